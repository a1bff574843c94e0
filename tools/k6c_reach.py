#!/usr/bin/env python
"""Share of an event's hits a K6c warp keeps in reach at each Truncated-Newton step, for several
ways of grouping the seeds into warps (a design probe for the culled Newton kernel, not a test).

    python tools/k6c_reach.py --config cfg3 --events 8

The trajectories come from the library (theta after 0, 1, .. q-1 steps = the kernel run with that
prefix of the sigma schedule); the box bound is the one of cull.cuh (K s^2 <= 128 kept), in fp64.
Groupings: 'morton' = 32 S consecutive seeds of the per-event Morton order of the SEEDS (K6c);
'cta_resort' = each CTA's 512 such seeds re-ordered by Morton code of their CURRENT theta, then
split into warps; 'event_resort' = the event's seeds re-ordered by current theta (upper bound).
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import configs as C  # noqa: E402
from synth import events as G  # noqa: E402
import paper_1709_08610_b200 as R  # noqa: E402
from paper_1709_08610_b200 import retina as RT  # noqa: E402

LOG2E = 1.4426950408889634


def morton(th, lo, hi, bits):
    q = np.clip((th - lo) / np.maximum(hi - lo, 1e-30) * ((1 << bits) - 1), 0, (1 << bits) - 1).astype(np.uint64)
    m = np.zeros(th.shape[0], np.uint64)
    P = th.shape[1]
    for b in range(bits):
        for d in range(P):
            m |= ((q[:, d] >> np.uint64(b)) & np.uint64(1)) << np.uint64(P * b + d)
    return m


def kept_share(hits, groups, K, P):
    """mean over groups of the share of hits within reach of the group's box"""
    x, y, z = hits[:, 0].astype(np.float64), hits[:, 1].astype(np.float64), hits[:, 2].astype(np.float64)
    out = []
    for g in groups:
        lo, hi = g.min(axis=0).astype(np.float64), g.max(axis=0).astype(np.float64)
        if P == 3:
            d0, d1 = z - hi[2], z - lo[2]
        else:
            d0 = d1 = z

        def min_abs(v, t0, t1):
            p = np.stack([t0 * d0, t0 * d1, t1 * d0, t1 * d1])
            pmin, pmax = p.min(axis=0), p.max(axis=0)
            a, b = v - pmax, v - pmin
            return np.where(a > 0, a, np.where(b < 0, -b, 0.0))
        mx, my = min_abs(x, lo[0], hi[0]), min_abs(y, lo[1], hi[1])
        out.append(float(np.mean(K * (mx * mx + my * my) <= 128.0)))
    return float(np.mean(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--events", type=int, default=8)
    a = ap.parse_args()
    cfg = C.get_config(a.config)
    ids = list(range(a.events))
    b = G.make_batch(cfg, ids)
    seeds_np = G.make_seeds(cfg, ids)
    seeds = torch.from_numpy(seeds_np).cuda()
    ev = R.Events.from_numpy(b.offsets, b.hits)
    sig, eta, fsig, mh = C.newton_schedule(cfg)
    P, S = cfg.P, cfg.n_seeds
    warp = 32 * (4 if P == 2 else 4)
    lo, hi = np.asarray(cfg.box_lo), np.asarray(cfg.box_hi)
    bits = 16 if P == 2 else 10
    thetas = [seeds_np]
    for j in range(1, len(sig)):
        th, _, _, _ = R.retina_multistart_newton_ex(ev, cfg.model, seeds, sig[:j], eta[:j], sig[j - 1], mh, cfg.box_lo,
                                                    cfg.box_hi, want_grad=False)
        torch.cuda.synchronize()
        thetas.append(th.cpu().numpy())
    res = {}
    for j, s_j in enumerate(sig):
        K = LOG2E / (s_j * s_j)
        acc = {"morton": [], "cta_resort": [], "event_resort": [], "morton_64": []}
        for e in range(a.events):
            hits = b.event_hits(e)
            order0 = np.argsort(morton(seeds_np[e].astype(np.float64), lo, hi, bits), kind="stable")
            th = thetas[j][e].astype(np.float64)
            acc["morton"].append(kept_share(hits, [th[order0[i:i + warp]] for i in range(0, S, warp)], K, P))
            acc["morton_64"].append(kept_share(hits, [th[order0[i:i + 64]] for i in range(0, S, 64)], K, P))
            gs = []
            for c in range(0, S, 512):
                idx = order0[c:c + 512]
                o = idx[np.argsort(morton(th[idx], lo, hi, bits), kind="stable")]
                gs += [th[o[i:i + warp]] for i in range(0, len(o), warp)]
            acc["cta_resort"].append(kept_share(hits, gs, K, P))
            o = np.argsort(morton(th, lo, hi, bits), kind="stable")
            acc["event_resort"].append(kept_share(hits, [th[o[i:i + warp]] for i in range(0, S, warp)], K, P))
        res[f"step{j + 1} (sigma x {s_j / cfg.sigma:.2f})"] = {k: round(float(np.mean(v)), 4) for k, v in acc.items()}
    print(json.dumps({"config": cfg.name, "events": a.events, "kept_share": res}, indent=1))


if __name__ == "__main__":
    main()
