#!/usr/bin/env python
"""Time the hot-path kernels of one library build (RETINA_LIB) on a cfg subset.

    RETINA_LIB=/path/lib.so python tools/variant_bench.py [--config cfg3] [--events 1000]
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

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--events", type=int, default=1000)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--algo", type=int, default=0)
a = ap.parse_args()
cfg = C.get_config(a.config)
ev_ids = range(a.events)
b = G.make_batch(cfg, ev_ids)
seeds = torch.from_numpy(G.make_seeds(cfg, ev_ids)).cuda()
ev = R.Events.from_numpy(b.offsets, b.hits)
nodes = [torch.from_numpy(n).cuda() for n in G.axis_nodes(cfg)]
chunk = max(1, min(a.events, int(2e9 // (4 * cfg.n_units))))
grid = torch.empty(R.retina.grid_shape(chunk, [len(n) for n in nodes]), device="cuda")
out = (torch.empty_like(seeds), torch.empty(seeds.shape[:2], device="cuda"), None)
nh = float(b.n_hits)


def timeit(fn):
    fn()
    torch.cuda.synchronize()
    t = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        t.append(e0.elapsed_time(e1))
    return min(t)


def run_grid():
    for e0 in range(0, a.events, chunk):
        e1 = min(a.events, e0 + chunk)
        sub = R.Events(ev.offsets[e0:e1 + 1], ev.hits, 0.0, int(np.diff(b.offsets).max()))
        R.retina_grid_response(sub, cfg.model, cfg.sigma, nodes, out=grid[:e1 - e0], algorithm=a.algo)


def run_ms():
    R.retina_multistart_optimize(ev, cfg.model, cfg.sigma, seeds, cfg.n_iters, cfg.step, cfg.box_lo, cfg.box_hi,
                                 want_grad=False, out=out)


tg = timeit(run_grid)
tm = timeit(run_ms)
res = {"lib": os.environ.get("RETINA_LIB", RT.LIB), "config": a.config, "events": a.events,
       "grid_ms": tg, "grid_pairs_per_s": nh * cfg.n_units / (tg * 1e-3),
       "ms_ms": tm, "ms_pairs_per_s": nh * cfg.n_seeds * (cfg.n_iters + 1) / (tm * 1e-3)}
res["ms_frac_mufu"] = res["ms_pairs_per_s"] / 4.6531e12
res["grid_frac_fma"] = res["grid_pairs_per_s"] / 3.7225e13
print(json.dumps(res))
