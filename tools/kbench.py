#!/usr/bin/env python
"""Time single hot-path phases of one library build (RETINA_LIB may point at a variant build).

    RETINA_LIB=/path/lib.so python tools/kbench.py --config cfg4 --events 200 --phases grid,peaks,ms,newton

Prints one JSON line per phase: median / min of --reps CUDA-event timings (after one warm-up),
the algorithmic work and the fraction of the bound the phase is measured against.
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import configs as C  # noqa: E402
from synth import events as G  # noqa: E402
import paper_1709_08610_b200 as R  # noqa: E402
from paper_1709_08610_b200 import retina as RT  # noqa: E402

MUFU = 148 * 16 * 1.965e9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--events", type=int, default=1000)
    ap.add_argument("--seeds", type=int, default=None)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--algo", type=int, default=0)
    ap.add_argument("--dense", action="store_true")
    ap.add_argument("--phases", default="grid,peaks,ms")
    ap.add_argument("--tag", default="")
    ap.add_argument("--peaks-ws", action="store_true", help="peaks: always the many-CTA workspace path")
    a = ap.parse_args()
    cfg = C.get_config(a.config, dense=True) if a.dense else C.get_config(a.config)
    if a.seeds:
        cfg = cfg.replace(n_seeds=a.seeds)
    ev_ids = range(a.events)
    b = G.make_batch(cfg, ev_ids)
    ev = R.Events.from_numpy(b.offsets, b.hits)
    nh = float(b.n_hits)
    phases = a.phases.split(",")
    out = []

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
        return statistics.median(t), min(t)

    def emit(phase, med, mn, **kw):
        d = {"tag": a.tag, "lib": os.environ.get("RETINA_LIB", RT.LIB), "config": cfg.name, "dense": a.dense,
             "events": a.events, "phase": phase, "ms_median": med, "ms_min": mn, **kw}
        out.append(d)
        print(json.dumps(d), flush=True)

    if cfg.axes and ({"grid", "peaks"} & set(phases)):
        nodes = [torch.from_numpy(n).cuda() for n in G.axis_nodes(cfg)]
        shape = RT.grid_shape(1, [len(n) for n in nodes])[1:]
        chunk = max(1, min(a.events, int(4e9 // (4 * cfg.n_units))))
        grid = torch.empty((chunk,) + shape, device="cuda")
        cap = cfg.peak_capacity
        pk = (torch.empty((chunk, cap), dtype=torch.int32, device="cuda"),
              torch.empty((chunk, cap), device="cuda"), torch.empty((chunk,), dtype=torch.int32, device="cuda"))
        ws = None
        if chunk < 2 * 148 or a.peaks_ws:
            ws = torch.empty((RT.find_peaks_workspace_size(chunk, shape) // 4 + 1,), dtype=torch.int32, device="cuda")
        maxh = int(np.diff(b.offsets).max())
        if "grid" in phases:
            def run_grid():
                for e0 in range(0, a.events, chunk):
                    e1 = min(a.events, e0 + chunk)
                    sub = R.Events(ev.offsets[e0:e1 + 1], ev.hits, 0.0, maxh)
                    R.retina_grid_response(sub, cfg.model, cfg.sigma, nodes, out=grid[:e1 - e0], algorithm=a.algo)
            med, mn = timeit(run_grid)
            pairs = nh * cfg.n_units
            emit("grid", med, mn, pairs=pairs, tflops_fp32acc=2 * pairs / (med * 1e-3) / 1e12,
                 frac_f16_acc=2 * pairs / (med * 1e-3) / (1673.1e12 / 3))
        if "peaks" in phases:
            # the peak scan reads a filled grid chunk (values from the grid kernel)
            sub = R.Events(ev.offsets[0:chunk + 1], ev.hits, 0.0, maxh)
            R.retina_grid_response(sub, cfg.model, cfg.sigma, nodes, out=grid[:chunk])
            n_chunks = (a.events + chunk - 1) // chunk

            def run_peaks():
                for _ in range(n_chunks):
                    R.retina_find_peaks(grid, cfg.P, cfg.peak_threshold, cap, out=pk, workspace=ws)
            med, mn = timeit(run_peaks)
            byts = 4.0 * cfg.n_units * chunk * n_chunks
            emit("peaks", med, mn, grid_bytes=byts, gbs=byts / (med * 1e-3) / 1e9, frac_hbm=byts / (med * 1e-3) / 6550.7e9)
    if "ms" in phases or "newton" in phases or "culled" in phases or "newton_culled" in phases:
        seeds = torch.from_numpy(G.make_seeds(cfg, ev_ids)).cuda()
        th = torch.empty_like(seeds)
        Rr = torch.empty(seeds.shape[:2], device="cuda")
        if "ms" in phases:
            def run_ms():
                R.retina_multistart_optimize(ev, cfg.model, cfg.sigma, seeds, cfg.n_iters, cfg.step, cfg.box_lo,
                                             cfg.box_hi, want_grad=False, out=(th, Rr, None))
            med, mn = timeit(run_ms)
            pairs = nh * cfg.n_seeds * (cfg.n_iters + 1)
            emit("ms", med, mn, pairs=pairs, frac_mufu=pairs / (med * 1e-3) / MUFU)
        if "culled" in phases:  # K4c: same results, only the pairs that can contribute
            ws = torch.empty((RT.multistart_workspace_size(len(ev_ids), cfg.n_seeds) // 4 + 1,), dtype=torch.int32,
                             device="cuda")
            pc = torch.zeros(1, dtype=torch.int64, device="cuda")

            def run_mc():
                R.retina_multistart_optimize(ev, cfg.model, cfg.sigma, seeds, cfg.n_iters, cfg.step, cfg.box_lo,
                                             cfg.box_hi, want_grad=False, out=(th, Rr, None),
                                             algorithm=RT.MS_CULLED, workspace=ws, pairs_evaluated=pc)
            med, mn = timeit(run_mc)
            pc.zero_()
            run_mc()
            torch.cuda.synchronize()
            pairs = nh * cfg.n_seeds * (cfg.n_iters + 1)
            ev_pairs = float(pc.item())
            emit("culled", med, mn, pairs=pairs, pairs_evaluated=ev_pairs, evaluated_frac=ev_pairs / pairs,
                 frac_mufu_evaluated=ev_pairs / (med * 1e-3) / MUFU, events_per_s=len(ev_ids) / (med * 1e-3))
        if "newton" in phases:
            sig, eta, fsig, mh = C.newton_schedule(cfg)
            ne = torch.empty(seeds.shape[:2], dtype=torch.int32, device="cuda")

            def run_nt():
                R.retina_multistart_newton_ex(ev, cfg.model, seeds, sig, eta, fsig, mh, cfg.box_lo, cfg.box_hi,
                                              want_grad=False, out=(th, Rr, None, ne))
            med, mn = timeit(run_nt)
            nev = ne.to(torch.float64).sum(dim=1).cpu().numpy()
            pairs = float((np.diff(b.offsets).astype(np.float64) * nev).sum())
            emit("newton", med, mn, pairs=pairs, frac_mufu=pairs / (med * 1e-3) / MUFU,
                 evals_per_seed=float(nev.sum() / ne.numel()))
        if "newton_culled" in phases:  # K6c: the same results, only the pairs that can contribute
            sig, eta, fsig, mh = C.newton_schedule(cfg)
            ne = torch.empty(seeds.shape[:2], dtype=torch.int32, device="cuda")
            ws = torch.empty((RT.multistart_workspace_size(len(ev_ids), cfg.n_seeds) // 4 + 1,), dtype=torch.int32,
                             device="cuda")
            pc = torch.zeros(1, dtype=torch.int64, device="cuda")

            def run_ntc():
                R.retina_multistart_newton_ex(ev, cfg.model, seeds, sig, eta, fsig, mh, cfg.box_lo, cfg.box_hi,
                                              want_grad=False, out=(th, Rr, None, ne), algorithm=RT.MS_CULLED,
                                              workspace=ws, pairs_evaluated=pc)
            med, mn = timeit(run_ntc)
            pc.zero_()
            run_ntc()
            torch.cuda.synchronize()
            nev = ne.to(torch.float64).sum(dim=1).cpu().numpy()
            pairs = float((np.diff(b.offsets).astype(np.float64) * nev).sum())
            ev_pairs = float(pc.item())
            emit("newton_culled", med, mn, pairs=pairs, pairs_evaluated=ev_pairs, evaluated_frac=ev_pairs / pairs,
                 frac_mufu_evaluated=ev_pairs / (med * 1e-3) / MUFU, events_per_s=len(ev_ids) / (med * 1e-3))


if __name__ == "__main__":
    main()
