#!/usr/bin/env python
"""Small invocation of every kernel (direct, separable and default tensor-core grids, all models,
resident and streaming hit stages, both peak paths, estimates, multi-start with/without grad, merge,
Truncated Newton) for compute-sanitizer runs."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import configs as C  # noqa: E402
from synth import events as G  # noqa: E402
import paper_1709_08610_b200 as R  # noqa: E402
from paper_1709_08610_b200 import retina as RT  # noqa: E402

for name, n_ev in (("cfg0", 1), ("cfg2", 3), ("cfg4", 1)):
    cfg = C.CONFIGS[name]
    b = G.make_batch(cfg, range(n_ev))
    for hint in (None, 0):  # resident vs streaming hit stage (default cap 2048 / 4096)
        ev = R.Events.from_numpy(b.offsets, b.hits, max_event_hits=hint)
        if cfg.axes:
            axes = [a for a in cfg.axes]
            if name == "cfg4":
                axes = [(-0.3, 0.3, 40), (-0.3, 0.3, 33), (-150.0, 150.0, 37)]
            nodes = [torch.linspace(lo, hi, n, device="cuda") for lo, hi, n in axes]
            for algo in (RT.GRID_DIRECT, RT.GRID_SEPARABLE, RT.GRID_AUTO):
                if algo != RT.GRID_DIRECT and cfg.model == C.LINE2D:
                    continue
                g = R.retina_grid_response(ev, cfg.model, cfg.sigma, nodes, algorithm=algo)
                idx, val, cnt = R.retina_find_peaks(g, cfg.P, 0.0, 64)
                ws = torch.empty((RT.find_peaks_workspace_size(n_ev, g.shape[1:]) // 4 + 1,), dtype=torch.int32,
                                 device="cuda")
                R.retina_find_peaks(g, cfg.P, 0.0, 64, workspace=ws)
                R.retina_estimate_peaks(g, nodes, idx, cnt)
        n_seeds = 300
        seeds = torch.from_numpy(G.make_seeds(cfg, range(n_ev), n_seeds=n_seeds)).cuda()
        lo, hi = (cfg.box_lo, cfg.box_hi) if cfg.box_lo else ((-1,) * cfg.P, (1,) * cfg.P)
        for want_grad in (True, False):
            th, Rr, _ = R.retina_multistart_optimize(ev, cfg.model, cfg.sigma, seeds, 3, cfg.step, lo, hi,
                                                     want_grad=want_grad)
        rad = cfg.merge_radius or (1e-3,) * cfg.P
        R.retina_merge_tracks(th, Rr, rad, 0.0, 16)
        if cfg.model != C.LINE2D:
            sig, eta, fsig, mh = C.newton_schedule(cfg)
            R.retina_multistart_newton_ex(ev, cfg.model, seeds, sig, eta, fsig, mh, lo, hi)
torch.cuda.synchronize()
print("sanitize case ok")
