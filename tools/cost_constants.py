#!/usr/bin/env python
"""Measure the paper's cost constants on B200:
C  = time(R + grad R + Hessian) / time(R)   (paper: "around 3", constant C = 3)
C0 = time of one Truncated-Newton step (incl. line search) / time(R)   (paper: C0 ~ 30)
on a cfg3 (or other) event subset, per (seed, hit) pass, with the kernels of libretina.so.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import configs as C  # noqa: E402
from synth import events as G  # noqa: E402
import paper_1709_08610_b200 as R  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--events", type=int, default=500)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
cfg = C.get_config(a.config)
ids = range(a.events)
b = G.make_batch(cfg, ids)
seeds = torch.from_numpy(G.make_seeds(cfg, ids)).cuda()
ev = R.Events.from_numpy(b.offsets, b.hits)
out = (torch.empty_like(seeds), torch.empty(seeds.shape[:2], device="cuda"), None)
sig, eta, fsig, mh = C.newton_schedule(cfg)


def t(fn):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def ms(n_iters, grad=False):
    return lambda: R.retina_multistart_optimize(ev, cfg.model, cfg.sigma, seeds, n_iters, cfg.step, cfg.box_lo,
                                                cfg.box_hi, want_grad=grad, out=out if not grad else None)


def nt(steps, halvings):
    return lambda: R.retina_multistart_newton(ev, cfg.model, seeds, sig[:steps] if steps <= 3 else sig * 2,
                                              eta[:steps] if steps <= 3 else eta * 2, fsig, halvings, cfg.box_lo,
                                              cfg.box_hi, want_grad=False, out=out)


T_R = t(ms(0))                    # 1 R-only pass
T_10 = t(ms(10))                  # 10 gradient passes + 1 R pass
T_grad = (T_10 - T_R) / 10
T_n1 = t(nt(1, 0))                # 1 Hessian pass + 1 trial (R) + final R
T_hess = T_n1 - 2 * T_R
T_q = t(nt(3, mh))                # the paper's q = 3 steps with backtracking + final R
C0 = (T_q - T_R) / 3 / T_R
res = {"config": a.config, "events": a.events, "seeds": cfg.n_seeds, "T_R_ms": T_R, "T_grad_pass_ms": T_grad,
       "T_hess_pass_ms": T_hess, "C_grad": T_grad / T_R, "C_hess": T_hess / T_R, "C0_newton_step": C0,
       "newton_q3_ms": T_q, "gradient_50_ms_equiv": T_grad * 50 + T_R,
       "paper": {"C": 3, "C0": 30}}
print(json.dumps(res))
