"""ctypes front end of the fp64 C oracle (oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product package.
Every function takes the same fp32 arrays the CUDA path receives and returns
float64 results; the arithmetic lives in oracle.c (see its header for the
PAPER.md passages each function follows).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

LINE2D, SLOPE2, SLOPE3 = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile oracle.c (plain C, -O2, no fast-math, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i, d = ctypes.c_int, ctypes.c_double
        L.ora_num_threads.restype = i
        L.ora_set_num_threads.argtypes = [i]
        L.ora_set_num_threads.restype = None
        L.ora_point.argtypes = [i, P, i, d, P, d, P, P, P]
        L.ora_grid.argtypes = [i, i, P, P, d, d, P, P, P, P, P]
        L.ora_peaks.argtypes = [P, i, i, P, d, i, P, P, P]
        L.ora_multistart.argtypes = [i, i, P, P, d, d, i, P, i, d, P, P, P, P, P]
        L.ora_merge.argtypes = [i, i, i, P, P, P, d, i, P, P, P, P, P, P]
        L.ora_estimate.argtypes = [P, i, i, P, P, P, P, P, P, i, P]
        L.ora_point_hess.argtypes = [i, P, i, d, P, d, P, P, P]
        L.ora_newton.argtypes = [i, i, P, P, d, i, P, i, P, P, d, i, P, P, P, P, P, P, P, P, P, i, d, ctypes.c_uint64]
        for f in (L.ora_point, L.ora_grid, L.ora_peaks, L.ora_multistart, L.ora_merge, L.ora_estimate,
                  L.ora_point_hess, L.ora_newton):
            f.restype = None
        _lib = L
    return _lib


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


def _f(v) -> float:
    """Reading Z18: scalars reach the GPU as fp32; the oracle uses that fp32 value promoted."""
    return float(np.float32(v))


def _P(model: int) -> int:
    return 3 if model == SLOPE3 else 2


def num_threads() -> int:
    return int(lib().ora_num_threads())


def set_num_threads(n: int) -> None:
    """OpenMP threads of the following oracle calls (timing only; results do not depend on it)."""
    lib().ora_set_num_threads(int(n))


def point(model: int, hits, theta, sigma: float, z_ref: float = 0.0):
    """Eq. (1) and its gradient at one theta: returns (R, grad[P], A[P])."""
    h = _f32(hits).reshape(-1, 4)
    th = np.ascontiguousarray(np.asarray(theta, np.float64))
    R = np.zeros(1)
    g = np.zeros(_P(model))
    A = np.zeros(_P(model))
    lib().ora_point(model, _p(h), len(h), _f(z_ref), _p(th), _f(sigma), _p(R), _p(g), _p(A))
    return float(R[0]), g, A


def grid(model: int, offsets, hits, nodes: Sequence[np.ndarray], sigma: float,
         z_ref: float = 0.0) -> np.ndarray:
    """Eq. (2): float64 [E, n0, n1] (P = 2) or [E, n2, n0, n1] (P = 3, z0 planes; reading Z37)."""
    off = np.ascontiguousarray(np.asarray(offsets, np.int32))
    h = _f32(hits).reshape(-1, 4)
    nd = [_f32(n) for n in nodes]
    P = _P(model)
    assert len(nd) == P
    alen = np.array([len(n) for n in nd], np.int32)
    E = len(off) - 1
    shape = tuple(alen) if P == 2 else (alen[2], alen[0], alen[1])
    out = np.zeros((E,) + shape, np.float64)
    lib().ora_grid(model, E, _p(off), _p(h), _f(z_ref), _f(sigma), _p(alen),
                   _p(nd[0]), _p(nd[1]), _p(nd[2]) if P == 3 else None, _p(out))
    return out


def peaks(grid_values: np.ndarray, P: int, threshold: float, capacity: int):
    """Reading Z6 peaks of a [E, d0, d1(, d2)] grid (any axis order: the rule is symmetric; a
    P = 3 response grid is [E, n2, n0, n1]): (index[E,cap], value[E,cap], count[E]), index =
    flat offset within the event's grid."""
    g = np.ascontiguousarray(np.asarray(grid_values, np.float64))
    E = g.shape[0]
    alen = np.array(g.shape[1:], np.int32)
    assert len(alen) == P
    idx = np.full((E, max(capacity, 1)), -1, np.int32)
    val = np.zeros((E, max(capacity, 1)), np.float64)
    cnt = np.zeros(E, np.int32)
    lib().ora_peaks(_p(g), E, P, _p(alen), _f(threshold), int(capacity), _p(idx), _p(val), _p(cnt))
    return idx[:, :capacity], val[:, :capacity], cnt


def multistart(model: int, offsets, hits, seeds, sigma: float, n_iters: int, step: float,
               box_lo, box_hi, z_ref: float = 0.0, want_grad: bool = True):
    """Algorithm 1 update loop (reading Z7): (theta[E,S,P], R[E,S], grad[E,S,P] or None)."""
    off = np.ascontiguousarray(np.asarray(offsets, np.int32))
    h = _f32(hits).reshape(-1, 4)
    sd = _f32(seeds)
    E, S, P = sd.shape
    assert P == _P(model) and E == len(off) - 1
    lo = np.ascontiguousarray(np.asarray(box_lo, np.float32).astype(np.float64))
    hi = np.ascontiguousarray(np.asarray(box_hi, np.float32).astype(np.float64))
    th = np.zeros((E, S, P))
    R = np.zeros((E, S))
    g = np.zeros((E, S, P)) if want_grad else None
    lib().ora_multistart(model, E, _p(off), _p(h), _f(z_ref), _f(sigma), S, _p(sd),
                         int(n_iters), _f(step), _p(lo), _p(hi), _p(th), _p(R), _p(g))
    return th, R, g


def merge(theta, R, radius, threshold: float, capacity: int, want_members: bool = False):
    """Algorithm 1 "cluster ... select highest response above R0" (readings Z9/Z10).
    Returns (track_theta[E,cap,P], track_R[E,cap], seed[E,cap], size[E,cap], count[E]), plus
    with want_members the leader ordinal each seed joined ([E,S], -1 below the threshold)."""
    th = np.ascontiguousarray(np.asarray(theta, np.float64))
    r = np.ascontiguousarray(np.asarray(R, np.float64))
    E, S, P = th.shape
    rad = np.ascontiguousarray(np.asarray(radius, np.float32).astype(np.float64))
    cap = max(capacity, 1)
    tt = np.zeros((E, cap, P))
    tr = np.zeros((E, cap))
    ts = np.full((E, cap), -1, np.int32)
    tz = np.zeros((E, cap), np.int32)
    tc = np.zeros(E, np.int32)
    mem = np.zeros((E, S), np.int32) if want_members else None
    lib().ora_merge(E, S, P, _p(th), _p(r), _p(rad), _f(threshold), int(capacity),
                    _p(tt), _p(tr), _p(ts), _p(tz), _p(tc), _p(mem))
    res = (tt[:, :capacity], tr[:, :capacity], ts[:, :capacity], tz[:, :capacity], tc)
    return res + ((mem,) if want_members else ())


def estimate(grid_values, nodes: Sequence[np.ndarray], peak_index, peak_count, capacity: int):
    """Step (iv) quadratic sub-cell estimate (reading Z21) on a response grid in the Z37 layout
    ([E, n0, n1] or [E, n2, n0, n1]); nodes in parameter order: float64 [E, capacity, P]."""
    g = np.ascontiguousarray(np.asarray(grid_values, np.float64))
    E = g.shape[0]
    P = g.ndim - 1
    nd = [_f32(n) for n in nodes]
    alen = np.array([len(n) for n in nd], np.int32)
    idx = np.ascontiguousarray(np.asarray(peak_index, np.int32))
    cnt = np.ascontiguousarray(np.asarray(peak_count, np.int32))
    out = np.zeros((E, max(capacity, 1), P))
    lib().ora_estimate(_p(g), E, P, _p(alen), _p(nd[0]), _p(nd[1]), _p(nd[2]) if P == 3 else None,
                       _p(idx), _p(cnt), int(capacity), _p(out))
    return out[:, :capacity]


def point_hess(model: int, hits, theta, sigma: float, z_ref: float = 0.0):
    """R, grad R and the Hessian (P x P) at one theta (chain rule through s^2; oracle.c)."""
    h = _f32(hits).reshape(-1, 4)
    th = np.ascontiguousarray(np.asarray(theta, np.float64))
    P = _P(model)
    R = np.zeros(1)
    g = np.zeros(P)
    H = np.zeros((P, P))
    lib().ora_point_hess(model, _p(h), len(h), _f(z_ref), _p(th), _f(sigma), _p(R), _p(g), _p(H))
    return float(R[0]), g, H


def newton(model: int, offsets, hits, seeds, sigmas, etas, final_sigma: float, max_halvings: int,
           box_lo, box_hi, z_ref: float = 0.0, want_grad: bool = True, want_margin: bool = False,
           want_evals: bool = False, flip=None, log_len: int = 0, perturb: float = 0.0, perturb_key: int = 0):
    """Algorithm 1 with Truncated-Newton updates and a sigma schedule (readings Z22-Z25).
    Returns (theta, R, grad), plus margin with want_margin, plus the per-seed response
    evaluation count (q + line-search trials + 1) with want_evals.  Test attribution only:
    `flip` ([E,S,log_len] bool) inverts the outcomes of the flagged numbered discrete decisions of
    each seed, and log_len > 0 appends each seed's per-decision margins ([E,S,log_len], -1 = unused);
    perturb > 0 multiplies every evaluated R, grad R and H entry by 1 + perturb u, u ~ U[-1, 1]
    keyed by perturb_key."""
    off = np.ascontiguousarray(np.asarray(offsets, np.int32))
    h = _f32(hits).reshape(-1, 4)
    sd = _f32(seeds)
    E, S, P = sd.shape
    sg = np.ascontiguousarray(np.asarray(sigmas, np.float32).astype(np.float64))
    et = np.ascontiguousarray(np.asarray(etas, np.float32).astype(np.float64))
    assert len(sg) == len(et)
    lo = np.ascontiguousarray(np.asarray(box_lo, np.float32).astype(np.float64))
    hi = np.ascontiguousarray(np.asarray(box_hi, np.float32).astype(np.float64))
    th = np.zeros((E, S, P))
    R = np.zeros((E, S))
    g = np.zeros((E, S, P)) if want_grad else None
    m = np.zeros((E, S)) if want_margin else None
    ne = np.zeros((E, S), np.int32) if want_evals else None
    assert flip is None or log_len > 0
    fl = None if flip is None else np.ascontiguousarray(np.broadcast_to(np.asarray(flip, np.uint8), (E, S, log_len)))
    lg = np.zeros((E, S, log_len)) if log_len > 0 else None
    lib().ora_newton(model, E, _p(off), _p(h), _f(z_ref), S, _p(sd), len(sg), _p(sg), _p(et), _f(final_sigma),
                     int(max_halvings), _p(lo), _p(hi), _p(th), _p(R), _p(g), _p(m), _p(ne), _p(fl), _p(lg),
                     int(log_len), float(perturb), int(perturb_key))
    res = (th, R, g) + ((m,) if want_margin else ()) + ((ne,) if want_evals else ()) + \
        ((lg,) if log_len > 0 else ())
    return res
