"""Comparators T1..T7 of DESIGN.md §5 (GPU result vs the fp64 oracle)."""
from __future__ import annotations

import math

import numpy as np

from oracle import oracle as ora

# T1 / T2 tolerance: north star "max relative error 1e-5 (fp32 vs fp64)"
REL = 1e-5
FLOOR = 1e-6


def t1_response(gpu, ref):
    """|R_gpu - R_ref| <= 1e-5 max(R_ref, 1e-6).  Returns (ok, worst ratio)."""
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    err = np.abs(gpu - ref) / (REL * np.maximum(ref, FLOOR))
    worst = float(err.max()) if err.size else 0.0
    return worst <= 1.0, worst


def grad_floor_scale(model, hits, sigma, theta):
    """G_i = (sqrt(2) e^-1/2 / sigma) max_k |ds_k/dtheta_i|: the largest possible
    single-hit gradient contribution (used as the T2 floor scale)."""
    h = np.asarray(hits, np.float64).reshape(-1, 4)
    c = math.sqrt(2.0) * math.exp(-0.5) / sigma
    if len(h) == 0:
        return np.zeros(len(theta))
    if model == ora.LINE2D:
        return c * np.array([np.abs(h[:, 0]).max(), 1.0])
    d = np.abs(h[:, 2] - (theta[2] if model == ora.SLOPE3 else 0.0))
    g = [d.max(), d.max()]
    if model == ora.SLOPE3:
        g.append(abs(theta[0]) + abs(theta[1]))
    return c * np.array(g)


def t2_gradient(gpu, ref, A, G):
    """|g_gpu - g_ref| <= 1e-5 max(A_i, 1e-6 G_i) per component."""
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    scale = REL * np.maximum(A, FLOOR * G)
    scale = np.where(scale > 0, scale, 1e-300)
    err = np.abs(gpu - ref) / scale
    worst = float(err.max()) if err.size else 0.0
    return worst <= 1.0, worst


def near_tie_cells(grid64, P, threshold):
    """T4 exemption: cells with some existing neighbour within 2e-5 relative, or within
    1e-5 relative of the threshold, in the ORACLE grid.  Returns a boolean mask."""
    g = np.asarray(grid64, np.float64)
    tie = np.abs(g - threshold) <= 1e-5 * max(abs(threshold), FLOOR)
    shape = g.shape
    for off in np.ndindex(*(3,) * P):
        d = tuple(o - 1 for o in off)
        if all(x == 0 for x in d):
            continue
        src = tuple(slice(max(0, -x), shape[i] - max(0, x)) for i, x in enumerate(d))
        dst = tuple(slice(max(0, x), shape[i] - max(0, -x)) for i, x in enumerate(d))
        a, b = g[dst], g[src]
        close = np.abs(a - b) <= 2e-5 * np.maximum(np.maximum(a, b), FLOOR)
        tie[dst] |= close
    return tie


def t4_peak_sets(idx_gpu, cnt_gpu, grid64, P, threshold, capacity):
    """Symmetric difference of GPU peaks (from the fp32 grid) and oracle peaks (from the
    fp64 grid) is empty except near-tie cells.  Returns (ok, n_diff, n_excused)."""
    ref_idx, _, ref_cnt = ora.peaks(grid64[None], P, threshold, capacity)
    a = set(int(v) for v in idx_gpu[:min(int(cnt_gpu), capacity)])
    b = set(int(v) for v in ref_idx[0, :min(int(ref_cnt[0]), capacity)])
    diff = a ^ b
    if not diff:
        return True, 0, 0
    tie = near_tie_cells(grid64, P, threshold).ravel()
    bad = [c for c in diff if not tie[c]]
    return len(bad) == 0, len(diff), len(diff) - len(bad)


def sensitive_seeds(model, offsets, hits, seeds, sigma, n_iters, step, lo, hi, ref_theta, ranges,
                    which):
    """T5 exemption: seed (e, s) is sensitive when the oracle re-run from theta^0 nudged by
    +-1 fp32 ulp per axis ends more than 1e-4 x range away from the unperturbed run."""
    out = np.zeros(len(which), bool)
    for k, (e, s) in enumerate(which):
        off = [0, int(offsets[e + 1] - offsets[e])]
        h = hits[offsets[e]:offsets[e + 1]]
        base = seeds[e, s].astype(np.float32)
        for sign in (+1, -1):
            nudged = np.nextafter(base, np.float32(sign * np.inf)).astype(np.float32)
            th, _, _ = ora.multistart(model, off, h, nudged[None, None], sigma, n_iters, step, lo, hi,
                                      want_grad=False)
            if np.any(np.abs(th[0, 0] - ref_theta[e, s]) > 1e-4 * np.asarray(ranges)):
                out[k] = True
    return out
