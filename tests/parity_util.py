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


# --------------------------------------------------------------------------- excused-fraction bookkeeping
def report(test: str, **stats):
    """One machine-readable line per comparator run (pytest -s | grep PARITY-STATS): how many
    items each named oracle-side rule excused, so the excused fractions are logged and bounded."""
    import json
    print("PARITY-STATS " + json.dumps({"test": test, **stats}, default=float), flush=True)


def t5_states(model, offsets, hits, seeds, sigma, n_iters, step, lo, hi, th_gpu, th_ref, ranges):
    """T5: every seed ends within 1e-3 x range of the oracle's end point unless it is
    sensitive (the only excuse).  Returns (unexcused list, stats dict, sensitive-cache)."""
    dev_rel = np.max(np.abs(np.asarray(th_gpu, np.float64) - th_ref) / ranges, axis=2)
    bad = [tuple(x) for x in np.argwhere(dev_rel > 1e-3)]
    sens = sensitive_seeds(model, offsets, hits, seeds, sigma, n_iters, step, lo, hi, th_ref, ranges, bad) \
        if bad else np.zeros(0, bool)
    cache = {k: bool(v) for k, v in zip(bad, sens)}
    unexcused = [k for k, v in cache.items() if not v]
    n = dev_rel.size
    return unexcused, {"seeds": n, "off_gt_1e-3": len(bad), "excused_sensitive": int(sens.sum()),
                       "excused_frac": float(sens.sum()) / max(n, 1),
                       "max_dev_nonexcused": float(dev_rel[dev_rel <= 1e-3].max()) if n else 0.0}, cache


def _match_one_to_one(A, B, ranges, tol=1e-3):
    """Greedy one-to-one matching of two track lists by ascending normalised Chebyshev distance
    (each track used at most once).  Returns (unmatched A indices, unmatched B indices)."""
    if len(A) == 0 or len(B) == 0:
        return list(range(len(A))), list(range(len(B)))
    d = np.max(np.abs(A[:, None, :] - B[None, :, :]) / ranges, axis=2)
    ia, ib = np.nonzero(d <= tol)
    order = np.argsort(d[ia, ib], kind="stable")
    ua, ub = np.ones(len(A), bool), np.ones(len(B), bool)
    for k in order:
        a, b = ia[k], ib[k]
        if ua[a] and ub[b]:
            ua[a] = ub[b] = False
    return list(np.nonzero(ua)[0]), list(np.nonzero(ub)[0])


def t6_tracks(side_gpu, side_ref, ranges, radius, R0, sensitive):
    """T6: merged tracks of the GPU pipeline and the oracle pipeline match one
    to one within 1e-3 x range per axis.  Each side is (theta[S,P] f64, R[S], leader seeds in
    creation order, member ordinal per seed).  An unmatched track is excused only by an
    oracle-side rule, named in the returned counts:
      near_R0     its leader's R is within 1e-5 relative of R0;
      near_radius its closest leader-to-leader distance on its own side is within 1e-5 x range
                  of the merge radius (the binding axis of the Chebyshev box);
      sensitive   every member seed is sensitive (T5 nudge rule; `sensitive(s)` decides).
    Returns (list of unexcused (side, leader seed), counts dict)."""
    ranges = np.asarray(ranges, np.float64)
    radius = np.asarray(radius, np.float64)
    lead = [np.asarray(s[2], np.int64) for s in (side_gpu, side_ref)]
    pos = [np.asarray(s[0], np.float64)[l] for s, l in zip((side_gpu, side_ref), lead)]
    un = _match_one_to_one(pos[0], pos[1], ranges)
    counts = {"tracks_gpu": len(lead[0]), "tracks_ref": len(lead[1]), "unmatched": len(un[0]) + len(un[1]),
              "near_R0": 0, "near_radius": 0, "sensitive": 0}
    bad = []
    for side, (th, R, _, mem) in enumerate((side_gpu, side_ref)):
        th = np.asarray(th, np.float64)
        for j in un[side]:
            L = int(lead[side][j])
            if abs(float(R[L]) - R0) <= 1e-5 * R0:
                counts["near_R0"] += 1
                continue
            others = np.delete(pos[side], j, axis=0)
            if len(others):
                excess = np.max((np.abs(others - th[L]) - radius) / ranges, axis=1)
                if np.min(np.abs(excess)) <= 1e-5:
                    counts["near_radius"] += 1
                    continue
            members = np.nonzero(np.asarray(mem) == j)[0]
            if len(members) and all(sensitive(int(s)) for s in members):
                counts["sensitive"] += 1
                continue
            bad.append(("gpu" if side == 0 else "ref", L))
    return bad, counts


def newton_sensitive(model, lo, hi, h, seed, end, ranges, sig, eta, fsig, mh, evals=None, z_ref=0.0):
    """T5n sensitivity (oracle-side): the oracle run perturbed at fp32 resolution -- from the seed
    nudged by +-1 ulp on every axis, or by 4 random-sign draws of 1e-7 x range per axis, or (the
    arithmetic form) from the seed itself with every evaluated R, grad R and H entry scaled by
    1 + 1e-6 u (u ~ U[-1, 1]; 4 keys; 1e-6 is the GPU's measured relative error, T1 ratios
    0.2-0.5 of 1e-5) -- ends more than 1e-4 x range from its unperturbed end point (or, with
    `evals`, spends another number of response evaluations).  fp32 arithmetic perturbs the GPU
    trajectory by that much, so such a seed may legitimately end elsewhere."""
    seed = np.asarray(seed, np.float32)
    ranges = np.asarray(ranges, np.float64)
    rng = np.random.default_rng(int(seed.view(np.uint32).sum()))
    trials = [np.nextafter(seed, np.float32(sgn * np.inf)).astype(np.float32) for sgn in (+1, -1)]
    trials += [(seed.astype(np.float64) + rng.choice([-1.0, 1.0], len(ranges)) * 1e-7 * ranges).astype(np.float32)
               for _ in range(4)]
    runs = [(t, 0.0, 0) for t in trials] + [(seed, 1e-6, key) for key in (1, 2, 3, 4)]
    for t, eps, key in runs:
        # want_grad=True: counts include the final pass, as in the GPU runs the tests compare
        t2, _, _, n2 = ora.newton(model, [0, len(h)], h, t[None, None], sig, eta, fsig, mh, lo, hi, z_ref=z_ref,
                                  want_grad=True, want_evals=True, perturb=eps, perturb_key=key)
        if np.any(np.abs(t2[0, 0] - end) > 1e-4 * ranges) or (evals is not None and n2[0, 0] != evals):
            return True
    return False


def newton_flip_explains(model, lo, hi, h, seeds, th_gpu, evals_gpu, ranges, sig, eta, fsig, mh, z_ref=0.0,
                         max_margin=1e-4, max_runs=256, max_flips=24):
    """T5n attribution rule "near-tie flips" (oracle-side).  A discrete decision of the Newton
    path (Armijo accept, CG curvature sign) whose relative margin in the oracle run is <= 1e-4
    is inside what fp32 R and fp32 H can move (T1 is 1e-5), so either outcome is a correct
    execution of the algorithm.  The rule searches (depth first, decisions in the order taken,
    at most `max_flips` flips and `max_runs` oracle runs per seed) for a set of such near-tie
    decisions whose inverted outcomes make the oracle reproduce the GPU's end point within
    1e-3 x range (and, when given, its evaluation count).  Every decision flipped is a near-tie
    of the oracle run it occurs in.  Returns (bool array, number of flips used or -1)."""
    seeds = np.ascontiguousarray(np.asarray(seeds, np.float32))
    n = len(seeds)
    ranges = np.asarray(ranges, np.float64)
    found = np.full(n, -1)
    if n == 0:
        return found >= 0, found
    off = [0, len(h)]
    LOG = 128
    # per seed: DFS stack of flip sets (sorted tuples); each popped state is one oracle run
    stacks = [[()] for _ in range(n)]
    runs = np.zeros(n, int)
    while True:
        rows = [i for i in range(n) if found[i] < 0 and stacks[i] and runs[i] < max_runs]
        if not rows:
            break
        states = [stacks[i].pop() for i in rows]
        fl = np.zeros((1, len(rows), LOG), np.uint8)
        for j, st in enumerate(states):
            fl[0, j, list(st)] = 1
        t2, _, _, _, n2, log = ora.newton(model, off, h, seeds[rows][None], sig, eta, fsig, mh, lo, hi, z_ref=z_ref,
                                          want_grad=True, want_margin=True, want_evals=True, flip=fl, log_len=LOG)
        for j, i in enumerate(rows):
            runs[i] += 1
            ok = np.all(np.abs(t2[0, j] - th_gpu[i]) <= 1e-3 * ranges)
            if evals_gpu is not None:
                ok = ok and int(n2[0, j]) == int(evals_gpu[i])
            if ok:
                found[i] = len(states[j])
                continue
            st = states[j]
            if len(st) >= max_flips:
                continue
            m = log[0, j]
            last = st[-1] if st else -1
            nxt = [k for k in range(last + 1, LOG) if 0 <= m[k] <= max_margin]
            # push in reverse so the earliest near-tie decision is explored first
            for k in reversed(nxt):
                stacks[i].append(st + (k,))
    return found >= 0, found


def t5n_states(model, lo, hi, batch, seeds, sig, eta, fsig, mh, th_gpu, th_ref, ranges,
               evals_gpu=None, evals_ref=None, z_ref=0.0, R_ref=None, R0=None):
    """T5n: Newton end states within 1e-3 x range, and (when given) per-seed
    evaluation counts identical, for every seed not explained by a named oracle-side rule:
      flip       inverting ONE of the seed's near-tie decisions (Armijo accept or CG curvature
                 sign with relative margin <= 1e-4 in the oracle run) makes the oracle reproduce
                 the GPU's end point (and count): newton_flip_explains();
      sensitive  newton_sensitive() (the oracle end point or count moves under fp32-size nudges).
    Returns (unexcused list, stats dict, excused set of (e, s))."""
    th_gpu = np.asarray(th_gpu, np.float64)
    dev_rel = np.max(np.abs(th_gpu - th_ref) / ranges, axis=2)
    bad = dev_rel > 1e-3
    mism = np.zeros_like(bad) if evals_gpu is None else (np.asarray(evals_gpu) != np.asarray(evals_ref))
    unexcused, excused = [], set()
    n_flip = n_sens = 0
    flip_counts = []
    for e in range(bad.shape[0]):
        rows = np.nonzero(bad[e] | mism[e])[0]
        if len(rows) == 0:
            continue
        h = batch.event_hits(e)
        ok, mexp = newton_flip_explains(model, lo, hi, h, seeds[e, rows], th_gpu[e, rows],
                                        None if evals_gpu is None else np.asarray(evals_gpu)[e, rows], ranges,
                                        sig, eta, fsig, mh, z_ref=z_ref)
        for j, s in enumerate(rows):
            if ok[j]:
                n_flip += 1
                flip_counts.append(int(mexp[j]))
                excused.add((e, int(s)))
                continue
            ev = None if not mism[e, s] else int(evals_ref[e, s])
            if newton_sensitive(model, lo, hi, h, seeds[e, s], th_ref[e, s], ranges, sig, eta, fsig, mh,
                                evals=ev, z_ref=z_ref):
                n_sens += 1
                excused.add((e, int(s)))
            else:
                unexcused.append((e, int(s)))
    n = bad.size
    st = {"seeds": n, "off_gt_1e-3": int(bad.sum()), "evals_mismatch": int(mism.sum()),
          "excused_flip": n_flip, "excused_sensitive": n_sens,
          "excused_frac": (n_flip + n_sens) / max(n, 1),
          "flips_per_excused_seed_max": max(flip_counts) if flip_counts else None,
          "max_dev_nonexcused": float(dev_rel[~bad].max()) if (~bad).any() else 0.0}
    if R_ref is not None and R0 is not None:
        # how many of the far (excused) seeds end as track candidates (oracle R >= R0)
        st["far_seeds_with_R_ge_R0"] = int((bad & (np.asarray(R_ref) >= R0)).sum())
        st["seeds_with_R_ge_R0"] = int((np.asarray(R_ref) >= R0).sum())
    return unexcused, st, excused
