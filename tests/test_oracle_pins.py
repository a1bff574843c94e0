"""Pins of the fp64 oracle against what the paper and mathematics fix (CPU only).

Each test names the pin id of DESIGN.md §5 (P1..P13) and the passage it
follows.  None of them re-types oracle.c's formula: they use closed forms,
invariants, special cases, independent numerical differentiation, library
routines (scipy.ndimage) and brute force on tiny inputs.
"""
import math
import os

import numpy as np
import pytest
from scipy import ndimage

from oracle import brute
from oracle import oracle as ora
from synth import configs as C
from synth import events as G

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "closed_forms.txt")


def golden():
    out = {}
    for line in open(GOLDEN):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        k, v = line.split()
        out[k] = float(v)
    return out


def h4(rows):
    a = np.zeros((len(rows), 4), np.float32)
    for i, r in enumerate(rows):
        a[i, :len(r)] = r
    return a


# ---------------------------------------------------------------- P1
def test_P1_hit_on_pattern_contributes_exactly_one():
    # tx = k / 2^10, integer z: x = tx z is exact, so s = 0 exactly in every model.
    tx, ty = 77 / 1024, -301 / 1024
    rows = [(tx * z, ty * z, z) for z in (30.0, 60.0, 450.0, 750.0)]
    R, g, _ = ora.point(C.SLOPE2, h4(rows), (tx, ty), 0.44)
    assert R == 4.0 and np.all(g == 0.0)
    z0 = -37.0
    rows3 = [(tx * (z - z0), ty * (z - z0), z) for z in (30.0, 60.0, 750.0)]
    R3, g3, _ = ora.point(C.SLOPE3, h4(rows3), (tx, ty, z0), 0.88)
    assert R3 == 3.0 and np.all(g3 == 0.0)
    a, b = 0.25, -0.375
    rows2 = [(x, a * x + b) for x in (1.0, 2.0, 7.0)]
    R2, g2, _ = ora.point(C.LINE2D, h4(rows2), (a, b), 0.005)
    assert R2 == 3.0 and np.all(g2 == 0.0)


# ---------------------------------------------------------------- P2
def test_P2_bounds_0_le_R_le_N():
    rng = np.random.default_rng(0)
    for model in (C.LINE2D, C.SLOPE2, C.SLOPE3):
        for _ in range(20):
            n = int(rng.integers(0, 40))
            h = rng.normal(0, 3, (n, 4)).astype(np.float32)
            h[:, 2] = np.abs(h[:, 2]) * 100
            th = rng.normal(0, 0.2, 3)[: 3 if model == C.SLOPE3 else 2]
            R, _, _ = ora.point(model, h, th, float(rng.uniform(0.05, 5)))
            assert 0.0 <= R <= n


# ---------------------------------------------------------------- P3
def test_P3_closed_form_distances():
    gv = golden()
    sig = float(np.float32(0.44031311))
    # SLOPE2, theta = 0: s = |(x, y)| in the plane
    assert ora.point(C.SLOPE2, h4([]), (0, 0), sig)[0] == 0.0
    assert ora.point(C.SLOPE2, h4([(0, 0, 100)]), (0, 0), sig)[0] == gv["one_hit_s0"]
    R1 = ora.point(C.SLOPE2, h4([(sig, 0, 100)]), (0, 0), sig)[0]
    assert abs(R1 - gv["one_hit_s_sigma"]) <= 1e-15
    # distance 2 sigma along y -- also pins that s^2 = s_x^2 + s_y^2 (no sqrt, no 1/2)
    R2 = ora.point(C.SLOPE2, h4([(0, -sig, 30), (0, 2 * sig, 30)]), (0, 0), sig)[0]
    assert abs(R2 - gv["hits_sigma_2sigma"]) <= 1e-15
    # 3 sigma split over both coordinates as a 3-4-5 triangle: sigma = 5/8,
    # (s_x, s_y) = (9/8, 3/2) are exact binaries with s_x^2 + s_y^2 = 9 sigma^2
    R3 = ora.point(C.SLOPE2, h4([(1.125, 1.5, 1)]), (0, 0), 0.625)[0]
    assert abs(R3 - gv["one_hit_s_3sigma"]) <= 1e-15
    # LINE2D: vertical residual y - (a x + b)
    RL = ora.point(C.LINE2D, h4([(3.0, 1.0 + 0.25), (5.0, 1.0 - 0.5)]), (0.0, 1.0), 0.25)[0]
    assert abs(RL - gv["hits_sigma_2sigma"]) <= 1e-15


# ---------------------------------------------------------------- P4 (north star: brute force)
@pytest.mark.parametrize("model", [C.LINE2D, C.SLOPE2, C.SLOPE3])
def test_P4_brute_force_mpmath(model):
    rng = np.random.default_rng(10 + model)
    for _ in range(6):
        n = int(rng.integers(1, 16))
        P = 3 if model == C.SLOPE3 else 2
        th_true = np.array([rng.uniform(-0.3, 0.3), rng.uniform(-0.3, 0.3), rng.uniform(-20, 20)])[:P]
        z = np.sort(rng.choice(C.VELO_PLANES[1:], n))
        if model == C.LINE2D:
            x = rng.integers(1, 11, n).astype(float)
            rows = [(xi, th_true[0] * xi + th_true[1] + rng.normal(0, 0.01)) for xi in x]
        else:
            d = z - (th_true[2] if model == C.SLOPE3 else 0.0)
            rows = [(th_true[0] * di + rng.normal(0, .05), th_true[1] * di + rng.normal(0, .05), zi)
                    for di, zi in zip(d, z)]
        h = h4(rows)
        sigma = float(np.float32(0.05 if model == C.LINE2D else 0.3))
        th = th_true + rng.normal(0, [1e-3, 1e-3, 0.1][:P])
        R, g, A = ora.point(model, h, th, sigma)
        Rb = float(brute.response(model, h, th, sigma))
        gb = [float(v) for v in brute.gradient(model, h, th, sigma)]
        assert abs(R - Rb) <= 1e-13 * max(Rb, 1e-300)
        for i in range(P):
            assert abs(g[i] - gb[i]) <= 1e-12 * max(A[i], 1e-300)


# ---------------------------------------------------------------- P5
@pytest.mark.parametrize("model", [C.LINE2D, C.SLOPE2, C.SLOPE3])
def test_P5_gradient_vs_central_differences(model):
    cfg = {C.LINE2D: C.CFG0, C.SLOPE2: C.CFG2, C.SLOPE3: C.CFG4}[model]
    b = G.make_batch(cfg, [0])
    h = b.event_hits(0)
    rng = np.random.default_rng(5)
    P = cfg.P
    for k in range(8):
        t0 = b.truth[0][k % len(b.truth[0])]
        th = np.array(t0, float) + rng.normal(0, [2e-3, 2e-3, 0.5][:P])
        _, g, A = ora.point(model, h, th, cfg.sigma)
        scale = np.array([1e-6, 1e-6, 1e-4][:P])
        for i in range(P):
            e = np.zeros(P)
            e[i] = scale[i]
            # Richardson-extrapolated central difference: O(h^4)
            d1 = (ora.point(model, h, th + e, cfg.sigma)[0] - ora.point(model, h, th - e, cfg.sigma)[0]) / (2 * e[i])
            d2 = (ora.point(model, h, th + 2 * e, cfg.sigma)[0] - ora.point(model, h, th - 2 * e, cfg.sigma)[0]) / (4 * e[i])
            fd = (4 * d1 - d2) / 3
            assert abs(g[i] - fd) <= 1e-5 * max(A[i], 1e-9), (i, g[i], fd, A[i])


# ---------------------------------------------------------------- P6
def test_P6_mirror_pair_zero_gradient():
    tx, ty, d = 0.1, -0.05, 300.0
    cx, cy = tx * d, ty * d
    for dx, dy, axis in ((0.2, 0.0, 0), (0.0, 0.3, 1)):
        h = h4([(cx + dx, cy + dy, d), (cx - dx, cy - dy, d)])
        _, g, A = ora.point(C.SLOPE2, h, (tx, ty), 0.44)
        assert abs(g[axis]) <= 1e-12 * A[axis]
        assert A[axis] > 0
    # LINE2D: hits mirrored about the line in y at the same x -> dR/db = 0
    h = h4([(4.0, 2.125 + 0.015625), (4.0, 2.125 - 0.015625)])  # exact binaries
    _, g, A = ora.point(C.LINE2D, h, (0.5, 0.125), 0.03125)
    assert abs(g[1]) <= 1e-12 * A[1] and abs(g[0]) <= 1e-12 * A[0]


# ---------------------------------------------------------------- P7
def test_P7_invariants():
    b = G.make_batch(C.CFG2, [3])
    h = b.event_hits(0)
    th = b.truth[0][0] + 1e-3
    s = C.CFG2.sigma
    RA = ora.point(C.SLOPE2, h[:400], th, s)[0]
    RB = ora.point(C.SLOPE2, h[400:], th, s)[0]
    R = ora.point(C.SLOPE2, h, th, s)[0]
    assert abs(R - (RA + RB)) <= 1e-13 * R  # additivity
    Rs = [ora.point(C.SLOPE2, h, th, sg)[0] for sg in (0.1, 0.2, 0.44, 1.0, 3.0)]
    assert all(a <= b for a, b in zip(Rs, Rs[1:]))  # non-decreasing in sigma
    # LINE2D translation: y -> y + delta and b -> b + delta leaves R unchanged
    b0 = G.make_batch(C.CFG0, [0])
    h0 = b0.event_hits(0).copy()
    h0[:, 1] = np.round(h0[:, 1] * 2.0 ** 16) / 2.0 ** 16  # so that y + delta is exact in fp32
    delta = 0.5
    h1 = h0.copy()
    h1[:, 1] += np.float32(delta)
    for a_, b_ in ((0.1, 0.2), (-0.3, 0.7)):
        r0 = ora.point(C.LINE2D, h0, (a_, b_), 0.02)[0]
        r1 = ora.point(C.LINE2D, h1, (a_, b_ + delta), 0.02)[0]
        assert abs(r0 - r1) <= 1e-12 * max(r0, 1e-3)
    # special-case reductions between models: SLOPE3 with z0 = c == SLOPE2 with z_ref = c
    for c in (0.0, -42.5, 17.25):
        r2, g2, _ = ora.point(C.SLOPE2, h, th, s, z_ref=c)
        r3, g3, _ = ora.point(C.SLOPE3, h, (th[0], th[1], c), s)
        assert r2 == r3 and np.all(g2 == g3[:2])


# ---------------------------------------------------------------- P8 (derived from PAPER.md:38)
def test_P8_single_hit_closed_form_and_grid_argmax():
    sig = 0.44031311
    x, y, d = 7.3, -4.1, 270.0
    h = h4([(x, y, d)])
    rng = np.random.default_rng(1)
    for _ in range(10):
        t = rng.uniform(-0.3, 0.3, 2)
        # R(t) = exp(-d^2 |t - h/d|^2 / sigma^2)
        u = np.array([x, y]) / d
        closed = math.exp(-d * d * float(np.sum((t - u) ** 2)) / (sig * sig))
        R, g, _ = ora.point(C.SLOPE2, h, t, float(np.float32(sig)))
        sig32 = float(np.float32(sig))
        closed32 = math.exp(-d * d * float(np.sum((t - np.array([np.float32(x), np.float32(y)]) / d) ** 2)) / sig32 ** 2)
        assert abs(R - closed32) <= 1e-12
        gc = 2 * d * d / sig32 ** 2 * closed32 * (np.array([np.float32(x), np.float32(y)]) / d - t)
        assert np.allclose(g, gc, rtol=1e-9, atol=1e-300)
    # the grid argmax is the node nearest h/d (per axis, the grid is separable)
    nodes = G.axis_nodes(C.CFG1)
    Rg = ora.grid(C.SLOPE2, [0, 1], h, nodes, 0.05)
    i, j = np.unravel_index(np.argmax(Rg[0]), Rg[0].shape)
    assert i == np.argmin(np.abs(nodes[0].astype(float) - np.float32(x) / d))
    assert j == np.argmin(np.abs(nodes[1].astype(float) - np.float32(y) / d))


# ---------------------------------------------------------------- P9
def test_P9_noiseless_recovery_grid_and_multistart():
    nodes = [np.linspace(-0.3, 0.3, 61).astype(np.float32)] * 2
    truth_ij = [(10, 12), (30, 45), (50, 20)]
    rows = []
    nh = []
    for (i, j) in truth_ij:
        tx, ty = float(nodes[0][i]), float(nodes[1][j])
        k = 0
        for z in C.VELO_PLANES[1:]:
            r = math.hypot(tx * z, ty * z)
            if 5 < r < 40:
                rows.append((np.float32(tx) * z, np.float32(ty) * z, z))
                k += 1
        nh.append(k)
    rows.sort(key=lambda r: r[2])
    h = h4(rows)
    sig = 0.05
    Rg = ora.grid(C.SLOPE2, [0, len(h)], h, nodes, sig)
    idx, val, cnt = ora.peaks(Rg, 2, 2.5, 64)
    found = sorted(int(v) for v in idx[0, :cnt[0]])
    assert found == sorted(i * 61 + j for i, j in truth_ij)
    for (i, j), n in zip(truth_ij, nh):
        # each own hit contributes 1 up to the fp32 rounding of its coordinates (s ~ 1e-6 mm)
        assert Rg[0, i, j] >= n * (1 - 1e-7)
    # multi-start from seeds inside a basin converges monotonically toward theta_true
    tt = np.array([[nodes[0][i], nodes[1][j]] for i, j in truth_ij], np.float64)
    seeds = (tt + np.array([[2e-5, -1.5e-5]])).astype(np.float32)[None]
    step = C.step_slope2(sig)
    prev = first = np.abs(seeds[0].astype(float) - tt).max(axis=1)
    for n_it in (1, 2, 5, 20, 100, 2000):
        th, R, _ = ora.multistart(C.SLOPE2, [0, len(h)], h, seeds, sig, n_it, step, (-.3, -.3), (.3, .3))
        dist = np.abs(th[0] - tt).max(axis=1)
        assert np.all(dist <= prev + 1e-12)
        prev = dist
    assert np.all(prev < 0.01 * first)


def test_P9_slope3_noiseless_recovery_and_layout():
    """P = 3 (PAPER.md:47-48 with a free origin z0): noiseless tracks whose (tx, ty, z0) sit on
    lattice nodes are the grid's peaks, at flat offsets (l n0 + i) n1 + j of the z0-plane layout
    (reading Z37), and each cell equals the point response at its node tuple."""
    nodes = [np.linspace(-0.3, 0.3, 31).astype(np.float32), np.linspace(-0.3, 0.3, 29).astype(np.float32),
             np.linspace(-40.0, 40.0, 9).astype(np.float32)]
    truth = [(5, 20, 2), (22, 7, 6)]
    rows = []
    for (i, j, l) in truth:
        tx, ty, z0 = (float(nodes[0][i]), float(nodes[1][j]), float(nodes[2][l]))
        for z in C.VELO_PLANES[1:]:
            d = z - z0
            if 5 < math.hypot(tx * d, ty * d) < 40:
                rows.append((tx * d, ty * d, z))
    rows.sort(key=lambda r: r[2])
    h = h4(rows)
    sig = 0.05
    Rg = ora.grid(C.SLOPE3, [0, len(h)], h, nodes, sig)
    assert Rg.shape == (1, 9, 31, 29)
    idx, _, cnt = ora.peaks(Rg, 3, 2.5, 64)
    assert sorted(int(v) for v in idx[0, :cnt[0]]) == sorted((l * 31 + i) * 29 + j for i, j, l in truth)
    rng = np.random.default_rng(7)
    for _ in range(20):
        i, j, l = int(rng.integers(31)), int(rng.integers(29)), int(rng.integers(9))
        R, _, _ = ora.point(C.SLOPE3, h, [nodes[0][i], nodes[1][j], nodes[2][l]], float(np.float32(sig)))
        assert Rg[0, l, i, j] == R


# ---------------------------------------------------------------- P10
def _strict_max_scipy(g, thr):
    P = g.ndim
    fp = np.ones((3,) * P, bool)
    fp[(1,) * P] = False
    nb = ndimage.maximum_filter(g, footprint=fp, mode="constant", cval=-np.inf)
    return np.flatnonzero((g > nb) & (g >= thr))


@pytest.mark.parametrize("P", [2, 3])
def test_P10_peak_rule(P):
    rng = np.random.default_rng(P)
    shape = (9, 13) if P == 2 else (7, 6, 9)
    for trial in range(30):
        g = rng.integers(0, 4, shape).astype(np.float64)  # many planted ties
        thr = float(rng.choice([0.0, 1.0, 2.5]))
        idx, val, cnt = ora.peaks(g[None], P, thr, 10_000)
        exp = _strict_max_scipy(g, thr)
        assert cnt[0] == len(exp) and np.array_equal(idx[0, :cnt[0]], exp)
        assert np.array_equal(val[0, :cnt[0]], g.ravel()[exp])
        # adding a constant to grid and R0 leaves the peaks unchanged
        idx2, _, cnt2 = ora.peaks(g[None] + 8.0, P, thr + 8.0, 10_000)
        assert cnt2[0] == cnt[0] and np.array_equal(idx2[0, :cnt[0]], idx[0, :cnt[0]])
    # constant grid -> none; single peak -> argmax
    assert ora.peaks(np.ones((1,) + shape), P, 0.0, 10)[2][0] == 0
    g = np.zeros(shape)
    c = tuple(s // 2 for s in shape)
    g[c] = 3.0
    idx, _, cnt = ora.peaks(g[None], P, 0.0, 10)
    assert cnt[0] == 1 and idx[0, 0] == np.ravel_multi_index(c, shape)
    # capacity: the true count is reported, only `cap` entries written
    g = rng.random(shape)
    idx, _, cnt = ora.peaks(g[None], P, 0.0, 2)
    assert cnt[0] == len(_strict_max_scipy(g, 0.0)) and idx.shape[1] == 2


# ---------------------------------------------------------------- P11 (Z7)
def test_P11_multistart_identities():
    cfg = C.CFG2
    b = G.make_batch(cfg, [0, 1])
    seeds = G.make_seeds(cfg, [0, 1], n_seeds=64)
    th, R, g = ora.multistart(cfg.model, b.offsets, b.hits, seeds, cfg.sigma, 0, cfg.step,
                              cfg.box_lo, cfg.box_hi)
    assert np.array_equal(th, seeds.astype(np.float64))
    for e in range(2):
        for s in (0, 17, 63):
            R1, g1, _ = ora.point(cfg.model, b.event_hits(e), seeds[e, s], cfg.sigma)
            assert R[e, s] == R1 and np.array_equal(g[e, s], g1)
    th0, _, _ = ora.multistart(cfg.model, b.offsets, b.hits, seeds, cfg.sigma, 7, 0.0, cfg.box_lo, cfg.box_hi)
    assert np.array_equal(th0, seeds.astype(np.float64))
    thb, _, _ = ora.multistart(cfg.model, b.offsets, b.hits, seeds, cfg.sigma, 10, cfg.step * 1e4,
                               cfg.box_lo, cfg.box_hi)
    assert np.all(thb >= np.float32(-0.3)) and np.all(thb <= np.float32(0.3))


def test_P11_single_hit_trajectory_is_a_straight_contraction():
    # one hit: grad R is parallel to (h/d - t) so ascent moves t straight toward h/d
    x, y, d = 9.0, -3.0, 300.0
    h = h4([(x, y, d)])
    u = np.array([x, y]) / d
    sig = 2.0
    seeds = np.array([[[0.02, -0.015], [0.035, 0.0]]], np.float32)
    th, R, _ = ora.multistart(C.SLOPE2, [0, 1], h, seeds, sig, 3, C.step_slope2(sig) * 30,
                              (-.3, -.3), (.3, .3))
    for s in range(2):
        v0 = seeds[0, s].astype(float) - u
        v1 = th[0, s] - u
        assert abs(v0[0] * v1[1] - v0[1] * v1[0]) <= 1e-12 * np.linalg.norm(v0) ** 2
        assert 0 < np.linalg.norm(v1) < np.linalg.norm(v0)
        assert np.dot(v0, v1) > 0


def test_P11_single_hit_one_step_closed_form():
    """One fixed-step update on one SLOPE2 hit, in closed form: with u = (x, y)/d,
    R(t) = exp(-d^2 |t - u|^2 / sigma^2) and grad R = (2 d^2 / sigma^2) R(t) (u - t), so
    t^1 = t^0 + eta (2 d^2 / sigma^2) R(t^0) (u - t^0)   (Alg. 1 update, reading Z7).
    Also with z_ref != 0 (d = z - z_ref) and for SLOPE3 at fixed z0 (d = z - z0; the z0 component
    of the step is then -eta (2/sigma^2) R sum (s_x tx + s_y ty), checked in closed form too)."""
    x, y, z = np.float32(7.25), np.float32(-4.5), np.float32(330.0)
    h = h4([(x, y, z)])
    sig = np.float32(1.5)
    eta = np.float32(3e-7)
    for z_ref in (0.0, 30.0):
        d = float(z) - z_ref
        u = np.array([float(x), float(y)]) / d
        seeds = np.array([[[0.0213, -0.0141], [0.026, -0.011], [-0.2, 0.25]]], np.float32)
        th, R, _ = ora.multistart(C.SLOPE2, [0, 1], h, seeds, float(sig), 1, float(eta), (-.3, -.3), (.3, .3),
                                  z_ref=z_ref)
        for s in range(seeds.shape[1]):
            t0 = seeds[0, s].astype(np.float64)
            R0 = math.exp(-d * d * float(np.sum((t0 - u) ** 2)) / float(sig) ** 2)
            t1 = t0 + float(eta) * (2 * d * d / float(sig) ** 2) * R0 * (u - t0)
            assert np.allclose(th[0, s], t1, rtol=0, atol=1e-15), (s, th[0, s], t1)
            if s < 2:
                assert np.linalg.norm(th[0, s] - t0) > 1e-6   # the step is not negligible
    # SLOPE3: theta = (tx, ty, z0); d = z - z0, s = (x - tx d, y - ty d)
    t0 = np.array([0.0215, -0.0138, 4.0])
    seeds = t0.astype(np.float32)[None, None]
    t0 = seeds[0, 0].astype(np.float64)
    th, _, _ = ora.multistart(C.SLOPE3, [0, 1], h, seeds, float(sig), 1, float(eta), (-.3, -.3, -150.), (.3, .3, 150.))
    d = float(z) - t0[2]
    sx, sy = float(x) - t0[0] * d, float(y) - t0[1] * d
    R0 = math.exp(-(sx * sx + sy * sy) / float(sig) ** 2)
    c = 2 / float(sig) ** 2 * R0
    t1 = t0 + float(eta) * c * np.array([sx * d, sy * d, -(sx * t0[0] + sy * t0[1])])
    assert np.allclose(th[0, 0], t1, rtol=0, atol=1e-13), (th[0, 0], t1)


# ---------------------------------------------------------------- P12
def _merge_cluster_all_then_select(theta, R, radius, thr):
    """Alternative formulation of PAPER.md:154-155: greedy leader clustering of
    ALL solutions in order (R desc, theta lex, index), then keep clusters whose
    leader (= highest R member) is >= R0."""
    n, P = theta.shape
    order = sorted(range(n), key=lambda s: (-R[s],) + tuple(theta[s]) + (s,))
    leaders, members = [], []
    for s in order:
        for li, l in enumerate(leaders):
            if all(abs(theta[s, i] - theta[l, i]) <= radius[i] for i in range(P)):
                members[li].append(s)
                break
        else:
            leaders.append(s)
            members.append([s])
    return [(l, sum(1 for m in mem if R[m] >= thr)) for l, mem in zip(leaders, members) if R[l] >= thr]


def test_P12_merge_examples_and_equivalence():
    rad = (6e-4, 6e-4)
    r32 = np.float32(6e-4).astype(float)
    th = np.array([[[0.1, 0.1], [0.1, 0.1], [0.1, 0.1]]])
    _, _, seed, size, cnt = ora.merge(th, np.array([[6.0, 6.0, 6.0]]), rad, 5.0, 8)
    assert cnt[0] == 1 and size[0, 0] == 3 and seed[0, 0] == 0
    th = np.array([[[0.1, 0.1], [0.1 + 10 * r32, 0.1]]])
    _, _, _, _, cnt = ora.merge(th, np.array([[6.0, 7.0]]), rad, 5.0, 8)
    assert cnt[0] == 2
    _, _, _, _, cnt = ora.merge(th, np.array([[4.0, 4.9]]), rad, 5.0, 8)
    assert cnt[0] == 0
    # equal R: the theta-lexicographically smaller one leads
    th = np.array([[[0.2, 0.1], [0.2, 0.0999], [0.1998, 0.3]]])
    _, _, seed, _, cnt = ora.merge(th, np.array([[6.0, 6.0, 6.0]]), rad, 5.0, 8)
    assert list(seed[0, :cnt[0]]) == [2, 1]
    # random sets vs the cluster-all formulation, and permutation invariance
    rng = np.random.default_rng(3)
    for trial in range(20):
        n = 300
        centers = rng.uniform(-0.3, 0.3, (12, 2))
        theta = centers[rng.integers(0, 12, n)] + rng.normal(0, 3e-4, (n, 2))
        R = rng.uniform(0, 12, n).round(1)  # planted R ties
        tt, tr, seed, size, cnt = ora.merge(theta[None], R[None], rad, 5.0, n)
        rad64 = np.array(rad, np.float32).astype(float)
        ref = _merge_cluster_all_then_select(theta, R, rad64, 5.0)
        assert [(int(a), int(b)) for a, b in zip(seed[0, :cnt[0]], size[0, :cnt[0]])] == ref
        perm = rng.permutation(n)
        _, _, seed2, size2, cnt2 = ora.merge(theta[perm][None], R[perm][None], rad, 5.0, n)
        assert cnt2[0] == cnt[0]
        assert list(perm[seed2[0, :cnt2[0]]]) == list(seed[0, :cnt[0]])
        assert np.array_equal(size2[0, :cnt2[0]], size[0, :cnt[0]])


# ---------------------------------------------------------------- P13
def test_P13_determinism_and_shard_invariance():
    cfg = C.CFG3
    full = G.make_batch(cfg, range(6))
    part = G.make_batch(cfg, [4, 5])
    assert np.array_equal(full.hits[full.offsets[4]:], part.hits)
    s_full = G.make_seeds(cfg, range(6), n_seeds=32)
    s_part = G.make_seeds(cfg, [4, 5], n_seeds=32)
    assert np.array_equal(s_full[4:], s_part)
    cfg2 = C.CFG2
    b = G.make_batch(cfg2, range(3))
    sd = G.make_seeds(cfg2, range(3), n_seeds=16)
    a1 = ora.multistart(cfg2.model, b.offsets, b.hits, sd, cfg2.sigma, 3, cfg2.step, cfg2.box_lo, cfg2.box_hi)
    a2 = ora.multistart(cfg2.model, b.offsets, b.hits, sd, cfg2.sigma, 3, cfg2.step, cfg2.box_lo, cfg2.box_hi)
    for x, y in zip(a1, a2):
        assert np.array_equal(x, y)


def test_generator_shapes_and_sorting():
    for name in ("cfg0", "cfg1", "cfg2", "cfg3", "cfg4"):
        cfg = C.CONFIGS[name]
        b = G.make_batch(cfg, range(min(cfg.n_events, 3)))
        assert b.hits.dtype == np.float32 and b.hits.shape[1] == 4
        for e in range(b.n_events):
            h = b.event_hits(e)
            key = h[:, 0] if cfg.model == C.LINE2D else h[:, 2]
            assert np.all(np.diff(key) >= 0)
        if cfg.n_seeds:
            s = G.make_seeds(cfg, [0], n_seeds=100)
            assert np.all(s >= np.float32(np.array(cfg.box_lo))) and np.all(s <= np.float32(np.array(cfg.box_hi)))


# ---------------------------------------------------------------- P14 step (iv)
@pytest.mark.parametrize("P", [2, 3])
def test_P14_estimate_exact_on_quadratics(P):
    """3-point quadratic interpolation is exact on a parabola: a quadratic bump centred between
    nodes is recovered to rounding, per axis, in parameter units."""
    rng = np.random.default_rng(40 + P)
    shape = (21, 17, 13)[:P]
    nodes = [np.linspace(-0.3, 0.3, n).astype(np.float32) for n in shape]
    for trial in range(10):
        c = [int(rng.integers(2, n - 2)) for n in shape]
        off = rng.uniform(-0.45, 0.45, P)
        curv = rng.uniform(0.5, 3.0, P)
        grids = np.meshgrid(*[np.arange(n, dtype=np.float64) for n in shape], indexing="ij")
        g = 100.0 - sum(curv[i] * (grids[i] - (c[i] + off[i])) ** 2 for i in range(P))
        if P == 3:  # the response layout stores z0 planes outermost (reading Z37)
            g = np.ascontiguousarray(g.transpose(2, 0, 1))
        mem_c, mem_shape = (c, shape) if P == 2 else ((c[2], c[0], c[1]), (shape[2], shape[0], shape[1]))
        idx, _, cnt = ora.peaks(g[None], P, 0.0, 16)
        assert cnt[0] == 1 and idx[0, 0] == np.ravel_multi_index(mem_c, mem_shape)
        th = ora.estimate(g[None], nodes, idx, cnt, 16)[0, 0]
        for i in range(P):
            step = float(nodes[i][c[i] + 1]) - float(nodes[i][c[i]])
            truth = float(nodes[i][c[i]]) + off[i] * 0.5 * (float(nodes[i][c[i] + 1]) - float(nodes[i][c[i] - 1]))
            assert abs(th[i] - truth) <= 1e-9 * abs(step), (i, th[i], truth)


def test_P14_estimate_centre_boundary_and_single_track():
    nodes = [np.linspace(-0.3, 0.3, 31).astype(np.float32)] * 2
    g = np.zeros((31, 31))
    g[10, 12] = 5.0
    g[9, 12] = g[11, 12] = 2.0   # symmetric along axis 0
    g[10, 11], g[10, 13] = 1.0, 1.0  # symmetric along axis 1
    g[0, 5] = 4.0                # boundary peak along axis 0
    g[1, 5] = 1.0
    idx, _, cnt = ora.peaks(g[None], 2, 0.5, 8)
    th = ora.estimate(g[None], nodes, idx, cnt, 8)[0]
    k = {int(v): i for i, v in enumerate(idx[0, :cnt[0]])}
    assert th[k[10 * 31 + 12]][0] == float(nodes[0][10]) and th[k[10 * 31 + 12]][1] == float(nodes[1][12])
    assert th[k[0 * 31 + 5]][0] == float(nodes[0][0])  # falls back to the cell centre
    # noiseless single track: the estimate is within half a step of the truth per axis and
    # at least as close as the peak cell's node ("maximal activation in the unit
    # with pattern parameters closest to the tracks parameters")
    cfg = C.CFG1
    nd = G.axis_nodes(cfg)
    tx, ty = 0.1234, -0.0567
    rows = [(tx * z, ty * z, z) for z in C.VELO_PLANES[1:] if 5 < np.hypot(tx * z, ty * z) < 40]
    h = h4(rows)
    grid = ora.grid(C.SLOPE2, [0, len(h)], h, nd, cfg.sigma)
    idx, _, cnt = ora.peaks(grid, 2, 2.5, 8)
    assert cnt[0] == 1
    th = ora.estimate(grid, nd, idx, cnt, 8)[0, 0]
    i, j = np.unravel_index(idx[0, 0], grid.shape[1:])
    step = float(nd[0][1] - nd[0][0])
    assert abs(th[0] - tx) <= 0.5 * step and abs(th[1] - ty) <= 0.5 * step
    assert abs(th[0] - tx) <= abs(float(nd[0][i]) - tx) + 1e-12
    assert abs(th[1] - ty) <= abs(float(nd[1][j]) - ty) + 1e-12


# ---------------------------------------------------------------- P15 Hessian
@pytest.mark.parametrize("model", [C.LINE2D, C.SLOPE2, C.SLOPE3])
def test_P15_hessian_vs_mpmath_and_fd(model):
    rng = np.random.default_rng(70 + model)
    P = 3 if model == C.SLOPE3 else 2
    for _ in range(4):
        n = int(rng.integers(2, 8))
        tt = np.array([rng.uniform(-0.3, 0.3), rng.uniform(-0.3, 0.3), rng.uniform(-20, 20)])[:P]
        z = np.sort(rng.choice(C.VELO_PLANES[1:], n))
        if model == C.LINE2D:
            rows = [(float(xi), tt[0] * xi + tt[1] + rng.normal(0, 0.01)) for xi in rng.integers(1, 11, n)]
            sigma = float(np.float32(0.05))
        else:
            d = z - (tt[2] if model == C.SLOPE3 else 0.0)
            rows = [(tt[0] * di + rng.normal(0, .05), tt[1] * di + rng.normal(0, .05), zi) for di, zi in zip(d, z)]
            sigma = float(np.float32(0.3))
        h = h4(rows)
        th = tt + rng.normal(0, [1e-3, 1e-3, 0.2][:P])
        R, g, H = ora.point_hess(model, h, th, sigma)
        Rp, gp, _ = ora.point(model, h, th, sigma)
        assert abs(R - Rp) <= 1e-14 * R and np.allclose(g, gp, rtol=1e-12, atol=0)  # = ora_point
        assert np.allclose(H, H.T, rtol=1e-12, atol=0)
        Hb = np.array([[float(v) for v in row] for row in brute.hessian(model, h, th, sigma)])
        scale = np.abs(Hb).max()
        assert np.abs(H - Hb).max() <= 1e-9 * scale, (H, Hb)
        # central differences of the (independently pinned) gradient
        for a in range(P):
            e = np.zeros(P)
            e[a] = [1e-7, 1e-7, 1e-5][a]
            fd = (ora.point(model, h, th + e, sigma)[1] - ora.point(model, h, th - e, sigma)[1]) / (2 * e[a])
            assert np.abs(fd - H[:, a]).max() <= 1e-5 * scale


# ---------------------------------------------------------------- P16 Truncated Newton
def _velo_track_hits(t, z0=0.0, smear=0.0, seed=0):
    rng = np.random.default_rng(seed)
    rows = []
    for z in C.VELO_PLANES:
        if z <= z0:
            continue
        x, y = t[0] * (z - z0), t[1] * (z - z0)
        if 5 < np.hypot(x, y) < 40:
            rows.append((x + rng.normal(0, smear) if smear else x, y + rng.normal(0, smear) if smear else y, z))
    return rows


def test_P16_newton_converges_to_the_maximiser_found_by_scipy():
    from scipy.optimize import minimize
    rows = _velo_track_hits((0.11, -0.07), smear=0.012, seed=1) + _velo_track_hits((-0.2, 0.15), smear=0.012, seed=2)
    rows.sort(key=lambda r: r[2])
    h = h4(rows)
    sig = float(np.float32(0.44))
    res = minimize(lambda t: -ora.point(C.SLOPE2, h, t, sig)[0], x0=[0.1105, -0.0695],
                   jac=lambda t: -ora.point(C.SLOPE2, h, t, sig)[1], method="BFGS",
                   options={"gtol": 1e-12, "maxiter": 500})
    seeds = np.array([[[0.1108, -0.0703], [0.1097, -0.0690]]], np.float32)
    th, R, g = ora.newton(C.SLOPE2, [0, len(h)], h, seeds, [sig] * 4, [C.step_slope2(sig)] * 4, sig, 8,
                          (-.3, -.3), (.3, .3))
    for s in range(2):
        assert np.abs(th[0, s] - res.x).max() <= 1e-9, (th[0, s], res.x)
        assert R[0, s] >= -res.fun - 1e-12


def test_P16_single_hit_newton_step_closed_form():
    """One Truncated-Newton step on ONE SLOPE2 hit, in closed form.  With u = (x, y)/d, v = u - t,
    c = 2 d^2 / sigma^2: grad R = R c v and -H = R c (I - c v v^T).  v is an eigenvector of -H with
    eigenvalue R c (1 - c |v|^2) > 0 when c |v|^2 < 1, and the gradient lies along it, so CG ends
    after one iteration with p = v / (1 - c |v|^2) (Z23).  For c |v|^2 = 1/4 the full step lands at
    u - v/3, closer to u, so Armijo accepts alpha = 1 (Z25):  t^1 = t + v / (1 - c |v|^2)."""
    x, y, z = np.float32(7.25), np.float32(-4.5), np.float32(330.0)
    h = h4([(x, y, z)])
    sig = float(np.float32(2.0))
    d = float(z)
    u = np.array([float(x), float(y)]) / d
    c = 2 * d * d / sig ** 2
    for direction in ([1.0, 0.0], [0.6, -0.8], [-0.28, 0.96]):
        v = np.array(direction) * np.sqrt(0.25 / c)          # c |v|^2 = 1/4
        t0 = (u - v).astype(np.float32)
        v = u - t0.astype(np.float64)                         # exact v for the fp32 seed
        th, R, _ = ora.newton(C.SLOPE2, [0, 1], h, t0[None, None], [sig], [C.step_slope2(sig)], sig, 8,
                              (-.3, -.3), (.3, .3))
        expect = t0.astype(np.float64) + v / (1.0 - c * float(v @ v))
        assert np.allclose(th[0, 0], expect, rtol=0, atol=1e-13), (th[0, 0], expect)
        assert np.linalg.norm(th[0, 0] - u) < np.linalg.norm(t0 - u)   # moved toward the hit
    # beyond the inflection (c |v|^2 > 1) -H is indefinite along v: the CG curvature test fails at
    # the first iteration and the step falls back to eta grad R (Z24), i.e. t + eta R c v
    v = np.array([0.6, -0.8]) * np.sqrt(1.5 / c)
    t0 = (u - v).astype(np.float32)
    v = u - t0.astype(np.float64)
    eta = float(np.float32(C.step_slope2(sig)))
    th, R, _ = ora.newton(C.SLOPE2, [0, 1], h, t0[None, None], [sig], [eta], sig, 8, (-.3, -.3), (.3, .3))
    R0 = np.exp(-d * d * float(v @ v) / sig ** 2)
    step = eta * R0 * c * v
    # Armijo on the fallback step: alpha = 2^-k for the first k whose trial passes; the
    # closed-form trial t0 + alpha step must be the result for some k <= 8
    cands = [t0.astype(np.float64) + 0.5 ** k * step for k in range(9)]
    assert min(np.abs(th[0, 0] - q).max() for q in cands) <= 1e-13


def test_P16_newton_ascent_identities_and_fallback():
    cfg = C.CFG2
    b = G.make_batch(cfg, [0])
    seeds = G.make_seeds(cfg, [0], n_seeds=64)
    sig = cfg.sigma
    # n_steps = 0: identity
    th, R, _ = ora.newton(cfg.model, b.offsets, b.hits, seeds, [], [], sig, 8, cfg.box_lo, cfg.box_hi)
    assert np.array_equal(th, seeds.astype(np.float64))
    # R is non-decreasing step by step at fixed sigma (Armijo acceptance or no move)
    prev = np.array([ora.point(cfg.model, b.event_hits(0), s, sig)[0] for s in seeds[0].astype(np.float64)])
    cur = seeds
    for j in range(4):
        th, R, _ = ora.newton(cfg.model, b.offsets, b.hits, cur, [sig], [cfg.step], sig, 8, cfg.box_lo, cfg.box_hi)
        assert np.all(R[0] >= prev - 1e-12)
        assert np.all(th >= np.float32(-0.3)) and np.all(th <= np.float32(0.3))
        prev, cur = R[0], th.astype(np.float32)
    # single hit far outside the Gaussian core: -H is not positive definite there, the first CG
    # iteration falls back to the gradient direction, which points straight at the hit
    x, y, d = 6.0, -3.0, 300.0
    h = h4([(x, y, d)])
    u = np.array([x, y]) / d
    s0 = np.array([[[0.02 + 0.004, -0.01 + 0.003]]], np.float32)  # 1.5 mm = 1.5 sigma from the hit
    sig1 = 1.0
    Rh, gh, Hh = ora.point_hess(C.SLOPE2, h, s0[0, 0].astype(np.float64), sig1)
    assert np.linalg.eigvalsh(-Hh).min() < 0  # indefinite: fallback path exercised
    th, R, _ = ora.newton(C.SLOPE2, [0, 1], h, s0, [sig1], [C.step_slope2(sig1) * 50], sig1, 30, (-.3, -.3), (.3, .3))
    v0, v1 = s0[0, 0].astype(float) - u, th[0, 0] - u
    assert abs(v0[0] * v1[1] - v0[1] * v1[0]) <= 1e-9 * np.dot(v0, v0)
    assert R[0, 0] > Rh


def test_P17_newton_evaluation_count():
    """Cost accounting of Algorithm 1 in response evaluations:
    q Hessian-mode evaluations + every line-search trial + the final evaluation."""
    cfg = C.CFG2
    b = G.make_batch(cfg, [0])
    seeds = G.make_seeds(cfg, [0], n_seeds=16)
    # no optimisation step: only the final evaluation
    *_, ne = ora.newton(cfg.model, b.offsets, b.hits, seeds, [], [], cfg.sigma, 8, cfg.box_lo, cfg.box_hi,
                        want_evals=True)
    assert np.all(ne == 1)
    # empty event: R = 0, grad = 0, p = 0, the first trial is accepted -> 2q + 1
    sig = [cfg.sigma * 3, cfg.sigma]
    eta = [cfg.step * 9, cfg.step]
    *_, ne = ora.newton(cfg.model, [0, 0], np.zeros((0, 4), np.float32), seeds, sig, eta, cfg.sigma, 8,
                        cfg.box_lo, cfg.box_hi, want_evals=True)
    assert np.all(ne == 2 * 2 + 1)
    # no gradient wanted and the final sigma is the last step's: the final evaluation repeats the
    # last step's value at that point and is not counted again (Z36); a different final sigma is
    th, R, _, ne = ora.newton(cfg.model, [0, 0], np.zeros((0, 4), np.float32), seeds, sig, eta, cfg.sigma, 8,
                              cfg.box_lo, cfg.box_hi, want_grad=False, want_evals=True)
    assert np.all(ne == 2 * 2)
    *_, ne = ora.newton(cfg.model, [0, 0], np.zeros((0, 4), np.float32), seeds, sig, eta, 2 * cfg.sigma, 8,
                        cfg.box_lo, cfg.box_hi, want_grad=False, want_evals=True)
    assert np.all(ne == 2 * 2 + 1)
    # seed on the box edge with the (fallback) ascent direction pointing out of the box: every
    # clamped trial equals the start, Armijo fails at every halving -> q (M + 1) + q + 1
    d = 300.0
    h = h4([(0.35 * d, 0.0, d)])  # the hit's slope lies outside the prior box in tx
    s0 = np.array([[[0.3, 0.0]]], np.float32)
    M = 8
    th, R, _, ne = ora.newton(C.SLOPE2, [0, 1], h, s0, [10.0, 10.0], [1e-6, 1e-6], 10.0, M, (-.3, -.3), (.3, .3),
                              want_evals=True)
    assert ne[0, 0] == 2 * (M + 1) + 2 + 1
    assert np.array_equal(th[0, 0], s0[0, 0].astype(np.float64))
