"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle on the same seeded
inputs (comparators T1..T7 of DESIGN.md §5).  Needs a B200."""
import numpy as np
import pytest
import torch

from oracle import oracle as ora
from synth import configs as C
from synth import events as G
from tests import parity_util as PU

import paper_1709_08610_b200 as R

pytestmark = pytest.mark.gpu
DEV = "cuda"


def dev(a, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV, dtype)


def events_of(batch, z_ref=0.0, hint=True):
    return R.Events.from_numpy(batch.offsets, batch.hits, z_ref=z_ref,
                               max_event_hits=None if hint else 0)


ALGOS = [R.retina.GRID_DIRECT, R.retina.GRID_SEPARABLE]


def gpu_grid(batch, cfg, nodes, z_ref=0.0, hint=True, sigma=None, algo=0):
    ev = events_of(batch, z_ref, hint)
    if algo == R.retina.GRID_SEPARABLE and cfg.model == C.LINE2D:
        algo = R.retina.GRID_DIRECT
    out = R.retina_grid_response(ev, cfg.model, cfg.sigma if sigma is None else sigma,
                                 [dev(n) for n in nodes], algorithm=algo)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def sub_lattice(g, pick):
    """Cells of a response grid [E, ...] (memory order: z0 planes outermost for P = 3, DESIGN.md
    Z37) on the sub-lattice of node subsets `pick` given in parameter order (tx, ty[, z0])."""
    mem = pick if len(pick) == 2 else [pick[2], pick[0], pick[1]]
    return g[(slice(None),) + np.ix_(*mem)]


def param_cells(flat, grid_dims):
    """Node indices in parameter order (tx, ty[, z0]) of flat cell offsets in a grid of per-event
    dims `grid_dims` (memory order)."""
    c = np.array(np.unravel_index(flat, grid_dims)).T
    return c if len(grid_dims) == 2 else c[:, [1, 2, 0]]


def synthetic_batch(model, counts, seed=0):
    """Events with given hit counts, VELO-like coordinates (or toy for LINE2D)."""
    rng = np.random.default_rng(seed)
    hs = []
    for n in counts:
        h = np.zeros((n, 4), np.float32)
        if model == C.LINE2D:
            h[:, 0] = rng.integers(1, 11, n)
            h[:, 1] = rng.uniform(-2, 2, n)
            h = h[np.argsort(h[:, 0], kind="stable")]
        else:
            z = rng.choice(C.VELO_PLANES, n)
            t = rng.uniform(-0.3, 0.3, (n, 2))
            h[:, 0] = t[:, 0] * z + rng.normal(0, 0.5, n)
            h[:, 1] = t[:, 1] * z + rng.normal(0, 0.5, n)
            h[:, 2] = z
            h = h[np.argsort(h[:, 2], kind="stable")]
        hs.append(h)
    off = np.zeros(len(counts) + 1, np.int32)
    off[1:] = np.cumsum(counts)
    hits = np.concatenate(hs) if hs else np.zeros((0, 4), np.float32)
    return G.EventBatch(offsets=off, hits=hits, event_ids=np.arange(len(counts)), truth=[None] * len(counts),
                        n_track_hits=np.zeros(len(counts)))


# --------------------------------------------------------------------------- T1
@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("name", ["cfg0", "cfg1"])
def test_T1_grid_full_single_event(name, algo):
    cfg = C.CONFIGS[name]
    b = G.make_batch(cfg, [0])
    nodes = G.axis_nodes(cfg)
    g = gpu_grid(b, cfg, nodes, algo=algo)
    ref = ora.grid(cfg.model, b.offsets, b.hits, nodes, cfg.sigma)
    ok, worst = PU.t1_response(g, ref)
    assert ok, worst


@pytest.mark.parametrize("model,z_ref,shape", [
    (C.SLOPE2, 0.0, (37, 70)), (C.SLOPE2, -12.345, (41, 33)), (C.LINE2D, 0.0, (29, 90)),
    (C.SLOPE3, 0.0, (5, 37, 45)), (C.SLOPE3, 0.0, (3, 70, 33))])
@pytest.mark.parametrize("hint", [True, False])
@pytest.mark.parametrize("algo", ALGOS)
def test_T1_grid_ragged_edges(model, z_ref, shape, hint, algo):
    # events: typical, empty, single hit, and one larger than the default hit stage (streaming)
    b = synthetic_batch(model, [700, 0, 1, 5000, 37], seed=len(shape) + model)
    P = len(shape)
    lo = [-0.3, -0.3, -150.0] if model != C.LINE2D else [-0.5, -1.0]
    hi = [0.3, 0.3, 150.0] if model != C.LINE2D else [0.5, 1.0]
    nodes = [np.linspace(lo[i], hi[i], shape[i]).astype(np.float32) for i in range(P)]
    sigma = 0.05 if model == C.LINE2D else 0.44
    cfg = C.Config(name="t", model=model, n_events=5, seed=0, n_tracks=0, sigma=sigma)
    g = gpu_grid(b, cfg, nodes, z_ref=z_ref, hint=hint, algo=algo)
    ref = ora.grid(model, b.offsets, b.hits, nodes, sigma, z_ref=z_ref)
    assert np.all(g[1] == 0.0)
    ok, worst = PU.t1_response(g, ref)
    assert ok, worst


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("name,events,sub", [("cfg3", [0, 9999], 48), ("cfg4", [0], 12)])
def test_T1_grid_full_size_sampled(name, events, sub, algo):
    """BASELINE full sizes (1024^2, 256^3) in the bench launch configuration; the oracle
    recomputes a sampled sub-lattice (random node subsets per axis)."""
    cfg = C.CONFIGS[name]
    b = G.make_batch(cfg, events)
    nodes = G.axis_nodes(cfg)
    g = gpu_grid(b, cfg, nodes, algo=algo)
    rng = np.random.default_rng(7)
    pick = [np.sort(rng.choice(len(n), sub, replace=False)) for n in nodes]
    pick = [np.unique(np.concatenate([p, [0, len(n) - 1]])) for p, n in zip(pick, nodes)]
    ref = ora.grid(cfg.model, b.offsets, b.hits, [n[p] for n, p in zip(nodes, pick)], cfg.sigma)
    sub_gpu = sub_lattice(g, pick)
    ok, worst = PU.t1_response(sub_gpu, ref)
    assert ok, worst


# --------------------------------------------------------------------------- T2
@pytest.mark.parametrize("name,z_ref", [("cfg0", 0.0), ("cfg2", 0.0), ("cfg2", 23.5), ("cfg4", 0.0)])
def test_T2_gradient_at_points(name, z_ref):
    cfg = C.CONFIGS[name]
    ev_ids = [0] if cfg.n_events == 1 else [0, 1, 2]
    b = G.make_batch(cfg, ev_ids)
    n = 256
    seeds = G.make_seeds(cfg, ev_ids, n_seeds=n)
    # half the points next to true tracks (where gradients cancel), half random
    for e in range(len(ev_ids)):
        t = b.truth[e]
        k = min(n // 2, len(t))
        rng = np.random.default_rng(e)
        near = t[rng.integers(0, len(t), k)] + rng.normal(0, [1e-4, 1e-4, 0.05][:cfg.P], (k, cfg.P))
        seeds[e, :k] = near.astype(np.float32)
    ev = events_of(b, z_ref)
    th, Rg, gg = R.retina_multistart_optimize(ev, cfg.model, cfg.sigma, dev(seeds), 0, 0.0,
                                              cfg.box_lo, cfg.box_hi)
    torch.cuda.synchronize()
    th, Rg, gg = th.cpu().numpy(), Rg.cpu().numpy(), gg.cpu().numpy()
    assert np.array_equal(th, seeds)
    worst1 = worst2 = 0.0
    for e in range(len(ev_ids)):
        h = b.event_hits(e)
        for s in range(n):
            r, g, A = ora.point(cfg.model, h, seeds[e, s].astype(np.float64), cfg.sigma, z_ref=z_ref)
            ok1, w1 = PU.t1_response(Rg[e, s], r)
            Gs = PU.grad_floor_scale(cfg.model, h, cfg.sigma, seeds[e, s].astype(np.float64))
            ok2, w2 = PU.t2_gradient(gg[e, s], g, A, Gs)
            worst1, worst2 = max(worst1, w1), max(worst2, w2)
    assert worst1 <= 1.0 and worst2 <= 1.0, (worst1, worst2)


# --------------------------------------------------------------------------- T3 / T4
@pytest.mark.parametrize("name", ["cfg0", "cfg1"])
@pytest.mark.parametrize("thr", [0.0, 2.5])
def test_T3_T4_peaks(name, thr):
    cfg = C.CONFIGS[name]
    b = G.make_batch(cfg, [0])
    nodes = G.axis_nodes(cfg)
    ev = events_of(b)
    grid = R.retina_grid_response(ev, cfg.model, cfg.sigma, [dev(n) for n in nodes])
    cap = 4096
    idx, val, cnt = R.retina_find_peaks(grid, cfg.P, thr, cap)
    torch.cuda.synchronize()
    g32 = grid.cpu().numpy()
    idx, val, cnt = idx.cpu().numpy(), val.cpu().numpy(), cnt.cpu().numpy()
    # T3: bit-exact on the same fp32 grid
    ri, rv, rc = ora.peaks(g32.astype(np.float64), cfg.P, thr, cap)
    assert cnt[0] == rc[0]
    k = min(cnt[0], cap)
    assert np.array_equal(idx[0, :k], ri[0, :k]) and np.array_equal(val[0, :k].astype(np.float64), rv[0, :k])
    # T4: vs the fp64 oracle grid, near-ties excused
    ref = ora.grid(cfg.model, b.offsets, b.hits, nodes, cfg.sigma)[0]
    ok, ndiff, nexc = PU.t4_peak_sets(idx[0], cnt[0], ref, cfg.P, thr, cap)
    assert ok, (ndiff, nexc)


@pytest.mark.parametrize("P,shape", [(2, (1, 37, 61)), (2, (3, 1024, 1024)), (3, (2, 19, 23, 29)),
                                     (3, (1, 64, 64, 64))])
def test_T3_peaks_bitexact_planted_ties(P, shape):
    rng = np.random.default_rng(P)
    g = rng.integers(0, 5, shape).astype(np.float32)  # many plateaus and ties
    g[0].flat[::97] = 7.0
    for thr, cap in ((0.0, 1 << 20), (3.0, 1 << 20), (0.0, 5)):
        idx, val, cnt = R.retina_find_peaks(dev(g), P, thr, cap)
        torch.cuda.synchronize()
        ri, rv, rc = ora.peaks(g.astype(np.float64), P, thr, cap)
        cnt = cnt.cpu().numpy()
        assert np.array_equal(cnt, rc)
        idx, val = idx.cpu().numpy(), val.cpu().numpy()
        for e in range(shape[0]):
            k = min(cnt[e], cap)
            assert np.array_equal(idx[e, :k], ri[e, :k])
            assert np.array_equal(val[e, :k].astype(np.float64), rv[e, :k])


@pytest.mark.parametrize("P,shape", [(2, (3, 1024, 1024)), (2, (5, 37, 61)), (3, (2, 64, 64, 64)),
                                     (3, (1, 256, 256, 256)), (2, (2, 700, 900)),
                                     # P = 3 plane-block (TMA ring) path: small rows, one block, max row
                                     # length, ragged last block, and a row length that is not a multiple
                                     # of 4 (slab path)
                                     (3, (2, 19, 23, 28)), (3, (1, 9, 300, 12)), (3, (1, 5, 7, 2048)),
                                     (3, (2, 4, 70, 36)), (3, (3, 40, 33, 200)), (3, (2, 33, 17, 29))])
def test_T3_peaks_workspace_path_identical(P, shape):
    """retina_find_peaks_ws (many CTAs per event) == retina_find_peaks (one CTA per event) ==
    the oracle rule, bit for bit, including ties and capacity overflow."""
    rng = np.random.default_rng(P + shape[1])
    g = rng.integers(0, 6, shape).astype(np.float32)
    dg = dev(g)
    ws = torch.empty((R.retina.find_peaks_workspace_size(shape[0], shape[1:]) // 4 + 1,), dtype=torch.int32,
                     device=DEV)
    for thr, cap in ((0.0, 1 << 21), (4.0, 1 << 20), (0.0, 7)):
        a = R.retina_find_peaks(dg, P, thr, cap)
        b = R.retina_find_peaks(dg, P, thr, cap, workspace=ws)
        torch.cuda.synchronize()
        assert torch.equal(a[2], b[2])
        for e in range(shape[0]):
            k = min(int(a[2][e]), cap)
            assert torch.equal(a[0][e, :k], b[0][e, :k]) and torch.equal(a[1][e, :k], b[1][e, :k])
        if np.prod(shape) <= 2e7:
            ri, rv, rc = ora.peaks(g.astype(np.float64), P, thr, cap)
            assert np.array_equal(b[2].cpu().numpy(), rc)
            for e in range(shape[0]):
                k = min(int(rc[e]), cap)
                assert np.array_equal(b[0][e, :k].cpu().numpy(), ri[e, :k])
                assert np.array_equal(b[1][e, :k].cpu().numpy().astype(np.float64), rv[e, :k])


@pytest.mark.parametrize("P,shape", [(2, (3, 1024, 1024)), (3, (2, 96, 96, 96))])
def test_T3_peaks_workspace_slab_lists_and_rescans(P, shape):
    """Sparse peaks (kept in the per-slab lists of pass 1 and copied) next to a dense region
    (P = 2: ~3,200 strict maxima in one slab, more than its list keeps, so pass 2 rescans it), in
    the same event: the workspace path equals the single-CTA path and the oracle bit for bit, for
    several capacities."""
    rng = np.random.default_rng(40 + P)
    g = rng.uniform(0.0, 1.0, shape).astype(np.float32)          # below threshold everywhere
    flat = g.reshape(shape[0], -1)
    cells = flat.shape[1]
    for e in range(shape[0]):
        pk = rng.choice(cells, 300, replace=False)                 # isolated planted peaks
        flat[e, pk] = rng.uniform(3.0, 9.0, 300).astype(np.float32)
        d0 = 131072 * (e % max(1, cells // 131072))                # one dense slab per event
        flat[e, d0:d0 + 60000] = rng.integers(2, 9, 60000).astype(np.float32)
    g = flat.reshape(shape)
    dg = dev(g)
    ws = torch.empty((R.retina.find_peaks_workspace_size(shape[0], shape[1:]) // 4 + 1,), dtype=torch.int32,
                     device=DEV)
    for thr, cap in ((2.5, 1 << 20), (2.5, 100), (2.5, 4000)):
        a = R.retina_find_peaks(dg, P, thr, cap)
        b = R.retina_find_peaks(dg, P, thr, cap, workspace=ws)
        torch.cuda.synchronize()
        assert torch.equal(a[2], b[2])
        ri, rv, rc = ora.peaks(g.astype(np.float64), P, thr, cap)
        assert np.array_equal(b[2].cpu().numpy(), rc)
        for e in range(shape[0]):
            k = min(int(rc[e]), cap)
            assert np.array_equal(b[0][e, :k].cpu().numpy(), ri[e, :k])
            assert np.array_equal(b[1][e, :k].cpu().numpy().astype(np.float64), rv[e, :k])
            assert torch.equal(a[0][e, :k], b[0][e, :k])


def test_T3_peaks_cfg4_slope3_sampled():
    cfg = C.CFG4
    b = G.make_batch(cfg, [1])
    nodes = G.axis_nodes(cfg)
    grid = R.retina_grid_response(events_of(b), cfg.model, cfg.sigma, [dev(n) for n in nodes])
    idx, val, cnt = R.retina_find_peaks(grid, 3, cfg.peak_threshold, cfg.peak_capacity)
    torch.cuda.synchronize()
    g32 = grid.cpu().numpy().astype(np.float64)
    ri, rv, rc = ora.peaks(g32, 3, cfg.peak_threshold, cfg.peak_capacity)
    cnt = cnt.cpu().numpy()
    assert cnt[0] == rc[0] and cnt[0] > 0
    k = min(cnt[0], cfg.peak_capacity)
    assert np.array_equal(idx.cpu().numpy()[0, :k], ri[0, :k])


# --------------------------------------------------------------------------- T5 / T6 / T7
def _run_multistart(cfg, ev_ids, n_seeds, n_iters=None, step=None, z_ref=0.0):
    b = G.make_batch(cfg, ev_ids)
    seeds = G.make_seeds(cfg, ev_ids, n_seeds=n_seeds)
    n_iters = cfg.n_iters if n_iters is None else n_iters
    step = cfg.step if step is None else step
    ev = events_of(b, z_ref)
    th, Rg, gg = R.retina_multistart_optimize(ev, cfg.model, cfg.sigma, dev(seeds), n_iters, step,
                                              cfg.box_lo, cfg.box_hi)
    torch.cuda.synchronize()
    return b, seeds, th, Rg, gg


# Bounds on the fraction of seeds (T5) / oracle tracks (T6) the oracle-side rules may excuse per
# config: about twice what the measured runs excuse (PARITY-STATS lines), so a
# kernel regression that moved many sensitive seeds (or dissolved tracks) still fails.
T5_EXCUSE_BOUND = {("cfg2", 1.0): 0.002, ("cfg2", 20.0): 0.005, ("cfg3", 1.0): 0.002, ("cfg4", 1.0): 0.002,
                   ("cfg0", 1e3): 0.12}   # measured (round 2): 0, 0.0020, 0, 0, 0.0625
T6_EXCUSE_BOUND = {("cfg2", 1.0): 0.03, ("cfg2", 20.0): 0.05, ("cfg3", 1.0): 0.03, ("cfg4", 1.0): 0.03}
# measured: 0/38, 1/48 (all members sensitive), 0/2, 0/1 and 0/96 oracle tracks excused


@pytest.mark.parametrize("name,n_ev,n_seeds,step_mult", [("cfg2", 4, 1024, 1.0), ("cfg2", 2, 512, 20.0),
                                                          ("cfg3", 2, 8192, 1.0),  # bench launch config
                                                          ("cfg4", 1, 256, 1.0), ("cfg4", 1, 16384, 1.0),
                                                          ("cfg0", 1, 256, 1e3)])
def test_T5_T6_T7_multistart_and_merge(name, n_ev, n_seeds, step_mult):
    cfg = C.CONFIGS[name]
    ev_ids = list(range(n_ev))
    n_iters = cfg.n_iters if cfg.n_iters else 20
    step = cfg.step * step_mult
    b, seeds, th_d, R_d, g_d = _run_multistart(cfg, ev_ids, n_seeds, n_iters, step)
    th, Rg = th_d.cpu().numpy(), R_d.cpu().numpy()
    rth, rR, rg = ora.multistart(cfg.model, b.offsets, b.hits, seeds, cfg.sigma, n_iters, step,
                                 cfg.box_lo, cfg.box_hi)
    ranges = np.array(cfg.box_hi, np.float64) - np.array(cfg.box_lo, np.float64)
    tag = f"T5/T6 {name} E={n_ev} S={n_seeds} step x{step_mult:g}"
    # T5: states within 1e-3 x range unless the seed is sensitive (the one oracle-side rule)
    unexcused, st5, sens_cache = PU.t5_states(cfg.model, b.offsets, b.hits, seeds, cfg.sigma, n_iters, step,
                                              cfg.box_lo, cfg.box_hi, th, rth, ranges)
    PU.report(tag, **st5)
    assert not unexcused, f"{len(unexcused)} non-sensitive seeds off by > 1e-3 range: {unexcused[:5]}"
    assert st5["excused_frac"] <= T5_EXCUSE_BOUND[(name, step_mult)], st5
    assert np.all(th >= np.float32(cfg.box_lo)) and np.all(th <= np.float32(cfg.box_hi))
    # T1 on the final responses: response_out = R(theta_out), checked at the GPU's own theta_out
    rng = np.random.default_rng(0)
    for e in range(len(ev_ids)):
        for s in rng.choice(th.shape[1], 64, replace=False):
            r, _, _ = ora.point(cfg.model, b.event_hits(e), th[e, s].astype(np.float64), cfg.sigma)
            ok, worst = PU.t1_response(Rg[e, s], r)
            assert ok, (e, s, worst)
    if cfg.P == 0 or name == "cfg0":
        return
    # T7: merge bit-exact vs the oracle merge on the GPU's fp32 outputs
    cap = cfg.track_capacity
    tt, tr, ts, tz, tc = R.retina_merge_tracks(th_d, R_d, cfg.merge_radius, cfg.track_threshold, cap)
    torch.cuda.synchronize()
    ts, tz, tc = ts.cpu().numpy(), tz.cpu().numpy(), tc.cpu().numpy()
    ott, otr, ots, otz, otc, gmem = ora.merge(th.astype(np.float64), Rg.astype(np.float64), cfg.merge_radius,
                                              cfg.track_threshold, cap, want_members=True)
    assert np.array_equal(tc, otc)
    for e in range(len(ev_ids)):
        k = min(tc[e], cap)
        assert np.array_equal(ts[e, :k], ots[e, :k]) and np.array_equal(tz[e, :k], otz[e, :k])
    assert np.array_equal(tt.cpu().numpy()[0, :min(tc[0], cap)], th[0, ts[0, :min(tc[0], cap)]])
    # T6: merged track sets of the GPU and oracle pipelines match one to one within 1e-3 range;
    # an unmatched track is excused only by a named oracle-side rule (near R0, near the merge
    # radius, all members sensitive)
    _, _, ots64, _, otc64, rmem = ora.merge(rth, rR, cfg.merge_radius, cfg.track_threshold, cap, want_members=True)
    assert np.all(otc64 <= cap) and np.all(tc <= cap)
    tot = {}
    for e in range(len(ev_ids)):
        def sensitive(s, e=e):
            if (e, s) not in sens_cache:
                sens_cache[(e, s)] = bool(PU.sensitive_seeds(cfg.model, b.offsets, b.hits, seeds, cfg.sigma, n_iters,
                                                             step, cfg.box_lo, cfg.box_hi, rth, ranges, [(e, s)])[0])
            return sens_cache[(e, s)]
        bad, cnt = PU.t6_tracks((th[e], Rg[e], ts[e, :tc[e]], gmem[e]), (rth[e], rR[e], ots64[e, :otc64[e]], rmem[e]),
                                ranges, cfg.merge_radius, cfg.track_threshold, sensitive)
        assert not bad, (e, bad, cnt)
        for k, v in cnt.items():
            tot[k] = tot.get(k, 0) + v
    excused = tot["near_R0"] + tot["near_radius"] + tot["sensitive"]
    PU.report(tag + " T6", **tot, excused_frac=excused / max(1, tot["tracks_ref"]))
    assert excused <= max(1, T6_EXCUSE_BOUND[(name, step_mult)] * tot["tracks_ref"]), tot


def test_T7_merge_synthetic_ties_and_capacity():
    rng = np.random.default_rng(11)
    E, S, P = 3, 16384, 3
    centers = rng.uniform(-0.3, 0.3, (40, P)).astype(np.float32)
    lab = rng.integers(0, 40, (E, S))
    th = (centers[lab] + rng.normal(0, 2e-4, (E, S, P))).astype(np.float32)
    th[:, ::7] = th[:, 3:4]  # exact duplicates
    Rv = rng.uniform(0, 12, (E, S)).round(1).astype(np.float32)  # exact R ties
    rad = (6e-4, 6e-4, 6e-4)
    for cap in (4096, 3):
        tt, tr, ts, tz, tc = R.retina_merge_tracks(dev(th), dev(Rv), rad, 5.0, cap)
        torch.cuda.synchronize()
        _, _, ots, otz, otc = ora.merge(th.astype(np.float64), Rv.astype(np.float64), rad, 5.0, cap)
        assert np.array_equal(tc.cpu().numpy(), otc)
        for e in range(E):
            k = min(otc[e], cap)
            assert np.array_equal(ts.cpu().numpy()[e, :k], ots[e, :k])
            assert np.array_equal(tz.cpu().numpy()[e, :k], otz[e, :k])


# --------------------------------------------------------------------------- K4c: culled = dense, bit for bit
@pytest.mark.parametrize("name,n_ev,n_seeds,n_iters,z_ref,want_grad,hint", [
    ("cfg2", 4, 4096, 50, 0.0, True, None), ("cfg2", 3, 1000, 20, 23.5, True, None),
    ("cfg3", 2, 8192, 50, 0.0, False, None),  # the bench launch configuration
    ("cfg3", 2, 8192, 0, 0.0, True, None), ("cfg2", 3, 777, 7, 0.0, True, 64),  # hint 64: events run dense
    ("cfg4", 1, 16384, 50, 0.0, False, None), ("cfg4", 2, 2000, 10, 0.0, True, None)])  # SLOPE3
def test_multistart_culled_bitwise_equal_to_dense(name, n_ev, n_seeds, n_iters, z_ref, want_grad, hint):
    """RETINA_MS_CULLED skips only pairs whose ex2.approx.ftz weight is exactly +0 and visits the
    others in hit order with K4's arithmetic: theta, R and grad R equal the dense kernel's bit for
    bit; it evaluates fewer pairs than the dense count (all pairs of all passes)."""
    cfg = C.CONFIGS[name]
    ev_ids = list(range(n_ev))
    b = G.make_batch(cfg, ev_ids)
    # plus an empty event and a single-hit event
    off = np.concatenate([b.offsets, [b.offsets[-1], b.offsets[-1] + 1]]).astype(np.int32)
    hits = np.concatenate([b.hits, b.hits[:1]])
    seeds = np.concatenate([G.make_seeds(cfg, ev_ids, n_seeds=n_seeds)] * 1 +
                           [G.make_seeds(cfg, [0, 1], n_seeds=n_seeds)], axis=0)
    ev = R.Events.from_numpy(off, hits, z_ref=z_ref, max_event_hits=hint)
    step = cfg.step if cfg.step else C.step_slope2(cfg.sigma)
    dense = R.retina_multistart_optimize(ev, cfg.model, cfg.sigma, dev(seeds), n_iters, step, cfg.box_lo,
                                         cfg.box_hi, want_grad=want_grad)
    pd = torch.zeros(1, dtype=torch.int64, device=DEV)
    pc = torch.zeros(1, dtype=torch.int64, device=DEV)
    dense2 = R.retina_multistart_optimize(ev, cfg.model, cfg.sigma, dev(seeds), n_iters, step, cfg.box_lo,
                                          cfg.box_hi, want_grad=want_grad, pairs_evaluated=pd)
    culled = R.retina_multistart_optimize(ev, cfg.model, cfg.sigma, dev(seeds), n_iters, step, cfg.box_lo,
                                          cfg.box_hi, want_grad=want_grad, algorithm=R.retina.MS_CULLED,
                                          pairs_evaluated=pc)
    torch.cuda.synchronize()
    for x, y, z in zip(dense, dense2, culled):
        if x is None:
            assert y is None and z is None
            continue
        assert torch.equal(x, y)
        assert torch.equal(x.view(torch.int32), z.view(torch.int32))  # bit for bit, signs of zeros included
    total = int(off[-1]) * seeds.shape[1] * (n_iters + 1)
    assert int(pd.item()) == total
    n_pc = int(pc.item())
    assert 0 < n_pc <= total
    if hint is None:
        assert n_pc < total
    PU.report(f"K4c {name} S={n_seeds} it={n_iters}", pairs_all=total, pairs_evaluated=n_pc,
              evaluated_frac=n_pc / total)


def test_multistart_culled_unsupported_and_workspace():
    cfg = C.CFG0
    b = G.make_batch(cfg, [0])
    ev = events_of(b)
    seeds = dev(G.make_seeds(cfg, [0], n_seeds=64))
    with pytest.raises(R.retina.RetinaError):  # LINE2D
        R.retina_multistart_optimize(ev, cfg.model, cfg.sigma, seeds, 1, 1e-8, (-0.5, -1.0), (0.5, 1.0),
                                     algorithm=R.retina.MS_CULLED)
    c2 = C.CFG2
    b2 = G.make_batch(c2, [0])
    s2 = dev(G.make_seeds(c2, [0], n_seeds=32))
    ws = torch.empty(1, dtype=torch.int32, device=DEV)  # 4 bytes: too small for 32 seeds
    with pytest.raises(R.retina.RetinaError):
        R.retina_multistart_optimize(events_of(b2), c2.model, c2.sigma, s2, 1, c2.step, c2.box_lo, c2.box_hi,
                                     algorithm=R.retina.MS_CULLED, workspace=ws)
    assert R.retina.multistart_workspace_size(3, 100) == 3 * 100 * 8  # permutation + Newton evaluation counts
    assert R.retina.multistart_workspace_size(3, 100, R.retina.MS_DENSE) == 0


# --------------------------------------------------------------------------- identities / edges
def test_multistart_identities_and_determinism():
    cfg = C.CFG2
    b = G.make_batch(cfg, [0, 1])
    seeds = G.make_seeds(cfg, [0, 1], n_seeds=1000)
    ev = events_of(b)
    sd = dev(seeds)
    th0, R0, _ = R.retina_multistart_optimize(ev, cfg.model, cfg.sigma, sd, 7, 0.0, cfg.box_lo, cfg.box_hi)
    torch.cuda.synchronize()
    assert torch.equal(th0, sd)
    a = R.retina_multistart_optimize(ev, cfg.model, cfg.sigma, sd, 10, cfg.step, cfg.box_lo, cfg.box_hi)
    bb = R.retina_multistart_optimize(ev, cfg.model, cfg.sigma, sd, 10, cfg.step, cfg.box_lo, cfg.box_hi)
    torch.cuda.synchronize()
    for x, y in zip(a, bb):
        assert torch.equal(x, y)
    # theta_out aliasing seeds; grad_out = NULL gives the same R
    alias = sd.clone()
    _, Ra, _ = R.retina_multistart_optimize(ev, cfg.model, cfg.sigma, alias, 10, cfg.step, cfg.box_lo,
                                            cfg.box_hi, want_grad=False,
                                            out=(alias, torch.empty_like(a[1]), None))
    torch.cuda.synchronize()
    assert torch.equal(alias, a[0]) and torch.equal(Ra, a[1])


def test_empty_batch_and_zero_hit_events():
    cfg = C.CFG1
    b = synthetic_batch(C.SLOPE2, [0, 0])
    nodes = [dev(n) for n in G.axis_nodes(cfg)]
    ev = events_of(b)
    g = R.retina_grid_response(ev, cfg.model, cfg.sigma, nodes)
    idx, val, cnt = R.retina_find_peaks(g, 2, 0.0, 16)
    seeds = dev(np.zeros((2, 10, 2), np.float32))
    th, Rr, gg = R.retina_multistart_optimize(ev, cfg.model, cfg.sigma, seeds, 5, 1e-3, (-.3, -.3), (.3, .3))
    torch.cuda.synchronize()
    assert torch.all(g == 0) and torch.all(cnt == 0) and torch.all(Rr == 0) and torch.all(gg == 0)
    e0 = R.Events(torch.zeros(1, dtype=torch.int32, device=DEV), torch.zeros((0, 4), device=DEV))
    out = R.retina_grid_response(e0, cfg.model, cfg.sigma, nodes)
    assert out.shape[0] == 0


def test_direct_and_separable_agree_cfg3_batch():
    """Both grid kernels on a 64-event cfg3 batch: each within T1 of the other's oracle-checked
    values (the pair is compared elementwise; both were checked against the oracle above)."""
    cfg = C.CFG3
    b = G.make_batch(cfg, range(64))
    nodes = G.axis_nodes(cfg)
    gd = gpu_grid(b, cfg, nodes, algo=R.retina.GRID_DIRECT)
    gs = gpu_grid(b, cfg, nodes, algo=R.retina.GRID_SEPARABLE)
    err = np.abs(gd.astype(np.float64) - gs) / (2e-5 * np.maximum(gd, 1e-6))
    assert err.max() <= 1.0, err.max()
    # peak sets from the two kernels agree up to near-ties of the direct grid
    for e in (0, 31, 63):
        idx, _, cnt = R.retina_find_peaks(dev(gs[e:e + 1]), 2, 2.5, 4096)
        ok, nd, ne = PU.t4_peak_sets(idx.cpu().numpy()[0], int(cnt[0]), gd[e].astype(np.float64), 2, 2.5, 4096)
        assert ok, (nd, ne)


# --------------------------------------------------------------------------- tensor-core grid (SLOPE2)
TENSOR = R.retina.GRID_TENSOR
TENSORS = [R.retina.GRID_TENSOR, R.retina.GRID_TENSOR_F16,  # 3xTF32 and the fp16-split kernels (default:
           R.retina.GRID_TENSOR_F16_PAIR, R.retina.GRID_TENSOR_F16_SINGLE]  # persistent pairs; per-tile pair, single)


@pytest.mark.parametrize("tensor", TENSORS)
def test_T1_tensor_grid_cfg1_full(tensor):
    cfg = C.CFG1
    b = G.make_batch(cfg, [0])
    nodes = G.axis_nodes(cfg)
    g = gpu_grid(b, cfg, nodes, algo=tensor)
    ref = ora.grid(cfg.model, b.offsets, b.hits, nodes, cfg.sigma)
    ok, worst = PU.t1_response(g, ref)
    assert ok, worst


@pytest.mark.parametrize("z_ref,shape", [(0.0, (37, 70)), (-12.345, (41, 33)), (0.0, (130, 300)),
                                         (0.0, (256, 512))])
@pytest.mark.parametrize("hint", [True, False])
@pytest.mark.parametrize("tensor", TENSORS)
def test_T1_tensor_grid_ragged_edges(z_ref, shape, hint, tensor):
    b = synthetic_batch(C.SLOPE2, [700, 0, 1, 5000, 37, 33], seed=3)
    nodes = [np.linspace(-0.3, 0.3, n).astype(np.float32) for n in shape]
    cfg = C.Config(name="t", model=C.SLOPE2, n_events=6, seed=0, n_tracks=0, sigma=0.44)
    g = gpu_grid(b, cfg, nodes, z_ref=z_ref, hint=hint, algo=tensor)
    ref = ora.grid(C.SLOPE2, b.offsets, b.hits, nodes, 0.44, z_ref=z_ref)
    assert np.all(g[1] == 0.0)
    ok, worst = PU.t1_response(g, ref)
    assert ok, worst


@pytest.mark.parametrize("tensor", TENSORS)
def test_T1_tensor_grid_cfg3_full_size_sampled(tensor):
    cfg = C.CFG3
    b = G.make_batch(cfg, [0, 5000, 9999])
    nodes = G.axis_nodes(cfg)
    g = gpu_grid(b, cfg, nodes, algo=tensor)
    rng = np.random.default_rng(9)
    pick = [np.unique(np.concatenate([np.sort(rng.choice(len(n), 48, replace=False)), [0, len(n) - 1]]))
            for n in nodes]
    ref = ora.grid(cfg.model, b.offsets, b.hits, [n[p] for n, p in zip(nodes, pick)], cfg.sigma)
    ok, worst = PU.t1_response(sub_lattice(g, pick), ref)
    assert ok, worst


@pytest.mark.parametrize("tensor", TENSORS)
def test_tensor_vs_separable_cfg3_batch_and_peaks(tensor):
    cfg = C.CFG3
    b = G.make_batch(cfg, range(32))
    nodes = G.axis_nodes(cfg)
    gt = gpu_grid(b, cfg, nodes, algo=tensor)
    gs = gpu_grid(b, cfg, nodes, algo=R.retina.GRID_SEPARABLE)
    err = np.abs(gt.astype(np.float64) - gs) / (2e-5 * np.maximum(gs, 1e-6))
    assert err.max() <= 1.0, err.max()
    for e in (0, 17, 31):
        idx, _, cnt = R.retina_find_peaks(dev(gt[e:e + 1]), 2, 2.5, 4096)
        ok, nd, ne = PU.t4_peak_sets(idx.cpu().numpy()[0], int(cnt[0]), gs[e].astype(np.float64), 2, 2.5, 4096)
        assert ok, (nd, ne)


# --------------------------------------------------------------------------- step (iv) estimate
@pytest.mark.parametrize("name,ev", [("cfg1", [0]), ("cfg3", [0, 1, 2]), ("cfg4", [0]), ("cfg0", [0])])
def test_estimate_peaks_vs_oracle(name, ev):
    cfg = C.CONFIGS[name]
    b = G.make_batch(cfg, ev)
    nodes = G.axis_nodes(cfg)
    dnodes = [dev(n) for n in nodes]
    grid = R.retina_grid_response(events_of(b), cfg.model, cfg.sigma, dnodes)
    cap = cfg.peak_capacity
    idx, val, cnt = R.retina_find_peaks(grid, cfg.P, cfg.peak_threshold, cap)
    th = R.retina_estimate_peaks(grid, dnodes, idx, cnt)
    torch.cuda.synchronize()
    g64 = grid.cpu().numpy().astype(np.float64)
    idx, cnt, th = idx.cpu().numpy(), cnt.cpu().numpy(), th.cpu().numpy()
    ref = ora.estimate(g64, nodes, idx, cnt, cap)
    steps = np.array([float(n[1] - n[0]) for n in nodes])
    n_checked = 0
    for e in range(len(ev)):
        k = min(cnt[e], cap)
        assert k > 0
        err = np.abs(th[e, :k].astype(np.float64) - ref[e, :k]) / steps
        assert err.max() <= 1e-3, err.max()  # fp32 vertex arithmetic vs fp64, in grid steps
        # every estimate stays inside its peak's cell (|delta| <= 1/2)
        cells = param_cells(idx[e, :k], g64.shape[1:])
        centre = np.stack([nodes[i][cells[:, i]] for i in range(cfg.P)], 1)
        assert np.all(np.abs(th[e, :k] - centre) <= 0.5 * steps * (1 + 1e-5))
        n_checked += k
    assert n_checked > 0


# --------------------------------------------------------------------------- NEXT #1: Truncated Newton
T5N_EXCUSE_BOUND = {"cfg2": 0.012, "cfg3": 0.02, "cfg4": 0.05}  # see T5_EXCUSE_BOUND
# measured (round 2, fp64 CG): cfg2 0.0054, cfg3 0.0068 / 0.0096 (512 / 8192 seeds), cfg4 0.027 / 0.018
# (256 / 16,384 seeds), most by the near-tie flip rule (seeds in empty regions whose Armijo tests
# compare R ~ 1e-200 in fp64 with R = 0 in fp32)
T6N_EXCUSE_BOUND = {"cfg2": 0.05, "cfg3": 0.05, "cfg4": 0.12}
# measured: 0/48, 0/0, 0/3; cfg4 1/6 and 19/331 -- cfg4's q = 3 Newton steps leave every candidate a
# single-seed cluster, so each excused far seed with R >= R0 is an unmatched track on both sides


@pytest.mark.parametrize("name,n_ev,n_seeds", [("cfg2", 4, 512), ("cfg3", 2, 512), ("cfg3", 2, 8192),
                                               ("cfg4", 1, 256), ("cfg4", 1, 16384)])
def test_newton_multistart_vs_oracle(name, n_ev, n_seeds):
    cfg = C.CONFIGS[name]
    ev_ids = list(range(n_ev))
    b = G.make_batch(cfg, ev_ids)
    seeds = G.make_seeds(cfg, ev_ids, n_seeds=n_seeds)
    sig, eta, fsig, mh = C.newton_schedule(cfg)
    th_d, R_d, g_d, ne_d = R.retina_multistart_newton_ex(events_of(b), cfg.model, dev(seeds), sig, eta, fsig, mh,
                                                         cfg.box_lo, cfg.box_hi)
    torch.cuda.synchronize()
    th, Rg = th_d.cpu().numpy(), R_d.cpu().numpy()
    rth, rR, _, margin, rne = ora.newton(cfg.model, b.offsets, b.hits, seeds, sig, eta, fsig, mh, cfg.box_lo,
                                         cfg.box_hi, want_margin=True, want_evals=True)
    # the paper's cost accounting (response evaluations per seed) is an integer: identical to the
    # oracle's for every seed whose discrete decisions were not oracle near-ties, unless the seed is
    # sensitive (its oracle run changes its evaluation count or end point under a +-1 ulp nudge:
    # the fp32 trajectory then legitimately takes other decisions further on)
    ne = ne_d.cpu().numpy()
    assert np.all(ne >= 2 * len(sig) + 1) and np.all(ne <= len(sig) * (mh + 2) + 1)
    ranges = np.array(cfg.box_hi, np.float64) - np.array(cfg.box_lo, np.float64)
    unexcused, st, excused_set = PU.t5n_states(cfg.model, cfg.box_lo, cfg.box_hi, b, seeds, sig, eta, fsig, mh, th,
                                               rth, ranges, ne, rne, R_ref=rR, R0=cfg.track_threshold)
    PU.report(f"T5n {name} E={n_ev} S={n_seeds}", **st)
    assert not unexcused, unexcused[:5]
    assert st["excused_frac"] <= T5N_EXCUSE_BOUND[name], st
    assert np.all(th >= np.float32(cfg.box_lo)) and np.all(th <= np.float32(cfg.box_hi))
    rng = np.random.default_rng(1)
    for e in range(n_ev):
        for s in rng.choice(n_seeds, 32, replace=False):
            r, _, _ = ora.point(cfg.model, b.event_hits(e), th[e, s].astype(np.float64), fsig)
            ok, worst = PU.t1_response(Rg[e, s], r)
            assert ok, (e, s, worst)
    # merge of the Newton solutions: bit-exact vs the oracle merge on the GPU's outputs
    tt, tr, ts, tz, tc = R.retina_merge_tracks(th_d, R_d, cfg.merge_radius, cfg.track_threshold, cfg.track_capacity)
    torch.cuda.synchronize()
    _, _, ots, otz, otc = ora.merge(th.astype(np.float64), Rg.astype(np.float64), cfg.merge_radius,
                                    cfg.track_threshold, cfg.track_capacity)
    assert np.array_equal(tc.cpu().numpy(), otc)
    if name == "cfg2":  # vertex at the origin: the pattern model is exact and tracks are found
        assert np.all(otc > 0)
    # T6 on the Newton path: GPU and oracle track sets match one to one; a track is excused only
    # by the named rules (near R0, near the radius, all members excused by the T5n rules)
    tc = tc.cpu().numpy()
    _, _, gts, _, gtc, gmem = ora.merge(th.astype(np.float64), Rg.astype(np.float64), cfg.merge_radius,
                                        cfg.track_threshold, cfg.track_capacity, want_members=True)
    _, _, rts, _, rtc, rmem = ora.merge(rth, rR, cfg.merge_radius, cfg.track_threshold, cfg.track_capacity,
                                        want_members=True)
    tot = {}
    for e in range(n_ev):
        def excused_seed(s, e=e):
            if (e, s) in excused_set:      # already attributed by T5n (flip or sensitivity)
                return True
            ok, _ = PU.newton_flip_explains(cfg.model, cfg.box_lo, cfg.box_hi, b.event_hits(e), seeds[e, s:s + 1],
                                            th[e, s:s + 1], None, ranges, sig, eta, fsig, mh)
            return bool(ok[0]) or PU.newton_sensitive(cfg.model, cfg.box_lo, cfg.box_hi, b.event_hits(e), seeds[e, s],
                                                      rth[e, s], ranges, sig, eta, fsig, mh)
        bad, cnt = PU.t6_tracks((th[e], Rg[e], gts[e, :gtc[e]], gmem[e]), (rth[e], rR[e], rts[e, :rtc[e]], rmem[e]),
                                ranges, cfg.merge_radius, cfg.track_threshold, excused_seed)
        assert not bad, (e, bad, cnt)
        for k, v in cnt.items():
            tot[k] = tot.get(k, 0) + v
    excused = tot["near_R0"] + tot["near_radius"] + tot["sensitive"]
    PU.report(f"T6n {name} E={n_ev} S={n_seeds}", **tot)
    assert excused <= max(1, T6N_EXCUSE_BOUND[name] * tot["tracks_ref"]), tot


def test_newton_line_search_queue_deterministic():
    """The line-search queue is filled with shared-memory atomics (entry order varies run to
    run); every seed's result and evaluation count must not: two runs agree bit for bit, and
    the run exercises the queue (seeds with more than one trial in some step)."""
    cfg = C.CFG3
    b = G.make_batch(cfg, [0, 1])
    seeds = dev(G.make_seeds(cfg, [0, 1], n_seeds=2048))
    sig, eta, fsig, mh = C.newton_schedule(cfg)
    runs = []
    for _ in range(2):
        out = R.retina_multistart_newton_ex(events_of(b), cfg.model, seeds, sig, eta, fsig, mh, cfg.box_lo,
                                            cfg.box_hi)
        torch.cuda.synchronize()
        runs.append([x.clone() for x in out])
    for x, y in zip(*runs):
        assert torch.equal(x, y)
    ne = runs[0][3]
    assert int((ne > 2 * len(sig) + 1).sum()) > 0  # some seeds needed halvings (queue path)


def test_newton_final_pass_reuse():
    """With no gradient wanted and the final sigma equal to the last step's, R(theta^q) comes from
    the last step's own evaluation at theta^q (its accepted trial, else its Hessian-mode pass):
    same trajectory bit for bit, one evaluation fewer per seed, R within T1 of a final pass (and
    bitwise equal to it wherever the value came from an accepted trial)."""
    cfg = C.CFG3
    b = G.make_batch(cfg, [3, 4])
    seeds = dev(G.make_seeds(cfg, [3, 4], n_seeds=2048))
    sig, eta, fsig, mh = C.newton_schedule(cfg)
    assert np.float32(sig[-1]) == np.float32(fsig)
    t1, r1, _, n1 = R.retina_multistart_newton_ex(events_of(b), cfg.model, seeds, sig, eta, fsig, mh, cfg.box_lo,
                                                  cfg.box_hi, want_grad=True)
    t0, r0, g0, n0 = R.retina_multistart_newton_ex(events_of(b), cfg.model, seeds, sig, eta, fsig, mh, cfg.box_lo,
                                                   cfg.box_hi, want_grad=False)
    torch.cuda.synchronize()
    assert g0 is None and torch.equal(t0, t1) and torch.equal(n0, n1 - 1)
    a, c = r0.cpu().numpy().astype(np.float64), r1.cpu().numpy().astype(np.float64)
    assert np.all(np.abs(a - c) <= 1e-5 * np.maximum(c, 1e-6))
    assert (a == c).mean() >= 0.5
    th = t0.cpu().numpy()
    for e in range(2):
        for s in range(0, 2048, 211):
            r, _, _ = ora.point(cfg.model, b.event_hits(e), th[e, s].astype(np.float64), fsig)
            assert PU.t1_response(float(a[e, s]), r)[0]


def test_newton_identities():
    cfg = C.CFG2
    b = G.make_batch(cfg, [0])
    seeds = dev(G.make_seeds(cfg, [0], n_seeds=300))
    th, Rn, _ = R.retina_multistart_newton(events_of(b), cfg.model, seeds, [], [], cfg.sigma, 8, cfg.box_lo,
                                           cfg.box_hi)
    th2, R2, _ = R.retina_multistart_optimize(events_of(b), cfg.model, cfg.sigma, seeds, 0, 0.0, cfg.box_lo,
                                              cfg.box_hi)
    torch.cuda.synchronize()
    assert torch.equal(th, seeds)
    assert torch.allclose(Rn, R2, rtol=2e-6, atol=1e-6)


@pytest.mark.parametrize("name,n_ev,n_seeds,z_ref,want_grad,hint,halvings", [
    ("cfg2", 3, 4096, 0.0, True, None, None), ("cfg2", 3, 1000, 23.5, False, None, None),
    ("cfg3", 2, 8192, 0.0, False, None, None),  # the bench's --update newton launch configuration
    ("cfg3", 2, 2048, 0.0, True, None, 30), ("cfg2", 3, 777, 0.0, True, 64, None),  # hint 64: events run dense
    ("cfg4", 1, 16384, 0.0, False, None, None), ("cfg4", 2, 2000, 0.0, True, None, None)])  # SLOPE3
def test_newton_culled_bitwise_equal_to_dense(name, n_ev, n_seeds, z_ref, want_grad, hint, halvings):
    """K6c (retina_multistart_newton_ex2, RETINA_MS_CULLED) skips only pairs whose ex2.approx.ftz
    weight is exactly +0 (Hessian-mode, line-search and final passes) and keeps every decision:
    theta, R, grad R and the per-seed evaluation counts equal the dense kernel's bit for bit; it
    evaluates fewer pairs than the dense count (evaluations x hits)."""
    cfg = C.CONFIGS[name]
    ev_ids = list(range(n_ev))
    b = G.make_batch(cfg, ev_ids)
    off = np.concatenate([b.offsets, [b.offsets[-1], b.offsets[-1] + 1]]).astype(np.int32)  # + empty, one hit
    hits = np.concatenate([b.hits, b.hits[:1]])
    seeds = np.concatenate([G.make_seeds(cfg, ev_ids, n_seeds=n_seeds), G.make_seeds(cfg, [0, 1], n_seeds=n_seeds)])
    ev = R.Events.from_numpy(off, hits, z_ref=z_ref, max_event_hits=hint)
    sig, eta, fsig, mh = C.newton_schedule(cfg)
    if halvings is not None:
        mh = halvings
    pd = torch.zeros(1, dtype=torch.int64, device=DEV)
    pc = torch.zeros(1, dtype=torch.int64, device=DEV)
    dense = R.retina_multistart_newton_ex(ev, cfg.model, dev(seeds), sig, eta, fsig, mh, cfg.box_lo, cfg.box_hi,
                                          want_grad=want_grad, pairs_evaluated=pd)
    culled = R.retina_multistart_newton_ex(ev, cfg.model, dev(seeds), sig, eta, fsig, mh, cfg.box_lo, cfg.box_hi,
                                           want_grad=want_grad, algorithm=R.retina.MS_CULLED, pairs_evaluated=pc)
    plain = R.retina_multistart_newton_ex(ev, cfg.model, dev(seeds), sig, eta, fsig, mh, cfg.box_lo, cfg.box_hi,
                                          want_grad=want_grad)
    torch.cuda.synchronize()
    for x, y, z in zip(plain, dense, culled):
        if x is None:
            assert y is None and z is None
            continue
        assert torch.equal(x, y)
        assert torch.equal(x.view(torch.int32), z.view(torch.int32))  # bit for bit, signs of zeros included
    n_hits = np.diff(off).astype(np.int64)
    total = int((plain[3].cpu().numpy().astype(np.int64) * n_hits[:, None]).sum())
    assert int(pd.item()) == total
    n_pc = int(pc.item())
    assert n_pc > 0
    if hint is None and cfg.model == C.SLOPE2:  # (SLOPE3's wide early sigmas keep nearly every hit in reach)
        assert n_pc < total
    PU.report(f"K6c {name} S={n_seeds}", pairs_dense=total, pairs_evaluated=n_pc, evaluated_frac=n_pc / total)


def test_newton_culled_no_steps_and_aliasing():
    """K6c with an empty schedule (one launch: the final pass only) and with theta_out aliasing the
    seeds (each launch reads the theta the previous one wrote) equals K6 bit for bit."""
    cfg = C.CFG2
    b = G.make_batch(cfg, [0, 1])
    seeds = G.make_seeds(cfg, [0, 1], n_seeds=1500)
    ev = events_of(b)
    sig, eta, fsig, mh = C.newton_schedule(cfg)
    for steps in (0, len(sig)):
        d = R.retina_multistart_newton_ex(ev, cfg.model, dev(seeds), sig[:steps], eta[:steps], fsig, mh, cfg.box_lo,
                                          cfg.box_hi)
        sd = dev(seeds)
        Rc = torch.empty(sd.shape[:2], dtype=torch.float32, device=DEV)
        gc = torch.empty_like(sd)
        nc = torch.empty(sd.shape[:2], dtype=torch.int32, device=DEV)
        c = R.retina_multistart_newton_ex(ev, cfg.model, sd, sig[:steps], eta[:steps], fsig, mh, cfg.box_lo,
                                          cfg.box_hi, out=(sd, Rc, gc, nc), algorithm=R.retina.MS_CULLED)
        torch.cuda.synchronize()
        for x, y in zip(d, c):
            assert torch.equal(x.view(torch.int32), y.view(torch.int32))


def test_newton_culled_unsupported_and_workspace():
    c2 = C.CFG2
    b2 = G.make_batch(c2, [0])
    s2 = dev(G.make_seeds(c2, [0], n_seeds=32))
    sig, eta, fsig, mh = C.newton_schedule(c2)
    ws = torch.empty(1, dtype=torch.int32, device=DEV)  # 4 bytes: too small for 32 seeds
    with pytest.raises(R.retina.RetinaError):
        R.retina_multistart_newton_ex(events_of(b2), c2.model, s2, sig, eta, fsig, mh, c2.box_lo, c2.box_hi,
                                      algorithm=R.retina.MS_CULLED, workspace=ws)
    with pytest.raises(R.retina.RetinaError):  # unknown algorithm
        R.retina_multistart_newton_ex(events_of(b2), c2.model, s2, sig, eta, fsig, mh, c2.box_lo, c2.box_hi,
                                      algorithm=5)


# --------------------------------------------------------------------------- tensor-core grid (SLOPE3)
@pytest.mark.parametrize("shape", [(5, 37, 45), (3, 70, 33), (130, 260, 3)])
@pytest.mark.parametrize("hint", [True, False])
@pytest.mark.parametrize("tensor", TENSORS)
def test_T1_tensor_grid_slope3_ragged(shape, hint, tensor):
    b = synthetic_batch(C.SLOPE3, [700, 0, 1, 5000, 37], seed=11)
    nodes = [np.linspace(lo, hi, n).astype(np.float32) for (lo, hi), n in
             zip([(-0.3, 0.3), (-0.3, 0.3), (-150.0, 150.0)], shape)]
    cfg = C.Config(name="t", model=C.SLOPE3, n_events=5, seed=0, n_tracks=0, sigma=0.88)
    g = gpu_grid(b, cfg, nodes, hint=hint, algo=tensor)
    ref = ora.grid(C.SLOPE3, b.offsets, b.hits, nodes, 0.88)
    assert np.all(g[1] == 0.0)
    ok, worst = PU.t1_response(g, ref)
    assert ok, worst


@pytest.mark.parametrize("model,z_ref,shape", [(C.SLOPE2, 0.0, (300, 516)), (C.SLOPE2, 7.5, (260, 132)),
                                               (C.SLOPE3, 0.0, (130, 260, 5)), (C.SLOPE3, 0.0, (40, 36, 7))])
def test_T1_default_grid_tma_store_ragged_tiles(model, z_ref, shape):
    """The default kernel's TMA-store epilogue (row pitch a multiple of 16 bytes): partial 256 x 256
    tiles at both edges, clipped by the tensor map's bounds (nothing written past n0 / n1, nor into
    the next z0 plane or event: the output buffer is pre-filled with a sentinel and the whole grid
    compared), empty / single-hit events, and an event longer than the hit window."""
    b = synthetic_batch(model, [700, 0, 1, 5000, 37], seed=21 + len(shape))
    P = len(shape)
    nodes = [np.linspace(lo, hi, n).astype(np.float32) for (lo, hi), n in
             zip([(-0.3, 0.3), (-0.3, 0.3), (-150.0, 150.0)], shape)]
    sigma = 0.44
    ev = events_of(b, z_ref)
    gshape = R.retina.grid_shape(5, shape)
    n_cells = int(np.prod(gshape))
    buf = torch.full((n_cells + 4096,), 7.25, device="cuda")   # sentinel tail right after the grid
    out = buf[:n_cells].view(gshape)
    R.retina_grid_response(ev, model, sigma, [dev(n) for n in nodes], out=out)
    torch.cuda.synchronize()
    g = out.cpu().numpy()
    ref = ora.grid(model, b.offsets, b.hits, nodes, sigma, z_ref=z_ref)
    assert g.shape == ref.shape and np.all(g[1] == 0.0)
    ok, worst = PU.t1_response(g, ref)
    assert ok, worst
    assert torch.all(buf[n_cells:] == 7.25)


@pytest.mark.parametrize("name,ev,model_shape", [
    ("cfg3", [0, 4999], None), ("cfg1", [0], None),
    ("ragged2", [700, 0, 1, 5000, 37], (C.SLOPE2, (300, 516))), ("ragged3", [700, 0, 1, 5000, 37], (C.SLOPE3, (130, 260, 5)))])
def test_T1_culled_tensor_grid_vs_fp64_oracle(name, ev, model_shape):
    """RETINA_GRID_TENSOR_F16_CULLED (each tile contracts only the hits that can reach it) against the
    fp64 oracle on whole grids: T1 on every cell; its peaks equal the dense kernel's up to T4 near-ties."""
    if model_shape is None:
        cfg = C.CONFIGS[name]
        b = G.make_batch(cfg, ev)
        nodes = G.axis_nodes(cfg)
        sigma, model = cfg.sigma, cfg.model
    else:
        model, shape = model_shape
        b = synthetic_batch(model, ev, seed=5)
        nodes = [np.linspace(lo, hi, n).astype(np.float32) for (lo, hi), n in
                 zip([(-0.3, 0.3), (-0.3, 0.3), (-150.0, 150.0)], shape)]
        sigma = 0.44
        cfg = C.Config(name="t", model=model, n_events=len(ev), seed=0, n_tracks=0, sigma=sigma)
    g = gpu_grid(b, cfg, nodes, algo=R.retina.GRID_TENSOR_F16_CULLED)
    ref = ora.grid(model, b.offsets, b.hits, nodes, sigma)
    ok, worst = PU.t1_response(g, ref)
    assert ok, worst
    P = len(nodes)
    for e in range(g.shape[0]):
        idx, _, cnt = R.retina_find_peaks(dev(g[e:e + 1]), P, 2.5, 1 << 16)
        okp, nd, ne = PU.t4_peak_sets(idx.cpu().numpy()[0], int(cnt[0]), ref[e], P, 2.5, 1 << 16)
        assert okp, (e, nd, ne)
    PU.report(f"T1/T4 culled grid {name}", t1_worst=worst)


@pytest.mark.parametrize("name,n_ev", [("cfg3", 160), ("cfg4", 12)])
def test_culled_tensor_grid_many_tiles_per_cluster(name, n_ev):
    """Many tiles per persistent CTA pair (the per-tile windows, the 'last chunk' flags and the ring
    phases carried from tile to tile): the culled grid equals the dense one within 2e-5 relative
    (each within 1e-5 of fp64, T1) on every cell of every event."""
    cfg = C.CONFIGS[name]
    b = G.make_batch(cfg, range(n_ev))
    nodes = G.axis_nodes(cfg)
    gd = gpu_grid(b, cfg, nodes, algo=R.retina.GRID_TENSOR_F16)
    gc = gpu_grid(b, cfg, nodes, algo=R.retina.GRID_TENSOR_F16_CULLED)
    err = np.abs(gc.astype(np.float64) - gd) / (2e-5 * np.maximum(gd.astype(np.float64), 1e-6))
    assert err.max() <= 1.0, err.max()
    # the pair counters: every pair for the dense kernel, the kept (tile, hit) pairs for the culled one
    ev = events_of(b)
    dn = [dev(n) for n in nodes]
    pd = torch.zeros(1, dtype=torch.int64, device=DEV)
    pc = torch.zeros(1, dtype=torch.int64, device=DEV)
    R.retina_grid_response(ev, cfg.model, cfg.sigma, dn, algorithm=R.retina.GRID_TENSOR_F16, pairs_evaluated=pd)
    R.retina_grid_response(ev, cfg.model, cfg.sigma, dn, algorithm=R.retina.GRID_TENSOR_F16_CULLED,
                           pairs_evaluated=pc)
    torch.cuda.synchronize()
    assert int(pd.item()) == int(b.offsets[-1]) * int(np.prod([len(n) for n in nodes]))
    assert 0 < int(pc.item()) <= int(pd.item())
    PU.report(f"culled grid {name} x{n_ev}", pairs_all=int(pd.item()), pairs_contracted=int(pc.item()),
              frac=int(pc.item()) / int(pd.item()))


@pytest.mark.parametrize("tensor", TENSORS)
def test_T1_tensor_grid_cfg4_full_size_sampled_and_peaks(tensor):
    cfg = C.CFG4
    b = G.make_batch(cfg, [0, 1])
    nodes = G.axis_nodes(cfg)
    g = gpu_grid(b, cfg, nodes, algo=tensor)
    rng = np.random.default_rng(12)
    pick = [np.unique(np.concatenate([np.sort(rng.choice(len(n), 12, replace=False)), [0, len(n) - 1]]))
            for n in nodes]
    ref = ora.grid(cfg.model, b.offsets, b.hits, [n[p] for n, p in zip(nodes, pick)], cfg.sigma)
    ok, worst = PU.t1_response(sub_lattice(g, pick), ref)
    assert ok, worst
    gs = gpu_grid(b, cfg, nodes, algo=R.retina.GRID_SEPARABLE)
    err = np.abs(g.astype(np.float64) - gs) / (2e-5 * np.maximum(gs, 1e-6))
    assert err.max() <= 1.0, err.max()
    idx, _, cnt = R.retina_find_peaks(dev(g[:1]), 3, cfg.peak_threshold, cfg.peak_capacity)
    ok, nd, ne = PU.t4_peak_sets(idx.cpu().numpy()[0], int(cnt[0]), gs[0].astype(np.float64), 3,
                                 cfg.peak_threshold, cfg.peak_capacity)
    assert ok, (nd, ne)


@pytest.mark.parametrize("model,z_ref", [(C.SLOPE2, 0.0), (C.SLOPE2, 17.5), (C.SLOPE3, 0.0)])
def test_multistart_and_newton_streaming_hits(model, z_ref):
    """Events larger than the shared-memory hit stage (no size hint -> 4096-hit stage, 5000-hit
    event) stream their hits through the double buffer on every pass; results must equal the
    resident path bit for bit (same hit order, same arithmetic)."""
    b = synthetic_batch(model, [5000, 300, 0], seed=21)
    P = 3 if model == C.SLOPE3 else 2
    lo = (-0.3, -0.3, -150.0)[:P]
    hi = (0.3, 0.3, 150.0)[:P]
    rng = np.random.default_rng(4)
    seeds = np.stack([rng.uniform(l, h, (3, 700)) for l, h in zip(lo, hi)], axis=-1).astype(np.float32)
    sigma = 0.44
    step = C.step_slope3(sigma) if model == C.SLOPE3 else C.step_slope2(sigma)
    res = []
    for hint in (True, False):
        ev = events_of(b, z_ref, hint)
        a = R.retina_multistart_optimize(ev, model, sigma, dev(seeds), 5, step * 10, lo, hi)
        n = R.retina_multistart_newton(ev, model, dev(seeds), [sigma * 3, sigma], [step * 9, step], sigma, 8, lo, hi)
        torch.cuda.synchronize()
        res.append([x.cpu().numpy() for x in a + n])
    for x, y in zip(*res):
        assert np.array_equal(x, y)
    # and the streaming result is right: R at theta_out vs the oracle
    th, Rr = res[1][0], res[1][1]
    for s in range(0, 700, 97):
        r, _, _ = ora.point(model, b.event_hits(0), th[0, s].astype(np.float64), sigma, z_ref=z_ref)
        assert PU.t1_response(Rr[0, s], r)[0]


def test_multistart_slope3_compact_stage_and_many_planes():
    """SLOPE3 events too large for six float4 stages per SM are staged compactly ((x, y) pairs + a
    plane table): a dense 26-plane event (compact path) and an event whose hits all have distinct
    z (more than 64 planes: the compact attempt falls back to the float4 stage, streaming) both
    match the oracle: states (T5, 20 small steps) and R at theta_out (T1)."""
    rng = np.random.default_rng(8)
    hs = []
    for n, planes in ((6000, True), (3000, False)):
        h = np.zeros((n, 4), np.float32)
        z = rng.choice(C.VELO_PLANES, n) if planes else rng.uniform(0.0, 750.0, n)
        t = rng.uniform(-0.3, 0.3, (n, 2))
        h[:, 0] = t[:, 0] * z + rng.normal(0, 0.5, n)
        h[:, 1] = t[:, 1] * z + rng.normal(0, 0.5, n)
        h[:, 2] = z
        hs.append(h[np.argsort(h[:, 2], kind="stable")])
    off = np.array([0, len(hs[0]), len(hs[0]) + len(hs[1])], np.int32)
    hits = np.concatenate(hs)
    lo, hi = (-0.3, -0.3, -150.0), (0.3, 0.3, 150.0)
    seeds = np.stack([rng.uniform(l, u, (2, 600)) for l, u in zip(lo, hi)], axis=-1).astype(np.float32)
    sigma = 0.88
    step = C.step_slope3(sigma)
    ev = R.Events.from_numpy(off, hits)
    th, Rr, _ = R.retina_multistart_optimize(ev, C.SLOPE3, sigma, dev(seeds), 20, step, lo, hi)
    torch.cuda.synchronize()
    th, Rr = th.cpu().numpy(), Rr.cpu().numpy()
    rth, _, _ = ora.multistart(C.SLOPE3, off, hits, seeds, sigma, 20, step, lo, hi, want_grad=False)
    ranges = np.array(hi) - np.array(lo)
    assert np.max(np.abs(th - rth) / ranges) <= 1e-3
    for e in range(2):
        for s in range(0, 600, 61):
            r, _, _ = ora.point(C.SLOPE3, hits[off[e]:off[e + 1]], th[e, s].astype(np.float64), sigma)
            assert PU.t1_response(Rr[e, s], r)[0], (e, s)


@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfg4"])
def test_pipeline_cuda_graph_replay_bitwise(name):
    """The whole pass captured in a CUDA graph and replayed gives the eager results bit for bit;
    replaying after new inputs are copied into the batch buffers recomputes them."""
    from paper_1709_08610_b200.pipeline import RetinaPipeline, upload
    import bench
    cfg = C.CONFIGS[name]
    if name == "cfg2":
        cfg = cfg.replace(axes=((-0.3, 0.3, 64), (-0.3, 0.3, 64)))
    if name == "cfg4":
        cfg = cfg.replace(n_seeds=1024)
    E = 3
    b = G.make_batch(cfg, range(E))
    sd = G.make_seeds(cfg, range(E))
    spec = bench.make_spec(cfg)
    pipe = RetinaPipeline(spec, E, chunk_events=2)
    db = upload(b.offsets, b.hits, sd)
    pipe.run(db)
    torch.cuda.synchronize()
    outs = [pipe.peak_cnt, pipe.peak_idx, pipe.peak_theta, pipe.theta, pipe.resp, pipe.t_count, pipe.t_seed]
    eager = [x[:E].clone() for x in outs]
    for x in outs:
        x.zero_()
    g = pipe.capture(db)
    for x in outs:
        x.zero_()
    g.replay()
    torch.cuda.synchronize()
    pc, tc = eager[0].cpu().numpy(), eager[5].cpu().numpy()
    assert torch.equal(outs[0][:E], eager[0]) and torch.equal(outs[5][:E], eager[5])
    assert torch.equal(outs[3][:E], eager[3]) and torch.equal(outs[4][:E], eager[4])
    for e in range(E):  # list entries past the true counts are unspecified
        k = min(int(pc[e]), spec.peak_capacity)
        assert torch.equal(outs[1][e, :k], eager[1][e, :k]) and torch.equal(outs[2][e, :k], eager[2][e, :k])
        k = min(int(tc[e]), spec.track_capacity)
        assert torch.equal(outs[6][e, :k], eager[6][e, :k])
    # new inputs into the same device buffers: the replay follows them
    b2 = G.make_batch(cfg, range(E, 2 * E))
    if b2.n_hits <= db.hits.shape[0]:
        db.offsets.copy_(torch.from_numpy(b2.offsets))
        db.hits[:b2.n_hits].copy_(torch.from_numpy(b2.hits))
        g.replay()
        torch.cuda.synchronize()
        ref = RetinaPipeline(spec, E, chunk_events=2)
        ref.run(upload(b2.offsets, b2.hits, sd))
        torch.cuda.synchronize()
        assert torch.equal(pipe.theta[:E], ref.theta[:E]) and torch.equal(pipe.peak_cnt[:E], ref.peak_cnt[:E])


def test_many_events_launch_chunking():
    """More than 65,535 events: the launchers split gridDim.y; tiny grid so the test stays small."""
    E = 70_000
    rng = np.random.default_rng(5)
    counts = rng.integers(0, 4, E)
    off = np.zeros(E + 1, np.int32)
    off[1:] = np.cumsum(counts)
    hits = np.zeros((int(off[-1]), 4), np.float32)
    hits[:, 2] = rng.choice(C.VELO_PLANES[1:], len(hits))
    hits[:, 0] = rng.uniform(-0.3, 0.3, len(hits)) * hits[:, 2]
    hits[:, 1] = rng.uniform(-0.3, 0.3, len(hits)) * hits[:, 2]
    b = G.EventBatch(offsets=off, hits=hits, event_ids=np.arange(E), truth=[None] * E, n_track_hits=counts)
    nodes = [np.linspace(-0.3, 0.3, 3).astype(np.float32)] * 2
    cfg = C.Config(name="t", model=C.SLOPE2, n_events=E, seed=0, n_tracks=0, sigma=0.44)
    for algo in (R.retina.GRID_DIRECT, R.retina.GRID_SEPARABLE, *TENSORS):
        g = gpu_grid(b, cfg, nodes, algo=algo)
        sel = np.r_[0:5, 65530:65540, E - 5:E]
        sub = G.EventBatch(offsets=np.concatenate([[0], np.cumsum(counts[sel])]).astype(np.int32),
                           hits=np.concatenate([hits[off[e]:off[e + 1]] for e in sel]), event_ids=sel,
                           truth=[None] * len(sel), n_track_hits=counts[sel])
        ref = ora.grid(C.SLOPE2, sub.offsets, sub.hits, nodes, 0.44)
        ok, worst = PU.t1_response(g[sel], ref)
        assert ok, (algo, worst)
    seeds = np.zeros((E, 3, 2), np.float32)
    seeds[:, :, 0] = rng.uniform(-0.3, 0.3, (E, 3))
    th, Rr, _ = R.retina_multistart_optimize(events_of(b), C.SLOPE2, 0.44, dev(seeds), 0, 0.0, (-.3, -.3), (.3, .3))
    torch.cuda.synchronize()
    e = E - 1
    for s in range(3):
        r, _, _ = ora.point(C.SLOPE2, hits[off[e]:off[e + 1]], seeds[e, s].astype(np.float64), 0.44)
        assert PU.t1_response(float(Rr[e, s]), r)[0]


# --------------------------------------------------------------------------- T1/T3/T4 at full BASELINE size vs fp64
def _t4_restricted(gpu_idx, ref_idx, tie_mask, keep):
    """Symmetric difference of two sets of flat indices restricted by `keep` (flat bool mask),
    excusing oracle near-tie cells.  Returns (n_diff, n_excused, unexcused list)."""
    a = {int(c) for c in gpu_idx if keep[c]}
    b = {int(c) for c in ref_idx if keep[c]}
    diff = a ^ b
    bad = [c for c in diff if not tie_mask[c]]
    return len(diff), len(diff) - len(bad), bad


def test_T1_T3_T4_full_cfg3_events_vs_fp64_oracle():
    """Whole 1024 x 1024 cfg3 grids (steps ii-iii; SURVEY §8(d) parity sample)
    from the default grid kernel, compared with the full fp64 oracle grid: T1 on every cell, T3
    bit-exact peaks both ways (GPU grid and oracle grid rounded to fp32), T4 peak sets from the
    fp32 and fp64 grids equal up to oracle near-ties, at R0 = 2.5 and R0 = 0."""
    cfg = C.CFG3
    ev = [0, 4999, 9998]
    b = G.make_batch(cfg, ev)
    nodes = G.axis_nodes(cfg)
    g = gpu_grid(b, cfg, nodes)                                     # AUTO: the bench's kernel
    ref = ora.grid(cfg.model, b.offsets, b.hits, nodes, cfg.sigma)  # 3 x 1.05e9 pairs in fp64
    ok, worst = PU.t1_response(g, ref)
    assert ok, worst
    stats = {"cells": int(ref.size), "t1_worst": worst}
    for thr, cap in ((cfg.peak_threshold, cfg.peak_capacity), (0.0, 1 << 20)):
        idx, val, cnt = R.retina_find_peaks(dev(g), 2, thr, cap)
        r32 = ref.astype(np.float32)
        idx2, val2, cnt2 = R.retina_find_peaks(dev(r32), 2, thr, cap)
        torch.cuda.synchronize()
        idx, cnt, idx2, cnt2 = idx.cpu().numpy(), cnt.cpu().numpy(), idx2.cpu().numpy(), cnt2.cpu().numpy()
        for grid32, i_, c_ in ((g, idx, cnt), (r32, idx2, cnt2)):         # T3 both ways
            ri, rv, rc = ora.peaks(grid32.astype(np.float64), 2, thr, cap)
            assert np.array_equal(c_, rc)
            for e in range(len(ev)):
                assert np.array_equal(i_[e, :min(rc[e], cap)], ri[e, :min(rc[e], cap)])
        n_diff = n_exc = n_pk = 0
        for e in range(len(ev)):
            assert cnt[e] <= cap
            ok, nd, ne = PU.t4_peak_sets(idx[e], cnt[e], ref[e], 2, thr, cap)
            assert ok, (e, thr, nd, ne)
            n_diff, n_exc, n_pk = n_diff + nd, n_exc + ne, n_pk + int(cnt[e])
        stats[f"R0={thr}"] = {"peaks": n_pk, "sym_diff": n_diff, "excused_near_tie": n_exc}
        if thr > 0:
            assert n_pk > 20   # 52 strict maxima with R >= 2.5 in these three events
    PU.report("T1/T3/T4 cfg3 full 1024^2 x 3 events", **stats)


def test_T1_T4_full_cfg4_slab_vs_fp64_oracle():
    """cfg4 (256^3 SLOPE3): the default grid kernel's full grid, compared on a 256 x 256 x 34 slab
    of z0 nodes around a true vertex with the fp64 oracle: T1 on every slab cell; T4 (3 x 3 x 3
    strict maxima from the fp32 and fp64 grids) on the slab's 32 interior z0 planes, where every
    cell's 26 neighbours lie inside the slab."""
    cfg = C.CFG4
    nodes = G.axis_nodes(cfg)
    stats = {}
    for e_id in (0, 1):
        b = G.make_batch(cfg, [e_id])
        g = gpu_grid(b, cfg, nodes)[0]
        z0 = float(b.truth[0][0, 2])
        kc = int(np.clip(np.argmin(np.abs(nodes[2] - z0)), 17, len(nodes[2]) - 18))
        k0, k1 = kc - 17, kc + 17                                     # slab node range [k0, k1)
        ref = ora.grid(cfg.model, b.offsets, b.hits, [nodes[0], nodes[1], nodes[2][k0:k1]], cfg.sigma)[0]
        ok, worst = PU.t1_response(g[k0:k1], ref)                     # z0 planes k0..k1-1 (Z37)
        assert ok, (e_id, worst)
        cap = 1 << 20
        for thr in (cfg.peak_threshold, 0.0):
            idx, _, cnt = R.retina_find_peaks(dev(g[None]), 3, thr, cap)
            torch.cuda.synchronize()
            gi = idx.cpu().numpy()[0, :int(cnt[0])]
            ci = np.array(np.unravel_index(gi, g.shape)).T                # (l, i, j)
            inside = (ci[:, 0] >= k0 + 1) & (ci[:, 0] < k1 - 1)
            # GPU peaks in the interior planes, as flat indices of the slab
            gpu_slab = np.ravel_multi_index((ci[inside, 0] - k0, ci[inside, 1], ci[inside, 2]), ref.shape)
            ri, _, rc = ora.peaks(ref[None], 3, thr, cap)
            keep = np.zeros(ref.shape, bool)
            keep[1:-1] = True
            tie = PU.near_tie_cells(ref, 3, thr).ravel()
            nd, ne, bad = _t4_restricted(gpu_slab, ri[0, :rc[0]], tie, keep.ravel())
            assert not bad, (e_id, thr, nd, ne, bad[:5])
            stats[f"event {e_id} R0={thr}"] = {"peaks_interior": int(inside.sum()), "sym_diff": nd,
                                               "excused_near_tie": ne}
        stats[f"event {e_id} t1_worst"] = worst
    PU.report("T1/T4 cfg4 256x256x34 slab", **stats)


def test_concurrent_host_threads_on_two_streams_bitwise():
    """include/retina.h promises calls are safe from several host threads on different streams
    (no global mutable state besides the once-per-kernel shared-memory attribute cache): two
    threads, each on its own stream, run cfg2 multi-start + merge and a cfg1 grid + peaks (first
    calls of their kernels included, so the attribute cache is filled concurrently); every result
    equals the serial run bit for bit."""
    import threading
    cfg, c1 = C.CFG2, C.CFG1
    jobs = []
    for k in range(2):
        b = G.make_batch(cfg, [2 * k, 2 * k + 1])
        sd = dev(G.make_seeds(cfg, [2 * k, 2 * k + 1], n_seeds=2048))
        b1 = G.make_batch(c1, [k])
        jobs.append((events_of(b), sd, events_of(b1), [dev(n) for n in G.axis_nodes(c1)]))

    def work(job, stream=None):
        ev, sd, ev1, nodes = job
        with torch.cuda.stream(stream) if stream is not None else torch.cuda.stream(torch.cuda.current_stream()):
            out = R.retina_multistart_optimize(ev, cfg.model, cfg.sigma, sd, cfg.n_iters, cfg.step, cfg.box_lo,
                                               cfg.box_hi, stream=stream)
            m = R.retina_merge_tracks(out[0], out[1], cfg.merge_radius, cfg.track_threshold, 256, stream=stream)
            g = R.retina_grid_response(ev1, c1.model, c1.sigma, nodes, stream=stream,
                                       algorithm=R.retina.GRID_TENSOR_F16_SINGLE)
            p = R.retina_find_peaks(g, 2, c1.peak_threshold, 4096, stream=stream)
        return list(out) + list(m) + [g] + list(p)

    results = [None, None]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]

    def thread_main(k):
        torch.cuda.set_device(0)
        results[k] = work(jobs[k], streams[k])
        streams[k].synchronize()

    ts = [threading.Thread(target=thread_main, args=(k,)) for k in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    torch.cuda.synchronize()
    for k in range(2):
        serial = work(jobs[k])
        torch.cuda.synchronize()
        a, b = results[k], serial
        for i in (0, 1, 2, 7, 8, 11):  # theta, R, grad, track_count, grid, peak_count: whole tensors
            assert torch.equal(a[i], b[i]), i
        for e in range(a[7].shape[0]):  # list entries up to the true counts
            kt = min(int(a[7][e]), 256)
            for i in (3, 4, 5, 6):
                assert torch.equal(a[i][e, :kt], b[i][e, :kt])
        for e in range(a[11].shape[0]):
            kp = min(int(a[11][e]), 4096)
            for i in (9, 10):
                assert torch.equal(a[i][e, :kp], b[i][e, :kp])
