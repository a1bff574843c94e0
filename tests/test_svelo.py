"""NEXT #2: sVELO generator, Eq. (3) budget, epsilon matching (CPU), and GPU
parity of the Truncated-Newton path on sVELO events."""
import math

import numpy as np
import pytest

from synth import configs as C
from synth import svelo as S
from tests import parity_util as PU
from tools import svelo_eval as EV


def test_generator_rules_and_determinism():
    cfg = S.SVELO
    for n in (50, 200):
        h, truth = S.make_svelo_event(n, 3)
        assert truth.shape == (n, 2)  # exactly n reconstructible tracks (Z31)
        assert np.all(np.diff(h[:, 2]) >= 0)
        assert set(np.unique(h[:, 2])) <= set(cfg.layers.astype(np.float32))
        r = np.hypot(h[:, 0], h[:, 1])
        assert np.all(r > cfg.r_inner - 0.1) and np.all(r < cfg.r_outer + 0.1)
        # true directions respect eta in [1, 6]: polar angle in [2 atan e^-6, 2 atan e^-1]
        polar = np.arctan(np.hypot(truth[:, 0], truth[:, 1]))
        assert polar.min() >= 2 * math.atan(math.exp(-6)) - 1e-12 and polar.max() <= cfg.max_polar + 1e-12
        h2, t2 = S.make_svelo_event(n, 3)
        assert np.array_equal(h, h2) and np.array_equal(truth, t2)
    # each reconstructible track leaves >= 2 hits within 5 sigma of its line
    h, truth = S.make_svelo_event(60, 9)
    for tx, ty in truth:
        d = np.hypot(h[:, 0] - tx * h[:, 2], h[:, 1] - ty * h[:, 2])
        assert np.sum(d < 5 * cfg.smear) >= cfg.n_min


def test_eta_and_noise_distributions():
    rng = np.random.default_rng(0)
    tx, ty = S.draw_prior(rng, 200_000)
    polar = np.arctan(np.hypot(tx, ty))
    eta = -np.log(np.tan(polar / 2))
    hist, _ = np.histogram(eta, bins=10, range=(1, 6))
    assert np.all(np.abs(hist / len(eta) - 0.1) < 0.005)  # eta ~ U[1, 6]
    n_noise = []
    for e in range(200):
        h, truth = S.make_svelo_event(1, e)
        n_noise.append(len(h))
    assert abs(np.mean(n_noise) - 250 - 5) < 5  # Poisson(250) noise + one track's few hits


def test_eq3_budget_and_matching():
    # Eq. (3): n = alpha n_grid / (C0 q)
    assert EV.seed_budget(1 / 3, 900_000, C0=30, q=3) == 3333
    assert EV.seed_budget(0.1, 900_000, C0=30, q=3) == 1000
    t = math.tan(S.SVELO.max_polar)
    n_axis = int(math.ceil(2 * t / 1e-3)) + 1
    assert EV.grid_cells_for_resolution(1e-3) == n_axis * n_axis
    # angle between two lines through the origin: closed form for lines in the x-z plane
    a = math.atan(0.2)
    b = math.atan(0.2) + 7e-4
    assert abs(EV.angle_between(0.2, 0.0, math.tan(b), 0.0) - 7e-4) < 1e-15
    truth = np.array([[0.2, 0.0], [0.0, -0.1]])
    eff, m, n = EV.match_efficiency([math.tan(a + 9e-4), 0.0], [0.0, -0.1 + 2e-3], truth, 1e-3)
    assert (m, n) == (1, 2) and eff == 0.5
    # one-to-one: two candidates within eps of ONE truth give 1 match + 1 ghost; the closer one
    # takes it, so a second truth near the farther candidate can still match it
    two = [math.tan(a + 3e-4), math.tan(a + 8e-4)]
    assert EV.match_tracks(two, [0.0, 0.0], truth[:1], 1e-3) == (1, 0, 1)
    pair = np.array([[0.2, 0.0], [math.tan(a + 1.0e-3), 0.0]])
    assert EV.match_tracks(two, [0.0, 0.0], pair, 1e-3) == (2, 0, 0)
    assert EV.match_tracks([], [], truth, 1e-3) == (0, 2, 0)


@pytest.mark.gpu
def test_svelo_newton_gpu_vs_oracle():
    import torch

    import paper_1709_08610_b200 as R
    from oracle import oracle as ora
    cfg = S.SVELO
    b = S.make_svelo_batch(50, [0, 1])
    seeds = S.svelo_seeds(50, [0, 1], 512)
    t = math.tan(cfg.max_polar)
    sig = [0.3, 0.175, 0.05]
    eta = [C.step_slope2(s, planes=cfg.layers) for s in sig]
    ev = R.Events.from_numpy(b.offsets, b.hits)
    th, Rg, _ = R.retina_multistart_newton(ev, C.SLOPE2, torch.from_numpy(seeds).cuda(), sig, eta, 0.05, 8,
                                           (-t, -t), (t, t))
    torch.cuda.synchronize()
    th, Rg = th.cpu().numpy(), Rg.cpu().numpy()
    rth, rR, _, margin = ora.newton(C.SLOPE2, b.offsets, b.hits, seeds, sig, eta, 0.05, 8, (-t, -t), (t, t),
                                    want_margin=True)
    # T5n with its named oracle-side rules only (decision margin, fp32-size sensitivity)
    unexcused, st, _ = PU.t5n_states(C.SLOPE2, (-t, -t), (t, t), b, seeds, sig, eta, 0.05, 8, th, rth,
                                     np.array([2 * t, 2 * t]))
    PU.report("T5n sVELO E=2 S=512", **st)
    assert not unexcused, unexcused[:5]
    assert st["excused_frac"] <= 0.05, st
    # the merged candidates find most reconstructible tracks at this seed density
    tt, tr, ts, tz, tc = R.retina_merge_tracks(torch.from_numpy(th).cuda(), torch.from_numpy(Rg).cuda(),
                                               (1e-3, 1e-3), 1.5, 512)
    torch.cuda.synchronize()
    _, _, ots, _, otc = ora.merge(th.astype(np.float64), Rg.astype(np.float64), (1e-3, 1e-3), 1.5, 512)
    assert np.array_equal(tc.cpu().numpy(), otc)
