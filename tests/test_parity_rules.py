"""CPU checks of the parity comparators' oracle-side rules (tests/parity_util.py): the rules
must excuse exactly what they name, so they are exercised here on oracle-made "GPU" results."""
import numpy as np

from oracle import oracle as ora
from synth import configs as C
from synth import events as G
from tests import parity_util as PU


def _newton_case(n_seeds=64):
    cfg = C.CFG2
    b = G.make_batch(cfg, [0])
    seeds = G.make_seeds(cfg, [0], n_seeds=n_seeds)
    sig, eta, fsig, mh = C.newton_schedule(cfg)
    return cfg, b, seeds, sig, eta, fsig, mh


def test_flip_rule_finds_planted_near_tie_flips_and_nothing_else():
    cfg, b, seeds, sig, eta, fsig, mh = _newton_case()
    ranges = np.array(cfg.box_hi, np.float64) - np.array(cfg.box_lo, np.float64)
    th, R, _, m, ne, log = ora.newton(cfg.model, b.offsets, b.hits, seeds, sig, eta, fsig, mh, cfg.box_lo,
                                      cfg.box_hi, want_margin=True, want_evals=True, log_len=128)
    # "GPU" = the oracle with the smallest-margin near-tie decision of each seed flipped (when it
    # has one) -- a result the rule must attribute
    flip = np.zeros((1, seeds.shape[1], 128), np.uint8)
    planted = []
    for s in range(seeds.shape[1]):
        k = [k for k in np.argsort(log[0, s]) if 0 <= log[0, s, k] <= 1e-4]
        if k:
            flip[0, s, k[0]] = 1
            planted.append(s)
    assert len(planted) >= 8
    th2, _, _, ne2, _ = ora.newton(cfg.model, b.offsets, b.hits, seeds, sig, eta, fsig, mh, cfg.box_lo, cfg.box_hi,
                                want_evals=True, flip=flip, log_len=128)
    changed = [s for s in planted if ne2[0, s] != ne[0, s] or np.any(np.abs(th2[0, s] - th[0, s]) > 1e-3 * ranges)]
    assert changed, "no planted flip changed an outcome"
    ok, nflips = PU.newton_flip_explains(cfg.model, cfg.box_lo, cfg.box_hi, b.event_hits(0), seeds[0, changed],
                                         th2[0, changed], ne2[0, changed], ranges, sig, eta, fsig, mh)
    assert ok.all() and np.all(nflips >= 1)
    # a result no set of near-tie flips can produce (the end point moved by 2e-3 x range) is not excused
    fake = th[0, :8] + 2e-3 * ranges
    ok, _ = PU.newton_flip_explains(cfg.model, cfg.box_lo, cfg.box_hi, b.event_hits(0), seeds[0, :8], fake,
                                    ne[0, :8], ranges, sig, eta, fsig, mh, max_runs=32)
    assert not ok.any()


def test_t6_rules_excuse_only_what_they_name():
    ranges = np.array([0.6, 0.6])
    radius = np.array([6e-4, 6e-4])
    th = np.array([[0.0, 0.0], [0.0, 5e-4], [0.1, 0.1], [0.2, 0.2]])
    R = np.array([9.0, 8.0, 7.0, 6.0])
    # identical sides: nothing unmatched
    side = (th, R, np.array([0, 2, 3]), np.array([0, 0, 1, 2]))
    bad, cnt = PU.t6_tracks(side, side, ranges, radius, 5.0, lambda s: False)
    assert not bad and cnt["unmatched"] == 0
    # a missing track that is not near R0, not near the radius, with a non-sensitive member: reported
    other = (th, R, np.array([0, 2]), np.array([0, 0, 1, -1]))
    bad, cnt = PU.t6_tracks(side, other, ranges, radius, 5.0, lambda s: False)
    assert bad == [("gpu", 3)]
    # ... excused when all its members are sensitive
    bad, cnt = PU.t6_tracks(side, other, ranges, radius, 5.0, lambda s: s == 3)
    assert not bad and cnt["sensitive"] == 1
    # ... or when its leader's R is within 1e-5 of R0
    R2 = R.copy()
    R2[3] = 5.0 * (1 + 5e-6)
    bad, cnt = PU.t6_tracks((th, R2) + side[2:], (th, R2) + other[2:], ranges, radius, 5.0, lambda s: False)
    assert not bad and cnt["near_R0"] == 1
    # a second leader just outside the first leader's radius (binding axis within 1e-5 range)
    th3 = np.array([[0.0, 0.0], [0.0, 6e-4 + 3e-6], [0.1, 0.1]])
    R3 = np.array([9.0, 8.0, 7.0])
    a = (th3, R3, np.array([0, 1, 2]), np.array([0, 1, 2]))
    c = (th3, R3, np.array([0, 2]), np.array([0, 0, 1]))
    bad, cnt = PU.t6_tracks(a, c, ranges, radius, 5.0, lambda s: False)
    assert not bad and cnt["near_radius"] == 1
    # one-to-one: two GPU tracks within tolerance of ONE oracle track leave one unmatched
    th4 = np.array([[0.0, 0.0], [0.0, 7e-4], [0.3, 0.3]])
    g = (th4, np.array([9.0, 8.0, 7.0]), np.array([0, 1]), np.array([0, 1, -1]))
    r = (th4, np.array([9.0, 8.0, 7.0]), np.array([0]), np.array([0, 0, -1]))
    bad, cnt = PU.t6_tracks(g, r, ranges, radius, 5.0, lambda s: False)
    assert cnt["unmatched"] == 1 and bad == [("gpu", 1)]


def test_arithmetic_perturbation_is_fp32_sized_and_off_by_default():
    cfg, b, seeds, sig, eta, fsig, mh = _newton_case(16)
    a = ora.newton(cfg.model, b.offsets, b.hits, seeds, sig, eta, fsig, mh, cfg.box_lo, cfg.box_hi)
    z = ora.newton(cfg.model, b.offsets, b.hits, seeds, sig, eta, fsig, mh, cfg.box_lo, cfg.box_hi, perturb=0.0,
                   perturb_key=7)
    assert all(np.array_equal(x, y) for x, y in zip(a, z))
    p1 = ora.newton(cfg.model, b.offsets, b.hits, seeds, sig, eta, fsig, mh, cfg.box_lo, cfg.box_hi, perturb=1e-6,
                    perturb_key=1)
    p2 = ora.newton(cfg.model, b.offsets, b.hits, seeds, sig, eta, fsig, mh, cfg.box_lo, cfg.box_hi, perturb=1e-6,
                    perturb_key=2)
    assert not np.array_equal(p1[0], p2[0])                      # the key changes the perturbation
    ranges = np.array(cfg.box_hi) - np.array(cfg.box_lo)
    moved = np.max(np.abs(p1[0] - a[0]) / ranges, axis=2)
    assert np.median(moved) < 1e-6                               # fp32-sized for a typical seed
