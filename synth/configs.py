"""BASELINE.json configs cfg0..cfg4 with every reading made explicit.

Readings (DESIGN.md §3 lists them with their justification; ids follow
SURVEY.md §8(c) Z1..Z20):

* Z1  "config-1 geometry" = configs[1] (0-based): 26 planes at z = 30 p mm.
* Z2  sigma = grid step in slope x z_mid, z_mid = 375 mm (middle of [0, 750]).
* Z3  cfg2 inherits cfg1's sigma, cfg3 multi-start uses cfg3's grid sigma,
      cfg4 applies Z2 to its tx step.
* Z4  node tables = fp32(lo + i (hi - lo)/(n - 1)) computed in fp64 (inclusive
      linspace); cfg4's z0 table is additionally snapped to multiples of
      2^-14 mm.
* Z5  cfg0 sigma = alpha step = 1/199.
* Z6  peaks: strict local max over existing 3^P - 1 neighbours, R >= R0,
      R0 = 2.5 for the physics list, 0 for the integer (bit-exact) tests.
* Z7  fixed step eta = sigma^2 / (2 lambda_max(sum_p J_p^T J_p)).
* Z8  seeds i.i.d. uniform on the prior box.
* Z9  merge radius = 1e-3 x axis range (Chebyshev, per axis).
* Z10 merge threshold R(theta^n) >= 5.
* Z11 noise = round(0.1 n_track_hits), plane uniform, (x, y) area-uniform on
      the annulus 5 < r < 40 mm.
* Z12 hit counts follow the stated generation rules (realised ~1,000 / ~2,000
      hits for cfg3 / cfg4); the "dense" variant drops the r-cut.
* Z13 forward tracks only (z_p > z0), p_hit = 1, smear N(0, 0.012 mm) per
      coordinate, acceptance on the true intersection, hits sorted by z.
* Z14 cfg3's 2-parameter grid keeps the pattern origin at z_ref = 0.
* Z15 cfg3/cfg4 multi-start inherit cfg2's 50 iterations, R0 = 5, 1e-3 range.
* Z16 cfg0 noise x uniform over the integer planes {1..10}, y ~ U[-6, 6].

Nothing here evaluates the response: only geometry constants and the step
size rule (a property of the plane positions, not of any event).
"""
from __future__ import annotations

import dataclasses
from typing import Tuple

import numpy as np

LINE2D, SLOPE2, SLOPE3 = 0, 1, 2
MODEL_P = {LINE2D: 2, SLOPE2: 2, SLOPE3: 3}
MODEL_NAME = {LINE2D: "line2d", SLOPE2: "slope2", SLOPE3: "slope3"}

# VELO-like geometry of BASELINE configs[1] (reading Z1): 26 planes over [0, 750] mm.
VELO_PLANES = 30.0 * np.arange(26)
VELO_R_MIN, VELO_R_MAX = 5.0, 40.0
VELO_SMEAR = 0.012
Z_MID = 375.0  # Z2

# 2-D toy of BASELINE configs[0]
TOY_PLANES = np.arange(1, 11, dtype=np.float64)
TOY_SMEAR = 0.01


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    model: int
    n_events: int
    seed: int
    # event generation
    n_tracks: int                 # fixed count, or Poisson mean if poisson_tracks
    poisson_tracks: bool = False
    z0_sigma: float = 0.0         # vertex z spread (mm); 0 = origin
    dense: bool = False           # Z12 variant: no acceptance cut
    # grid path
    axes: Tuple[Tuple[float, float, int], ...] = ()
    snap_last_axis: float = 0.0   # Z4: snap last-axis nodes to this quantum (0 = none)
    sigma: float = 1.0
    peak_threshold: float = 2.5
    peak_capacity: int = 4096
    # multi-start path
    n_seeds: int = 0
    n_iters: int = 0
    step: float = 0.0
    box_lo: Tuple[float, ...] = ()
    box_hi: Tuple[float, ...] = ()
    merge_radius: Tuple[float, ...] = ()
    track_threshold: float = 5.0
    track_capacity: int = 1024
    z_ref: float = 0.0

    @property
    def P(self) -> int:
        return MODEL_P[self.model]

    @property
    def n_units(self) -> int:
        return int(np.prod([a[2] for a in self.axes])) if self.axes else 0

    def replace(self, **kw) -> "Config":
        return dataclasses.replace(self, **kw)


def sigma_from_step(lo: float, hi: float, n: int, z_mid: float = Z_MID) -> float:
    """Z2: sigma = (grid step in slope) x z_mid, mapping the step into mm."""
    return (hi - lo) / (n - 1) * z_mid


def step_slope2(sigma: float, planes=VELO_PLANES) -> float:
    """Z7 for SLOPE2 with z_ref = 0: J_p = -z_p I, lambda_max = sum_p z_p^2."""
    lam = float(np.sum(np.asarray(planes, np.float64) ** 2))
    return sigma * sigma / (2.0 * lam)


def step_slope3(sigma: float, z0_max: float = 150.0, t_max: float = 0.3,
                planes=VELO_PLANES) -> float:
    """Z7 for SLOPE3: trace bound of sum_p J_p^T J_p over the prior box,
    J_p = [[-d, 0, tx], [0, -d, ty]], d = z_p - z0, |z0| <= 150, |t| <= 0.3."""
    d = np.asarray(planes, np.float64) + z0_max
    lam = float(np.sum(2.0 * d * d + 2.0 * t_max * t_max))
    return sigma * sigma / (2.0 * lam)


def step_line2d(sigma: float, planes=TOY_PLANES) -> float:
    """Z7 for LINE2D: J_p = [-x_p, -1]; lambda_max of [[sum x^2, sum x], [sum x, n]]."""
    x = np.asarray(planes, np.float64)
    m = np.array([[np.sum(x * x), np.sum(x)], [np.sum(x), float(len(x))]])
    lam = float(np.linalg.eigvalsh(m).max())
    return sigma * sigma / (2.0 * lam)


_S1 = sigma_from_step(-0.3, 0.3, 512)
_S3 = sigma_from_step(-0.3, 0.3, 1024)
_S4 = sigma_from_step(-0.3, 0.3, 256)

CFG0 = Config(
    name="cfg0", model=LINE2D, n_events=1, seed=0, n_tracks=5,
    axes=((-0.5, 0.5, 200), (-1.0, 1.0, 200)), sigma=1.0 / 199.0,  # Z5
    n_seeds=256, n_iters=0, step=step_line2d(1.0 / 199.0),
    box_lo=(-0.5, -1.0), box_hi=(0.5, 1.0),
    merge_radius=(1e-3, 2e-3), track_threshold=2.5,
)
CFG1 = Config(
    name="cfg1", model=SLOPE2, n_events=1, seed=1, n_tracks=100,
    axes=((-0.3, 0.3, 512), (-0.3, 0.3, 512)), sigma=_S1,
)
CFG2 = Config(
    name="cfg2", model=SLOPE2, n_events=200, seed=2, n_tracks=150, sigma=_S1,
    n_seeds=4096, n_iters=50, step=step_slope2(_S1),
    box_lo=(-0.3, -0.3), box_hi=(0.3, 0.3), merge_radius=(6e-4, 6e-4),
)
CFG3 = Config(
    name="cfg3", model=SLOPE2, n_events=10_000, seed=3, n_tracks=150, poisson_tracks=True,
    z0_sigma=50.0, axes=((-0.3, 0.3, 1024), (-0.3, 0.3, 1024)), sigma=_S3,
    n_seeds=8192, n_iters=50, step=step_slope2(_S3),
    box_lo=(-0.3, -0.3), box_hi=(0.3, 0.3), merge_radius=(6e-4, 6e-4),
)
CFG4 = Config(
    name="cfg4", model=SLOPE3, n_events=1_000, seed=4, n_tracks=300, z0_sigma=50.0,
    axes=((-0.3, 0.3, 256), (-0.3, 0.3, 256), (-150.0, 150.0, 256)),
    snap_last_axis=2.0 ** -14, sigma=_S4, peak_capacity=8192,
    n_seeds=16384, n_iters=50, step=step_slope3(_S4),
    box_lo=(-0.3, -0.3, -150.0), box_hi=(0.3, 0.3, 150.0),
    merge_radius=(6e-4, 6e-4, 0.3), track_capacity=2048,
)

CONFIGS = {c.name: c for c in (CFG0, CFG1, CFG2, CFG3, CFG4)}


def get_config(name: str, **overrides) -> Config:
    cfg = CONFIGS[name]
    return cfg.replace(**overrides) if overrides else cfg


def describe(cfg: Config) -> dict:
    d = dataclasses.asdict(cfg)
    d["model"] = MODEL_NAME[cfg.model]
    d["P"] = cfg.P
    return d


# ---------------------------------------------------------------------------------------------
# NEXT #1: the paper's own update.  Readings:
# Z22 the schedule sigma = 0.3, 0.175, 0.05 (q = 3) is applied as RATIOS to the config's sigma,
#     which is the last (finest) value: sigma_j = sigma_cfg x (6, 3.5, 1); final R at sigma_cfg.
# Z23 Truncated Newton = conjugate gradients on (-H) p = grad R, <= P iterations, stopped at
#     non-positive curvature.
# Z24 the negative-curvature fallback at the first CG iteration is the fixed-step ascent step
#     of reading Z7 at sigma_j: p = eta_j grad R, eta_j = sigma_j^2 / (2 lambda_max).
# Z25 Armijo backtracking on R, c1 = 1e-4, alpha = 1, 1/2, ..., at most 8 halvings
#     (SPEC.md:396), trial points clamped to the prior box; no accepted trial = no move.
PAPER_SIGMA_SCHEDULE = (0.3, 0.175, 0.05)


def newton_schedule(cfg: Config):
    """(sigmas, etas, final_sigma, max_halvings) for the Truncated-Newton path of `cfg`."""
    ratios = [s / PAPER_SIGMA_SCHEDULE[-1] for s in PAPER_SIGMA_SCHEDULE]
    sigmas = [cfg.sigma * r for r in ratios]
    if cfg.model == SLOPE3:
        etas = [step_slope3(s) for s in sigmas]
    elif cfg.model == SLOPE2:
        etas = [step_slope2(s) for s in sigmas]
    else:
        etas = [step_line2d(s) for s in sigmas]
    return sigmas, etas, cfg.sigma, 8
