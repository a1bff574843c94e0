"""sVELO: the paper's simplified LHCb VELO model, NEXT #2 of SURVEY.md §8(f).

Seeded synthetic events only (no method arithmetic).  Every bulleted sVELO assumption of
PAPER.md:173-185 is a field of SveloConfig; the places the text is silent are readings
(Z26-Z31):

* Z26 layers: N_l = 20 disks "equally spaced within 700 mm along z" are placed at
      z_l = 700 (l + 1) / N_l mm, l = 0..19 (35 .. 700 mm; the interaction point is at the origin
      and a disk at z = 0 could not be hit outside its 8 mm inner radius).
* Z27 directions: eta ~ U[1, 6] gives the polar angle to the beam axis, theta_p = 2 atan(e^-eta)
      (PAPER.md:179); the transverse angle phi ~ U[0, 2 pi); all tracks go
      forward from the origin ("primary vertex").  In the kernels' SLOPE2 model the
      line is x = tx z, y = ty z with tx = tan(theta_p) cos(phi), ty = tan(theta_p) sin(phi); the
      paper's (theta, phi) of PAPER.md:189-194 is the same line family (tx = tan(theta)/cos(phi),
      ty = tan(phi) in its convention), so the search runs in slope space and converts at the end.
* Z28 a track interacts with each layer it crosses (8 < r < 42 mm at that z) with probability
      p_hit = 0.5; tracks with fewer than N_min = 2 hits are not reconstructible and
      their hits are kept as noise.
* Z29 measurement errors eps_x, eps_y ~ N(0, 1e-2) are standard deviations in mm.
* Z30 N_noise ~ Poisson(250) noise hits, each on a uniformly chosen layer, area-
      uniform on the 8 < r < 42 mm annulus.
* Z31 "number of reconstructible tracks varied between 50 and 350": an event is
      generated with exactly n_reco reconstructible tracks (tracks are drawn until n_reco have
      >= 2 hits; the non-reconstructible ones drawn on the way contribute their hits as noise).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Sequence

import numpy as np

from .events import EventBatch, _rng

STREAM_SVELO = 3


@dataclasses.dataclass(frozen=True)
class SveloConfig:
    n_layers: int = 20
    z_span: float = 700.0
    r_inner: float = 8.0
    r_outer: float = 42.0
    eta_lo: float = 1.0
    eta_hi: float = 6.0
    p_hit: float = 0.5
    n_min: int = 2
    smear: float = 1e-2
    noise_mean: float = 250.0
    seed: int = 17

    @property
    def layers(self) -> np.ndarray:
        return self.z_span * (np.arange(self.n_layers) + 1.0) / self.n_layers

    @property
    def max_polar(self) -> float:
        """Largest polar angle in the prior: eta = eta_lo."""
        return 2.0 * math.atan(math.exp(-self.eta_lo))


SVELO = SveloConfig()


def polar_from_eta(eta):
    """eta = -ln tan(theta/2)  <=>  theta = 2 atan(exp(-eta))."""
    return 2.0 * np.arctan(np.exp(-np.asarray(eta, np.float64)))


def slopes_from_direction(polar, phi):
    """Z27: forward line through the origin with polar angle `polar` and azimuth `phi`."""
    t = np.tan(np.asarray(polar, np.float64))
    return t * np.cos(phi), t * np.sin(phi)


def draw_prior(rng: np.random.Generator, n: int, cfg: SveloConfig = SVELO):
    """The physical track prior of PAPER.md:179-180 in slope coordinates (Z27)."""
    eta = rng.uniform(cfg.eta_lo, cfg.eta_hi, n)
    phi = rng.uniform(0.0, 2.0 * math.pi, n)
    return slopes_from_direction(polar_from_eta(eta), phi)


def make_svelo_event(n_reco: int, event_id: int, cfg: SveloConfig = SVELO):
    """One sVELO event with exactly n_reco reconstructible tracks (Z31).
    Returns (hits float32 [N, 4] sorted by z, truth slopes float64 [n_reco, 2])."""
    rng = _rng(cfg.seed, STREAM_SVELO, (int(n_reco) << 32) | int(event_id))
    z = cfg.layers
    xs, ys, zs, truth = [], [], [], []
    n_found = 0
    while n_found < n_reco:
        tx, ty = draw_prior(rng, 1, cfg)
        tx, ty = float(tx[0]), float(ty[0])
        r = math.hypot(tx, ty) * z
        cross = (r > cfg.r_inner) & (r < cfg.r_outer)
        hit = cross & (rng.random(len(z)) < cfg.p_hit)
        k = np.nonzero(hit)[0]
        hx = tx * z[k] + rng.normal(0.0, cfg.smear, len(k))
        hy = ty * z[k] + rng.normal(0.0, cfg.smear, len(k))
        xs.append(hx)
        ys.append(hy)
        zs.append(z[k])
        if len(k) >= cfg.n_min:
            truth.append((tx, ty))
            n_found += 1
    n_noise = int(rng.poisson(cfg.noise_mean))
    lay = rng.integers(0, len(z), n_noise)
    rr = np.sqrt(rng.uniform(cfg.r_inner ** 2, cfg.r_outer ** 2, n_noise))
    ph = rng.uniform(0.0, 2.0 * math.pi, n_noise)
    xs.append(rr * np.cos(ph))
    ys.append(rr * np.sin(ph))
    zs.append(z[lay])
    x = np.concatenate(xs)
    y = np.concatenate(ys)
    zz = np.concatenate(zs)
    order = np.argsort(zz, kind="stable")
    h = np.zeros((len(x), 4), np.float32)
    h[:, 0] = x[order]
    h[:, 1] = y[order]
    h[:, 2] = zz[order]
    return h, np.asarray(truth, np.float64).reshape(-1, 2)


def make_svelo_batch(n_reco: int, event_ids: Sequence[int], cfg: SveloConfig = SVELO) -> EventBatch:
    hs, truths = [], []
    for e in event_ids:
        h, t = make_svelo_event(n_reco, int(e), cfg)
        hs.append(h)
        truths.append(t)
    counts = np.array([len(h) for h in hs], np.int64)
    off = np.zeros(len(hs) + 1, np.int64)
    np.cumsum(counts, out=off[1:])
    return EventBatch(offsets=off.astype(np.int32), hits=np.ascontiguousarray(np.concatenate(hs)),
                      event_ids=np.asarray(list(event_ids), np.int64), truth=truths,
                      n_track_hits=np.full(len(hs), -1))


def svelo_seeds(n_reco: int, event_ids: Sequence[int], n_seeds: int, cfg: SveloConfig = SVELO) -> np.ndarray:
    """Seeds drawn from the physical prior (SPEC.md:346-354 default prior), fp32 [E, n, 2]."""
    out = np.empty((len(event_ids), n_seeds, 2), np.float32)
    for i, e in enumerate(event_ids):
        rng = _rng(cfg.seed, STREAM_SVELO + 1, (int(n_reco) << 32) | int(e))
        tx, ty = draw_prior(rng, n_seeds, cfg)
        out[i, :, 0] = tx
        out[i, :, 1] = ty
    return out
