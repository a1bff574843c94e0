"""Keyed, seeded event / node-table / seed generation (no method arithmetic).

Every event e of config c is drawn from its own Philox stream keyed
(c.seed << 8 | stream, e), so event e's hits and seeds are the same whatever
range of events a caller (or a rank) asks for.

Hit layout: float32 [N, 4] = (x, y, z, 0) per hit, events in
CSR form with int32 offsets[E + 1]; hits of one event are sorted by their
plane coordinate (z for the VELO-like models, x for the 2-D toy, whose hits
are stored as (x, y, 0, 0)).
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional, Sequence

import numpy as np

from .configs import (LINE2D, SLOPE3, TOY_PLANES, TOY_SMEAR, VELO_PLANES,
                      VELO_R_MAX, VELO_R_MIN, VELO_SMEAR, Config)

STREAM_HITS, STREAM_SEEDS = 1, 2


def _rng(cfg_seed: int, stream: int, event: int) -> np.random.Generator:
    key = np.array([(int(cfg_seed) << 8) | int(stream), int(event)], dtype=np.uint64)
    return np.random.Generator(np.random.Philox(key=key))


@dataclasses.dataclass
class EventBatch:
    """A CSR batch of events. `truth` is harness-only (never passed to kernels)."""
    offsets: np.ndarray          # int32 [E+1]
    hits: np.ndarray             # float32 [N, 4]
    event_ids: np.ndarray        # int64 [E]
    truth: List[np.ndarray]      # per event float64 [T, P]: true track parameters
    n_track_hits: np.ndarray     # int64 [E]

    @property
    def n_events(self) -> int:
        return len(self.offsets) - 1

    @property
    def n_hits(self) -> int:
        return int(self.offsets[-1])

    def event_hits(self, e: int) -> np.ndarray:
        return self.hits[self.offsets[e]:self.offsets[e + 1]]


def _toy_event(cfg: Config, rng: np.random.Generator):
    """BASELINE configs[0]: 5 lines y = a x + b, one hit per plane x = 1..10,
    y smeared N(0, 0.01); 20 noise hits x in {1..10}, y ~ U[-6, 6] (Z16)."""
    T = cfg.n_tracks
    a = rng.uniform(-0.5, 0.5, T)
    b = rng.uniform(-1.0, 1.0, T)
    xs, ys = [], []
    for t in range(T):
        y = a[t] * TOY_PLANES + b[t] + rng.normal(0.0, TOY_SMEAR, len(TOY_PLANES))
        xs.append(TOY_PLANES.copy())
        ys.append(y)
    n_track_hits = T * len(TOY_PLANES)
    nx = rng.integers(1, 11, 20).astype(np.float64)
    ny = rng.uniform(-6.0, 6.0, 20)
    x = np.concatenate(xs + [nx])
    y = np.concatenate(ys + [ny])
    order = np.argsort(x, kind="stable")
    h = np.zeros((len(x), 4), np.float32)
    h[:, 0] = x[order]
    h[:, 1] = y[order]
    truth = np.stack([a, b], axis=1)
    return h, truth, n_track_hits


def _velo_event(cfg: Config, rng: np.random.Generator):
    """BASELINE configs[1..4]: straight tracks from (0, 0, z0), slopes
    tx, ty ~ U(-0.3, 0.3), hit at every plane z_p > z0 whose TRUE intersection
    lies in 5 < r < 40 mm (Z13; no cut if cfg.dense), smeared N(0, 0.012) in x
    and y; + round(0.1 n_track_hits) noise hits (Z11); sorted by z."""
    T = int(rng.poisson(cfg.n_tracks)) if cfg.poisson_tracks else cfg.n_tracks
    tx = rng.uniform(-0.3, 0.3, T)
    ty = rng.uniform(-0.3, 0.3, T)
    z0 = rng.normal(0.0, cfg.z0_sigma, T) if cfg.z0_sigma > 0 else np.zeros(T)
    planes = VELO_PLANES
    d = planes[None, :] - z0[:, None]                    # [T, L]
    xt = tx[:, None] * d
    yt = ty[:, None] * d
    r = np.hypot(xt, yt)
    keep = d > 0
    if not cfg.dense:
        keep &= (r > VELO_R_MIN) & (r < VELO_R_MAX)
    ti, pi = np.nonzero(keep)
    n_tr = len(ti)
    hx = xt[ti, pi] + rng.normal(0.0, VELO_SMEAR, n_tr)
    hy = yt[ti, pi] + rng.normal(0.0, VELO_SMEAR, n_tr)
    hz = planes[pi]
    n_noise = int(round(0.1 * n_tr))
    npl = rng.integers(0, len(planes), n_noise)
    rr = np.sqrt(rng.uniform(VELO_R_MIN ** 2, VELO_R_MAX ** 2, n_noise))
    ph = rng.uniform(0.0, 2.0 * np.pi, n_noise)
    x = np.concatenate([hx, rr * np.cos(ph)])
    y = np.concatenate([hy, rr * np.sin(ph)])
    z = np.concatenate([hz, planes[npl]])
    order = np.argsort(z, kind="stable")
    h = np.zeros((len(x), 4), np.float32)
    h[:, 0] = x[order]
    h[:, 1] = y[order]
    h[:, 2] = z[order]
    if cfg.model == SLOPE3:
        truth = np.stack([tx, ty, z0], axis=1)
    else:
        truth = np.stack([tx, ty], axis=1)
    return h, truth, n_tr


def make_event(cfg: Config, event_id: int):
    rng = _rng(cfg.seed, STREAM_HITS, event_id)
    if cfg.model == LINE2D:
        return _toy_event(cfg, rng)
    return _velo_event(cfg, rng)


def make_batch(cfg: Config, event_ids: Optional[Sequence[int]] = None) -> EventBatch:
    """Events `event_ids` (default: 0..cfg.n_events-1) of config `cfg`."""
    if event_ids is None:
        event_ids = range(cfg.n_events)
    event_ids = np.asarray(list(event_ids), dtype=np.int64)
    hs, truths, nth = [], [], []
    for e in event_ids:
        h, t, n = make_event(cfg, int(e))
        hs.append(h)
        truths.append(t)
        nth.append(n)
    counts = np.array([len(h) for h in hs], dtype=np.int64)
    offsets = np.zeros(len(hs) + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    assert offsets[-1] < 2 ** 31
    hits = np.concatenate(hs, axis=0) if hs else np.zeros((0, 4), np.float32)
    return EventBatch(offsets=offsets.astype(np.int32), hits=np.ascontiguousarray(hits),
                      event_ids=event_ids, truth=truths, n_track_hits=np.asarray(nth))


def make_seeds(cfg: Config, event_ids: Optional[Sequence[int]] = None,
               n_seeds: Optional[int] = None) -> np.ndarray:
    """Z8: seeds i.i.d. uniform on the prior box, float32 [E, n_seeds, P]."""
    if event_ids is None:
        event_ids = range(cfg.n_events)
    n = cfg.n_seeds if n_seeds is None else n_seeds
    lo = np.asarray(cfg.box_lo, np.float64)
    hi = np.asarray(cfg.box_hi, np.float64)
    out = np.empty((len(list(event_ids)), n, cfg.P), np.float32)
    if n == 0 or len(cfg.box_lo) == 0:  # grid-only configs (cfg1) draw no seeds
        return np.zeros((out.shape[0], n, cfg.P), np.float32)
    for i, e in enumerate(event_ids):
        rng = _rng(cfg.seed, STREAM_SEEDS, int(e))
        u = rng.random((n, cfg.P))
        out[i] = (lo + u * (hi - lo)).astype(np.float32)
    return out


def axis_nodes(cfg: Config) -> List[np.ndarray]:
    """Z4: inclusive linspace nodes computed in fp64 and rounded to fp32; the
    last axis optionally snapped to a multiple of cfg.snap_last_axis."""
    out = []
    for i, (lo, hi, n) in enumerate(cfg.axes):
        v = lo + np.arange(n, dtype=np.float64) * ((hi - lo) / (n - 1))
        if cfg.snap_last_axis and i == len(cfg.axes) - 1:
            q = cfg.snap_last_axis
            v = np.round(v / q) * q
        out.append(v.astype(np.float32))
    return out
