"""sVELO evaluation (NEXT #2): Eq. (3) seed budget, epsilon-matching and efficiency, and the
paper's experiment shape (efficiency vs reconstructible tracks at alpha = 1/3 and 1/10,
PAPER.md:197-241).  Harness code: runs the CUDA path through the public binding.
"""
from __future__ import annotations

import math

import numpy as np

from synth.svelo import SVELO, SveloConfig


def direction_from_slopes(tx, ty):
    """Unit direction (x, y, z) of the line x = tx z, y = ty z (z > 0)."""
    tx = np.asarray(tx, np.float64)
    ty = np.asarray(ty, np.float64)
    n = np.sqrt(tx * tx + ty * ty + 1.0)
    return np.stack([tx / n, ty / n, 1.0 / n], axis=-1)


def angle_between(a_tx, a_ty, b_tx, b_ty):
    """Angle (rad) between the directions of two lines through the origin (matching metric,
    PAPER.md:197 'within epsilon = 1e-3 radians'), computed stably with atan2(|a x b|, a . b)."""
    a = direction_from_slopes(a_tx, a_ty)
    b = direction_from_slopes(b_tx, b_ty)
    cross = np.linalg.norm(np.cross(a, b), axis=-1)
    dot = np.sum(a * b, axis=-1)
    return np.arctan2(cross, dot)


def grid_cells_for_resolution(eps: float = 1e-3, cfg: SveloConfig = SVELO) -> int:
    """n_grid of Eq. (3): cells of a slope lattice with step eps covering the
    prior, |tx|, |ty| <= tan(max polar) (reading Z32: the kernels' lattice is in slopes)."""
    t = math.tan(cfg.max_polar)
    n = int(math.ceil(2.0 * t / eps)) + 1
    return n * n


def seed_budget(alpha: float, n_grid: int, C0: float = 30.0, q: int = 3) -> int:
    """Eq. (3): n = alpha * n_grid * (1/C0) * (1/q)."""
    return int(math.floor(alpha * n_grid / (C0 * q)))


def match_tracks(found_tx, found_ty, truth: np.ndarray, eps: float = 1e-3):
    """PAPER.md:197-198 ("a track is reconstructed if the found parameters are within
    epsilon = 1e-3 radians"), as a one-to-one matching: every (truth,
    candidate) pair within eps, taken in ascending angle (ties: truth index, then candidate
    index), matches when neither side is matched yet.  Returns (n_matched, n_missed, n_ghosts)."""
    n_t, n_f = len(truth), len(found_tx)
    if n_t == 0 or n_f == 0:
        return 0, n_t, n_f
    ang = angle_between(truth[:, 0][:, None], truth[:, 1][:, None], np.asarray(found_tx)[None, :],
                        np.asarray(found_ty)[None, :])
    ti, fi = np.nonzero(ang <= eps)
    order = np.lexsort((fi, ti, ang[ti, fi]))
    used_t, used_f = np.zeros(n_t, bool), np.zeros(n_f, bool)
    m = 0
    for k in order:
        if not used_t[ti[k]] and not used_f[fi[k]]:
            used_t[ti[k]] = used_f[fi[k]] = True
            m += 1
    return m, n_t - m, n_f - m


def match_efficiency(found_tx, found_ty, truth: np.ndarray, eps: float = 1e-3):
    """Efficiency = matched / true tracks under the one-to-one matching of match_tracks().
    Returns (efficiency, n_matched, n_true)."""
    if len(truth) == 0:
        return 1.0, 0, 0
    m, _, _ = match_tracks(found_tx, found_ty, truth, eps)
    return m / len(truth), m, len(truth)
