"""50-digit mpmath evaluation of Eq. (1) and its gradient for tiny inputs.

TEST INFRASTRUCTURE ONLY.  Used by tests to bound the C oracle's fp64
rounding (north star: "agreement with brute-force evaluation on tiny
inputs").  Eq. (1): R = sum_k exp(-s_k^2 / sigma^2); the
gradient here is taken by mpmath's numerical differentiation (mp.diff), not
by the analytic chain rule the C oracle uses, so a wrong derivative formula
in oracle.c cannot be reproduced here.
"""
from __future__ import annotations

import mpmath as mp

mp.mp.dps = 50


def _s2(model, h, th, z_ref):
    x, y, z = mp.mpf(float(h[0])), mp.mpf(float(h[1])), mp.mpf(float(h[2]))
    if model == 0:
        s = y - (th[0] * x + th[1])
        return s * s
    d = z - (th[2] if model == 2 else mp.mpf(float(z_ref)))
    sx = x - th[0] * d
    sy = y - th[1] * d
    return sx * sx + sy * sy


def response(model, hits, theta, sigma, z_ref=0.0):
    th = [mp.mpf(float(t)) for t in theta]
    sg = mp.mpf(float(sigma))
    return mp.fsum(mp.exp(-_s2(model, h, th, z_ref) / (sg * sg)) for h in hits)


def gradient(model, hits, theta, sigma, z_ref=0.0):
    P = len(theta)
    out = []
    for i in range(P):
        def f(t, i=i):
            th = [mp.mpf(float(v)) for v in theta]
            th[i] = t
            sg = mp.mpf(float(sigma))
            return mp.fsum(mp.exp(-_s2(model, h, th, z_ref) / (sg * sg)) for h in hits)
        out.append(mp.diff(f, mp.mpf(float(theta[i]))))
    return out


def hessian(model, hits, theta, sigma, z_ref=0.0):
    """Second partial derivatives of Eq. (1) by mpmath numerical differentiation."""
    P = len(theta)
    sg = mp.mpf(float(sigma))

    def f(*t):
        return mp.fsum(mp.exp(-_s2(model, h, list(t), z_ref) / (sg * sg)) for h in hits)

    x0 = [mp.mpf(float(v)) for v in theta]
    H = [[None] * P for _ in range(P)]
    for a in range(P):
        for b in range(P):
            orders = [0] * P
            orders[a] += 1
            orders[b] += 1
            H[a][b] = mp.diff(f, x0, tuple(orders))
    return H
