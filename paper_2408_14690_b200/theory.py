"""Exact Gaussian magnitude quantile used to pick synthetic thresholds
(pkg/src/actsparse/theory.py:34-63): t_p with P(|Z| <= t_p) = p, bisection on
erf to 1e-12; p = 1 -> inf.  Host arithmetic (a scalar formula, not a kernel)."""

from __future__ import annotations

import math


def _abs_normal_mass(t: float) -> float:
    # P(|Z| <= t) = 2 Phi(t) - 1 with Phi(t) = (1 + erf(t / sqrt 2)) / 2
    return 2.0 * (0.5 * (1.0 + math.erf(t / math.sqrt(2.0)))) - 1.0


def gaussian_threshold(p: float, sigma_x: float = 1.0) -> float:
    if not 0.0 <= p <= 1.0:
        raise ValueError(f"sparsity must lie in [0, 1], got {p}")
    if not sigma_x > 0:
        raise ValueError(f"sigma_x must be positive, got {sigma_x}")
    if p == 0.0:
        return 0.0
    if p == 1.0:
        return math.inf
    lo, hi = 0.0, 1.0
    while _abs_normal_mass(hi) < p:
        hi *= 2.0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if _abs_normal_mass(mid) < p:
            lo = mid
        else:
            hi = mid
        if hi - lo <= 1e-12:
            break
    return sigma_x * 0.5 * (lo + hi)
