"""Noise-bound calculator for the LWE-PIR decode (DESIGN R8 / SURVEY 8(c)).

TEST INFRASTRUCTURE ONLY (see oracle/oracle.py header).

The paper prints no noise bound (it has no LWE PIR; DESIGN R1).  The bound is
derived from the decode identity (DESIGN R8):
    x_r = Delta * D[r][c*] + N_r  (mod 2^32),   N_r = sum_c D[r][c] e_c,
decode is correct iff |N_r| < 2^23 = Delta / 2.  With e_c ~ round(N(0, sigma^2))
i.i.d., N_r has mean 0 and variance ~ sigma^2 * sum_c D[r][c]^2, so the
per-entry failure probability is about erfc(z / sqrt(2)) with
    z = 2^23 / (sigma * sqrt(sum_c D[r][c]^2)).
Worst case (every byte 255): sum_c D^2 = m * 255^2.
"""
from __future__ import annotations

import math

import numpy as np

HALF_DELTA = 2.0 ** 23


def z_score(sigma: float, sum_sq: float) -> float:
    return HALF_DELTA / (sigma * math.sqrt(sum_sq))


def worst_case_z(sigma: float, m: int, p_max: int = 255) -> float:
    return z_score(sigma, m * float(p_max) ** 2)


def failure_prob(z: float) -> float:
    return math.erfc(z / math.sqrt(2.0))


def row_z(D: np.ndarray, sigma: float) -> np.ndarray:
    """Per-row z for an explicit D (rows x m, u8)."""
    sq = (D.astype(np.float64) ** 2).sum(axis=1)
    sq = np.maximum(sq, 1.0)
    return HALF_DELTA / (sigma * np.sqrt(sq))


def max_m_for(sigma: float, log2_fail: float = -40.0, p_max: int = 255) -> int:
    """Largest m whose worst-case per-entry failure probability is <= 2^log2_fail."""
    target = 2.0 ** log2_fail
    lo, hi = 1, 1 << 40
    while lo < hi:
        mid = (lo + hi + 1) // 2
        if failure_prob(worst_case_z(sigma, mid, p_max)) <= target:
            lo = mid
        else:
            hi = mid - 1
    return lo
