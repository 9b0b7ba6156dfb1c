"""Parity metrics of the paper's study.  TEST INFRASTRUCTURE.

Eq. 1:
  delta = log10( max_i || C_before(x_i) - V_before(x_i) ||_inf + eps ), eps = 1e-10
  eta   = (1/N) sum_i 1[ V_post(x_i) != C_post(x_i) ]
Base 10 and the L-inf norm: reading R14 (Table 3's -10.00 = log10(1e-10), L808).
Unequal-length generations count as inconsistent (reading R15).
"""
from __future__ import annotations

import math

import numpy as np


def delta(compiled, vendor, eps: float = 1e-10) -> float:
    m = 0.0
    for c, v in zip(compiled, vendor):
        c = np.asarray(c, np.float64)
        v = np.asarray(v, np.float64)
        if c.shape != v.shape:
            raise ValueError(f"shape mismatch {c.shape} vs {v.shape}")
        if c.size:
            m = max(m, float(np.max(np.abs(c - v))))
    return math.log10(m + eps)


def eta(compiled_post, vendor_post) -> float:
    n = 0
    bad = 0
    for c, v in zip(compiled_post, vendor_post):
        n += 1
        c = np.asarray(c)
        v = np.asarray(v)
        if c.shape != v.shape or not np.array_equal(c, v):
            bad += 1
    return bad / n if n else 0.0


def in_band(preds, band: float = 1e-3) -> bool:
    """True if any predicate on the sample's path lies within `band` of its threshold
    (north_star: such samples are excluded from decision parity and counted)."""
    return any(abs(v - t) < band for (_, v, t) in preds)
