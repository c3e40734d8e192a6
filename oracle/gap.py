"""Oracle of the performance-gap diagnosis (PAPER §VII; SURVEY §8(f)
NEXT-3).  TEST INFRASTRUCTURE ONLY (see oracle/oracle.py's header).

  y_actual = t_theory / measured latency     (efficiency)
  gap      = y_p80 - y_actual
  underperforming <=> gap > 0.1

The threshold decides an integer, so -- as the CUDA path -- the arithmetic is
fp32 (IEEE division, subtraction), written out one pair at a time.
"""
from __future__ import annotations

import numpy as np

THRESHOLD = np.float32(0.1)


def perf_gap(t_theory, status, eff_p80, measured, spec_of, n_specs, n_bins=100, lo=-0.5, hi=0.5):
    """Per pair gap (NaN when skipped), per spec {valid, underperforming}
    counts and the gap histogram on [lo, hi) with clamped end bins."""
    n = len(t_theory)
    gap = np.full(n, np.nan, np.float32)
    counts = np.zeros((n_specs, 2), np.int64)
    hist = np.zeros((n_specs, n_bins), np.int64)
    f32 = np.float32
    lo32, hi32 = f32(lo), f32(hi)
    for p in range(n):
        g = int(spec_of[p])
        t, m, y80 = f32(t_theory[p]), f32(measured[p]), f32(eff_p80[p])
        if status[p] != 0 or not (0 <= g < n_specs) or not m > 0 or np.isnan(t) or np.isnan(y80):
            continue
        y = f32(t / m)
        d = f32(y80 - y)
        if np.isnan(d):
            continue
        gap[p] = d
        counts[g, 0] += 1
        if d > THRESHOLD:
            counts[g, 1] += 1
        x = f32(f32(f32(d - lo32) / f32(hi32 - lo32)) * f32(n_bins))
        b = 0 if x < 0 else (n_bins - 1 if x >= n_bins else int(x))
        hist[g, b] += 1
    return gap, counts, hist
