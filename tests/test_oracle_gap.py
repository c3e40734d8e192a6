"""Pins of the gap-diagnosis oracle (oracle/gap.py; PAPER §VII-B P:675-683,
SPEC S:433-445): SPEC's worked examples, the constructed fixture of S:441,
the all-at-ceiling case (the paper's H20, "zero such points"), histogram
bookkeeping, and SPEC's monotone-diagnosis invariant."""
import numpy as np

from oracle import gap as G


def one(p80, y):
    # t_theory = y, measured = 1  ->  y_actual = y exactly
    return G.perf_gap(np.array([y], np.float32), np.zeros(1, np.uint8), np.array([p80], np.float32),
                      np.ones(1, np.float32), np.zeros(1, np.int64), 1)


def test_spec_examples():
    g, c, _ = one(0.60, 0.45)  # gap 0.15, underperforming
    assert abs(float(g[0]) - 0.15) < 1e-6 and c.tolist() == [[1, 1]]
    g, c, _ = one(0.60, 0.55)  # gap 0.05, not underperforming
    assert abs(float(g[0]) - 0.05) < 1e-6 and c.tolist() == [[1, 0]]
    g, c, _ = one(0.50, 0.70)  # y > y_p80 -> negative gap
    assert g[0] < 0 and c.tolist() == [[1, 0]]


def test_constructed_fixture_and_ceiling():
    """20% of one virtual GPU's samples degraded by 0.2 -> that GPU
    dominates; S:442 / P:683: all samples at the ceiling -> zero points."""
    rng = np.random.default_rng(0)
    n_per, n_gpu = 500, 3
    p80 = rng.uniform(0.3, 0.9, n_per * n_gpu).astype(np.float32)
    y = (p80 - rng.uniform(0.0, 0.05, p80.size)).astype(np.float32)  # near the ceiling
    spec = np.repeat(np.arange(n_gpu), n_per)
    _, c0, _ = G.perf_gap(y, np.zeros(y.size, np.uint8), p80, np.ones(y.size, np.float32), spec, n_gpu)
    assert c0[:, 1].sum() == 0 and c0[:, 0].tolist() == [n_per] * n_gpu
    bad = (spec == 1) & (rng.uniform(0, 1, y.size) < 0.2)
    y2 = np.where(bad, y - np.float32(0.2), y).astype(np.float32)
    _, c, _ = G.perf_gap(y2, np.zeros(y.size, np.uint8), p80, np.ones(y.size, np.float32), spec, n_gpu)
    assert c[1, 1] == bad.sum() and c[0, 1] == 0 and c[2, 1] == 0


def test_histogram_and_skips():
    t = np.array([0.45, 0.2, np.nan, 0.3, 0.1], np.float32)
    st = np.array([0, 0, 0, 3, 0], np.uint8)
    p80 = np.array([0.6, 0.9, 0.5, 0.5, 0.5], np.float32)
    m = np.array([1, 1, 1, 1, 0], np.float32)  # last pair: measured <= 0 -> skipped
    gap, c, h = G.perf_gap(t, st, p80, m, np.zeros(5, np.int64), 1, n_bins=10, lo=-0.5, hi=0.5)
    assert c.tolist() == [[2, 2]]  # pairs 0 and 1 valid (gap 0.15, 0.7)
    assert np.isnan(gap[2:]).all()
    assert h[0, 6] == 1 and h[0, 9] == 1 and h.sum() == 2  # 0.15 -> bin 6; 0.7 clamps to the top bin


def test_monotone_diagnosis():
    """lowering a measured latency never flips healthy -> underperforming."""
    rng = np.random.default_rng(1)
    n = 400
    t = rng.uniform(1, 100, n).astype(np.float32)
    m = (t / rng.uniform(0.2, 0.95, n)).astype(np.float32)
    p80 = rng.uniform(0.3, 0.99, n).astype(np.float32)
    z = np.zeros(n, np.int64)
    g1, _, _ = G.perf_gap(t, np.zeros(n, np.uint8), p80, m, z, 1)
    g2, _, _ = G.perf_gap(t, np.zeros(n, np.uint8), p80, (m * np.float32(0.8)).astype(np.float32), z, 1)
    assert not np.any((g1 <= G.THRESHOLD) & (g2 > G.THRESHOLD))
