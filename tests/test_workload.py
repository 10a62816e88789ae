"""Seeded input generator: determinism, layout, and the Eq. 1 data model (CPU)."""
import math

import numpy as np
import pytest

import workload


def test_deterministic_and_row_consistent():
    w1 = workload.Workload(300, 3, p_missing=0.1, seed=11)
    w2 = workload.Workload(300, 3, p_missing=0.1, seed=11)
    np.testing.assert_array_equal(w1.x0, w2.x0)
    a = w1.y_packed()
    b = w2.y_packed()
    np.testing.assert_array_equal(a, b)
    # row ranges concatenate to the full packing
    parts = np.concatenate([w1.y_rows(0, 97), w1.y_rows(97, 200), w1.y_rows(200, 300)])
    np.testing.assert_array_equal(parts, a)
    # full rows are the symmetric view of the packing
    full = workload.unpack_lower(a, 300)
    rows = np.array([0, 5, 150, 299])
    np.testing.assert_array_equal(w1.y_full_rows(rows), full[rows])


def test_values_positive_and_missing_rate():
    w = workload.Workload(800, 2, p_missing=0.1, seed=3)
    y = w.y_packed()
    obs = y[~np.isnan(y)]
    assert np.all(obs > 0)
    frac = np.isnan(y).mean()
    assert abs(frac - 0.1) < 0.005


def test_truncated_normal_mean_at_zero_distance():
    """With all latent points coincident, y ~ N(0, s^2) truncated to > 0:
    half-normal mean s sqrt(2/pi) (Eq. 1, SPEC.md:520 idea)."""
    w = workload.Workload(600, 2, seed=5, sigma=1.0)
    w.x_true[:] = 0.0
    y = w.y_packed()
    se = math.sqrt(1 - 2 / math.pi) / math.sqrt(y.size)
    assert abs(y.mean() - math.sqrt(2 / math.pi)) < 4 * se


def test_configs_shapes():
    for name, (idx, n, d, kind, pm) in workload.CONFIGS.items():
        assert n >= 64 and d in (2, 6)
    w = workload.config("C1")
    assert w.x0.shape == (64, 2)
    assert w.sigma == pytest.approx(0.6)
