"""Host-side adjoint machinery (no device work): Taylor test and the optimizer driver,
after the reference's tests/test_adjoint.py:173-275."""

import numpy as np
import pytest

from paper_2212_00964_b200.adjoint import OptimizeHistory, optimize, taylor_test


def test_taylor_quadratic_exact(rng):
    Q = rng.standard_normal((6, 6))
    Q = Q @ Q.T + 6 * np.eye(6)
    theta = rng.standard_normal(6)
    rep = taylor_test(lambda t: float(t @ Q @ t), lambda t: 2.0 * Q @ t, theta, rng.standard_normal(6),
                      [1e-1, 1e-2, 1e-3, 1e-4])
    assert np.all(np.abs(rep.orders_zeroth - 1.0) < 0.05)
    assert np.all(np.abs(rep.orders_first - 2.0) < 1e-6)
    assert abs(rep.fitted_first - 2.0) < 1e-6


def test_taylor_rejects_bad_steps():
    with pytest.raises(ValueError):
        taylor_test(lambda t: 0.0, lambda t: t, np.zeros(2), np.ones(2), [1e-1, -1e-2])


def test_taylor_rejects_nonfinite_objective():
    with pytest.raises(ValueError):
        taylor_test(lambda t: float("nan") if t[0] > 0 else 0.0, lambda t: t, np.zeros(2), np.ones(2), [1e-1])


def test_taylor_csv(tmp_path, rng):
    rep = taylor_test(lambda t: float(t @ t), lambda t: 2 * t, rng.standard_normal(3), rng.standard_normal(3),
                      [1e-1, 1e-2])
    path = tmp_path / "taylor.csv"
    rep.write_csv(path)
    text = path.read_text()
    assert "r_zeroth" in text and "fitted_order_first" in text


def test_optimize_lbfgs_quadratic(rng):
    Q = rng.standard_normal((8, 8))
    Q = Q @ Q.T + 8 * np.eye(8)
    b = rng.standard_normal(8)
    theta, hist = optimize(lambda t: (float(0.5 * t @ Q @ t - b @ t), Q @ t - b), np.zeros(8), method="lbfgs",
                           max_iters=30, gtol=1e-12)
    assert np.linalg.norm(Q @ theta - b) < 1e-8
    assert len(hist.objective) >= 1


def test_optimize_lbfgs_zero_gradient_terminates_immediately():
    calls = []

    def vg(t):
        calls.append(1)
        return 0.0, np.zeros(4)

    theta, _ = optimize(vg, np.ones(4), method="lbfgs", max_iters=50)
    assert np.array_equal(theta, np.ones(4))
    assert len(calls) == 1


def test_optimize_unknown_method():
    with pytest.raises(ValueError):
        optimize(lambda t: (0.0, t), np.zeros(2), method="sgd")


def test_optimize_mma_needs_bounds_and_constraint():
    with pytest.raises(ValueError):
        optimize(lambda t: (0.0, t), np.zeros(2), method="mma")


def test_history_csv(tmp_path):
    h = OptimizeHistory()
    h.record(2.0, np.array([3.0, 4.0]))
    path = tmp_path / "h.csv"
    h.write_csv(path)
    assert h.gradient_norm == [5.0]
    assert "gradient_norm" in path.read_text()
