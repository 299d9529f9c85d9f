"""Prediction metrics (exact.cpp:79-92) and the dense predictive oracle --
host-side, no GPU."""
import numpy as np
import pytest

import paper_2405_18328_b200 as wg
from oracle import dense_ref


def test_metrics_formula():
    pred = wg.PredictiveDistribution(np.array([0.0, 1.0, 2.0]), np.array([0.5, 0.25, 1.0]), 0.5)
    y = np.array([0.5, 1.0, 1.0])
    m = wg.test_metrics(pred, y)
    err = pred.means - y
    var = pred.variances + 0.5
    assert m.rmse == pytest.approx(np.sqrt(np.mean(err ** 2)))
    assert m.mean_loglik == pytest.approx(np.mean(-0.5 * (np.log(var) + np.log(2 * np.pi)) - 0.5 * err ** 2 / var))
    assert wg.test_metrics(wg.PredictiveDistribution(np.zeros(0), np.zeros(0)), np.zeros(0)).rmse == 0.0
    with pytest.raises(ValueError, match="length mismatch"):
        wg.test_metrics(pred, y[:2])


def test_dense_predict_interpolates_training_points():
    """Noise-free limit: the posterior mean at training inputs reproduces y and
    the latent variance vanishes (exact.cpp:52-77)."""
    rng = np.random.default_rng(0)
    X = rng.standard_normal((60, 2))
    y = np.sin(X[:, 0]) + X[:, 1]
    means, var, nv = dense_ref.predict(X, y, X, np.ones(2), 1.0, 1e-4)
    assert np.max(np.abs(means - y)) < 1e-4
    assert np.max(var) < 1e-6 and nv == pytest.approx(1e-8)
