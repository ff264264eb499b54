"""Pins of the match-predictor oracle."""
import numpy as np
import pytest

import synth
from oracle import predictor as P


def _cone(n, seed=1, d=768, axis_w=0.8):
    rng = np.random.default_rng(seed)
    c = rng.standard_normal(d)
    c /= np.linalg.norm(c)
    e, _ = synth.entries(n, seed=seed)
    X = axis_w * c + np.sqrt(1 - axis_w ** 2) * e
    return X / np.linalg.norm(X, axis=1, keepdims=True), c


def _objective(X, w, rho, nu):
    return 0.5 * w @ w - rho + np.maximum(0.0, rho - X @ w).sum() / (nu * len(X))


def test_retrain_rule():
    """retrain when embeddings change by > 5% (strict)."""
    assert not P.needs_retrain(0.04) and P.needs_retrain(0.06) and not P.needs_retrain(0.05)


def test_precision_recall_examples():
    """all correct -> (1, 1); all-true predictor on 50/50 labels -> (0.5, 1)."""
    t = np.array([1, 0, 1, 0], bool)
    assert P.precision_recall(t, t) == (1.0, 1.0)
    assert P.precision_recall(np.ones(4, bool), t) == (0.5, 1.0)


def test_rho_is_the_exact_minimiser_in_rho():
    """At the returned (w, rho), J(w, .) is minimal over rho (checked against the objective
    itself on a grid around rho) and at most a nu fraction of points violates."""
    X, _ = _cone(3000)
    nu = 0.01
    w, rho = P.train(X, nu=nu, epochs=20)
    j0 = _objective(X, w, rho, nu)
    for d in np.linspace(-0.05, 0.05, 41):
        assert j0 <= _objective(X, w, rho + d, nu) + 1e-12
    assert ((X @ w) < rho).mean() <= nu


def test_overfit_membership_and_far_outliers():
    """P:476-478 "we effectively overfit": training members -> true (>= 1 - 2 nu of them);
    SPEC S:385-392: a point far from every positive -> false; determinism."""
    X, c = _cone(4000)
    nu = 0.001
    w, rho = P.train(X, nu=nu)
    f = P.decision(w, rho, X)
    assert (f >= 0).mean() >= 1 - 2 * nu
    assert (P.decision(w, rho, -X[:200]) < 0).all()
    assert P.decision(w, rho, c[None, :])[0] > 0                 # the cluster centre
    w2, rho2 = P.train(X, nu=nu)
    assert np.array_equal(w, w2) and rho == rho2
