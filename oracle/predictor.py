"""fp64 oracle of the match predictor -- TEST INFRASTRUCTURE ONLY.

One-Class SVM with a linear decision function f(x) = <w, x> - rho, trained "by utilizing all
prompt embeddings stored in the VDB, and assigning them a positive label" with
nu = 0.001, minimising the one-class objective

    J(w, rho) = 1/2 ||w||^2 - rho + 1/(nu n) sum_i max(0, rho - <w, x_i>).

Reading R22 (the paper says only "SGD"): J is convex and piecewise linear in rho with its
exact minimiser at the k-th smallest margin, k = ceil(nu n); so each epoch sets rho to that
order statistic and then takes one subgradient step in w on nu * J:

    viol   = { i : <w, x_i> < rho }           (strict; max(0, 0) has subgradient 0)
    w     <- w - eta_t (nu w - (1/n) sum_viol x_i) / nu,   eta_t = lr0 / sqrt(1 + t)

starting from w = mean(x_i) (the one-class direction of the data).  x_i are the STORED
cached embeddings scaled to unit norm (x~ / ||x~||), the same vectors the lookup scores.
predict(q) = f(q~ / ||q~||) >= 0 ("likely a close match"; >= 0 inclusive).
"""
from __future__ import annotations

import math

import numpy as np


def kth(n: int, nu: float) -> int:
    return max(1, int(math.ceil(nu * n)))


def train(X: np.ndarray, nu: float = 0.001, epochs: int = 50, lr0: float = 0.5):
    """X: [n][d] fp64 unit rows.  Returns (w [d], rho)."""
    X = np.asarray(X, dtype=np.float64)
    n, d = X.shape
    k = kth(n, nu)
    w = X.mean(axis=0)
    rho = 0.0
    for t in range(epochs):
        margins = X @ w
        rho = float(np.partition(margins, k - 1)[k - 1])     # k-th smallest margin
        viol = margins < rho
        g = X[viol].sum(axis=0) if viol.any() else np.zeros(d)
        eta = lr0 / math.sqrt(1.0 + t)
        w = w - eta * (nu * w - g / n) / nu
    margins = X @ w
    rho = float(np.partition(margins, k - 1)[k - 1])
    return w, rho


def decision(w: np.ndarray, rho: float, Q: np.ndarray) -> np.ndarray:
    """f(q) = <w, q> - rho for unit rows Q."""
    return np.asarray(Q, dtype=np.float64) @ w - rho


def needs_retrain(change_fraction: float, threshold: float = 0.05) -> bool:
    """Retrain "when embeddings in VDB changes significantly (i.e., > 5%)", strict."""
    return change_fraction > threshold


def precision_recall(pred: np.ndarray, truth: np.ndarray):
    pred = np.asarray(pred, bool)
    truth = np.asarray(truth, bool)
    tp = int((pred & truth).sum())
    p = tp / max(1, int(pred.sum()))
    r = tp / max(1, int(truth.sum()))
    return p, r
