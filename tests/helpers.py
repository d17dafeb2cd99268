"""Shared test helpers: parity tolerances and comparisons (test infrastructure)."""
import numpy as np

# Stated tolerances: histograms bit-exact (unit weights) / 1e-12 relative
# (fractional weights); FP64 EM parameters and final log-likelihood 1e-9 relative.
TOL_EM = 1e-9
TOL_WEIGHTED_HIST = 1e-12


def model_close(a, b, tol=TOL_EM):
    """Component-wise relative distance between two canonical models (same order).
    Means are compared relative to the component scale (|mu| + sqrt(tr Sigma))."""
    assert a.size() == b.size(), (a.size(), b.size())
    worst = 0.0
    for ca, cb in zip(a.components, b.components):
        worst = max(worst, abs(ca.weight - cb.weight) / max(abs(cb.weight), 1e-300))
        scale = np.linalg.norm(cb.mean) + np.sqrt(np.trace(cb.covariance))
        worst = max(worst, np.linalg.norm(ca.mean - cb.mean) / scale)
        worst = max(worst, np.linalg.norm(ca.covariance - cb.covariance) / np.linalg.norm(cb.covariance))
    return worst


def rel(a, b):
    return abs(a - b) / max(abs(a), abs(b), 1e-300)
