"""Workload metrics used by the harness reports (harness.py:245-253, 480-505) and the
cluster telemetry (cluster.py:77-78): set overlap, load spread, and how well an
access-count histogram follows a power law or an exponential.

Semantics follow the reference metrics.py:8-64; the fits run the same numpy
least-squares calls so the reported R^2 values are the same floats.
"""

from __future__ import annotations

import numpy as np

__all__ = ["jaccard", "coefficient_of_variation", "access_distribution"]


def jaccard(set_a, set_b) -> float:
    """Intersection over union of two id collections (metrics.py:8-14); two empty sets give 0."""
    left, right = set(set_a), set(set_b)
    both = len(left & right)
    either = len(left) + len(right) - both
    return both / either if either else 0.0


def coefficient_of_variation(values) -> float:
    """Population std over mean (metrics.py:17-25); 0 when empty or the mean is 0."""
    v = np.asarray(values, dtype=np.float64)
    mu = v.mean() if v.size else 0.0
    return float(v.std() / mu) if mu != 0 else 0.0


def _line_fit_quality(x: np.ndarray, y: np.ndarray) -> float:
    """Coefficient of determination of the degree-1 least-squares fit y ~ x (metrics.py:28-36)."""
    fitted = np.polyval(np.polyfit(x, y, 1), x)
    resid = float(((y - fitted) ** 2).sum())
    spread = float(((y - y.mean()) ** 2).sum())
    return 1.0 - resid / spread if spread != 0.0 else 1.0


def access_distribution(counts) -> dict:
    """Rank-frequency curve of the positive counts plus two fit qualities (metrics.py:39-64):
    ``powerlaw_r2`` (log rank vs log frequency) and ``exponential_r2`` (rank vs log
    frequency).  Both are NaN when the curve is flat or has fewer than 3 points; an input
    without a positive count raises ValueError."""
    c = np.asarray(counts, dtype=np.float64)
    positive = c[c > 0]
    if positive.size == 0:
        raise ValueError("access counts are all zero; distribution fit undefined")
    freq = -np.sort(-positive)
    ranks = np.arange(1, freq.size + 1, dtype=np.float64)
    flat = bool((freq == freq[0]).all())
    nan = float("nan")
    fits = (nan, nan)
    if not flat and freq.size >= 3:
        log_f = np.log(freq)
        fits = (_line_fit_quality(np.log(ranks), log_f), _line_fit_quality(ranks, log_f))
    return {"ranks": ranks, "frequencies": freq, "powerlaw_r2": fits[0], "exponential_r2": fits[1],
            "degenerate": flat}
