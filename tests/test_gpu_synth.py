"""The on-device stream generator (synth.generate_synthetic_device) draws the reference generator's law.

bench.py builds every benchmark graph with generate_synthetic_device (numpy's generator alone takes about
a minute for the 191M-edge GDELT shape).  It is not bit-identical to numpy's PCG64 stream, so this module
checks it against the numpy restatement -- itself digest-pinned to the unmodified reference
(tests/test_synth.py, /root/reference/pkg/src/ctdg/synth.py:15-53) -- as a distribution: two-sample chi^2
over destination and source node frequencies (each of the heaviest nodes its own bin, the tail in
equal-mass bins), two-sample Kolmogorov-Smirnov over timestamps, and the structural properties
(sorted timestamps, no self-loops, node ids in range).
"""

from __future__ import annotations

import numpy as np
import pytest
from scipy import stats

pytestmark = pytest.mark.gpu

P_MIN = 1e-4


def _binned(a: np.ndarray, b: np.ndarray, nodes: int, heads: int = 60, tail_bins: int = 40):
    """Counts of a and b over bins: the `heads` most frequent nodes of the pooled sample individually,
    the rest in `tail_bins` bins of about equal pooled mass."""
    ca = np.bincount(a, minlength=nodes).astype(np.float64)
    cb = np.bincount(b, minlength=nodes).astype(np.float64)
    order = np.argsort(-(ca + cb), kind="stable")
    head, rest = order[:heads], order[heads:]
    cum = np.cumsum((ca + cb)[rest])
    cut = np.searchsorted(cum, np.linspace(0, cum[-1], tail_bins + 1)[1:-1])
    ra = [ca[head]] + [np.array([x.sum()]) for x in np.split(ca[rest], cut)]
    rb = [cb[head]] + [np.array([x.sum()]) for x in np.split(cb[rest], cut)]
    fa, fb = np.concatenate(ra), np.concatenate(rb)
    keep = (fa + fb) > 0
    return fa[keep], fb[keep]


def _two_sample_chi2(fa: np.ndarray, fb: np.ndarray) -> float:
    table = np.stack([fa, fb])
    return stats.chi2_contingency(table, correction=False)[1]


@pytest.mark.parametrize("src_skew", [None, 2.2])
def test_device_generator_draws_the_reference_law(cuda_device, src_skew):
    import paper_2311_17410_b200 as gf

    nodes, edges, span = 3_000, 1_000_000, 500_000
    s_np, d_np, t_np = gf.generate_synthetic_arrays(nodes, edges, 2.2, span, seed=11, src_skew=src_skew)
    s_d, d_d, t_d = gf.generate_synthetic_device(nodes, edges, 2.2, span, seed=11, src_skew=src_skew,
                                                 device=cuda_device)
    s_g, d_g, t_g = (x.cpu().numpy() for x in (s_d, d_d, t_d))
    # structure: ids in range, no self-loops, timestamps sorted inside [0, span)
    for x in (s_g, d_g):
        assert x.dtype == np.int64 and x.min() >= 0 and x.max() < nodes
    assert not np.any(s_g == d_g)
    assert np.all(np.diff(t_g) >= 0) and t_g.min() >= 0 and t_g.max() < span
    # destination (power law, skew 2.2) and source (uniform or power law, resampled off self-loops)
    assert _two_sample_chi2(*_binned(d_np, d_g, nodes)) > P_MIN
    assert _two_sample_chi2(*_binned(s_np, s_g, nodes)) > P_MIN
    # timestamps: sorted uniform integers over the span
    assert stats.ks_2samp(t_np, t_g).pvalue > P_MIN
    # the heaviest destination's share matches the law's weight (rank 1 of n^(-1/(skew-1)))
    w = np.arange(1, nodes + 1, dtype=np.float64) ** (-1.0 / 1.2)
    p0 = w[0] / w.sum()
    sd = np.sqrt(p0 * (1 - p0) / edges)
    assert abs(np.mean(d_g == 0) - p0) < 5 * sd


def test_device_generator_is_seeded(cuda_device):
    import paper_2311_17410_b200 as gf

    a = gf.generate_synthetic_device(500, 50_000, 2.2, 10_000, seed=5, src_skew=2.2, device=cuda_device)
    b = gf.generate_synthetic_device(500, 50_000, 2.2, 10_000, seed=5, src_skew=2.2, device=cuda_device)
    c = gf.generate_synthetic_device(500, 50_000, 2.2, 10_000, seed=6, src_skew=2.2, device=cuda_device)
    for x, y in zip(a, b):
        assert bool((x == y).all())
    assert not all(bool((x == y).all()) for x, y in zip(a, c))
