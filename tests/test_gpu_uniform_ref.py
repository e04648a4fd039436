"""Uniform sampling vs the REFERENCE sampler's own draws (two-sample tests).

tests/golden/make_uniform_ref.py ran the unmodified reference ``sample_layer``
(uniform, fanout 10: PCG64 partial Fisher-Yates, sampling.py:185-198) on six
GDELT-1/50 queries with n = 12 ... 1,000 in-window candidates, each repeated R
times, and stored its inclusion counts, its k-subset counts (n <= 14) and its
pair-inclusion counts (n = 30).  The CUDA sampler (Philox + Floyd, DESIGN.md
section 2) runs the same queries on the same graph, and the two samplers must
be indistinguishable:

* exact count min(fanout, n) and no repeated candidate per query;
* inclusions: two-sample chi^2 (reference vs GPU) and goodness of fit to k/n;
* joint law, n <= 14: every k-subset is equally likely (C(12,10) = 66 and
  C(14,10) = 1001 cells), two-sample and goodness of fit -- a sampler with
  the right marginals but a biased joint law fails here;
* pairs, n = 30: per-pair z scores of GPU vs reference counts.
Thresholds: p > 1e-4 per test (SPEC.md:220,587 uses 1e-4), |z| < 5.
"""

from __future__ import annotations

import os
from itertools import combinations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "uniform_ref.npz")
TS_MIN = -(2**63)


@pytest.fixture(scope="module")
def graph_and_ref(cuda_device):
    import paper_2311_17410_b200 as gf

    ref = np.load(GOLD)
    src, dst, ts = gf.generate_synthetic_arrays(int(ref["nodes"]), int(ref["edges"]), 2.2, 175_200, seed=0,
                                                src_skew=2.2)
    g = gf.DynamicGraph(directed=True, tau=8192, device=cuda_device)
    for lo in range(0, len(src), 100_000):
        g.add_edges_arrays(src[lo:lo + 100_000], dst[lo:lo + 100_000], ts[lo:lo + 100_000])
    return g, ref


def _gpu_positions(g, ref, qi, seed):
    import torch

    import paper_2311_17410_b200 as gf

    v, t_end, R = int(ref[f"q{qi}_node"]), int(ref[f"q{qi}_t_end"]), int(ref[f"q{qi}_reps"])
    dev = g.device
    lay = gf.sample_layer(g, torch.full((R,), v, device=dev), torch.full((R,), TS_MIN, device=dev),
                          torch.full((R,), t_end, device=dev), int(ref["fanout"]), gf.SamplingPolicy.uniform(), seed=seed)
    cand = ref[f"q{qi}_candidates"]
    order = np.argsort(cand)
    eids = lay.edge_ids.cpu().numpy()
    pos = order[np.searchsorted(cand[order], eids)]
    assert np.array_equal(cand[pos], eids), "sampled an edge outside the reference candidate set"
    k = min(int(ref["fanout"]), len(cand))
    assert np.all(np.diff(lay.offsets.cpu().numpy()) == k)
    return pos.reshape(R, k)


def _queries():
    return range(int(np.load(GOLD)["n_queries"]))


@pytest.mark.parametrize("qi", list(_queries()))
def test_inclusion_two_sample_vs_reference(graph_and_ref, qi):
    from scipy.stats import chi2_contingency, chisquare

    g, ref = graph_and_ref
    pos = _gpu_positions(g, ref, qi, seed=1000 + qi)
    srt = np.sort(pos, axis=1)
    assert not np.any(srt[:, 1:] == srt[:, :-1]), "a candidate drawn twice in one query"
    n = int(ref[f"q{qi}_n"])
    gpu = np.bincount(pos.ravel(), minlength=n)
    refc = ref[f"q{qi}_incl"]
    assert gpu.sum() == refc.sum()
    p2 = chi2_contingency(np.stack([refc, gpu])).pvalue
    assert p2 > 1e-4, f"q{qi} (n={n}): GPU inclusions differ from the reference sampler's, p={p2:.2e}"
    assert chisquare(gpu).pvalue > 1e-4


@pytest.mark.parametrize("qi", [q for q in _queries() if int(np.load(GOLD)[f"q{q}_n"]) <= 14])
def test_joint_subset_law_vs_reference(graph_and_ref, qi):
    from scipy.stats import chi2_contingency, chisquare

    g, ref = graph_and_ref
    pos = _gpu_positions(g, ref, qi, seed=2000 + qi)
    n, k = int(ref[f"q{qi}_n"]), pos.shape[1]
    masks = np.zeros(len(pos), np.int64)
    for j in range(k):
        masks |= np.left_shift(1, pos[:, j])
    all_masks = np.array(sorted(sum(1 << i for i in c) for c in combinations(range(n), k)), np.int64)
    gpu = np.zeros(len(all_masks), np.int64)
    u, c = np.unique(masks, return_counts=True)
    gpu[np.searchsorted(all_masks, u)] = c
    refc = np.zeros(len(all_masks), np.int64)
    refc[np.searchsorted(all_masks, ref[f"q{qi}_subset_masks"])] = ref[f"q{qi}_subset_counts"]
    assert np.all(refc > 0) and np.all(gpu > 0), "some k-subset never drawn"
    assert chisquare(gpu).pvalue > 1e-4, "GPU k-subsets not uniform"
    p2 = chi2_contingency(np.stack([refc, gpu])).pvalue
    assert p2 > 1e-4, f"q{qi}: GPU subset law differs from the reference sampler's, p={p2:.2e}"


@pytest.mark.parametrize("qi", [q for q in _queries() if int(np.load(GOLD)[f"q{q}_n"]) == 30])
def test_pair_inclusion_vs_reference(graph_and_ref, qi):
    g, ref = graph_and_ref
    pos = _gpu_positions(g, ref, qi, seed=3000 + qi)
    n, k, R = int(ref[f"q{qi}_n"]), pos.shape[1], len(pos)
    pair = np.zeros((n, n), np.int64)
    srt = np.sort(pos, axis=1)
    ii, jj = np.triu_indices(k, 1)
    np.add.at(pair, (srt[:, ii].ravel(), srt[:, jj].ravel()), 1)
    iu = np.triu_indices(n, 1)
    a, b = pair[iu].astype(np.float64), ref[f"q{qi}_pairs"][iu].astype(np.float64)
    expect = R * k * (k - 1) / (n * (n - 1))
    assert abs(a.mean() - expect) < 1e-9 * expect + 1e-6 and abs(b.mean() - expect) < 1e-6 + 1e-9 * expect
    z = (a - b) / np.sqrt(a + b)
    assert np.abs(z).max() < 5.0, f"pair counts differ: max |z| = {np.abs(z).max():.2f}"
    assert 0.6 < float(np.mean(z * z)) < 1.4, f"pair z^2 mean {np.mean(z * z):.3f}"
    zg = (a - expect) / np.sqrt(expect * (1 - expect / R))
    assert np.abs(zg).max() < 5.0
