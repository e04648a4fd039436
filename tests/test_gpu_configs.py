"""Parity at the BASELINE.json config sizes (CUDA path vs the CPU oracle on identical inputs).

configs[0] WIKI-shaped, 1-hop recent           -- bitwise on every root
configs[1] REDDIT-shaped, 2-hop uniform        -- bitwise vs the oracle's Philox stream; inclusion
                                                  frequencies vs the expected k/n (chi^2)
configs[3] GDELT-shaped, 191M edges, 2-hop f10 -- bitwise on a 4,096-root subset, recent and uniform
                                                  after 1% edge + 3 hub deletions (general path)
configs[4] MAG-shaped, one GPU's 1/8 share     -- bitwise on a 4,096-root subset, uniform [15,10] and
                                                  recent [10,10] (the bench's mag8 workload)
(configs[2] is covered by tests/test_gpu_harness.py.)
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _build_pair(src, dst, ts, directed, tau, batch):
    import paper_2311_17410_b200 as gf
    from oracle import OracleGraph

    g = gf.DynamicGraph(directed=directed, tau=tau)
    o = OracleGraph(directed, tau)
    for lo in range(0, len(src), batch):
        sl = slice(lo, lo + batch)
        g.add_edges_arrays(src[sl], dst[sl], ts[sl])
        o.add_edges(src[sl], dst[sl], ts[sl])
    return g, o


def _compare(got, want):
    for lay, ref in zip(got.layers, want):
        for nm, w in zip(("source_nodes", "source_times", "offsets", "neighbors", "edge_ids", "timestamps"), ref):
            np.testing.assert_array_equal(getattr(lay, nm).cpu().numpy(), w, err_msg=nm)


def test_wiki_shape_recent_one_hop_bitwise(cuda_device):
    import torch

    import paper_2311_17410_b200 as gf

    src, dst, ts = gf.generate_synthetic_arrays(9_000, 157_000, 2.2, 2_592_000, seed=0)
    g, o = _build_pair(src, dst, ts, False, 48, 10_000)
    roots = np.concatenate([src[-4000:], dst[-4000:]])
    rts = np.concatenate([ts[-4000:], ts[-4000:]])
    got = gf.TemporalSampler(g, [10], "recent").sample(torch.from_numpy(roots).cuda(), torch.from_numpy(rts).cuda())
    _compare(got, o.sample_khop(roots, rts, [10], "recent", threads=8))


def test_reddit_shape_uniform_two_hop(cuda_device):
    import torch
    from scipy.stats import chisquare

    import paper_2311_17410_b200 as gf

    src, dst, ts = gf.generate_synthetic_arrays(11_000, 672_000, 2.2, 2_592_000, seed=0)
    g, o = _build_pair(src, dst, ts, False, 48, 100_000)
    rng = np.random.default_rng(1)
    pick = rng.choice(len(src), 600, replace=False)
    roots = np.concatenate([src[-600:], dst[-600:], src[pick]])
    rts = np.concatenate([ts[-600:], ts[-600:], ts[pick]])
    got = gf.TemporalSampler(g, [10, 10], "uniform", seed=5).sample(torch.from_numpy(roots).cuda(),
                                                                    torch.from_numpy(rts).cuda())
    _compare(got, o.sample_khop(roots, rts, [10, 10], "uniform", seed=5, threads=8))
    # distribution: one busy node queried many times at a fixed time -> each in-window
    # candidate appears with probability k/n
    hub = int(np.bincount(src).argmax())
    q = 30_000
    t_end = int(ts[len(ts) // 2])
    lay = gf.sample_layer(g, torch.full((q,), hub, device="cuda"), torch.full((q,), -2**63, device="cuda"),
                          torch.full((q,), t_end, device="cuda"), 10, gf.SamplingPolicy.uniform(), seed=9)
    eids = lay.edge_ids.cpu().numpy()
    offs, nb, cand_eids, _ = o.sample_layer([hub], [-2**63], [t_end], 10**9, "recent")
    n = len(cand_eids)
    assert n > 10
    idx = {int(e): i for i, e in enumerate(cand_eids.tolist())}
    cnt = np.bincount([idx[int(e)] for e in eids], minlength=n)
    assert cnt.sum() == 10 * q
    assert chisquare(cnt).pvalue > 1e-4


@pytest.fixture(scope="module")
def gdelt_pair(cuda_device):
    """The full GDELT-shaped graph (191M directed edges) on the GPU and in the oracle."""
    import paper_2311_17410_b200 as gf
    from oracle import OracleGraph

    src_d, dst_d, ts_d = gf.generate_synthetic_device(17_000, 191_000_000, 2.2, 175_200, seed=0, src_skew=2.2)
    g = gf.DynamicGraph(directed=True, tau=8192)
    n = src_d.numel()
    g.reserve(17_000, 17_000 * 16 + n // 8192 + 1024, n + 17_000 * 8192)
    for lo in range(0, n, 1_000_000):
        g.add_edges_arrays(src_d[lo:lo + 1_000_000], dst_d[lo:lo + 1_000_000], ts_d[lo:lo + 1_000_000])
    src, dst, ts = src_d.cpu().numpy(), dst_d.cpu().numpy(), ts_d.cpu().numpy()
    del src_d, dst_d, ts_d
    o = OracleGraph(True, 8192)
    for lo in range(0, n, 1_000_000):
        o.add_edges(src[lo:lo + 1_000_000], dst[lo:lo + 1_000_000], ts[lo:lo + 1_000_000])
    assert g.num_nodes == o.num_nodes and g.total_edges_inserted == o.total_edges_inserted
    rng = np.random.default_rng(2)
    pick = rng.choice(n, 2048, replace=False)
    roots = np.concatenate([src[-1024:], dst[-1024:], src[pick]])
    rts = np.concatenate([ts[-1024:], ts[-1024:], ts[pick]])
    return g, o, roots, rts, src


def test_gdelt_full_shape_two_hop_bitwise_subset(gdelt_pair):
    import torch

    import paper_2311_17410_b200 as gf

    g, o, roots, rts, _ = gdelt_pair
    for policy in ("recent", "uniform"):
        got = gf.TemporalSampler(g, [10, 10], policy, seed=1).sample(torch.from_numpy(roots).cuda(),
                                                                     torch.from_numpy(rts).cuda())
        _compare(got, o.sample_khop(roots, rts, [10, 10], policy, seed=1, threads=16))


def test_gdelt_full_shape_after_deletions_bitwise(gdelt_pair):
    """The general (post-deletion) sampler at full GDELT scale: 1% of the edges and the three
    largest hubs deleted (storage.py:479-512), then 2-hop recent / uniform / time-window on 4,096
    roots, bitwise vs the oracle (sampling.py:153-155,178)."""
    import torch

    import paper_2311_17410_b200 as gf

    g, o, roots, rts, src = gdelt_pair
    n = len(src)
    rng = np.random.default_rng(3)
    dele = np.sort(rng.choice(n, n // 100, replace=False)).astype(np.int64)
    assert g.delete_edges(dele) == o.delete_edges(dele) == len(dele)
    hubs = np.argsort(np.bincount(src, minlength=17_000))[::-1][:3]
    for v in hubs:
        assert g.delete_node(int(v)) and o.delete_node(int(v))
    for policy, delta in (("recent", 0), ("uniform", 0), ("time_window", 5_000)):
        got = gf.TemporalSampler(g, [10, 10], policy, delta=delta, seed=4).sample(torch.from_numpy(roots).cuda(),
                                                                                  torch.from_numpy(rts).cuda())
        want = o.sample_khop(roots, rts, [10, 10], policy, delta=delta, seed=4, threads=16)
        _compare(got, want)
        assert sum(len(w[3]) for w in want) > 0


def test_mag8_shape_bitwise_subset(cuda_device):
    """configs[4] at one GPU's share of the 8-way partition (the bench's mag8 shape): 15.25M nodes,
    162.5M directed edges, span 120 ticks, tau 8192, 10M-edge ingest batches; 4,096 roots,
    uniform [15, 10] and recent [10, 10], bitwise vs the oracle."""
    import torch

    import paper_2311_17410_b200 as gf
    from oracle import OracleGraph

    nodes, edges, batch = 15_250_000, 162_500_000, 10_000_000
    src_d, dst_d, ts_d = gf.generate_synthetic_device(nodes, edges, 2.2, 120, seed=0, src_skew=2.2)
    g = gf.DynamicGraph(directed=True, tau=8192)
    g.reserve(nodes, nodes * 4 + edges // 8192 + 1024, edges + edges // 2)
    for lo in range(0, edges, batch):
        g.add_edges_arrays(src_d[lo:lo + batch], dst_d[lo:lo + batch], ts_d[lo:lo + batch])
    src, dst, ts = src_d.cpu().numpy(), dst_d.cpu().numpy(), ts_d.cpu().numpy()
    del src_d, dst_d, ts_d
    o = OracleGraph(True, 8192)
    for lo in range(0, edges, batch):
        o.add_edges(src[lo:lo + batch], dst[lo:lo + batch], ts[lo:lo + batch])
    assert g.num_nodes == o.num_nodes and g.total_edges_inserted == o.total_edges_inserted
    rng = np.random.default_rng(5)
    pick = rng.choice(edges, 2048, replace=False)
    roots = np.concatenate([src[-1024:], dst[-1024:], src[pick]])
    rts = np.concatenate([ts[-1024:], ts[-1024:], ts[pick]])
    for policy, fan in (("uniform", [15, 10]), ("recent", [10, 10])):
        got = gf.TemporalSampler(g, fan, policy, seed=6).sample(torch.from_numpy(roots).cuda(),
                                                                torch.from_numpy(rts).cuda())
        _compare(got, o.sample_khop(roots, rts, fan, policy, seed=6, threads=16))
