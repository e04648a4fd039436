"""K1 sync-free path: replayed launch graphs, device-side node growth and pool-overflow replay.

Same-size batches replay one captured launch sequence with new inputs every call; node ids
beyond the table capacity and slot/directory pool overflow abort a batch before any mutation
and replay it after the host grows the pools.  The store must still equal the oracle's
(itself pinned to the reference, tests/test_oracle_golden.py) field by field, and sampling
over it must match the oracle bit for bit.
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("directed", [True, False])
def test_replayed_batches_with_growth_match_oracle(cuda_device, ingest_path, directed):
    import torch

    import paper_2311_17410_b200 as gf
    from gpu_helpers import assert_store_equal, export_store, oracle_store
    from oracle import OracleGraph

    rng = np.random.default_rng(7 + directed)
    g = gf.DynamicGraph(directed=directed, tau=8)
    o = OracleGraph(directed, 8)
    t0 = 0
    next_pre = 10_000_000
    for b in range(12):
        m = 5000  # same shape every batch: the captured sequence is replayed
        hi = 300 * (b + 1) ** 2  # node ids outgrow the table (1024 rows at first) -> device abort + replay
        src = rng.integers(0, hi, m)
        dst = rng.integers(0, hi, m)
        ts = np.sort(rng.integers(t0, t0 + 5000, m))
        t0 += 5000
        if b == 5:  # a batch with out-of-order edges: rejections through the serial resolve
            k = rng.choice(m, size=50, replace=False)
            ts = ts.copy()
            ts[k] -= 20_000
        pre = None
        if b in (3, 8):  # preassigned ids through the replayed sequence
            pre = np.arange(next_pre, next_pre + m, dtype=np.int64)
            next_pre += 2 * m
        out, rej = g.add_edges_arrays(src, dst, ts, pre)
        want = o.add_edges(src, dst, ts, pre)
        np.testing.assert_array_equal(out.cpu().numpy(), want, err_msg=f"batch {b}")
        assert rej == int((want < 0).sum())
    assert g.num_nodes == o.num_nodes
    assert_store_equal(export_store(g), oracle_store(o), f"directed={directed}")
    roots = rng.integers(0, g.num_nodes, 2000)
    rts = rng.integers(0, t0, 2000)
    for policy in ("recent", "uniform"):
        got = gf.TemporalSampler(g, [10, 10], policy, seed=3).sample(torch.from_numpy(roots).cuda(),
                                                                     torch.from_numpy(rts).cuda())
        ref = o.sample_khop(roots, rts, [10, 10], policy, seed=3)
        for lay, r in zip(got.layers, ref):
            for a, w in zip((lay.offsets, lay.neighbors, lay.edge_ids, lay.timestamps), (r[2], r[3], r[4], r[5])):
                np.testing.assert_array_equal(a.cpu().numpy(), w)


def test_negative_id_batch_leaves_graph_unchanged(cuda_device):
    import paper_2311_17410_b200 as gf
    from gpu_helpers import assert_store_equal, export_store, oracle_store
    from oracle import OracleGraph

    g = gf.DynamicGraph(directed=True, tau=4)
    o = OracleGraph(True, 4)
    src, dst, ts = np.arange(100) % 7, (np.arange(100) * 3) % 11, np.arange(100)
    g.add_edges_arrays(src, dst, ts)
    o.add_edges(src, dst, ts)
    with pytest.raises(ValueError):
        g.add_edges_arrays(np.array([1, -2]), np.array([0, 1]), np.array([200, 201]))
    assert_store_equal(export_store(g), oracle_store(o), "after rejected batch")
    out, _ = g.add_edges_arrays(np.array([1, 2]), np.array([0, 1]), np.array([200, 201]))
    np.testing.assert_array_equal(out.cpu().numpy(), o.add_edges(np.array([1, 2]), np.array([0, 1]),
                                                                 np.array([200, 201])))


@pytest.mark.parametrize("offset", [0, 1 << 40])
def test_window_search_with_and_without_32bit_fence(cuda_device, offset):
    """Timestamps beyond int32 switch the sampler from the 32-bit fence to the int64 one; both match the oracle."""
    import torch

    import paper_2311_17410_b200 as gf
    from oracle import OracleGraph

    src, dst, ts = gf.generate_synthetic_arrays(200, 60_000, 2.2, 5_000, seed=11, src_skew=2.2)
    ts = ts + offset
    g = gf.DynamicGraph(directed=True, tau=256)
    o = OracleGraph(True, 256)
    for lo in range(0, len(src), 20_000):
        sl = slice(lo, lo + 20_000)
        g.add_edges_arrays(src[sl], dst[sl], ts[sl])
        o.add_edges(src[sl], dst[sl], ts[sl])
    rng = np.random.default_rng(5)
    pick = rng.integers(0, len(src), 3000)
    roots = np.concatenate([src[pick], dst[pick]])
    rts = np.concatenate([ts[pick], ts[pick] + rng.integers(0, 3, 3000)])
    for policy in ("recent", "uniform"):
        got = gf.TemporalSampler(g, [10, 10], policy, seed=1).sample(torch.from_numpy(roots).cuda(),
                                                                     torch.from_numpy(rts).cuda())
        ref = o.sample_khop(roots, rts, [10, 10], policy, seed=1)
        for lay, r in zip(got.layers, ref):
            for a, w in zip((lay.offsets, lay.neighbors, lay.edge_ids, lay.timestamps), (r[2], r[3], r[4], r[5])):
                np.testing.assert_array_equal(a.cpu().numpy(), w)
