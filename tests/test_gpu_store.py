"""K1 (batch append) parity: the device block store equals the reference's, field by field.

Golden fixtures come from the unmodified reference (tests/golden/store_cases.npz);
larger randomized streams are checked against the CPU oracle (itself pinned to
the reference in tests/test_oracle_golden.py).
"""

from __future__ import annotations

import numpy as np
import pytest

from fixtures import load, replay_build

pytestmark = pytest.mark.gpu


def test_store_layout_matches_reference_fixtures(cuda_device, ingest_path):
    from gpu_helpers import assert_store_equal, export_store, gpu_factory

    fx, meta = load("store_cases.npz")
    for m in meta:
        p = f"c{m['id']}/"
        g, eids = replay_build(gpu_factory, fx, p, m)
        np.testing.assert_array_equal(eids, fx[p + "eids"], err_msg=p)
        want = {k: fx[p + k] for k in ("head", "tail", "num_blocks", "degree", "node_valid", "blk_capacity", "blk_size",
                                         "blk_tmin", "blk_tmax", "blk_prev", "blk_next", "slot_offsets", "slot_nbr",
                                         "slot_eid", "slot_ts", "slot_valid")}
        assert_store_equal(export_store(g.g), want, p)
        ne = fx[p + "next_edge_id"]
        assert g.g.next_edge_id == ne[0] and g.g.total_edges_inserted == ne[1]


@pytest.mark.parametrize("directed", [True, False])
@pytest.mark.parametrize("sizing", ["adaptive", "fixed", "batch"])
def test_store_matches_oracle_random_streams(cuda_device, ingest_path, directed, sizing):
    from gpu_helpers import GpuGraphAdapter, assert_store_equal, export_store, oracle_store
    from oracle import OracleGraph

    rng = np.random.default_rng(hash((directed, sizing)) & 0xFFFF)
    for case in range(4):
        nn = int(rng.integers(2, 400))
        tau = int(rng.choice([1, 3, 8, 48, 8192]))
        param = int(rng.integers(1, 9))
        gg = GpuGraphAdapter(directed, tau, sizing, param)
        o = OracleGraph(directed, tau, sizing, param)
        for b in range(int(rng.integers(1, 6))):
            m = int(rng.integers(1, 3000))
            src = rng.integers(0, nn, m); dst = rng.integers(0, nn, m)
            base = b * 10_000
            ts = np.sort(rng.integers(base, base + 10_000, m))
            if case % 2:  # out-of-order tail: rejections
                ts = ts.copy()
                k = rng.choice(m, size=max(1, m // 20), replace=False)
                ts[k] -= rng.integers(0, 20_000, size=len(k))
            got = gg.add_edges(src, dst, ts)
            want = o.add_edges(src, dst, ts)
            np.testing.assert_array_equal(got, want)
        assert_store_equal(export_store(gg.g), oracle_store(o), f"{directed} {sizing} case {case}")


def test_add_edges_api_semantics(cuda_device):
    import paper_2311_17410_b200 as gf

    g = gf.new_graph(directed=True)
    r = g.add_edges([(0, 1, 10), (0, 2, 5), (0, 3, 11)])  # reference tests/test_storage.py:99-105
    assert r.rejected == [1] and r.edge_ids[1] is None and g.degree(0) == 2
    assert [t for _, _, t, _ in g.iter_edges(0)] == [10, 11]
    with pytest.raises(ValueError):
        g.add_edges([(-1, 0, 3)])
    with pytest.raises(ValueError):
        gf.new_graph(tau=0)
    g2 = gf.new_graph(directed=False)
    assert g2.add_edges([(0, 1, 5), (1, 2, 5), (2, 0, 4), (3, 4, 1)]).edge_ids == [0, 1, None, 2]
    g3 = gf.new_graph(directed=True, tau=8192)
    g3.add_edges([(0, 1, t) for t in range(10_000)])
    assert g3.new_block_capacity(0) == 8192
    with pytest.raises(gf.NodeNotFoundError):
        g3.new_block_capacity(5)
    ids = g3.add_edges([(0, 1, 20_000)]).accepted_ids
    assert ids == [10_000]
    assert g3.delete_edges(ids) == 1 and g3.delete_edges(ids) == 0
    assert g3.delete_node(0) is True and g3.delete_node(0) is False
    with pytest.raises(gf.NodeNotFoundError):
        g3.degree(0)


def test_preassigned_ids_and_empty_batches(cuda_device):
    import paper_2311_17410_b200 as gf

    g = gf.new_graph(directed=True)
    assert g.add_edges([]).edge_ids == []
    r = g.add_edges([(0, 1, 1), (1, 2, 2)], edge_ids=[40, 41])
    assert r.edge_ids == [40, 41] and g.next_edge_id == 42
    with pytest.raises(ValueError):
        g.add_edges([(0, 1, 3)], edge_ids=[1, 2])


@pytest.mark.parametrize("directed", [True, False])
def test_cooperative_ingest_taken_and_equal(cuda_device, directed):
    """A time-sorted stream is committed by the cooperative single launch (k_ingest_coop), with hub
    segments above one warp (CTA radix sort), node-table growth and pool growth on the way; a batch
    with an out-of-order edge falls back to the general sequence.  Both equal the oracle."""
    import paper_2311_17410_b200 as gf
    from paper_2311_17410_b200 import _lib
    from gpu_helpers import assert_store_equal, export_store, oracle_store
    from oracle import OracleGraph

    rng = np.random.default_rng(11 + directed)
    g = gf.DynamicGraph(directed=directed, tau=48)
    o = OracleGraph(directed, 48)
    w = np.arange(1, 3001, dtype=np.float64) ** -1.2
    w /= w.sum()
    t0 = 0
    for b in range(8):
        m = int(rng.integers(1000, 20_000))
        nn = 500 * (b + 1)
        src = rng.choice(3000, size=m, p=w) % nn
        dst = rng.integers(0, nn, m)
        ts = np.sort(rng.integers(t0, t0 + 1000, m))
        t0 += 1000
        if b == 6:  # the same source earlier in the batch at a later time: a rejection, general sequence
            ts = ts.copy()
            src[m // 2] = src[0]
            ts[m // 2] = ts[0] - 1
        _lib.profile_enable(True)
        out, rej = g.add_edges_arrays(src, dst, ts)
        prof = _lib.profile_summary()
        _lib.profile_enable(False)
        want = o.add_edges(src, dst, ts)
        np.testing.assert_array_equal(out.cpu().numpy(), want, err_msg=f"batch {b}")
        assert rej == int((want < 0).sum())
        assert "k_ingest_coop" in prof
        assert ("k_commit" in prof) == (b == 6), (b, sorted(prof))
    assert_store_equal(export_store(g), oracle_store(o), f"directed={directed}")
