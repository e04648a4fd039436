"""Device offload (storage.py:516-574): TGOF blob bytes, unlink, LIFO handle reuse, sampling after offload."""

from __future__ import annotations

import io

import numpy as np
import pytest

from fixtures import TS_MIN, live_layout_from, load, replay_offload_case

pytestmark = pytest.mark.gpu


class _GpuOffloadAdapter:
    def __init__(self, m):
        import paper_2311_17410_b200 as gf

        sz = {"adaptive": None, "fixed": gf.FixedSizing(m["param"]), "batch": gf.BatchSizing()}[m["sizing"]]
        self.g = gf.DynamicGraph(directed=m["directed"], tau=m["tau"], sizing=sz)

    def add_edges(self, s, d, t):
        return self.g.add_edges_arrays(s, d, t)[0].cpu().numpy()

    def delete_edges(self, ids):
        return self.g.delete_edges(np.asarray(ids, dtype=np.int64))

    def offload(self, cutoff):
        buf = io.BytesIO()
        n = self.g.offload_before(cutoff, buf)
        return buf.getvalue(), n


def test_offload_matches_reference_fixtures(cuda_device):
    fx, meta = load("offload_cases.npz")
    for m in meta:
        p = f"o{m['id']}/"
        a = _GpuOffloadAdapter(m)
        for what, step, got, want in replay_offload_case(a, fx, p, m):
            if what == "n":
                assert got == want, (p, step)
            else:
                np.testing.assert_array_equal(got, want, err_msg=f"{p} {what} {step}")
        live = fx[p + "live"]
        arrs = a.g._block_arrays()
        sizes = a.g._export_blocks()["size"]

        def slots(h):
            x = arrs[h]
            s = int(sizes[h])
            return x.neighbors[:s], x.edge_ids[:s], x.timestamps[:s], x.valid[:s]

        lay = live_layout_from(a.g._export_nodes(), a.g._export_blocks(), slots, live)
        for k, v in lay.items():
            np.testing.assert_array_equal(v, fx[p + k], err_msg=f"{p} {k}")
        assert a.g.info().num_block_handles == m["num_block_handles"]
        st = a.g.storage_stats()
        assert [st.avg_list_len, st.max_list_len, st.edge_data_bytes, st.metadata_bytes, st.wasted_slots] == m["stats"]


def test_sampling_after_offload_matches_oracle(cuda_device):
    import paper_2311_17410_b200 as gf
    from oracle import OracleGraph

    rng = np.random.default_rng(4)
    for policy in ("recent", "uniform"):
        g = gf.DynamicGraph(directed=True, tau=8)
        o = OracleGraph(True, 8)
        t0 = 0
        for step in range(4):
            m = 3000
            s = rng.integers(0, 50, m); d = rng.integers(0, 50, m); ts = np.sort(rng.integers(t0, t0 + 10 * m, m))
            t0 = int(ts[-1])
            g.add_edges_arrays(s, d, ts)
            o.add_edges(s, d, ts)
            cut = int(rng.integers(0, t0))
            blob, n = o.offload_before(cut)
            buf = io.BytesIO()
            assert g.offload_before(cut, buf) == n and buf.getvalue() == blob
        q = rng.integers(0, 50, 2000); t1 = rng.integers(0, t0 + 5, 2000)
        t_lo = np.where(rng.random(2000) < 0.5, TS_MIN, t1 - rng.integers(0, t0, 2000))
        lay = gf.sample_layer(g, q, t_lo, t1, 7, gf.SamplingPolicy(policy), seed=3)
        want = o.sample_layer(q, t_lo, t1, 7, policy, seed=3)
        for nm, w in zip(("offsets", "neighbors", "edge_ids", "timestamps"), want):
            np.testing.assert_array_equal(getattr(lay, nm), w, err_msg=f"{policy} {nm}")


def test_offload_reference_goldens(cuda_device):
    """Reference tests/test_storage.py:167-232 on the device store."""
    import paper_2311_17410_b200 as gf

    def three_blocks():
        g = gf.DynamicGraph(directed=True, sizing=gf.FixedSizing(2))
        g.add_edges([(0, 1, 1), (0, 2, 5), (0, 3, 10), (0, 4, 15), (0, 5, 20), (0, 6, 30)])
        assert g.node_entry(0).num_blocks == 3
        return g

    g = three_blocks()
    sink = io.BytesIO()
    assert g.offload_before(0, sink) == 0 and sink.getvalue() == b"TGOF" + (1).to_bytes(4, "little")
    g = three_blocks()
    assert g.offload_before(31, io.BytesIO()) == 6
    e = g.node_entry(0)
    assert e.num_blocks == 0 and e.head_block is None and e.tail_block is None and e.degree == 0
    g = three_blocks()
    sink = io.BytesIO()
    assert g.offload_before(20, sink) == 4
    assert g.node_entry(0).num_blocks == 1 and [t for _, _, t, _ in g.iter_edges(0)] == [20, 30]
    recs = gf.parse_offload(io.BytesIO(sink.getvalue()))
    assert [(n, [r[2] for r in rs]) for n, rs in recs] == [(0, [1, 5]), (0, [10, 15])]
    assert gf.write_offload_records(recs) == sink.getvalue()
    lay = gf.sample_layer(g, [0], [TS_MIN], [100], 50, gf.SamplingPolicy.recent(), seed=0)
    assert sorted(lay.timestamps.tolist()) == [20, 30]

    class FailingSink:
        def write(self, data):
            raise OSError("disk full")

    g = three_blocks()
    with pytest.raises(OSError):
        g.offload_before(31, FailingSink())
    assert g.node_entry(0).num_blocks == 3 and g.degree(0) == 6
