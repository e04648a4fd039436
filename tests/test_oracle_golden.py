"""Pin the CPU oracle against the reference's golden fixtures (CPU only).

Every fixture was produced by the unmodified reference (tests/golden/make_golden.py).
When /root/reference is present (build container) a few tests also run the
live reference side by side.
"""

from __future__ import annotations

import os
import sys
from collections import Counter

import numpy as np
import pytest

from fixtures import TS_MIN, load, misc, replay_build
from oracle import CacheOracle, EdgeFeatureOracle, NodeFeatureOracle, OracleGraph, child_key, hop_seed
from oracle.oracle import build as build_oracle

REF = "/root/reference/pkg/src"


def setup_module(_):
    build_oracle()


def _oracle_factory(directed, tau, sizing, param):
    return OracleGraph(directed=directed, tau=tau, sizing=sizing, sizing_param=param)


def _check_store(g: OracleGraph, fx: dict, p: str):
    nodes = g.export_nodes()
    for k in ("head", "tail", "num_blocks", "degree", "node_valid"):
        np.testing.assert_array_equal(nodes[k], fx[p + k], err_msg=p + k)
    blks = g.export_blocks()
    for ours, theirs in (("capacity", "blk_capacity"), ("size", "blk_size"), ("tmin", "blk_tmin"),
                         ("tmax", "blk_tmax"), ("prev", "blk_prev"), ("next", "blk_next")):
        np.testing.assert_array_equal(blks[ours], fx[p + theirs], err_msg=p + theirs)
    offs = fx[p + "slot_offsets"]
    for h in range(len(offs) - 1):
        nbr, eid, ts, valid = g.block_edges(h)
        sl = slice(offs[h], offs[h + 1])
        np.testing.assert_array_equal(nbr, fx[p + "slot_nbr"][sl])
        np.testing.assert_array_equal(eid, fx[p + "slot_eid"][sl])
        np.testing.assert_array_equal(ts, fx[p + "slot_ts"][sl])
        np.testing.assert_array_equal(valid, fx[p + "slot_valid"][sl])
    ne = fx[p + "next_edge_id"]
    assert g.next_edge_id == ne[0] and g.total_edges_inserted == ne[1]


def test_oracle_store_layout_matches_reference():
    fx, meta = load("store_cases.npz")
    for m in meta:
        p = f"c{m['id']}/"
        g, eids = replay_build(_oracle_factory, fx, p, m)
        np.testing.assert_array_equal(eids, fx[p + "eids"], err_msg=p)
        _check_store(g, fx, p)


def test_oracle_recent_matches_reference_bitwise():
    fx, meta = load("sample_cases.npz")
    for m in meta:
        p = f"s{m['id']}/"
        g, _ = replay_build(_oracle_factory, fx, p, {**m, "sizing": "adaptive", "param": 0})
        for faithful in (True, False):
            for f in (1, 3, 10):
                offs, nb, eid, ts = g.sample_layer(fx[p + "q_src"], fx[p + "q_t0"], fx[p + "q_t1"], f, "recent",
                                                   faithful=faithful)
                np.testing.assert_array_equal(offs, fx[p + f"recent_f{f}_offsets"])
                np.testing.assert_array_equal(nb, fx[p + f"recent_f{f}_neighbors"])
                np.testing.assert_array_equal(eid, fx[p + f"recent_f{f}_edge_ids"])
                np.testing.assert_array_equal(ts, fx[p + f"recent_f{f}_timestamps"])


@pytest.mark.parametrize("kind", ["full", "tw"])
def test_oracle_complete_fanout_multisets(kind):
    """At fanout 1e9 uniform/time_window return every candidate: multisets must match."""
    fx, meta = load("sample_cases.npz")
    for m in meta:
        p = f"s{m['id']}/"
        g, _ = replay_build(_oracle_factory, fx, p, {**m, "sizing": "adaptive", "param": 0})
        policy, delta = ("uniform", 0) if kind == "full" else ("time_window", m["tw_delta"])
        for faithful in (True, False):
            offs, nb, eid, ts = g.sample_layer(fx[p + "q_src"], fx[p + "q_t0"], fx[p + "q_t1"], 10**9, policy, delta,
                                               seed=5, faithful=faithful)
            np.testing.assert_array_equal(offs, fx[p + f"{kind}_offsets"])
            for i in range(len(offs) - 1):
                a = slice(offs[i], offs[i + 1])
                got = Counter(zip(nb[a].tolist(), eid[a].tolist(), ts[a].tolist()))
                want = Counter(zip(fx[p + f"{kind}_neighbors"][a].tolist(), fx[p + f"{kind}_edge_ids"][a].tolist(),
                                   fx[p + f"{kind}_timestamps"][a].tolist()))
                assert got == want


def test_oracle_khop_recent_matches_reference():
    fx, meta = load("sample_cases.npz")
    for m in meta:
        p = f"s{m['id']}/"
        g, _ = replay_build(_oracle_factory, fx, p, {**m, "sizing": "adaptive", "param": 0})
        layers = g.sample_khop(fx[p + "khop_roots"], fx[p + "khop_ts"], [4, 3], "recent")
        for h, lay in enumerate(layers):
            for nm, arr in zip(("source_nodes", "source_times", "offsets", "neighbors", "edge_ids", "timestamps"), lay):
                np.testing.assert_array_equal(arr, fx[p + f"khop{h}_{nm}"], err_msg=f"{p} hop{h} {nm}")


def test_hop_seed_matches_numpy_seedsequence():
    for k, v in misc()["hop_seed"].items():
        s, h = (int(x) for x in k.split(":"))
        assert hop_seed(s, h) == int(v), k
    # measured in SURVEY.md A3
    assert hop_seed(0, 0) == 15793235383387715774
    assert hop_seed(0, 1) == 5836529245451711556
    rng = np.random.default_rng(3)
    for s in rng.integers(0, 2**63, size=50).tolist():
        for h in (0, 1, 2, 70000, 2**33):
            want = int(np.random.SeedSequence([s, h]).generate_state(1, dtype=np.uint64)[0])
            assert hop_seed(s, h) == want


def test_child_keys_vectorised_match_scalar():
    from oracle.oracle import _child_keys_vec

    parent = np.array([0, 1, 2**63, 2**64 - 1, 12345], dtype=np.uint64)
    j = np.array([0, 5, 9, 1, 100], dtype=np.int64)
    v = _child_keys_vec(parent, j)
    for a, b, c in zip(parent.tolist(), j.tolist(), v.tolist()):
        assert child_key(a, b) == c


def test_cache_oracle_matches_reference_traces():
    fx, meta = load("cache_cases.npz")
    for m in meta:
        p = f"k{m['id']}/"
        c = CacheOracle(m["policy"], m["capacity"], m["dim"], m["lam"])
        for step, call in enumerate(m["calls"]):
            keys = fx[p + f"{step}_keys"]
            values, hit, miss = c.fetch(keys)
            np.testing.assert_array_equal(hit, fx[p + f"{step}_hit"])
            np.testing.assert_array_equal(miss, fx[p + f"{step}_miss"])
            np.testing.assert_array_equal(values, fx[p + f"{step}_values"])
            rows = (miss[:, None] * 10 + np.arange(m["dim"])[None, :]).astype(np.float32) + 0.5
            assert c.insert_batch(miss, rows) == call["admitted"]
            np.testing.assert_array_equal(c.keys, fx[p + f"{step}_cache_keys"])
            np.testing.assert_array_equal(c.scores, fx[p + f"{step}_cache_scores"])
            assert c.fifo_head == call["fifo_head"]
            st = c.stats()
            assert (st["hits"], st["misses"], st["evictions"]) == (call["hits"], call["misses"], call["evictions"])
        np.testing.assert_array_equal(c.storage, fx[p + "storage"])


def test_feature_oracles_match_reference():
    fx, _ = load("feature_cases.npz")
    n = NodeFeatureOracle(7)
    n.set_many(fx["node_ids"], fx["node_rows"])
    v, f = n.get(fx["node_q"])
    np.testing.assert_array_equal(v, fx["node_v"])
    np.testing.assert_array_equal(f, fx["node_f"])
    e = EdgeFeatureOracle(6)
    e.append(fx["edge_ids"], fx["edge_rows"])
    v, f = e.get(fx["edge_q"])
    np.testing.assert_array_equal(v, fx["edge_v"])
    np.testing.assert_array_equal(f, fx["edge_f"])


def test_oracle_fig1_goldens():
    """Reference tests/test_sampling.py:44-62,137-167,189-208 restated on the oracle."""
    g = OracleGraph(directed=False, tau=48)
    A, B, C, D = 0, 1, 2, 3
    g.add_edges([A, B, C, A], [C, C, D, C], [12, 14, 16, 23])
    offs, nb, eid, ts = g.sample_layer([A], [TS_MIN], [24], 10)
    assert nb.tolist() == [C, C] and sorted(ts.tolist()) == [12, 23]
    layers = g.sample_khop([A], [24], [10, 10], "recent")
    hop2 = layers[1]
    assert hop2[0].tolist() == [C, C]
    by = {(int(hop2[0][i]), int(hop2[1][i])): sorted(hop2[3][hop2[2][i]:hop2[2][i + 1]].tolist())
          for i in range(len(hop2[0]))}
    assert by[(C, 23)] == [A, B, D] and by[(C, 12)] == []
    g2 = OracleGraph(directed=True)
    g2.add_edges([0, 0, 0, 0], [1, 2, 3, 4], [1, 5, 9, 12])
    assert g2.sample_layer([0], [0], [10], 2)[3].tolist() == [9, 5]
    g3 = OracleGraph(directed=True)
    ids = g3.add_edges([0, 0, 0], [1, 2, 3], [7, 7, 7])
    assert g3.sample_layer([0], [TS_MIN], [8], 2)[2].tolist() == [ids[2], ids[1]]
    g4 = OracleGraph(directed=True)
    g4.add_edges([0, 0, 0], [1, 2, 3], [1, 5, 9])
    assert sorted(g4.sample_layer([0], [TS_MIN], [10], 10**9, "time_window", 5)[3].tolist()) == [5, 9]
    assert g4.sample_layer([0, 99], [0, 0], [10, 10], 10**9)[0].tolist() == [0, 3, 3]
    # rejection example measured in SURVEY.md 8(a') rule 11
    g5 = OracleGraph(directed=False)
    assert g5.add_edges([0, 1, 2, 3], [1, 2, 0, 4], [5, 5, 4, 1]).tolist() == [0, 1, -1, 2]


def test_oracle_uniform_frequencies_within_4_sigma():
    """Reference tests/test_sampling.py:93-105 on the oracle's Philox+Floyd stream."""
    g = OracleGraph(directed=True)
    g.add_edges([0] * 20, list(range(1, 21)), list(range(20)))
    reps, f, n = 10_000, 5, 20
    counts = Counter()
    for seed in range(reps):
        counts.update(g.sample_layer([0], [TS_MIN], [100], f, "uniform", seed=seed)[1].tolist())
    p = f / n
    sigma = (p * (1 - p) / reps) ** 0.5
    for nbr in range(1, n + 1):
        assert abs(counts[nbr] / reps - p) <= 4 * sigma


def test_oracle_thread_count_invariance():
    fx, meta = load("sample_cases.npz")
    m = meta[3]
    p = f"s{m['id']}/"
    g, _ = replay_build(_oracle_factory, fx, p, {**m, "sizing": "adaptive", "param": 0})
    base = g.sample_layer(fx[p + "q_src"], fx[p + "q_t0"], fx[p + "q_t1"], 3, "uniform", seed=9, threads=1)
    for t in (2, 4, 7):
        got = g.sample_layer(fx[p + "q_src"], fx[p + "q_t0"], fx[p + "q_t1"], 3, "uniform", seed=9, threads=t)
        for a, b in zip(base, got):
            np.testing.assert_array_equal(a, b)


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted (GPU box)")
def test_oracle_against_live_reference_random_corpus():
    """Side-by-side with the live reference on fresh random cases (build container only)."""
    sys.path.insert(0, REF)
    import ctdg  # noqa: F401
    from ctdg import DynamicGraph, SamplingPolicy, sample_layer

    rng = np.random.default_rng(11)
    for case in range(15):
        directed = bool(case % 2)
        tau = int(rng.choice([1, 2, 4, 16, 48]))
        m = int(rng.integers(1, 400))
        nn = int(rng.integers(2, 40))
        src = rng.integers(0, nn, m); dst = rng.integers(0, nn, m); ts = rng.integers(0, 3 * m, m)
        ref = DynamicGraph(directed=directed, tau=tau)
        r = ref.add_edges(list(zip(src.tolist(), dst.tolist(), ts.tolist())))
        ora = OracleGraph(directed=directed, tau=tau)
        got = ora.add_edges(src, dst, ts)
        assert got.tolist() == [-1 if e is None else e for e in r.edge_ids]
        q = rng.integers(0, nn, 40); t1 = rng.integers(0, 3 * m + 2, 40)
        lay = sample_layer(ref, q, np.full(40, TS_MIN), t1, 4, SamplingPolicy.recent(), 0)
        offs, nb, eid, tts = ora.sample_layer(q, np.full(40, TS_MIN), t1, 4)
        assert offs.tolist() == lay.offsets.tolist() and nb.tolist() == lay.neighbors.tolist()
        assert eid.tolist() == lay.edge_ids.tolist() and tts.tolist() == lay.timestamps.tolist()


class _OracleOffloadAdapter:
    def __init__(self, m):
        self.g = OracleGraph(m["directed"], m["tau"], m["sizing"], m["param"])

    def add_edges(self, s, d, t):
        return self.g.add_edges(s, d, t)

    def delete_edges(self, ids):
        return self.g.delete_edges(ids)

    def offload(self, cutoff):
        return self.g.offload_before(cutoff)


def test_oracle_offload_matches_reference():
    """storage.py:516-574 incl. TGOF bytes and LIFO handle reuse by later ingests."""
    from fixtures import live_layout_from, replay_offload_case

    fx, meta = load("offload_cases.npz")
    for m in meta:
        p = f"o{m['id']}/"
        a = _OracleOffloadAdapter(m)
        for what, step, got, want in replay_offload_case(a, fx, p, m):
            if what == "n":
                assert got == want, (p, step)
            else:
                np.testing.assert_array_equal(got, want, err_msg=f"{p} {what} {step}")
        live = fx[p + "live"]
        lay = live_layout_from(a.g.export_nodes(), a.g.export_blocks(), lambda h: a.g.block_edges(h), live)
        for k, v in lay.items():
            np.testing.assert_array_equal(v, fx[p + k], err_msg=f"{p} {k}")
        assert a.g.num_block_handles == m["num_block_handles"]
