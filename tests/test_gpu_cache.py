"""K4-K7 parity: the device VectorCache, feature tables and fetch block vs the reference."""

from __future__ import annotations

import io
from collections import OrderedDict

import numpy as np
import pytest

from fixtures import load

pytestmark = pytest.mark.gpu


def rows(keys, dim=2):
    return np.array([np.full(dim, float(k), np.float32) for k in keys], np.float32).reshape(len(list(keys)), dim)


def test_cache_traces_match_reference_fixtures(cuda_device):
    import paper_2311_17410_b200 as gf

    fx, meta = load("cache_cases.npz")
    for m in meta:
        p = f"k{m['id']}/"
        c = gf.VectorCache(m["policy"], m["capacity"], m["dim"], m["lam"])
        for step, call in enumerate(m["calls"]):
            keys = fx[p + f"{step}_keys"]
            values, hit, miss = c.fetch(keys)
            np.testing.assert_array_equal(hit, fx[p + f"{step}_hit"], err_msg=f"{p}{step}")
            np.testing.assert_array_equal(miss, fx[p + f"{step}_miss"], err_msg=f"{p}{step}")
            np.testing.assert_array_equal(values, fx[p + f"{step}_values"], err_msg=f"{p}{step}")
            r = (miss[:, None] * 10 + np.arange(m["dim"])[None, :]).astype(np.float32) + 0.5
            assert c.insert_batch(miss, r) == call["admitted"]
            np.testing.assert_array_equal(c.keys, fx[p + f"{step}_cache_keys"], err_msg=f"{p}{step}")
            np.testing.assert_array_equal(c.scores, fx[p + f"{step}_cache_scores"], err_msg=f"{p}{step}")
            assert c.fifo_head == call["fifo_head"]
            st = c.stats()
            assert (st["hits"], st["misses"], st["evictions"]) == (call["hits"], call["misses"], call["evictions"])
        np.testing.assert_array_equal(c.storage, fx[p + "storage"])


class ScalarLRU:  # reference tests/test_cache.py:24-42 (restated)
    def __init__(self, cap):
        self.cap, self.e, self.trace, self.evicted = cap, OrderedDict(), [], []

    def access(self, k):
        hit = k in self.e
        self.trace.append(hit)
        if hit:
            self.e.move_to_end(k)
        else:
            if len(self.e) == self.cap:
                self.evicted.append(self.e.popitem(last=False)[0])
            self.e[k] = None


class ScalarFIFO(ScalarLRU):
    def access(self, k):
        hit = k in self.e
        self.trace.append(hit)
        if not hit:
            if len(self.e) == self.cap:
                self.evicted.append(self.e.popitem(last=False)[0])
            self.e[k] = None


class ScalarLFU:  # reference tests/test_cache.py:45-72
    def __init__(self, cap):
        self.cap, self.slots, self.count, self.trace, self.evicted = cap, [None] * cap, {}, [], []

    def access(self, k):
        hit = k in self.count
        self.trace.append(hit)
        if hit:
            self.count[k] += 1
            return
        if None in self.slots:
            s = self.slots.index(None)
        else:
            s = min(range(self.cap), key=lambda i: (self.count[self.slots[i]], i))
            v = self.slots[s]
            self.evicted.append(v)
            del self.count[v]
        self.slots[s] = k
        self.count[k] = 1


@pytest.mark.parametrize("policy,ref", [("lru", ScalarLRU), ("lfu", ScalarLFU), ("fifo", ScalarFIFO)])
def test_single_key_trace_matches_scalar_reference(cuda_device, policy, ref):
    import paper_2311_17410_b200 as gf

    rng = np.random.default_rng(99)
    keys = rng.integers(0, 120, size=2500).tolist()
    c = gf.VectorCache(policy, 32, 2, lam=1.0)
    trace, ev = [], []
    for k in keys:
        _, hit, miss = c.fetch([k])
        trace.append(bool(hit[0]))
        if len(miss):
            before = {int(x) for x in c.keys if x != -1}
            c.insert_batch(miss, rows(miss))
            after = {int(x) for x in c.keys if x != -1}
            ev.extend(sorted(before - after))
    r = ref(32)
    for k in keys:
        r.access(k)
    assert trace == r.trace and ev == r.evicted


def test_cache_semantics_goldens(cuda_device):
    import paper_2311_17410_b200 as gf
    from paper_2311_17410_b200.cache import SnapshotFormatError, SnapshotMismatchError

    c = gf.VectorCache("lru", 4, 2, lam=1.0)
    v, h, m = c.fetch([1, 2])
    assert h.tolist() == [False, False] and m.tolist() == [1, 2] and np.all(v == 0)
    c.insert_batch([1], rows([1]))
    v, h, m = c.fetch([1, 1, 2])
    assert h.tolist() == [True, True, False] and m.tolist() == [2] and np.array_equal(v[1], rows([1])[0])
    c = gf.VectorCache("lru", 4, 2, lam=1.0)
    c.insert_batch([1, 2, 3], rows([1, 2, 3]))
    c.fetch([1, 1])
    s = {int(c.keys[i]): int(c.scores[i]) for i in range(4) if c.keys[i] != -1}
    assert s == {1: 0, 2: -1, 3: -1}
    c = gf.VectorCache("lfu", 4, 2, lam=1.0)
    c.insert_batch([1, 2], rows([1, 2]))
    c.fetch([1, 1, 2])
    s = {int(c.keys[i]): int(c.scores[i]) for i in range(4) if c.keys[i] != -1}
    assert s == {1: 3, 2: 2}
    c = gf.VectorCache("lru", 100, 2, lam=0.2)
    assert c.insert_batch(list(range(50)), rows(range(50))) == 20 and sorted(c.slot_of) == list(range(20))
    c = gf.VectorCache("lru", 4, 2, lam=1.0)
    c.insert_batch([10, 11, 12, 13], rows([10, 11, 12, 13]))
    c.scores[:] = np.array([-3, -1, 0, -2])  # write-through, reference tests/test_cache.py:171
    c.insert_batch([99], rows([99]))
    assert 10 not in c.slot_of and 99 in c.slot_of
    c = gf.VectorCache("fifo", 3, 2, lam=1.0)
    for k in (1, 2, 3, 4):
        c.insert_batch([k], rows([k]))
    assert sorted(c.slot_of) == [2, 3, 4]
    with pytest.raises(ValueError):
        gf.VectorCache("lru", 4, 3, lam=1.0).insert_batch([1], np.zeros((1, 2), np.float32))
    c = gf.VectorCache("lru", 4, 2, lam=1.0)
    c.insert_batch([1], rows([1]))
    with pytest.raises(ValueError):
        c.insert_batch([1], rows([1]))
    with pytest.raises(ValueError):
        gf.VectorCache("mru", 4, 2)
    # snapshot / restore / persist (reference tests/test_cache.py:268-327)
    c = gf.VectorCache("lru", 8, 2, lam=1.0)
    c.insert_batch([1, 2, 3], rows([1, 2, 3]))
    snap = c.snapshot()
    dsnap = c.device_snapshot()
    c.fetch([9, 9, 9])
    c.insert_batch([9], rows([9]))
    c.restore(snap)
    assert np.array_equal(c.keys, snap.keys) and np.array_equal(c.scores, snap.scores)
    c.fetch([1, 5])
    dsnap.restore_into(c)
    assert np.array_equal(c.keys, snap.keys) and np.array_equal(c.scores, snap.scores)
    with pytest.raises(SnapshotMismatchError):
        c.restore(gf.VectorCache("lfu", 8, 2, lam=1.0).snapshot())
    for policy in ("lru", "lfu", "fifo"):
        c = gf.VectorCache(policy, 8, 3, lam=0.5)
        c.insert_batch([4, 1], rows([4, 1], 3))
        c.fetch([4, 7])
        buf = io.BytesIO()
        c.persist(buf)
        blob = buf.getvalue()
        loaded = gf.load_cache(io.BytesIO(blob))
        buf2 = io.BytesIO()
        loaded.persist(buf2)
        assert buf2.getvalue() == blob
        assert loaded.fetch([4, 1, 2])[1].tolist() == [True, True, False]
    with pytest.raises(SnapshotFormatError):
        gf.load_cache(io.BytesIO(b"garbage"))


def test_feature_tables_match_reference_fixtures(cuda_device):
    import paper_2311_17410_b200 as gf

    fx, _ = load("feature_cases.npz")
    n = gf.NodeFeatureTable(7)
    n.set_many(fx["node_ids"], fx["node_rows"])
    v, f = n.get(fx["node_q"])
    np.testing.assert_array_equal(v, fx["node_v"])
    np.testing.assert_array_equal(f, fx["node_f"])
    e = gf.EdgeFeatureTable(6)
    ids, rws = fx["edge_ids"], fx["edge_rows"]
    for chunk in np.array_split(np.arange(len(ids)), 7):
        e.append(ids[chunk], rws[chunk])
    v, f = e.get(fx["edge_q"])
    np.testing.assert_array_equal(v, fx["edge_v"])
    np.testing.assert_array_equal(f, fx["edge_f"])
    with pytest.raises(ValueError):
        e.append([int(ids[-1])], rws[:1])


@pytest.mark.parametrize("policy", ["lru", "lfu", "fifo"])
@pytest.mark.parametrize("dim", [16, 186, 413])
def test_fetch_block_matches_harness_semantics(cuda_device, policy, dim):
    """harness.py:438-446 (fetch -> table.get(miss) -> insert_batch(found)) vs the oracle."""
    import torch

    import paper_2311_17410_b200 as gf
    from oracle import CacheOracle, EdgeFeatureOracle

    rng = np.random.default_rng(dim)
    m = 5000
    ids = np.cumsum(rng.integers(1, 3, m)).astype(np.int64)
    feats = rng.random((m, dim), dtype=np.float32)
    table = gf.EdgeFeatureTable(dim)
    table.append(ids, feats)
    ot = EdgeFeatureOracle(dim)
    ot.append(ids, feats)
    cache = gf.VectorCache(policy, 300, dim, 0.2)
    oc = CacheOracle(policy, 300, dim, 0.2)
    for it in range(12):
        keys = rng.choice(np.concatenate([ids[: 400 + 300 * it], [10**9, -5]]), size=2000)
        vals, hit, nm, adm = gf.fetch_features(cache, table, torch.from_numpy(keys).cuda())
        _, ohit, omiss = oc.fetch(keys)
        r, found = ot.get(omiss)
        oadm = oc.insert_batch(omiss[found], r[found])
        assert np.array_equal(hit.cpu().numpy(), ohit) and nm == len(omiss) and adm == oadm
        full, _ = ot.get(keys)
        np.testing.assert_array_equal(vals.cpu().numpy(), full)
    np.testing.assert_array_equal(cache.keys, oc.keys)
    np.testing.assert_array_equal(cache.scores, oc.scores)
    np.testing.assert_array_equal(cache.storage, oc.storage)
    st = cache.stats()
    assert (st["hits"], st["misses"], st["evictions"]) == (oc.hits, oc.misses, oc.evictions)
