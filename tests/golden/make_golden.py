"""Generate golden fixtures from the UNMODIFIED reference (``ctdg``).

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``ctdg`` from /root/reference/pkg/src and the reference's own test
corpus builder (``make_random_case`` in /root/reference/pkg/tests/conftest.py,
seed 20240817), drives the reference through the hot-path calls, and stores
inputs + outputs as small compressed ``.npz`` files next to this script.  The
fixtures travel with the repo; /root/reference does not.

Fixtures:
  store_cases.npz   ingest batches (incl. rejections, preassigned ids, all
                    sizing kinds, deletions) -> full block-store layout
  sample_cases.npz  recent sample_layer / sample_khop outputs (bit-exact) and
                    complete-fanout uniform/time_window outputs (as multisets)
  cache_cases.npz   fetch/insert traces for lru/lfu/fifo with per-call outputs
  feature_cases.npz NodeFeatureTable / EdgeFeatureTable lookups
  misc.json         hop_seed values, generator digests, Fig.1 goldens
"""

from __future__ import annotations

import hashlib
import importlib.util
import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
HERE = os.path.dirname(os.path.abspath(__file__))

sys.path.insert(0, REF_SRC)
sys.dont_write_bytecode = True
import ctdg  # noqa: E402
from ctdg import (  # noqa: E402
    BatchSizing,
    DynamicGraph,
    EdgeFeatureTable,
    FixedSizing,
    NodeFeatureTable,
    SampleRequest,
    SamplingPolicy,
    VectorCache,
    sample_khop,
    sample_layer,
)
from ctdg.sampling import hop_seed  # noqa: E402
from ctdg.storage import TS_MIN  # noqa: E402


def _ref_conftest():
    spec = importlib.util.spec_from_file_location("ref_conftest", os.path.join(REF_TESTS, "conftest.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules["ref_conftest"] = mod
    spec.loader.exec_module(mod)
    return mod


def dump_store(g: DynamicGraph, out: dict, p: str) -> None:
    f = g.fast
    out[p + "head"] = f.head.copy()
    out[p + "tail"] = f.tail.copy()
    out[p + "num_blocks"] = f.num_blocks.copy()
    out[p + "degree"] = f.degree.copy()
    out[p + "node_valid"] = f.node_valid.copy()
    nb = f._blk_used
    for name in ("blk_capacity", "blk_size", "blk_tmin", "blk_tmax", "blk_prev", "blk_next"):
        out[p + name] = getattr(f, name)[:nb].copy()
    offs, nbr, eid, ts, valid = [0], [], [], [], []
    for h in range(nb):
        a = g.shared.get(h)
        s = int(f.blk_size[h])
        nbr.append(a.neighbors[:s]); eid.append(a.edge_ids[:s]); ts.append(a.timestamps[:s]); valid.append(a.valid[:s])
        offs.append(offs[-1] + s)
    cat = (lambda xs, dt: np.concatenate(xs).astype(dt) if xs else np.zeros(0, dt))
    out[p + "slot_offsets"] = np.array(offs, np.int64)
    out[p + "slot_nbr"] = cat(nbr, np.int64)
    out[p + "slot_eid"] = cat(eid, np.int64)
    out[p + "slot_ts"] = cat(ts, np.int64)
    out[p + "slot_valid"] = cat(valid, bool)
    out[p + "next_edge_id"] = np.array([g.next_edge_id, g.total_edges_inserted], np.int64)


def store_cases() -> dict:
    rng = np.random.default_rng(20240817)
    cf = _ref_conftest()
    out: dict = {}
    meta = []
    i = 0
    # (a) the reference's own randomized corpus (sorted streams, deletions)
    for _ in range(40):
        case_rng_state = rng.bit_generator.state
        case = cf.make_random_case(rng, max_edges=300)
        # replay the exact batches: rebuild from the log with a fresh rng copy
        r2 = np.random.default_rng()
        r2.bit_generator.state = case_rng_state
        n_nodes = int(r2.integers(2, 60)); n_edges = int(r2.integers(1, 301)); directed = bool(r2.integers(0, 2))
        tau = int(r2.choice([1, 2, 4, 16, 48]))
        srcs = r2.integers(0, n_nodes, size=n_edges); dsts = r2.integers(0, n_nodes, size=n_edges)
        ts = np.sort(r2.integers(0, 10 * n_edges, size=n_edges))
        n_batches = int(r2.integers(1, 5))
        bounds = [len(c) for c in np.array_split(np.arange(n_edges), n_batches)]
        p = f"c{i}/"
        out[p + "src"], out[p + "dst"], out[p + "ts"] = srcs.astype(np.int64), dsts.astype(np.int64), ts.astype(np.int64)
        out[p + "batches"] = np.array(bounds, np.int64)
        out[p + "eids"] = np.array([e for _, _, _, e in case.edges], np.int64)
        out[p + "del_edges"] = np.array(sorted(case.deleted_edges), np.int64)
        out[p + "del_nodes"] = np.array(sorted(case.deleted_nodes), np.int64)
        assert case.graph.directed == directed and case.graph.tau == tau
        dump_store(case.graph, out, p)
        meta.append({"id": i, "directed": directed, "tau": tau, "sizing": "adaptive", "param": 0, "kind": "corpus"})
        i += 1
    # (b) unsorted streams -> rejections; preassigned ids; fixed/batch sizing
    for k in range(24):
        directed = bool(k % 2)
        n_nodes = int(rng.integers(2, 30))
        m = int(rng.integers(5, 200))
        src = rng.integers(0, n_nodes, size=m); dst = rng.integers(0, n_nodes, size=m)
        ts = rng.integers(0, 50, size=m)  # unsorted: rejections
        if k % 3 == 1:
            ts = np.sort(ts)
        sizing_kind = ["adaptive", "fixed", "batch"][k % 3]
        param = int(rng.integers(1, 6)) if sizing_kind == "fixed" else 0
        tau = int(rng.choice([1, 2, 3, 8, 48]))
        sizing = {"adaptive": None, "fixed": FixedSizing(max(param, 1)), "batch": BatchSizing()}[sizing_kind]
        g = DynamicGraph(directed=directed, tau=tau, sizing=sizing)
        n_batches = int(rng.integers(1, 4))
        bounds = [len(c) for c in np.array_split(np.arange(m), n_batches)]
        preassign = (k % 4 == 3)
        eids_in = (np.cumsum(rng.integers(1, 4, size=m)) + 5).astype(np.int64) if preassign else None
        res_ids = []
        pos = 0
        for b in bounds:
            batch = list(zip(src[pos:pos + b].tolist(), dst[pos:pos + b].tolist(), ts[pos:pos + b].tolist()))
            r = g.add_edges(batch, edge_ids=None if eids_in is None else eids_in[pos:pos + b].tolist())
            res_ids.extend(-1 if e is None else e for e in r.edge_ids)
            pos += b
        p = f"c{i}/"
        out[p + "src"], out[p + "dst"], out[p + "ts"] = src.astype(np.int64), dst.astype(np.int64), ts.astype(np.int64)
        out[p + "batches"] = np.array(bounds, np.int64)
        out[p + "eids"] = np.array(res_ids, np.int64)
        out[p + "eids_in"] = eids_in if eids_in is not None else np.zeros(0, np.int64)
        out[p + "del_edges"] = np.zeros(0, np.int64)
        out[p + "del_nodes"] = np.zeros(0, np.int64)
        dump_store(g, out, p)
        meta.append({"id": i, "directed": directed, "tau": tau, "sizing": sizing_kind, "param": param,
                     "kind": "reject" if k % 3 != 1 else "sorted", "preassigned": preassign})
        i += 1
    out["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    return out


def sample_cases() -> dict:
    """Recent outputs (bit-exact) on the reference corpus + complete-fanout uniform."""
    rng = np.random.default_rng(777)
    cf = _ref_conftest()
    out: dict = {}
    meta = []
    crng = np.random.default_rng(20240817)
    for i in range(30):
        st = crng.bit_generator.state
        case = cf.make_random_case(crng, max_edges=400)
        p = f"s{i}/"
        # record the build inputs by replaying the rng (same as store_cases)
        r2 = np.random.default_rng(); r2.bit_generator.state = st
        n_nodes = int(r2.integers(2, 60)); n_edges = int(r2.integers(1, 401)); directed = bool(r2.integers(0, 2))
        tau = int(r2.choice([1, 2, 4, 16, 48]))
        srcs = r2.integers(0, n_nodes, size=n_edges); dsts = r2.integers(0, n_nodes, size=n_edges)
        ts = np.sort(r2.integers(0, 10 * n_edges, size=n_edges))
        n_batches = int(r2.integers(1, 5))
        out[p + "src"], out[p + "dst"], out[p + "ts"] = srcs.astype(np.int64), dsts.astype(np.int64), ts.astype(np.int64)
        out[p + "batches"] = np.array([len(c) for c in np.array_split(np.arange(n_edges), n_batches)], np.int64)
        out[p + "del_edges"] = np.array(sorted(case.deleted_edges), np.int64)
        out[p + "del_nodes"] = np.array(sorted(case.deleted_nodes), np.int64)
        g = case.graph
        t_hi = case.max_ts() + 2
        nq = 64
        q_src = rng.integers(-2, g.num_nodes + 3, size=nq)
        q_t1 = rng.integers(-1, t_hi + 1, size=nq)
        q_t0 = np.where(rng.random(nq) < 0.5, TS_MIN, q_t1 - rng.integers(0, t_hi + 1, size=nq))
        for fi, f in enumerate((1, 3, 10)):
            lay = sample_layer(g, q_src, q_t0, q_t1, f, SamplingPolicy.recent(), seed=0)
            for nm in ("offsets", "neighbors", "edge_ids", "timestamps"):
                out[p + f"recent_f{f}_{nm}"] = getattr(lay, nm)
        lay = sample_layer(g, q_src, q_t0, q_t1, 10**9, SamplingPolicy.uniform(), seed=5)
        for nm in ("offsets", "neighbors", "edge_ids", "timestamps"):
            out[p + f"full_{nm}"] = getattr(lay, nm)
        lay = sample_layer(g, q_src, q_t0, q_t1, 10**9, SamplingPolicy.time_window(max(1, t_hi // 4)), seed=5)
        for nm in ("offsets", "neighbors", "edge_ids", "timestamps"):
            out[p + f"tw_{nm}"] = getattr(lay, nm)
        out[p + "q_src"], out[p + "q_t0"], out[p + "q_t1"] = q_src, q_t0, q_t1
        # multi-hop recent
        roots = rng.integers(0, g.num_nodes, size=16)
        rts = rng.integers(0, t_hi, size=16)
        lays = sample_khop(g, SampleRequest(roots.tolist(), rts.tolist(), [4, 3], SamplingPolicy.recent(), 0)).layers
        out[p + "khop_roots"], out[p + "khop_ts"] = roots, rts
        for h, lay in enumerate(lays):
            for nm in ("source_nodes", "source_times", "offsets", "neighbors", "edge_ids", "timestamps"):
                out[p + f"khop{h}_{nm}"] = getattr(lay, nm)
        meta.append({"id": i, "directed": directed, "tau": tau, "tw_delta": max(1, t_hi // 4)})
    out["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    return out


def cache_cases() -> dict:
    rng = np.random.default_rng(4242)
    out: dict = {}
    meta = []
    i = 0
    for policy in ("lru", "lfu", "fifo"):
        for capacity, lam, keyspace, dim in ((8, 1.0, 30, 3), (32, 0.2, 200, 5), (16, 0.5, 60, 4), (5, 0.25, 20, 2)):
            c = VectorCache(policy, capacity, dim, lam)
            p = f"k{i}/"
            calls = []
            for step in range(40):
                n = int(rng.integers(0, 25))
                keys = rng.integers(0, keyspace, size=n).astype(np.int64)
                values, hit, miss = c.fetch(keys)
                rows = (miss[:, None] * 10 + np.arange(dim)[None, :]).astype(np.float32) + 0.5
                admitted = c.insert_batch(miss, rows)
                out[p + f"{step}_keys"] = keys
                out[p + f"{step}_values"] = values
                out[p + f"{step}_hit"] = hit
                out[p + f"{step}_miss"] = miss
                out[p + f"{step}_cache_keys"] = c.keys.copy()
                out[p + f"{step}_cache_scores"] = c.scores.copy()
                calls.append({"admitted": admitted, "fifo_head": c.fifo_head, **c.stats()})
            out[p + "storage"] = c.storage.copy()
            meta.append({"id": i, "policy": policy, "capacity": capacity, "lam": lam, "dim": dim, "calls": calls})
            i += 1
    out["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    return out


def feature_cases() -> dict:
    rng = np.random.default_rng(99)
    out: dict = {}
    node = NodeFeatureTable(7)
    ids = rng.choice(500, size=120, replace=False)
    rows = rng.random((120, 7), dtype=np.float32)
    node.set_many(ids.tolist(), rows)
    q = rng.integers(-5, 520, size=300)
    v, f = node.get(q)
    out.update(node_ids=ids, node_rows=rows, node_q=q, node_v=v, node_f=f)
    edge = EdgeFeatureTable(6)
    all_ids, all_rows = [], []
    nxt = 0
    for _ in range(30):
        k = int(rng.integers(1, 12))
        e = nxt + np.cumsum(rng.integers(1, 4, size=k))
        nxt = int(e[-1])
        r = rng.random((k, 6), dtype=np.float32)
        edge.append(e, r)
        all_ids.append(e); all_rows.append(r)
    q = rng.integers(-3, nxt + 5, size=400)
    v, f = edge.get(q)
    out.update(edge_ids=np.concatenate(all_ids).astype(np.int64), edge_rows=np.concatenate(all_rows),
               edge_q=q, edge_v=v, edge_f=f)
    return out


def misc() -> dict:
    seeds = [0, 1, 7, 123, 2**31, 2**32 + 5, 2**63 + 11, 2**64 - 1, -1, -12345]
    hs = {f"{s}:{h}": str(hop_seed(s, h)) for s in seeds for h in range(4)}
    gens = {}
    for args in ((9000, 157000, 2.2, 2592000, 0, None), (17000, 200000, 2.2, 175200, 0, 2.2), (150, 6000, 2.0, 100000, 2, 2.0)):
        stream = ctdg.generate_synthetic(*args[:5], src_skew=args[5])
        a = np.asarray(stream, dtype=np.int64).reshape(-1, 3)
        gens[json.dumps(args)] = hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
    return {"hop_seed": hs, "generate_synthetic_sha256": gens}


def offload_cases() -> dict:
    """ingest -> offload(c1) -> ingest -> offload(c2) -> ingest: TGOF blobs, eids and the live layout.

    Later ingests reuse the freed block handles (LIFO, storage.py:171-191)."""
    import io

    rng = np.random.default_rng(31337)
    out: dict = {}
    meta = []
    for i in range(24):
        directed = bool(i % 2)
        tau = int(rng.choice([1, 2, 4, 16, 48]))
        sizing_kind = ["adaptive", "fixed", "adaptive", "batch"][i % 4]
        param = int(rng.integers(1, 6))
        sizing = {"adaptive": None, "fixed": FixedSizing(param), "batch": BatchSizing()}[sizing_kind]
        g = DynamicGraph(directed=directed, tau=tau, sizing=sizing)
        nn = int(rng.integers(2, 40))
        p = f"o{i}/"
        t0 = 0
        steps = []
        for step in range(3):
            m = int(rng.integers(1, 250))
            src = rng.integers(0, nn, m); dst = rng.integers(0, nn, m)
            ts = np.sort(rng.integers(t0, t0 + 5 * m, m))
            t0 = int(ts[-1])
            r = g.add_edges(list(zip(src.tolist(), dst.tolist(), ts.tolist())))
            out[p + f"{step}_src"], out[p + f"{step}_dst"], out[p + f"{step}_ts"] = src, dst, ts
            out[p + f"{step}_eids"] = np.array([-1 if e is None else e for e in r.edge_ids], np.int64)
            if step < 2:
                cutoff = int(rng.integers(0, t0 + 2))
                if i % 5 == 0 and step == 1:  # an edge deletion between offloads
                    ids = [e for e in r.edge_ids if e is not None][:3]
                    g.delete_edges(ids)
                    out[p + f"{step}_del"] = np.array(ids, np.int64)
                buf = io.BytesIO()
                n_off = g.offload_before(cutoff, buf)
                out[p + f"{step}_blob"] = np.frombuffer(buf.getvalue(), np.uint8).copy()
                steps.append({"cutoff": cutoff, "n": n_off})
        f = g.fast
        live = []
        for v in range(g.num_nodes):
            live.extend(g.blocks_of(v))
        out[p + "live"] = np.array(live, np.int64)
        for name in ("head", "tail", "num_blocks", "degree", "node_valid"):
            out[p + name] = getattr(f, name).copy()
        for name in ("blk_capacity", "blk_size", "blk_tmin", "blk_tmax", "blk_prev", "blk_next"):
            out[p + name] = getattr(f, name)[live].copy() if live else np.zeros(0, np.int64)
        offs, cols = [0], {"nbr": [], "eid": [], "ts": [], "valid": []}
        for h in live:
            a = g.shared.get(h)
            s = int(f.blk_size[h])
            cols["nbr"].append(a.neighbors[:s]); cols["eid"].append(a.edge_ids[:s])
            cols["ts"].append(a.timestamps[:s]); cols["valid"].append(a.valid[:s])
            offs.append(offs[-1] + s)
        out[p + "slot_offsets"] = np.array(offs, np.int64)
        for k, dt in (("nbr", np.int64), ("eid", np.int64), ("ts", np.int64), ("valid", bool)):
            out[p + "slot_" + k] = np.concatenate(cols[k]).astype(dt) if cols[k] else np.zeros(0, dt)
        st = g.storage_stats()
        meta.append({"id": i, "directed": directed, "tau": tau, "sizing": sizing_kind, "param": param, "steps": steps,
                     "stats": [st.avg_list_len, st.max_list_len, st.edge_data_bytes, st.metadata_bytes, st.wasted_slots],
                     "num_block_handles": int(f._blk_used)})
    out["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    return out


HARNESS_CONFIGS = [
    dict(generate_nodes=300, generate_edges=6000, generate_time_span=200_000, batch_edges=1000, epochs_per_round=2,
         replay_ratio=0.2, minibatch_size=200, fanouts=(5, 5), seed=3, label="lru"),
    dict(generate_nodes=500, generate_edges=8000, generate_time_span=500_000, batch_edges=2000, epochs_per_round=3,
         replay_ratio=0.0, minibatch_size=300, fanouts=(4, 3), seed=5, directed=True, tau=16, label="mixed",
         cache=dict(node_policy="lfu", edge_policy="fifo", node_capacity_frac=0.05, edge_capacity_frac=0.01, lam=0.5,
                    reuse=False, restore=False)),
    dict(generate_nodes=200, generate_edges=5000, generate_time_span=100_000, batch_by="time", batch_interval=20_000,
         epochs_per_round=2, replay_ratio=0.5, minibatch_size=150, fanouts=(6,), seed=7, label="time-batches",
         memory_dim=4, cache=dict(node_policy="lru", edge_policy="lfu", node_capacity_frac=0.1, edge_capacity_frac=0.02)),
]


def harness_reports() -> dict:
    """RoundReports of the reference's continuous loop (recent policy) for HARNESS_CONFIGS."""
    from ctdg.harness import CacheConfig, RunConfig, run_continuous

    out = {}
    for i, kw in enumerate(HARNESS_CONFIGS):
        kw = dict(kw)
        cache = CacheConfig(**kw.pop("cache", {}))
        cfg = RunConfig(**kw, cache=cache)
        out[str(i)] = {"config": HARNESS_CONFIGS[i], "reports": [r.to_json() for r in run_continuous(cfg)]}
    return out


def main() -> None:
    np.savez_compressed(os.path.join(HERE, "store_cases.npz"), **store_cases())
    np.savez_compressed(os.path.join(HERE, "sample_cases.npz"), **sample_cases())
    np.savez_compressed(os.path.join(HERE, "cache_cases.npz"), **cache_cases())
    np.savez_compressed(os.path.join(HERE, "feature_cases.npz"), **feature_cases())
    with open(os.path.join(HERE, "misc.json"), "w") as fh:
        json.dump(misc(), fh, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "offload_cases.npz"), **offload_cases())
    if not os.path.exists(os.path.join(HERE, "harness_reports.json")) or os.environ.get("GOLDEN_HARNESS"):
        with open(os.path.join(HERE, "harness_reports.json"), "w") as fh:
            json.dump(harness_reports(), fh, indent=1)


if __name__ == "__main__":
    main()
