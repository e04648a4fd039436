"""Two processes driving libgfb200 on one GPU, collectives over gloo (world_size 2).

The multi-GPU paths (replicated ingest + root sharding, SURVEY.md 8(e);
partitioned sampling, cluster.py:226-292) run their real per-rank engine --
the CUDA library, not the oracle -- in two ranks that share cuda:0 (NCCL
refuses two ranks on one device, so the collectives go over gloo on host
buffers).  The union of the ranks' outputs must equal a one-process sample of
all roots bit for bit, the reference's distributed == local property
(tests/test_cluster.py:62-84).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _stream():
    from paper_2311_17410_b200.synth import generate_synthetic_arrays

    return generate_synthetic_arrays(700, 60_000, 2.2, 80_000, seed=5, src_skew=2.2)


def _roots(src, dst, ts):
    return np.concatenate([src[-500:], dst[-500:]]), np.concatenate([ts[-500:], ts[-500:]])


POLICIES = ("recent", "uniform", "time_window")


def _policy(name):
    import paper_2311_17410_b200 as gf

    return gf.SamplingPolicy(name, 2_000) if name == "time_window" else gf.SamplingPolicy(name)


def _replicated_worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2311_17410_b200 as gf
        from paper_2311_17410_b200.distributed import ReplicatedGraph, exclusive_prefix, shard_range

        dev = torch.device("cuda:0")
        torch.cuda.set_device(dev)
        rg = ReplicatedGraph(gf.DynamicGraph(directed=True, tau=64, device=dev))
        src, dst, ts = _stream()
        for lo in range(0, len(src), 9_000):
            hi = min(len(src), lo + 9_000)
            a, b = shard_range(hi - lo, world, rank)
            eids, rej = rg.ingest(torch.from_numpy(src[lo + a:lo + b]).to(dev), torch.from_numpy(dst[lo + a:lo + b]).to(dev),
                                  torch.from_numpy(ts[lo + a:lo + b]).to(dev))
            assert rej == 0
        roots, rts = _roots(src, dst, ts)
        lo, hi = (0, 333) if rank == 0 else (333, len(roots))  # uneven root shards
        base, total = exclusive_prefix(hi - lo)
        assert base == lo and total == len(roots)
        res = {}
        for pol in POLICIES:
            s = gf.sample_khop_device(rg.graph, torch.from_numpy(roots[lo:hi]).to(dev), torch.from_numpy(rts[lo:hi]).to(dev),
                                      [6, 4], _policy(pol), seed=9, root_key_base=base)
            for h, lay in enumerate(s.layers):
                for nm in ("offsets", "neighbors", "edge_ids", "timestamps"):
                    res[f"{pol}_{h}_{nm}"] = getattr(lay, nm).cpu().numpy()
        f = rg.graph.fast
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), degree=f.degree, num_blocks=f.num_blocks,
                 blk_capacity=f.blk_capacity, **res)
    finally:
        dist.destroy_process_group()


def _single_process(directed):
    import paper_2311_17410_b200 as gf

    dev = torch.device("cuda:0")
    g = gf.DynamicGraph(directed=directed, tau=64 if directed else 32, device=dev)
    src, dst, ts = _stream()
    step = 9_000 if directed else 5_000
    for lo in range(0, len(src), step):
        g.add_edges_arrays(src[lo:lo + step], dst[lo:lo + step], ts[lo:lo + step])
    return g, src, dst, ts


def test_replicated_two_ranks_libgfb200_equal_single_process(tmp_path):
    mp.spawn(_replicated_worker, args=(2, _port(), str(tmp_path)), nprocs=2, join=True)
    import paper_2311_17410_b200 as gf

    g, src, dst, ts = _single_process(True)
    parts = [np.load(tmp_path / f"rank{r}.npz") for r in range(2)]
    f = g.fast
    for p in parts:  # identical replicas
        for k in ("degree", "num_blocks", "blk_capacity"):
            np.testing.assert_array_equal(p[k], getattr(f, k))
    roots, rts = _roots(src, dst, ts)
    dev = torch.device("cuda:0")
    for pol in POLICIES:
        want = gf.sample_khop_device(g, torch.from_numpy(roots).to(dev), torch.from_numpy(rts).to(dev), [6, 4],
                                     _policy(pol), seed=9)
        for h, lay in enumerate(want.layers):
            for nm in ("neighbors", "edge_ids", "timestamps"):
                got = np.concatenate([p[f"{pol}_{h}_{nm}"] for p in parts])
                np.testing.assert_array_equal(got, getattr(lay, nm).cpu().numpy(), err_msg=f"{pol} hop{h} {nm}")
            cnt = np.concatenate([np.diff(p[f"{pol}_{h}_offsets"]) for p in parts])
            np.testing.assert_array_equal(cnt, np.diff(lay.offsets.cpu().numpy()))


def _partitioned_worker(rank, world, port, out_dir, directed):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2311_17410_b200.distributed import shard_range
        from paper_2311_17410_b200.partitioned import DistTransport, GpuEngine, PartitionedGraph

        dev = torch.device("cuda:0")
        torch.cuda.set_device(dev)
        pg = PartitionedGraph(DistTransport(), GpuEngine(tau=64 if directed else 32, device=dev), directed=directed)
        src, dst, ts = _stream()
        step = 9_000 if directed else 5_000
        for lo in range(0, len(src), step):
            hi = min(len(src), lo + step)
            a, b = shard_range(hi - lo, world, rank)
            pg.add_edges(torch.from_numpy(src[lo + a:lo + b]), torch.from_numpy(dst[lo + a:lo + b]),
                         torch.from_numpy(ts[lo + a:lo + b]))
        roots, rts = _roots(src, dst, ts)
        lo, hi = shard_range(len(roots), world, rank)
        res = {}
        for pol in POLICIES:
            s = pg.sample_khop(torch.from_numpy(roots[lo:hi]), torch.from_numpy(rts[lo:hi]), [6, 4], _policy(pol),
                               seed=9, root_key_base=lo)
            for h, lay in enumerate(s.layers):
                for nm in ("offsets", "neighbors", "edge_ids", "timestamps"):
                    res[f"{pol}_{h}_{nm}"] = getattr(lay, nm).cpu().numpy()
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("directed", [True, False])
def test_partitioned_two_ranks_libgfb200_equal_unpartitioned(tmp_path, directed):
    mp.spawn(_partitioned_worker, args=(2, _port(), str(tmp_path), directed), nprocs=2, join=True)
    import paper_2311_17410_b200 as gf

    g, src, dst, ts = _single_process(directed)
    parts = [np.load(tmp_path / f"rank{r}.npz") for r in range(2)]
    roots, rts = _roots(src, dst, ts)
    dev = torch.device("cuda:0")
    for pol in POLICIES:
        want = gf.sample_khop_device(g, torch.from_numpy(roots).to(dev), torch.from_numpy(rts).to(dev), [6, 4],
                                     _policy(pol), seed=9)
        for h, lay in enumerate(want.layers):
            for nm in ("neighbors", "edge_ids", "timestamps"):
                got = np.concatenate([p[f"{pol}_{h}_{nm}"] for p in parts])
                np.testing.assert_array_equal(got, getattr(lay, nm).cpu().numpy(), err_msg=f"{pol} hop{h} {nm}")


def _feature_batches(seed, n_ids, dim):
    rng = np.random.default_rng(seed)
    rows = rng.random((n_ids, dim), dtype=np.float32)
    # power-law-ish key batches with repeats and unknown ids (>= n_ids)
    batches = [np.minimum(rng.zipf(1.3, 3_000) - 1, n_ids + 50).astype(np.int64) for _ in range(6)]
    return rows, batches


def _sharded_worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2311_17410_b200 as gf
        from paper_2311_17410_b200.distributed import ShardedFeatureTable, fetch_features_sharded

        dev = torch.device("cuda:0")
        torch.cuda.set_device(dev)
        n_ids, dim = 5_000, 186
        rows, batches = _feature_batches(rank, n_ids, dim)
        rows_all, _ = _feature_batches(0, n_ids, dim)  # the shared table contents (rank-0 seed)
        ids = np.arange(n_ids, dtype=np.int64)
        mine = ids[ShardedFeatureTable.owns(ids, world, rank)]
        tab = gf.EdgeFeatureTable(dim, device=dev)
        tab.append(mine, rows_all[mine])
        sharded = ShardedFeatureTable(tab)
        cache = gf.VectorCache("lru", 400, dim, 0.2, device=dev)
        res = {}
        for b, keys in enumerate(batches):
            vals, hit, nm, adm = fetch_features_sharded(cache, sharded, torch.from_numpy(keys).to(dev))
            res[f"v{b}"] = vals.cpu().numpy()
            res[f"h{b}"] = hit.cpu().numpy()
            res[f"c{b}"] = np.array([nm, adm])
        res["keys"] = cache.keys
        res["scores"] = cache.scores
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
    finally:
        dist.destroy_process_group()


def test_sharded_feature_fetch_two_ranks_equal_local_table(tmp_path):
    """Replicated mode, features sharded by id % world: each rank's fetch block (cache probe, owner
    fetch of the misses over the all-to-all, insert) equals the fused local block over the whole
    table -- rows, hit masks, miss / admitted counts and the final cache state."""
    mp.spawn(_sharded_worker, args=(2, _port(), str(tmp_path)), nprocs=2, join=True)
    import paper_2311_17410_b200 as gf

    dev = torch.device("cuda:0")
    n_ids, dim = 5_000, 186
    rows_all, _ = _feature_batches(0, n_ids, dim)
    for rank in range(2):
        _, batches = _feature_batches(rank, n_ids, dim)
        got = np.load(tmp_path / f"rank{rank}.npz")
        tab = gf.EdgeFeatureTable(dim, device=dev)
        tab.append(np.arange(n_ids), rows_all)
        cache = gf.VectorCache("lru", 400, dim, 0.2, device=dev)
        for b, keys in enumerate(batches):
            vals, hit, nm, adm = gf.fetch_features(cache, tab, torch.from_numpy(keys).to(dev))
            np.testing.assert_array_equal(got[f"v{b}"], vals.cpu().numpy(), err_msg=f"rank {rank} batch {b} rows")
            np.testing.assert_array_equal(got[f"h{b}"], hit.cpu().numpy())
            assert list(got[f"c{b}"]) == [nm, adm]
        np.testing.assert_array_equal(got["keys"], cache.keys)
        np.testing.assert_array_equal(got["scores"], cache.scores)
