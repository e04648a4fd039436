"""world_size-2 gloo tests (CPU) for the replicated multi-GPU host logic.

Each process holds a shard of every ingest batch and of the root set.  The
all-gather ingest and the per-rank key bases are exercised with the CPU
oracle as the per-rank engine (the CUDA kernels need a GPU; their shard
invariance is covered by tests/test_gpu_sampling.py).  The union of the two
ranks' samples must equal a single-process sample of all roots, bitwise.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import OracleGraph
        from paper_2311_17410_b200.distributed import exclusive_prefix, gather_edge_batch, shard_range
        from paper_2311_17410_b200.synth import generate_synthetic_arrays

        src, dst, ts = generate_synthetic_arrays(500, 30_000, 2.2, 50_000, seed=7, src_skew=2.2)
        g = OracleGraph(directed=True, tau=64)
        for lo in range(0, len(src), 7_000):
            hi = min(len(src), lo + 7_000)
            a, b = shard_range(hi - lo, world, rank)
            # uneven shards on purpose: rank 1 also gets nothing for the last batch piece
            s, d, t = gather_edge_batch(torch.from_numpy(src[lo + a:lo + b]), torch.from_numpy(dst[lo + a:lo + b]),
                                        torch.from_numpy(ts[lo + a:lo + b]))
            g.add_edges(s.numpy(), d.numpy(), t.numpy())
        roots = np.concatenate([src[-300:], dst[-300:]])
        rts = np.concatenate([ts[-300:], ts[-300:]])
        # unequal root shards: rank 0 takes 250, rank 1 the rest
        lo, hi = (0, 250) if rank == 0 else (250, len(roots))
        base, total = exclusive_prefix(hi - lo)
        assert base == lo and total == len(roots)
        res = {}
        for pol in ("recent", "uniform"):
            lays = g.sample_khop(roots[lo:hi], rts[lo:hi], [5, 4], pol, seed=3, root_key_base=base)
            res[pol] = [lay[3] for lay in lays]  # neighbours per hop
        exp = g.export_nodes()
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"),
                 **{f"{p}_{h}": v for p, hops in res.items() for h, v in enumerate(hops)},
                 degree=exp["degree"], num_blocks=exp["num_blocks"])
    finally:
        dist.destroy_process_group()


def test_two_rank_ingest_and_sharded_sampling_equal_single_process(tmp_path):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    from oracle import OracleGraph
    from paper_2311_17410_b200.synth import generate_synthetic_arrays

    src, dst, ts = generate_synthetic_arrays(500, 30_000, 2.2, 50_000, seed=7, src_skew=2.2)
    g = OracleGraph(directed=True, tau=64)
    for lo in range(0, len(src), 7_000):
        g.add_edges(src[lo:lo + 7_000], dst[lo:lo + 7_000], ts[lo:lo + 7_000])
    roots = np.concatenate([src[-300:], dst[-300:]])
    rts = np.concatenate([ts[-300:], ts[-300:]])
    r0, r1 = np.load(tmp_path / "rank0.npz"), np.load(tmp_path / "rank1.npz")
    exp = g.export_nodes()
    for r in (r0, r1):  # identical replicas
        np.testing.assert_array_equal(r["degree"], exp["degree"])
        np.testing.assert_array_equal(r["num_blocks"], exp["num_blocks"])
    for pol in ("recent", "uniform"):
        lays = g.sample_khop(roots, rts, [5, 4], pol, seed=3)
        for h, lay in enumerate(lays):
            np.testing.assert_array_equal(np.concatenate([r0[f"{pol}_{h}"], r1[f"{pol}_{h}"]]), lay[3])


def test_shard_range_covers_everything():
    from paper_2311_17410_b200.distributed import shard_range

    for total in (0, 1, 7, 100, 101):
        for n in (1, 2, 3, 8):
            seen = []
            for r in range(n):
                lo, hi = shard_range(total, n, r)
                seen.extend(range(lo, hi))
            assert seen == list(range(total))
