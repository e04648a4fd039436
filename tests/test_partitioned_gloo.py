"""Partitioned mode host logic, world_size 2 over gloo (CPU), with the oracle as each rank's engine.

Every rank ingests its shard of every batch (all-to-all dispatch by owner) and
samples its own roots through per-hop all-to-all exchanges; the union must
equal single-process sampling of the unpartitioned graph, bitwise.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class OracleEngine:
    def __init__(self, tau):
        from oracle import OracleGraph

        self.g = OracleGraph(True, tau)
        self.device = torch.device("cpu")

    def add(self, src, dst, ts, eids):
        out = self.g.add_edges(src.numpy(), dst.numpy(), ts.numpy(), eids.numpy())
        return int((out < 0).sum())

    def delete_node(self, v):
        return self.g.delete_node(v)

    def sample(self, src, tend, keys, fanout, policy, seed):
        from oracle.oracle import _child_keys_vec

        k = keys.numpy().view(np.uint64)
        offs, nb, eid, ts = self.g.sample_layer(src.numpy(), np.full(len(src), -2**63, np.int64), tend.numpy(), fanout,
                                                policy.kind, policy.delta, seed, keys=k)
        cnt = np.diff(offs)
        ok = _child_keys_vec(np.repeat(k, cnt), np.arange(len(nb)) - np.repeat(offs[:-1], cnt)).view(np.int64)
        return tuple(torch.from_numpy(np.ascontiguousarray(a)) for a in (offs, nb, eid, ts, ok))


def _host_partitioned_graph():
    """PartitionedGraph whose bucketing / merge run on host tensors: the CPU engine here is the
    oracle, so the device kernels (gf_part.cu) are replaced by their numpy statement; the GPU
    tests (tests/test_gpu_multiproc.py) cover the kernels themselves."""
    from paper_2311_17410_b200.partitioned import PartitionedGraph

    class HostPartitionedGraph(PartitionedGraph):
        def _bucket(self, keys):
            k = keys.numpy()
            owner = np.mod(k, self.P)
            perm = np.argsort(owner, kind="stable")
            counts = np.bincount(owner, minlength=self.P).tolist()
            return torch.from_numpy(perm), torch.from_numpy(k[perm]), counts

        def _merge(self, perm, cnt_sorted, arrays):
            perm_np, cnt = perm.numpy(), cnt_sorted.numpy()
            n = len(perm_np)
            cnt_orig = np.zeros(n, np.int64)
            cnt_orig[perm_np] = cnt
            offsets = np.concatenate([[0], np.cumsum(cnt_orig)]).astype(np.int64)
            start = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
            outs = []
            for a in arrays:
                a = a.numpy()
                o = np.empty_like(a)
                for i in range(n):
                    d = offsets[perm_np[i]]
                    o[d:d + cnt[i]] = a[start[i]:start[i] + cnt[i]]
                outs.append(torch.from_numpy(o))
            return torch.from_numpy(offsets), outs, int(offsets[-1])

    return HostPartitionedGraph


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _stream():
    from paper_2311_17410_b200.synth import generate_synthetic_arrays

    return generate_synthetic_arrays(400, 20_000, 2.2, 40_000, seed=11, src_skew=2.2)


def _worker(rank, world, port, out_dir, directed):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2311_17410_b200 import SamplingPolicy
        from paper_2311_17410_b200.distributed import shard_range
        from paper_2311_17410_b200.partitioned import DistTransport, PartitionedGraph

        pg = _host_partitioned_graph()(DistTransport(), OracleEngine(32), directed=directed)
        src, dst, ts = _stream()
        for lo in range(0, len(src), 5_000):
            hi = min(len(src), lo + 5_000)
            a, b = shard_range(hi - lo, world, rank)
            pg.add_edges(torch.from_numpy(src[lo + a:lo + b]), torch.from_numpy(dst[lo + a:lo + b]),
                         torch.from_numpy(ts[lo + a:lo + b]))
        roots = np.concatenate([src[-200:], dst[-200:]])
        rts = np.concatenate([ts[-200:], ts[-200:]])
        lo, hi = shard_range(len(roots), world, rank)
        res = {}
        for pol in ("recent", "uniform"):
            s = pg.sample_khop(torch.from_numpy(roots[lo:hi]), torch.from_numpy(rts[lo:hi]), [4, 3],
                               SamplingPolicy(pol), seed=2, root_key_base=lo)
            for h, lay in enumerate(s.layers):
                for nm in ("offsets", "neighbors", "edge_ids", "timestamps"):
                    res[f"{pol}_{h}_{nm}"] = getattr(lay, nm).numpy()
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
    finally:
        dist.destroy_process_group()


def _check(tmp_path, directed):
    from oracle import OracleGraph

    src, dst, ts = _stream()
    g = OracleGraph(directed, 32)
    for lo in range(0, len(src), 5_000):
        g.add_edges(src[lo:lo + 5_000], dst[lo:lo + 5_000], ts[lo:lo + 5_000])
    roots = np.concatenate([src[-200:], dst[-200:]])
    rts = np.concatenate([ts[-200:], ts[-200:]])
    parts = [np.load(tmp_path / f"rank{r}.npz") for r in range(2)]
    for pol in ("recent", "uniform"):
        want = g.sample_khop(roots, rts, [4, 3], pol, seed=2)
        # per-rank layer h covers the rank's share of layer h's queries, in order
        for h, lay in enumerate(want):
            nb = np.concatenate([p[f"{pol}_{h}_neighbors"] for p in parts])
            eid = np.concatenate([p[f"{pol}_{h}_edge_ids"] for p in parts])
            tts = np.concatenate([p[f"{pol}_{h}_timestamps"] for p in parts])
            np.testing.assert_array_equal(nb, lay[3], err_msg=f"{pol} hop{h}")
            np.testing.assert_array_equal(eid, lay[4])
            np.testing.assert_array_equal(tts, lay[5])


def test_partitioned_two_ranks_equal_unpartitioned_directed(tmp_path):
    mp.spawn(_worker, args=(2, _port(), str(tmp_path), True), nprocs=2, join=True)
    _check(tmp_path, True)


def test_partitioned_two_ranks_equal_unpartitioned_undirected(tmp_path):
    mp.spawn(_worker, args=(2, _port(), str(tmp_path), False), nprocs=2, join=True)
    _check(tmp_path, False)


def _failed_worker(rank, world, port, out_dir):
    """cluster.py:97-98,264-265 (tests/test_cluster.py:101-108): a failed owner surfaces as a
    RemoteRequestError carrying the request id -- here on every rank of the SPMD group, in the
    same hop, so no rank is left waiting in the next exchange."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2311_17410_b200 import RemoteRequestError, SamplingPolicy
        from paper_2311_17410_b200.distributed import shard_range
        from paper_2311_17410_b200.partitioned import DistTransport

        pg = _host_partitioned_graph()(DistTransport(), OracleEngine(32), directed=False)
        src, dst, ts = _stream()
        a, b = shard_range(len(src), world, rank)
        pg.add_edges(torch.from_numpy(src[a:b]), torch.from_numpy(dst[a:b]), torch.from_numpy(ts[a:b]))
        roots = torch.tensor([1, 2, 3], dtype=torch.int64)
        rts = torch.full((3,), int(ts[-1]), dtype=torch.int64)
        # healthy group first: the layer completes on both ranks
        pg.sample_khop(roots, rts, [4], SamplingPolicy("recent"), seed=0)
        pg.failed = rank == 1
        got = -1
        try:
            pg.sample_khop(roots, rts, [4, 3], SamplingPolicy("recent"), seed=0)
        except RemoteRequestError as err:
            got = err.request_id
        # the group is still usable afterwards: the exchanges stayed matched
        pg.failed = False
        ok = pg.sample_khop(roots, rts, [4], SamplingPolicy("recent"), seed=0)
        np.save(os.path.join(out_dir, f"fail{rank}.npy"),
                np.array([got, int(ok.layers[0].offsets[-1])], dtype=np.int64))
    finally:
        dist.destroy_process_group()


def test_partitioned_failed_owner_raises_request_id(tmp_path):
    mp.spawn(_failed_worker, args=(2, _port(), str(tmp_path)), nprocs=2, join=True)
    a, b = (np.load(tmp_path / f"fail{r}.npy") for r in range(2))
    # hop 0 of the second sample_khop call (ids 2P..3P-1 after the first call's one hop); owner 1
    assert a[0] == b[0] == 2 + 1
    assert a[1] > 0 and b[1] > 0
