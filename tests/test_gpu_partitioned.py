"""Partitioned mode on the GPU: P partitions (threads, one GPU) equal the unpartitioned graph bitwise."""

from __future__ import annotations

import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("P,directed", [(2, True), (3, False), (4, True)])
def test_partitioned_threads_equal_single_gpu(cuda_device, P, directed):
    import torch

    import paper_2311_17410_b200 as gf
    from paper_2311_17410_b200.distributed import shard_range
    from paper_2311_17410_b200.partitioned import GpuEngine, PartitionedGraph, ThreadTransport

    src, dst, ts = gf.generate_synthetic_arrays(3000, 300_000, 2.2, 175_200, seed=4, src_skew=2.2)
    roots = np.concatenate([src[-3000:], dst[-3000:]])
    rts = np.concatenate([ts[-3000:], ts[-3000:]])
    transports = ThreadTransport.group(P)
    results = [None] * P
    errors = []

    def rank_main(r):
        try:
            pg = PartitionedGraph(transports[r], GpuEngine(tau=64), directed=directed)
            for lo in range(0, len(src), 50_000):
                hi = min(len(src), lo + 50_000)
                a, b = shard_range(hi - lo, P, r)
                pg.add_edges(src[lo + a:lo + b], dst[lo + a:lo + b], ts[lo + a:lo + b])
            a, b = shard_range(len(roots), P, r)
            out = {}
            for pol in ("recent", "uniform"):
                s = pg.sample_khop(roots[a:b], rts[a:b], [10, 10], gf.SamplingPolicy(pol), seed=8, root_key_base=a)
                out[pol] = [(lay.neighbors.cpu().numpy(), lay.edge_ids.cpu().numpy(), lay.timestamps.cpu().numpy())
                            for lay in s.layers]
            torch.cuda.synchronize()
            results[r] = out
        except Exception as e:  # surface thread failures
            errors.append(e)
            transports[r].shared.barrier.abort()

    threads = [threading.Thread(target=rank_main, args=(r,)) for r in range(P)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    g = gf.DynamicGraph(directed=directed, tau=64)
    for lo in range(0, len(src), 50_000):
        g.add_edges_arrays(src[lo:lo + 50_000], dst[lo:lo + 50_000], ts[lo:lo + 50_000])
    dev = torch.device("cuda:0")
    for pol in ("recent", "uniform"):
        want = gf.TemporalSampler(g, [10, 10], pol, seed=8).sample(torch.from_numpy(roots).to(dev),
                                                                   torch.from_numpy(rts).to(dev))
        for h, lay in enumerate(want.layers):
            for i, nm in enumerate(("neighbors", "edge_ids", "timestamps")):
                got = np.concatenate([results[r][pol][h][i] for r in range(P)])
                np.testing.assert_array_equal(got, getattr(lay, nm).cpu().numpy(), err_msg=f"{pol} hop{h} {nm}")


def test_peer_feature_fetch_threads(cuda_device):
    """Rows owned by other partitions come back through the transport, bit-exact; cache state
    equals a single-table fetch block (harness.py:438-446)."""
    import torch

    import paper_2311_17410_b200 as gf
    from paper_2311_17410_b200.partitioned import PartitionedFeatures, ThreadTransport, fetch_features_partitioned

    P, dim = 3, 19
    rng = np.random.default_rng(3)
    n_nodes = 5000
    rows = rng.random((n_nodes, dim), dtype=np.float32)
    keys_all = [rng.integers(-5, n_nodes + 50, 4000) for _ in range(6)]
    transports = ThreadTransport.group(P)
    out = [None] * P
    errors = []

    def rank_main(r):
        try:
            table = gf.NodeFeatureTable(dim)
            mine = np.arange(r, n_nodes, P)
            table.set_many(mine, rows[mine])
            feats = PartitionedFeatures(transports[r], table, dim)
            cache = gf.VectorCache("lru", 300, dim, 0.3)
            res = []
            for keys in keys_all:
                k = torch.from_numpy(keys).cuda()
                got, found = feats.get(k)
                res.append((got.cpu().numpy(), found.cpu().numpy()))
                fetch_features_partitioned(cache, feats, k)
            res.append((cache.keys, cache.scores))
            out[r] = res
        except Exception as e:
            errors.append(e)
            transports[r].shared.barrier.abort()

    threads = [threading.Thread(target=rank_main, args=(r,)) for r in range(P)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    single = gf.NodeFeatureTable(dim)
    single.set_many(np.arange(n_nodes), rows)
    ref_cache = gf.VectorCache("lru", 300, dim, 0.3)
    for i, keys in enumerate(keys_all):
        want_rows, want_found = single.get(keys)
        for r in range(P):
            np.testing.assert_array_equal(out[r][i][0], want_rows)
            np.testing.assert_array_equal(out[r][i][1], want_found)
        gf.fetch_features(ref_cache, single, keys)
    for r in range(P):
        np.testing.assert_array_equal(out[r][-1][0], ref_cache.keys)
        np.testing.assert_array_equal(out[r][-1][1], ref_cache.scores)


def test_partitioned_failed_owner_raises_on_every_rank(cuda_device):
    """cluster.py:97-98,264-265 on libgfb200 (3 thread ranks, one GPU): a failed owner makes every
    rank raise RemoteRequestError with the same request id in the same hop; the group recovers."""
    import paper_2311_17410_b200 as gf
    from paper_2311_17410_b200.distributed import shard_range
    from paper_2311_17410_b200.partitioned import GpuEngine, PartitionedGraph, ThreadTransport

    P = 3
    src, dst, ts = gf.generate_synthetic_arrays(500, 40_000, 2.2, 20_000, seed=2, src_skew=2.2)
    transports = ThreadTransport.group(P)
    got = [None] * P
    errors = []

    def rank_main(r):
        try:
            pg = PartitionedGraph(transports[r], GpuEngine(tau=32), directed=False)
            a, b = shard_range(len(src), P, r)
            pg.add_edges(src[a:b], dst[a:b], ts[a:b])
            roots, rts = src[-30:][r::P], ts[-30:][r::P]
            pg.failed = r == 2
            rid = None
            try:
                pg.sample_khop(roots, rts, [5, 5], gf.SamplingPolicy("uniform"), seed=1)
            except gf.RemoteRequestError as e:
                rid = e.request_id
            pg.failed = False
            s = pg.sample_khop(roots, rts, [5], gf.SamplingPolicy("recent"), seed=1)
            got[r] = (rid, int(s.layers[0].offsets[-1]))
        except Exception as e:  # surface thread failures
            errors.append(e)
            transports[r].shared.barrier.abort()

    threads = [threading.Thread(target=rank_main, args=(r,)) for r in range(P)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    assert [g[0] for g in got] == [2] * P  # hop 0, owner 2
    assert all(g[1] > 0 for g in got)
