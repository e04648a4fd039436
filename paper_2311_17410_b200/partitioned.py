"""Partitioned multi-GPU mode (MAG config): the graph is edge-cut hash partitioned.

Rank r owns the nodes v with v % P == r (partition.py:38-39) and stores each
owned node's whole list (cluster.py:126-140): a directed edge lives with
the owner of its source, an undirected edge additionally as (dst, src) with
the owner of its destination, under one global edge id (cluster.py:178-201).

Ingest: every rank holds a contiguous shard of the new batch (rank order);
global ids are the batch base plus the shard offset; entries are bucketed by
owner and exchanged with one all-to-all, then appended on the owner in
stream order (received chunks are concatenated in source-rank order, so the
per-node append order equals the unpartitioned store's).

Sampling, per hop (cluster.py:242-292): queries are bucketed by the owner of
their source and exchanged (node, t_end, query key); the owner runs the
device sampler with the given keys; counts and sampled (nbr, eid, ts, child
key) go back with a second all-to-all and are merged into the original
query order.  Because the sampler's randomness is keyed by the query key,
not by where the query runs, the result equals a single-GPU sample of the
unpartitioned graph bit for bit (tests/test_partitioned*.py), the property
the reference checks for its cluster (tests/test_cluster.py:62-84).

Data movement around the all-to-alls runs on the GPU (exchange.py -> gf_part.cu): owner
bucketing is a stable counting sort, the answers are merged into request order by one CSR-merge
kernel and feature rows by a row scatter.  The host sees only the per-owner counts the
all-to-all needs for its split sizes (one small copy per exchange, not one per source rank).

Transports: ``DistTransport`` (torch.distributed all_to_all_single: NCCL over
NVLink between GPUs, gloo on CPU) and ``ThreadTransport`` (P ranks as
threads of one process on one GPU, the counterpart of the reference's
in-process LocalTransport, cluster.py:143-157).
"""

from __future__ import annotations

import threading

import numpy as np

from . import exchange as X
from .sampling import LayeredSample, SampleLayer, SamplingPolicy, hop_seed


class DistTransport:
    """all_to_all over the default torch.distributed process group."""

    def __init__(self):
        import torch.distributed as dist

        self.dist = dist
        self.P = dist.get_world_size()
        self.rank = dist.get_rank()
        # gloo's all_to_all runs on host tensors (CPU tests, several ranks sharing one GPU)
        self.host = dist.get_backend() != "nccl"

    def exchange(self, chunks):
        """chunks[d]: int64 tensor [k, n_d] for rank d -> list of tensors received from each rank."""
        import torch

        if self.host and chunks and chunks[0].is_cuda:
            dev0 = chunks[0].device
            return [c.to(dev0) for c in self.exchange([c.cpu() for c in chunks])]
        k = chunks[0].shape[0]
        dev = chunks[0].device
        send_n = torch.tensor([c.shape[1] for c in chunks], dtype=torch.int64, device=dev)
        recv_n = torch.empty_like(send_n)
        self.dist.all_to_all_single(recv_n, send_n)
        rn = recv_n.tolist()
        send = torch.cat([c.t().contiguous() for c in chunks]) if chunks else torch.empty((0, k), dtype=torch.int64)
        recv = torch.empty((sum(rn), k), dtype=torch.int64, device=dev)
        self.dist.all_to_all_single(recv, send, [int(x) for x in rn], [int(c.shape[1]) for c in chunks])
        out, pos = [], 0
        for n in rn:
            out.append(recv[pos:pos + n].t().contiguous())
            pos += n
        return out

    def allgather_int(self, x: int) -> list[int]:
        import torch

        t = torch.tensor([x], dtype=torch.int64)
        if self.dist.get_backend() == "nccl":
            t = t.cuda()
        parts = [torch.zeros_like(t) for _ in range(self.P)]
        self.dist.all_gather(parts, t)
        return [int(p.item()) for p in parts]


class ThreadTransport:
    """P ranks as threads of one process (single-GPU simulation of the partitioned mode)."""

    class _Shared:
        def __init__(self, P):
            self.P = P
            self.table = [None] * P
            self.barrier = threading.Barrier(P)

    def __init__(self, shared: "_Shared", rank: int):
        self.shared, self.P, self.rank = shared, shared.P, rank

    @classmethod
    def group(cls, P: int):
        sh = cls._Shared(P)
        return [cls(sh, r) for r in range(P)]

    def exchange(self, chunks):
        sh = self.shared
        sh.table[self.rank] = chunks
        sh.barrier.wait()
        out = [sh.table[s][self.rank] for s in range(self.P)]
        sh.barrier.wait()
        return out

    def allgather_int(self, x: int) -> list[int]:
        sh = self.shared
        sh.table[self.rank] = x
        sh.barrier.wait()
        out = list(sh.table)
        sh.barrier.wait()
        return out


def _exchange_rows(transport, chunks):
    """Exchange float32 [n_d, dim] row blocks (viewed as int32 columns for the int64 exchange)."""
    import torch

    dim = chunks[0].shape[1] if chunks else 0
    as_int = [torch.cat([c.contiguous().view(torch.int32).to(torch.int64).t(),
                         torch.zeros((0, c.shape[0]), dtype=torch.int64, device=c.device)]) for c in chunks]
    got = transport.exchange(as_int)
    return [g.t().to(torch.int32).contiguous().view(torch.float32).reshape(-1, dim) for g in got]


class PartitionedFeatures:
    """Feature rows sharded by owner = id % P (cluster.py:296-325), fetched over the transport.

    ``table`` is this rank's local feature table (NodeFeatureTable /
    EdgeFeatureTable on the GPU) holding the rows of the ids it owns.
    """

    def __init__(self, transport, table, dim: int):
        self.t, self.table, self.dim = transport, table, dim
        self.P, self.rank = transport.P, transport.rank

    def get(self, ids):
        """(rows, found) for arbitrary ids, in order; one id/rows all-to-all round trip."""
        import torch

        dev = ids.device
        n = int(ids.numel())
        perm, ids_sorted, counts = X.bucket_by_owner(ids, self.P)
        chunks, pos = [], 0
        for c in counts:
            chunks.append(ids_sorted[pos:pos + c].reshape(1, -1))
            pos += c
        asked = self.t.exchange(chunks)
        sizes = [int(q.shape[1]) for q in asked]
        qall = torch.cat([q.reshape(-1) for q in asked]) if asked else torch.zeros(0, dtype=torch.int64, device=dev)
        if qall.numel():
            rows, found = self.table.get(qall)  # one lookup for every requester
        else:
            rows = torch.zeros((0, self.dim), dtype=torch.float32, device=dev)
            found = torch.zeros(0, dtype=torch.bool, device=dev)
        rows, found = rows.to(torch.float32), found.to(torch.int64)
        replies_rows, replies_found, pos = [], [], 0
        for c in sizes:
            replies_rows.append(rows[pos:pos + c])
            replies_found.append(found[pos:pos + c].reshape(1, -1))
            pos += c
        rows_back = torch.cat(_exchange_rows(self.t, replies_rows)) if n else torch.zeros((0, self.dim), device=dev)
        found_back = torch.cat([f.reshape(-1) for f in self.t.exchange(replies_found)])
        out = X.scatter_rows(rows_back, perm, n) if n else torch.zeros((0, self.dim), dtype=torch.float32, device=dev)
        found = torch.zeros(n, dtype=torch.bool, device=dev)
        found[perm] = found_back.bool()
        return out, found


def fetch_features_partitioned(cache, features: PartitionedFeatures, keys):
    """The harness fetch block (harness.py:438-446) with peer-owned rows:
    cache.fetch -> owner fetch of the distinct misses -> cache.insert_batch(found).

    Like the local block (features.fetch_features / gf_fetch_features) it returns COMPLETE rows:
    cached rows for hits, the owners' rows for misses (zeros for ids no owner holds)."""
    import torch

    k = keys.to(device=cache.device, dtype=torch.int64).contiguous()
    values, hit, miss = cache.fetch_device(k)
    admitted = 0
    if miss.numel():
        rows, found = features.get(miss)
        # every missed occurrence takes its distinct key's row (miss keys are unique)
        order = torch.argsort(miss)
        occ = (~hit).nonzero().reshape(-1)
        pos = order[torch.searchsorted(miss[order], k[occ])]
        values[occ] = rows[pos]
        if bool(found.any()):
            admitted = cache.insert_batch(miss[found].contiguous(), rows[found].contiguous())
    return values, hit, int(miss.numel()), admitted


class GpuEngine:
    """This rank's partition on its GPU (libgfb200)."""

    def __init__(self, tau: int = 48, sizing=None, device=None):
        from .storage import DynamicGraph

        # a partition stores directed per-endpoint entries (cluster.py:131-140)
        self.graph = DynamicGraph(directed=True, tau=tau, sizing=sizing, device=device)
        self.device = self.graph.device

    def add(self, src, dst, ts, eids) -> int:
        """Append owner entries with their global ids; returns the number rejected as out of order."""
        return self.graph.add_edges_arrays(src, dst, ts, eids)[1]

    def delete_node(self, v: int) -> bool:
        return self.graph.delete_node(v)

    def sample(self, src, tend, keys, fanout, policy: SamplingPolicy, seed):
        from .sampling import _layer_device

        offs, nbr, eid, ts, okeys = _layer_device(self.graph, src, None, tend, fanout, policy, seed, keys=keys,
                                                  want_keys=True)
        return offs, nbr, eid, ts, okeys


class PartitionedGraph:
    def __init__(self, transport, engine, directed: bool = False):
        self.t = transport
        self.e = engine
        self.P, self.rank = transport.P, transport.rank
        self.directed = directed
        self.next_edge_id = 0
        # cluster.py:88,97-98: a failed worker answers requests with ErrorMsg(1, "worker failed")
        self.failed = False
        self._next_request_id = 0

    @property
    def device(self):
        return self.e.device

    # -- ingest -------------------------------------------------------------------
    def add_edges(self, src, dst, ts):
        """Append this rank's shard of a global batch; returns the shard's global edge ids."""
        import torch

        dev = self.device
        src = torch.as_tensor(src, dtype=torch.int64, device=dev)
        dst = torch.as_tensor(dst, dtype=torch.int64, device=dev)
        ts = torch.as_tensor(ts, dtype=torch.int64, device=dev)
        sizes = self.t.allgather_int(int(src.numel()))
        base = self.next_edge_id + sum(sizes[: self.rank])
        ids = base + torch.arange(src.numel(), dtype=torch.int64, device=dev)
        self.next_edge_id += sum(sizes)
        # entries in stream order: edge j -> (src, dst) [, (dst, src)]
        if self.directed:
            es, ed, et, ei = src, dst, ts, ids
        else:
            es = torch.stack([src, dst], 1).reshape(-1)
            ed = torch.stack([dst, src], 1).reshape(-1)
            et = torch.stack([ts, ts], 1).reshape(-1)
            ei = torch.stack([ids, ids], 1).reshape(-1)
        perm, es_s, owner_counts = self._bucket(es)
        ent = torch.stack([es_s, ed[perm], et[perm], ei[perm]])
        chunks, pos = [], 0
        for c in owner_counts:
            chunks.append(ent[:, pos:pos + c])
            pos += c
        got = torch.cat(self.t.exchange(chunks), dim=1)  # source-rank order = stream order
        rejected = 0
        if got.shape[1]:
            rejected = int(self.e.add(got[0].contiguous(), got[1].contiguous(), got[2].contiguous(),
                                      got[3].contiguous()))
        # cluster.py:199-200 asserts a time-sorted stream; a rejection at one owner would leave the
        # partitions disagreeing about an edge, so every rank learns of it and fails loudly
        if any(self.t.allgather_int(rejected)):
            raise ValueError("partitioned ingestion requires a time-sorted stream (an owner rejected an edge)")
        return ids

    def delete_node(self, v: int) -> bool:
        # node validity is checked at the sampling owner for sources and neighbours: every partition
        return bool(self.e.delete_node(v))

    # -- sampling -------------------------------------------------------------------
    # owner bucketing and the request-order merge run on the GPU (gf_part.cu)
    def _bucket(self, keys):
        return X.bucket_by_owner(keys, self.P)

    def _merge(self, perm, cnt_sorted, arrays):
        return X.csr_merge(perm, cnt_sorted, arrays)

    @staticmethod
    def _raise_failed(rid0, sent, cnt_recv):
        """RemoteRequestError for the first owner whose count chunk does not match the request
        (cluster.py:264-265): the request to owner d carries id rid0 + d."""
        for d, (ns, c) in enumerate(zip(sent, cnt_recv)):
            if int(c.shape[-1]) != int(ns):
                from .cluster import RemoteRequestError

                raise RemoteRequestError(rid0 + d, "worker failed")

    def sample_layer(self, src, tend, keys, fanout: int, policy: SamplingPolicy, seed_h: int):
        import torch

        dev = self.device
        n = int(src.numel())
        perm, src_s, owner_counts = self._bucket(src)
        qs = torch.stack([src_s, tend[perm], keys[perm]])  # keys: uint64 bit patterns in int64
        chunks, pos = [], 0
        for c in owner_counts:
            chunks.append(qs[:, pos:pos + c])
            pos += c
        # one request id per (hop, owner), as the reference's origin numbers its requests
        # (cluster.py:251-252); every rank numbers them the same way
        rid0 = self._next_request_id
        self._next_request_id += self.P
        recv = self.t.exchange(chunks)
        q = torch.cat(recv, dim=1)
        per_src = [int(c.shape[1]) for c in recv]
        if self.failed:
            # cluster.py:97-98: a failed owner serves nothing.  It still takes part in both answer
            # exchanges (the collectives stay matched on every rank) and signals the failure through
            # the split sizes the all-to-all already moves to the host: a count chunk one longer than
            # the origin's request.  Every origin therefore sees it, fails over the same hop and raises
            # -- fail-stop, instead of the ranks that sent no request to it hanging in the next hop.
            back_counts = [torch.full((1, nq + 1), -1, dtype=torch.int64, device=dev) for nq in per_src]
            back_edges = [torch.zeros((4, 0), dtype=torch.int64, device=dev) for _ in per_src]
            cnt_recv = self.t.exchange(back_counts)
            self.t.exchange(back_edges)
            self._raise_failed(rid0, owner_counts, cnt_recv)
        if q.shape[1]:
            offs, nbr, eid, ts, okeys = self.e.sample(q[0].contiguous(), q[1].contiguous(), q[2].contiguous(), fanout,
                                                      policy, seed_h)
            counts = offs[1:] - offs[:-1]
        else:
            counts = torch.zeros(0, dtype=torch.int64, device=dev)
            nbr = eid = ts = okeys = torch.zeros(0, dtype=torch.int64, device=dev)
            offs = torch.zeros(1, dtype=torch.int64, device=dev)
        # answers back to each origin: per query counts, then the flat edges (the owner's offsets at
        # the source-rank boundaries: one small host copy)
        bounds = [0]
        for nq in per_src:
            bounds.append(bounds[-1] + nq)
        eb = offs[torch.tensor(bounds, device=offs.device)].tolist()
        edges = torch.stack([nbr, eid, ts, okeys])
        back_counts = [counts[bounds[i]:bounds[i + 1]].reshape(1, -1) for i in range(len(per_src))]
        back_edges = [edges[:, eb[i]:eb[i + 1]] for i in range(len(per_src))]
        cnt_recv = self.t.exchange(back_counts)
        edge_recv = self.t.exchange(back_edges)
        self._raise_failed(rid0, owner_counts, cnt_recv)
        # merge into the original query order (send order -> request order, one kernel)
        cnt_sorted = torch.cat([c.reshape(-1) for c in cnt_recv])
        edges_sorted = torch.cat(edge_recv, dim=1)
        offsets, out, _ = self._merge(perm, cnt_sorted, [edges_sorted[0], edges_sorted[1], edges_sorted[2],
                                                         edges_sorted[3]])
        return SampleLayer(src, tend, offsets, out[0], out[1], out[2]), out[3]

    def sample_khop(self, roots, ts, fanouts, policy: SamplingPolicy, seed: int = 0, root_key_base: int = 0):
        """This rank's roots; keys root_key_base + i (cf. sampling.sample_khop)."""
        import torch

        dev = self.device
        src = torch.as_tensor(roots, dtype=torch.int64, device=dev)
        tend = torch.as_tensor(ts, dtype=torch.int64, device=dev)
        keys = (torch.arange(src.numel(), dtype=torch.int64, device=dev) + int(root_key_base))
        layers = []
        for hop, f in enumerate(fanouts):
            lay, keys = self.sample_layer(src, tend, keys, int(f), policy, hop_seed(seed, hop))
            layers.append(lay)
            src, tend = lay.neighbors, lay.timestamps
        return LayeredSample(layers)
