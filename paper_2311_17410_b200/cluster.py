"""``ClusterSim`` facade (reference cluster.py:33-345) over device partitions.

The reference simulates M machines x W worker ranks in one process: every
machine stores the whole block lists of the nodes it owns (``node % M``),
directed per-endpoint entries under global edge ids (cluster.py:126-140,
178-201); a k-hop request is split per hop by owner, served by the worker of
the same rank on every machine (static scheduling, cluster.py:72-75,91-97),
and merged back into query order (cluster.py:242-292).

Here each machine's store is a ``DynamicGraph`` in HBM (all machines share
one GPU; ``partitioned.PartitionedGraph`` is the one-rank-per-GPU form with
NCCL all-to-all).  Per hop the owner buckets, the per-machine
``gf_sample_layer`` calls and the merge all stay on the device.  Query keys
travel with the queries (hop 0: the root index; hop l+1: the child key of
the sampled edge), so a cluster sample equals ``sample_khop`` on one
unpartitioned graph bit for bit for every policy -- the property the
reference tests for its cluster (tests/test_cluster.py:62-84).

Not built: the TCP transport and servers (cluster.py:350-444) -- networking is
outside the hot path.  ``transport`` is the in-process
``LocalTransport``; the TGRP frames it would carry are in ``wire.py``.
"""

from __future__ import annotations

import threading
import time
from dataclasses import dataclass

import numpy as np

from .features import EdgeFeatureTable, NodeFeatureTable
from .metrics import coefficient_of_variation
from .partition import PartitionSpec, assign
from .sampling import LayeredSample, SampleLayer, SamplingPolicy, SampleRequest, _layer_device, hop_seed
from .storage import TS_MIN, BlockSizing, DynamicGraph, InsertionBatch


@dataclass(frozen=True)
class ClusterSpec:
    machines: int
    workers_per_machine: int

    def __post_init__(self):
        if self.machines < 1 or self.workers_per_machine < 1:
            raise ValueError("need at least one machine and one worker")

    @property
    def partition(self) -> PartitionSpec:
        return PartitionSpec(self.machines)


@dataclass(frozen=True)
class Origin:
    machine: int
    rank: int


@dataclass
class WorkerTelemetry:
    requests_served: int = 0
    targets_sampled: int = 0
    busy_time: float = 0.0


class RemoteRequestError(RuntimeError):
    def __init__(self, request_id: int, message: str):
        super().__init__(f"request {request_id}: {message}")
        self.request_id = request_id


def route(spec: ClusterSpec, origin: Origin, target: int) -> tuple[int, int]:
    """cluster.py:72-75: the owner machine, same worker rank as the origin."""
    return assign(spec.partition, target), origin.rank


def measure_cv(values) -> float:
    return coefficient_of_variation(values)


@dataclass
class LayerRequest:
    """One per-machine slice of a hop: device tensors plus the sampling parameters
    (the content of a TGRP sample request, wire.py, plus the query keys)."""
    targets: object
    t_starts: object
    timestamps: object
    keys: object
    fanout: int
    policy: SamplingPolicy
    seed: int


class Worker:
    """Serial server of one machine's partition for one rank (cluster.py:81-123)."""

    def __init__(self, machine: "Machine", rank: int):
        self.machine = machine
        self.rank = rank
        self.telemetry = WorkerTelemetry()
        self.failed = False
        self._lock = threading.Lock()

    def serve_sample(self, origin: Origin, req: LayerRequest):
        with self._lock:
            if origin.rank != self.rank:
                raise AssertionError(f"static scheduling violated: rank {self.rank} got a request from rank "
                                     f"{origin.rank}")
            if self.failed:
                return None
            t0 = time.perf_counter()
            out = _layer_device(self.machine.graph, req.targets, req.t_starts, req.timestamps, req.fanout, req.policy,
                                req.seed, keys=req.keys, want_keys=True)
            self.telemetry.requests_served += 1
            self.telemetry.targets_sampled += int(req.targets.numel())
            self.telemetry.busy_time += time.perf_counter() - t0
            return out

    def serve_features(self, kind: int, ids):
        with self._lock:
            table = self.machine.node_features if kind == 0 else self.machine.edge_features
            return table.get(ids)


class Machine:
    """cluster.py:126-140: one partition's store (directed per-endpoint entries) and feature shards."""

    def __init__(self, index: int, tau: int, sizing: BlockSizing | None, spec: ClusterSpec, node_dim: int = 0,
                 edge_dim: int = 0, device=None):
        self.index = index
        self.graph = DynamicGraph(directed=True, tau=tau, sizing=sizing, device=device)
        self.node_features = NodeFeatureTable(node_dim, device=self.graph.device)
        self.edge_features = EdgeFeatureTable(edge_dim, device=self.graph.device)
        self.workers = [Worker(self, r) for r in range(spec.workers_per_machine)]


class LocalTransport:
    """cluster.py:143-157: direct calls into the machines' workers."""

    def __init__(self, cluster: "ClusterSim"):
        self.cluster = cluster

    def sample(self, machine: int, rank: int, origin: Origin, request_id: int, req: LayerRequest):
        return self.cluster.machines[machine].workers[rank].serve_sample(origin, req)

    def features(self, machine: int, rank: int, kind: int, ids):
        return self.cluster.machines[machine].workers[rank].serve_features(kind, ids)

    def close(self) -> None:
        pass


class ClusterSim:
    def __init__(self, spec: ClusterSpec, directed: bool = False, tau: int = 48, sizing: BlockSizing | None = None,
                 node_dim: int = 0, edge_dim: int = 0, device=None):
        self.spec = spec
        self.directed = directed
        self.machines = [Machine(i, tau, sizing, spec, node_dim, edge_dim, device) for i in range(spec.machines)]
        self.device = self.machines[0].graph.device
        self.transport = LocalTransport(self)
        self._next_request_id = 0

    # -- ingest (cluster.py:178-224) ------------------------------------------------------------
    def add_edges(self, batch, *, first_edge_id: int | None = None) -> list[int]:
        """Route a time-sorted batch to the owners under shared global edge ids; an undirected
        edge becomes one directed entry per endpoint owner (both on one machine for a self loop)."""
        import torch

        edges = batch.edges if isinstance(batch, InsertionBatch) else batch
        arr = np.asarray(list(edges), dtype=np.int64).reshape(-1, 3)
        base = self._peek_edge_id() if first_edge_id is None else int(first_edge_id)
        ids = np.arange(base, base + len(arr), dtype=np.int64)
        if not len(arr):
            return []
        src, dst, ts = arr[:, 0], arr[:, 1], arr[:, 2]
        if self.directed:
            es, ed, et, ei = src, dst, ts, ids
        else:  # entry order per edge: (src, dst) then (dst, src), as an undirected graph appends
            es = np.stack([src, dst], 1).reshape(-1)
            ed = np.stack([dst, src], 1).reshape(-1)
            et = np.repeat(ts, 2)
            ei = np.repeat(ids, 2)
        owner = es % self.spec.machines
        for m, machine in enumerate(self.machines):
            sel = owner == m
            if sel.any():
                dev = machine.graph.device
                cols = [torch.from_numpy(np.ascontiguousarray(c[sel])).to(dev) for c in (es, ed, et, ei)]
                _, rejected = machine.graph.add_edges_arrays(*cols)
                if rejected:
                    raise AssertionError("cluster ingestion requires a time-sorted stream")
        return ids.tolist()

    def _peek_edge_id(self) -> int:
        return max((m.graph.next_edge_id for m in self.machines), default=0)

    def delete_edges(self, edge_ids) -> int:
        """cluster.py:206-213: an id counts once however many partitions held a copy."""
        wanted = {int(e) for e in edge_ids}
        deleted: set[int] = set()
        for m in self.machines:
            deleted |= m.graph.delete_edges_set(wanted)
        return len(deleted)

    def delete_nodes(self, nodes) -> int:
        """cluster.py:215-224: a node is invalidated on every machine (validity of neighbours
        is checked where they are sampled)."""
        count = 0
        for node in nodes:
            hit = False
            for m in self.machines:
                hit = m.graph.delete_node(int(node)) or hit
            count += int(hit)
        return count

    # -- sampling (cluster.py:226-292) -----------------------------------------------------------
    def sample_khop(self, request: SampleRequest, origin: Origin, root_key_base: int = 0) -> LayeredSample:
        import torch

        request.validate()
        dev = self.device
        on_dev = isinstance(request.targets, torch.Tensor) and request.targets.is_cuda
        src = torch.as_tensor(np.asarray(request.targets, dtype=np.int64) if not on_dev else request.targets,
                              dtype=torch.int64).to(dev)
        tend = torch.as_tensor(np.asarray(request.timestamps, dtype=np.int64) if not on_dev else request.timestamps,
                               dtype=torch.int64).to(dev)
        keys = torch.arange(src.numel(), dtype=torch.int64, device=dev) + int(root_key_base)
        out = LayeredSample()
        for hop, fanout in enumerate(request.fanouts):
            tstart = torch.full_like(src, TS_MIN)
            layer, keys = self._sample_layer_distributed(src, tstart, tend, keys, int(fanout), request.policy,
                                                         hop_seed(request.seed, hop), origin)
            out.layers.append(layer)
            src, tend = layer.neighbors, layer.timestamps
        return out if on_dev else out.to_host()

    def _sample_layer_distributed(self, src, tstart, tend, keys, fanout, policy, seed, origin):
        import torch

        dev = self.device
        n = int(src.numel())
        M = self.spec.machines
        owner = torch.remainder(src, M)
        order = torch.argsort(owner, stable=True)
        per_machine = torch.bincount(owner, minlength=M).tolist() if n else [0] * M
        counts_sorted, pieces, pos = [], [], 0
        for m in range(M):
            sel = order[pos:pos + per_machine[m]]
            pos += per_machine[m]
            if sel.numel() == 0:
                continue
            rid = self._next_request_id
            self._next_request_id += 1
            req = LayerRequest(src[sel], tstart[sel], tend[sel], keys[sel], fanout, policy, seed)
            resp = self.transport.sample(m, origin.rank, origin, rid, req)
            if resp is None:
                raise RemoteRequestError(rid, "worker failed")
            offs, nbr, eid, ts, okeys = resp
            counts_sorted.append(offs[1:] - offs[:-1])
            pieces.append(torch.stack([nbr, eid, ts, okeys]))
        cnt_sorted = torch.cat(counts_sorted) if counts_sorted else torch.zeros(0, dtype=torch.int64, device=dev)
        edges_sorted = torch.cat(pieces, 1) if pieces else torch.zeros((4, 0), dtype=torch.int64, device=dev)
        counts = torch.empty(n, dtype=torch.int64, device=dev)
        counts[order] = cnt_sorted
        offsets = torch.zeros(n + 1, dtype=torch.int64, device=dev)
        torch.cumsum(counts, 0, out=offsets[1:])
        total = int(edges_sorted.shape[1])
        # the i-th sorted query's edges land at offsets[order[i]] onwards
        qid = torch.repeat_interleave(torch.arange(n, device=dev), cnt_sorted)
        first = torch.cumsum(cnt_sorted, 0) - cnt_sorted
        dest = offsets[order[qid]] + torch.arange(total, device=dev) - first[qid]
        merged = torch.empty((4, total), dtype=torch.int64, device=dev)
        merged[:, dest] = edges_sorted
        return SampleLayer(src, tend, offsets, merged[0], merged[1], merged[2]), merged[3]

    # -- feature fetch (cluster.py:296-325) ------------------------------------------------------
    def _fetch(self, kind: int, ids, owners_of, origin: Origin):
        ids = np.asarray(ids, dtype=np.int64)
        owners = np.asarray(owners_of, dtype=np.int64) % self.spec.machines
        table0 = self.machines[0].node_features if kind == 0 else self.machines[0].edge_features
        rows = np.zeros((len(ids), table0.dim), dtype=np.float32)
        found = np.zeros(len(ids), dtype=bool)
        for m in range(self.spec.machines):
            idx = np.flatnonzero(owners == m)
            if len(idx):
                r, f = self.transport.features(m, origin.rank, kind, ids[idx])
                rows[idx] = r
                found[idx] = f
        return rows, found

    def fetch_node_features(self, ids, origin: Origin):
        return self._fetch(0, ids, ids, origin)

    def fetch_edge_features(self, edge_ids, src_nodes, origin: Origin):
        """Edge rows live with the owner of the edge's source (cluster.py:311-325)."""
        return self._fetch(1, edge_ids, src_nodes, origin)

    # -- telemetry (cluster.py:329-345) ----------------------------------------------------------
    def all_telemetry(self) -> list[tuple[int, int, WorkerTelemetry]]:
        return [(m.index, w.rank, w.telemetry) for m in self.machines for w in m.workers]

    def rank_group_cv(self, metric: str = "requests_served") -> dict[int, float]:
        return {r: measure_cv([getattr(m.workers[r].telemetry, metric) for m in self.machines])
                for r in range(self.spec.workers_per_machine)}
