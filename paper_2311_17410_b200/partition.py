"""Edge-cut hash partitioning helpers (reference partition.py:1-83), vectorised.

Same names and results as the reference: ``assign`` is ``node % P``
(partition.py:38-39); ``dispatch`` splits a batch into per-partition batches
in stream order, a directed edge going to its source's owner and an
undirected edge to both endpoints' owners, once when they coincide
(partition.py:42-55); ``balance_stats`` counts first-seen nodes and routed
edges per partition with their coefficient of variation (partition.py:58-83).
The device-side counterpart used by the partitioned sampler is the owner
bucketing in ``partitioned.PartitionedGraph``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .storage import InsertionBatch


@dataclass(frozen=True)
class PartitionSpec:
    num_partitions: int
    hash_kind: str = "identity"

    def __post_init__(self):
        if self.num_partitions < 1:
            raise ValueError("need at least one partition")
        if self.hash_kind != "identity":
            raise ValueError(f"unknown hash kind {self.hash_kind!r}")


@dataclass(frozen=True)
class BalanceStats:
    node_counts: tuple[int, ...]
    edge_counts: tuple[int, ...]
    node_cv: float
    edge_cv: float


def assign(spec: PartitionSpec, node: int) -> int:
    return int(node) % spec.num_partitions


def _columns(batch) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    edges = batch.edges if isinstance(batch, InsertionBatch) else batch
    arr = np.asarray(list(edges), dtype=np.int64).reshape(-1, 3)
    return arr[:, 0], arr[:, 1], arr[:, 2]


def _routes(spec: PartitionSpec, src: np.ndarray, dst: np.ndarray, directed: bool) -> np.ndarray:
    """bool [P, m]: edge j is stored by partition p."""
    P = spec.num_partitions
    p = np.arange(P, dtype=np.int64)[:, None]
    hit = (src % P)[None, :] == p
    if not directed:
        hit |= (dst % P)[None, :] == p
    return hit


def dispatch(spec: PartitionSpec, batch, directed: bool) -> list[InsertionBatch]:
    src, dst, ts = _columns(batch)
    hit = _routes(spec, src, dst, directed)
    return [InsertionBatch(list(zip(src[h].tolist(), dst[h].tolist(), ts[h].tolist()))) for h in hit]


def _cv(counts: np.ndarray) -> float:
    mean = counts.mean()
    if mean == 0:
        return 0.0
    return float(counts.std() / mean)


def balance_stats(spec: PartitionSpec, batch, directed: bool) -> BalanceStats:
    src, dst, _ = _columns(batch)
    P = spec.num_partitions
    # distinct nodes in first-seen order (src before dst per edge) -> owner counts
    nodes = np.unique(np.stack([src, dst], 1).reshape(-1))
    node_counts = np.bincount(nodes % P, minlength=P).astype(np.int64) if len(nodes) else np.zeros(P, np.int64)
    edge_counts = _routes(spec, src, dst, directed).sum(axis=1).astype(np.int64)
    return BalanceStats(node_counts=tuple(int(c) for c in node_counts), edge_counts=tuple(int(c) for c in edge_counts),
                        node_cv=_cv(node_counts), edge_cv=_cv(edge_counts))
