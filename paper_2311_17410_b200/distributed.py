"""Multi-GPU replicated mode: one process per GPU, full graph replica per rank.

* Ingest: each rank holds a shard of the new edge batch; ``gather_edge_batch``
  all-gathers the shards (NCCL over NVLink on GPUs, gloo on CPU) into the
  global batch in rank order, and every rank appends it with the same
  deterministic K1 -- replicas stay identical (block handles are assigned by
  scan, not atomics).
* Sampling: each rank samples its own root shard.  ``root_key_base`` places
  the shard in the global root order (an exclusive prefix of per-rank root
  counts -- one integer per rank, not a data-path collective), so the union of
  the ranks' samples equals a single-GPU sample of all roots bit for bit
  (query keys are root_key_base + i and path-derived below that).
* No collective on the sampling path; the reference's distributed sampler
  reaches the same invariance with its content-keyed RNG (sampling.py:140-142,
  cluster.py:226-292).
* Features: tables too large to replicate (GDELT edge features are 142 GB) are
  sharded by owner = id % world (``ShardedFeatureTable``); a rank's cache misses
  are fetched from their owners with one id/row all-to-all round trip inside the
  fetch block (``fetch_features_sharded``; cluster.py:296-325 routes feature
  requests to the owner the same way).
"""

from __future__ import annotations


def _dist():
    import torch.distributed as dist

    return dist


def world() -> tuple[int, int]:
    dist = _dist()
    if not dist.is_available() or not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(), dist.get_rank()


def _coll_device(dev):
    """Device for collective buffers: the data's device under NCCL, the host under gloo (whose
    collectives run on CPU tensors; the CPU tests and 2-ranks-on-one-GPU tests use it)."""
    import torch

    return dev if _dist().get_backend() == "nccl" else torch.device("cpu")


def exclusive_prefix(count: int, device=None) -> tuple[int, int]:
    """(sum of counts on lower ranks, global total) for this rank's count."""
    import torch

    n, r = world()
    if n == 1:
        return 0, int(count)
    dist = _dist()
    t = torch.tensor([int(count)], dtype=torch.int64, device=_coll_device(device or torch.device("cpu")))
    allc = [torch.zeros_like(t) for _ in range(n)]
    dist.all_gather(allc, t)
    vals = [int(x.item()) for x in allc]
    return sum(vals[:r]), sum(vals)


def gather_edge_batch(src, dst, ts):
    """All-gather per-rank edge shards into the global batch (rank order).

    Shards may have different lengths: lengths are exchanged first and the
    shards padded to the longest one for a single all_gather_into_tensor.
    """
    import torch

    n, r = world()
    if n == 1:
        return src, dst, ts
    dist = _dist()
    out_dev = src.device
    dev = _coll_device(out_dev)
    local = torch.stack([src.to(dev, torch.int64), dst.to(dev, torch.int64), ts.to(dev, torch.int64)])  # [3, m]
    m = torch.tensor([local.shape[1]], dtype=torch.int64, device=dev)
    lens = [torch.zeros_like(m) for _ in range(n)]
    dist.all_gather(lens, m)
    lens = [int(x.item()) for x in lens]
    per = max(lens)
    pad = torch.zeros((3, per), dtype=torch.int64, device=dev)
    pad[:, : local.shape[1]] = local
    full = torch.empty((n, 3, per), dtype=torch.int64, device=dev)
    if hasattr(dist, "all_gather_into_tensor") and dev.type == "cuda":
        dist.all_gather_into_tensor(full, pad)
    else:
        parts = [torch.empty_like(pad) for _ in range(n)]
        dist.all_gather(parts, pad)
        full = torch.stack(parts)
    cols = [full[i, :, : lens[i]] for i in range(n)]
    batch = torch.cat(cols, dim=1).to(out_dev)
    return batch[0].contiguous(), batch[1].contiguous(), batch[2].contiguous()


def shard_range(total: int, n: int, r: int) -> tuple[int, int]:
    """Contiguous [lo, hi) slice of `total` items for rank r of n."""
    per = (total + n - 1) // n
    lo = min(total, r * per)
    return lo, min(total, lo + per)


class ReplicatedGraph:
    """A DynamicGraph replica per rank with all-gather ingest and sharded sampling."""

    def __init__(self, graph):
        self.graph = graph

    def ingest(self, src, dst, ts):
        """Append this rank's shard of a new batch; every rank applies the whole batch."""
        s, d, t = gather_edge_batch(src, dst, ts)
        return self.graph.add_edges_arrays(s, d, t)

    def sample(self, roots, ts, fanouts, strategy="recent", delta=0, seed=0):
        """Sample this rank's root shard; keys are positioned in the global root order."""
        from .sampling import TemporalSampler

        base, _ = exclusive_prefix(int(roots.numel()), device=roots.device)
        return TemporalSampler(self.graph, fanouts, strategy, delta, seed).sample(roots, ts, root_key_base=base)


class ShardedFeatureTable:
    """A feature table sharded over the ranks by owner = id % world.

    ``table`` is this rank's NodeFeatureTable / EdgeFeatureTable holding the rows of the ids it
    owns.  ``get`` answers any id: the ids are bucketed by owner on the GPU, exchanged with one
    all-to-all (NCCL over NVLink), looked up by their owners and the rows returned with a second
    all-to-all (partitioned.PartitionedFeatures).  With one rank it is the local table."""

    def __init__(self, table, transport=None):
        self.table = table
        self.dim = table.dim
        self.world, self.rank = world()
        self.remote = None
        if self.world > 1:
            from .partitioned import DistTransport, PartitionedFeatures

            self.remote = PartitionedFeatures(transport or DistTransport(), table, table.dim)

    @staticmethod
    def owns(ids, world_size: int, rank: int):
        """Mask of the ids a rank stores."""
        return (ids % world_size) == rank

    def get(self, ids):
        return self.remote.get(ids) if self.remote is not None else self.table.get(ids)


def fetch_features_sharded(cache, sharded: ShardedFeatureTable, keys):
    """The fetch block (harness.py:438-446) over a sharded table: one rank -> the fused local
    block (gf_fetch_features); several -> cache probe, owner fetch of the distinct misses over
    NCCL, insert.  Returns (values, hit_mask, n_miss, admitted) with complete rows either way."""
    if sharded.remote is None:
        from .features import fetch_features

        return fetch_features(cache, sharded.table, keys)
    from .partitioned import fetch_features_partitioned

    return fetch_features_partitioned(cache, sharded.remote, keys)
