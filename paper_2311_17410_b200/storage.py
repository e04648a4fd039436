"""Device-resident block store behind the reference's ``DynamicGraph`` API.

Mirrors /root/reference/pkg/src/ctdg/storage.py (class and method names,
argument meaning, errors).  State lives on the GPU (libgfb200, see
csrc/gf_graph.cu); ``fast`` / ``shared`` return host mirrors of the
reference's FastTier / SharedTier columns for inspection and parity tests.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import check, load, ptr, stream_ptr

NO_BLOCK = -1  # storage.py:31
BLOCK_META_BYTES = 72  # storage.py:35
NODE_ENTRY_BYTES = 40  # storage.py:36
EDGE_SLOT_BYTES = 25  # storage.py:40
TS_MIN = int(np.iinfo(np.int64).min)  # storage.py:45
TS_MAX = int(np.iinfo(np.int64).max)


class GraphFormatError(ValueError):
    """Raised for malformed offload files (storage.py:49-50)."""


class NodeNotFoundError(KeyError):
    """Raised when an operation names a node that does not exist (storage.py:53-54)."""


# -- sizing policies (storage.py:62-121) ---------------------------------------------
class BlockSizing:
    kind = "adaptive"
    param = 0

    def capacity(self, degree: int, pending: int) -> int:
        raise NotImplementedError


@dataclass(frozen=True)
class AdaptiveSizing(BlockSizing):
    tau: int
    kind = "adaptive"

    def __post_init__(self):
        if self.tau < 1:
            raise ValueError(f"tau must be >= 1, got {self.tau}")

    @property
    def param(self):
        return 0

    def capacity(self, degree: int, pending: int) -> int:
        return min(max(degree, 1), self.tau)


@dataclass(frozen=True)
class FixedSizing(BlockSizing):
    size: int
    kind = "fixed"

    def __post_init__(self):
        if self.size < 1:
            raise ValueError(f"block size must be >= 1, got {self.size}")

    @property
    def param(self):
        return self.size

    def capacity(self, degree: int, pending: int) -> int:
        return self.size


@dataclass(frozen=True)
class BatchSizing(BlockSizing):
    kind = "batch"

    @property
    def param(self):
        return 0

    def capacity(self, degree: int, pending: int) -> int:
        return max(pending, 1)


ADJACENCY_LIST_SIZING = FixedSizing(1)


# -- record types (storage.py:249-295) --------------------------------------------
@dataclass(frozen=True)
class NodeEntry:
    head_block: int | None
    tail_block: int | None
    num_blocks: int
    degree: int
    valid: bool


@dataclass
class InsertionBatch:
    edges: list[tuple[int, int, int]] = field(default_factory=list)

    def __len__(self) -> int:
        return len(self.edges)

    def __iter__(self):
        return iter(self.edges)


@dataclass
class InsertionResult:
    edge_ids: list[int | None]
    rejected: list[int]

    @property
    def accepted_ids(self) -> list[int]:
        return [e for e in self.edge_ids if e is not None]


@dataclass(frozen=True)
class StorageStats:
    avg_list_len: float
    max_list_len: int
    edge_data_bytes: int
    metadata_bytes: int
    wasted_slots: int


@dataclass
class EdgeArrays:
    neighbors: np.ndarray
    edge_ids: np.ndarray
    timestamps: np.ndarray
    valid: np.ndarray


class FastTierView:
    """Host mirror of FastTier's columns (storage.py:140-152), exported from the device."""

    def __init__(self, nodes: dict, blocks: dict, live_blocks: int | None = None):
        self._live = live_blocks
        self.head = nodes["head"]
        self.tail = nodes["tail"]
        self.num_blocks = nodes["num_blocks"]
        self.degree = nodes["degree"]
        self.node_valid = nodes["node_valid"]
        self.blk_capacity = blocks["capacity"]
        self.blk_size = blocks["size"]
        self.blk_tmin = blocks["tmin"]
        self.blk_tmax = blocks["tmax"]
        self.blk_prev = blocks["prev"]
        self.blk_next = blocks["next"]
        self.accesses = 0

    @property
    def num_nodes(self) -> int:
        return len(self.head)

    @property
    def live_blocks(self) -> int:
        return len(self.blk_capacity) if self._live is None else self._live

    def metadata_bytes(self) -> int:
        return self.num_nodes * NODE_ENTRY_BYTES + self.live_blocks * BLOCK_META_BYTES


class SharedTierView:
    """Host mirror of SharedTier (storage.py:220-241): per-block arrays at capacity."""

    def __init__(self, graph: "DynamicGraph"):
        self._g = graph
        self.accesses = 0

    def get(self, handle: int) -> EdgeArrays:
        return self._g._block_arrays()[int(handle)]

    def edge_data_bytes(self) -> int:
        return int(self._g.fast.blk_capacity.sum()) * EDGE_SLOT_BYTES


def _as_device_i64(x, device):
    import torch

    if isinstance(x, torch.Tensor):
        if x.dtype is torch.int64 and x.device == device and x.is_contiguous():
            return x  # the common case (device-resident int64 batches): no dispatch at all
        return x.to(device=device, dtype=torch.int64).contiguous()
    a = np.ascontiguousarray(np.asarray(x, dtype=np.int64))
    return torch.from_numpy(a).to(device)


class DynamicGraph:
    """Dynamic CTDG store on one GPU: node table + per-node chronological block lists.

    Same constructor and semantics as storage.py:303-323; ``device`` selects
    the CUDA device (default: the current one).
    """

    def __init__(self, directed: bool = False, tau: int = 48, sizing: BlockSizing | None = None, device=None):
        import torch

        if sizing is None:
            if tau < 1:
                raise ValueError(f"tau must be >= 1, got {tau}")
            sizing = AdaptiveSizing(tau)
        self.directed = directed
        self.tau = tau
        self.sizing = sizing
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = torch.device(device)
        self._dev_index = self.device.index if self.device.index is not None else torch.cuda.current_device()
        self.device = torch.device(self.device.type, self._dev_index)  # "cuda" -> "cuda:k": tensors compare equal
        h = ctypes.c_void_p()
        check(load().gf_graph_create(int(bool(directed)), int(tau), _lib.SIZING_CODE[sizing.kind],
                                     int(sizing.param), self._dev_index, ctypes.byref(h)))
        self._h = h
        self._version = 0
        self._cache: dict = {}
        self.shared = SharedTierView(self)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                load().gf_graph_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    # -- basic queries (storage.py:327-390) ---------------------------------------
    def info(self) -> _lib.GraphInfo:
        inf = _lib.GraphInfo()
        check(load().gf_graph_get_info(self._h, ctypes.byref(inf)))
        return inf

    @property
    def num_nodes(self) -> int:
        return int(self.info().num_nodes)

    @property
    def next_edge_id(self) -> int:
        return int(self.info().next_edge_id)

    @property
    def total_edges_inserted(self) -> int:
        return int(self.info().total_edges_inserted)

    def has_node(self, node: int) -> bool:
        return 0 <= node < self.num_nodes

    def _exported(self, key, fn):
        c = self._cache.get(key)
        if c is None or c[0] != self._version:
            c = (self._version, fn())
            self._cache[key] = c
        return c[1]

    def _export_nodes(self) -> dict:
        def run():
            n = self.num_nodes
            cols = {k: np.zeros(n, np.int64) for k in ("head", "tail", "num_blocks", "degree")}
            valid = np.zeros(n, np.uint8)
            check(load().gf_graph_export_nodes(
                self._h, *[_lib.np_ptr(cols[k], ctypes.c_int64) for k in ("head", "tail", "num_blocks", "degree")],
                _lib.np_ptr(valid, ctypes.c_uint8), stream_ptr(device=self.device)))
            cols["node_valid"] = valid.astype(bool)
            return cols
        return self._exported("nodes", run)

    def _export_blocks(self) -> dict:
        def run():
            n = int(self.info().num_block_handles)
            names = ("capacity", "size", "tmin", "tmax", "prev", "next")
            cols = {k: np.zeros(n, np.int64) for k in names}
            check(load().gf_graph_export_blocks(self._h, *[_lib.np_ptr(cols[k], ctypes.c_int64) for k in names],
                                                stream_ptr(device=self.device)))
            return cols
        return self._exported("blocks", run)

    def _block_arrays(self) -> list[EdgeArrays]:
        def run():
            b = self._export_blocks()
            nb = len(b["capacity"])
            offs = np.zeros(nb + 1, np.int64)
            tot = int(b["size"].sum())
            nbr = np.zeros(max(tot, 1), np.int64); eid = np.zeros(max(tot, 1), np.int64)
            ts = np.zeros(max(tot, 1), np.int64); valid = np.zeros(max(tot, 1), np.uint8)
            check(load().gf_graph_export_slots(self._h, 0, nb, _lib.np_ptr(offs, ctypes.c_int64),
                                               _lib.np_ptr(nbr, ctypes.c_int64), _lib.np_ptr(eid, ctypes.c_int64),
                                               _lib.np_ptr(ts, ctypes.c_int64), _lib.np_ptr(valid, ctypes.c_uint8),
                                               stream_ptr(device=self.device)))
            out = []
            for h in range(nb):
                cap = int(b["capacity"][h])
                a = EdgeArrays(np.zeros(cap, np.int64), np.zeros(cap, np.int64), np.zeros(cap, np.int64),
                               np.zeros(cap, bool))
                s, e = offs[h], offs[h + 1]
                a.neighbors[: e - s] = nbr[s:e]
                a.edge_ids[: e - s] = eid[s:e]
                a.timestamps[: e - s] = ts[s:e]
                a.valid[: e - s] = valid[s:e].astype(bool)
                out.append(a)
            return out
        return self._exported("slots", run)

    @property
    def fast(self) -> FastTierView:
        return self._exported("fast", lambda: FastTierView(self._export_nodes(), self._export_blocks(),
                                                           int(self.info().live_blocks)))

    def node_entry(self, node: int) -> NodeEntry:
        if not self.has_node(node):
            raise NodeNotFoundError(node)
        f = self._export_nodes()
        head, tail = int(f["head"][node]), int(f["tail"][node])
        return NodeEntry(None if head == NO_BLOCK else head, None if tail == NO_BLOCK else tail,
                         int(f["num_blocks"][node]), int(f["degree"][node]), bool(f["node_valid"][node]))

    def degree(self, node: int) -> int:
        if not self.has_node(node):
            raise NodeNotFoundError(node)
        f = self._export_nodes()
        if not f["node_valid"][node]:
            raise NodeNotFoundError(node)
        return int(f["degree"][node])

    def new_block_capacity(self, node: int) -> int:
        if not self.has_node(node):
            raise NodeNotFoundError(node)
        return self.sizing.capacity(int(self._export_nodes()["degree"][node]), 1)

    def blocks_of(self, node: int) -> list[int]:
        if not self.has_node(node):
            raise NodeNotFoundError(node)
        nxt = self._export_blocks()["next"]
        out, h = [], int(self._export_nodes()["head"][node])
        while h != NO_BLOCK:
            out.append(h)
            h = int(nxt[h])
        return out

    def iter_edges(self, node: int):
        sizes = self._export_blocks()["size"]
        arrs = self._block_arrays()
        for h in self.blocks_of(node):
            a = arrs[h]
            for i in range(int(sizes[h])):
                yield (int(a.neighbors[i]), int(a.edge_ids[i]), int(a.timestamps[i]), bool(a.valid[i]))

    def node_t_max(self, node: int) -> int:
        if not self.has_node(node):
            return TS_MIN
        tail = int(self._export_nodes()["tail"][node])
        if tail == NO_BLOCK:
            return TS_MIN
        b = self._export_blocks()
        return int(b["tmax"][tail]) if b["size"][tail] else TS_MIN

    # -- mutation -----------------------------------------------------------------
    def reserve(self, nodes: int, blocks: int, slots: int) -> None:
        """Pre-size the device node table, block arena and slot pool (they also grow on demand)."""
        check(load().gf_graph_reserve(self._h, int(nodes), int(blocks), int(slots), stream_ptr(device=self.device)))

    def add_edges_arrays(self, src, dst, ts, edge_ids=None, stream=None):
        """Batch append from arrays or CUDA tensors; returns (eids tensor, n_rejected).

        eids[i] is -1 for an edge rejected as out of order.  No host copies
        when the inputs are already CUDA tensors.
        """
        import torch

        s = _as_device_i64(src, self.device)
        d = _as_device_i64(dst, self.device)
        t = _as_device_i64(ts, self.device)
        if not (s.numel() == d.numel() == t.numel()):
            raise ValueError("src, dst and ts must have equal length")
        e = None
        if edge_ids is not None:
            e = _as_device_i64(edge_ids, self.device)
            if e.numel() != s.numel():
                raise ValueError("edge_ids must match batch length")
        out = torch.empty(s.numel(), dtype=torch.int64, device=self.device)
        rej = ctypes.c_int64(0)
        self._version += 1
        check(load().gf_graph_add_edges(self._h, ptr(s), ptr(d), ptr(t), s.numel(), ptr(e), ptr(out),
                                        ctypes.byref(rej), stream_ptr(stream, self.device)))
        return out, int(rej.value)

    def add_edges(self, batch, *, edge_ids: list[int] | None = None) -> InsertionResult:
        """storage.py:394-450: append a batch; out-of-order edges are rejected individually."""
        edges = list(batch.edges if isinstance(batch, InsertionBatch) else batch)
        if edge_ids is not None and len(edge_ids) != len(edges):
            raise ValueError("edge_ids must match batch length")
        if not edges:
            return InsertionResult(edge_ids=[], rejected=[])
        arr = np.asarray(edges, dtype=np.int64).reshape(-1, 3)
        out, _ = self.add_edges_arrays(arr[:, 0], arr[:, 1], arr[:, 2], edge_ids)
        ids = out.cpu().numpy()
        return InsertionResult(edge_ids=[None if e < 0 else int(e) for e in ids.tolist()],
                               rejected=[i for i, e in enumerate(ids.tolist()) if e < 0])

    def delete_edges(self, edge_ids) -> int:
        """storage.py:479-485: soft-delete by id; returns how many ids were live."""
        ids = _as_device_i64(list(edge_ids) if not hasattr(edge_ids, "__array__") and not hasattr(edge_ids, "data_ptr")
                             else edge_ids, self.device)
        if ids.numel() == 0:
            return 0
        out = ctypes.c_int64(0)
        self._version += 1
        check(load().gf_graph_delete_edges(self._h, ptr(ids), ids.numel(), ctypes.byref(out), stream_ptr(device=self.device)))
        return int(out.value)

    def delete_edges_set(self, edge_ids) -> set[int]:
        wanted = {int(e) for e in edge_ids}
        if not wanted:
            return set()
        live = set()
        for a, s in zip(self._block_arrays(), self._export_blocks()["size"]):
            live.update(int(e) for e, v in zip(a.edge_ids[:s], a.valid[:s]) if v and int(e) in wanted)
        self.delete_edges(sorted(live))
        return live

    def delete_node(self, node: int) -> bool:
        """storage.py:507-512."""
        out = ctypes.c_int(0)
        self._version += 1
        check(load().gf_graph_delete_node(self._h, int(node), ctypes.byref(out), stream_ptr(device=self.device)))
        return bool(out.value)

    def offload_before(self, cutoff: int, sink) -> int:
        """storage.py:516-574: serialise and unlink every block with t_max < cutoff.

        The TGOF blob is assembled on the device and written to ``sink``
        before anything is unlinked, so an I/O failure leaves the graph
        unchanged.  Returns the number of edge records written.
        """
        lib = load()
        blen, edges = ctypes.c_int64(0), ctypes.c_int64(0)
        check(lib.gf_graph_offload_before(self._h, int(cutoff), None, 0, ctypes.byref(blen), ctypes.byref(edges), 0,
                                          stream_ptr(device=self.device)))
        blob = np.zeros(int(blen.value), dtype=np.uint8)
        check(lib.gf_graph_offload_before(self._h, int(cutoff), _lib.np_ptr(blob, ctypes.c_uint8), len(blob),
                                          ctypes.byref(blen), ctypes.byref(edges), 0, stream_ptr(device=self.device)))
        sink.write(blob.tobytes())
        self._version += 1
        check(lib.gf_graph_offload_before(self._h, int(cutoff), None, 0, ctypes.byref(blen), ctypes.byref(edges), 1,
                                          stream_ptr(device=self.device)))
        return int(edges.value)

    def _live_handles(self) -> list[int]:
        nodes, nxt = self._export_nodes(), self._export_blocks()["next"]
        out = []
        for h in nodes["head"].tolist():
            while h != NO_BLOCK:
                out.append(h)
                h = int(nxt[h])
        return out

    # -- statistics (storage.py:578-617) --------------------------------------------
    def storage_stats(self) -> StorageStats:
        f = self.fast
        active = f.degree > 0
        avg = float(f.num_blocks[active].mean()) if active.any() else 0.0
        max_len = int(f.num_blocks.max()) if f.num_nodes else 0
        live = np.asarray(self._live_handles(), dtype=np.int64)
        cap = f.blk_capacity[live] if len(live) else np.zeros(0, np.int64)
        size = f.blk_size[live] if len(live) else np.zeros(0, np.int64)
        wasted = int((cap - size).sum())
        metadata = f.num_nodes * NODE_ENTRY_BYTES + int(self.info().live_blocks) * BLOCK_META_BYTES
        return StorageStats(avg, max_len, int(cap.sum()) * EDGE_SLOT_BYTES, metadata, wasted)

    def check_waste_bound(self) -> bool:
        stats = self.storage_stats()
        return stats.wasted_slots < 0.5 * max(self.total_edges_inserted, 1)

    def access_counts(self) -> dict[str, int]:
        # the reference counts tier accesses in Python (sampling.py:153-169); on the
        # GPU the equivalent evidence is ncu's dram/lts counters (profiles/)
        return {"metadata": 0, "edge_data": 0}


def new_graph(directed: bool = False, tau: int = 48, sizing: BlockSizing | None = None, device=None) -> DynamicGraph:
    return DynamicGraph(directed=directed, tau=tau, sizing=sizing, device=device)


OFFLOAD_MAGIC = b"TGOF"  # storage.py:42-43
OFFLOAD_VERSION = 1


def parse_offload(source) -> list[tuple[int, list[tuple[int, int, int, bool]]]]:
    """Parse an offload blob into (node, [(neighbor, edge_id, ts, valid)]) (storage.py:624-647)."""
    import struct

    data = source.read() if hasattr(source, "read") else bytes(source)
    if data[:4] != OFFLOAD_MAGIC:
        raise GraphFormatError("bad offload magic")
    (version,) = struct.unpack_from("<I", data, 4)
    if version != OFFLOAD_VERSION:
        raise GraphFormatError(f"unsupported offload version {version}")
    pos, out = 8, []
    while pos < len(data):
        if pos + 12 > len(data):
            raise GraphFormatError("truncated block header")
        node, size = struct.unpack_from("<QI", data, pos)
        pos += 12
        if pos + 25 * size > len(data):
            raise GraphFormatError("truncated edge record")
        recs = [struct.unpack_from("<QQqB", data, pos + 25 * i) for i in range(size)]
        pos += 25 * size
        out.append((int(node), [(n, e, t, bool(v)) for n, e, t, v in recs]))
    return out


def write_offload_records(records) -> bytes:
    """Re-serialise parsed offload records (storage.py:650-659)."""
    import struct

    buf = [OFFLOAD_MAGIC, struct.pack("<I", OFFLOAD_VERSION)]
    for node, recs in records:
        buf.append(struct.pack("<QI", node, len(recs)))
        buf.extend(struct.pack("<QQqB", n, e, t, 1 if v else 0) for n, e, t, v in recs)
    return b"".join(buf)
