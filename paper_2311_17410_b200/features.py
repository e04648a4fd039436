"""Device feature tables, the harness fetch block, and the TGFF feature file.

``NodeFeatureTable`` / ``EdgeFeatureTable`` / ``NodeMemoryTable`` mirror
/root/reference/pkg/src/ctdg/features.py:27-157 (same names, zeros + found
mask for unknown ids, strictly increasing edge ids) with rows in HBM.
``fetch_features`` is the per-minibatch block of harness.py:438-446:
cache.fetch -> table.get(miss) -> cache.insert_batch(found), in one call.
``save_features`` / ``load_features`` / ``load_feature_table`` write and read the
reference's TGFF byte format (features.py:159-207), byte for byte.
"""

from __future__ import annotations

import csv
import ctypes
import struct

import numpy as np

FEATURE_MAGIC = b"TGFF"  # features.py:17-20
FEATURE_VERSION = 1
KIND_NODE = 0
KIND_EDGE = 1


class FeatureFormatError(ValueError):
    """Raised for malformed feature files (features.py:23-24)."""

from ._lib import check, load, ptr, stream_ptr


class _DeviceTable:
    _KIND = 0

    def __init__(self, dim: int, device=None):
        import torch

        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = torch.device(device)
        self.dim = int(dim)
        idx = self.device.index if self.device.index is not None else torch.cuda.current_device()
        h = ctypes.c_void_p()
        check(load().gf_ftable_create(self._KIND, self.dim, idx, ctypes.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                load().gf_ftable_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    def __len__(self) -> int:
        n = ctypes.c_int64()
        check(load().gf_ftable_size(self._h, ctypes.byref(n)))
        return int(n.value)

    def _stored_ids(self):
        """Stored ids ascending, as a device tensor (gf_ftable_ids)."""
        import torch

        n = len(self)
        out = torch.empty(max(n, 1), dtype=torch.int64, device=self.device)
        got = ctypes.c_int64()
        check(load().gf_ftable_ids(self._h, ptr(out), n, ctypes.byref(got), stream_ptr(device=self.device)))
        return out[: got.value]

    def _put(self, ids, rows):
        import torch

        if isinstance(ids, torch.Tensor) and ids.is_cuda:
            i = ids.to(device=self.device, dtype=torch.int64).contiguous()
            r = rows.to(device=self.device, dtype=torch.float32).contiguous()
        else:
            i = torch.from_numpy(np.ascontiguousarray(np.asarray(ids, dtype=np.int64))).to(self.device)
            r = torch.from_numpy(np.ascontiguousarray(np.asarray(rows, dtype=np.float32))).to(self.device)
        if tuple(r.shape) != (i.numel(), self.dim):
            raise ValueError(f"rows must be ({i.numel()}, {self.dim}), got {tuple(r.shape)}")
        check(load().gf_ftable_put(self._h, ptr(i), int(i.numel()), ptr(r), stream_ptr(device=self.device)))

    def get(self, ids):
        """Rows for ids (zeros where unknown) and the found mask."""
        import torch

        on_dev = isinstance(ids, torch.Tensor) and ids.is_cuda
        i = ids.to(device=self.device, dtype=torch.int64).contiguous() if on_dev else \
            torch.from_numpy(np.ascontiguousarray(np.asarray(ids, dtype=np.int64))).to(self.device)
        n = int(i.numel())
        out = torch.zeros((n, self.dim), dtype=torch.float32, device=self.device)
        found = torch.zeros(n, dtype=torch.uint8, device=self.device)
        if n:
            check(load().gf_ftable_get(self._h, ptr(i), n, ptr(out), ptr(found), stream_ptr(device=self.device)))
        if on_dev:
            return out, found.bool()
        return out.cpu().numpy(), found.cpu().numpy().astype(bool)


class NodeFeatureTable(_DeviceTable):
    """features.py:27-61 (rows indexed by non-negative node id; last write wins)."""

    _KIND = 0

    def set(self, node: int, row) -> None:
        row = np.asarray(row, dtype=np.float32)
        if row.shape != (self.dim,):
            raise ValueError(f"expected row of dim {self.dim}, got shape {row.shape}")
        self._put([int(node)], row.reshape(1, -1))

    def set_many(self, ids, rows) -> None:
        self._put(ids, rows)

    def __contains__(self, node: int) -> bool:
        return bool(self.get([int(node)])[1][0])

    def ids_sorted(self) -> np.ndarray:
        """features.py:60-61."""
        return self._stored_ids().cpu().numpy()

    @property
    def _rows(self) -> dict[int, np.ndarray]:
        """Host snapshot {node: row} of the device table (the reference keeps its rows in this dict,
        features.py:30; its harness tests read it)."""
        ids = self._stored_ids()
        if ids.numel() == 0:
            return {}
        rows = self.get(ids)[0].cpu().numpy()
        return {int(i): r for i, r in zip(ids.cpu().numpy().tolist(), rows)}


class EdgeFeatureTable(_DeviceTable):
    """features.py:64-120 (append-only, strictly increasing ids; binary-search lookup)."""

    _KIND = 1

    def append(self, ids, rows) -> None:
        self._put(ids, rows)

    @property
    def ids(self) -> np.ndarray:
        """features.py:76-78."""
        return self._stored_ids().cpu().numpy()

    @property
    def values(self) -> np.ndarray:
        """features.py:80-82 (rows in id order)."""
        ids = self._stored_ids()
        if ids.numel() == 0:
            return np.zeros((0, self.dim), dtype=np.float32)
        return self.get(ids)[0].cpu().numpy()


class NodeMemoryTable(NodeFeatureTable):
    """features.py:123-156: per-node state rows in HBM (upsert) plus the host-side
    ``last_update`` map the reference exposes."""

    def __init__(self, dim: int, device=None):
        super().__init__(dim, device)
        self.last_update: dict[int, int] = {}

    def update(self, ids, rows, timestamps) -> None:
        ids_np = np.asarray(ids.cpu() if hasattr(ids, "cpu") else ids, dtype=np.int64)
        shape = tuple(rows.shape) if hasattr(rows, "shape") else np.asarray(rows).shape
        if shape != (len(ids_np), self.dim):
            raise ValueError(f"rows must be ({len(ids_np)}, {self.dim}), got {shape}")
        if len(ids_np) == 0:
            return
        self._put(ids, rows)
        ts_np = np.asarray(timestamps.cpu() if hasattr(timestamps, "cpu") else timestamps, dtype=np.int64)
        for node, t in zip(ids_np.tolist(), ts_np.tolist()):
            self.last_update[node] = t


def fetch_features(cache, table, keys, stream=None):
    """harness.py:438-446 as one device call.

    Returns (values, hit_mask, n_miss, admitted): ``values`` are complete rows
    (cache hits, and table rows for the misses; zeros for unknown ids).
    """
    import torch

    # host tensors and tensors on another device are moved to the cache's device first: the kernels
    # dereference the key pointer on that device
    k = keys.to(device=cache.device, dtype=torch.int64).contiguous() if isinstance(keys, torch.Tensor) else \
        torch.from_numpy(np.ascontiguousarray(np.asarray(keys, dtype=np.int64))).to(cache.device)
    n = int(k.numel())
    values = torch.empty((n, cache.dim), dtype=torch.float32, device=cache.device)
    hit = torch.empty(max(n, 1), dtype=torch.uint8, device=cache.device)
    if stream is not None:  # the block's last kernels (the insert) still read values on that stream
        for t in (k, values, hit):
            t.record_stream(stream)
    nm, adm = ctypes.c_int64(), ctypes.c_int64()
    check(load().gf_fetch_features(cache.handle, table.handle, ptr(k), n, ptr(values), ptr(hit), ctypes.byref(nm),
                                   ctypes.byref(adm), stream_ptr(stream, cache.device)))
    return values, hit[:n].bool(), int(nm.value), int(adm.value)


# ---------------------------------------------------------------------------
# TGFF feature files (features.py:159-221); host byte format, identical bytes
# ---------------------------------------------------------------------------

_HDR = "<IBIQ"


def save_features(sink, kind: int, dim: int, ids, rows) -> None:
    """features.py:159-166: magic, version, kind, dim, count, ids (u64), f32 rows."""
    ids = np.asarray(ids, dtype="<i8")
    rows = np.ascontiguousarray(rows, dtype="<f4")
    sink.write(FEATURE_MAGIC)
    sink.write(struct.pack(_HDR, FEATURE_VERSION, kind, dim, len(ids)))
    sink.write(ids.astype("<u8").tobytes())
    sink.write(rows.tobytes())


def load_features(source):
    """features.py:169-184 -> (kind, dim, ids int64, rows f32 [count, dim])."""
    data = source.read() if hasattr(source, "read") else bytes(source)
    if data[:4] != FEATURE_MAGIC:
        raise FeatureFormatError("bad feature-file magic")
    version, kind, dim, count = struct.unpack_from(_HDR, data, 4)
    if version != FEATURE_VERSION:
        raise FeatureFormatError(f"unsupported feature-file version {version}")
    pos = 4 + struct.calcsize(_HDR)
    if len(data) != pos + count * 8 + count * dim * 4:
        raise FeatureFormatError("feature file length mismatch")
    ids = np.frombuffer(data, dtype="<u8", count=count, offset=pos).astype(np.int64)
    rows = np.frombuffer(data, dtype="<f4", count=count * dim, offset=pos + count * 8)
    return kind, dim, ids, rows.reshape(count, dim).copy()


def save_node_features(table: NodeFeatureTable, sink) -> None:
    """features.py:187-190 (ids ascending)."""
    ids = table._stored_ids()
    rows = table.get(ids)[0].cpu().numpy() if ids.numel() else np.zeros((0, table.dim), np.float32)
    save_features(sink, KIND_NODE, table.dim, ids.cpu().numpy(), rows)


def save_edge_features(table: EdgeFeatureTable, sink) -> None:
    """features.py:193-194."""
    save_features(sink, KIND_EDGE, table.dim, table.ids, table.values)


def load_feature_table(source, device=None):
    """features.py:197-207: a device table of the file's kind."""
    kind, dim, ids, rows = load_features(source)
    if kind == KIND_NODE:
        table = NodeFeatureTable(dim, device)
        if len(ids):
            table.set_many(ids, rows)
        return table
    if kind == KIND_EDGE:
        table = EdgeFeatureTable(dim, device)
        if len(ids):
            table.append(ids, rows)
        return table
    raise FeatureFormatError(f"unknown feature kind {kind}")


def load_features_csv(path, dim: int):
    """features.py:210-221: id,v0,v1,... per line -> (ids int64, rows f32)."""
    ids, rows = [], []
    with open(path, newline="") as fh:
        for row in csv.reader(fh):
            if not row or row[0].startswith("#"):
                continue
            ids.append(int(row[0]))
            vals = [float(x) for x in row[1:]]
            if len(vals) != dim:
                raise FeatureFormatError(f"expected {dim} values, got {len(vals)}")
            rows.append(vals)
    return np.array(ids, dtype=np.int64), np.array(rows, dtype=np.float32)
