"""Device feature tables and the harness fetch block.

``NodeFeatureTable`` / ``EdgeFeatureTable`` mirror
/root/reference/pkg/src/ctdg/features.py:27-120 (same names, zeros + found
mask for unknown ids, strictly increasing edge ids) with rows in HBM.
``fetch_features`` is the per-minibatch block of harness.py:438-446:
cache.fetch -> table.get(miss) -> cache.insert_batch(found), in one call.
"""

from __future__ import annotations

import ctypes

import numpy as np

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

    def _put(self, ids, rows):
        import torch

        if isinstance(ids, torch.Tensor) and ids.is_cuda:
            i = ids.to(torch.int64).contiguous()
            r = rows.to(device=self.device, dtype=torch.float32).contiguous()
        else:
            i = torch.from_numpy(np.ascontiguousarray(np.asarray(ids, dtype=np.int64))).to(self.device)
            r = torch.from_numpy(np.ascontiguousarray(np.asarray(rows, dtype=np.float32))).to(self.device)
        if tuple(r.shape) != (i.numel(), self.dim):
            raise ValueError(f"rows must be ({i.numel()}, {self.dim}), got {tuple(r.shape)}")
        check(load().gf_ftable_put(self._h, ptr(i), int(i.numel()), ptr(r), stream_ptr()))

    def get(self, ids):
        """Rows for ids (zeros where unknown) and the found mask."""
        import torch

        on_dev = isinstance(ids, torch.Tensor) and ids.is_cuda
        i = ids.to(torch.int64).contiguous() if on_dev else \
            torch.from_numpy(np.ascontiguousarray(np.asarray(ids, dtype=np.int64))).to(self.device)
        n = int(i.numel())
        out = torch.zeros((n, self.dim), dtype=torch.float32, device=self.device)
        found = torch.zeros(n, dtype=torch.uint8, device=self.device)
        if n:
            check(load().gf_ftable_get(self._h, ptr(i), n, ptr(out), ptr(found), stream_ptr()))
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


class EdgeFeatureTable(_DeviceTable):
    """features.py:64-120 (append-only, strictly increasing ids; binary-search lookup)."""

    _KIND = 1

    def append(self, ids, rows) -> None:
        self._put(ids, rows)


def fetch_features(cache, table, keys, stream=None):
    """harness.py:438-446 as one device call.

    Returns (values, hit_mask, n_miss, admitted): ``values`` are complete rows
    (cache hits, and table rows for the misses; zeros for unknown ids).
    """
    import torch

    k = keys.to(torch.int64).contiguous() if isinstance(keys, torch.Tensor) else \
        torch.from_numpy(np.ascontiguousarray(np.asarray(keys, dtype=np.int64))).to(cache.device)
    n = int(k.numel())
    values = torch.empty((n, cache.dim), dtype=torch.float32, device=cache.device)
    hit = torch.empty(max(n, 1), dtype=torch.uint8, device=cache.device)
    nm, adm = ctypes.c_int64(), ctypes.c_int64()
    check(load().gf_fetch_features(cache.handle, table.handle, ptr(k), n, ptr(values), ptr(hit), ctypes.byref(nm),
                                   ctypes.byref(adm), stream_ptr(stream)))
    return values, hit[:n].bool(), int(nm.value), int(adm.value)
