"""GPU-resident vectorised feature cache behind the reference's ``VectorCache`` API.

Mirrors /root/reference/pkg/src/ctdg/cache.py (policies lru/lfu/fifo, the
per-call admission cap floor(lam * capacity), batch scoring, lowest
(score, slot) eviction, snapshot/restore, TGCS persist/load).  State lives in
device memory (csrc/gf_cache.cu); ``keys``/``scores``/``storage``/``slot_of``
are host mirrors for inspection; assigning ``scores`` writes through.
"""

from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check, load, ptr, stream_ptr

POLICIES = ("lru", "lfu", "fifo")
_POLICY_CODE = {"lru": 0, "lfu": 1, "fifo": 2}
_POLICY_NAME = {v: k for k, v in _POLICY_CODE.items()}
EMPTY_KEY = -1
SNAPSHOT_MAGIC = b"TGCS"
SNAPSHOT_VERSION = 1


class SnapshotMismatchError(ValueError):
    """cache.py:35-36."""


class SnapshotFormatError(ValueError):
    """cache.py:39-40."""


@dataclass
class CacheSnapshot:
    """cache.py:43-52.  Holds host copies plus (optionally) a device snapshot handle."""

    policy: str
    capacity: int
    dim: int
    lam: float
    keys: np.ndarray
    scores: np.ndarray
    fifo_head: int
    storage: np.ndarray


class _ScoresView(np.ndarray):
    """Host copy of scores whose slice assignment writes through to the device."""

    def __setitem__(self, idx, value):
        super().__setitem__(idx, value)
        owner = getattr(self, "_owner", None)
        if owner is not None:
            owner._set_state(scores=np.asarray(self, dtype=np.int64))


class VectorCache:
    def __init__(self, policy: str, capacity: int, dim: int, lam: float = 0.2, device=None):
        import torch

        if policy not in POLICIES:
            raise ValueError(f"unknown cache policy {policy!r}")
        if capacity < 1:
            raise ValueError("capacity must be >= 1")
        if not 0.0 < lam <= 1.0:
            raise ValueError("lam must be in (0, 1]")
        self.policy, self.capacity, self.dim, self.lam = policy, int(capacity), int(dim), float(lam)
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = torch.device(device)
        idx = self.device.index if self.device.index is not None else torch.cuda.current_device()
        h = ctypes.c_void_p()
        check(load().gf_cache_create(_POLICY_CODE[policy], self.capacity, self.dim, self.lam, idx, ctypes.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                load().gf_cache_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def max_update(self) -> int:  # cache.py:79-81
        return int(self.lam * self.capacity)

    # -- state mirrors -----------------------------------------------------------------
    def _get_state(self):
        keys = np.zeros(self.capacity, np.int64)
        scores = np.zeros(self.capacity, np.int64)
        storage = np.zeros((self.capacity, self.dim), np.float32)
        head = ctypes.c_int64(0)
        check(load().gf_cache_get_state(self._h, _lib.np_ptr(keys, ctypes.c_int64), _lib.np_ptr(scores, ctypes.c_int64),
                                        _lib.np_ptr(storage, ctypes.c_float), ctypes.byref(head), stream_ptr(device=self.device)))
        return keys, scores, storage, int(head.value)

    def _set_state(self, keys=None, scores=None, storage=None, fifo_head=None):
        k = None if keys is None else np.ascontiguousarray(keys, dtype=np.int64)
        s = None if scores is None else np.ascontiguousarray(scores, dtype=np.int64)
        r = None if storage is None else np.ascontiguousarray(storage, dtype=np.float32)
        head = self.fifo_head if fifo_head is None else int(fifo_head)
        check(load().gf_cache_set_state(self._h, None if k is None else _lib.np_ptr(k, ctypes.c_int64),
                                        None if s is None else _lib.np_ptr(s, ctypes.c_int64),
                                        None if r is None else _lib.np_ptr(r, ctypes.c_float), head, stream_ptr(device=self.device)))

    @property
    def keys(self) -> np.ndarray:
        return self._get_state()[0]

    @property
    def scores(self) -> np.ndarray:
        v = self._get_state()[1].view(_ScoresView)
        v._owner = self
        return v

    @scores.setter
    def scores(self, value):
        self._set_state(scores=np.asarray(value, dtype=np.int64))

    @property
    def storage(self) -> np.ndarray:
        return self._get_state()[2]

    @property
    def fifo_head(self) -> int:
        head = ctypes.c_int64(0)
        check(load().gf_cache_get_state(self._h, None, None, None, ctypes.byref(head), stream_ptr(device=self.device)))
        return int(head.value)

    @property
    def slot_of(self) -> dict[int, int]:
        return {int(k): i for i, k in enumerate(self.keys.tolist()) if k != EMPTY_KEY}

    def __len__(self) -> int:
        return int(np.count_nonzero(self.keys != EMPTY_KEY))

    # -- core operations (cache.py:85-177) ---------------------------------------------
    def fetch_device(self, keys, stream=None):
        """Device fetch: keys CUDA int64 tensor -> (values, hit_mask, miss_keys) CUDA tensors."""
        import torch

        n = int(keys.numel())
        values = torch.empty((n, self.dim), dtype=torch.float32, device=self.device)
        hit = torch.empty(n, dtype=torch.uint8, device=self.device)
        miss = torch.empty(max(n, 1), dtype=torch.int64, device=self.device)
        nm = ctypes.c_int64(0)
        check(load().gf_cache_fetch(self._h, ptr(keys), n, ptr(values), ptr(hit), ptr(miss), ctypes.byref(nm),
                                    stream_ptr(stream, self.device)))
        return values, hit.bool(), miss[: int(nm.value)]

    def fetch(self, keys):
        """Batched lookup: (values, hit_mask, miss_keys) as in cache.py:85-121."""
        import torch

        if isinstance(keys, torch.Tensor) and keys.is_cuda:
            return self.fetch_device(keys.to(torch.int64).contiguous())
        k = np.ascontiguousarray(np.asarray(keys, dtype=np.int64))
        if len(k) == 0:
            return np.zeros((0, self.dim), np.float32), np.zeros(0, bool), np.empty(0, np.int64)
        v, h, m = self.fetch_device(torch.from_numpy(k).to(self.device))
        return v.cpu().numpy(), h.cpu().numpy(), m.cpu().numpy()

    def insert_batch(self, keys, values) -> int:
        """Admit at most floor(lam * capacity) new entries (cache.py:123-167)."""
        import torch

        on_dev = isinstance(keys, torch.Tensor) and keys.is_cuda
        if on_dev:
            k = keys.to(torch.int64).contiguous()
            v = values.to(device=self.device, dtype=torch.float32).contiguous()
            if tuple(v.shape) != (k.numel(), self.dim):
                raise ValueError(f"values must be ({k.numel()}, {self.dim}), got {tuple(v.shape)}")
        else:
            kn = np.ascontiguousarray(np.asarray(keys, dtype=np.int64))
            vn = np.ascontiguousarray(np.asarray(values, dtype=np.float32))
            if vn.shape != (len(kn), self.dim):
                raise ValueError(f"values must be ({len(kn)}, {self.dim}), got {vn.shape}")
            if len(kn) == 0:
                return 0
            k = torch.from_numpy(kn).to(self.device)
            v = torch.from_numpy(vn.reshape(len(kn), self.dim)).to(self.device)
        adm = ctypes.c_int64(0)
        check(load().gf_cache_insert(self._h, ptr(k), int(k.numel()), ptr(v), ctypes.byref(adm), stream_ptr(device=self.device)))
        return int(adm.value)

    # -- snapshot / persistence (cache.py:181-233) --------------------------------------
    def snapshot(self) -> CacheSnapshot:
        keys, scores, storage, head = self._get_state()
        return CacheSnapshot(self.policy, self.capacity, self.dim, self.lam, keys, scores, head, storage)

    def restore(self, snap: CacheSnapshot) -> None:
        if (snap.policy, snap.capacity, snap.dim) != (self.policy, self.capacity, self.dim):
            raise SnapshotMismatchError(
                f"snapshot is ({snap.policy}, {snap.capacity}, {snap.dim}), "
                f"cache is ({self.policy}, {self.capacity}, {self.dim})")
        self._set_state(snap.keys, snap.scores, snap.storage, snap.fifo_head)

    def device_snapshot(self) -> "DeviceCacheSnapshot":
        """Device-to-device snapshot for per-epoch restoration (no host copies)."""
        return DeviceCacheSnapshot(self)

    def persist(self, sink) -> None:
        snap = self.snapshot()
        sink.write(SNAPSHOT_MAGIC)
        sink.write(struct.pack("<IBQId", SNAPSHOT_VERSION, _POLICY_CODE[snap.policy], snap.capacity, snap.dim, snap.lam))
        sink.write(snap.keys.astype("<i8").tobytes())
        sink.write(snap.scores.astype("<i8").tobytes())
        sink.write(struct.pack("<Q", snap.fifo_head))
        sink.write(np.ascontiguousarray(snap.storage, dtype="<f4").tobytes())

    def stats(self) -> dict:
        h, m, e = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        check(load().gf_cache_stats(self._h, ctypes.byref(h), ctypes.byref(m), ctypes.byref(e)))
        total = h.value + m.value
        return {"hits": int(h.value), "misses": int(m.value), "hit_rate": h.value / total if total else 0.0,
                "evictions": int(e.value)}

    def reset_stats(self) -> None:
        check(load().gf_cache_reset_stats(self._h))


class DeviceCacheSnapshot:
    def __init__(self, cache: VectorCache):
        h = ctypes.c_void_p()
        check(load().gf_cache_snapshot(cache.handle, ctypes.byref(h), stream_ptr(device=cache.device)))
        self._h = h
        self.shape = (cache.policy, cache.capacity, cache.dim)

    def restore_into(self, cache: VectorCache) -> None:
        if self.shape != (cache.policy, cache.capacity, cache.dim):
            raise SnapshotMismatchError("snapshot shape does not match the cache")
        check(load().gf_cache_restore(cache.handle, self._h, stream_ptr(device=cache.device)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                load().gf_cache_snapshot_free(h)
            except Exception:
                pass
            self._h = None


def load_cache(source, device=None) -> VectorCache:
    """cache.py:236-273: parse a TGCS blob into a device cache."""
    data = source.read() if hasattr(source, "read") else bytes(source)
    if data[:4] != SNAPSHOT_MAGIC:
        raise SnapshotFormatError("bad snapshot magic")
    header_fmt = "<IBQId"
    header_size = struct.calcsize(header_fmt)
    if len(data) < 4 + header_size:
        raise SnapshotFormatError("truncated snapshot header")
    version, policy_code, capacity, dim, lam = struct.unpack_from(header_fmt, data, 4)
    if version != SNAPSHOT_VERSION:
        raise SnapshotFormatError(f"unsupported snapshot version {version}")
    if policy_code not in _POLICY_NAME:
        raise SnapshotFormatError(f"unknown policy code {policy_code}")
    pos = 4 + header_size
    expected = pos + capacity * 8 * 2 + 8 + capacity * dim * 4
    if len(data) != expected:
        raise SnapshotFormatError("snapshot length mismatch")
    keys = np.frombuffer(data, dtype="<i8", count=capacity, offset=pos).copy()
    pos += capacity * 8
    scores = np.frombuffer(data, dtype="<i8", count=capacity, offset=pos).copy()
    pos += capacity * 8
    (fifo_head,) = struct.unpack_from("<Q", data, pos)
    pos += 8
    storage = np.frombuffer(data, dtype="<f4", count=capacity * dim, offset=pos).reshape(capacity, dim).copy()
    cache = VectorCache(_POLICY_NAME[policy_code], capacity, dim, lam, device=device)
    cache.restore(CacheSnapshot(cache.policy, capacity, dim, lam, keys, scores, int(fifo_head), storage))
    return cache
