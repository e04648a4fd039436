"""Feature-cache and feature-table restatements (CPU ORACLE -- test infrastructure only).

Restates the reference's ``VectorCache`` (cache.py:55-233) and the
``NodeFeatureTable``/``EdgeFeatureTable`` lookups (features.py:27-120) in
numpy so the CUDA cache can be checked call-by-call.  Pinned against the
reference's scalar LRU/LFU/FIFO oracles and fixtures (tests/test_oracle_golden.py).
"""

from __future__ import annotations

import numpy as np

EMPTY_KEY = -1  # cache.py:30
POLICIES = ("lru", "lfu", "fifo")  # cache.py:26


class CacheOracle:
    def __init__(self, policy: str, capacity: int, dim: int, lam: float = 0.2):
        # cache.py:56-74
        if policy not in POLICIES:
            raise ValueError(f"unknown cache policy {policy!r}")
        if capacity < 1:
            raise ValueError("capacity must be >= 1")
        if not 0.0 < lam <= 1.0:
            raise ValueError("lam must be in (0, 1]")
        self.policy, self.capacity, self.dim, self.lam = policy, capacity, dim, lam
        self.keys = np.full(capacity, EMPTY_KEY, dtype=np.int64)
        self.scores = np.zeros(capacity, dtype=np.int64)
        self.storage = np.zeros((capacity, dim), dtype=np.float32)
        self.fifo_head = 0
        self.slot_of: dict[int, int] = {}
        self.hits = self.misses = self.evictions = 0

    @property
    def max_update(self) -> int:  # cache.py:79-81
        return int(self.lam * self.capacity)

    def fetch(self, keys):
        """cache.py:85-121."""
        keys = np.asarray(keys, dtype=np.int64)
        values = np.zeros((len(keys), self.dim), dtype=np.float32)
        if len(keys) == 0:
            return values, np.zeros(0, bool), np.empty(0, np.int64)
        slots = np.array([self.slot_of.get(int(k), -1) for k in keys], dtype=np.int64)
        hit = slots >= 0
        values[hit] = self.storage[slots[hit]]
        occupied = self.keys != EMPTY_KEY
        if self.policy == "lru":
            self.scores[occupied] -= 1
            self.scores[np.unique(slots[hit])] = 0
        elif self.policy == "lfu":
            hs, cnt = np.unique(slots[hit], return_counts=True)
            self.scores[hs] += cnt
        miss_keys, seen = [], set()
        for k, h in zip(keys.tolist(), hit.tolist()):
            if not h and k not in seen:
                seen.add(k)
                miss_keys.append(k)
        self.hits += int(hit.sum())
        self.misses += int(len(keys) - hit.sum())
        return values, hit, np.array(miss_keys, dtype=np.int64)

    def insert_batch(self, keys, values) -> int:
        """cache.py:123-177."""
        keys = np.asarray(keys, dtype=np.int64)
        values = np.asarray(values, dtype=np.float32)
        if values.shape != (len(keys), self.dim):
            raise ValueError(f"values must be ({len(keys)}, {self.dim}), got {values.shape}")
        uniq, seen = [], set()
        for i, k in enumerate(keys.tolist()):
            if k in self.slot_of:
                raise ValueError(f"key {k} is already cached")
            if k not in seen:
                seen.add(k)
                uniq.append(i)
        admit = uniq[: self.max_update]
        if not admit:
            return 0
        if self.policy == "fifo":
            for i in admit:
                self._place(int(keys[i]), self.fifo_head, values[i], 0)
                self.fifo_head = (self.fifo_head + 1) % self.capacity
            return len(admit)
        new_score = 0 if self.policy == "lru" else 1
        free = np.flatnonzero(self.keys == EMPTY_KEY)
        n_free = min(len(free), len(admit))
        for j in range(n_free):
            self._place(int(keys[admit[j]]), int(free[j]), values[admit[j]], new_score)
        rest = admit[n_free:]
        if rest:
            occ = np.flatnonzero(self.keys != EMPTY_KEY)
            order = np.lexsort((occ, self.scores[occ]))
            for i, slot in zip(rest, occ[order[: len(rest)]]):
                self._place(int(keys[i]), int(slot), values[i], new_score)
        return len(admit)

    def _place(self, key, slot, row, score):  # cache.py:169-177
        old = int(self.keys[slot])
        if old != EMPTY_KEY:
            del self.slot_of[old]
            self.evictions += 1
        self.keys[slot] = key
        self.scores[slot] = score
        self.storage[slot] = row
        self.slot_of[key] = slot

    def stats(self) -> dict:  # cache.py:223-230
        tot = self.hits + self.misses
        return {"hits": self.hits, "misses": self.misses, "hit_rate": self.hits / tot if tot else 0.0,
                "evictions": self.evictions}


class NodeFeatureOracle:
    """features.py:27-61 (dict of rows; zeros + found=False for unknown ids)."""

    def __init__(self, dim: int):
        self.dim = dim
        self.rows: dict[int, np.ndarray] = {}

    def set_many(self, ids, rows):
        rows = np.asarray(rows, dtype=np.float32)
        for i, k in enumerate(np.asarray(ids).tolist()):
            self.rows[int(k)] = rows[i].copy()

    def get(self, ids):
        ids = np.asarray(ids, dtype=np.int64)
        out = np.zeros((len(ids), self.dim), np.float32)
        found = np.zeros(len(ids), bool)
        for i, k in enumerate(ids.tolist()):
            r = self.rows.get(k)
            if r is not None:
                out[i] = r
                found[i] = True
        return out, found


class EdgeFeatureOracle:
    """features.py:64-120 (sorted ids + searchsorted exact match)."""

    def __init__(self, dim: int):
        self.dim = dim
        self.ids = np.empty(0, np.int64)
        self.values = np.empty((0, dim), np.float32)

    def append(self, ids, rows):
        ids = np.asarray(ids, dtype=np.int64)
        rows = np.asarray(rows, dtype=np.float32)
        if rows.shape != (len(ids), self.dim):
            raise ValueError("shape mismatch")
        if len(ids) == 0:
            return
        if np.any(np.diff(ids) <= 0) or (len(self.ids) and ids[0] <= self.ids[-1]):
            raise ValueError("edge ids must be strictly increasing")
        self.ids = np.concatenate([self.ids, ids])
        self.values = np.concatenate([self.values, rows])

    def get(self, ids):
        ids = np.asarray(ids, dtype=np.int64)
        out = np.zeros((len(ids), self.dim), np.float32)
        found = np.zeros(len(ids), bool)
        if len(self.ids) == 0 or len(ids) == 0:
            return out, found
        pos = np.searchsorted(self.ids, ids)
        ok = pos < len(self.ids)
        hit = ok.copy()
        hit[ok] = self.ids[pos[ok]] == ids[ok]
        out[hit] = self.values[pos[hit]]
        found[hit] = True
        return out, found
