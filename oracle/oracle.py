"""ctypes wrapper over liboracle.so (CPU ORACLE -- test infrastructure only)."""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

TS_MIN = int(np.iinfo(np.int64).min)
_HERE = os.path.dirname(os.path.abspath(__file__))
lib_path = os.path.join(_HERE, "liboracle.so")

_POLICY = {"recent": 0, "uniform": 1, "time_window": 2}
_SIZING = {"adaptive": 0, "fixed": 1, "batch": 2}

_i64p = ctypes.POINTER(ctypes.c_int64)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_u32p = ctypes.POINTER(ctypes.c_uint32)


def build() -> str:
    """Compile liboracle.so in place (gcc)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return lib_path


def _load():
    if not os.path.exists(lib_path):
        build()
    lib = ctypes.CDLL(lib_path)
    lib.or_graph_create.restype = ctypes.c_void_p
    lib.or_graph_create.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int, ctypes.c_int64]
    lib.or_graph_destroy.argtypes = [ctypes.c_void_p]
    lib.or_add_edges.restype = ctypes.c_int64
    lib.or_add_edges.argtypes = [ctypes.c_void_p, _i64p, _i64p, _i64p, ctypes.c_int64, _i64p, _i64p]
    lib.or_delete_edges.restype = ctypes.c_int64
    lib.or_delete_edges.argtypes = [ctypes.c_void_p, _i64p, ctypes.c_int64]
    lib.or_delete_node.restype = ctypes.c_int
    lib.or_delete_node.argtypes = [ctypes.c_void_p, ctypes.c_int64]
    for name in ("or_num_nodes", "or_num_block_handles", "or_next_edge_id", "or_total_edges_inserted"):
        getattr(lib, name).restype = ctypes.c_int64
        getattr(lib, name).argtypes = [ctypes.c_void_p]
    lib.or_offload_before.restype = ctypes.c_int64
    lib.or_offload_before.argtypes = [ctypes.c_void_p, ctypes.c_int64, _u8p, ctypes.c_int64, _i64p]
    lib.or_export_nodes.argtypes = [ctypes.c_void_p, _i64p, _i64p, _i64p, _i64p, _u8p]
    lib.or_export_blocks.argtypes = [ctypes.c_void_p] + [_i64p] * 6
    lib.or_export_block_edges.restype = ctypes.c_int64
    lib.or_export_block_edges.argtypes = [ctypes.c_void_p, ctypes.c_int64, _i64p, _i64p, _i64p, _u8p]
    lib.or_sample_layer.restype = ctypes.c_int64
    lib.or_sample_layer.argtypes = [
        ctypes.c_void_p, _i64p, _i64p, _i64p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
        ctypes.c_int64, ctypes.c_uint64, _u64p, _i64p, _i64p, _i64p, _i64p, ctypes.c_int64,
        ctypes.c_int, ctypes.c_int,
    ]
    lib.or_hop_seed.restype = ctypes.c_uint64
    lib.or_hop_seed.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
    lib.or_child_key.restype = ctypes.c_uint64
    lib.or_child_key.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
    lib.or_philox4x32_10.argtypes = [_u32p, _u32p, _u32p]
    return lib


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = _load()
    return _lib


def _p(a, t=_i64p):
    return a.ctypes.data_as(t) if a is not None else None


def hop_seed(seed: int, hop: int) -> int:
    return int(lib().or_hop_seed(seed & 0xFFFFFFFFFFFFFFFF, hop))


def child_key(parent: int, j: int) -> int:
    return int(lib().or_child_key(parent & 0xFFFFFFFFFFFFFFFF, j))


def philox4x32_10(ctr, key) -> np.ndarray:
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().or_philox4x32_10(_p(c, _u32p), _p(k, _u32p), _p(out, _u32p))
    return out


class OracleGraph:
    """CPU restatement of ``ctdg.DynamicGraph`` (storage.py:303-621)."""

    def __init__(self, directed: bool = False, tau: int = 48, sizing: str = "adaptive", sizing_param: int = 0):
        if sizing == "adaptive" and tau < 1:
            raise ValueError(f"tau must be >= 1, got {tau}")
        self.directed = bool(directed)
        self.tau = tau
        self._h = lib().or_graph_create(int(directed), int(tau), _SIZING[sizing], int(sizing_param))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().or_graph_destroy(h)
            self._h = None

    # -- mutation ---------------------------------------------------------
    def add_edges(self, src, dst, ts, edge_ids=None) -> np.ndarray:
        src = np.ascontiguousarray(src, dtype=np.int64)
        dst = np.ascontiguousarray(dst, dtype=np.int64)
        ts = np.ascontiguousarray(ts, dtype=np.int64)
        if not (len(src) == len(dst) == len(ts)):
            raise ValueError("src, dst, ts must have equal length")
        eids = None if edge_ids is None else np.ascontiguousarray(edge_ids, dtype=np.int64)
        if eids is not None and len(eids) != len(src):
            raise ValueError("edge_ids must match batch length")
        out = np.empty(len(src), dtype=np.int64)
        rc = lib().or_add_edges(self._h, _p(src), _p(dst), _p(ts), len(src), _p(eids), _p(out))
        if rc < 0:
            raise ValueError("node ids must be non-negative")
        return out

    def delete_edges(self, edge_ids) -> int:
        e = np.ascontiguousarray(edge_ids, dtype=np.int64)
        return int(lib().or_delete_edges(self._h, _p(e), len(e)))

    def delete_node(self, node: int) -> bool:
        return bool(lib().or_delete_node(self._h, int(node)))

    def offload_before(self, cutoff: int):
        """storage.py:516-574: returns (TGOF blob bytes, edge records)."""
        blen = ctypes.c_int64(0)
        lib().or_offload_before(self._h, int(cutoff), None, 0, ctypes.byref(blen))
        buf = np.zeros(blen.value, dtype=np.uint8)
        n = lib().or_offload_before(self._h, int(cutoff), _p(buf, _u8p), len(buf), ctypes.byref(blen))
        return buf.tobytes(), int(n)

    # -- inspection -------------------------------------------------------
    @property
    def num_nodes(self) -> int:
        return int(lib().or_num_nodes(self._h))

    @property
    def num_block_handles(self) -> int:
        return int(lib().or_num_block_handles(self._h))

    @property
    def next_edge_id(self) -> int:
        return int(lib().or_next_edge_id(self._h))

    @property
    def total_edges_inserted(self) -> int:
        return int(lib().or_total_edges_inserted(self._h))

    def export_nodes(self) -> dict:
        n = self.num_nodes
        cols = {k: np.zeros(n, dtype=np.int64) for k in ("head", "tail", "num_blocks", "degree")}
        valid = np.zeros(n, dtype=np.uint8)
        lib().or_export_nodes(self._h, _p(cols["head"]), _p(cols["tail"]), _p(cols["num_blocks"]),
                              _p(cols["degree"]), _p(valid, _u8p))
        cols["node_valid"] = valid.astype(bool)
        return cols

    def export_blocks(self) -> dict:
        n = self.num_block_handles
        names = ("capacity", "size", "tmin", "tmax", "prev", "next")
        cols = {k: np.zeros(n, dtype=np.int64) for k in names}
        lib().or_export_blocks(self._h, *[_p(cols[k]) for k in names])
        return cols

    def block_edges(self, handle: int):
        cap = self.export_blocks()["size"][handle]
        nbr = np.zeros(cap, np.int64); eid = np.zeros(cap, np.int64); ts = np.zeros(cap, np.int64)
        valid = np.zeros(cap, np.uint8)
        lib().or_export_block_edges(self._h, int(handle), _p(nbr), _p(eid), _p(ts), _p(valid, _u8p))
        return nbr, eid, ts, valid.astype(bool)

    def blocks_of(self, node: int) -> list[int]:
        nodes = self.export_nodes()
        nxt = self.export_blocks()["next"]
        out, h = [], int(nodes["head"][node])
        while h != -1:
            out.append(h)
            h = int(nxt[h])
        return out

    # -- sampling ---------------------------------------------------------
    def sample_layer(self, sources, t_starts, t_ends, fanout: int, policy: str = "recent", delta: int = 0,
                     seed: int = 0, keys=None, threads: int = 1, faithful: bool = False):
        """Returns (offsets, neighbors, edge_ids, timestamps) as int64 arrays."""
        src = np.ascontiguousarray(sources, dtype=np.int64)
        t0 = np.ascontiguousarray(t_starts, dtype=np.int64)
        t1 = np.ascontiguousarray(t_ends, dtype=np.int64)
        if not (len(src) == len(t0) == len(t1)):
            raise ValueError("sources, t_starts and t_ends must have equal length")
        if fanout < 1:
            raise ValueError("fanout must be >= 1")
        n = len(src)
        k = None if keys is None else np.ascontiguousarray(keys, dtype=np.uint64)
        cap = int(min(n * min(fanout, 64), 1 << 26))
        while True:
            offs = np.zeros(n + 1, dtype=np.int64)
            nb = np.zeros(max(cap, 1), np.int64); eid = np.zeros(max(cap, 1), np.int64)
            ts = np.zeros(max(cap, 1), np.int64)
            tot = lib().or_sample_layer(self._h, _p(src), _p(t0), _p(t1), n, int(fanout), _POLICY[policy],
                                        int(delta), seed & 0xFFFFFFFFFFFFFFFF, _p(k, _u64p), _p(offs), _p(nb),
                                        _p(eid), _p(ts), cap, int(threads), int(faithful))
            if tot < 0:
                raise ValueError("bad sampling arguments")
            if tot <= cap:
                return offs, nb[:tot].copy(), eid[:tot].copy(), ts[:tot].copy()
            cap = int(tot)

    def sample_khop(self, roots, ts, fanouts, policy: str = "recent", delta: int = 0, seed: int = 0,
                    root_key_base: int = 0, threads: int = 1, faithful: bool = False):
        """sampling.py:276-299 with path-derived keys.  Returns a list of
        (source_nodes, source_times, offsets, neighbors, edge_ids, timestamps)."""
        roots = np.ascontiguousarray(roots, dtype=np.int64)
        tends = np.ascontiguousarray(ts, dtype=np.int64)
        if len(roots) != len(tends):
            raise ValueError("targets and timestamps must have equal length")
        if any(f < 1 for f in fanouts):
            raise ValueError("every fanout must be >= 1")
        keys = np.arange(len(roots), dtype=np.uint64) + np.uint64(root_key_base)
        layers = []
        for hop, f in enumerate(fanouts):
            offs, nb, eid, tts = self.sample_layer(roots, np.full(len(roots), TS_MIN, np.int64), tends, f, policy,
                                                   delta, hop_seed(seed, hop), keys, threads, faithful)
            layers.append((roots.copy(), tends.copy(), offs, nb, eid, tts))
            counts = np.diff(offs)
            parent = np.repeat(keys, counts)
            j = np.arange(len(nb), dtype=np.int64) - np.repeat(offs[:-1], counts)
            keys = _child_keys_vec(parent, j)
            roots, tends = nb, tts
        return layers


def _child_keys_vec(parent: np.ndarray, j: np.ndarray) -> np.ndarray:
    """Vectorised or_child_key (splitmix64 of parent ^ golden*(j+1))."""
    with np.errstate(over="ignore"):
        z = parent.astype(np.uint64) ^ (np.uint64(0x9E3779B97F4A7C15) * (j.astype(np.uint64) + np.uint64(1)))
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))
