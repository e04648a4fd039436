"""ctypes binding of libgfb200.so (the C ABI declared in include/gfb200.h).

The library is built in-tree (``python __graft_entry__.py`` or
``make -C paper_2311_17410_b200/csrc``).  There is no fallback: if the shared
object is missing or a call fails, the error propagates.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GF_LIB_PATH") or os.path.join(HERE, "libgfb200.so")  # override for A/B builds

GF_OK, GF_EINVAL, GF_ENOTFOUND, GF_ENOMEM, GF_ECUDA, GF_ERANGE, GF_EFORMAT = range(7)
POLICY_CODE = {"recent": 0, "uniform": 1, "time_window": 2}  # wire.py:27
CACHE_CODE = {"lru": 0, "lfu": 1, "fifo": 2}  # cache.py:27
SIZING_CODE = {"adaptive": 0, "fixed": 1, "batch": 2}

c_i64 = ctypes.c_int64
c_u64 = ctypes.c_uint64
c_int = ctypes.c_int
c_vp = ctypes.c_void_p
P_i64 = ctypes.POINTER(ctypes.c_int64)
P_u8 = ctypes.POINTER(ctypes.c_uint8)
P_f32 = ctypes.POINTER(ctypes.c_float)


class GraphInfo(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in (
        "num_nodes", "num_block_handles", "live_blocks", "slots_allocated", "next_edge_id",
        "total_edges_inserted", "any_deleted", "directed", "tau", "sizing_kind", "sizing_param", "device_bytes")]


# name -> (restype, argtypes)
_SIGS = {
    "gf_last_error": (ctypes.c_char_p, []),
    "gf_version": (ctypes.c_char_p, []),
    "gf_launch_count": (c_u64, []),
    "gf_profile_enable": (None, [c_int]),
    "gf_profile_summary": (c_int, [ctypes.c_char_p, c_i64]),
    "gf_hop_seed": (c_u64, [c_u64, c_u64]),
    "gf_child_key": (c_u64, [c_u64, c_u64]),
    "gf_graph_create": (c_int, [c_int, c_i64, c_int, c_i64, c_int, ctypes.POINTER(c_vp)]),
    "gf_graph_destroy": (c_int, [c_vp]),
    "gf_graph_reserve": (c_int, [c_vp, c_i64, c_i64, c_i64, c_vp]),
    "gf_graph_add_edges": (c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, P_i64, c_vp]),
    "gf_graph_delete_edges": (c_int, [c_vp, c_vp, c_i64, P_i64, c_vp]),
    "gf_graph_delete_node": (c_int, [c_vp, c_i64, ctypes.POINTER(c_int), c_vp]),
    "gf_graph_get_info": (c_int, [c_vp, ctypes.POINTER(GraphInfo)]),
    "gf_graph_offload_before": (c_int, [c_vp, c_i64, P_u8, c_i64, P_i64, P_i64, c_int, c_vp]),
    "gf_graph_export_nodes": (c_int, [c_vp, P_i64, P_i64, P_i64, P_i64, P_u8, c_vp]),
    "gf_graph_export_blocks": (c_int, [c_vp, P_i64, P_i64, P_i64, P_i64, P_i64, P_i64, c_vp]),
    "gf_graph_export_slots": (c_int, [c_vp, c_i64, c_i64, P_i64, P_i64, P_i64, P_i64, P_u8, c_vp]),
    "gf_sample_layer": (c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_int, c_i64, c_u64, c_vp, c_u64, c_vp, c_vp,
                                c_vp, c_vp, c_vp, c_i64, P_i64, c_vp]),
    "gf_sample_khop": (c_int, [c_vp, c_vp, c_vp, c_i64, P_i64, c_int, c_int, c_i64, c_u64, c_u64,
                               ctypes.POINTER(c_vp), ctypes.POINTER(c_vp), ctypes.POINTER(c_vp), ctypes.POINTER(c_vp),
                               P_i64, P_i64, c_vp]),
    "gf_cache_create": (c_int, [c_int, c_i64, c_i64, ctypes.c_double, c_int, ctypes.POINTER(c_vp)]),
    "gf_cache_destroy": (c_int, [c_vp]),
    "gf_cache_fetch": (c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, P_i64, c_vp]),
    "gf_cache_insert": (c_int, [c_vp, c_vp, c_i64, c_vp, P_i64, c_vp]),
    "gf_cache_stats": (c_int, [c_vp, P_i64, P_i64, P_i64]),
    "gf_cache_reset_stats": (c_int, [c_vp]),
    "gf_cache_get_state": (c_int, [c_vp, P_i64, P_i64, P_f32, P_i64, c_vp]),
    "gf_cache_set_state": (c_int, [c_vp, P_i64, P_i64, P_f32, c_i64, c_vp]),
    "gf_cache_snapshot": (c_int, [c_vp, ctypes.POINTER(c_vp), c_vp]),
    "gf_cache_restore": (c_int, [c_vp, c_vp, c_vp]),
    "gf_cache_snapshot_free": (c_int, [c_vp]),
    "gf_ftable_create": (c_int, [c_int, c_i64, c_int, ctypes.POINTER(c_vp)]),
    "gf_ftable_destroy": (c_int, [c_vp]),
    "gf_ftable_put": (c_int, [c_vp, c_vp, c_i64, c_vp, c_vp]),
    "gf_ftable_get": (c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "gf_ftable_size": (c_int, [c_vp, P_i64]),
    "gf_ftable_ids": (c_int, [c_vp, c_vp, c_i64, P_i64, c_vp]),
    "gf_fetch_features": (c_int, [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, P_i64, P_i64, c_vp]),
    "gf_gather_rows": (c_int, [c_vp, c_i64, c_vp, c_i64, c_i64, c_vp, c_vp]),
    "gf_bucket_by_owner": (c_int, [c_vp, c_i64, c_int, c_vp, c_vp, P_i64, c_vp]),
    "gf_csr_merge": (c_int, [c_vp, c_vp, c_i64, c_int, ctypes.POINTER(c_vp), c_vp, ctypes.POINTER(c_vp), P_i64, c_vp]),
    "gf_scatter_rows": (c_int, [c_vp, c_i64, c_vp, c_i64, c_i64, c_vp, c_i64, c_vp]),
}

EXPORTED = tuple(_SIGS)

_lib = None


class GFError(RuntimeError):
    pass


def load():
    """Load libgfb200.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python __graft_entry__.py` "
                              "(make -C paper_2311_17410_b200/csrc)")
        lib = ctypes.CDLL(LIB_PATH)
        ab = os.environ.get("GF_LIB_AB") == "1"  # A/B against an older build: tolerate missing entry points
        for name, (res, args) in _SIGS.items():
            if ab and not hasattr(lib, name):
                continue
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(status: int, value_error=ValueError, not_found=KeyError) -> None:
    if status == GF_OK:
        return
    msg = load().gf_last_error().decode(errors="replace")
    if status == GF_EINVAL:
        raise value_error(msg)
    if status == GF_ENOTFOUND:
        raise not_found(msg)
    if status == GF_ENOMEM:
        raise MemoryError(msg)
    raise GFError(f"gfb200 status {status}: {msg}")


def ptr(t) -> int | None:
    """Device (or host numpy) data pointer, or None."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def np_ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(ctypes.POINTER(ctype))


def stream_ptr(stream=None, device=None) -> int:
    """Raw cudaStream_t of ``stream`` or of the current stream (of ``device``, default: current)."""
    import torch

    if stream is not None:
        return stream.cuda_stream
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:  # fast path: no Stream object construction
        idx = torch.cuda.current_device() if device is None else (device.index if device.index is not None
                                                                   else torch.cuda.current_device())
        return raw(idx)
    return torch.cuda.current_stream(device).cuda_stream


def launch_count() -> int:
    return int(load().gf_launch_count())


def profile_enable(on: bool) -> None:
    load().gf_profile_enable(1 if on else 0)


def profile_summary() -> dict[str, tuple[int, float]]:
    """{kernel name: (launches, total ms)} from CUDA events around every library launch."""
    buf = ctypes.create_string_buffer(1 << 16)
    check(load().gf_profile_summary(buf, len(buf)))
    out = {}
    for line in buf.value.decode().splitlines():
        name, cnt, ms = line.split("\t")
        out[name] = (int(cnt), float(ms))
    return out
