"""Device-side halves of the multi-GPU exchanges (libgfb200 gf_part.cu).

The reference routes each request to the machine that owns it and merges the answers back in
request order (cluster.py:242-292 for sampling, cluster.py:296-325 for features).  Around every
all-to-all these three calls do the data movement on the GPU:

* ``bucket_by_owner``  stable counting sort of keys by owner = key mod P -> send order + counts
* ``csr_merge``        owners' per-query counts + flat edge arrays -> request-order CSR layer
* ``scatter_rows``     owners' feature rows -> request order

The only host values are the per-owner counts that the all-to-all needs for its split sizes.
"""

from __future__ import annotations

import ctypes

from ._lib import check, load, ptr, stream_ptr

_I64 = ctypes.c_int64


def bucket_by_owner(keys, nparts: int, want_keys: bool = True, stream=None):
    """(perm, keys in send order or None, per-owner counts) for a CUDA int64 tensor of keys."""
    import torch

    k = keys.to(torch.int64).contiguous()
    n = int(k.numel())
    perm = torch.empty(n, dtype=torch.int64, device=k.device)
    ks = torch.empty(n, dtype=torch.int64, device=k.device) if want_keys else None
    counts = (_I64 * nparts)()
    check(load().gf_bucket_by_owner(ptr(k), n, int(nparts), ptr(perm), ptr(ks), counts, stream_ptr(stream, k.device)))
    return perm, ks, [int(c) for c in counts]


def csr_merge(perm, cnt_sorted, arrays, stream=None):
    """Request-order (offsets, arrays) from send-order per-query counts and edge arrays."""
    import torch

    n = int(perm.numel())
    dev = perm.device
    offsets = torch.empty(n + 1, dtype=torch.int64, device=dev)
    ins = [a.to(torch.int64).contiguous() for a in arrays]
    outs = [torch.empty_like(a) for a in ins]
    VP = ctypes.c_void_p * max(1, len(ins))
    total = _I64(0)
    check(load().gf_csr_merge(ptr(perm), ptr(cnt_sorted.contiguous()), n, len(ins), VP(*[ptr(a) for a in ins]),
                              ptr(offsets), VP(*[ptr(a) for a in outs]), ctypes.byref(total), stream_ptr(stream, dev)))
    return offsets, outs, int(total.value)


def scatter_rows(rows, dest, n_out: int, out=None, stream=None):
    """out[dest[i], :] = rows[i, :] for float32 rows [n, dim] (out zero-initialised when not given)."""
    import torch

    r = rows.to(torch.float32).contiguous()
    dim = int(r.shape[1]) if r.dim() == 2 else 0
    if out is None:
        out = torch.zeros((n_out, dim), dtype=torch.float32, device=r.device)
    d = dest.to(torch.int64).contiguous()
    check(load().gf_scatter_rows(ptr(r), dim, ptr(d), int(d.numel()), dim, ptr(out), int(out.shape[1]),
                                 stream_ptr(stream, r.device)))
    return out
