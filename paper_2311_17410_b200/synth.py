"""Seeded synthetic edge streams (input generator for tests and bench.py).

``generate_synthetic_arrays`` restates the reference generator
(/root/reference/pkg/src/ctdg/synth.py:15-53) with the identical numpy calls
in the identical order, but returns int64 columns instead of a list of
Python tuples (the only non-vectorised part of the reference, synth.py:53).
Array-identical to the reference (tests/test_synth.py pins it against the
digests in tests/golden/misc.json).

``generate_synthetic_device`` draws the same law on the GPU with torch
(inverse-CDF of the rank weights, uniform self-loop resampling, sorted
uniform integer timestamps).  It is NOT bit-identical to numpy's PCG64
stream; bench.py uses it for the 191M-edge GDELT shape, where the numpy
generator alone takes about a minute of host time.
"""

from __future__ import annotations

import numpy as np


def _weights(nodes: int, exponent: float) -> np.ndarray:
    # synth.py:32-34
    w = (np.arange(1, nodes + 1, dtype=np.float64)) ** (-1.0 / (exponent - 1.0))
    return w / w.sum()


def generate_synthetic_arrays(nodes: int, edges: int, skew: float = 2.2, time_span: int = 1_000_000,
                              seed: int = 0, src_skew: float | None = None):
    """Returns (src, dst, ts) int64 arrays; same stream as ctdg.generate_synthetic."""
    if nodes < 1 or edges < 1:
        raise ValueError("need at least one node and one edge")
    if skew <= 1.0:
        raise ValueError("skew must exceed 1 (power-law tail exponent)")
    if nodes == 1:
        z = np.zeros(0, dtype=np.int64)
        return z, z.copy(), z.copy()
    rng = np.random.default_rng(seed)
    dst = rng.choice(nodes, size=edges, p=_weights(nodes, skew))
    if src_skew is None:
        src = rng.integers(0, nodes, size=edges)
    else:
        src = rng.choice(nodes, size=edges, p=_weights(nodes, src_skew))
    loops = np.flatnonzero(src == dst)
    while len(loops):
        src[loops] = rng.integers(0, nodes, size=len(loops))
        loops = loops[src[loops] == dst[loops]]
    ts = np.sort(rng.integers(0, time_span, size=edges))
    return src.astype(np.int64), dst.astype(np.int64), ts.astype(np.int64)


def generate_synthetic_device(nodes: int, edges: int, skew: float = 2.2, time_span: int = 1_000_000,
                              seed: int = 0, src_skew: float | None = None, device="cuda"):
    """Same law as generate_synthetic, drawn on the GPU (torch tensors)."""
    import torch

    gen = torch.Generator(device=device)
    gen.manual_seed(seed)

    def draw(exponent):
        w = torch.arange(1, nodes + 1, dtype=torch.float64, device=device) ** (-1.0 / (exponent - 1.0))
        cdf = torch.cumsum(w, 0)
        cdf = cdf / cdf[-1]
        u = torch.rand(edges, dtype=torch.float64, device=device, generator=gen)
        return torch.searchsorted(cdf, u, right=True).clamp_(max=nodes - 1)

    dst = draw(skew)
    if src_skew is None:
        src = torch.randint(0, nodes, (edges,), device=device, generator=gen)
    else:
        src = draw(src_skew)
    loops = torch.nonzero(src == dst).flatten()
    while loops.numel():
        src[loops] = torch.randint(0, nodes, (loops.numel(),), device=device, generator=gen)
        loops = loops[src[loops] == dst[loops]]
    ts = torch.sort(torch.randint(0, time_span, (edges,), device=device, generator=gen)).values
    return src.to(torch.int64), dst.to(torch.int64), ts.to(torch.int64)


def generate_synthetic(nodes: int, edges: int, skew: float = 2.2, time_span: int = 1_000_000, seed: int = 0,
                       src_skew: float | None = None) -> list[tuple[int, int, int]]:
    """synth.py:15-53 signature and return type: the stream as (src, dst, ts) tuples."""
    s, d, t = generate_synthetic_arrays(nodes, edges, skew, time_span, seed, src_skew)
    return list(zip(s.tolist(), d.tolist(), t.tolist()))
