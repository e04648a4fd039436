"""Temporal k-hop sampling on the GPU behind the reference's sampling API.

Mirrors /root/reference/pkg/src/ctdg/sampling.py: ``SamplingPolicy``,
``SampleRequest``, ``SampleLayer``, ``LayeredSample``, ``sample_layer``,
``sample_khop``, ``random_walk``, ``hop_seed``; plus the paper-level
``TemporalSampler(graph, fanouts, strategy).sample(roots, ts)``.

Host inputs (lists / numpy) give numpy outputs, like the reference; CUDA
tensor inputs give CUDA tensor outputs with no host round trip except the
per-hop sample counts.

Randomness (uniform / time_window): Philox4x32-10 keyed by the hop seed,
counter = (query key, draw index); Floyd's algorithm picks k distinct
candidates.  sample_layer's query key is ``key_base + i``; sample_khop keys
root i with ``root_key_base + i`` and the j-th edge sampled by a query with
key K gets child key mix(K, j), so a root batch split across GPUs reproduces
the single-GPU sample exactly.  The reference instead seeds numpy PCG64 per
(seed, node, window, occurrence) (sampling.py:140-142); the two streams
differ, their distributions match (tests/test_gpu_sampling.py).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import check, load, ptr, stream_ptr
from .storage import TS_MIN, DynamicGraph

POLICY_KINDS = ("recent", "uniform", "time_window")  # sampling.py:28
_U64 = 0xFFFFFFFFFFFFFFFF


@dataclass(frozen=True)
class SamplingPolicy:
    kind: str
    delta: int = 0

    def __post_init__(self):
        if self.kind not in POLICY_KINDS:
            raise ValueError(f"unknown policy kind {self.kind!r}")
        if self.kind == "time_window" and self.delta <= 0:
            raise ValueError("time_window policy requires delta > 0")

    @classmethod
    def recent(cls) -> "SamplingPolicy":
        return cls("recent")

    @classmethod
    def uniform(cls) -> "SamplingPolicy":
        return cls("uniform")

    @classmethod
    def time_window(cls, delta: int) -> "SamplingPolicy":
        return cls("time_window", delta)


@dataclass
class SampleRequest:
    targets: list[int]
    timestamps: list[int]
    fanouts: list[int]
    policy: SamplingPolicy
    seed: int = 0

    def validate(self) -> None:
        if len(self.targets) != len(self.timestamps):
            raise ValueError("targets and timestamps must have equal length")
        if any(f < 1 for f in self.fanouts):
            raise ValueError("every fanout must be >= 1")


def _np(x) -> np.ndarray:
    if isinstance(x, np.ndarray):
        return x
    if hasattr(x, "detach"):
        return x.detach().cpu().numpy()
    return np.asarray(x)


@dataclass
class SampleLayer:
    """One hop in CSR form (sampling.py:71-106); arrays are numpy or CUDA tensors."""

    source_nodes: object
    source_times: object
    offsets: object
    neighbors: object
    edge_ids: object
    timestamps: object

    _FIELDS = ("source_nodes", "source_times", "offsets", "neighbors", "edge_ids", "timestamps")

    def __eq__(self, other) -> bool:
        if not isinstance(other, SampleLayer) and not hasattr(other, "offsets"):
            return NotImplemented
        return all(np.array_equal(_np(getattr(self, f)), _np(getattr(other, f))) for f in self._FIELDS)

    def slice_of(self, i: int) -> slice:
        return slice(int(self.offsets[i]), int(self.offsets[i + 1]))

    def to_host(self) -> "SampleLayer":
        return SampleLayer(*[_np(getattr(self, f)) for f in self._FIELDS])

    def to_json_dict(self) -> dict:
        return {f: _np(getattr(self, f)).tolist() for f in ("offsets", "neighbors", "edge_ids", "timestamps")}


@dataclass
class LayeredSample:
    layers: list[SampleLayer] = field(default_factory=list)

    def __eq__(self, other) -> bool:
        if not hasattr(other, "layers"):
            return NotImplemented
        return len(self.layers) == len(other.layers) and all(a == b for a, b in zip(self.layers, other.layers))

    def to_host(self) -> "LayeredSample":
        return LayeredSample([lay.to_host() for lay in self.layers])

    def to_json_dict(self) -> dict:
        return {"layers": [layer.to_json_dict() for layer in self.layers]}

    def sampled_nodes(self) -> set[int]:
        out: set[int] = set()
        for layer in self.layers:
            out.update(_np(layer.source_nodes).tolist())
            out.update(_np(layer.neighbors).tolist())
        return out

    def sampled_edges(self) -> set[int]:
        out: set[int] = set()
        for layer in self.layers:
            out.update(_np(layer.edge_ids).tolist())
        return out

    def num_sampled_edges(self) -> int:
        return sum(int(layer.neighbors.shape[0]) for layer in self.layers)


def hop_seed(seed: int, hop: int) -> int:
    """sampling.py:135-137 (numpy SeedSequence, restated natively in libgfb200)."""
    return int(load().gf_hop_seed(seed & _U64, hop & _U64))


def _policy_args(policy: SamplingPolicy):
    return _lib.POLICY_CODE[policy.kind], int(policy.delta)


def _to_dev(x, device):
    import torch

    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=torch.int64).contiguous(), True
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.int64))).to(device), False


def _layer_device(graph: DynamicGraph, src, t_start, t_end, fanout: int, policy: SamplingPolicy, seed: int,
                  keys=None, key_base: int = 0, want_keys: bool = False, stream=None):
    """One gf_sample_layer call on device tensors; retries on GF_ERANGE."""
    import torch

    n = int(src.numel())
    code, delta = _policy_args(policy)
    offsets = torch.empty(n + 1, dtype=torch.int64, device=graph.device)
    cap = max(1, min(n * min(int(fanout), 64), 1 << 28))
    lib = load()
    while True:
        nbr = torch.empty(cap, dtype=torch.int64, device=graph.device)
        eid = torch.empty(cap, dtype=torch.int64, device=graph.device)
        ts = torch.empty(cap, dtype=torch.int64, device=graph.device)
        okeys = torch.empty(cap, dtype=torch.int64, device=graph.device) if want_keys else None
        total = ctypes.c_int64(0)
        st = lib.gf_sample_layer(graph.handle, ptr(src), ptr(t_start), ptr(t_end), n, int(fanout), code, delta,
                                 seed & _U64, ptr(keys), key_base & _U64, ptr(offsets), ptr(nbr), ptr(eid), ptr(ts),
                                 ptr(okeys), cap, ctypes.byref(total), stream_ptr(stream, graph.device))
        if st == _lib.GF_ERANGE:
            cap = int(total.value)
            continue
        check(st)
        t = int(total.value)
        return offsets, nbr[:t], eid[:t], ts[:t], (okeys[:t] if want_keys else None)


def sample_layer(graph: DynamicGraph, sources, t_starts, t_ends, fanout: int, policy: SamplingPolicy, seed: int,
                 workers: int = 1) -> SampleLayer:
    """sampling.py:219-273.  ``workers`` is accepted for API parity (the GPU runs every query in parallel)."""
    import torch

    s, on_dev = _to_dev(sources, graph.device)
    t0, _ = _to_dev(t_starts, graph.device)
    t1, _ = _to_dev(t_ends, graph.device)
    if not (s.numel() == t0.numel() == t1.numel()):
        raise ValueError("sources, t_starts and t_ends must have equal length")
    if fanout < 1:
        raise ValueError("fanout must be >= 1")
    offs, nbr, eid, ts, _ = _layer_device(graph, s, t0, t1, fanout, policy, seed)
    lay = SampleLayer(s.clone(), t1.clone(), offs, nbr, eid, ts)
    return lay if on_dev else lay.to_host()


def sample_khop(graph: DynamicGraph, request: SampleRequest, workers: int = 1, root_key_base: int = 0,
                stream=None) -> LayeredSample:
    """sampling.py:276-299: hop l+1 queries each sampled neighbour at the edge's timestamp."""
    import torch

    request.validate()
    roots, on_dev = _to_dev(request.targets, graph.device)
    tends, _ = _to_dev(request.timestamps, graph.device)
    out = sample_khop_device(graph, roots, tends, list(request.fanouts), request.policy, request.seed, root_key_base,
                             stream)
    return out if on_dev else out.to_host()


_ARR_TYPES: dict[int, tuple] = {}


def _arr_types(n: int):
    """ctypes array types for n hops (cached: building them costs more than the C call's setup)."""
    t = _ARR_TYPES.get(n)
    if t is None:
        t = _ARR_TYPES[n] = (ctypes.c_void_p * n, ctypes.c_int64 * n)
    return t


def sample_khop_device(graph: DynamicGraph, roots, tends, fanouts, policy: SamplingPolicy, seed: int = 0,
                       root_key_base: int = 0, stream=None) -> LayeredSample:
    """Fused multi-hop driver (gf_sample_khop) on CUDA tensors; one host sync per hop."""
    import torch

    fanouts = [int(f) for f in fanouts]
    if any(f < 1 for f in fanouts):
        raise ValueError("every fanout must be >= 1")
    if roots.numel() != tends.numel():
        raise ValueError("targets and timestamps must have equal length")
    n_hops = len(fanouts)
    if n_hops == 0:
        return LayeredSample()
    caps, n = [], int(roots.numel())
    for f in fanouts:
        n = n * f
        caps.append(n)
    if max(caps) > (1 << 30):
        return _khop_layerwise(graph, roots, tends, fanouts, policy, seed, root_key_base, stream)
    dev = graph.device
    nq = [int(roots.numel())] + caps[:-1]
    # one allocation for every output of the call, carved into disjoint views
    sizes = [max(c, 1) for c in caps] * 3 + [q + 1 for q in nq]
    flat = torch.empty(sum(sizes), dtype=torch.int64, device=dev)
    parts = list(torch.split(flat, sizes))
    nbr, eid, tss, offs = (parts[i * n_hops:(i + 1) * n_hops] for i in range(4))
    VP, I64 = _arr_types(n_hops)
    totals = I64()
    code, delta = _policy_args(policy)
    st = load().gf_sample_khop(graph.handle, ptr(roots), ptr(tends), int(roots.numel()), I64(*fanouts), n_hops, code,
                               delta, seed & _U64, root_key_base & _U64, VP(*[ptr(o) for o in offs]),
                               VP(*[ptr(x) for x in nbr]), VP(*[ptr(x) for x in eid]), VP(*[ptr(x) for x in tss]),
                               I64(*caps), totals, stream_ptr(stream, graph.device))
    check(st)
    layers = []
    src, te = roots, tends
    for h in range(n_hops):
        t = int(totals[h])
        nq_h = int(src.numel())
        layers.append(SampleLayer(src, te, offs[h][: nq_h + 1], nbr[h][:t], eid[h][:t], tss[h][:t]))
        src, te = nbr[h][:t], tss[h][:t]
    return LayeredSample(layers)


def _khop_layerwise(graph, roots, tends, fanouts, policy, seed, root_key_base, stream):
    """Hop-by-hop driver for fanout products too large to pre-size (e.g. fanout 1e9)."""
    import torch

    layers = []
    src, te = roots, tends
    keys = None
    for h, f in enumerate(fanouts):
        want = policy.kind != "recent" and h + 1 < len(fanouts)
        offs, nbr, eid, ts, okeys = _layer_device(graph, src, None, te, f, policy, hop_seed(seed, h), keys,
                                                  root_key_base, want, stream)
        layers.append(SampleLayer(src, te, offs, nbr, eid, ts))
        src, te, keys = nbr, ts, okeys
    return LayeredSample(layers)


def random_walk(graph: DynamicGraph, start: int, t: int, length: int, policy: SamplingPolicy,
                seed: int = 0) -> list[tuple[int, int]]:
    """sampling.py:302-324."""
    if length < 1:
        raise ValueError("length must be >= 1")
    sample = sample_khop(graph, SampleRequest([start], [t], [1] * length, policy, seed))
    walk: list[tuple[int, int]] = []
    for layer in sample.layers:
        if len(layer.neighbors) == 0:
            break
        walk.append((int(layer.neighbors[0]), int(layer.timestamps[0])))
    return walk


class TemporalSampler:
    """Paper-level sampler: ``TemporalSampler(graph, fanouts, strategy).sample(roots, ts)``.

    Equivalent to sample_khop(graph, SampleRequest(roots, ts, fanouts,
    SamplingPolicy(strategy, delta), seed)).  Returns device tensors when
    given device tensors; ``root_key_base`` positions this root batch in a
    larger (multi-GPU) batch.
    """

    def __init__(self, graph: DynamicGraph, fanouts, strategy: str = "recent", delta: int = 0, seed: int = 0):
        self.graph = graph
        self.fanouts = [int(f) for f in fanouts]
        if any(f < 1 for f in self.fanouts):
            raise ValueError("every fanout must be >= 1")
        self.policy = SamplingPolicy(strategy, delta)
        self.seed = seed

    def sample(self, roots, ts, fanouts=None, strategy: str | None = None, seed: int | None = None,
               root_key_base: int = 0, stream=None, delta: int | None = None) -> LayeredSample:
        """``sample(roots, ts)`` with the constructor's settings, or the north-star form
        ``sample(roots, ts, fanouts, strategy)`` overriding them for this call."""
        fo = self.fanouts if fanouts is None else [int(f) for f in fanouts]
        pol = self.policy if strategy is None else SamplingPolicy(strategy, self.policy.delta if delta is None else delta)
        req = SampleRequest(roots, ts, fo, pol, self.seed if seed is None else seed)
        return sample_khop(self.graph, req, root_key_base=root_key_base, stream=stream)
