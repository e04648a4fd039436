"""Probe: how much of the uniform hop-1 pick traffic is line reuse that a node-grouped processing order
could capture?  (GDELT bench shape; run on a B200 under gpurun.)

Builds the bench graph, samples 2-hop uniform [10, 10] from the bench roots, maps every hop-1 pick to its
node-major list position (a stand-in for its slot: blocks are contiguous runs of a node's list), and
times a 32-byte-record gather over a 191M-record array in four orders: the output order the sampler
uses today, grouped by the query's node (stable), fully sorted, and shuffled.  Also counts distinct
128 B lines and times scattered (partial-line) vs contiguous output writes.
"""

from __future__ import annotations

import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2311_17410_b200 as gf  # noqa: E402


def timeit(fn, reps=3):
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    best = 1e9
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def main():
    dev = torch.device("cuda:0")
    cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "gdelt"]
    src, dst, ts = bench.make_stream(cfg, dev)
    g, _ = bench.build_graph(cfg, src, dst, ts, 1, 0, dev)
    roots, rts = bench.roots_for_rank(src, dst, ts, cfg["roots"], 0)
    fan = cfg.get("fanouts", [10, 10])
    s = gf.sample_khop_device(g, roots, rts, fan, gf.SamplingPolicy("uniform"), seed=0, root_key_base=0)
    lay = s.layers[-1]
    Q = lay.source_nodes.numel()
    S = lay.edge_ids.numel()
    counts = lay.offsets[1:] - lay.offsets[:-1]
    print(f"hop-1 queries {Q}, picks {S}")
    # node-major list position of every edge (directed: stored at src, in eid order)
    E = src.numel()
    order = torch.sort(src, stable=True).indices
    pos = torch.empty(E, dtype=torch.int64, device=dev)
    pos[order] = torch.arange(E, device=dev)
    del order
    idx = pos[lay.edge_ids]
    del pos
    torch.cuda.synchronize()
    lines = idx // 4
    dl = torch.unique(lines).numel()
    print(f"distinct 128B lines {dl} ({dl / S:.3f} per pick)")
    qnode = torch.repeat_interleave(lay.source_nodes, counts)
    perm_node = torch.sort(qnode, stable=True).indices
    idx_node = idx[perm_node]
    idx_sorted = torch.sort(idx).values
    idx_shuf = idx[torch.randperm(S, device=dev)]
    import ctypes
    lib = ctypes.CDLL(os.path.join(ROOT, "scripts", "locality_probe.so"))
    lib.probe_gather.restype = ctypes.c_float
    lib.probe_gather.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int64] + [ctypes.c_void_p] * 3 + [ctypes.c_int]
    rec = torch.zeros(E, 4, dtype=torch.int64, device=dev)
    outs = [torch.empty(S, dtype=torch.int64, device=dev) for _ in range(3)]
    P = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
    for name, ix, pm in (("output order", idx, None), ("node-grouped, contiguous stores", idx_node, None),
                         ("node-grouped, stores in output order", idx_node, perm_node), ("sorted", idx_sorted, None),
                         ("shuffled", idx_shuf, None)):
        torch.cuda.synchronize()
        ms = lib.probe_gather(P(rec), P(ix), P(pm), S, *[P(o) for o in outs], 3)
        print(f"gather {name:38s} {ms:.3f} ms  {S / ms / 1e6:.1f} G records/s")
    # per-node stats: queries per node and list length
    deg = torch.bincount(src, minlength=cfg["nodes"])
    qn = torch.bincount(lay.source_nodes, minlength=cfg["nodes"])
    top = torch.topk(deg, 5)
    print("top degrees", top.values.tolist(), "their hop-1 queries", qn[top.indices].tolist())


if __name__ == "__main__":
    main()
