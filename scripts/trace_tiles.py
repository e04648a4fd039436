"""Per-tile phase times of the fused sampler (A/B trace build: scripts/build_variant.sh trace -DGF_AB_TRACE=1).

    GF_LIB_PATH=scripts/lib_trace.so python scripts/trace_tiles.py

Runs hop 1 of the GDELT bench step alone (recent and uniform) with sample_layer and prints the mean
time from a tile's ticket to: publication of its counts, end of its selection, its output base
(look-back done), and the end of its gather/store; plus the launch span and tiles in flight.
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2311_17410_b200 as gf  # noqa: E402
from paper_2311_17410_b200 import _lib  # noqa: E402

lib = _lib.load()
lib.gf_ab_trace_dump.argtypes = [ctypes.c_void_p, ctypes.c_int]
name = sys.argv[1] if len(sys.argv) > 1 else "gdelt"
cfg = bench.CONFIGS[name]
fan = cfg.get("fanouts", [10, 10])
pols = cfg.get("policies", ("recent", "uniform"))
dev = torch.device("cuda", 0)
src, dst, ts = bench.make_stream(cfg, dev)
g, _ = bench.build_graph(cfg, src, dst, ts, 1, 0, dev)
roots, rts = bench.roots_for_rank(src, dst, ts, cfg["roots"], 0)
for pol, ft in (("recent", 128), ("uniform", 256)):
    if pol not in pols:
        continue
    p = gf.SamplingPolicy(pol)
    h0 = gf.sample_khop_device(g, roots, rts, [fan[0]], p, seed=0).layers[0]
    q, t = h0.neighbors.contiguous(), h0.timestamps.contiguous()
    t0 = torch.full_like(t, -2**63)
    for _ in range(2):
        lib.gf_ab_trace_clear()
        torch.cuda.synchronize()
        gf.sample_layer(g, q, t0, t, fan[1], p, seed=1)
        torch.cuda.synchronize()
    tiles = (q.numel() + ft - 1) // ft
    buf = np.zeros((tiles, 5), np.uint64)
    lib.gf_ab_trace_dump(buf.ctypes.data, tiles)
    b = buf.astype(np.float64)
    b -= b[:, :1].min()
    d = lambda i, j: np.mean(b[:, j] - b[:, i]) / 1e3  # noqa: E731
    span = (b[:, 4].max() - b[:, 0].min()) / 1e3
    life = np.mean(b[:, 4] - b[:, 0]) / 1e3
    print(f"{pol} hop1: {tiles} tiles, launch span {span:.0f} us, mean tile life {life:.2f} us, "
          f"tiles in flight ~{tiles * life / span:.0f}")
    print(f"   ticket->publish {d(0, 1):.2f}  publish->selection {d(1, 2):.2f}  "
          f"selection->base (look-back) {d(2, 3):.2f}  base->end (gather/store) {d(3, 4):.2f} us")
