"""Where ingest time goes: GDELT-law stream, 100K-edge batches through gf_graph_add_edges.

Prints edges/s (device events around the loop), the per-kernel device time from the library's
launch profiler, and host wall time per batch.
Usage: python scripts/ingest_profile.py [edges] [batch] [nodes] [span] [d|u]
(GDELT: 17000 nodes, span 175200 -- the defaults; mag8: 15250000 nodes, span 120, 10M batches)
"""

import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_17410_b200 as gf  # noqa: E402
from paper_2311_17410_b200 import _lib  # noqa: E402

E = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
B = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000
NODES = int(sys.argv[3]) if len(sys.argv) > 3 else 17_000
SPAN = int(sys.argv[4]) if len(sys.argv) > 4 else 175_200
DIRECTED = (sys.argv[5] != "u") if len(sys.argv) > 5 else True  # "u": undirected stream (WIKI / REDDIT law)
dev = torch.device("cuda", 0)
src, dst, ts = gf.generate_synthetic_device(NODES, E, 2.2, SPAN, seed=0, src_skew=2.2 if DIRECTED else None, device=dev)
TAU = 8192 if DIRECTED else 48
g = gf.DynamicGraph(directed=DIRECTED, tau=TAU, device=dev)
g.reserve(NODES, NODES * 16 + 2 * E // TAU + 1024, 2 * E + min(NODES * TAU, E))
half = E // 2
for lo in range(0, half, B):  # warm half
    g.add_edges_arrays(src[lo:lo + B], dst[lo:lo + B], ts[lo:lo + B])
torch.cuda.synchronize()
_lib.profile_enable(True)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
a.record()
nb = 0
for lo in range(half, E, B):
    g.add_edges_arrays(src[lo:lo + B], dst[lo:lo + B], ts[lo:lo + B])
    nb += 1
b.record()
torch.cuda.synchronize()
wall = time.perf_counter() - t0
prof = _lib.profile_summary()
_lib.profile_enable(False)
ms = a.elapsed_time(b)
print(f"profiled: {nb} batches of {B}: {ms:.1f} ms device, {wall * 1e3:.1f} ms wall -> {(E - half) / (ms / 1e3) / 1e6:.1f} M edges/s"
      f" ({ms / nb * 1e3:.0f} us/batch)")
tot = sum(v[1] for v in prof.values())
for k, (c, kms) in sorted(prof.items(), key=lambda kv: -kv[1][1]):
    print(f"  {k:40s} {c:6d} launches {kms:8.2f} ms  {kms / nb * 1e3:7.1f} us/batch")
print(f"  kernel sum {tot:.1f} ms = {tot / nb * 1e3:.0f} us/batch")
# unprofiled rate
torch.cuda.synchronize()
g2 = gf.DynamicGraph(directed=DIRECTED, tau=TAU, device=dev)
g2.reserve(NODES, NODES * 16 + 2 * E // TAU + 1024, 2 * E + min(NODES * TAU, E))
a.record()
for lo in range(0, E, B):
    g2.add_edges_arrays(src[lo:lo + B], dst[lo:lo + B], ts[lo:lo + B])
b.record()
torch.cuda.synchronize()
print(f"unprofiled: {E / (a.elapsed_time(b) / 1e3) / 1e6:.1f} M edges/s, {a.elapsed_time(b) / (E // B) * 1e3:.0f} us/batch")
