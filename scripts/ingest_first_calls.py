"""Per-call wall time of the first ingest calls on a fresh graph (WIKI / REDDIT shapes, undirected)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_17410_b200 as gf  # noqa: E402

for name, nodes, edges, tau in (("wiki", 9000, 157_000, 48), ("reddit", 11_000, 672_000, 48), ("wiki2", 9000, 157_000, 48)):
    dev = torch.device("cuda", 0)
    src, dst, ts = gf.generate_synthetic_device(nodes, edges, 2.2, 2_592_000, seed=0, device=dev)
    g = gf.DynamicGraph(directed=False, tau=tau, device=dev)
    g.reserve(nodes, nodes * 16 + 2 * edges // tau + 1024, 2 * edges + min(nodes * tau, edges))
    torch.cuda.synchronize()
    times = []
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for lo in range(0, edges, 100_000):
        t0 = time.perf_counter()
        g.add_edges_arrays(src[lo:lo + 100_000], dst[lo:lo + 100_000], ts[lo:lo + 100_000])
        times.append((time.perf_counter() - t0) * 1e6)
    b.record()
    torch.cuda.synchronize()
    print(name, "calls us:", [round(t) for t in times], "device ms", round(a.elapsed_time(b), 3),
          "edges/s %.1f M" % (edges / a.elapsed_time(b) / 1e3))
