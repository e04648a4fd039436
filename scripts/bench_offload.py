"""Offload (storage.py:516-574): serialise and unlink every block older than a cutoff.

    python scripts/bench_offload.py [--impl ours|reference] [--edges E]

A GDELT-law stream (directed, tau 8192) is ingested, then everything before the median timestamp is
offloaded into an in-memory TGOF blob.  Reports offloaded edge records/s and blob bytes; `ours` times
DynamicGraph.offload_before on cuda:0 (device-built blob, D2H, unlink), `reference` the unmodified
reference on the host (build container only).
"""

from __future__ import annotations

import argparse
import io
import json
import os
import sys
import time

import numpy as np


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--edges", type=int, default=20_000_000)
    args = ap.parse_args()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import paper_2311_17410_b200 as gf

    src, dst, ts = gf.generate_synthetic_arrays(17_000, args.edges, 2.2, 175_200, seed=0, src_skew=2.2)
    cutoff = int(ts[len(ts) // 2])
    if args.impl == "reference":
        sys.path.insert(0, "/root/reference/pkg/src")
        from ctdg.storage import DynamicGraph, InsertionBatch

        g = DynamicGraph(directed=True, tau=8192)
        edges = list(zip(src.tolist(), dst.tolist(), ts.tolist()))
        for lo in range(0, len(edges), 100_000):
            g.add_edges(InsertionBatch(edges[lo:lo + 100_000]))
        sync = lambda: None  # noqa: E731
    else:
        import torch

        g = gf.DynamicGraph(directed=True, tau=8192, device=torch.device("cuda", 0))
        for lo in range(0, len(src), 100_000):
            g.add_edges_arrays(src[lo:lo + 100_000], dst[lo:lo + 100_000], ts[lo:lo + 100_000])
        sync = torch.cuda.synchronize
    sync()
    buf = io.BytesIO()
    t0 = time.perf_counter()
    n = g.offload_before(cutoff, buf)
    sync()
    dt = time.perf_counter() - t0
    print(json.dumps({"impl": args.impl, "workload": f"GDELT-law {args.edges} edges, directed, tau 8192; offload "
                      "everything before the median timestamp (storage.py:516-574)",
                      "offloaded_edges": n, "blob_bytes": len(buf.getvalue()), "seconds": round(dt, 4),
                      "edges_per_s": round(n / dt, 1), "blob_GB_per_s": round(len(buf.getvalue()) / dt / 1e9, 3)}))


if __name__ == "__main__":
    main()
