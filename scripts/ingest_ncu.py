"""ncu helper: warm a GDELT-law graph, then ingest a few 100K-edge batches (the profiled ones).
Usage: ncu ... python scripts/ingest_ncu.py [warm_edges] [batches] [batch] [nodes] [span]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_17410_b200 as gf  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
NB = int(sys.argv[2]) if len(sys.argv) > 2 else 5
B = int(sys.argv[3]) if len(sys.argv) > 3 else 100_000
NODES = int(sys.argv[4]) if len(sys.argv) > 4 else 17_000
SPAN = int(sys.argv[5]) if len(sys.argv) > 5 else 175_200
dev = torch.device("cuda", 0)
E = W + NB * B
src, dst, ts = gf.generate_synthetic_device(NODES, E, 2.2, SPAN, seed=0, src_skew=2.2, device=dev)
g = gf.DynamicGraph(directed=True, tau=8192, device=dev)
g.reserve(NODES, NODES * 16 + E // 8192 + 1024, E + min(NODES * 8192, E // 2))
g.add_edges_arrays(src[:W], dst[:W], ts[:W])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for lo in range(W, E, B):
    g.add_edges_arrays(src[lo:lo + B], dst[lo:lo + B], ts[lo:lo + B])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
