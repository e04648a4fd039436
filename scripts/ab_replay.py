"""Per-policy latest-root and replay-root step times for the current library (or GF_LIB_PATH):
    python scripts/ab_replay.py  ->  one JSON line."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

cfg = bench.CONFIGS["gdelt"]
dev = torch.device("cuda", 0)
src, dst, ts = bench.make_stream(cfg, dev)
g, _ = bench.build_graph(cfg, src, dst, ts, 1, 0, dev)
out = {"lib": os.environ.get("GF_LIB_PATH", "current")}
for name, (r, t) in {"latest": bench.roots_for_rank(src, dst, ts, 1 << 20, 0),
                     "replay": bench.replay_roots_for_rank(src, dst, ts, 1 << 20, 0)}.items():
    for pol in ("recent", "uniform"):
        bench.run_step(g, r, t, 0, (pol,))
        ms, e = bench.timed_steps(g, r, t, 0, 5, (pol,))
        out[f"{name}/{pol}"] = round(ms / 5, 4)
print(json.dumps(out))
