"""Reference uniform-sampling statistics on GDELT-1/50 queries (run in the build container).

    python tests/golden/make_uniform_ref.py

Builds the GDELT-shaped stream at 1/50 scale (17,000 nodes, 3,820,000 directed
edges, tau 8192, skew and src_skew 2.2, span 175,200) with the
UNMODIFIED reference (``ctdg.generate_synthetic`` + ``DynamicGraph.add_edges``
in 100K batches), picks queries (node, t_end) whose in-window candidate
counts n cover 12 ... 1,000, and runs the reference ``sample_layer`` (uniform,
fanout 10; PCG64 partial Fisher-Yates, sampling.py:185-198) on each query
repeated R times in one call -- the reference keys each repetition by its
occurrence rank (sampling.py:140-142,243-248), so the R draws are
independent.  Stored per query (tests/golden/uniform_ref.npz):

  * inclusion counts per candidate (chronological candidate order),
  * for n <= 14: counts of every drawn k-subset (as bitmasks),
  * for n == 30: the pair-inclusion count matrix.

tests/test_gpu_uniform_ref.py runs the CUDA sampler on the same queries and
compares: two-sample chi^2 on inclusions, subset and pair tables (p > 1e-4).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF_SRC)
sys.dont_write_bytecode = True
import ctdg  # noqa: E402
from ctdg import DynamicGraph, SamplingPolicy, generate_synthetic, sample_layer  # noqa: E402
from ctdg.storage import TS_MIN  # noqa: E402

NODES, EDGES, SKEW, SPAN = 17_000, 3_820_000, 2.2, 175_200
FANOUT = 10
TARGET_N = (12, 14, 30, 64, 200, 1000)
REPS = {12: 20_000, 14: 40_000, 30: 40_000, 64: 20_000, 200: 20_000, 1000: 20_000}
SEED = 4242


def main():
    t0 = time.time()
    edges = generate_synthetic(NODES, EDGES, SKEW, SPAN, seed=0, src_skew=SKEW)
    g = DynamicGraph(directed=True, tau=8192)
    for lo in range(0, len(edges), 100_000):
        g.add_edges(edges[lo:lo + 100_000])
    src = np.fromiter((e[0] for e in edges), np.int64, len(edges))
    ts = np.fromiter((e[2] for e in edges), np.int64, len(edges))
    print(f"built in {time.time() - t0:.1f}s", flush=True)
    deg = np.bincount(src, minlength=NODES)
    rng = np.random.default_rng(11)
    out = {"nodes": NODES, "edges": EDGES, "fanout": FANOUT, "seed": SEED}
    for qi, n in enumerate(TARGET_N):
        # a node with at least n + 50 out-edges (hubs for large n, mid-degree nodes for small n);
        # t_end = the timestamp at chronological position n of its list, so the window
        # [TS_MIN, t_end) holds the first n' >= ... candidates (ties counted by the reference itself)
        cands = np.flatnonzero((deg >= n + 50) & (deg <= max(40 * n, 5_000)))
        v = int(rng.choice(cands))
        vts = np.sort(ts[src == v])
        t_end = int(vts[n])
        # the reference's own candidate list for the query (recent at a huge fanout = all, newest first)
        full = sample_layer(g, [v], [TS_MIN], [t_end], 10**9, SamplingPolicy.recent(), seed=0)
        cand = full.edge_ids[::-1].copy()  # chronological
        m = len(cand)
        R = REPS[n]
        t1 = time.time()
        lay = sample_layer(g, [v] * R, [TS_MIN] * R, [t_end] * R, FANOUT, SamplingPolicy.uniform(), seed=SEED + qi)
        pos_of = {int(e): i for i, e in enumerate(cand.tolist())}
        offs = lay.offsets
        assert np.all(np.diff(offs) == min(FANOUT, m))
        pos = np.array([pos_of[int(e)] for e in lay.edge_ids.tolist()], np.int64).reshape(R, -1)
        incl = np.bincount(pos.ravel(), minlength=m)
        out[f"q{qi}_node"] = v
        out[f"q{qi}_t_end"] = t_end
        out[f"q{qi}_n"] = m
        out[f"q{qi}_reps"] = R
        out[f"q{qi}_candidates"] = cand
        out[f"q{qi}_incl"] = incl
        if m <= 14:
            masks = np.zeros(R, np.int64)
            for j in range(pos.shape[1]):
                masks |= np.left_shift(1, pos[:, j])
            u, c = np.unique(masks, return_counts=True)
            out[f"q{qi}_subset_masks"] = u
            out[f"q{qi}_subset_counts"] = c
        if m == 30:
            pair = np.zeros((m, m), np.int64)
            for row in pos:
                a = np.sort(row)
                ii, jj = np.triu_indices(len(a), 1)
                np.add.at(pair, (a[ii], a[jj]), 1)
            out[f"q{qi}_pairs"] = pair
        print(f"q{qi}: node {v} t_end {t_end} n {m} R {R} in {time.time() - t1:.1f}s", flush=True)
    out["n_queries"] = len(TARGET_N)
    np.savez_compressed(os.path.join(HERE, "uniform_ref.npz"), **out)
    print("ctdg", getattr(ctdg, "__version__", "?"), f"total {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
