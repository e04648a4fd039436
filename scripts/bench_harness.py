"""configs[2]: MOOC/LASTFM-shaped streaming -- the continuous-learning round loop (harness.py:371-513).

    python scripts/bench_harness.py [--impl ours|reference] [--shape mooc|lastfm] [--rounds R]

Each round ingests one incremental batch (10 batches after a 30% initial load, harness.py:256-277),
then runs 3 epochs x minibatches of 600 training edges: sample_khop (recent, fanout [10]) over the
minibatch's src+dst, then the node and edge fetch blocks through LRU caches (node/edge dims 16).
`--impl ours` runs paper_2311_17410_b200.harness on cuda:0; `--impl reference` runs the unmodified
reference harness on the host (build container only: /root/reference).  Prints one JSON line with
per-round wall-clock stage times (the RoundReport fields) and minibatch iterations/s.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

SHAPES = {  # public dataset statistics; synthetic streams with the reference generator law
    "mooc": dict(generate_nodes=7_144, generate_edges=411_749),
    "lastfm": dict(generate_nodes=1_980, generate_edges=1_293_103),
}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--shape", choices=sorted(SHAPES), default="mooc")
    ap.add_argument("--rounds", type=int, default=10)
    args = ap.parse_args()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if args.impl == "reference":
        sys.path.insert(0, "/root/reference/pkg/src")
        from ctdg.harness import CacheConfig, RunConfig, run_continuous
    else:
        sys.path.insert(0, root)
        from paper_2311_17410_b200.harness import CacheConfig, RunConfig, run_continuous
    n_edges = SHAPES[args.shape]["generate_edges"]
    cfg = RunConfig(**SHAPES[args.shape], generate_skew=2.2, generate_time_span=2_592_000, directed=False, tau=48,
                    initial_fraction=0.3, batch_by="count", batch_edges=-(-int(0.7 * n_edges) // 10),
                    epochs_per_round=3, minibatch_size=600, fanouts=(10,), policy_kind="recent", node_dim=16,
                    edge_dim=16, cache=CacheConfig(), seed=0, label=args.shape)
    t0 = time.perf_counter()
    rounds = []
    for rep in run_continuous(cfg):
        rounds.append(rep)
        if len(rounds) >= args.rounds:
            break
    wall = time.perf_counter() - t0
    its = sum(r.n_iterations for r in rounds)
    upd = sum(r.graph_update_time for r in rounds)
    smp = sum(r.sampling_time for r in rounds)
    fch = sum(r.fetch_time for r in rounds)
    ing = sum(r.n_new_edges for r in rounds)
    print(json.dumps({
        "impl": args.impl, "workload": f"{args.shape}-shaped continuous learning (harness.py:371-513)",
        "rounds": len(rounds), "iterations": its, "iterations_per_s": round(its / (smp + fch), 1),
        "ingest_edges_per_s": round(ing / upd, 1) if upd else None,
        "sampling_s": round(smp, 4), "fetch_s": round(fch, 4), "graph_update_s": round(upd, 4),
        "wall_s_incl_setup": round(wall, 2),
        "node_hit_rate_last": rounds[-1].node_hit_rates[-1] if rounds and rounds[-1].node_hit_rates else None,
        "config": {"minibatch": 600, "fanouts": [10], "policy": "recent", "epochs_per_round": 3,
                   "node_dim": 16, "edge_dim": 16, "cache": "lru 3% / 3 per mille, reuse + restore"}}))


if __name__ == "__main__":
    main()
