"""Golden fixtures for the data formats and host helpers either side of the hot path,
generated from the UNMODIFIED reference (``ctdg``) in the build container:

    python tests/golden/make_golden_formats.py

formats.npz holds
  wire_<i>          TGRP frames the reference encoded (wire.encode_message) for a
                    fixed set of messages; the messages themselves are rebuilt by
                    tests/test_formats.py from the same seeds
  tgff_node/edge    TGFF feature files (features.save_features)
  metrics / partition / cluster results as JSON strings
"""

from __future__ import annotations

import io
import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF_SRC)
sys.dont_write_bytecode = True
import ctdg  # noqa: E402
from ctdg import wire  # noqa: E402
from ctdg.features import KIND_EDGE, KIND_NODE, save_features  # noqa: E402

sys.path.insert(0, os.path.dirname(HERE))
from format_cases import cluster_case, feature_rows, metric_inputs, partition_edges, wire_messages  # noqa: E402


def ref_msg(kind, d):
    return getattr(wire, kind)(**d)


def main():
    out = {}
    for i, (rid, kind, d) in enumerate(wire_messages()):
        out[f"wire_{i}"] = np.frombuffer(wire.encode_message(rid, ref_msg(kind, d)), dtype=np.uint8)
    for name, kind in (("tgff_node", KIND_NODE), ("tgff_edge", KIND_EDGE)):
        ids, rows = feature_rows(kind)
        buf = io.BytesIO()
        save_features(buf, kind, rows.shape[1], ids, rows)
        out[name] = np.frombuffer(buf.getvalue(), dtype=np.uint8)
    res = {}
    for i, counts in enumerate(metric_inputs()):
        try:
            fit = ctdg.access_distribution(counts)
            res[f"access_{i}"] = {"powerlaw_r2": repr(fit["powerlaw_r2"]), "exponential_r2": repr(fit["exponential_r2"]),
                                  "degenerate": fit["degenerate"], "frequencies": fit["frequencies"].tolist()}
        except ValueError as e:
            res[f"access_{i}"] = {"error": str(e)}
        res[f"cv_{i}"] = repr(ctdg.coefficient_of_variation(counts))
    res["jaccard"] = [repr(ctdg.jaccard(a, b)) for a, b in (([1, 2, 3], [2, 3, 4]), ([], []), ([5], [6]))]
    for P in (1, 3, 4):
        for directed in (True, False):
            edges = partition_edges()
            spec = ctdg.PartitionSpec(P)
            shards = ctdg.dispatch(spec, edges, directed)
            st = ctdg.balance_stats(spec, edges, directed)
            res[f"partition_{P}_{int(directed)}"] = {
                "shards": [list(map(list, s.edges)) for s in shards],
                "stats": [list(st.node_counts), list(st.edge_counts), repr(st.node_cv), repr(st.edge_cv)]}
    # cluster: recent sampling is content-deterministic -> bit-exact reference outputs
    for directed in (True, False):
        edges, targets, times, fanouts = cluster_case(directed)
        cl = ctdg.ClusterSim(ctdg.ClusterSpec(3, 2), directed=directed, tau=8)
        ids = cl.add_edges(edges)
        req = ctdg.SampleRequest(targets, times, fanouts, ctdg.SamplingPolicy("recent"), 5)
        s = cl.sample_khop(req, ctdg.Origin(0, 1))
        res[f"cluster_{int(directed)}"] = {"ids": ids, "sample": s.to_json_dict(),
                                           "requests": [t.requests_served for _, _, t in cl.all_telemetry()]}
    # CLI: the reference's JSON for ingest / sample on a generated CSV (tests/test_gpu_cluster.py)
    import contextlib
    import tempfile

    from ctdg import cli

    with tempfile.TemporaryDirectory() as tmp:
        csv_path = os.path.join(tmp, "g.csv")
        cli.main(["generate", "--nodes", "60", "--edges", "800", "--time-span", "5000", "--seed", "4",
                  "--out", csv_path])
        for name, argv in (("cli_ingest", ["ingest", "--data", csv_path, "--tau", "8", "--batch-edges", "100"]),
                           ("cli_sample", ["sample", "--data", csv_path, "--targets", "0,5,7,59,61",
                                           "--times", "4000,2000,5000,100,5000", "--fanouts", "3,2"]),
                           ("cli_sample_dir", ["sample", "--data", csv_path, "--directed", "--tau", "4",
                                               "--targets", "1,2,3", "--times", "5000,2500,10", "--fanouts", "5"])):
            buf = io.StringIO()
            with contextlib.redirect_stdout(buf):
                cli.main(argv)
            res[name] = buf.getvalue()
    out["results"] = np.frombuffer(json.dumps(res).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "formats.npz"), **out)
    print("wrote", os.path.join(HERE, "formats.npz"), sorted(out))


if __name__ == "__main__":
    main()
