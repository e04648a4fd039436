"""The ``python -m paper_2311_17410_b200`` command line (reference cli.py:193-263).

CPU: generate / partition outputs and CSV validation.  GPU: ingest / sample JSON equal to
the reference CLI's output on the same generated CSV (tests/golden/formats.npz), cluster and
bench run end to end.
"""

from __future__ import annotations

import contextlib
import io
import json
import os

import numpy as np
import pytest

from paper_2311_17410_b200 import cli
from paper_2311_17410_b200.harness import IngestFormatError, load_edge_csv
from paper_2311_17410_b200.partition import PartitionSpec, dispatch
from paper_2311_17410_b200.synth import generate_synthetic_arrays

GOLD = json.loads(np.load(os.path.join(os.path.dirname(__file__), "golden", "formats.npz"))["results"]
                  .tobytes().decode())


def run(argv):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        code = cli.main(argv)
    return code, buf.getvalue()


@pytest.fixture
def gen_csv(tmp_path):
    path = str(tmp_path / "g.csv")
    code, out = run(["generate", "--nodes", "60", "--edges", "800", "--time-span", "5000", "--seed", "4", "--out", path])
    assert code == 0 and json.loads(out) == {"edges": 800, "out": path}
    return path


def test_generate_and_partition(gen_csv, tmp_path):
    s, d, t = generate_synthetic_arrays(60, 800, 2.2, 5000, 4)
    edges = load_edge_csv(gen_csv)
    assert edges == list(zip(s.tolist(), d.tolist(), t.tolist()))
    prefix = str(tmp_path / "parts.csv")
    code, out = run(["partition", "--data", gen_csv, "--partitions", "3", "--out-prefix", prefix])
    res = json.loads(out)
    want = dispatch(PartitionSpec(3), edges, False)
    for p, path in enumerate(res["shards"]):
        assert load_edge_csv(path) == list(want[p].edges)
    stats = json.load(open(res["stats"]))
    assert sum(stats["node_counts"]) == len(set(s.tolist()) | set(d.tolist()))


def test_csv_errors(tmp_path):
    bad = tmp_path / "bad.csv"
    bad.write_text("a,b,c\n1,2,3\n")
    with pytest.raises(IngestFormatError, match="row 1"):
        load_edge_csv(bad)
    bad.write_text("src,dst,timestamp\n1,2,5\n2,3,4\n")
    with pytest.raises(IngestFormatError, match="row 3: timestamps not sorted"):
        load_edge_csv(bad)
    bad.write_text("src,dst,timestamp\n1,x,5\n")
    assert run(["partition", "--data", str(bad), "--partitions", "2", "--out-prefix", str(tmp_path / "p")])[0] == 2


@pytest.mark.gpu
def test_ingest_and_sample_equal_reference_cli(cuda_device, gen_csv):
    code, out = run(["ingest", "--data", gen_csv, "--tau", "8", "--batch-edges", "100"])
    assert code == 0 and json.loads(out) == json.loads(GOLD["cli_ingest"])
    code, out = run(["sample", "--data", gen_csv, "--targets", "0,5,7,59,61", "--times", "4000,2000,5000,100,5000",
                     "--fanouts", "3,2"])
    assert json.loads(out) == json.loads(GOLD["cli_sample"])
    code, out = run(["sample", "--data", gen_csv, "--directed", "--tau", "4", "--targets", "1,2,3",
                     "--times", "5000,2500,10", "--fanouts", "5"])
    assert json.loads(out) == json.loads(GOLD["cli_sample_dir"])


@pytest.mark.gpu
@pytest.mark.parametrize("policy", ["recent", "uniform"])
def test_cluster_and_bench_commands(cuda_device, gen_csv, policy):
    code, out = run(["cluster", "--data", gen_csv, "--machines", "3", "--workers", "2", "--policy", policy,
                     "--requests", "6", "--fanouts", "4,3"])
    res = json.loads(out)
    assert code == 0 and res["bitwise_matches"] == 6 and len(res["telemetry"]) == 6
    code, out = run(["bench", "--data", gen_csv, "--repeats", "2"])
    res = json.loads(out)
    assert res["sampling_throughput"] > 0 and res["fetch_throughput"] > 0 and res["avg_list_len"] > 0
