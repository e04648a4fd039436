"""Summarise scripts/ncu_sampler.sh output into profiles/.

Reads gpurun_out/prof.ncu-rep (ncu --set full, the 4 fused sampler launches of one step, in launch
order recent/hop0, recent/hop1, uniform/hop0, uniform/hop1) and
gpurun_out/launches.csv (the launch list), writes
  profiles/<round>_ncu_sampler_launches.json  per-launch metrics
  profiles/ncu_traffic.json                   dram read+write bytes per launch, averaged per kernel
  profiles/<round>_launches.csv               copy of the launch list
Usage: python scripts/ncu_summarize.py r02 [report] [config]

profiles/ncu_traffic.json records, per launch (k_sample_fused[<policy>/hop<h>]), the DRAM bytes
and ncu duration, the config the capture ran (bench.py --config), and the hash of the sources
(bench.TRAFFIC_SOURCES) at summary time, so bench.py can tell a stale capture from a current one.
"""

from __future__ import annotations

import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TAGS = ["recent/hop0", "recent/hop1", "uniform/hop0", "uniform/hop1"]
METRICS = {
    "gpu__time_duration.sum": "ns",
    "dram__bytes_read.sum": "bytes",
    "dram__bytes_write.sum": "bytes",
    "lts__t_sector_hit_rate.pct": "pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "pct",
    "launch__registers_per_thread": "n",
    "smsp__issue_active.avg.per_cycle_active": "n",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum": "n",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum": "n",
}


def to_float(s: str) -> float:
    return float(s.replace(",", ""))


def raw_rows(rep: str) -> list[dict]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                         check=True, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    header = rows[0]
    return [dict(zip(header, r)) for r in rows[2:]]  # row 1 holds units


def main() -> None:
    rnd = sys.argv[1] if len(sys.argv) > 1 else "r02"
    rep = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", "prof.ncu-rep")
    config = sys.argv[3] if len(sys.argv) > 3 else "gdelt"
    rows = raw_rows(rep)
    summ, traffic = {}, {}
    for i, r in enumerate(rows):
        # launches come in step order; the tag follows the launch index (template args stripped)
        name = r["Kernel Name"].split("(")[0].split()[-1].split("::")[-1].split("<")[0]
        tag = TAGS[i % len(TAGS)] if len(rows) <= len(TAGS) else f"#{i}"
        e = {
            "ms": round(to_float(r["gpu__time_duration.sum"]) / 1e6, 6),
            "dram_read_GB": round(to_float(r["dram__bytes_read.sum"]) / 1e9, 6),
            "dram_write_GB": round(to_float(r["dram__bytes_write.sum"]) / 1e9, 6),
            "l2_hit_pct": round(to_float(r["lts__t_sector_hit_rate.pct"]), 3),
            "warps_active_pct": round(to_float(r["sm__warps_active.avg.pct_of_peak_sustained_active"]), 3),
            "regs": to_float(r["launch__registers_per_thread"]),
            "issue_per_sched": round(to_float(r["smsp__issue_active.avg.per_cycle_active"]), 3),
        }
        te = r.get("smsp__thread_inst_executed_per_inst_executed.ratio")
        if te:
            e["warp_exec_efficiency_pct"] = round(100 * to_float(te) / 32, 1)
        req = r.get("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum")
        sec = r.get("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum")
        if req and sec:
            e["ld_sectors_per_request"] = round(to_float(sec) / max(1.0, to_float(req)), 2)
        summ[f"{name}[{tag}]"] = e
        traffic[f"{name}[{tag}]"] = {"dram_bytes": int(to_float(r["dram__bytes_read.sum"]) + to_float(r["dram__bytes_write.sum"])),
                                     "ms": e["ms"]}
    with open(os.path.join(ROOT, "profiles", f"{rnd}_ncu_sampler_launches.json"), "w") as f:
        json.dump(summ, f, indent=1)
    sys.path.insert(0, ROOT)
    import bench

    with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as f:
        json.dump({"config": config, "source_sha16": bench.source_sha16(), "sources": list(bench.TRAFFIC_SOURCES),
                   "report": os.path.basename(rep), "metric": "dram__bytes_read.sum + dram__bytes_write.sum per launch",
                   "launches": traffic}, f, indent=1)
    launches = os.path.join(ROOT, "gpurun_out", "launches.csv")
    if os.path.exists(launches):
        shutil.copy(launches, os.path.join(ROOT, "profiles", f"{rnd}_launches.csv"))
    for k, v in summ.items():
        print(k, v)


if __name__ == "__main__":
    main()
