#!/bin/bash
# Sampler-only bench line (no CPU baseline / e2e / fetch) and a compact summary of it.
# Usage (repo root, under gpurun): scripts/quick_bench.sh TAG [bench.py args...]
tag=$1; shift
timeout 400 python bench.py --no-cpu --no-e2e --no-fetch "$@" > gpurun_out/qb_$tag.json 2> gpurun_out/qb_$tag.err
python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/qb_{tag}.json").read().strip().splitlines()[-1])
except Exception as e:
    print("bench failed:", e); print(open(f"gpurun_out/qb_{tag}.err").read()[-2000:]); sys.exit(1)
print(tag, "value %.2f G/s" % (d["value"] / 1e9), "frac", d["roofline"]["frac"], "ms/step", d["ms_per_step"])
for p, v in d["per_policy"].items():
    print("  ", p, "%.2f G/s" % (v["value"] / 1e9), "frac", v.get("frac"), "ms", v["ms_per_step"])
for k, v in d["kernels"].items():
    print("  ", k, v["ms"], "frac", v.get("frac"))
print("  replay %.2f G/s" % (d["replay"]["value"] / 1e9), "ingest %.3f G/s" % (d["ingest"]["value"] / 1e9))
PY
