"""Top SASS instructions by warp-stall samples from `ncu -i X --page source --csv --print-source sass`.
Usage: python scripts/ncu_sass_hot.py dump.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
cs, ci = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
data = [(int(r[cs]), int(r[ci]), i, r[1].strip()) for i, r in enumerate(rows[hi + 1:]) if len(r) > ci and r[cs].isdigit()]
ts = sum(d[0] for d in data) or 1
print(f"samples {ts}")
for s, e, i, src in sorted(data, reverse=True)[:n]:
    print(f"{100 * s / ts:5.1f}%  #{i:5d} exec {e:9d}  {src}")
