"""Top source lines by warp-stall samples / executed instructions from an
`ncu --page source --csv --print-source cuda,sass` dump.  Usage: python scripts/ncu_hot_lines.py dump.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
cs, ci = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
data = []
for r in rows[hi + 1:]:
    if len(r) < len(h) or not r[0]:
        continue
    try:
        data.append((int(r[cs]), int(r[ci]), r[0], r[1][:120]))
    except ValueError:
        pass
ts, ti = sum(d[0] for d in data) or 1, sum(d[1] for d in data) or 1
print(f"samples {ts} warp-instructions {ti}")
for s, i, ln, src in sorted(data, reverse=True)[:n]:
    print(f"{100 * s / ts:5.1f}% stall  {100 * i / ti:5.1f}% inst  L{ln}: {src.strip()}")
