"""Aggregate an ncu 'cuda,sass' source-page CSV by CUDA source line
(the line rows carry the aggregated metrics): warp instructions executed
and stall samples per line, hottest first."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hdr_i]
iexec = hdr.index("Instructions Executed")
istall = hdr.index("Warp Stall Sampling (All Samples)")
items = []
for r in rows[hdr_i + 1:]:
    if r and r[0].strip():
        try:
            items.append((int(r[0]), r[1].strip(), int(float(r[iexec])), int(float(r[istall]))))
        except ValueError:
            pass
tot = sum(i[2] for i in items)
tots = max(sum(i[3] for i in items), 1)
print(f"total warp instructions {tot:,}")
for ln, s, n, st in sorted(items, key=lambda x: -x[2])[:top]:
    print(f"{ln:4d} {100*n/tot:5.1f}% stall {100*st/tots:5.1f}%  {s[:80]}")
