"""Per CUDA source line: warp-stall samples by reason (ncu 'cuda,sass'
source-page CSV).  Usage: stall_lines.py <csv> [reason] [top]"""
import csv
import os
import sys
from collections import Counter, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
reason = sys.argv[2] if len(sys.argv) > 2 else "stall_wait"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
hdr = None
fname = "?"
key = None
per = defaultdict(Counter)
src = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = os.path.splitext(os.path.basename(r[1]))[0]
        continue
    if r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None:
        continue
    if r[0].strip():
        try:
            key = (fname, int(r[0]))
            src[key] = r[1].strip()
        except ValueError:
            pass
        continue
    if key is None or len(r) < len(hdr) or not r[2].startswith("0x"):
        continue
    for h, i in hdr.items():
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                per[key][h] += int(float(r[i] or 0))
            except ValueError:
                pass
tot = Counter()
for k in per:
    tot.update(per[k])
allt = sum(tot.values())
print("all reasons:", ", ".join(f"{h[6:]} {100*n/allt:.1f}%" for h, n in tot.most_common(10)))
print(f"\ntop lines for {reason} ({100*tot[reason]/allt:.1f}% of samples):")
for k in sorted(per, key=lambda k: -per[k][reason])[:top]:
    print(f"{100*per[k][reason]/allt:5.1f}%  {k[0]}:{k[1]}  {src.get(k, '')[:90]}")
