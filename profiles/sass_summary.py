"""Summarise an ncu SASS source-page CSV: instructions executed per opcode
and warp-stall samples per opcode (used for the profiles/ summaries)."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
ins, stall = Counter(), Counter()
tot_i = tot_s = 0
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    toks = r[ix["Source"]].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    op = op.split(".")[0]
    n = int(float(r[ix["Instructions Executed"]] or 0))
    s = int(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
    ins[op] += n
    stall[op] += s
    tot_i += n
    tot_s += s
print(f"total warp instructions executed {tot_i:,}  stall samples {tot_s:,}")
for op, n in ins.most_common(25):
    print(f"{op:10s} {n:14,d} {100*n/tot_i:5.1f}%   stalls {100*stall[op]/max(tot_s,1):5.1f}%")
