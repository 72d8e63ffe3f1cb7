"""Per CUDA source line: warp instructions by opcode (from an ncu
'cuda,sass' source-page CSV).  Lines are keyed by (file, line); the report
prints <file-stem>:<line>.  Usage: line_ops.py <csv> [top-ops] [--lines]"""
import csv
import os
import sys
from collections import Counter, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 12
ops = defaultdict(Counter)
src = {}
fname = "?"
iexec = None
key = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = os.path.splitext(os.path.basename(r[1]))[0]
        continue
    if r[0] == "Line No":
        iexec = r.index("Instructions Executed")
        continue
    if iexec is None:
        continue
    if r[0].strip():
        try:
            key = (fname, int(r[0]))
            src[key] = r[1].strip()
        except ValueError:
            pass
        continue
    if len(r) > iexec and r[2].startswith("0x") and key is not None:
        try:
            n = int(float(r[iexec]))
        except ValueError:
            continue
        toks = r[3].split()
        op = toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "?")
        ops[key][op.split(".")[0]] += n
tot_by_op = Counter()
for k in ops:
    tot_by_op.update(ops[k])
tot = sum(tot_by_op.values())
print(f"total warp instructions {tot:,}")
for op in [o for o, _ in tot_by_op.most_common(top)]:
    keys = sorted(ops, key=lambda k: -ops[k][op])[:6]
    print(f"{op:8s} {100*tot_by_op[op]/tot:5.1f}%  " +
          "; ".join(f"{k[0]}:{k[1]}:{100*ops[k][op]/tot:.1f}%" for k in keys if ops[k][op]))
if "--lines" in sys.argv:
    print("\nheaviest source lines:")
    for k in sorted(ops, key=lambda k: -sum(ops[k].values()))[:40]:
        n = sum(ops[k].values())
        print(f"{100*n/tot:5.1f}%  {k[0]}:{k[1]}  {src.get(k, '')[:90]}")
