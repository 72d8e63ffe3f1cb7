"""Per CUDA source line: warp instructions by opcode (from an ncu
'cuda,sass' source-page CSV)."""
import csv
import sys
from collections import Counter, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hdr_i]
iexec = hdr.index("Instructions Executed")
ops = defaultdict(Counter)
src = {}
line = None
for r in rows[hdr_i + 1:]:
    if not r:
        continue
    if r[0].strip():
        try:
            line = int(r[0]); src[line] = r[1].strip()
        except ValueError:
            pass
        continue
    if len(r) > iexec and r[2].startswith("0x") and line is not None:
        try:
            n = int(float(r[iexec]))
        except ValueError:
            continue
        toks = r[3].split()
        op = toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "?")
        ops[line][op.split(".")[0]] += n
tot_by_op = Counter()
for l in ops:
    tot_by_op.update(ops[l])
tot = sum(tot_by_op.values())
for op in [o for o, _ in tot_by_op.most_common(12)]:
    lines = sorted(ops, key=lambda l: -ops[l][op])[:6]
    print(f"{op:8s} {100*tot_by_op[op]/tot:5.1f}%  " +
          "; ".join(f"L{l}:{100*ops[l][op]/tot:.1f}%" for l in lines if ops[l][op]))
