"""Per CUDA source line: total warp-stall samples (all reasons) and executed
warp instructions, from an ncu 'cuda,sass' source-page CSV.
Usage: lines.py <csv> [top] [file-filter]"""
import csv, os, sys
from collections import Counter, defaultdict
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
filt = sys.argv[3] if len(sys.argv) > 3 else ""
hdr = None; fname = "?"; key = None
st = Counter(); ins = Counter(); src = {}; reasons = defaultdict(Counter)
for r in rows:
    if not r: continue
    if r[0] == "File Path":
        fname = os.path.splitext(os.path.basename(r[1]))[0]; continue
    if r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}; continue
    if hdr is None: continue
    if r[0].strip():
        try:
            key = (fname, int(r[0])); src[key] = r[1].strip()
        except ValueError: pass
        continue
    if key is None or len(r) < len(hdr) or not r[2].startswith("0x"): continue
    for h, i in hdr.items():
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                v = int(float(r[i] or 0)); st[key] += v; reasons[key][h[6:]] += v
            except ValueError: pass
    try: ins[key] += int(float(r[hdr["Instructions Executed"]] or 0))
    except (ValueError, KeyError): pass
ts = sum(st.values()); ti = sum(ins.values())
print(f"samples {ts}  warp-instr {ti}")
for k in sorted(st, key=lambda k: -st[k])[:top]:
    if filt and filt not in k[0]: continue
    rs = ", ".join(f"{a} {100*b/max(st[k],1):.0f}%" for a, b in reasons[k].most_common(3))
    print(f"{100*st[k]/ts:5.1f}% st {100*ins[k]/ti:5.1f}% in {k[0]}:{k[1]:<4} {src.get(k,'')[:70]:70s} [{rs}]")
