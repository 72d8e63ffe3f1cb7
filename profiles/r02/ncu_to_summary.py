"""ncu --set full capture of the headline vmult kernel -> the summary entry
bench.py reads (profiles/ncu_laplace.json, key k<degree>): kernel identifier
in dg_laplace_kernel_name's format, DRAM bytes per launch, fp64 instruction
counts per DoF (from the per-cycle SASS counters x elapsed cycles), pipe /
issue / occupancy figures.
usage: ncu_to_summary.py <rep> <k> <dofs> <source-note> [json]"""
import csv, json, os, re, subprocess, sys

rep, k, dofs, note = sys.argv[1], int(sys.argv[2]), float(sys.argv[3]), sys.argv[4]
out = sys.argv[5] if len(sys.argv) > 5 else os.path.join(os.path.dirname(os.path.dirname(
    os.path.abspath(__file__))), "ncu_laplace.json")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, units, v = rows[0], rows[1], rows[2]
m = dict(zip(h, v))


def num(key):
    return float(m[key].replace(",", ""))


def scale(key):
    u = units[h.index(key)]
    return {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6,
            "ns": 1e-9}.get(u, 1.0)


name = m["Kernel Name"]
mt = re.match(r"void (?:dg::)?(\w+)<([^>]*)>", name)
ident = mt.group(1) + "<" + ",".join(
    {"false": "0", "true": "1"}.get(a.strip(), a.strip()) for a in mt.group(2).split(",")) + ">"
cyc = num("sm__cycles_elapsed.avg") if "sm__cycles_elapsed.avg" in m else None
sms = 148
per_dof = {}
for op in ("dfma", "dadd", "dmul"):
    key = f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed"
    if key in m and cyc:
        per_dof[op] = num(key) * cyc / dofs
entry = {
    "kernel": ident,
    "source": note,
    "dram_bytes_per_launch": num("dram__bytes_read.sum") * scale("dram__bytes_read.sum")
    + num("dram__bytes_write.sum") * scale("dram__bytes_write.sum"),
    "dram_read_bytes": num("dram__bytes_read.sum") * scale("dram__bytes_read.sum"),
    "dram_write_bytes": num("dram__bytes_write.sum") * scale("dram__bytes_write.sum"),
    "duration_ms_ncu": num("gpu__time_duration.sum") * scale("gpu__time_duration.sum") * 1e3,
    "fp64_pipe_pct": num("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "warps_active_pct": num("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "inst_executed": num("smsp__inst_executed.sum"),
    "registers_per_thread": num("launch__registers_per_thread"),
    "grid": num("launch__grid_size"), "block": num("launch__block_size"),
    "l2_hit_pct": num("lts__t_sector_hit_rate.pct"),
}
for op, val in per_dof.items():
    entry[f"{op}_per_dof"] = round(val, 2)
if per_dof:
    entry["flop_per_dof"] = round(2 * per_dof.get("dfma", 0) + per_dof.get("dadd", 0)
                                  + per_dof.get("dmul", 0), 1)
    entry["fp64_inst_per_dof"] = round(sum(per_dof.values()), 1)
entry["thread_inst_per_dof"] = round(entry["inst_executed"] * 32 / dofs, 1)
data = json.load(open(out)) if os.path.exists(out) else {}
old = data.get(f"k{k}")
if old and old.get("kernel") != ident:
    data[f"k{k}_previous_{old.get('kernel', '?').split('<')[0]}"] = old
data[f"k{k}"] = entry
data["comment"] = ("Per launch of the default vmult kernel per degree from one ncu --set full "
                   "capture (profiles/r02/ncu_to_summary.py); bench.py uses an entry only if "
                   "its 'kernel' equals dg_laplace_kernel_name of the benched context.")
json.dump(data, open(out, "w"), indent=1)
print(json.dumps(entry, indent=1))
