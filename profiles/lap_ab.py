"""A/B helper for Laplace-kernel changes: the 64^3 degree sweep (Q2-Q7),
the config-2 Chebyshev / multigrid PCG solves and the config-4 step, one
JSON line (run once per library build, e.g. DG_LIB=... python profiles/lap_ab.py)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

out = {"sweep": {k: round(v["dof_per_s"] / 1e9, 1)
                 for k, v in bench.run_degree_sweep(bench.hbm_peak()[0]).items()}}
cg = bench.run_cg(False)
out["cg_ms"] = round(cg["solve_ms"], 1)
out["cg_it"] = cg["iterations"]
out["mg_ms"] = round(cg["multigrid"]["solve_ms"], 2)
if "--step" in sys.argv:
    st = bench.run_c4_step(3)
    out["c4_ms"] = round(st["ms_per_step_steady"], 1)
print(json.dumps(out), flush=True)
