"""C2 (32^3 Q4) Chebyshev(5,20)-Jacobi PCG: fused v4-brick epilogues (default)
vs unfused column-kernel vmult + vector kernels (DG_NO_FUSED_CG=1 is read once
per process: run twice)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench
import torch
r = bench.run_cg(False)
print(json.dumps({"fused_off": os.environ.get("DG_NO_FUSED_CG"), "its": r["iterations"],
                  "solve_ms": round(r["solve_ms"], 2), "ms_per_it": round(r["ms_per_iteration"], 4),
                  "mg_ms": round(r["multigrid"]["solve_ms"], 2)}))
