"""Kernel breakdown of C2 (32^3 Q4 Chebyshev(5,20)-Jacobi PCG, 50 iterations)
from a CUPTI trace (torch.profiler): real durations inside the solve graph."""
import collections, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1607_01323_b200 import mesh as M, operators as ops, solvers as sol
from paper_1607_01323_b200.spaces import DgSpace
mesh = M.build_box_mesh(((0, 1),) * 3, (32, 32, 32), periodic=(True, False, True))
sp = DgSpace(mesh, 4)
bcs = ops.BoundarySpec({"ymin": ops.DirichletBC(None), "ymax": ops.DirichletBC(None)}).resolve(sp)
b = sol.zero_mean_project_dual(sp, torch.rand(sp.n_dofs, dtype=torch.float64, device="cuda"))
diag = ops.laplace_diagonal(sp, bcs)
cfg = sol.ChebyshevConfig(5, 20.0, 3.0)
run = lambda: sol.laplace_pcg(sp, bcs, b, project_dual=True, cheb=cfg, diag=diag, rel_tol=0, max_iter=50)
run(); torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
out = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", "c2_trace.json")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    run(); torch.cuda.synchronize()
prof.export_chrome_trace(out)
tr = json.load(open(out))
agg, cnt = collections.Counter(), collections.Counter()
tot = 0.0
for e in tr["traceEvents"]:
    if e.get("cat") != "kernel":
        continue
    key = (e["name"][:80], tuple(e.get("args", {}).get("grid", [])))
    agg[key] += e["dur"]; cnt[key] += 1; tot += e["dur"]
print("total kernel us %.0f for 50 iterations" % tot)
for k, v in agg.most_common(15):
    print("%5.1f%% %9.1f us %5d x %7.2f us  %s %s" % (100 * v / tot, v, cnt[k], v / cnt[k], k[1], k[0]))
