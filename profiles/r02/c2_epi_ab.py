"""C2 (32^3 Q4) Chebyshev(5,20)-Jacobi PCG, 100 fixed iterations, per Q4
column-epilogue configuration (DG_EPI_CFG read per call), interleaved
rounds, best ms per iteration; the solution checked against config 0."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1607_01323_b200 import mesh as M, operators as ops, solvers as sol
from paper_1607_01323_b200.spaces import DgSpace
cfgs = (sys.argv[1] if len(sys.argv) > 1 else "0 1 2").split()
mesh = M.build_box_mesh(((0, 1),) * 3, (32, 32, 32), periodic=(True, False, True))
sp = DgSpace(mesh, 4)
bcs = ops.BoundarySpec({"ymin": ops.DirichletBC(None), "ymax": ops.DirichletBC(None)}).resolve(sp)
b = sol.zero_mean_project_dual(sp, torch.rand(sp.n_dofs, dtype=torch.float64, device="cuda"))
diag = ops.laplace_diagonal(sp, bcs)
cfg = sol.ChebyshevConfig(5, 20.0, 3.0)
best, xs = {c: 1e9 for c in cfgs}, {}
for rnd in range(3):
    for c in cfgs:
        os.environ["DG_EPI_CFG"] = c
        run = lambda: sol.laplace_pcg(sp, bcs, b, project_dual=True, cheb=cfg, diag=diag, rel_tol=0, max_iter=100)
        x, _ = run(); torch.cuda.synchronize()
        xs[c] = x
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); run(); e1.record(); torch.cuda.synchronize()
        best[c] = min(best[c], e0.elapsed_time(e1) / 100)
ref = xs[cfgs[0]]
print({c: (round(best[c], 4), f"{float((xs[c] - ref).norm() / ref.norm()):.1e}") for c in cfgs})
