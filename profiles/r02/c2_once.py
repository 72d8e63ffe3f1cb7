"""A few C2 (32^3 Q4) Chebyshev-Jacobi PCG iterations (launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_1607_01323_b200 import mesh as M, operators as ops, solvers as sol
from paper_1607_01323_b200.spaces import DgSpace
mesh = M.build_box_mesh(((0, 1),) * 3, (32, 32, 32), periodic=(True, False, True))
sp = DgSpace(mesh, 4)
bcs = ops.BoundarySpec({"ymin": ops.DirichletBC(None), "ymax": ops.DirichletBC(None)}).resolve(sp)
b = sol.zero_mean_project_dual(sp, torch.rand(sp.n_dofs, dtype=torch.float64, device="cuda"))
diag = ops.laplace_diagonal(sp, bcs)
cfg = sol.ChebyshevConfig(5, 20.0, 3.0)
for it in (3, 3):
    x, st = sol.laplace_pcg(sp, bcs, b, project_dual=True, cheb=cfg, diag=diag, rel_tol=0, max_iter=it)
torch.cuda.synchronize()
print("ok")
