import os, sys, ctypes
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1607_01323_b200 import mesh as M, operators as ops, solvers as sol, _lib
from paper_1607_01323_b200.spaces import DgSpace
n_ = int(sys.argv[1]) if len(sys.argv) > 1 else 8
mesh = M.build_box_mesh(((0, 1),) * 3, (n_, n_, n_), periodic=(True, False, True))
space = DgSpace(mesh, 4)
bcs = ops.BoundarySpec({"ymin": ops.DirichletBC(None), "ymax": ops.DirichletBC(None)}).resolve(space)
b = sol.zero_mean_project_dual(space, torch.rand(space.n_dofs, dtype=torch.float64, device="cuda"))
diag = ops.laplace_diagonal(space, bcs)
cfg = sol.ChebyshevConfig(5, 20.0, 3.0)
orig = _lib.check
def chk(rc):
    if rc: print("rc", rc, "msg", repr(_lib.lib().dg_last_error()))
    orig(rc)
_lib.check = chk
x, st = sol.laplace_pcg(space, bcs, b, project_dual=True, cheb=cfg, diag=diag, rel_tol=1e-10, max_iter=50)
print(st.iterations, st.converged)
