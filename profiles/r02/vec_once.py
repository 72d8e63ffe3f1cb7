"""One application of each C4 vector operator (64x32x32 Q3 channel): viscous
Helmholtz, projection (div-div + continuity penalty), one fused M^-1-PCG
iteration pair and one MG Chebyshev smoothing step -- the ncu target."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_1607_01323_b200 import mesh as M, operators as ops, solvers as sol
from paper_1607_01323_b200.spaces import DgSpace

mesh = M.build_box_mesh(((0, 2 * np.pi), (-1, 1), (0, np.pi)), (64, 32, 32),
                        grading=(0.0, 1.8, 0.0), periodic=(True, False, True))
sp = DgSpace(mesh, 3)
bcs = ops.BoundarySpec({"ymin": ops.DirichletBC(None), "ymax": ops.DirichletBC(None)}).resolve(sp)
u = torch.rand(3 * sp.n_dofs, dtype=torch.float64, device="cuda")
tau_d = torch.rand(mesh.n_elements, dtype=torch.float64, device="cuda")
tau_c = torch.rand(3 * mesh.n_elements, dtype=torch.float64, device="cuda")
for _ in range(2):
    h = ops.apply_viscous_helmholtz(sp, u, 1500.0, 1 / 180, bcs)
    p = ops.apply_projection_operator(sp, u, tau_d, tau_c)
    x, st = sol.helmholtz_pcg(sp, bcs, h, 1500.0, 1 / 180, rel_tol=1e-30, max_iter=2)
torch.cuda.synchronize()
print("ok", float(h.norm()), float(p.norm()), st.iterations)
