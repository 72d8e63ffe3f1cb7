"""Times the C4 vector operators (64x32x32 Q3 channel) in one process: viscous
Helmholtz apply, projection apply, and 20 fused M^-1-PCG iterations of each
(CUDA events, after warm-up)."""
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
g = torch.Generator(device="cuda").manual_seed(0)
u = torch.rand(3 * sp.n_dofs, dtype=torch.float64, device="cuda", generator=g)
tau_d = torch.rand(mesh.n_elements, dtype=torch.float64, device="cuda", generator=g)
tau_c = torch.rand(3 * mesh.n_elements, dtype=torch.float64, device="cuda", generator=g)


def timed(f, reps=20):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


h = ops.apply_viscous_helmholtz(sp, u, 1500.0, 1 / 180, bcs)
p = ops.apply_projection_operator(sp, u, tau_d, tau_c)
print("helmholtz apply %.1f us  |h| %.15e" % (1e3 * timed(lambda: ops.apply_viscous_helmholtz(sp, u, 1500.0, 1 / 180, bcs)), float(h.norm())))
print("projection apply %.1f us  |p| %.15e" % (1e3 * timed(lambda: ops.apply_projection_operator(sp, u, tau_d, tau_c)), float(p.norm())))
print("helmholtz pcg 20 its %.2f ms" % timed(lambda: sol.helmholtz_pcg(sp, bcs, h, 1500.0, 1 / 180, rel_tol=1e-30, max_iter=20), 3))
print("projection pcg 20 its %.2f ms" % timed(lambda: sol.projection_pcg(sp, p, tau_d, tau_c, rel_tol=1e-30, max_iter=20), 3))
