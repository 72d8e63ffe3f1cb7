"""Throughput of the quadrature-point operators (CUDA events, 10 reps):
Helmholtz, projection, convective (C3 rule), divergence, gradient, element-local
PCG.  Usage: python profiles/vec_throughput.py [cells] [k]"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1607_01323_b200 import mesh as M, operators as ops, solvers as sol
from paper_1607_01323_b200.spaces import DgSpace

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
k = int(sys.argv[2]) if len(sys.argv) > 2 else 4
mesh = M.build_box_mesh(((0, 1),) * 3, (n, n, n), periodic=(True, False, True))
space = DgSpace(mesh, k)
bcs = ops.BoundarySpec({"ymin": ops.DirichletBC(None), "ymax": ops.DirichletBC(None)}).resolve(space)
nd = space.n_dofs
x1 = torch.rand(nd, dtype=torch.float64, device="cuda")
x3 = torch.rand(3 * nd, dtype=torch.float64, device="cuda")
tau_d = torch.rand(space.mesh.n_elements, dtype=torch.float64, device="cuda")
tau_c = torch.rand(3 * space.mesh.n_elements, dtype=torch.float64, device="cuda")


def timeit(f, reps=10):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for name, f, dofs in [
    ("laplace", lambda: ops.apply_pressure_laplace(space, x1, bcs), nd),
    ("helmholtz", lambda: ops.apply_viscous_helmholtz(space, x3, 1500.0, 1 / 180, bcs), 3 * nd),
    ("projection", lambda: ops.apply_projection_operator(space, x3, tau_d, tau_c), 3 * nd),
    ("convective", lambda: ops.eval_convective_rhs(space, bcs, [x3, x3], (2.0, -1.0), (0., 0.), 0.), 3 * nd),
    ("divergence(weak)", lambda: ops.eval_divergence_rhs(space, x3, bcs, 1.0, "weak"), 3 * nd),
    ("gradient(weak)", lambda: ops.eval_pressure_gradient_rhs(space, x1, bcs, 1.0, "weak"), nd),
    ("vorticity", lambda: ops.compute_vorticity(space, x3), 3 * nd),
    ("element_local_pcg", lambda: sol.projection_element_pcg(space, x3, tau_d, rel_tol=1e-12), 3 * nd),
]:
    ms = timeit(f, 3 if "pcg" in name else 10)
    print(f"{name:18s} {ms:9.3f} ms  {dofs / ms / 1e6:8.3f} GDoF/s")
