"""Throughput of the individual device operators at a given size (CUDA
events, inputs larger than L2).  Usage: python profiles/op_throughput.py [cells] [k]"""
import sys
import torch
sys.path.insert(0, ".")
from paper_1607_01323_b200 import mesh as M, operators as ops
from paper_1607_01323_b200.spaces import DgSpace

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
k = int(sys.argv[2]) if len(sys.argv) > 2 else 4
mesh = M.build_box_mesh(((0, 1),) * 3, (n, n, n))
space = DgSpace(mesh, k)
bcs = ops.BoundarySpec({t: ops.DirichletBC(None) for t in mesh.boundary_tags()}).resolve(space)
nd = space.n_dofs
x = torch.rand(nd, dtype=torch.float64, device="cuda")
x3 = torch.rand(3 * nd, dtype=torch.float64, device="cuda")


def timeit(f, reps=30):
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


y = torch.empty_like(x)
for name, f, dofs in [
    ("copy (torch)", lambda: y.copy_(x), nd),
    ("laplace", lambda: ops.apply_pressure_laplace(space, x, bcs), nd),
    ("mass", lambda: ops.mass_apply(space, x), nd),
    ("inverse_mass", lambda: ops.inverse_mass_apply(space, x), nd),
    ("helmholtz", lambda: ops.apply_viscous_helmholtz(space, x3, 1500.0, 1 / 180, bcs), 3 * nd),
    ("convective", lambda: ops.eval_convective_rhs(space, bcs, [x3], (1.0,), (0.0,), 0.0), 3 * nd),
]:
    ms = timeit(f)
    print(f"{name:14s} {ms:8.3f} ms  {dofs / ms / 1e6:8.2f} GDoF/s  {16 * dofs / ms / 1e6:8.1f} GB/s(16B/DoF)")
