"""2D Cartesian operator throughput (the reference's own dimension): Laplace,
Helmholtz, projection, convective on an n x n box, Q_k.
Usage: python profiles/vec2d_throughput.py [n] [k]"""
import sys
import torch
sys.path.insert(0, ".")
from paper_1607_01323_b200 import mesh as M, operators as ops
from paper_1607_01323_b200.spaces import DgSpace

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
k = int(sys.argv[2]) if len(sys.argv) > 2 else 3
mesh = M.build_box_mesh(((0, 1), (0, 1)), (n, n), periodic=(True, False))
space = DgSpace(mesh, k)
bcs = ops.BoundarySpec({"ymin": ops.DirichletBC(None), "ymax": ops.DirichletBC(None)}).resolve(space)
nd = space.n_dofs
p = torch.rand(nd, dtype=torch.float64, device="cuda")
u = torch.rand(2 * nd, dtype=torch.float64, device="cuda")
ne = mesh.n_elements
td = torch.rand(ne, dtype=torch.float64, device="cuda")
tc = torch.rand(2 * ne, dtype=torch.float64, device="cuda")


def t(f, reps=20):
    f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        f()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for name, f, d in (("laplace", lambda: ops.apply_pressure_laplace(space, p, bcs), nd),
                   ("helmholtz", lambda: ops.apply_viscous_helmholtz(space, u, 10.0, 0.01, bcs), 2 * nd),
                   ("projection", lambda: ops.apply_projection_operator(space, u, td, tc), 2 * nd),
                   ("convective", lambda: ops.eval_convective_rhs(space, bcs, [u], (1.0,), (0.0,), 0.0), 2 * nd),
                   ("inverse mass", lambda: ops.inverse_mass_apply(space, u), 2 * nd)):
    ms = t(f)
    print(f"2D {n}x{n} Q{k} {name:12s} {ms:8.3f} ms {d / ms / 1e6:8.2f} GDoF/s")
