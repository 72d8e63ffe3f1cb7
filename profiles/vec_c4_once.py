"""One viscous Helmholtz vmult and one projection vmult at config-4 size
(64x32x32 Q3, graded walls) and one config-3 convective term (32^3 Q5,
n_q = 8), after warm-up, for ncu captures of the Cartesian vector kernels."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1607_01323_b200 import mesh as M, operators as ops
from paper_1607_01323_b200.spaces import DgSpace

mesh = M.build_box_mesh(((0, 2 * np.pi), (-1, 1), (0, np.pi)), (64, 32, 32),
                        grading=(0.0, 1.8, 0.0), periodic=(True, False, True))
space = DgSpace(mesh, 3)
bcs = ops.BoundarySpec({"ymin": ops.DirichletBC(None), "ymax": ops.DirichletBC(None)}).resolve(space)
u = torch.rand(3 * space.n_dofs, dtype=torch.float64, device="cuda")
ne = mesh.n_elements
td = torch.rand(ne, dtype=torch.float64, device="cuda") * 0.01
tc = torch.rand(3 * ne, dtype=torch.float64, device="cuda") * 0.01
m3 = M.build_box_mesh(((0, 2 * np.pi),) * 3, (32, 32, 32), periodic=(True, True, True))
s3 = DgSpace(m3, 5)
u3 = torch.rand(3 * s3.n_dofs, dtype=torch.float64, device="cuda")
b3 = ops.BoundarySpec({}).resolve(s3)
for _ in range(3):
    ops.apply_viscous_helmholtz(space, u, 1500.0, 1 / 180, bcs)
    ops.apply_projection_operator(space, u, td, tc)
    ops.eval_convective_rhs(s3, b3, [u3], (1.0,), (0.0,), 0.0)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
ops.apply_viscous_helmholtz(space, u, 1500.0, 1 / 180, bcs)
ops.apply_projection_operator(space, u, td, tc)
ops.eval_convective_rhs(s3, b3, [u3], (1.0,), (0.0,), 0.0)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
