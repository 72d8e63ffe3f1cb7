import sys
import torch
sys.path.insert(0, ".")
from paper_1607_01323_b200 import mesh as M, operators as ops
from paper_1607_01323_b200.spaces import DgSpace
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
k = int(sys.argv[2]) if len(sys.argv) > 2 else 3
mesh = M.build_box_mesh(((0, 1),) * 3, (n, n, n), periodic=(True, False, True))
space = DgSpace(mesh, k)
bcs = ops.BoundarySpec({"ymin": ops.DirichletBC(None), "ymax": ops.DirichletBC(None)}).resolve(space)
x3 = torch.rand(3 * space.n_dofs, dtype=torch.float64, device="cuda")
for _ in range(2):
    y = ops.apply_viscous_helmholtz(space, x3, 1500.0, 1 / 180, bcs)
torch.cuda.synchronize()
