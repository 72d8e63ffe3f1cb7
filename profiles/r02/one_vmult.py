"""Run a few Laplace vmults (for ncu captures): python one_vmult.py cells k [reps]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1607_01323_b200 import mesh as M, operators as ops
from paper_1607_01323_b200.spaces import DgSpace
cells, k = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
mesh = M.build_box_mesh(((0, 1),) * 3, (cells,) * 3)
sp = DgSpace(mesh, k)
bcs = ops.BoundarySpec({t: ops.DirichletBC(None) for t in mesh.boundary_tags()}).resolve(sp)
x = torch.rand(sp.n_dofs, dtype=torch.float64, device="cuda")
for _ in range(reps):
    y = ops.apply_pressure_laplace(sp, x, bcs)
torch.cuda.synchronize()
print("ok", y.norm().item())
