"""Small invocations of every device operator family (usable under
compute-sanitizer memcheck / racecheck where the pool allows it; not on
this build's pool): Cartesian Laplace (k = 2..5, walls and
periodic), Helmholtz / projection / convective fast paths, the vector PCG,
the general 2D path (cylinder-like refined hierarchy is not needed: a warped
box through GeneralSpace2D), the fp64 and fp32 V-cycles."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1607_01323_b200 import mesh as M, operators as ops, solvers as sol, multigrid as MG
from paper_1607_01323_b200.spaces import DgSpace

for k in (2, 3, 4, 5):
    mesh = M.build_box_mesh(((0, 1), (0, 2), (0, 1)), (3, 4, 5), periodic=(True, False, False))
    space = DgSpace(mesh, k)
    bcs = ops.BoundarySpec({"ymin": ops.DirichletBC(None), "ymax": ops.NeumannBC(None, None),
                            "zmin": ops.DirichletBC(None), "zmax": ops.DirichletBC(None)}).resolve(space)
    p = torch.rand(space.n_dofs, dtype=torch.float64, device="cuda")
    u = torch.rand(3 * space.n_dofs, dtype=torch.float64, device="cuda")
    ops.apply_pressure_laplace(space, p, bcs)
    ops.laplace_diagonal(space, bcs)
    ops.apply_viscous_helmholtz(space, u, 10.0, 0.1, bcs)
    ne = mesh.n_elements
    ops.apply_projection_operator(space, u, torch.rand(ne, dtype=torch.float64, device="cuda"),
                                  torch.rand(3 * ne, dtype=torch.float64, device="cuda"))
    ops.eval_convective_rhs(space, bcs, [u, u], (2.0, -1.0), (0.1, 0.0), 0.2)
    sol.helmholtz_pcg(space, bcs, u, 10.0, 0.1, rel_tol=1e-6, max_iter=5)
meshes = MG.box_mesh_hierarchy(((0, 1),) * 3, (2, 2, 2), 2, periodic=(True, False, True))
spaces = [DgSpace(m, 3) for m in meshes]
spec = ops.BoundarySpec({"ymin": ops.DirichletBC(None), "ymax": ops.DirichletBC(None)})
b = torch.rand(spaces[-1].n_dofs, dtype=torch.float64, device="cuda")
b = sol.zero_mean_project_dual(spaces[-1], b)
for prec in ("fp64", "fp32"):
    mg = MG.MultigridHierarchy(spaces, spec, project=sol.zero_mean_project, precision=prec)
    MG.laplace_pcg_mg(mg, b, project_dual=True, rel_tol=1e-6, max_iter=5)
torch.cuda.synchronize()
print("sanitize-ops done")
