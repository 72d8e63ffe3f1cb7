"""One config-4 step after a warm-up step (for ncu launch lists)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1607_01323_b200 import multigrid as MG, operators as ops, stepper as S
from paper_1607_01323_b200.spaces import DgSpace
meshes = MG.box_mesh_hierarchy(((0, 2 * np.pi), (-1, 1), (0, np.pi)), (2, 1, 1), 5,
                               grading=(0.0, 1.8, 0.0), periodic=(True, False, True))
spaces = [DgSpace(m, 3) for m in meshes]
spec = ops.BoundarySpec({"ymin": ops.DirichletBC(None), "ymax": ops.DirichletBC(None)})
vc = S.VelocityCorrection(spaces, spec, S.StepConfig(dt=1e-3, nu=1 / 180, J=2,
                                                     variant=ops.VariantConfig("V4")))
x, y, z = spaces[-1].node_coords()
u0 = np.stack([1 - y ** 2, 0 * y, 0 * y]) + 0.1 * np.random.default_rng(3).uniform(-1, 1, (3,) + y.shape)
u0 = torch.as_tensor(u0.ravel(), device="cuda")
w0 = ops.compute_vorticity(spaces[-1], u0)
r = vc.step([u0, u0], [], [w0, w0], 0.0)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
r = vc.step([r.u, u0], [r.p], [r.w, w0], 1e-3)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print(r.times_ms, r.iters)
