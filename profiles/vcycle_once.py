"""One config-4 V-cycle (64x32x32 Q3 channel hierarchy, 6 levels) after a
warm-up, bracketed by cudaProfilerStart/Stop for ncu launch lists; also
prints the CUDA-event time of 20 V-cycles."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1607_01323_b200 import multigrid as MG, operators as ops, solvers as sol
from paper_1607_01323_b200.spaces import DgSpace

meshes = MG.box_mesh_hierarchy(((0, 2 * np.pi), (-1, 1), (0, np.pi)), (2, 1, 1), 5,
                               grading=(0.0, 1.8, 0.0), periodic=(True, False, True))
spaces = [DgSpace(m, 3) for m in meshes]
spec = ops.BoundarySpec({"ymin": ops.DirichletBC(None), "ymax": ops.DirichletBC(None)})
mg = MG.MultigridHierarchy(spaces, spec, project=sol.zero_mean_project)
print("levels", mg.n_levels, "coarse iters", mg.levels[0].coarse_iters,
      "dofs", [lv.space.n_dofs for lv in mg.levels])
b = torch.rand(spaces[-1].n_dofs, dtype=torch.float64, device="cuda")
for _ in range(3):
    x = mg.vcycle(b)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    x = mg.vcycle(b)
e1.record()
torch.cuda.synchronize()
print(f"V-cycle {e0.elapsed_time(e1) / 20:.3f} ms")
torch.cuda.cudart().cudaProfilerStart()
x = mg.vcycle(b)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
