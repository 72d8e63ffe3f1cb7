"""Laplace vmult timing ablations (CUDA events, 30 reps after warm-up).
DG_EXP bits (timing experiments only, results are wrong when set):
1 skip halo loads, 2 skip face lifts, 4 skip halo steps A/B.
Usage: DG_EXP=<bits> DG_LAP_VARIANT=<v> python profiles/lap_ablate.py [cells] [k]"""
import os
import sys
import torch
sys.path.insert(0, ".")
from paper_1607_01323_b200 import mesh as M, operators as ops
from paper_1607_01323_b200.spaces import DgSpace

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
k = int(sys.argv[2]) if len(sys.argv) > 2 else 4
mesh = M.build_box_mesh(((0, 1),) * 3, (n, n, n))
space = DgSpace(mesh, k)
bcs = ops.BoundarySpec({t: ops.DirichletBC(None) for t in mesh.boundary_tags()}).resolve(space)
x = torch.rand(space.n_dofs, dtype=torch.float64, device="cuda")
f = lambda: ops.apply_pressure_laplace(space, x, bcs)
for _ in range(3):
    f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(30):
    f()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 30
print(f"exp={os.environ.get('DG_EXP', '0'):>2s} var={os.environ.get('DG_LAP_VARIANT', '-'):>3s} "
      f"{n}^3 Q{k}: {ms:7.3f} ms {space.n_dofs / ms / 1e6:7.1f} GDoF/s")
