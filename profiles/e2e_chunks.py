"""e2e (pinned host in -> device -> host out) of apply_pressure_laplace at
128^3 Q4 for several chunk counts of the pipelined host-buffer path."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1607_01323_b200 import mesh as M, operators as ops
from paper_1607_01323_b200.spaces import DgSpace
n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
mesh = M.build_box_mesh(((0, 1),) * 3, (n, n, n))
space = DgSpace(mesh, 4)
bcs = ops.BoundarySpec({t: ops.DirichletBC(None) for t in mesh.boundary_tags()}).resolve(space)
h = torch.rand(space.n_dofs, dtype=torch.float64).pin_memory()
for ch in (1, 4, 8, 16, 32, 64):
    ops.HOST_CHUNKS = ch
    for _ in range(2):
        ops.apply_pressure_laplace(space, h, bcs)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        ops.apply_pressure_laplace(space, h, bcs)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"chunks {ch:3d}: {ms:7.2f} ms  {space.n_dofs / ms / 1e6:6.2f} GDoF/s")
