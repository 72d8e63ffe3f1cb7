"""C5 sharded Jacobi-PCG iteration (1 rank) with a per-kernel breakdown
(CUDA events): python cg_c5.py [cells] [k]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1607_01323_b200 import mesh as M, _lib
from paper_1607_01323_b200.parallel import SlabLaplace, SlabPCG
n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
k = int(sys.argv[2]) if len(sys.argv) > 2 else 4
mesh = M.build_box_mesh(((0, 1),) * 3, (n, n, n))
op = SlabLaplace(mesh, k, (_lib.BC_VELOCITY_DIRICHLET,) * 6, 0, 1)
src = torch.rand(op.n_dofs, dtype=torch.float64, device="cuda")
s = SlabPCG(op, op.diagonal(), project_dual=True)
s.start(src, rel_tol=0.0)
for _ in range(3):
    s.step()
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(20):
    s.step()
ev[1].record(); torch.cuda.synchronize()
it = ev[0].elapsed_time(ev[1]) / 20
# component timings
def t(f, reps=20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f(); torch.cuda.synchronize(); a.record()
    for _ in range(reps): f()
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b) / reps
o = s.ops; sc = s.scal
print({"ms_iter": round(it, 3), "gdofs_iter": round(op.n_dofs / it / 1e6, 1),
       "vmult": round(t(lambda: op.vmult(s.p, s.Lp)), 3),
       "dots": round(t(lambda: o.dots(s.p, s.Lp, sc[1:])), 3),
       "update": round(t(lambda: o.update(s.x, s.r, s.p, s.Lp, sc, True, s.diag, s.z, sc[4:])), 3),
       "pupdate": round(t(lambda: o.pupdate(s.p, s.z, sc)), 3)})
