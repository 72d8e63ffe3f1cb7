"""C5 (128^3 Q4 walls) CG-step pieces on one GPU: vmult, vmult + dg_cg_dots,
fused dg_laplace_vmult_dots; and the SlabPCG Jacobi iteration with / without
the fused launch (DG_NO_DOTS_FUSED is read at the first call: run twice)."""
import ctypes
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1607_01323_b200 import _lib, mesh as M, operators as ops
from paper_1607_01323_b200.parallel import SlabLaplace, SlabPCG
from paper_1607_01323_b200.spaces import DgSpace

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
mesh = M.build_box_mesh(((0, 1),) * 3, (n, n, n))
space = DgSpace(mesh, 4)
bcs = ops.BoundarySpec({t: ops.DirichletBC(None) for t in mesh.boundary_tags()}).resolve(space)
lap = SlabLaplace(mesh, 4, bcs.kinds, 0, 1)
g = torch.Generator(device="cuda").manual_seed(4)
p = torch.rand(space.n_dofs, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
Lp = torch.empty_like(p)
s = torch.zeros(3, dtype=torch.float64, device="cuda")
P = lambda t: ctypes.c_void_p(t.data_ptr())
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
h = lap.ctx.handle


def timeit(f, reps=30):
    for _ in range(5):
        f()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def unfused():
    _lib.call("dg_laplace_vmult", h, P(p), P(Lp), 1.0, st)
    _lib.call("dg_cg_dots", h, P(p), P(Lp), P(s), st)


for rnd in range(2):
    t0 = timeit(lambda: _lib.call("dg_laplace_vmult", h, P(p), P(Lp), 1.0, st))
    t1 = timeit(unfused)
    s1 = s.cpu().numpy().copy()
    t2 = timeit(lambda: _lib.call("dg_laplace_vmult_dots", h, P(p), P(Lp), 1.0, P(s), st))
    s2 = s.cpu().numpy().copy()
    print(f"vmult {t0:.3f} ms | vmult + dots {t1:.3f} ms | fused {t2:.3f} ms | sums {s1} vs {s2}")

diag = lap.diagonal()
b = torch.rand(space.n_dofs, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
pcg = SlabPCG(lap, diag)
pcg.start(b, rel_tol=1e-30)
for _ in range(3):
    pcg.step()
t = timeit(pcg.step, 20)
print(f"SlabPCG Jacobi iteration {t:.3f} ms ({space.n_dofs / t / 1e6:.1f} GDoF/s per iteration)")
