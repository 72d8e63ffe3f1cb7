"""Times the fused Chebyshev-step vmults: C2 (32^3 Q4) Chebyshev-Jacobi PCG,
100 iterations, and 64x32x32 Q3 (the C4 fine level) Chebyshev(5) smoothing
applications (CUDA events).  Run once with DG_EXP=16 (no bulk L2 prefetch of
the epilogue vectors) and once without for the A/B."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_1607_01323_b200 import mesh as M, operators as ops, solvers as sol
from paper_1607_01323_b200.spaces import DgSpace


def timed(f, reps):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


mesh = M.build_box_mesh(((0, 1),) * 3, (32, 32, 32), periodic=(True, False, True))
sp = DgSpace(mesh, 4)
bcs = ops.BoundarySpec({"ymin": ops.DirichletBC(None), "ymax": ops.DirichletBC(None)}).resolve(sp)
b = sol.zero_mean_project_dual(sp, torch.rand(sp.n_dofs, dtype=torch.float64, device="cuda"))
diag = ops.laplace_diagonal(sp, bcs)
cfg = sol.ChebyshevConfig(5, 20.0, 3.0)
ms = timed(lambda: sol.laplace_pcg(sp, bcs, b, project_dual=True, cheb=cfg, diag=diag, rel_tol=0,
                                   max_iter=100), 3)
print("DG_EXP=%s C2 PCG %.4f ms/iteration" % (os.environ.get("DG_EXP", "0"), ms / 100))
mesh = M.build_box_mesh(((0, 2 * np.pi), (-1, 1), (0, np.pi)), (64, 32, 32),
                        grading=(0.0, 1.8, 0.0), periodic=(True, False, True))
sp = DgSpace(mesh, 3)
bcs = ops.BoundarySpec({"ymin": ops.NeumannBC(None, None), "ymax": ops.NeumannBC(None, None)}).resolve(sp)
diag = ops.laplace_diagonal(sp, bcs)
r = torch.rand(sp.n_dofs, dtype=torch.float64, device="cuda")
for b in ("0",):
    ms = timed(lambda: sol.laplace_chebyshev_smooth(sp, bcs, diag, cfg, r), 20)
    print("DG_EXP=%s brick %s Q3 64x32x32 Chebyshev(5) %.4f ms (%.1f us per fused step)" % (
        os.environ.get("DG_EXP", "0"), b, ms, ms * 1e3 / 4))
