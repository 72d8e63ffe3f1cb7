"""Config-2 PCG solve timing breakdown (used with ncu --metrics gpu__time_duration.sum)."""
import sys
import time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1607_01323_b200 import mesh as M, operators as ops, solvers as sol
from paper_1607_01323_b200.spaces import DgSpace

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
mesh = M.build_box_mesh(((0, 1),) * 3, (32, 32, 32), periodic=(True, False, True))
space = DgSpace(mesh, 4)
bcs = ops.BoundarySpec({"ymin": ops.DirichletBC(None), "ymax": ops.DirichletBC(None)}).resolve(space)
xn = space.node_coords()
f = np.sin(2 * np.pi * xn[0]) * np.cos(np.pi * xn[1]) * np.sin(2 * np.pi * xn[2])
f = f + 1e-3 * np.random.default_rng(1).standard_normal(f.shape)
b = sol.zero_mean_project_dual(space, ops.mass_apply(space, torch.as_tensor(f.ravel(), device="cuda")))
diag = ops.laplace_diagonal(space, bcs)
lmax = sol.lanczos_lambda_max(space, bcs, diag, project=True)
cfg = sol.ChebyshevConfig(5, 20.0, lmax)
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, st = sol.laplace_pcg(space, bcs, b, project_dual=True, cheb=cfg, diag=diag,
                            rel_tol=1e-10, max_iter=iters)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"iterations {st.iterations} converged {st.converged} wall {1e3*dt:.1f} ms "
          f"({1e3*dt/max(st.iterations,1):.3f} ms/it)")
