"""Config-2 Poisson solve with the multigrid V-cycle preconditioner vs
Chebyshev(5,20)-Jacobi: iterations and device time (CUDA events).
Usage: python profiles/mg_profile.py [cells] [k] [base]"""
import sys
import time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1607_01323_b200 import mesh as M, operators as ops, solvers as sol, multigrid as MG
from paper_1607_01323_b200.spaces import DgSpace

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
k = int(sys.argv[2]) if len(sys.argv) > 2 else 4
base = int(sys.argv[3]) if len(sys.argv) > 3 else 4
levels = int(round(np.log2(n // base)))
meshes = MG.box_mesh_hierarchy(((0, 1),) * 3, (base,) * 3, levels, periodic=(True, False, True))
spaces = [DgSpace(m, k) for m in meshes]
spec = ops.BoundarySpec({"ymin": ops.DirichletBC(None), "ymax": ops.DirichletBC(None)})
space = spaces[-1]
bcs = spec.resolve(space)
xn = space.node_coords()
f = np.sin(2 * np.pi * xn[0]) * np.cos(np.pi * xn[1]) * np.sin(2 * np.pi * xn[2])
f = f + 1e-3 * np.random.default_rng(1).standard_normal(f.shape)
b = sol.zero_mean_project_dual(space, ops.mass_apply(space, torch.as_tensor(f.ravel(), device="cuda")))
torch.cuda.synchronize()
t0 = time.perf_counter()
mg = MG.MultigridHierarchy(spaces, spec, project=sol.zero_mean_project)
torch.cuda.synchronize()
print(f"{n}^3 Q{k}: {space.n_dofs} DoFs, {mg.n_levels} levels, setup {time.perf_counter()-t0:.2f} s, "
      f"coarse iters {mg.levels[0].coarse_iters}")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
x = mg.vcycle(b)
torch.cuda.synchronize()
e0.record()
for _ in range(10):
    x = mg.vcycle(b)
e1.record()
torch.cuda.synchronize()
print(f"vcycle {e0.elapsed_time(e1)/10:.3f} ms")
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, st = MG.laplace_pcg_mg(mg, b, project_dual=True, rel_tol=1e-10, max_iter=200)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"MG-PCG iterations {st.iterations} converged {st.converged} {1e3*dt:.1f} ms "
          f"({1e3*dt/max(st.iterations,1):.3f} ms/it)")
diag = ops.laplace_diagonal(space, bcs)
lmax = sol.lanczos_lambda_max(space, bcs, diag, project=True)
cfg = sol.ChebyshevConfig(5, 20.0, lmax)
torch.cuda.synchronize()
t0 = time.perf_counter()
x2, st2 = sol.laplace_pcg(space, bcs, b, project_dual=True, cheb=cfg, diag=diag, rel_tol=1e-10,
                          max_iter=5000)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"Chebyshev-PCG iterations {st2.iterations} {1e3*dt:.1f} ms; "
      f"rel diff of solutions {float((x - x2).norm() / x2.norm()):.2e}")
