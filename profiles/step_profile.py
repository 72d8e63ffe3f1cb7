"""BASELINE config 4: one dual-splitting step on the turbulent-channel box
(64 x 32 x 32 cells, Q3, y graded with grading_map(s, 1.8), periodic x/z,
no-slip walls), nu = 1/180, dt = 1e-3, BDF2, variant V4 (zeta* = 1, CFL = 1);
u0 = (1 - y^2, 0, 0) + 0.1 U(-1, 1) (seed 3), history [u0, u0].
Reports wall time per step and per substep and the solver iterations.
Usage: python profiles/step_profile.py [variant] [steps] [fused]"""
import sys
import time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1607_01323_b200 import multigrid as MG, operators as ops, stepper as S
from paper_1607_01323_b200.spaces import DgSpace

variant = sys.argv[1] if len(sys.argv) > 1 else "V4"
nsteps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
fused = (sys.argv[3] != "0") if len(sys.argv) > 3 else True
meshes = MG.box_mesh_hierarchy(((0, 2 * np.pi), (-1, 1), (0, np.pi)), (2, 1, 1), 5,
                               grading=(0.0, 1.8, 0.0), periodic=(True, False, True))
spaces = [DgSpace(m, 3) for m in meshes]
spec = ops.BoundarySpec({"ymin": ops.DirichletBC(None), "ymax": ops.DirichletBC(None)})
cfg = S.StepConfig(dt=1e-3, nu=1 / 180, J=2, variant=ops.VariantConfig(variant))
t0 = time.perf_counter()
vc = S.VelocityCorrection(spaces, spec, cfg, fused=fused)
torch.cuda.synchronize()
print(f"C4 {variant}: {spaces[-1].mesh.counts} cells Q3, {3 * spaces[-1].n_dofs} velocity DoFs, "
      f"MG levels {vc.mg.n_levels}, setup {time.perf_counter() - t0:.2f} s")
x, y, z = spaces[-1].node_coords()
rng = np.random.default_rng(3)
u0 = np.stack([1 - y ** 2, 0 * y, 0 * y]) + 0.1 * rng.uniform(-1, 1, (3,) + y.shape)
u0 = torch.as_tensor(u0.ravel(), device="cuda")
w0 = ops.compute_vorticity(spaces[-1], u0)
hu, hp, hw = [u0, u0], [], [w0, w0]
for n in range(nsteps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = vc.step(hu, hp, hw, n * 1e-3)
    torch.cuda.synchronize()
    dt = 1e3 * (time.perf_counter() - t0)
    print(f"step {n}: {dt:8.1f} ms  substeps " +
          ", ".join(f"{k} {v:.1f}" for k, v in r.times_ms.items()) + "  iterations " + str(r.iters))
    hu, hp, hw = [r.u, hu[0]], [r.p] + hp[:1], [r.w, hw[0]]
