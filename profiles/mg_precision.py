"""fp64 vs fp32 V-cycle (dg_mg_set_precision): V-cycle time and MG-PCG
iterations / time at config 4 (64x32x32 Q3 channel, 6 levels) and config 2
(32^3 Q4 pure Neumann, 4 levels).  Usage: python profiles/mg_precision.py"""
import sys
import time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1607_01323_b200 import multigrid as MG, operators as ops, solvers as sol
from paper_1607_01323_b200.spaces import DgSpace


def run(name, meshes, k, spec, singular):
    spaces = [DgSpace(m, k) for m in meshes]
    proj = sol.zero_mean_project if singular else None
    top = spaces[-1]
    b = torch.rand(top.n_dofs, dtype=torch.float64, device="cuda") - 0.5
    if singular:
        b = sol.zero_mean_project_dual(top, b)
    for prec in ("fp64", "fp32"):
        mg = MG.MultigridHierarchy(spaces, spec, project=proj, precision=prec)
        for _ in range(3):
            mg.vcycle(b)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            mg.vcycle(b)
        e1.record()
        torch.cuda.synchronize()
        vc = e0.elapsed_time(e1) / 20
        MG.laplace_pcg_mg(mg, b, project_dual=singular, rel_tol=1e-10)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x, st = MG.laplace_pcg_mg(mg, b, project_dual=singular, rel_tol=1e-10)
        torch.cuda.synchronize()
        ms = 1e3 * (time.perf_counter() - t0)
        print(f"{name} {prec}: V-cycle {vc:.3f} ms, MG-PCG {st.iterations} it {ms:.1f} ms")


m4 = MG.box_mesh_hierarchy(((0, 2 * np.pi), (-1, 1), (0, np.pi)), (2, 1, 1), 5,
                           grading=(0.0, 1.8, 0.0), periodic=(True, False, True))
run("C4", m4, 3, ops.BoundarySpec({"ymin": ops.DirichletBC(None), "ymax": ops.DirichletBC(None)}),
    True)
m2 = MG.box_mesh_hierarchy(((0, 1),) * 3, (4, 4, 4), 3, periodic=(True, False, True))
run("C2", m2, 4, ops.BoundarySpec({"ymin": ops.DirichletBC(None), "ymax": ops.DirichletBC(None)}),
    True)
