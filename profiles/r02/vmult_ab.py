"""In-process A/B of Laplace vmult kernels (DG_LAP_VARIANT / DG_L7CFG are read
per call): for each (cells, k) case, every configuration is timed with CUDA
events in interleaved rounds; prints the best GDoF/s per configuration and
checks every configuration's output against the default kernel's.
usage: vmult_ab.py "cells,k ..." "variant:cfg ..." """
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1607_01323_b200 import mesh as M, operators as ops
from paper_1607_01323_b200.spaces import DgSpace

cases = [tuple(map(int, a.split(","))) for a in (sys.argv[1] if len(sys.argv) > 1 else "128,4 64,3 96,3").split()]
cfgs = (sys.argv[2] if len(sys.argv) > 2 else "0:0 7:0 7:1").split()

def setcfg(c):
    v, k = c.split(":")
    os.environ["DG_LAP_VARIANT"] = v
    os.environ["DG_L7CFG"] = k

res = {}
for cells, k in cases:
    mesh = M.build_box_mesh(((0, 1),) * 3, (cells,) * 3)
    sp = DgSpace(mesh, k)
    bcs = ops.BoundarySpec({t: ops.DirichletBC(None) for t in mesh.boundary_tags()}).resolve(sp)
    g = torch.Generator(device="cuda").manual_seed(4)
    x = torch.rand(sp.n_dofs, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    setcfg(cfgs[0]); ref = ops.apply_pressure_laplace(sp, x, bcs)
    best = {c: 1e9 for c in cfgs}
    err = {}
    reps = max(3, int(2e9 / sp.n_dofs / 8))
    for rnd in range(4):
        for c in cfgs:
            setcfg(c)
            y = ops.apply_pressure_laplace(sp, x, bcs)
            if rnd == 0:
                err[c] = float(((y - ref).norm() / ref.norm()).item())
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                y = ops.apply_pressure_laplace(sp, x, bcs)
            b.record(); torch.cuda.synchronize()
            best[c] = min(best[c], a.elapsed_time(b) / reps)
    res[f"{cells}^3 Q{k}"] = {c: (round(sp.n_dofs / best[c] / 1e6, 1), f"{err[c]:.1e}") for c in cfgs}
    print(f"{cells}^3 Q{k}", res[f"{cells}^3 Q{k}"], flush=True)
print(json.dumps(res))
