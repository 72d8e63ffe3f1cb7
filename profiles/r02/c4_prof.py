"""Diagnostic: kernel time breakdown of the C4 step (bench.run_c4_step setup)
from a CUPTI trace (torch.profiler) of one steady step -- real durations
inside the CUDA-graph replays, unlike ncu's serialised per-kernel replay.
Prints device time per (kernel, grid) and the step's wall time."""
import collections
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_1607_01323_b200 import multigrid as MG, operators as ops, stepper as S
from paper_1607_01323_b200.spaces import DgSpace

meshes = MG.box_mesh_hierarchy(((0, 2 * np.pi), (-1, 1), (0, np.pi)), (2, 1, 1), 5,
                               grading=(0.0, 1.8, 0.0), periodic=(True, False, True))
spaces = [DgSpace(m, 3) for m in meshes]
print("levels", [m.n_elements for m in meshes])
spec = ops.BoundarySpec({"ymin": ops.DirichletBC(None), "ymax": ops.DirichletBC(None)})
cfg = S.StepConfig(dt=1e-3, nu=1 / 180, J=2, variant=ops.VariantConfig("V4"))
vc = S.VelocityCorrection(spaces, spec, cfg)
x, y, z = spaces[-1].node_coords()
rng = np.random.default_rng(3)
u0 = np.stack([1 - y ** 2, 0 * y, 0 * y]) + 0.1 * rng.uniform(-1, 1, (3,) + y.shape)
u0 = torch.as_tensor(u0.ravel(), device="cuda")
w0 = ops.compute_vorticity(spaces[-1], u0)
hu, hp, hw = [u0, u0], [], [w0, w0]
for n in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = vc.step(hu, hp, hw, n * 1e-3)
    torch.cuda.synchronize()
    print("step", n, "%.2f ms" % (1e3 * (time.perf_counter() - t0)), r.iters,
          {k: round(v, 2) for k, v in r.times_ms.items()}, flush=True)
    hu, hp, hw = [r.u, hu[0]], [r.p] + hp[:1], [r.w, hw[0]]

from torch.profiler import profile, ProfilerActivity
out = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", "c4_trace.json")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    r = vc.step(hu, hp, hw, 3e-3)
    torch.cuda.synchronize()
print("profiled step", r.iters, {k: round(v, 2) for k, v in r.times_ms.items()})
prof.export_chrome_trace(out)
tr = json.load(open(out))
agg, cnt = collections.Counter(), collections.Counter()
tot = 0.0
for e in tr["traceEvents"]:
    if e.get("cat") != "kernel":
        continue
    g = tuple(e.get("args", {}).get("grid", []))
    key = (e["name"][:70], g)
    agg[key] += e["dur"]
    cnt[key] += 1
    tot += e["dur"]
print("total kernel us %.0f" % tot)
for k, v in agg.most_common(45):
    print("%5.1f%% %9.1f us %5d x %7.2f us  %s %s" % (100 * v / tot, v, cnt[k], v / cnt[k], k[1], k[0]))
