"""A/B of the C3 convective kernel configurations (32^3 periodic Q5, n_q = 8,
Taylor-Green + 1e-2 noise, seed 2): DG_VCONV_CFG per call, same process,
interleaved rounds; outputs checked against configuration 0."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_1607_01323_b200 import mesh as M, operators as ops
from paper_1607_01323_b200.spaces import DgSpace

cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["0", "1", "2", "3", "4"]
mesh = M.build_box_mesh(((0, 2 * np.pi),) * 3, (32, 32, 32), periodic=(True, True, True))
space = DgSpace(mesh, 5, n_q_over=8)
x, y, z = space.node_coords()
rng = np.random.default_rng(2)
u = np.stack([np.sin(x) * np.cos(y) * np.cos(z), -np.cos(x) * np.sin(y) * np.cos(z), 0 * z])
u = u + 1e-2 * rng.uniform(-1, 1, u.shape)
ud = torch.as_tensor(u.ravel(), device="cuda")
bcs = ops.BoundarySpec({}).resolve(space)
f = lambda: ops.eval_convective_rhs(space, bcs, [ud], (1.0,), (0.0,), 0.0)
ref = None
res = {c: [] for c in cfgs}
for rnd in range(3):
    for c in cfgs:
        os.environ["DG_VCONV_CFG"] = c
        y = f()
        torch.cuda.synchronize()
        if ref is None:
            ref = y.clone()
        err = float((y - ref).norm() / ref.norm())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            f()
        e1.record()
        torch.cuda.synchronize()
        res[c].append((e0.elapsed_time(e1) / 10, err))
for c in cfgs:
    print("cfg %s: %s ms (err %.1e)" % (c, " ".join("%.3f" % t for t, _ in res[c]), res[c][-1][1]))
