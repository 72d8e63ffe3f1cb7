"""A/B: v4 brick sizes for the small (multigrid coarse-level) Q3 meshes of C4,
vmults replayed from a CUDA graph (as inside the V-cycle graph); DG_V4SMALL
selects the brick per call (0: 4x4x2, 1: 2x2x2, 2: 2x2x1, 3: 1x1x1, 4: 4x2x2),
DG_LAP_VARIANT=7 the column kernel."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_1607_01323_b200 import mesh as M, operators as ops
from paper_1607_01323_b200.spaces import DgSpace

CFGS = [("v4 4x4x2", "4", "0"), ("v4 2x2x2", "4", "1"), ("v4 2x2x1", "4", "2"),
        ("v4 1x1x1", "4", "3"), ("v4 4x2x2", "4", "4"), ("column", "7", "0")]
for counts in ((4, 2, 2), (8, 4, 4), (16, 8, 8), (32, 16, 16), (64, 32, 32)):
    mesh = M.build_box_mesh(((0, 2 * np.pi), (-1, 1), (0, np.pi)), counts,
                            grading=(0.0, 1.8, 0.0), periodic=(True, False, True))
    sp = DgSpace(mesh, 3)
    bcs = ops.BoundarySpec({"ymin": ops.DirichletBC(None), "ymax": ops.DirichletBC(None)}).resolve(sp)
    x = torch.rand(sp.n_dofs, dtype=torch.float64, device="cuda")
    ref = None
    res = []
    for name, var, small in CFGS:
        os.environ["DG_LAP_VARIANT"], os.environ["DG_V4SMALL"] = var, small
        y = ops.apply_pressure_laplace(sp, x, bcs)
        torch.cuda.synchronize()
        if ref is None:
            ref = y.clone()
        err = float((y - ref).norm() / ref.norm())
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(3):
                ops.apply_pressure_laplace(sp, x, bcs)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(20):
                ops.apply_pressure_laplace(sp, x, bcs)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        res.append("%s %.2f us (err %.0e)" % (name, e0.elapsed_time(e1) / 200 * 1e3, err))
    print(counts, " | ".join(res), flush=True)
