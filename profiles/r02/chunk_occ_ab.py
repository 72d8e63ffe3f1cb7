"""A/B of the z-chunk rule of the column kernels with several CTAs per SM (Q3,
Q5): 4-wave rule (default) vs list-scheduling model capped at the 4-wave
length (default; DG_CHUNK_MODEL=0 = the rule, read per call)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1607_01323_b200 import mesh as M, operators as ops
from paper_1607_01323_b200.spaces import DgSpace


def timeit(f, reps):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for counts, k in (((64, 64, 64), 3), ((96, 96, 96), 3), ((64, 32, 32), 3), ((128, 128, 128), 3),
                  ((48, 48, 48), 5), ((64, 64, 64), 5), ((96, 96, 96), 5)):
    mesh = M.build_box_mesh(((0, 1),) * 3, counts)
    sp = DgSpace(mesh, k)
    bcs = ops.BoundarySpec({t: ops.DirichletBC(None) for t in mesh.boundary_tags()}).resolve(sp)
    src = torch.rand(sp.n_dofs, dtype=torch.float64, device="cuda") * 2 - 1
    dst = torch.empty_like(src)
    import ctypes
    from paper_1607_01323_b200 import _lib
    h = sp.ctx(bcs.kinds).handle
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    f = lambda: _lib.call("dg_laplace_vmult", h, ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(dst.data_ptr()), 1.0, st)
    best, outs = {}, {}
    for rnd in range(3):
        for tag, env in (("rule", "0"), ("list", None)):
            if env is None:
                os.environ.pop("DG_CHUNK_MODEL", None)
            else:
                os.environ["DG_CHUNK_MODEL"] = env
            f(); f()
            torch.cuda.synchronize()
            t = timeit(f, 40)
            best[tag] = min(best.get(tag, 1e9), t)
            outs[tag] = dst.clone()
    os.environ.pop("DG_CHUNK_MODEL", None)
    print(f"{counts} Q{k}: rule {best['rule']:.4f} ms ({sp.n_dofs / best['rule'] / 1e6:.1f} GDoF/s)  "
          f"list {best['list']:.4f} ms ({100 * (best['rule'] / best['list'] - 1):+.1f} %)  "
          f"equal {torch.equal(outs['rule'], outs['list'])}", flush=True)
