"""A/B of the column kernels' z-chunk rule (DG_CHUNK_OLD=1 per call: about 4
waves; default: the wave-quantisation model of dgmf.cu chunk_len) on whole
meshes and on the interior x-slab of P ranks of the C5 mesh; interleaved
rounds in one process, outputs compared."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_1607_01323_b200 import mesh as M, _lib, operators as ops
from paper_1607_01323_b200.parallel import SlabPartition
from paper_1607_01323_b200.spaces import DgSpace, DeviceContext
from paper_1607_01323_b200.operators import ctypes_ptr

P = lambda t: ctypes_ptr(t.data_ptr())


def timed(f, reps=20):
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


cases = []
for n, k in ((128, 4), (96, 4), (64, 4), (48, 4), (32, 4), (64, 3), (96, 3), (64, 5), (48, 5)):
    mesh = M.build_box_mesh(((0, 1),) * 3, (n, n, n))
    sp = DgSpace(mesh, k)
    bcs = ops.BoundarySpec({t: ops.DirichletBC(None) for t in mesh.boundary_tags()}).resolve(sp)
    x = torch.rand(sp.n_dofs, dtype=torch.float64, device="cuda")
    cases.append((f"{n}^3 Q{k}", sp.n_dofs, lambda sp=sp, x=x, bcs=bcs: ops.apply_pressure_laplace(sp, x, bcs)))
mesh = M.build_box_mesh(((0, 2 * np.pi), (-1, 1), (0, np.pi)), (64, 32, 32), grading=(0.0, 1.8, 0.0),
                        periodic=(True, False, True))
sp = DgSpace(mesh, 3)
bcs = ops.BoundarySpec({"ymin": ops.DirichletBC(None), "ymax": ops.DirichletBC(None)}).resolve(sp)
xc = torch.rand(sp.n_dofs, dtype=torch.float64, device="cuda")
cases.append(("C4 fine 64x32x32 Q3", sp.n_dofs, lambda: ops.apply_pressure_laplace(sp, xc, bcs)))
mesh = M.build_box_mesh(((0, 1),) * 3, (128, 128, 128))
keep = []
for nranks in (2, 4, 8):
    part = SlabPartition(128, nranks, False)
    c = DeviceContext(mesh, 4, (_lib.BC_VELOCITY_DIRICHLET,) * 6, 0, part.range(1))
    cnt = ctypes.c_int64()
    _lib.call("dg_halo_count", c.handle, ctypes.byref(cnt))
    x0, x1 = part.range(1)
    nloc = (x1 - x0) * 128 * 128 * 125
    src = torch.rand(nloc, dtype=torch.float64, device="cuda")
    dst = torch.empty_like(src)
    rcv = [torch.rand(cnt.value, dtype=torch.float64, device="cuda") for _ in range(2)]
    _lib.call("dg_halo_attach", c.handle, P(rcv[0]), P(rcv[1]))
    keep.append((c, src, dst, rcv))
    cases.append((f"slab P={nranks}", nloc, lambda c=c, src=src, dst=dst: (_lib.call(
        "dg_laplace_vmult_part", c.handle, P(src), P(dst), 1.0, 0,
        ctypes_ptr(torch.cuda.current_stream().cuda_stream)), dst)[1]))
for name, nd, f in cases:
    res = {}
    outs = {}
    for rnd in range(3):
        for mode in ("old", "new"):
            if mode == "old":
                os.environ["DG_CHUNK_OLD"] = "1"
            else:
                os.environ.pop("DG_CHUNK_OLD", None)
            res.setdefault(mode, []).append(timed(f))
            outs[mode] = f().clone()
    err = float((outs["old"] - outs["new"]).norm() / outs["old"].norm())
    to, tn = min(res["old"]), min(res["new"])
    print(f"{name:22s} old {to:.4f} ms ({nd / to / 1e6:.1f} GDoF/s)  new {tn:.4f} ms "
          f"({nd / tn / 1e6:.1f} GDoF/s)  {to / tn:.3f}x  diff {err:.0e}", flush=True)
