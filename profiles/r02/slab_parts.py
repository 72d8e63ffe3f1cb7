"""x-slab vmult parts on one GPU: the interior slab of P ranks of the C5 mesh
(128^3 Q4 walls), ghost traces filled by device copies; times part 1
(columns not touching a ghost side: overlaps the exchange), part 2 (the rest)
and the whole-mesh vmult of the same slab size.  DG_L8SLAB=1 selected (knob
removed after this measurement: 4x8 slower at every P)
4x8 tiles (x-narrow) for slab contexts."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_1607_01323_b200 import mesh as M, _lib, operators as ops
from paper_1607_01323_b200.parallel import SlabPartition
from paper_1607_01323_b200.spaces import DeviceContext
from paper_1607_01323_b200.operators import ctypes_ptr

n, k = 128, 4
P = lambda t: ctypes_ptr(t.data_ptr())
for nranks in (2, 4, 8):
    mesh = M.build_box_mesh(((0, 1),) * 3, (n, n, n))
    part = SlabPartition(n, nranks, False)
    r = 1 if nranks > 1 else 0
    kinds = (_lib.BC_VELOCITY_DIRICHLET,) * 6
    c = DeviceContext(mesh, k, kinds, 0, part.range(r))
    cnt = ctypes.c_int64()
    _lib.call("dg_halo_count", c.handle, ctypes.byref(cnt))
    nd = c.n_dofs if hasattr(c, "n_dofs") else None
    x0, x1 = part.range(r)
    nloc = (x1 - x0) * n * n * (k + 1) ** 3
    src = torch.rand(nloc, dtype=torch.float64, device="cuda")
    dst = torch.empty_like(src)
    rcv = [torch.rand(cnt.value, dtype=torch.float64, device="cuda") for _ in range(2)]
    _lib.call("dg_halo_attach", c.handle, P(rcv[0]), P(rcv[1]))
    st = ctypes_ptr(torch.cuda.current_stream().cuda_stream)
    res = []
    for var in ("0", "1"):
        os.environ["DG_L8SLAB"] = var
        def t(prt, reps=20):
            f = lambda: _lib.call("dg_laplace_vmult_part", c.handle, P(src), P(dst), 1.0, prt, st)
            f(); torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                f()
            b.record(); torch.cuda.synchronize()
            return a.elapsed_time(b) / reps
        t1, t2, t0 = t(1), t(2), t(0)
        def ts_(ph, reps=20):
            f = lambda: _lib.call("dg_laplace_vmult_split", c.handle, P(src), P(dst), 1.0, ph, st)
            f(); torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                f()
            b.record(); torch.cuda.synchronize()
            return a.elapsed_time(b) / reps
        if var == "0":
            print(f"  P={nranks} split phase 1 {ts_(1):.3f} ms, phase 2 {ts_(2):.4f} ms", flush=True)
        _lib.call("dg_laplace_vmult_part", c.handle, P(src), P(dst), 1.0, 1, st)
        _lib.call("dg_laplace_vmult_part", c.handle, P(src), P(dst), 1.0, 2, st)
        torch.cuda.synchronize()
        res.append((var, t1, t2, dst.clone(), t0))
    err = float((res[0][3] - res[1][3]).norm() / res[0][3].norm())
    print(f"P={nranks} slab {x1-x0}x{n}x{n}: " + " | ".join(
        f"tiles {'4x8' if v == '1' else '8x4'}: part1 {a:.3f} part2 {b:.3f} sum {a+b:.3f} whole {w:.3f} ms" for v, a, b, _, w in res)
        + f"  (rel diff {err:.1e})", flush=True)
