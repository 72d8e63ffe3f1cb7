"""A/B of Q4 column-kernel configurations on the C5 x-slabs (interior slab of
P ranks, whole-slab launch): default laplace8<5,8,4,4,1> vs laplace7 tiles
(DG_LAP_VARIANT=7, DG_L7CFG per call)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1607_01323_b200 import mesh as M, _lib
from paper_1607_01323_b200.parallel import SlabPartition
from paper_1607_01323_b200.spaces import DeviceContext
from paper_1607_01323_b200.operators import ctypes_ptr
P = lambda t: ctypes_ptr(t.data_ptr())
mesh = M.build_box_mesh(((0, 1),) * 3, (128, 128, 128))
cfgs = [("laplace8 8x4", None, None), ("l7 <5,4,4,4,2>", "7", "4"), ("l7 <5,4,4,3,2>", "7", "2"),
        ("l7 <5,8,4,4,1>", "7", "1")]
for nranks in (1, 2, 4, 8):
    part = SlabPartition(128, nranks, False)
    c = DeviceContext(mesh, 4, (_lib.BC_VELOCITY_DIRICHLET,) * 6, 0, part.range(1) if nranks > 1 else None)
    if nranks > 1:
        cnt = ctypes.c_int64()
        _lib.call("dg_halo_count", c.handle, ctypes.byref(cnt))
        rcv = [torch.rand(cnt.value, dtype=torch.float64, device="cuda") for _ in range(2)]
        _lib.call("dg_halo_attach", c.handle, P(rcv[0]), P(rcv[1]))
    x0, x1 = part.range(1) if nranks > 1 else (0, 128)
    nloc = (x1 - x0) * 128 * 128 * 125
    src = torch.rand(nloc, dtype=torch.float64, device="cuda")
    dst = torch.empty_like(src)
    st = ctypes_ptr(torch.cuda.current_stream().cuda_stream)
    line = []
    ref = None
    for name, var, cfg in cfgs:
        for k_, v_ in (("DG_LAP_VARIANT", var), ("DG_L7CFG", cfg)):
            if v_ is None:
                os.environ.pop(k_, None)
            else:
                os.environ[k_] = v_
        f = lambda: _lib.call("dg_laplace_vmult_part", c.handle, P(src), P(dst), 1.0, 0, st)
        f(); torch.cuda.synchronize()
        if ref is None:
            ref = dst.clone()
        err = float((dst - ref).norm() / ref.norm())
        best = 1e9
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                f()
            b.record(); torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b) / 20)
        line.append(f"{name} {best:.4f} ms ({nloc / best / 1e6:.1f}) e{err:.0e}")
    print(f"P={nranks}: " + " | ".join(line), flush=True)
