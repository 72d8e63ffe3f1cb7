"""x-slab vmult (interior slab of P ranks of the C5 mesh, 128^3 Q4 walls,
ghost traces from device buffers) per Q4 column-kernel configuration
(DG_LAP_VARIANT=8, DG_L7CFG read per call): the whole-slab phase of the split
vmult and the ghost-lift phase, best of 3 rounds of 20 calls."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1607_01323_b200 import mesh as M, _lib
from paper_1607_01323_b200.parallel import SlabPartition
from paper_1607_01323_b200.spaces import DeviceContext
from paper_1607_01323_b200.operators import ctypes_ptr

cfgs = (sys.argv[1] if len(sys.argv) > 1 else "0 6").split()
n, k = 128, 4
P = lambda t: ctypes_ptr(t.data_ptr())
os.environ["DG_LAP_VARIANT"] = os.environ.get("SLAB_VARIANT", "8")
for nranks in (1, 2, 4, 8):
    mesh = M.build_box_mesh(((0, 1),) * 3, (n, n, n))
    part = SlabPartition(n, nranks, False)
    r = 1 if nranks > 1 else 0
    kinds = (_lib.BC_VELOCITY_DIRICHLET,) * 6
    c = DeviceContext(mesh, k, kinds, 0, part.range(r))
    cnt = ctypes.c_int64()
    _lib.call("dg_halo_count", c.handle, ctypes.byref(cnt))
    x0, x1 = part.range(r)
    nloc = (x1 - x0) * n * n * (k + 1) ** 3
    src = torch.rand(nloc, dtype=torch.float64, device="cuda")
    dst = torch.empty_like(src)
    if cnt.value:
        rcv = [torch.rand(cnt.value, dtype=torch.float64, device="cuda") for _ in range(2)]
        _lib.call("dg_halo_attach", c.handle, P(rcv[0]), P(rcv[1]))
    st = ctypes_ptr(torch.cuda.current_stream().cuda_stream)
    best = {cf: [1e9, 1e9] for cf in cfgs}
    outs = {}
    for rnd in range(3):
        for cf in cfgs:
            os.environ["DG_L7CFG"] = cf
            for ph in ((1, 2) if nranks > 1 else (0,)):
                if nranks > 1:
                    f = lambda: _lib.call("dg_laplace_vmult_split", c.handle, P(src), P(dst), 1.0, ph, st)
                else:
                    f = lambda: _lib.call("dg_laplace_vmult", c.handle, P(src), P(dst), 1.0, st)
                f(); torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(20):
                    f()
                b.record(); torch.cuda.synchronize()
                i = 0 if ph in (0, 1) else 1
                best[cf][i] = min(best[cf][i], a.elapsed_time(b) / 20)
            if rnd == 0:
                if nranks > 1:
                    _lib.call("dg_laplace_vmult_split", c.handle, P(src), P(dst), 1.0, 1, st)
                    _lib.call("dg_laplace_vmult_split", c.handle, P(src), P(dst), 1.0, 2, st)
                torch.cuda.synchronize()
                outs[cf] = dst.clone()
    ref = outs[cfgs[0]]
    print(f"P={nranks} slab {x1-x0}x{n}x{n}: " + " | ".join(
        f"cfg {cf}: phase1 {best[cf][0]:.3f} phase2 {best[cf][1] if nranks > 1 else 0:.3f} ms "
        f"(diff {float((outs[cf] - ref).norm() / ref.norm()):.1e})" for cf in cfgs), flush=True)
