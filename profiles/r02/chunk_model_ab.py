"""A/B of the z-chunk models of the column kernels (DG_CHUNK_MODEL is read per
call: 0 = wave model, unset = list-scheduling model): whole-slab vmult of the
interior C5 x-slab of P ranks (Q4) and cubes, CUDA events, interleaved rounds."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1607_01323_b200 import mesh as M, _lib
from paper_1607_01323_b200.parallel import SlabPartition
from paper_1607_01323_b200.spaces import DeviceContext
from paper_1607_01323_b200.operators import ctypes_ptr
P = lambda t: ctypes_ptr(t.data_ptr())


def timeit(f, reps):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


cases = [("C5 P=%d slab" % p, (128, 128, 128), p) for p in (1, 2, 4, 8)]
cases += [("%d^3" % n, (n, n, n), 1) for n in (48, 64, 96, 160)]
for name, counts, nranks in cases:
    mesh = M.build_box_mesh(((0, 1),) * 3, counts)
    part = SlabPartition(counts[0], nranks, False)
    c = DeviceContext(mesh, 4, (_lib.BC_VELOCITY_DIRICHLET,) * 6, 0,
                      part.range(1) if nranks > 1 else None)
    keep = []
    if nranks > 1:
        cnt = ctypes.c_int64()
        _lib.call("dg_halo_count", c.handle, ctypes.byref(cnt))
        keep = [torch.zeros(cnt.value, dtype=torch.float64, device="cuda") for _ in range(2)]
        _lib.call("dg_halo_attach", c.handle, P(keep[0]), P(keep[1]))
    n = c.n_dofs
    src = torch.rand(n, dtype=torch.float64, device="cuda") * 2 - 1
    dst = torch.empty_like(src)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    f = lambda: _lib.call("dg_laplace_vmult_part", c.handle, P(src), P(dst), 1.0, 0, st)
    best, outs = {}, {}
    for rnd in range(3):
        for tag, env in (("wave", "0"), ("list", None)):
            if env is None:
                os.environ.pop("DG_CHUNK_MODEL", None)
            else:
                os.environ["DG_CHUNK_MODEL"] = env
            f(); f()
            torch.cuda.synchronize()
            t = timeit(f, 40 if n < 1e8 else 15)
            best[tag] = min(best.get(tag, 1e9), t)
            outs[tag] = dst.clone()
    os.environ.pop("DG_CHUNK_MODEL", None)
    same = torch.equal(outs["wave"], outs["list"])
    print(f"{name:14s} wave {best['wave']:.4f} ms  list {best['list']:.4f} ms  "
          f"({100 * (best['wave'] / best['list'] - 1):+.1f} %)  bitwise equal {same}", flush=True)
