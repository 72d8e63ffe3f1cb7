"""x-slab domain decomposition over ranks (one process per GPU).

The reference is single-process; the paper's MPI
partitioning is replaced here by x-slabs of the structured box: rank r owns
cells [x_r, x_{r+1}) x all y x all z.  The only data-path exchange of the
SIP vmult is one ghost cell layer per slab face (owner-computed face data of
the neighbour), moved with point-to-point send/recv (NCCL over NVLink on
GPUs, gloo on CPU in the tests) and overlapped with the interior cells;
CG inner products are one all-reduce of the partial sums.

The exchange helpers are backend-agnostic (torch.distributed tensors); the
device-side pieces are the C ABI calls dg_halo_pack / dg_halo_attach /
dg_laplace_vmult_part.
"""

import ctypes
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib


@dataclass(frozen=True)
class SlabPartition:
    """Balanced split of nx cell layers over nranks (x-slabs)."""
    nx: int
    nranks: int
    periodic: bool

    def __post_init__(self):
        if self.nranks < 1 or self.nranks > self.nx:
            raise ValueError(f"cannot split {self.nx} x-layers over {self.nranks} ranks")

    def range(self, rank):
        base, extra = divmod(self.nx, self.nranks)
        a = rank * base + min(rank, extra)
        return a, a + base + (1 if rank < extra else 0)

    def neighbours(self, rank):
        """(lo, hi) neighbour ranks; None across a non-periodic boundary;
        a single rank on a periodic axis wraps locally (no exchange)."""
        if self.nranks == 1:
            return None, None
        lo = rank - 1 if rank > 0 else (self.nranks - 1 if self.periodic else None)
        hi = rank + 1 if rank < self.nranks - 1 else (0 if self.periodic else None)
        return lo, hi


def exchange_halos(send_lo, send_hi, recv_lo, recv_hi, lo_rank, hi_rank, group=None):
    """Send our first/last layer to the lo/hi neighbour and receive theirs.

    Messages between a pair of ranks are matched in issue order (NCCL has no
    tags).  Convention: sends are issued lo-layer first, receives hi-side
    first.  A peer's lo layer lands in our recv_hi (we are its lo
    neighbour) and its hi layer in our recv_lo, so with two ranks on a
    periodic axis (lo == hi) both messages still pair correctly.
    """
    import torch.distributed as dist
    ops = []
    if lo_rank is not None:
        ops.append(dist.P2POp(dist.isend, send_lo, lo_rank, group))
    if hi_rank is not None:
        ops.append(dist.P2POp(dist.isend, send_hi, hi_rank, group))
    if hi_rank is not None:
        ops.append(dist.P2POp(dist.irecv, recv_hi, hi_rank, group))
    if lo_rank is not None:
        ops.append(dist.P2POp(dist.irecv, recv_lo, lo_rank, group))
    if not ops:
        return []
    return dist.batch_isend_irecv(ops)


class SlabLaplace:
    """SIP Laplace vmult on this rank's x-slab with overlapped halo exchange.

    ``mesh`` is the GLOBAL box mesh; ``bc_kinds`` the per-tag kinds tuple
    (ResolvedBCs.kinds).  Vectors are this rank's element-major slab
    (cells ix in [a, b), local numbering ix-a + nxl*(iy + ny*iz)).
    """

    def __init__(self, mesh, k, bc_kinds, rank, nranks, group=None):
        import torch
        from .spaces import DeviceContext
        self.part = SlabPartition(mesh.counts[0], nranks, bool(mesh.periodic[0]))
        self.rank, self.nranks, self.group = rank, nranks, group
        self.range = self.part.range(rank)
        self.lo, self.hi = self.part.neighbours(rank)
        slab = self.range if nranks > 1 else None
        self.ctx = DeviceContext(mesh, k, bc_kinds, 0, slab)
        cnt = ctypes.c_int64()
        _lib.call("dg_halo_count", self.ctx.handle, ctypes.byref(cnt))
        self.halo_count = cnt.value
        dev = dict(dtype=torch.float64, device="cuda")
        self.send = [torch.empty(self.halo_count, **dev) for _ in range(2)]
        self.recv = [torch.zeros(self.halo_count, **dev) for _ in range(2)]
        self.has = [self.lo is not None, self.hi is not None]
        P = lambda t, on: ctypes.c_void_p(t.data_ptr() if on else 0)
        _lib.call("dg_halo_attach", self.ctx.handle, P(self.recv[0], self.has[0]),
                  P(self.recv[1], self.has[1]))
        self.comm = torch.cuda.Stream()
        self.n_dofs = self.ctx.n_dofs

    def vmult(self, src, dst, tau_scale=1.0):
        """dst = L src on this slab (interior cells overlap the exchange)."""
        import torch
        P = lambda t: ctypes.c_void_p(t.data_ptr())
        main = torch.cuda.current_stream()
        h = self.ctx.handle
        if self.nranks == 1:
            _lib.call("dg_laplace_vmult", h, P(src), P(dst), float(tau_scale),
                      ctypes.c_void_p(main.cuda_stream))
            return dst
        self.comm.wait_stream(main)
        with torch.cuda.stream(self.comm):
            _lib.call("dg_halo_pack", h, P(src),
                      ctypes.c_void_p(self.send[0].data_ptr() if self.has[0] else 0),
                      ctypes.c_void_p(self.send[1].data_ptr() if self.has[1] else 0),
                      ctypes.c_void_p(self.comm.cuda_stream))
            for r in exchange_halos(self.send[0], self.send[1], self.recv[0], self.recv[1],
                                    self.lo, self.hi, self.group):
                r.wait()
        _lib.call("dg_laplace_vmult_part", h, P(src), P(dst), float(tau_scale), 1,
                  ctypes.c_void_p(main.cuda_stream))
        main.wait_stream(self.comm)
        _lib.call("dg_laplace_vmult_part", h, P(src), P(dst), float(tau_scale), 2,
                  ctypes.c_void_p(main.cuda_stream))
        return dst


def allreduce_sum(t, group=None):
    """In-place sum over ranks (CG inner products)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def slab_of(global_field, part: SlabPartition, rank, counts, n_local):
    """Element-major global field -> this rank's slab (host numpy)."""
    a, b = part.range(rank)
    nz = counts[2] if len(counts) == 3 else 1
    g = np.asarray(global_field).reshape(nz, counts[1], counts[0], n_local)
    return np.ascontiguousarray(g[:, :, a:b]).ravel()
