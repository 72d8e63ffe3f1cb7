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


class TorchComm:
    """Communicator of the x-slab path over torch.distributed (NCCL between
    GPUs, gloo on CPU): point-to-point ghost exchange and fp64 sum
    all-reduce of CG partial sums."""

    def __init__(self, group=None):
        self.group = group

    def exchange(self, send_lo, send_hi, recv_lo, recv_hi, lo, hi):
        for r in exchange_halos(send_lo, send_hi, recv_lo, recv_hi, lo, hi, self.group):
            r.wait()

    def allreduce(self, t):
        return allreduce_sum(t, self.group)


class ThreadComm:
    """Ranks emulated by host threads of one process on ONE GPU (tests): each
    rank's kernels run on its own stream; exchanges and all-reduces meet at a
    host barrier after a stream synchronize, so no kernel ever waits on
    another rank's kernel.  ``view(rank)`` is the per-rank communicator."""

    def __init__(self, world):
        import threading
        self.world = world
        self.bar = threading.Barrier(world)
        self.slots = [None] * world

    def view(self, rank):
        return _ThreadRankComm(self, rank)


class _ThreadRankComm:
    def __init__(self, shared, rank):
        self.c, self.rank = shared, rank

    def exchange(self, send_lo, send_hi, recv_lo, recv_hi, lo, hi):
        import torch
        c = self.c
        torch.cuda.current_stream().synchronize()
        c.slots[self.rank] = (send_lo, send_hi)
        c.bar.wait()
        if lo is not None:
            recv_lo.copy_(c.slots[lo][1])  # the lo neighbour's last layer
        if hi is not None:
            recv_hi.copy_(c.slots[hi][0])  # the hi neighbour's first layer
        torch.cuda.current_stream().synchronize()
        c.bar.wait()

    def allreduce(self, t):
        import torch
        c = self.c
        torch.cuda.current_stream().synchronize()
        c.slots[self.rank] = t.clone()
        c.bar.wait()
        tot = c.slots[0].clone()
        for r in range(1, c.world):  # fixed rank order
            tot += c.slots[r]
        torch.cuda.current_stream().synchronize()
        c.bar.wait()
        t.copy_(tot)
        return t


class SlabLaplace:
    """SIP Laplace vmult on this rank's x-slab with overlapped halo exchange.

    ``mesh`` is the GLOBAL box mesh; ``bc_kinds`` the per-tag kinds tuple
    (ResolvedBCs.kinds).  Vectors are this rank's element-major slab
    (cells ix in [a, b), local numbering ix-a + nxl*(iy + ny*iz)).  The ghost
    payload is what dg_halo_pack writes: owner-computed face traces (value and
    x-derivative at the face points, 2 n^2 doubles per cell) for Q3-Q5, whole
    cells otherwise.  ``comm``: TorchComm (default) or a ThreadComm view.
    """

    def __init__(self, mesh, k, bc_kinds, rank, nranks, group=None, comm=None):
        import torch
        from .spaces import DeviceContext
        self.part = SlabPartition(mesh.counts[0], nranks, bool(mesh.periodic[0]))
        self.rank, self.nranks, self.group = rank, nranks, group
        self.comm_ops = comm if comm is not None else TorchComm(group)
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
        self.traced = mesh.dim == 3 and 3 <= k <= 5  # ghost payload: face traces
        self.n_dofs = self.ctx.n_dofs
        self.volume = float(np.prod([v[-1] - v[0] for v in mesh.axis_vertices[:mesh.dim]]))

    def vmult(self, src, dst, tau_scale=1.0, overlap=None):
        """dst = L src on this slab, the ghost exchange overlapped with the
        slab's own work.  Traced ghosts (Q3-Q5): ONE launch over the whole
        slab on zero ghost traces while the traces move, then the ghost-trace
        face terms on the boundary x-layers (dg_laplace_vmult_split; the
        operator is linear in the ghost data).  Other degrees: the columns
        that touch no ghost side while the traces move, the rest after
        (dg_laplace_vmult_part 1 / 2) -- splitting the column launch itself
        costs more than the exchange at Q4 (profiles/r02/slab_parts.py).
        ``overlap`` False: exchange first, then one launch (part 0)."""
        import torch
        P = lambda t: ctypes.c_void_p(t.data_ptr())
        main = torch.cuda.current_stream()
        h = self.ctx.handle
        ms = ctypes.c_void_p(main.cuda_stream)
        if self.nranks == 1:
            _lib.call("dg_laplace_vmult", h, P(src), P(dst), float(tau_scale), ms)
            return dst
        self.comm.wait_stream(main)
        with torch.cuda.stream(self.comm):
            _lib.call("dg_halo_pack", h, P(src),
                      ctypes.c_void_p(self.send[0].data_ptr() if self.has[0] else 0),
                      ctypes.c_void_p(self.send[1].data_ptr() if self.has[1] else 0),
                      ctypes.c_void_p(self.comm.cuda_stream))
            self.comm_ops.exchange(self.send[0], self.send[1], self.recv[0], self.recv[1],
                                   self.lo, self.hi)
        if overlap is None:
            overlap = True
        if overlap and self.traced:
            _lib.call("dg_laplace_vmult_split", h, P(src), P(dst), float(tau_scale), 1, ms)
            main.wait_stream(self.comm)
            _lib.call("dg_laplace_vmult_split", h, P(src), P(dst), float(tau_scale), 2, ms)
            return dst
        if overlap:
            _lib.call("dg_laplace_vmult_part", h, P(src), P(dst), float(tau_scale), 1, ms)
        main.wait_stream(self.comm)
        _lib.call("dg_laplace_vmult_part", h, P(src), P(dst), float(tau_scale),
                  2 if overlap else 0, ms)
        return dst

    def vmult_dots(self, p, Lp, tau_scale, out3):
        """Lp = L p with the rank-local [p.Lp, sum(Lp), p.w] in out3 (device):
        one fused launch on a single rank (dg_laplace_vmult_dots); x-slab
        ranks run the overlapped vmult, then dg_cg_dots."""
        import torch
        P = lambda t: ctypes.c_void_p(t.data_ptr())
        ms = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        h = self.ctx.handle
        if self.nranks == 1:
            _lib.call("dg_laplace_vmult_dots", h, P(p), P(Lp), float(tau_scale), P(out3), ms)
        elif self.traced:
            # as vmult(): traces move on the side stream during phase 1
            main = torch.cuda.current_stream()
            self.comm.wait_stream(main)
            with torch.cuda.stream(self.comm):
                _lib.call("dg_halo_pack", h, P(p),
                          ctypes.c_void_p(self.send[0].data_ptr() if self.has[0] else 0),
                          ctypes.c_void_p(self.send[1].data_ptr() if self.has[1] else 0),
                          ctypes.c_void_p(self.comm.cuda_stream))
                self.comm_ops.exchange(self.send[0], self.send[1], self.recv[0], self.recv[1],
                                       self.lo, self.hi)
            _lib.call("dg_laplace_vmult_split_dots", h, P(p), P(Lp), float(tau_scale), 1,
                      P(out3), ms)
            main.wait_stream(self.comm)
            _lib.call("dg_laplace_vmult_split_dots", h, P(p), P(Lp), float(tau_scale), 2,
                      P(out3), ms)
        else:
            self.vmult(p, Lp, tau_scale)
            _lib.call("dg_cg_dots", h, P(p), P(Lp), P(out3), ms)
        return Lp

    def diagonal(self, tau_scale=1.0):
        """Exact Jacobi diagonal of this slab (operators.py:675-730)."""
        import torch
        d = torch.empty(self.n_dofs, dtype=torch.float64, device="cuda")
        _lib.call("dg_laplace_diagonal", self.ctx.handle, ctypes.c_void_p(d.data_ptr()),
                  float(tau_scale), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        return d


class SlabPCG:
    """The reference pcg (solvers.py:30-73) sharded over x-slabs, one rank per
    GPU: op = L or zero_mean_project_dual o L (``project_dual``, folded
    algebraically: pAp = p.Lp - (sum(Lp)/|Omega|) p.w and r -= alpha (Lp -
    c w)), prec = point Jacobi (``cheb`` None) or chebyshev_smooth(L, diag,
    cheb) (solvers.py:93-129) with the slab vmult.  Each iteration: one slab
    vmult (ghost exchange overlapped with interior columns), dg_cg_dots,
    one all-reduce of [p.Lp, sum(Lp), p.w], dg_cg_update (x, r and, for
    Jacobi, z and r.z in one pass), one all-reduce of r.z, the stop test on
    the host, dg_cg_pupdate.  No torch or cuBLAS kernels in the loop; the
    iteration count and sqrt(r.z) history follow the reference exactly."""

    def __init__(self, lap, diag, cheb=None, project_dual=False, tau_scale=1.0, ops=None):
        import torch
        self.lap, self.diag, self.cheb = lap, diag, cheb
        self.project, self.ts = bool(project_dual), float(tau_scale)
        self.ops = ops if ops is not None else DeviceSlabOps(lap)
        n = lap.n_dofs
        dev = dict(dtype=torch.float64, device=diag.device)
        self.r, self.z, self.p, self.Lp = (torch.empty(n, **dev) for _ in range(4))
        if cheb is not None:
            if cheb.degree <= 0:
                raise ValueError("Chebyshev degree must be >= 1 inside the sharded PCG")
            self.rc, self.d, self.d2, self.Ld = (torch.empty(n, **dev) for _ in range(4))
        self.scal = torch.zeros(8, **dev)
        self.comm = lap.comm_ops

    def _precondition(self):
        """z = chebyshev_smooth(L, diag, cheb, r) from x = 0 (solvers.py:93-129)."""
        cfg, ops = self.cheb, self.ops
        lmax = cfg.lambda_max
        lmin = lmax / cfg.smoothing_range
        theta, delta = 0.5 * (lmax + lmin), 0.5 * (lmax - lmin)
        sigma1 = theta / delta
        rho = 1.0 / sigma1
        ops.cheb_init(self.r, self.diag, self.rc, self.d, self.z, theta)
        d, d2 = self.d, self.d2
        for _ in range(cfg.degree - 1):
            rho_new = 1.0 / (2.0 * sigma1 - rho)
            a, b = rho_new * rho, 2.0 * rho_new / delta
            self.lap.vmult(d, self.Ld, self.ts)
            ops.cheb_step(self.rc, self.Ld, d, d2, self.diag, self.z, a, b)
            d, d2 = d2, d
            rho = rho_new

    def _rz(self):
        """z = prec(r) and the REDUCED r.z in scal[4]."""
        sc = self.scal
        if self.cheb is None:
            sc[1:4].zero_()  # pAp = 0: no x/r update, only z = r/diag and r.z
            self.ops.update(self.r, self.r, self.r, self.r, sc, False, self.diag, self.z, sc[4:])
        else:
            self._precondition()
            self.ops.dot(self.r, self.z, sc[4:])
        self.comm.allreduce(sc[4:5])

    def start(self, b, x=None, rel_tol=1e-8, abs_tol=0.0):
        """Set up the solve of op x = b from x = 0 (x: this rank's slab,
        overwritten); returns False when already converged or broken down."""
        import math
        import torch
        from .solvers import SolverStats
        sc = self.scal
        self.x = torch.zeros_like(b) if x is None else x.zero_()
        self.r.copy_(b)
        self._rz()
        rz = float(sc[4].item())
        self.it = 0
        if rz < 0:
            self.stats = SolverStats(0, math.sqrt(abs(rz)), False, True, [])
            return False
        norm0 = math.sqrt(rz)
        self.hist = [norm0]
        self.tol = max(rel_tol * norm0, abs_tol)
        self.norm = norm0
        if norm0 <= self.tol:
            self.stats = SolverStats(0, norm0, True, False, self.hist)
            return False
        self.p.copy_(self.z)
        sc[0].copy_(sc[4])
        self.stats = None
        return True

    def step(self):
        """One PCG iteration; returns False once the solve has stopped
        (self.stats then holds the outcome)."""
        import math
        from .solvers import SolverStats
        sc, ops = self.scal, self.ops
        self.it += 1
        it = self.it
        if hasattr(self.lap, "vmult_dots"):  # device slabs: fused on a single rank
            self.lap.vmult_dots(self.p, self.Lp, self.ts, sc[1:])
        else:
            self.lap.vmult(self.p, self.Lp, self.ts)
            ops.dots(self.p, self.Lp, sc[1:])
        self.comm.allreduce(sc[1:4])
        ops.update(self.x, self.r, self.p, self.Lp, sc, self.project,
                   self.diag if self.cheb is None else None, self.z, sc[4:])
        if self.cheb is not None:
            self._precondition()
            ops.dot(self.r, self.z, sc[4:])
        self.comm.allreduce(sc[4:5])
        pLp, sLp, pw, rz_new = sc[1:5].tolist()
        pAp = pLp - (sLp / self.lap.volume) * pw if self.project else pLp
        if pAp <= 0.0:
            self.stats = SolverStats(it, self.norm, False, True, self.hist)
            return False
        self.norm = math.sqrt(max(rz_new, 0.0))
        self.hist.append(self.norm)
        if self.norm <= self.tol:
            self.stats = SolverStats(it, self.norm, True, False, self.hist)
            return False
        if rz_new <= 0.0:
            self.stats = SolverStats(it, self.norm, False, True, self.hist)
            return False
        ops.pupdate(self.p, self.z, sc)
        return True

    def solve(self, b, x=None, rel_tol=1e-8, abs_tol=0.0, max_iter=1000):
        """x (this rank's slab) solving op x = b from x = 0; returns
        (x, SolverStats) with the reference's iteration count, flags and
        sqrt(r.z) history (identical on every rank)."""
        from .solvers import SolverStats
        if self.start(b, x, rel_tol, abs_tol):
            while self.it < max_iter and self.step():
                pass
            if self.stats is None:
                self.stats = SolverStats(max_iter, self.norm, False, False, self.hist)
        return self.x, self.stats


class DeviceSlabOps:
    """The rank-local vector kernels of SlabPCG: the C ABI of include/dgmf.h
    (dg_cg_dots / dg_cg_update / dg_cg_pupdate / dg_cheb_vec_* / dg_dot) on
    the slab context, on torch's current stream."""

    def __init__(self, lap):
        self.h, self.n = lap.ctx.handle, lap.n_dofs

    @staticmethod
    def _P(t):
        return ctypes.c_void_p(0 if t is None else t.data_ptr())

    @staticmethod
    def _st():
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def dots(self, p, Lp, out3):
        _lib.call("dg_cg_dots", self.h, self._P(p), self._P(Lp), self._P(out3), self._st())

    def update(self, x, r, p, Lp, scal, project, diag, z, out_rz):
        _lib.call("dg_cg_update", self.h, self._P(x), self._P(r), self._P(p), self._P(Lp),
                  self._P(scal), int(project), self._P(diag), self._P(z), self._P(out_rz),
                  self._st())

    def pupdate(self, p, z, scal):
        _lib.call("dg_cg_pupdate", self.h, self._P(p), self._P(z), self._P(scal), self._st())

    def dot(self, a, b, out):
        _lib.call("dg_dot", self.h, self._P(a), self._P(b), self.n, self._P(out), self._st())

    def cheb_init(self, r, diag, rc, d, x, theta):
        _lib.call("dg_cheb_vec_init", self.h, self._P(r), self._P(diag), self._P(rc), self._P(d),
                  self._P(x), float(theta), self._st())

    def cheb_step(self, rc, Ld, d_old, d_new, diag, x, a, b):
        _lib.call("dg_cheb_vec_step", self.h, self._P(rc), self._P(Ld), self._P(d_old),
                  self._P(d_new), self._P(diag), self._P(x), float(a), float(b), self._st())


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
