"""Krylov solvers on the GPU (reference pkg/src/dgins/solvers.py).

Two levels:

* Reference-compatible callables: ``pcg``, ``chebyshev_smooth``,
  ``eigen_estimate_via_cg``, ``zero_mean_project[_dual]`` with the
  reference signatures (solvers.py:30-198), operating on CUDA tensors
  (numpy inputs are moved to the device once).
* The fused hot path ``laplace_pcg``: the whole PCG loop for the SIP
  Laplacian with Chebyshev(degree, range)-over-Jacobi or Jacobi
  preconditioning runs in libdgmf (dg_laplace_pcg): device-resident vectors,
  deterministic reductions, one host read of two scalars per iteration.
"""

import ctypes
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _lib
from .operators import apply_pressure_laplace, laplace_diagonal, ctypes_ptr, _stream
from .spaces import _torch


@dataclass
class SolverStats:
    iterations: int
    residual: float
    converged: bool
    breakdown: bool = False
    history: list = field(default_factory=list)


@dataclass
class ChebyshevConfig:
    """solvers.py:76-90."""
    degree: int = 5
    smoothing_range: float = 20.0
    lambda_max: float = 1.0

    def __post_init__(self):
        if self.degree < 0:
            raise ValueError("Chebyshev degree must be >= 0")
        if self.smoothing_range <= 1.0:
            raise ValueError("smoothing range must exceed 1")


def _to_dev(x):
    torch = _torch()
    if isinstance(x, torch.Tensor):
        return x
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64)).to("cuda")


def _vdot(a, b):
    return float((a.reshape(-1) @ b.reshape(-1)).item())


def pcg(op: Callable, prec: Optional[Callable], b, x0=None, rel_tol: float = 1e-8,
        abs_tol: float = 0.0, max_iter: int = 1000):
    """Preconditioned CG with the reference semantics (solvers.py:30-73):
    stops when sqrt(r.z) <= max(rel_tol*sqrt(r0.z0), abs_tol); breakdown
    on nonpositive curvature; iterations = operator applications."""
    b = _to_dev(b)
    prec = prec or (lambda v: v.clone())
    if x0 is None:
        x = b.new_zeros(b.shape)
        r = b.clone()
    else:
        x = _to_dev(x0).clone()
        r = b - op(x)
    z = prec(r)
    rz = _vdot(r, z)
    if rz < 0:
        return x, SolverStats(0, float(np.sqrt(abs(rz))), False, True, [])
    norm0 = float(np.sqrt(rz))
    hist = [norm0]
    tol = max(rel_tol * norm0, abs_tol)
    if norm0 <= tol:
        return x, SolverStats(0, norm0, True, False, hist)
    p = z.clone()
    norm = norm0
    for it in range(1, max_iter + 1):
        Ap = op(p)
        pAp = _vdot(p, Ap)
        if pAp <= 0.0:
            return x, SolverStats(it, norm, False, True, hist)
        alpha = rz / pAp
        x += alpha * p
        r -= alpha * Ap
        z = prec(r)
        rz_new = _vdot(r, z)
        norm = float(np.sqrt(max(rz_new, 0.0)))
        hist.append(norm)
        if norm <= tol:
            return x, SolverStats(it, norm, True, False, hist)
        if rz_new <= 0.0:
            return x, SolverStats(it, norm, False, True, hist)
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, SolverStats(max_iter, norm, False, False, hist)


def chebyshev_smooth(op: Callable, diag, cfg: ChebyshevConfig, rhs, x=None,
                     degree: Optional[int] = None):
    """Chebyshev iteration on [lmax/range, lmax] (solvers.py:93-129)."""
    deg = cfg.degree if degree is None else degree
    rhs = _to_dev(rhs)
    diag = _to_dev(diag).reshape(rhs.shape)
    if x is None:
        x = rhs.new_zeros(rhs.shape)
        r = rhs.clone()
    else:
        x = _to_dev(x).clone()
        if deg == 0:
            return x
        r = rhs - op(x)
    if deg == 0:
        return x
    lmax = cfg.lambda_max
    lmin = lmax / cfg.smoothing_range
    theta = 0.5 * (lmax + lmin)
    delta = 0.5 * (lmax - lmin)
    sigma1 = theta / delta
    rho = 1.0 / sigma1
    d = (r / diag) / theta
    x += d
    for _ in range(deg - 1):
        r -= op(d)
        rho_new = 1.0 / (2.0 * sigma1 - rho)
        d = (rho_new * rho) * d + (2.0 * rho_new / delta) * (r / diag)
        rho = rho_new
        x += d
    return x


def chebyshev_error_factor(kappa: float, n: int) -> float:
    """Classic Chebyshev error bound 2 q^n, q = (sqrt(kappa)-1)/(sqrt(kappa)+1)
    (solvers.py:132-135); host arithmetic, the bound behind the coarse count."""
    q = (np.sqrt(kappa) - 1.0) / (np.sqrt(kappa) + 1.0)
    return float(2.0 * q ** n)


def eigen_estimate_via_cg(op: Callable, prec_diag, b, n_iter: int = 20):
    """Lanczos estimates from CG coefficients (solvers.py:138-176)."""
    b = _to_dev(b)
    diag = _to_dev(prec_diag).reshape(b.shape) if prec_diag is not None else None
    x = b.new_zeros(b.shape)
    r = b.clone()
    z = r / diag if diag is not None else r.clone()
    rz = _vdot(r, z)
    alphas, betas = [], []
    p = z.clone()
    for _ in range(n_iter):
        Ap = op(p)
        pAp = _vdot(p, Ap)
        if pAp <= 0 or rz <= 0:
            break
        alpha = rz / pAp
        alphas.append(alpha)
        x += alpha * p
        r -= alpha * Ap
        z = r / diag if diag is not None else r.clone()
        rz_new = _vdot(r, z)
        if rz_new <= 1e-30 * rz or rz_new <= 0:
            break
        beta = rz_new / rz
        betas.append(beta)
        p = z + beta * p
        rz = rz_new
    if not alphas:
        return 1.0, 1.0
    n = len(alphas)
    T = np.zeros((n, n))
    T[0, 0] = 1.0 / alphas[0]
    for i in range(1, n):
        T[i, i] = 1.0 / alphas[i] + betas[i - 1] / alphas[i - 1]
        off = np.sqrt(betas[i - 1]) / alphas[i - 1]
        T[i, i - 1] = T[i - 1, i] = off
    ev = np.linalg.eigvalsh(T)
    return float(ev[-1]), float(max(ev[0], 1e-12 * ev[-1]))


def _zm(space, v, name):
    torch = _torch()
    is_t = isinstance(v, torch.Tensor)
    shape = v.shape
    if is_t:
        out = v.contiguous().clone().reshape(-1)
    else:
        out = torch.as_tensor(space.to_element_major(np.asarray(v), 1).ravel()).to("cuda")
    if out.numel() != space.n_dofs:
        raise ValueError("zero-mean projection acts on one scalar field")
    ctx = space.ctx(space.default_kinds())
    _lib.call(name, ctx.handle, ctypes_ptr(out.data_ptr()), _stream())
    if is_t:
        return out.view(shape)
    return space.from_element_major(out.cpu().numpy(), 1, shape)


def zero_mean_project(space, p):
    """Subtract the L2 mean (solvers.py:179-184)."""
    if getattr(space, "is_general", False):
        from . import general
        return general.zero_mean_project(space, p)
    return _zm(space, p, "dg_zero_mean")


def zero_mean_project_dual(space, b):
    """b - (sum b / |Omega|) w, w_i = integral of l_i (solvers.py:187-198)."""
    if getattr(space, "is_general", False):
        from . import general
        return general.zero_mean_project_dual(space, b)
    return _zm(space, b, "dg_zero_mean_dual")


def lanczos_lambda_max(space, bcs, diag, tau_scale=1.0, est_iters=20, safety=1.1,
                       seed=987, project=False):
    """lambda_max of the Jacobi-preconditioned Laplacian as the reference's MG
    level setup computes it (multigrid.py:100-114): a 20-step CG-Lanczos on
    default_rng(seed).standard_normal (element-major draw), projected on
    singular problems."""
    rng = np.random.default_rng(seed)
    seed_vec = _to_dev(rng.standard_normal(space.n_dofs))
    op = lambda v: apply_pressure_laplace(space, v, bcs, tau_scale)
    if project:
        seed_vec = zero_mean_project(space, seed_vec)
        est = lambda v: zero_mean_project(space, op(v))
    else:
        est = op
    lmax, _ = eigen_estimate_via_cg(est, diag, seed_vec, est_iters)
    return safety * lmax


def laplace_pcg(space, bcs, b, tau_scale: float = 1.0, project_dual: bool = False,
                cheb: Optional[ChebyshevConfig] = None, diag=None,
                rel_tol: float = 1e-8, abs_tol: float = 0.0, max_iter: int = 1000):
    """Fused device PCG for L x = b (L = SIP Laplacian, optionally composed
    with zero_mean_project_dual), preconditioned by Chebyshev over Jacobi
    (cheb given) or Jacobi (cheb None).  Equivalent to
    ``pcg(op, lambda r: chebyshev_smooth(L, diag, cheb, r), b, ...)`` of the
    reference (solvers.py:30-129).  Returns (x, SolverStats with history)."""
    torch = _torch()
    bt = _to_dev(b)
    is_np = not isinstance(b, torch.Tensor)
    shape = bt.shape
    if is_np:
        bt = torch.as_tensor(space.to_element_major(np.asarray(b), 1).ravel()).to("cuda")
    bt = bt.contiguous().reshape(-1)
    if diag is None:
        diag = laplace_diagonal(space, bcs, tau_scale)
    diag = _to_dev(diag).contiguous().reshape(-1)
    x = torch.empty_like(bt)
    prm = _lib.PcgParams()
    prm.tau_scale = tau_scale
    prm.project_dual = int(project_dual)
    prm.cheb_degree = cheb.degree if cheb is not None else 0
    prm.cheb_range = cheb.smoothing_range if cheb is not None else 20.0
    prm.cheb_lambda_max = cheb.lambda_max if cheb is not None else 1.0
    prm.rel_tol, prm.abs_tol, prm.max_iter = rel_tol, abs_tol, max_iter
    if cheb is not None and cheb.degree == 0:
        raise ValueError("degree-0 Chebyshev is the zero operator; use cheb=None for Jacobi")
    st = _lib.PcgStats()
    hist = np.zeros(max_iter + 1)
    ctx = space.ctx(bcs.kinds)
    _lib.call("dg_laplace_pcg", ctx.handle, ctypes_ptr(bt.data_ptr()), ctypes_ptr(x.data_ptr()),
              ctypes_ptr(diag.data_ptr()), ctypes.byref(prm), ctypes.byref(st),
              hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), _stream())
    stats = SolverStats(st.iterations, st.residual, bool(st.converged), bool(st.breakdown),
                        list(hist[:st.iterations + 1]))
    if is_np:
        return space.from_element_major(x.cpu().numpy(), 1, np.shape(b)), stats
    return x.view(shape), stats


def element_local_pcg(op_local: Callable, prec_local: Callable, b, rel_tol: float = 1e-12,
                      max_iter: int = 200, floor_factor: float = 8.0):
    """Batched per-cell CG on block-diagonal SPD systems with the reference
    semantics (solvers.py:201-256): every cell iterates with its own alpha,
    beta and stops individually; the tolerance is clipped at
    floor_factor * eps * lambda_max (running Lanczos diagonal).

    Device vectors: b is a CUDA tensor (or numpy array moved to the device)
    in element-major layout (ncomp, ne, ...), cell axis 1; the callables take
    and return tensors of that layout.  Returns (x, iterations per cell,
    converged per cell) as (tensor, numpy int array, numpy bool array).
    For the V3 projection (op = projection with tau_C = None, prec = inverse
    mass) use ``projection_element_pcg``, which runs all cells' iterations in
    one kernel."""
    torch = _torch()
    b = _to_dev(b)
    ne = b.shape[1]
    red = (0,) + tuple(range(2, b.dim()))
    bshape = (1, ne) + (1,) * (b.dim() - 2)

    def edot(u, v):
        return (u * v).sum(dim=red)

    x = torch.zeros_like(b)
    r = b.clone()
    z = prec_local(r)
    rz = edot(r, z)
    norm0 = torch.sqrt(torch.clamp(rz, min=0.0))
    active = norm0 > rel_tol * norm0
    iters = torch.zeros(ne, dtype=torch.int64, device=b.device)
    p = z.clone()
    eps = float(np.finfo(float).eps)
    lan_max = torch.ones(ne, dtype=b.dtype, device=b.device)
    alpha_prev = torch.ones_like(lan_max)
    beta_prev = torch.zeros_like(lan_max)
    one = torch.ones_like(lan_max)
    for it in range(1, max_iter + 1):
        if not bool(active.any()):
            break
        Ap = op_local(p)
        pAp = edot(p, Ap)
        safe = torch.where(active & (pAp > 0), pAp, one)
        alpha = torch.where(active, rz / safe, one)
        lan_max = torch.maximum(lan_max, 1.0 / alpha + beta_prev / alpha_prev)
        am = torch.where(active, alpha, torch.zeros_like(alpha)).view(bshape)
        x += am * p
        r -= am * Ap
        z = prec_local(r)
        rz_new = edot(r, z)
        norm = torch.sqrt(torch.clamp(rz_new, min=0.0))
        iters[active] = it
        tol = torch.clamp(floor_factor * eps * lan_max, min=rel_tol) * norm0
        active = active & (norm > tol)
        beta = torch.where(active, rz_new / torch.where(rz > 0, rz, one),
                           torch.zeros_like(rz))
        alpha_prev, beta_prev = alpha, beta
        p = z + beta.view(bshape) * p
        rz = rz_new
    return x, iters.cpu().numpy(), (~active).cpu().numpy()


def projection_element_pcg(space, b, tau_d, rel_tol: float = 1e-12, max_iter: int = 200,
                           floor_factor: float = 8.0):
    """Fused ``element_local_pcg`` for the V3 projection (solvers.py:201-256
    with op_local = apply_projection_operator(space, ., tau_d, None) and
    prec_local = inverse_mass_apply): one CTA per cell runs its whole CG in
    shared memory (dg_element_local_pcg).  b: velocity (dim components) as a
    CUDA tensor (element-major) or numpy in the reference layout; tau_d: per
    cell or None.  Returns (x, iterations per cell, converged per cell)."""
    torch = _torch()
    from .operators import _Arg
    a = _Arg(space, b, space.dim)
    x = a.new_out()
    ne = space.mesh.n_elements
    iters = torch.zeros(ne, dtype=torch.int32, device="cuda")
    conv = torch.zeros(ne, dtype=torch.int32, device="cuda")
    keep = None
    td = ctypes_ptr(0)
    if tau_d is not None:
        keep = _to_dev(tau_d).contiguous().reshape(-1)
        if keep.numel() != ne:
            raise ValueError(f"tau_d needs one entry per cell ({ne})")
        td = ctypes_ptr(keep.data_ptr())
    ctx = space.ctx(space.default_kinds())
    _lib.call("dg_element_local_pcg", ctx.handle, a.ptr(), ctypes_ptr(x.data_ptr()), td,
              float(rel_tol), int(max_iter), float(floor_factor),
              ctypes_ptr(iters.data_ptr()), ctypes_ptr(conv.data_ptr()), _stream())
    del keep
    return a.result(x), iters.cpu().numpy().astype(int), conv.cpu().numpy().astype(bool)


def laplace_chebyshev_smooth(space, bcs, diag, cfg: ChebyshevConfig, rhs, x=None,
                             degree: Optional[int] = None, tau_scale: float = 1.0):
    """chebyshev_smooth(L, diag, cfg, rhs, x) (solvers.py:93-129) for the SIP
    Laplacian with every step one fused kernel (dg_cheb_step: vmult +
    Chebyshev update in the epilogue).  Device tensors (element-major)."""
    torch = _torch()
    deg = cfg.degree if degree is None else degree
    rhs = _to_dev(rhs).reshape(-1)
    diag = _to_dev(diag).reshape(-1)
    if x is None:
        x = torch.zeros_like(rhs)
        r = rhs.clone()
    else:
        x = _to_dev(x).reshape(-1).clone()
        if deg == 0:
            return x
        r = rhs - apply_pressure_laplace(space, x, bcs, tau_scale)
    if deg == 0:
        return x
    lmax = cfg.lambda_max
    lmin = lmax / cfg.smoothing_range
    theta, delta = 0.5 * (lmax + lmin), 0.5 * (lmax - lmin)
    sigma1 = theta / delta
    rho = 1.0 / sigma1
    d = (r / diag) / theta
    x += d
    d2 = torch.empty_like(d)
    ctx = space.ctx(bcs.kinds)
    for _ in range(deg - 1):
        rho_new = 1.0 / (2.0 * sigma1 - rho)
        _lib.call("dg_cheb_step", ctx.handle, ctypes_ptr(d.data_ptr()), ctypes_ptr(d2.data_ptr()),
                  ctypes_ptr(r.data_ptr()), ctypes_ptr(x.data_ptr()), ctypes_ptr(diag.data_ptr()),
                  float(rho_new * rho), float(2.0 * rho_new / delta), float(tau_scale), _stream())
        d, d2 = d2, d
        rho = rho_new
    return x


def _vector_pcg(space, op, kinds, gamma0_dt, nu, tau_d, tau_c, b, x0, rel_tol, abs_tol, max_iter):
    torch = _torch()
    bt = _to_dev(b).contiguous().reshape(-1)
    if bt.numel() != 3 * space.n_dofs:
        raise ValueError(f"expected {3 * space.n_dofs} values, got {bt.numel()}")
    x = torch.zeros_like(bt) if x0 is None else _to_dev(x0).reshape(-1).clone()
    st = _lib.PcgStats()
    hist = np.zeros(max_iter + 1)
    ctx = space.ctx(kinds)
    keep = [t.contiguous() if t is not None else None for t in (tau_d, tau_c)]
    ptr = lambda t: ctypes_ptr(t.data_ptr() if t is not None else 0)
    _lib.call("dg_vector_pcg", ctx.handle, int(op), float(gamma0_dt), float(nu), ptr(keep[0]),
              ptr(keep[1]), ctypes_ptr(bt.data_ptr()), ctypes_ptr(x.data_ptr()), float(rel_tol),
              float(abs_tol), int(max_iter), ctypes.byref(st),
              hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), _stream())
    stats = SolverStats(st.iterations, st.residual, bool(st.converged), bool(st.breakdown),
                        list(hist[:st.iterations + 1]))
    return x.view(b.shape) if hasattr(b, "shape") else x, stats


def helmholtz_pcg(space, bcs, b, gamma0_dt: float, nu: float, x0=None, rel_tol: float = 1e-8,
                  abs_tol: float = 0.0, max_iter: int = 1000):
    """``pcg(lambda v: apply_viscous_helmholtz(space, v, gamma0_dt, nu, bcs),
    lambda r: inverse_mass_apply(space, r), b, x0, ...)`` (solvers.py:30-73,
    operators.py:418-491) as one device call (dg_vector_pcg): fast-path
    operator, fused update / inverse mass / r.z kernel.  3D, device tensors."""
    return _vector_pcg(space, 0, bcs.kinds, gamma0_dt, nu, None, None, b, x0, rel_tol, abs_tol,
                       max_iter)


def projection_pcg(space, b, tau_d=None, tau_c=None, x0=None, rel_tol: float = 1e-8,
                   abs_tol: float = 0.0, max_iter: int = 1000):
    """``pcg(lambda w: apply_projection_operator(space, w, tau_d, tau_c),
    lambda r: inverse_mass_apply(space, r), b, x0, ...)`` (operators.py:372-412)
    as one device call.  tau_d per cell, tau_c in the device face layout
    [d*ne + e] (compute_penalty_parameters returns both)."""
    torch = _torch()
    td = None if tau_d is None else _to_dev(tau_d).reshape(-1)
    tc = None
    if tau_c is not None:
        from .operators import face_penalty_layout
        tc = tau_c if isinstance(tau_c, torch.Tensor) else face_penalty_layout(space, tau_c)
        tc = _to_dev(tc).reshape(-1)
    return _vector_pcg(space, 1, space.default_kinds(), 0.0, 0.0, td, tc, b, x0, rel_tol,
                       abs_tol, max_iter)
