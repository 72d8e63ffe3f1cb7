"""Drop-in operator API (reference pkg/src/dgins/operators.py) on the GPU.

Same names, arguments and error behaviour as the reference:

  apply_pressure_laplace(space, p, bcs, tau_scale=1.0)      operators.py:187
  laplace_diagonal(space, bcs, tau_scale=1.0)               operators.py:717
  mass_apply(space, u) / inverse_mass_apply(space, r)        operators.py:167-181
  apply_viscous_helmholtz(space, u, gamma0_dt, nu, bcs)      operators.py:418
  apply_projection_operator(space, w, tau_d_e, tau_c_f)      operators.py:372
  eval_convective_rhs(space, bcs, history, betas, times, t_np1,
                      body_force=None)                       operators.py:533
  eval_divergence_rhs(space, u, bcs, scale, form)            operators.py:265
  eval_pressure_gradient_rhs(space, p, bcs, scale, form)     operators.py:322
  compute_vorticity(space, u)                                operators.py:610
  eval_pressure_neumann_rhs(space, bcs, history, vorticity_history, betas,
                            nu, t_np1, body_force=None)      operators.py:621
  gp_dirichlet_rhs(space, bcs, t, tau_scale=1.0)             operators.py:241
  viscous_rhs_bc(space, bcs, t, nu)                          operators.py:494

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
        if getattr(space, "is_general", False):
            from .general import GeneralBCs
            return GeneralBCs(space, self)
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


def _route_2d(space):
    """2D Cartesian spaces run the vector operators on their general-geometry
    view (gen2d kernels, several small cells per CTA); DG_2D_GENERIC=1 keeps
    the per-cell quadrature-point kernel (A/B timing)."""
    import os
    return (space.dim == 2 and not getattr(space, "is_general", False)
            and os.environ.get("DG_2D_GENERIC", "0") == "0")


def _to_dev_em(space, x, ncomp):
    """(CUDA element-major tensor, numpy shape or None) with the Cartesian
    space's own layout rules."""
    torch = _torch()
    if isinstance(x, torch.Tensor):
        return x, None
    a = np.asarray(x, dtype=np.float64)
    return torch.as_tensor(space.to_element_major(a, ncomp).ravel()).to("cuda"), a.shape


def _from_dev_em(space, out, ncomp, shape):
    if shape is None:
        return out
    return space.from_element_major(out.cpu().numpy(), ncomp, shape)


def _view_bcs(space, bcs):
    """(general view, its resolved BCs) of a 2D Cartesian space and BC set."""
    view = space.general_view()
    key = ("view", tuple(id(bc) for _, bc in bcs.dirichlet + bcs.neumann))
    cache = space.__dict__.setdefault("_view_bcs", {})
    if key not in cache:
        spec = BoundarySpec({t: bc for t, bc in bcs.dirichlet + bcs.neumann})
        cache[key] = (spec, spec.resolve(view))
    return view, cache[key][1]


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


HOST_CHUNKS = 32  # z-chunks of the pipelined host-buffer vmult (measured best at 128^3)


def _laplace_host(space, p, bcs, tau_scale):
    """Host (CPU torch) tensor in, host tensor out: dg_laplace_vmult_host
    overlaps the two PCIe directions with the kernel (pinned buffers)."""
    torch = _torch()
    if p.dtype != torch.float64 or p.numel() != space.n_dofs:
        raise ValueError(f"expected {space.n_dofs} float64 values")
    src = p.contiguous()
    out = torch.empty(src.shape, dtype=torch.float64, pin_memory=src.is_pinned())
    ctx = space.ctx(bcs.kinds)
    _lib.call("dg_laplace_vmult_host", ctx.handle, ctypes_ptr(src.data_ptr()),
              ctypes_ptr(out.data_ptr()), float(tau_scale), HOST_CHUNKS, _stream())
    torch.cuda.current_stream().synchronize()
    return out


def apply_pressure_laplace(space: DgSpace, p, bcs: ResolvedBCs, tau_scale: float = 1.0):
    """SIP pressure Laplacian (operators.py:187-238).  CUDA tensors stay on
    the device; CPU tensors (element-major, pinned for full overlap) take the
    pipelined host-buffer path; numpy arrays are converted from the
    reference layouts."""
    if getattr(space, "is_general", False):
        from . import general
        return general.apply_pressure_laplace(space, p, bcs, tau_scale)
    torch = _torch()
    if isinstance(p, torch.Tensor) and p.device.type == "cpu":
        return _laplace_host(space, p, bcs, tau_scale)
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
    if getattr(space, "is_general", False):
        from . import general
        return general.laplace_diagonal(space, bcs, tau_scale,
                                        "numpy" if isinstance(like, np.ndarray) else None)
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
    if getattr(space, "is_general", False):
        from . import general
        return general.mass_apply(space, u)
    return _mass(space, u, "dg_mass")


def inverse_mass_apply(space: DgSpace, r):
    """Exact inverse mass per component (operators.py:176-181)."""
    if getattr(space, "is_general", False):
        from . import general
        return general.inverse_mass_apply(space, r)
    return _mass(space, r, "dg_inverse_mass")


def apply_viscous_helmholtz(space: DgSpace, u, gamma0_dt: float, nu: float,
                            bcs: ResolvedBCs):
    """(gamma0/dt) M u + SIP of -div(2 nu eps(u)) (operators.py:418-491)."""
    if getattr(space, "is_general", False):
        from . import general
        return general.apply_viscous_helmholtz(space, u, gamma0_dt, nu, bcs)
    if _route_2d(space):
        from . import general
        view, vb = _view_bcs(space, bcs)
        t, shape = _to_dev_em(space, u, 2)
        return _from_dev_em(space, general.apply_viscous_helmholtz(view, t, gamma0_dt, nu, vb),
                            2, shape)
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


def _cart_tau_c_slots(space, tau_c_f):
    """Cartesian tau_C (reference face order, or the device layout [d*ne+e])
    -> the general view's [e][4] layout."""
    torch = _torch()
    if tau_c_f is None or not isinstance(tau_c_f, torch.Tensor):
        return tau_c_f  # reference face order = the view's interior order
    em, sm, ep, sp = space.interior_faces()
    key = "_tcs_index"
    if getattr(space, key, None) is None:
        ne = space.mesh.n_elements
        src = torch.as_tensor((sm // 2) * ne + em).to("cuda")
        setattr(space, key, (src, torch.as_tensor(em * 4 + sm).to("cuda"),
                             torch.as_tensor(ep * 4 + sp).to("cuda")))
    src, a, b = getattr(space, key)
    out = torch.zeros(space.mesh.n_elements * 4, dtype=torch.float64, device="cuda")
    vals = tau_c_f.reshape(-1)[src]
    out[a] = vals
    out[b] = vals
    return out.view(space.mesh.n_elements, 4)


def apply_projection_operator(space: DgSpace, w, tau_d_e, tau_c_f):
    """M + tau_D div-div + tau_C interior jump penalty (operators.py:372-412).

    tau_d_e: per cell (or None).  tau_c_f: per interior face in the order of
    ``space.interior_faces()`` as the reference passes it, or already in the
    device layout [d*ne + e] (a CUDA tensor of dim*ne entries), or None."""
    if getattr(space, "is_general", False):
        from . import general
        return general.apply_projection_operator(space, w, tau_d_e, tau_c_f)
    if _route_2d(space):
        from . import general
        t, shape = _to_dev_em(space, w, 2)
        out = general.apply_projection_operator(space.general_view(), t, tau_d_e,
                                                _cart_tau_c_slots(space, tau_c_f))
        return _from_dev_em(space, out, 2, shape)
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
    """sum_i beta_i [(grad v, u u) - (v, F*.n)] + (v, f) with the local
    Lax-Friedrichs flux on the over-integration rule (operators.py:533-594).
    Dirichlet data g(x, times[i]) enters the mirror state 2g - u (a None
    callable means homogeneous data, as for every boundary callable here); the data and
    the body force are sampled on the host (they are the caller's Python
    callables) and integrated on the device."""
    if getattr(space, "is_general", False):
        from . import general
        return general.eval_convective_rhs(space, bcs, history, betas, times, t_np1, body_force)
    # convective: the general kernel wins at k <= 3 (n_q <= 5), the per-cell
    # kernel above that (profiles/NOTES.md)
    if _route_2d(space) and space.k <= 3 and space.n_q_over == (3 * space.k) // 2 + 1:
        from . import general
        view, vb = _view_bcs(space, bcs)
        conv = [_to_dev_em(space, u, 2) for u in history]
        out = general.eval_convective_rhs(view, vb, [t for t, _ in conv], betas, times, t_np1,
                                          body_force)
        return _from_dev_em(space, out, 2, conv[0][1])
    import ctypes
    if len(times) < len(history) or len(betas) < len(history):
        raise ValueError("need one beta and one time per history level")
    args = [_Arg(space, u, space.dim) for u in history]
    out = args[0].new_out()
    ptrs = (ctypes.c_void_p * len(args))(*[a.t.data_ptr() for a in args])
    b = (ctypes.c_double * len(betas))(*[float(x) for x in betas])
    keep = []
    gd = None
    if bcs.dirichlet:
        pts = _rule_points(space, space.n_q_over)
        flat = []
        for t_i in times[:len(args)]:
            sides = _side_data(space, pts, [(tag, lambda x, bc=bc, t=t_i: bc.g(x, t))
                                            for tag, bc in bcs.dirichlet
                                            if bc.g is not None], keep)
            flat += sides
        gd = (ctypes.c_void_p * len(flat))(*flat)
    body = ctypes_ptr(0)
    if body_force is not None:
        fq = body_force(_volume_points(space, space.n_q_over), t_np1)
        fq = np.ascontiguousarray(np.asarray(fq, dtype=np.float64).reshape(space.dim, -1))
        keep.append(_dev(fq))
        body = ctypes_ptr(keep[-1].data_ptr())
    ctx = space.ctx(bcs.kinds)
    _lib.call("dg_convective_rhs_ex", ctx.handle, len(args), ctypes.cast(ptrs, ctypes.c_void_p),
              ctypes.cast(b, ctypes.c_void_p),
              ctypes.cast(gd, ctypes.c_void_p) if gd is not None else ctypes_ptr(0),
              body, ctypes_ptr(out.data_ptr()), _stream())
    return args[0].result(out)


# ---------------------------------------------------------------------------
# once-per-step right-hand sides (operators.py:241-366, 494-527, 610-672)

_FORMS = {"standard": 0, "weak": 1, "strong": 2}


def _dev(a):
    torch = _torch()
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64)).to("cuda")


def _rule_points(space, n_q):
    from .basis import get_basis
    return np.asarray(get_basis(space.k, n_q).points)


def _volume_points(space, n_q):
    """Physical coordinates of the tensor Gauss points of every cell,
    (dim, ne, [z,] y, x) in element-major order."""
    pts = _rule_points(space, n_q)
    dim, mesh = space.dim, space.mesh
    idx = np.indices(mesh.counts[::-1]).reshape(dim, -1)[::-1]      # ix, iy, iz
    out = []
    for d in range(dim):
        v = mesh.axis_vertices[d]
        c = v[idx[d]][:, None] + 0.5 * (pts[None, :] + 1.0) * np.diff(v)[idx[d]][:, None]
        shape = [mesh.n_elements] + [1] * dim
        shape[dim - d] = len(pts)
        out.append(np.broadcast_to(c.reshape(shape), (mesh.n_elements,) + (len(pts),) * dim))
    return np.stack(out)


def side_face_points(space, side, pts):
    """Physical coordinates of the face Gauss points of the boundary cells of
    one side (side = 2*d + s, TAG_NAMES order) in the device boundary-data
    layout of include/dgmf.h: (dim, ntan, [slow,] fast), tangential cells
    (slow, fast) and points [slow][fast] in decreasing axis order."""
    dim, mesh = space.dim, space.mesh
    d, s = divmod(side, 2)
    tang = [a for a in range(dim - 1, -1, -1) if a != d]
    counts = [mesh.counts[a] for a in tang]
    q = len(pts)
    nt = len(tang)
    X = np.empty((dim,) + tuple(counts) + (q,) * nt)
    for a in range(dim):
        v = mesh.axis_vertices[a]
        if a == d:
            X[a] = v[-1] if s else v[0]
            continue
        j = tang.index(a)
        c = v[:-1, None] + 0.5 * (pts[None, :] + 1.0) * np.diff(v)[:, None]
        shape = [1] * (2 * nt)
        shape[j] = counts[j]
        shape[nt + j] = q
        X[a] = c.reshape(shape)
    return X.reshape((dim, int(np.prod(counts))) + (q,) * nt)


def _side_data(space, pts, entries, keep):
    """Evaluate per-tag data callables fn(x) at the face points of their
    sides; returns 6 device pointers (0 where no data) in the layout
    [ntan][ncomp][n_f]."""
    ptrs = [0] * 6
    for tag, fn in entries:
        side = TAG_NAMES.index(tag)
        X = side_face_points(space, side, pts)
        val = np.asarray(fn(X), dtype=np.float64)
        if val.ndim == X.ndim - 1:          # scalar data
            val = val[None]
        nt = X.shape[1]
        val = np.ascontiguousarray(np.moveaxis(val.reshape(val.shape[0], nt, -1), 1, 0))
        t = _dev(val)
        keep.append(t)
        ptrs[side] = t.data_ptr()
    return ptrs


def _out_result(space, out, ncomp, like):
    """Result for calls whose only inputs are callables: a CUDA tensor if
    ``like`` is a tensor (or the string 'device'), else numpy in the layout
    of ``like`` (default: the 2D reference kernel layout / 3D element-major)."""
    torch = _torch()
    if isinstance(like, torch.Tensor) or (isinstance(like, str) and like == "device"):
        return out
    if like is None:
        m, ne = space.k + 1, space.mesh.n_elements
        if space.dim == 2:
            like_shape = (m, ne, m) if ncomp == 1 else (ncomp, m, ne, m)
        else:
            like_shape = space.field_shape(None if ncomp == 1 else ncomp)
    else:
        like_shape = np.shape(like)
    return space.from_element_major(out.cpu().numpy(), ncomp, like_shape)


def _bnd_call(name, space, bcs, entries, ncomp_out, like, *scalars):
    import ctypes
    torch = _torch()
    keep = []
    ptrs = _side_data(space, _rule_points(space, space.k + 1), entries, keep)
    arr = (ctypes.c_void_p * 6)(*ptrs)
    out = torch.empty(space.n_dofs * ncomp_out, dtype=torch.float64, device="cuda")
    ctx = space.ctx(bcs.kinds)
    _lib.call(name, ctx.handle, ctypes.cast(arr, ctypes.c_void_p),
              *[ctypes.c_double(v) for v in scalars], ctypes_ptr(out.data_ptr()), _stream())
    return _out_result(space, out, ncomp_out, like)


def gp_dirichlet_rhs(space: DgSpace, bcs: ResolvedBCs, t: float, tau_scale: float = 1.0,
                     like=None):
    """Pressure-Dirichlet data g_p on velocity-Neumann faces for the Poisson
    right side (operators.py:241-259)."""
    if getattr(space, "is_general", False):
        from . import general
        return general.gp_dirichlet_rhs(space, bcs, t, tau_scale, like)
    entries = [(tag, lambda x, bc=bc: bc.g_p(x, t)) for tag, bc in bcs.neumann
               if bc.g_p is not None]
    return _bnd_call("dg_gp_dirichlet_rhs", space, bcs, entries, 1, like, float(tau_scale))


def viscous_rhs_bc(space: DgSpace, bcs: ResolvedBCs, t: float, nu: float, like=None):
    """Boundary-data terms of the viscous solve (operators.py:494-527):
    Dirichlet g with 2 tau nu and the symmetric-gradient test, Neumann
    h + g_p n."""
    if getattr(space, "is_general", False):
        from . import general
        return general.viscous_rhs_bc(space, bcs, t, nu, like)
    entries = [(tag, lambda x, bc=bc: bc.g(x, t)) for tag, bc in bcs.dirichlet
               if bc.g is not None]

    def neu(bc):
        def f(x):
            h = (np.asarray(bc.h(x, t), dtype=np.float64) if bc.h is not None
                 else np.zeros((space.dim,) + x.shape[1:]))
            gp = (np.asarray(bc.g_p(x, t), dtype=np.float64) if bc.g_p is not None
                  else np.zeros(x.shape[1:]))
            return np.concatenate([h, np.broadcast_to(gp, h.shape[1:])[None]])
        return f
    entries += [(tag, neu(bc)) for tag, bc in bcs.neumann
                if bc.h is not None or bc.g_p is not None]
    return _bnd_call("dg_viscous_rhs_bc", space, bcs, entries, space.dim, like, float(nu))


def eval_divergence_rhs(space: DgSpace, u, bcs: ResolvedBCs, scale: float,
                        form: str = "standard"):
    """a(q, u) scaled: 'standard' volume form, 'weak' with central flux or
    its 'strong' rewrite (operators.py:265-316)."""
    if getattr(space, "is_general", False):
        from . import general
        return general.eval_divergence_rhs(space, u, bcs, scale, form)
    if form not in _FORMS:
        raise ValueError(f"unknown divergence form {form!r}")
    torch = _torch()
    a = _Arg(space, u, space.dim)
    out = torch.empty(space.n_dofs, dtype=torch.float64, device="cuda")
    ctx = space.ctx(bcs.kinds)
    _lib.call("dg_divergence_rhs", ctx.handle, a.ptr(), ctypes_ptr(out.data_ptr()),
              float(scale), _FORMS[form], _stream())
    return _scalar_like(space, a, out)


def _scalar_like(space, a, out):
    """Scalar result of a vector-input call, in the input's type/layout."""
    if a.is_torch:
        return out.view(a.shape[1:]) if len(a.shape) > 1 and a.shape[0] == space.dim \
            and int(np.prod(a.shape[1:])) == space.n_dofs else out
    like = a.shape[1:] if len(a.shape) > 1 else (space.n_dofs,)
    return space.from_element_major(out.cpu().numpy(), 1, like)


def _vector_like(space, a, out):
    """Vector result of a scalar-input call, in the input's type/layout."""
    ncomp = space.dim
    if a.is_torch:
        return out.view((ncomp,) + tuple(a.shape)) if len(a.shape) > 1 else out
    return space.from_element_major(out.cpu().numpy(), ncomp, (ncomp,) + tuple(a.shape))


def eval_pressure_gradient_rhs(space: DgSpace, p, bcs: ResolvedBCs, scale: float,
                               form: str = "standard"):
    """b(v, p) scaled: standard -(v, scale grad p) or weak with central flux
    (operators.py:322-366)."""
    if getattr(space, "is_general", False):
        from . import general
        return general.eval_pressure_gradient_rhs(space, p, bcs, scale, form)
    if form not in ("standard", "weak"):
        raise ValueError(f"unknown pressure-gradient form {form!r}")
    torch = _torch()
    a = _Arg(space, p, 1)
    out = torch.empty(space.n_dofs * space.dim, dtype=torch.float64, device="cuda")
    ctx = space.ctx(bcs.kinds)
    _lib.call("dg_pressure_gradient_rhs", ctx.handle, a.ptr(), ctypes_ptr(out.data_ptr()),
              float(scale), _FORMS[form], _stream())
    return _vector_like(space, a, out)


def compute_vorticity(space: DgSpace, u):
    """Element-local L2 projection of curl u (operators.py:610-618): a scalar
    field in 2D (the reference), the three curl components in 3D."""
    if getattr(space, "is_general", False):
        from . import general
        return general.compute_vorticity(space, u)
    torch = _torch()
    a = _Arg(space, u, space.dim)
    nw = 1 if space.dim == 2 else 3
    out = torch.empty(space.n_dofs * nw, dtype=torch.float64, device="cuda")
    ctx = space.ctx(space.default_kinds())
    _lib.call("dg_vorticity", ctx.handle, a.ptr(), ctypes_ptr(out.data_ptr()), _stream())
    if nw == 1:
        return _scalar_like(space, a, out)
    return a.result(out)


def eval_pressure_neumann_rhs(space: DgSpace, bcs: ResolvedBCs, history, vorticity_history,
                              betas, nu: float, t_np1: float,
                              body_force: Optional[Callable] = None, like=None):
    """Consistent pressure Neumann data on velocity-Dirichlet faces:
    -(dg/dt + sum_i beta_i (div(u u) + nu curl w) - f) . n
    (operators.py:621-672).  dg/dt and f are sampled on the host at the face
    points (caller's callables); the traces run on the device."""
    if getattr(space, "is_general", False):
        from . import general
        return general.eval_pressure_neumann_rhs(space, bcs, history, vorticity_history, betas, nu,
                                                 t_np1, body_force, like)
    import ctypes
    torch = _torch()
    nw = 1 if space.dim == 2 else 3
    hist = [_Arg(space, u, space.dim) for u in history]
    if not bcs.dirichlet:
        out = torch.zeros(space.n_dofs, dtype=torch.float64, device="cuda")
        return _out_result(space, out, 1, like) if like is not None else \
            _scalar_like(space, hist[0], out)
    vort = [_Arg(space, w, nw) for w in vorticity_history]
    if len(vort) < len(hist) or len(betas) < len(hist):
        raise ValueError("need one vorticity field and one beta per history level")
    keep = []
    entries = []
    for tag, bc in bcs.dirichlet:
        if bc.dg_dt is None and body_force is None:
            continue

        def f(x, bc=bc):
            h = (np.asarray(bc.dg_dt(x, t_np1), dtype=np.float64) if bc.dg_dt is not None
                 else np.zeros((space.dim,) + x.shape[1:]))
            if body_force is not None:
                h = h - np.asarray(body_force(x, t_np1), dtype=np.float64)
            return h
        entries.append((tag, f))
    ptrs = _side_data(space, _rule_points(space, space.k + 1), entries, keep)
    bnd = (ctypes.c_void_p * 6)(*ptrs)
    hp = (ctypes.c_void_p * len(hist))(*[a.t.data_ptr() for a in hist])
    wp = (ctypes.c_void_p * len(hist))(*[w.t.data_ptr() for w in vort[:len(hist)]])
    bt = (ctypes.c_double * len(hist))(*[float(x) for x in betas[:len(hist)]])
    out = torch.empty(space.n_dofs, dtype=torch.float64, device="cuda")
    ctx = space.ctx(bcs.kinds)
    _lib.call("dg_pressure_neumann_rhs", ctx.handle, len(hist), ctypes.cast(hp, ctypes.c_void_p),
              ctypes.cast(wp, ctypes.c_void_p), ctypes.cast(bt, ctypes.c_void_p), float(nu),
              ctypes.cast(bnd, ctypes.c_void_p), ctypes_ptr(out.data_ptr()), _stream())
    if like is not None:
        return _out_result(space, out, 1, like)
    return _scalar_like(space, hist[0], out)





# ---------------------------------------------------------------------------
# stabilisation variants and penalty parameters (operators.py:28-75, 736-755)

VARIANTS = ("VHW", "V1", "V2", "V3a", "V3b", "V3c", "V4")


@dataclass
class VariantConfig:
    """Stabilisation variant selector and penalty factors (operators.py:31-75)."""
    variant: str = "V3c"
    zeta_d_star: float = 1.0
    zeta_c_star: float = 1.0
    dt_ref: Optional[float] = None

    def __post_init__(self):
        if self.variant not in VARIANTS:
            raise ValueError(f"unknown variant {self.variant!r}")
        if self.zeta_d_star < 0 or self.zeta_c_star < 0:
            raise ValueError("penalty factors must be >= 0")
        if self.variant == "V1" and not (self.dt_ref and self.dt_ref > 0):
            raise ValueError("V1 needs a positive reference time step dt_ref")

    @property
    def uses_divdiv(self) -> bool:
        return self.variant in ("V3a", "V3b", "V3c", "V4")

    @property
    def uses_jump(self) -> bool:
        return self.variant == "V4"

    @property
    def a_form(self) -> str:
        return "weak" if self.variant in ("V3b", "V3c") else "standard"

    @property
    def b_form(self) -> str:
        return "weak" if self.variant == "V3c" else "standard"

    @property
    def local_projection(self) -> bool:
        return not self.uses_jump


def compute_penalty_parameters(space: DgSpace, u, dt: float, cfl: float, cfg: VariantConfig):
    """tau_D per cell and tau_C per face from the cell-mean velocity
    (operators.py:736-755; h = V^(1/dim)).  Returns device tensors (tau_c in
    the face layout apply_projection_operator accepts) or None where the
    variant has no such term."""
    if getattr(space, "is_general", False):
        from . import general
        return general.compute_penalty_parameters(space, u, dt, cfl, cfg)
    if cfl <= 0:
        raise ValueError(f"CFL must be positive, got {cfl}")
    torch = _torch()
    a = _Arg(space, u, space.dim)
    ne = space.mesh.n_elements
    td = torch.empty(ne, dtype=torch.float64, device="cuda") if cfg.uses_divdiv else None
    tc = torch.empty(space.dim * ne, dtype=torch.float64, device="cuda") if cfg.uses_jump else None
    ctx = space.ctx(space.default_kinds())
    _lib.call("dg_penalty_parameters", ctx.handle, a.ptr(), float(dt), float(cfl),
              float(cfg.zeta_d_star), float(cfg.zeta_c_star),
              ctypes_ptr(td.data_ptr() if td is not None else 0),
              ctypes_ptr(tc.data_ptr() if tc is not None else 0), _stream())
    return td, tc
