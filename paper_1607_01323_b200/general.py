"""General-geometry 2D path: the reference's own 2D setting — quadrilateral
meshes with iso-parametric (possibly curved, k_geo > 1) mappings, arbitrary
conforming connectivity and face-orientation flips (reference mesh.py,
geometry.py, spaces.py) — on the device (csrc/gen2d.cuh, dg_g2_*).

``GeneralSpace2D(mesh, k)`` takes any object with the reference ``Mesh``
fields (``geom_degree``, ``geom_nodes`` (2, mg, ne, mg), ``interior``
(em, sm, ep, sp, flip), ``boundary`` (elem, slot, tag), ``tag_names``), so a
reference user passes the meshes they already build (box, warped, cylinder).
The geometry at the quadrature points is restated here from
geometry.py:29-87 (host setup, numpy) and uploaded once; the operators
mirror operators.py under the same names and take reference-layout numpy
fields (m, ne, m) / (c, m, ne, m) or element-major CUDA tensors.
"""

import ctypes
from typing import Optional

import numpy as np

from . import _lib
from .basis import get_basis
from .spaces import _torch

_REF_NORMALS = ((-1.0, 0.0), (1.0, 0.0), (0.0, -1.0), (0.0, 1.0))


def _lagrange(nodes, x):
    """V[q][i] = l_i(x_q) for the Lagrange basis on `nodes`."""
    nodes, x = np.asarray(nodes, dtype=np.float64), np.asarray(x, dtype=np.float64)
    V = np.ones((x.size, nodes.size))
    for i in range(nodes.size):
        for j in range(nodes.size):
            if j != i:
                V[:, i] *= (x - nodes[j]) / (nodes[i] - nodes[j])
    return V


def _vol(F, S1, S2):
    """out[a, e, b] = sum_j sum_i S1[a, j] S2[b, i] F[j, e, i] (kernel layout)."""
    return np.einsum("aj,jei,bi->aeb", S1, F, S2, optimize=True)


def _face_values(F, t):
    S = t.S
    return np.stack([(S @ F[:, :, 0]).T, (S @ F[:, :, -1]).T, F[0] @ S.T, F[-1] @ S.T])


def _face_gradients(F, t):
    S, D, ld, rd = t.S, t.D, t.left_deriv, t.right_deriv
    m, ne, _ = F.shape
    Fr = F.reshape(m * ne, m)
    dxl = (Fr @ ld).reshape(m, ne)
    dxr = (Fr @ rd).reshape(m, ne)
    Fy = F.reshape(m, ne * m)
    dyb = (ld @ Fy).reshape(ne, m)
    dyt = (rd @ Fy).reshape(ne, m)
    gx = np.stack([(S @ dxl).T, (S @ dxr).T, F[0] @ D.T, F[-1] @ D.T])
    gy = np.stack([(D @ F[:, :, 0]).T, (D @ F[:, :, -1]).T, dyb @ S.T, dyt @ S.T])
    return gx, gy


class Geometry2D:
    """Mapped geometry at the Gauss points (restates geometry.py:29-87):
    xq, jxw, jinvT (volume) and xf, jinvT_f, normal, sjxw (faces), in the
    reference kernel layouts."""

    def __init__(self, mesh, n_q: int):
        gb = get_basis(mesh.geom_degree, n_q)
        w = gb.weights
        X, Y = mesh.geom_nodes[0], mesh.geom_nodes[1]
        xs, ys = _vol(X, gb.S, gb.S), _vol(Y, gb.S, gb.S)
        dxdxi, dydxi = _vol(X, gb.S, gb.D), _vol(Y, gb.S, gb.D)
        dxdeta, dydeta = _vol(X, gb.D, gb.S), _vol(Y, gb.D, gb.S)
        det = dxdxi * dydeta - dxdeta * dydxi
        if not (det > 0).all():
            bad = int(np.argwhere((det <= 0).any(axis=(0, 2)))[0, 0])
            raise ValueError(f"non-positive mapping Jacobian in element {bad}")
        self.xq = np.stack([xs, ys])
        self.jxw = det * np.multiply.outer(w, w)[:, None, :]
        self.jinvT = np.stack([np.stack([dydeta / det, -dydxi / det]),
                               np.stack([-dxdeta / det, dxdxi / det])])
        self.volumes = self.jxw.sum(axis=(0, 2))
        fx, fy = _face_values(X, gb), _face_values(Y, gb)
        gxx, gxy = _face_gradients(X, gb)
        gyx, gyy = _face_gradients(Y, gb)
        fdet = gxx * gyy - gxy * gyx
        if not (fdet > 0).all():
            bad = int(np.argwhere((fdet <= 0).any(axis=(0, 2)))[0, 0])
            raise ValueError(f"non-positive mapping Jacobian on a face of element {bad}")
        self.xf = np.stack([fx, fy])
        jit = np.stack([np.stack([gyy / fdet, -gyx / fdet]), np.stack([-gxy / fdet, gxx / fdet])])
        self.jinvT_f = jit
        ne = X.shape[1]
        normal = np.empty((2, 4, ne, n_q))
        sjxw = np.empty((4, ne, n_q))
        for s, nref in enumerate(_REF_NORMALS):
            v0 = jit[0, 0, s] * nref[0] + jit[0, 1, s] * nref[1]
            v1 = jit[1, 0, s] * nref[0] + jit[1, 1, s] * nref[1]
            norm = np.hypot(v0, v1)
            normal[0, s] = v0 / norm
            normal[1, s] = v1 / norm
            sjxw[s] = fdet[s] * norm * w[None, :]
        self.normal = normal
        self.sjxw = sjxw
        self.face_areas = sjxw.sum(axis=2)


def compute_tau_ip(mesh, geom: Geometry2D, k: int):
    """tau_e = (k+1)^2 (A_int/2 + A_bnd) / V_e (geometry.py:90-108)."""
    ne = mesh.geom_nodes.shape[2]
    a_int = np.zeros(ne)
    a_bnd = np.zeros(ne)
    f, b = mesh.interior, mesh.boundary
    np.add.at(a_int, f.em, geom.face_areas[f.sm, f.em])
    np.add.at(a_int, f.ep, geom.face_areas[f.sp, f.ep])
    np.add.at(a_bnd, b.elem, geom.face_areas[b.slot, b.elem])
    return (k + 1) ** 2 * (0.5 * a_int + a_bnd) / geom.volumes


class GeneralSpace2D:
    """Discontinuous Q_k space on a general quadrilateral mesh (reference
    spaces.py:61-81) with its device context."""

    dim = 2
    is_general = True

    def __init__(self, mesh, k: int):
        if k < 1:
            raise ValueError(f"polynomial degree must be >= 1, got k={k}")
        if k > 7:
            raise ValueError("general 2D path: k <= 7")
        torch = _torch()
        self.mesh, self.k = mesh, k
        n = k + 1
        self.n_q = n
        self.basis = get_basis(k, n)
        self.geom = Geometry2D(mesh, n)
        self.tau_e = compute_tau_ip(mesh, self.geom, k)
        ne = mesh.geom_nodes.shape[2]
        self.n_elements = ne
        f = mesh.interior
        em, sm = np.asarray(f.em, np.int64), np.asarray(f.sm, np.int64)
        ep, sp = np.asarray(f.ep, np.int64), np.asarray(f.sp, np.int64)
        flip = np.asarray(f.flip, bool)
        nbr = -np.ones((ne, 4), np.int64)
        nslot = np.zeros((ne, 4), np.int32)
        nflip = np.zeros((ne, 4), np.int32)
        nbr[em, sm], nslot[em, sm], nflip[em, sm] = ep, sp, flip
        nbr[ep, sp], nslot[ep, sp], nflip[ep, sp] = em, sm, flip
        self._nbr = (nbr, nslot, nflip, sm, em, sp, ep, flip)
        self._h, self._d, self._tabs = self._make_ctx(self.geom, self.basis, n)
        self._over = None
        self._kinds = {}
        b = mesh.boundary
        self.b_groups = {}
        for i, name in enumerate(mesh.tag_names):
            sel = np.asarray(b.tag) == i
            if sel.any():
                self.b_groups[name] = (np.asarray(b.elem)[sel], np.asarray(b.slot)[sel])

    def _make_ctx(self, g, t, q):
        """Device geometry arrays (element-major) and a dg_g2 context for one
        rule (the linear rule n_q = k+1, or the convective over-integration
        rule)."""
        torch = _torch()
        nbr, nslot, nflip, sm, em, sp, ep, flip = self._nbr
        ne = self.n_elements
        # own-frame face data; plus sides of interior faces take the minus
        # side's sJxW and (negated) normal, flip-mapped (spaces.py:140-163)
        fsj = g.sjxw.copy()
        fnrm = g.normal.copy()
        sjm = g.sjxw[sm, em]
        nm = g.normal[:, sm, em]
        sjm = np.where(flip[:, None], sjm[:, ::-1], sjm)
        nm = np.where(flip[None, :, None], nm[:, :, ::-1], nm)
        fsj[sp, ep] = sjm
        fnrm[:, sp, ep] = -nm
        dev = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to("cuda")
        d = {
            "jxw": dev(g.jxw.transpose(1, 0, 2)),
            "jit": dev(g.jinvT.reshape(4, q, ne, q).transpose(2, 0, 1, 3)),
            "fsj": dev(fsj.transpose(1, 0, 2)),
            "fnrm": dev(fnrm.transpose(2, 1, 0, 3)),
            "fjit": dev(g.jinvT_f.reshape(4, 4, ne, q).transpose(2, 1, 0, 3)),
            "tau": dev(self.tau_e),
            "nbr": dev(nbr),
            "nslot": dev(nslot),
            "nflip": dev(nflip),
        }
        desc = _lib.G2Desc()
        desc.n, desc.nq, desc.ncells = self.k + 1, q, ne
        P = lambda x: ctypes.c_void_p(x.data_ptr())
        for name in ("jxw", "jit", "fsj", "fnrm", "fjit", "tau", "nbr", "nslot", "nflip"):
            setattr(desc, name, P(d[name]))
        Si = np.linalg.inv(t.S) if q == self.k + 1 else np.zeros((self.k + 1, self.k + 1))
        tabs = [np.ascontiguousarray(a, dtype=np.float64)
                for a in (t.S, t.D, Si, t.left_deriv, t.right_deriv)]
        H = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        desc.S, desc.D, desc.Si, desc.ld, desc.rd = [H(a) for a in tabs]
        h = ctypes.c_void_p()
        _lib.call("dg_g2_create", ctypes.byref(desc), ctypes.byref(h))
        return h, d, tabs

    def over(self):
        """(handle, geometry) of the convective over-integration rule
        n_q = floor(3k/2) + 1 (basis.py:103-105, spaces.py:117-122)."""
        if self._over is None:
            nq = (3 * self.k) // 2 + 1
            if nq > 11:
                raise ValueError("general 2D convective term: n_q <= 11 (k <= 6)")
            g = Geometry2D(self.mesh, nq)
            h, d, tabs = self._make_ctx(g, get_basis(self.k, nq), nq)
            self._over = (h, g, d, tabs)
        return self._over

    def __del__(self):
        for h in (getattr(self, "_h", None),
                  (getattr(self, "_over", None) or (None,))[0]):
            if h is not None and h.value:
                try:
                    _lib.lib().dg_g2_destroy(h)
                except Exception:
                    pass
        self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def n_local(self):
        return (self.k + 1) ** 2

    @property
    def n_dofs(self):
        return self.n_elements * self.n_local

    def boundary_tags(self):
        return list(self.b_groups)

    def node_coords(self):
        """Physical coordinates of the field nodes, (2, m, ne, m) (restates
        spaces.py:86-105: the geometry mapping evaluated at the GLL nodes of
        degree k)."""
        if getattr(self, "_node_coords", None) is None:
            from .basis import gll_nodes
            gb = get_basis(self.mesh.geom_degree, 2)
            T = _lagrange(gb.nodes, gll_nodes(self.k))
            X, Y = self.mesh.geom_nodes[0], self.mesh.geom_nodes[1]
            self._node_coords = np.stack([_vol(X, T, T), _vol(Y, T, T)])
        return self._node_coords

    def interpolate(self, fn, t: float, ncomp: int):
        """Nodal interpolant of fn(x, t) (spaces.py:107-113)."""
        x = self.node_coords()
        vals = fn(x, t)
        if ncomp == 1 and np.asarray(vals).shape != (1,) + x.shape[1:]:
            vals = np.asarray(vals)[None]
        return np.ascontiguousarray(np.asarray(vals, dtype=float))

    def kinds(self, bcs):
        """Device int32 [e][4] boundary kinds of a resolved BC set."""
        key = bcs.key
        if key not in self._kinds:
            from .operators import DirichletBC, NeumannBC
            kd = np.zeros((self.n_elements, 4), np.int32)
            for tag, (eb, sb) in self.b_groups.items():
                kind = bcs.spec.kinds[tag]
                if isinstance(kind, DirichletBC):
                    kd[eb, sb] = _lib.BC_VELOCITY_DIRICHLET
                elif isinstance(kind, NeumannBC):
                    kd[eb, sb] = _lib.BC_VELOCITY_NEUMANN
                else:
                    raise TypeError(f"unsupported boundary kind for tag {tag!r}")
            self._kinds[key] = _torch().as_tensor(kd).to("cuda")
        return self._kinds[key]

    # layouts: reference kernel layout (m, ne, m) <-> element-major (ne, m, m)
    def to_element_major(self, a, ncomp):
        a = np.asarray(a, dtype=np.float64)
        m, ne = self.k + 1, self.n_elements
        if ncomp == 1:
            return np.ascontiguousarray(a.reshape(m, ne, m).transpose(1, 0, 2))
        return np.ascontiguousarray(a.reshape(ncomp, m, ne, m).transpose(0, 2, 1, 3))

    def from_element_major(self, a, ncomp):
        m, ne = self.k + 1, self.n_elements
        if ncomp == 1:
            return np.ascontiguousarray(a.reshape(ne, m, m).transpose(1, 0, 2))
        return np.ascontiguousarray(a.reshape(ncomp, ne, m, m).transpose(0, 2, 1, 3))


class GeneralBCs:
    """Resolved boundary conditions of a general space (operators.py:113-131)."""

    def __init__(self, space: GeneralSpace2D, spec):
        present = set(space.boundary_tags())
        missing = present - set(spec.kinds)
        if missing:
            raise ValueError(f"boundary tags without a condition: {missing}")
        from .operators import DirichletBC, NeumannBC
        self.space, self.spec = space, spec
        self.dirichlet, self.neumann = [], []
        for tag in space.boundary_tags():
            kind = spec.kinds[tag]
            if isinstance(kind, DirichletBC):
                self.dirichlet.append((tag, kind))
            elif isinstance(kind, NeumannBC):
                self.neumann.append((tag, kind))
            else:
                raise TypeError(f"unsupported boundary kind for tag {tag!r}")
        self.key = tuple((t, type(spec.kinds[t]).__name__) for t in space.boundary_tags())

    @property
    def has_outflow(self):
        return len(self.neumann) > 0


def _field(space, x, ncomp):
    """(device tensor, is_numpy, shape) of a field argument."""
    torch = _torch()
    if isinstance(x, torch.Tensor):
        if x.device.type != "cuda" or x.dtype != torch.float64:
            raise ValueError("device operands must be float64 CUDA tensors")
        if x.numel() != ncomp * space.n_dofs:
            raise ValueError(f"expected {ncomp * space.n_dofs} values, got {x.numel()}")
        return x.contiguous().reshape(-1), False, x.shape
    a = np.asarray(x, dtype=np.float64)
    if a.size != ncomp * space.n_dofs:
        raise ValueError(f"expected {ncomp * space.n_dofs} values, got {a.size}")
    return torch.as_tensor(space.to_element_major(a, ncomp).ravel()).to("cuda"), True, a.shape


def _result(space, out, is_np, shape, ncomp):
    if is_np:
        return space.from_element_major(out.cpu().numpy(), ncomp).reshape(shape)
    return out.view(shape)


def _ncomp_of(space, x):
    n = int(np.prod(np.shape(x)))
    if n % space.n_dofs:
        raise ValueError("field size is not a multiple of the space size")
    return n // space.n_dofs


def _stream():
    return ctypes.c_void_p(_torch().cuda.current_stream().cuda_stream)


def _apply(space, op, x, ncomp, tau_scale=1.0, kinds=None):
    t, is_np, shape = _field(space, x, ncomp)
    out = _torch().empty_like(t)
    kp = ctypes.c_void_p(kinds.data_ptr() if kinds is not None else 0)
    _lib.call("dg_g2_apply", space.handle, int(op), float(tau_scale), kp,
              ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(out.data_ptr()), int(ncomp),
              _stream())
    return _result(space, out, is_np, shape, ncomp)


def mass_apply(space: GeneralSpace2D, u):
    """Consistent mass per component (operators.py:167-173)."""
    return _apply(space, 0, u, _ncomp_of(space, u))


def inverse_mass_apply(space: GeneralSpace2D, r):
    """Exact inverse mass per component (operators.py:176-181)."""
    return _apply(space, 1, r, _ncomp_of(space, r))


def apply_pressure_laplace(space: GeneralSpace2D, p, bcs: GeneralBCs, tau_scale: float = 1.0):
    """SIP pressure Laplacian (operators.py:187-238)."""
    return _apply(space, 2, p, 1, tau_scale, space.kinds(bcs))


def laplace_diagonal(space: GeneralSpace2D, bcs: GeneralBCs, tau_scale: float = 1.0,
                     like: Optional[object] = None):
    """Exact Jacobi diagonal (operators.py:675-730): a CUDA tensor
    (element-major), or reference-layout numpy when ``like='numpy'``."""
    torch = _torch()
    out = torch.empty(space.n_dofs, dtype=torch.float64, device="cuda")
    _lib.call("dg_g2_laplace_diagonal", space.handle, float(tau_scale),
              ctypes.c_void_p(space.kinds(bcs).data_ptr()), ctypes.c_void_p(out.data_ptr()),
              _stream())
    if like == "numpy":
        return space.from_element_major(out.cpu().numpy(), 1)
    return out


# ---------------------------------------------------------------------------
# vector operators and right-hand sides (operators.py:262-618)

def _op(space, prm, src, dst, handle=None):
    _lib.call("dg_g2_operator", handle if handle is not None else space.handle,
              ctypes.byref(prm), ctypes.c_void_p(src.data_ptr() if src is not None else 0),
              ctypes.c_void_p(dst.data_ptr()), _stream())


def _params(space, op, bcs):
    prm = _lib.G2Params()
    prm.op = op
    prm.kind = ctypes.c_void_p(space.kinds(bcs).data_ptr())
    return prm


def _all_interior_kinds(space):
    """Kinds from the connectivity alone: 0 on interior (incl. periodic)
    slots, velocity-Dirichlet on boundary slots (operators whose face terms
    are interior-only: projection; and the face-free vorticity)."""
    key = ("__structural__",)
    if key not in space._kinds:
        nbr = space._d["nbr"]
        space._kinds[key] = torch_where_kinds(nbr)
    return space._kinds[key]


def torch_where_kinds(nbr):
    torch = _torch()
    return torch.where(nbr >= 0, torch.zeros_like(nbr), torch.full_like(nbr, _lib.BC_VELOCITY_DIRICHLET)
                       ).to(torch.int32).contiguous()


def apply_viscous_helmholtz(space: GeneralSpace2D, u, gamma0_dt: float, nu: float,
                            bcs: GeneralBCs):
    """(gamma0/dt) M u + SIP of -div(2 nu eps(u)) (operators.py:418-491)."""
    t, is_np, shape = _field(space, u, 2)
    out = _torch().empty_like(t)
    prm = _params(space, 3, bcs)
    prm.gamma0_dt, prm.nu = float(gamma0_dt), float(nu)
    _op(space, prm, t, out)
    return _result(space, out, is_np, shape, 2)


def face_penalty_slots(space: GeneralSpace2D, tau_c_f):
    """Reference per-interior-face tau_C (mesh.interior order) -> [e][4]."""
    f = space.mesh.interior
    tau_c_f = np.asarray(tau_c_f, dtype=np.float64)
    if tau_c_f.shape != np.shape(f.em):
        raise ValueError(f"tau_c_f needs one entry per interior face ({np.size(f.em)})")
    out = np.zeros((space.n_elements, 4))
    out[np.asarray(f.em), np.asarray(f.sm)] = tau_c_f
    out[np.asarray(f.ep), np.asarray(f.sp)] = tau_c_f
    return out


def apply_projection_operator(space: GeneralSpace2D, w, tau_d_e, tau_c_f):
    """M + tau_D div-div + tau_C interior jump penalty (operators.py:372-412).
    tau_c_f: per interior face (reference order) or a [e][4] CUDA tensor."""
    torch = _torch()
    t, is_np, shape = _field(space, w, 2)
    out = torch.empty_like(t)
    prm = _lib.G2Params()
    prm.op = 4
    prm.kind = ctypes.c_void_p(_all_interior_kinds(space).data_ptr())
    keep = []
    if tau_d_e is not None:
        td = tau_d_e if isinstance(tau_d_e, torch.Tensor) else torch.as_tensor(
            np.asarray(tau_d_e, dtype=np.float64)).to("cuda")
        td = td.contiguous()
        keep.append(td)
        prm.tau_d = ctypes.c_void_p(td.data_ptr())
    if tau_c_f is not None:
        tc = tau_c_f if isinstance(tau_c_f, torch.Tensor) else torch.as_tensor(
            face_penalty_slots(space, tau_c_f)).to("cuda")
        tc = tc.contiguous()
        keep.append(tc)
        prm.tau_c = ctypes.c_void_p(tc.data_ptr())
    _op(space, prm, t, out)
    return _result(space, out, is_np, shape, 2)


def eval_divergence_rhs(space: GeneralSpace2D, u, bcs: GeneralBCs, scale: float,
                        form: str = "standard"):
    """a(q, u) scaled (operators.py:265-316)."""
    forms = {"standard": 0, "weak": 1, "strong": 2}
    if form not in forms:
        raise ValueError(f"unknown divergence form {form!r}")
    t, is_np, shape = _field(space, u, 2)
    out = _torch().empty(space.n_dofs, dtype=_torch().float64, device="cuda")
    prm = _params(space, 6, bcs)
    prm.scale, prm.form = float(scale), forms[form]
    _op(space, prm, t, out)
    if is_np:
        return space.from_element_major(out.cpu().numpy(), 1)
    return out


def eval_pressure_gradient_rhs(space: GeneralSpace2D, p, bcs: GeneralBCs, scale: float,
                               form: str = "standard"):
    """b(v, p) scaled (operators.py:322-366)."""
    forms = {"standard": 0, "weak": 1}
    if form not in forms:
        raise ValueError(f"unknown pressure-gradient form {form!r}")
    t, is_np, shape = _field(space, p, 1)
    out = _torch().empty(2 * space.n_dofs, dtype=_torch().float64, device="cuda")
    prm = _params(space, 7, bcs)
    prm.scale, prm.form = float(scale), forms[form]
    _op(space, prm, t, out)
    if is_np:
        return space.from_element_major(out.cpu().numpy(), 2)
    return out


def compute_vorticity(space: GeneralSpace2D, u):
    """Element-local L2 projection of du2/dx - du1/dy (operators.py:610-618)."""
    torch = _torch()
    t, is_np, shape = _field(space, u, 2)
    r = torch.empty(space.n_dofs, dtype=torch.float64, device="cuda")
    prm = _lib.G2Params()
    prm.op = 8
    prm.kind = ctypes.c_void_p(_all_interior_kinds(space).data_ptr())
    _op(space, prm, t, r)
    out = inverse_mass_apply(space, r)
    if is_np:
        return space.from_element_major(out.cpu().numpy(), 1)
    return out


def eval_convective_rhs(space: GeneralSpace2D, bcs: GeneralBCs, history, betas, times,
                        t_np1: float, body_force=None):
    """sum_i beta_i [(grad v, u u) - (v, F*.n)] + (v, f) with the local
    Lax-Friedrichs flux on the over-integration rule (operators.py:533-594);
    Dirichlet data g(x, t_i) enters the mirror state 2g - u (a None callable
    means homogeneous data)."""
    torch = _torch()
    if len(history) < 1 or len(history) > 4:
        raise ValueError("need 1..4 history levels")
    if len(times) < len(history) or len(betas) < len(history):
        raise ValueError("need one beta and one time per history level")
    h, g, _, _ = space.over()
    nq = g.jxw.shape[0]
    ne = space.n_elements
    fields = [_field(space, u, 2) for u in history]
    is_np, shape = fields[0][1], fields[0][2]
    out = torch.empty(2 * space.n_dofs, dtype=torch.float64, device="cuda")
    prm = _params(space, 5, bcs)
    prm.n_hist = len(history)
    keep = []
    for j, (t, _, _) in enumerate(fields):
        prm.hist[j] = ctypes.c_void_p(t.data_ptr())
        prm.beta[j] = float(betas[j])
        gd = None
        for tag, bc in bcs.dirichlet:
            if bc.g is None:
                continue
            eb, sb = space.b_groups[tag]
            x = g.xf[:, sb, eb]                          # (2, nb, q)
            gu = np.asarray(bc.g(x, times[j]), dtype=np.float64)
            if gd is None:
                gd = np.zeros((ne, 4, 2, nq))
            gd[eb, sb] = np.moveaxis(gu, 0, 1)
        if gd is not None:
            tg = torch.as_tensor(gd).to("cuda")
            keep.append(tg)
            prm.gdata[j] = ctypes.c_void_p(tg.data_ptr())
    if body_force is not None:
        f = np.asarray(body_force(g.xq, t_np1), dtype=np.float64)  # (2, q, ne, q)
        tb = torch.as_tensor(np.ascontiguousarray(f.transpose(0, 2, 1, 3))).to("cuda")
        keep.append(tb)
        prm.body = ctypes.c_void_p(tb.data_ptr())
    _op(space, prm, None, out, handle=h)
    if is_np:
        return space.from_element_major(out.cpu().numpy(), 2).reshape(shape)
    return out.view(shape)


# ---------------------------------------------------------------------------
# boundary-data right-hand sides: the data callables are the caller's Python
# functions, sampled on the host at the face Gauss points (geometry xf);
# traces of device fields and the lifts run on the device

def _face_data(space, groups, ncomp):
    """[e][4][ncomp][q] device array from (tag, fn(x) -> (ncomp, nb, q)) entries,
    or None when there is no data."""
    g = space.geom
    out = None
    for tag, fn in groups:
        eb, sb = space.b_groups[tag]
        val = np.asarray(fn(g.xf[:, sb, eb]), dtype=np.float64)
        if val.ndim == 2:
            val = val[None]
        if out is None:
            out = np.zeros((space.n_elements, 4, ncomp, space.n_q))
        out[eb, sb, :val.shape[0]] = np.moveaxis(val, 0, 1)
    if out is None:
        return None
    return _torch().as_tensor(out).to("cuda")


def _like_out(space, out, ncomp, like):
    torch = _torch()
    if isinstance(like, torch.Tensor) or (isinstance(like, str) and like == "device"):
        return out
    return space.from_element_major(out.cpu().numpy(), ncomp)


def gp_dirichlet_rhs(space: GeneralSpace2D, bcs: GeneralBCs, t: float, tau_scale: float = 1.0,
                     like=None):
    """Pressure-Dirichlet data g_p on velocity-Neumann faces (operators.py:241-259)."""
    torch = _torch()
    fd = _face_data(space, [(tag, lambda x, bc=bc: bc.g_p(x, t)) for tag, bc in bcs.neumann
                            if bc.g_p is not None], 1)
    out = torch.empty(space.n_dofs, dtype=torch.float64, device="cuda")
    prm = _params(space, 10, bcs)
    prm.tau_scale = float(tau_scale)
    prm.fdata = ctypes.c_void_p(fd.data_ptr() if fd is not None else 0)
    _op(space, prm, None, out)
    return _like_out(space, out, 1, like)


def viscous_rhs_bc(space: GeneralSpace2D, bcs: GeneralBCs, t: float, nu: float, like=None):
    """Boundary-data terms of the viscous solve (operators.py:494-527)."""
    torch = _torch()
    groups = []
    for tag, bc in bcs.dirichlet:
        if bc.g is not None:
            groups.append((tag, lambda x, bc=bc: np.concatenate(
                [np.asarray(bc.g(x, t), dtype=np.float64), np.zeros((1,) + x.shape[1:])])))
    for tag, bc in bcs.neumann:
        if bc.h is None and bc.g_p is None:
            continue
        def fn(x, bc=bc):
            h = np.asarray(bc.h(x, t), dtype=np.float64) if bc.h is not None else \
                np.zeros((2,) + x.shape[1:])
            gp = np.asarray(bc.g_p(x, t), dtype=np.float64) if bc.g_p is not None else \
                np.zeros(x.shape[1:])
            return np.concatenate([h, gp[None]])
        groups.append((tag, fn))
    fd = _face_data(space, groups, 3)
    out = torch.empty(2 * space.n_dofs, dtype=torch.float64, device="cuda")
    prm = _params(space, 11, bcs)
    prm.nu = float(nu)
    prm.fdata = ctypes.c_void_p(fd.data_ptr() if fd is not None else 0)
    _op(space, prm, None, out)
    return _like_out(space, out, 2, like)


def eval_pressure_neumann_rhs(space: GeneralSpace2D, bcs: GeneralBCs, history, vorticity_history,
                              betas, nu: float, t_np1: float, body_force=None, like=None):
    """Consistent pressure Neumann data on velocity-Dirichlet faces
    (operators.py:621-672): -(dg/dt + sum_i beta_i (div(u u) + nu curl w)
    - f) . n against the pressure test functions."""
    torch = _torch()
    if len(history) < 1 or len(history) > 4:
        raise ValueError("need 1..4 history levels")
    if len(vorticity_history) < len(history) or len(betas) < len(history):
        raise ValueError("need one vorticity level and one beta per history level")
    out = torch.zeros(space.n_dofs, dtype=torch.float64, device="cuda")
    if not bcs.dirichlet:
        return _like_out(space, out, 1, like if like is not None else
                         (history[0] if isinstance(history[0], torch.Tensor) else None))
    groups = []
    for tag, bc in bcs.dirichlet:
        def fn(x, bc=bc):
            h = np.asarray(bc.dg_dt(x, t_np1), dtype=np.float64) if bc.dg_dt is not None else \
                np.zeros((2,) + x.shape[1:])
            if body_force is not None:
                h = h - np.asarray(body_force(x, t_np1), dtype=np.float64)
            return h
        if bc.dg_dt is not None or body_force is not None:
            groups.append((tag, fn))
    fd = _face_data(space, groups, 2)
    us = [_field(space, u, 2)[0] for u in history]
    ws = [_field(space, w, 1)[0] for w in vorticity_history[:len(history)]]
    prm = _params(space, 12, bcs)
    prm.nu = float(nu)
    prm.n_hist = len(us)
    for j, (u, w) in enumerate(zip(us, ws)):
        prm.hist[j] = ctypes.c_void_p(u.data_ptr())
        prm.vort[j] = ctypes.c_void_p(w.data_ptr())
        prm.beta[j] = float(betas[j])
    prm.fdata = ctypes.c_void_p(fd.data_ptr() if fd is not None else 0)
    _op(space, prm, None, out)
    if like is None and isinstance(history[0], torch.Tensor):
        like = "device"
    return _like_out(space, out, 1, like)


# ---------------------------------------------------------------------------
# zero-mean projections, penalty parameters (device tensors)

def _basis_integrals(space: GeneralSpace2D):
    """w_i = integral of l_i = (M 1)_i, element-major (device), cached."""
    if getattr(space, "_wint", None) is None:
        torch = _torch()
        ones = torch.ones(space.n_dofs, dtype=torch.float64, device="cuda")
        space._wint = mass_apply(space, ones)
        space._area = float(space.geom.volumes.sum())
    return space._wint, space._area


def zero_mean_project(space: GeneralSpace2D, p):
    """Subtract the L2 mean (solvers.py:179-184)."""
    t, is_np, shape = _field(space, p, 1)
    w, area = _basis_integrals(space)
    out = t - (t @ w) / area
    return _result(space, out, is_np, shape, 1)


def zero_mean_project_dual(space: GeneralSpace2D, b):
    """b - (sum b / |Omega|) w, w_i = integral of l_i (solvers.py:187-198)."""
    t, is_np, shape = _field(space, b, 1)
    w, area = _basis_integrals(space)
    out = t - (t.sum() / area) * w
    return _result(space, out, is_np, shape, 1)


def compute_penalty_parameters(space: GeneralSpace2D, u, dt: float, cfl: float, cfg):
    """tau_D per cell and tau_C per (cell, slot) (operators.py:736-755; 2D
    h = sqrt(V)); tau_c comes back in the [e][4] layout the general
    apply_projection_operator takes (0 on boundary sides)."""
    if cfl <= 0:
        raise ValueError(f"CFL must be positive, got {cfl}")
    torch = _torch()
    t, _, _ = _field(space, u, 2)
    w, _ = _basis_integrals(space)
    ne, npl = space.n_elements, space.n_local
    uw = (t.view(2, ne, npl) * w.view(1, ne, npl)).sum(dim=2)
    vol = torch.as_tensor(space.geom.volumes, device="cuda")
    norm = torch.hypot(uw[0], uw[1]) / vol
    td = tc = None
    if cfg.uses_divdiv:
        td = (cfg.zeta_d_star / cfl) * norm * torch.sqrt(vol) * dt
    if cfg.uses_jump:
        tce = (cfg.zeta_c_star / cfl) * norm * dt
        nbr = space._d["nbr"]
        inner = nbr >= 0
        tc = torch.where(inner, 0.5 * (tce[:, None] + tce[nbr.clamp(min=0)]),
                         torch.zeros(nbr.shape, dtype=torch.float64, device="cuda"))
    return td, tc


# ---------------------------------------------------------------------------
# geometric multigrid on refined general meshes (multigrid.py:33-175)

class Transfer2D:
    """Polynomial embedding between a general space and its refinement
    (multigrid.py:33-73): needs the fine mesh's parent / quadrant links."""

    def __init__(self, coarse: GeneralSpace2D, fine: GeneralSpace2D):
        if getattr(fine.mesh, "parent", None) is None:
            raise ValueError("fine mesh lacks parent links; build the hierarchy by refinement")
        if coarse.k != fine.k:
            raise ValueError("multigrid levels need the same degree")
        torch = _torch()
        parent = np.asarray(fine.mesh.parent, np.int64)
        quad = np.asarray(fine.mesh.quadrant, np.int32)
        children = -np.ones((coarse.n_elements, 4), np.int64)
        children[parent, quad] = np.arange(fine.n_elements)
        self.coarse, self.fine = coarse, fine
        self._parent = torch.as_tensor(parent).to("cuda")
        self._quad = torch.as_tensor(quad).to("cuda")
        self._children = torch.as_tensor(children).to("cuda")

    def _call(self, prolong, x, out, add=0):
        P = lambda t: ctypes.c_void_p(t.data_ptr())
        _lib.call("dg_g2_transfer", self.fine.k, int(prolong), self.fine.n_elements,
                  P(self._parent), P(self._quad), self.coarse.n_elements, P(self._children),
                  P(x), P(out), int(add), _stream())

    def prolong(self, xc, out=None, add=False):
        t, is_np, _ = _field(self.coarse, xc, 1)
        torch = _torch()
        if out is None:
            out = torch.empty(self.fine.n_dofs, dtype=torch.float64, device="cuda")
        self._call(True, t, out, int(add))
        return self.fine.from_element_major(out.cpu().numpy(), 1) if is_np else out

    def restrict(self, xf):
        torch = _torch()
        t, is_np, _ = _field(self.fine, xf, 1)
        out = torch.empty(self.coarse.n_dofs, dtype=torch.float64, device="cuda")
        self._call(False, t, out)
        return self.coarse.from_element_major(out.cpu().numpy(), 1) if is_np else out


class GeneralMultigrid:
    """V-cycle preconditioner on a refined general hierarchy (reference
    MultigridHierarchy, multigrid.py:76-151): Chebyshev(degree, range)-Jacobi
    smoothing with the device operator, a seeded 20-step Lanczos lambda_max
    per level, the fixed-count coarse Chebyshev; every operation is a device
    kernel.  ``vcycle`` drops into ``solvers.pcg(op, mg.vcycle, b)``."""

    def __init__(self, spaces, bc_spec, tau_scale: float = 1.0, degree: int = 5,
                 smoothing_range: float = 20.0, coarse_tol: float = 1e-3, est_iters: int = 20,
                 safety: float = 1.1, seed: int = 987, project=None):
        import math
        from .solvers import ChebyshevConfig, eigen_estimate_via_cg
        if len(spaces) < 1:
            raise ValueError("hierarchy needs at least one level")
        rng = np.random.default_rng(seed)
        self.levels = []
        self.tau_scale = tau_scale
        for lvl, space in enumerate(spaces):
            bcs = bc_spec.resolve(space)
            op = (lambda s, b: lambda p: apply_pressure_laplace(s, p, b, tau_scale))(space, bcs)
            diag = laplace_diagonal(space, bcs, tau_scale)
            m, ne = space.k + 1, space.n_elements
            seed_vec = _torch().as_tensor(space.to_element_major(
                rng.standard_normal((m, ne, m)), 1).ravel()).to("cuda")
            est_op = op
            if project is not None:
                seed_vec = project(space, seed_vec)
                est_op = (lambda o, s: lambda p: project(s, o(p)))(op, space)
            lmax, lmin = eigen_estimate_via_cg(est_op, diag, seed_vec, est_iters)
            level = {"space": space, "op": op, "diag": diag,
                     "cheb": ChebyshevConfig(degree, smoothing_range, safety * lmax),
                     "lambda_max": safety * lmax}
            if lvl == 0:
                kappa = (safety * lmax) / max(lmin / safety, 1e-12 * lmax)
                q = (math.sqrt(kappa) - 1.0) / (math.sqrt(kappa) + 1.0)
                n = math.ceil(math.log(2.0 / coarse_tol) / -math.log(max(q, 1e-12)))
                level["coarse_iters"] = max(n, 1)
                level["coarse_range"] = kappa
            self.levels.append(level)
        self.transfers = [Transfer2D(c["space"], f["space"])
                          for c, f in zip(self.levels[:-1], self.levels[1:])]

    @property
    def n_levels(self):
        return len(self.levels)

    def vcycle(self, b):
        top = self.levels[-1]["space"]
        t, is_np, shape = _field(top, b, 1)
        x = self._cycle(t, self.n_levels - 1)
        return top.from_element_major(x.cpu().numpy(), 1).reshape(shape) if is_np else x.view(shape)

    def _cycle(self, b, lvl):
        from .solvers import ChebyshevConfig, chebyshev_smooth
        lev = self.levels[lvl]
        if lvl == 0:
            cfg = ChebyshevConfig(lev["coarse_iters"], max(lev["coarse_range"], 1.0 + 1e-8),
                                  lev["cheb"].lambda_max)
            return chebyshev_smooth(lev["op"], lev["diag"], cfg, b)
        x = chebyshev_smooth(lev["op"], lev["diag"], lev["cheb"], b)
        r = b - lev["op"](x)
        tr = self.transfers[lvl - 1]
        xc = self._cycle(tr.restrict(r), lvl - 1)
        tr.prolong(xc, out=x, add=True)
        return chebyshev_smooth(lev["op"], lev["diag"], lev["cheb"], b, x)
