"""numpy restatement of the reference DG operators, DIM in {2, 3}.

TEST INFRASTRUCTURE -- the checker, never the product (see oracle/__init__.py).

This module restates, in dimension-generic numpy, the algorithm of the
reference package ``dgins`` (``/root/reference/pkg/src/dgins``; all
citations below are ``file:line`` into that tree).  The reference is
2D-only; the restatement keeps its structure (sum-factorised evaluation at
Gauss points, reference-gradient -> physical gradient via J^-T, face traces
per slot, gather/scatter of interior faces without accumulation, adjoint
lifts) and generalises the slot numbering from 4 to 2*DIM slots.

Layout (differs from the reference's ``(m, ne, m)`` kernel layout): a scalar
field is an array ``(ne,) + (m,)*DIM`` with axes ``(cell, [z,] y, x)`` -- the
element-major serialisation of ``FieldVector.element_major``
(spaces.py:49-51), extended to 3D.  Direction d (0=x, 1=y, 2=z) lives on
array axis ``DIM - d``.  Cells are numbered e = ix + nx*(iy + ny*iz)
(mesh.py:320-325 extended).  Face slot 2d is xi_d = -1, slot 2d+1 is
xi_d = +1 (kernels.py:224-227 extended).

Geometry is restricted to the meshes the hot path runs on: axis-aligned
boxes with per-axis (optionally tanh-graded) vertex coordinates, k_geo = 1.
On such cells the reference's general formulas (geometry.py:29-87: JxW,
J^-T, Nanson normals) reduce to per-cell constants, which are broadcast to
quadrature points here so the operator code keeps the reference's general
structure.
"""

from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

# ---------------------------------------------------------------------------
# 1D quadrature (reference quadrature.py)

_NEWTON_TOL = 1e-15
_NEWTON_MAXIT = 100


@dataclass(frozen=True)
class QuadratureRule:
    points: np.ndarray
    weights: np.ndarray

    @property
    def n(self):
        return len(self.points)


def _legendre_eval(n, x):
    """P_n and P_n' by the three-term recurrence (quadrature.py:31-45)."""
    p0 = np.ones_like(x)
    if n == 0:
        return p0, np.zeros_like(x)
    p1 = x.copy()
    for j in range(1, n):
        p0, p1 = p1, ((2 * j + 1) * x * p1 - j * p0) / (j + 1)
    with np.errstate(divide="ignore", invalid="ignore"):
        dp = n * (x * p1 - p0) / (x * x - 1.0)
    at_end = np.abs(np.abs(x) - 1.0) < 1e-300
    if at_end.any():
        dp = np.where(at_end, np.sign(x) ** (n - 1) * n * (n + 1) / 2.0, dp)
    return p1, dp


def gauss_rule(n):
    """Gauss-Legendre rule by Newton from Chebyshev seeds (quadrature.py:48-71)."""
    if n < 1:
        raise ValueError(f"need at least one quadrature point, got n={n}")
    if n == 1:
        return QuadratureRule(np.array([0.0]), np.array([2.0]))
    x = -np.cos(np.pi * (np.arange(n) + 0.75) / (n + 0.5))
    for _ in range(_NEWTON_MAXIT):
        p, dp = _legendre_eval(n, x)
        dx = p / dp
        x -= dx
        if np.max(np.abs(dx)) < _NEWTON_TOL:
            break
    p, dp = _legendre_eval(n, x)
    x -= p / dp
    x = 0.5 * (x - x[::-1])
    _, dp = _legendre_eval(n, x)
    w = 2.0 / ((1.0 - x * x) * dp * dp)
    return QuadratureRule(x, w)


def gll_nodes(k):
    """+-1 plus the roots of P_k' (quadrature.py:74-95)."""
    if k < 1:
        raise ValueError(f"polynomial degree must be >= 1, got k={k}")
    if k == 1:
        return np.array([-1.0, 1.0])
    x = -np.cos(np.pi * (np.arange(1, k) + 0.26) / k)
    for _ in range(_NEWTON_MAXIT):
        p, dp = _legendre_eval(k, x)
        ddp = (2 * x * dp - k * (k + 1) * p) / (1.0 - x * x)
        dx = dp / ddp
        x -= dx
        if np.max(np.abs(dx)) < _NEWTON_TOL:
            break
    x = 0.5 * (x - x[::-1])
    return np.concatenate(([-1.0], x, [1.0]))


# ---------------------------------------------------------------------------
# 1D Lagrange tables (reference basis.py)

def lagrange_values(nodes, x):
    """V[q, i] = l_i(x_q), barycentric (basis.py:15-35)."""
    nodes = np.asarray(nodes, dtype=float)
    x = np.atleast_1d(np.asarray(x, dtype=float))
    diff = nodes[None, :] - nodes[:, None]
    np.fill_diagonal(diff, 1.0)
    bw = 1.0 / np.prod(diff, axis=1)
    v = np.empty((len(x), len(nodes)))
    for q, xq in enumerate(x):
        d = xq - nodes
        hit = np.isclose(d, 0.0, atol=1e-14)
        if hit.any():
            v[q] = 0.0
            v[q, np.argmax(hit)] = 1.0
        else:
            t = bw / d
            v[q] = t / t.sum()
    return v


def lagrange_derivatives(nodes, x):
    """D[q, i] = l_i'(x_q) via the nodal differentiation matrix (basis.py:38-58)."""
    nodes = np.asarray(nodes, dtype=float)
    n = len(nodes)
    diff = nodes[None, :] - nodes[:, None]
    np.fill_diagonal(diff, 1.0)
    bw = 1.0 / np.prod(diff, axis=1)
    dn = np.empty((n, n))
    for j in range(n):
        for i in range(n):
            if i != j:
                dn[j, i] = bw[i] / bw[j] / (nodes[j] - nodes[i])
        dn[j, j] = 0.0
        dn[j, j] = -dn[j].sum()
    return lagrange_values(nodes, x) @ dn


class Basis1D:
    """Degree-k GLL Lagrange basis bound to a Gauss rule (basis.py:61-84)."""

    def __init__(self, k, rule):
        self.k = k
        self.nodes = gll_nodes(k)
        self.rule = rule
        self.S = lagrange_values(self.nodes, rule.points)
        self.D = lagrange_derivatives(self.nodes, rule.points)
        self.left_value = lagrange_values(self.nodes, np.array([-1.0]))[0]
        self.right_value = lagrange_values(self.nodes, np.array([1.0]))[0]
        self.left_deriv = lagrange_derivatives(self.nodes, np.array([-1.0]))[0]
        self.right_deriv = lagrange_derivatives(self.nodes, np.array([1.0]))[0]
        self.S_inv = np.linalg.inv(self.S) if rule.n == k + 1 else None

    @property
    def n_q(self):
        return self.rule.n

    def end_value(self, s):
        return self.right_value if s else self.left_value

    def end_deriv(self, s):
        return self.right_deriv if s else self.left_deriv


_basis_cache = {}


def get_basis(k, n_q):
    """Cached Basis1D (basis.py:90-95)."""
    key = (k, n_q)
    if key not in _basis_cache:
        _basis_cache[key] = Basis1D(k, gauss_rule(n_q))
    return _basis_cache[key]


def convective_rule_points(k):
    """floor(3k/2)+1 over-integration points (basis.py:103-105)."""
    return (3 * k) // 2 + 1


# ---------------------------------------------------------------------------
# sum-factorisation kernels (reference kernels.py), DIM-generic

def _ax(dim, d):
    """Array axis of direction d in a (ne, [z,] y, x) cell array."""
    return dim - d


def _contract(F, T, ax):
    """out[..., q(ax), ...] = sum_i T[q, i] F[..., i(ax), ...] (kernels.py:47-58)."""
    return np.moveaxis(np.tensordot(F, T, axes=([ax], [1])), -1, ax)


def vol_values(F, b, dim):
    """kernels.py:61-63."""
    for d in range(dim):
        F = _contract(F, b.S, _ax(dim, d))
    return F


def vol_gradients(F, b, dim):
    """Reference gradients d/dxi_d at tensor Gauss points (kernels.py:66-79)."""
    out = []
    for dg in range(dim):
        G = F
        for d in range(dim):
            G = _contract(G, b.D if d == dg else b.S, _ax(dim, d))
        out.append(G)
    return out


def vol_integrate_values(Q, b, dim):
    """Adjoint of vol_values (kernels.py:82-84)."""
    for d in range(dim):
        Q = _contract(Q, b.S.T, _ax(dim, d))
    return Q


def vol_integrate_gradients(G, b, dim):
    """Adjoint of vol_gradients (kernels.py:87-92)."""
    out = 0.0
    for dg in range(dim):
        H = G[dg]
        for d in range(dim):
            H = _contract(H, b.D.T if d == dg else b.S.T, _ax(dim, d))
        out = out + H
    return out


def apply_inverse_mass(R, b, jxw, dim):
    """Exact M^-1 via S^-1 (kernels.py:95-108)."""
    if b.S_inv is None:
        raise ValueError("inverse mass requires the n_q = k + 1 Gauss rule")
    Si = b.S_inv
    Q = R
    for d in range(dim):
        Q = _contract(Q, Si.T, _ax(dim, d))
    Q = Q / jxw
    for d in range(dim):
        Q = _contract(Q, Si, _ax(dim, d))
    return Q


def apply_mass(F, b, jxw, dim):
    """kernels.py:111-113."""
    return vol_integrate_values(vol_values(F, b, dim) * jxw, b, dim)


def _tangential(dim, d):
    """Directions of the face-array axes 1..dim-1 for a face normal to d."""
    return [dd for dd in range(dim - 1, -1, -1) if dd != d]


def face_values(F, b, dim):
    """Value traces on all 2*dim slots (kernels.py:119-130)."""
    out = []
    for d in range(dim):
        for s in (0, 1):
            T = np.tensordot(F, b.end_value(s), axes=([_ax(dim, d)], [0]))
            for j, dd in enumerate(_tangential(dim, d)):
                T = _contract(T, b.S, 1 + j)
            out.append(T)
    return np.stack(out)


def face_gradients(F, b, dim):
    """Reference-gradient traces on all slots, list over components
    (kernels.py:133-156)."""
    comps = []
    for dg in range(dim):
        per_slot = []
        for d in range(dim):
            for s in (0, 1):
                row = b.end_deriv(s) if dg == d else b.end_value(s)
                T = np.tensordot(F, row, axes=([_ax(dim, d)], [0]))
                for j, dd in enumerate(_tangential(dim, d)):
                    T = _contract(T, b.D if dd == dg else b.S, 1 + j)
                per_slot.append(T)
        comps.append(np.stack(per_slot))
    return comps


def _expand(T, row, ax):
    """Outer product of face data with a 1D row along cell axis ax."""
    T = np.expand_dims(T, ax)
    shape = [1] * T.ndim
    shape[ax] = len(row)
    return T * row.reshape(shape)


def face_lift_values(V, b, out, dim):
    """Adjoint of face_values, accumulated (kernels.py:159-168)."""
    for d in range(dim):
        for s in (0, 1):
            T = V[2 * d + s]
            for j, dd in enumerate(_tangential(dim, d)):
                T = _contract(T, b.S.T, 1 + j)
            out += _expand(T, b.end_value(s), _ax(dim, d))
    return out


def face_lift_gradients(G, b, out, dim):
    """Adjoint of face_gradients, accumulated (kernels.py:171-186)."""
    for dg in range(dim):
        for d in range(dim):
            for s in (0, 1):
                T = G[dg][2 * d + s]
                for j, dd in enumerate(_tangential(dim, d)):
                    T = _contract(T, b.D.T if dd == dg else b.S.T, 1 + j)
                row = b.end_deriv(s) if dg == d else b.end_value(s)
                out += _expand(T, row, _ax(dim, d))
    return out


# ---------------------------------------------------------------------------
# structured box meshes (reference mesh.py)

def grading_map(s, gamma, delta=1.0):
    """delta*tanh(gamma(2s-1))/tanh(gamma) (mesh.py:32-43)."""
    s = np.asarray(s, dtype=float)
    if gamma < 0:
        raise ValueError(f"grading parameter must be >= 0, got {gamma}")
    if gamma == 0.0:
        return delta * (2.0 * s - 1.0)
    return delta * np.tanh(gamma * (2.0 * s - 1.0)) / np.tanh(gamma)


TAG_NAMES = ("xmin", "xmax", "ymin", "ymax", "zmin", "zmax")


@dataclass
class InteriorFaces:
    em: np.ndarray
    sm: np.ndarray
    ep: np.ndarray
    sp: np.ndarray

    @property
    def n(self):
        return len(self.em)


@dataclass
class BoundaryFaces:
    elem: np.ndarray
    slot: np.ndarray
    tag: np.ndarray

    @property
    def n(self):
        return len(self.elem)


class BoxMesh:
    """Axis-aligned tensor-product box (mesh.py:279-351 generalised to DIM)."""

    def __init__(self, extents, counts, grading=None, delta=1.0,
                 periodic=None):
        dim = len(counts)
        if dim not in (2, 3) or len(extents) != dim:
            raise ValueError("need 2 or 3 axes")
        grading = tuple(grading) if grading is not None else (0.0,) * dim
        periodic = tuple(periodic) if periodic is not None else (False,) * dim
        for d in range(dim):
            if counts[d] < 1:
                raise ValueError(f"counts must be >= 1 per axis, got {counts}")
            if extents[d][1] <= extents[d][0]:
                raise ValueError(f"extents must have positive size, got {extents}")
            if grading[d] < 0:
                raise ValueError("grading must be >= 0")
            if periodic[d] and grading[d] > 0:
                raise ValueError(f"axis {d}: grading would break periodic "
                                 "translation matching across the wrap")
        self.dim = dim
        self.counts = tuple(int(c) for c in counts)
        self.extents = tuple(tuple(map(float, e)) for e in extents)
        self.grading = grading
        self.periodic = periodic

        def axis_nodes(n, gamma, lo, hi):   # mesh.py:306-310
            s = np.linspace(0.0, 1.0, n + 1)
            f = grading_map(s, gamma, delta)
            return lo + (f - f[0]) / (f[-1] - f[0]) * (hi - lo)

        self.axis_vertices = [axis_nodes(self.counts[d], grading[d],
                                         *self.extents[d]) for d in range(dim)]
        ne = int(np.prod(self.counts))
        self.n_elements = ne
        e = np.arange(ne)
        idx = []
        rem = e
        for d in range(dim):
            idx.append(rem % self.counts[d])
            rem = rem // self.counts[d]
        self.cell_index = np.stack(idx)               # (dim, ne)
        self.h = np.stack([np.diff(self.axis_vertices[d])[idx[d]]
                           for d in range(dim)], axis=1)   # (ne, dim)
        self.lower = np.stack([self.axis_vertices[d][idx[d]]
                               for d in range(dim)], axis=1)
        stride = np.cumprod((1,) + self.counts[:-1])

        em, sm, ep, sp = [], [], [], []
        be, bs, bt = [], [], []
        for d in range(dim):
            n = self.counts[d]
            lo = e[idx[d] < n - 1]
            em.append(lo); sm.append(np.full(lo.size, 2 * d + 1))
            ep.append(lo + stride[d]); sp.append(np.full(lo.size, 2 * d))
            last = e[idx[d] == n - 1]
            first = e[idx[d] == 0]
            if periodic[d]:
                em.append(last); sm.append(np.full(last.size, 2 * d + 1))
                ep.append(last - (n - 1) * stride[d])
                sp.append(np.full(last.size, 2 * d))
            else:
                be.append(first); bs.append(np.full(first.size, 2 * d))
                bt.append(np.full(first.size, 2 * d))
                be.append(last); bs.append(np.full(last.size, 2 * d + 1))
                bt.append(np.full(last.size, 2 * d + 1))
        cat = lambda a: (np.concatenate(a).astype(np.int64) if a
                         else np.zeros(0, np.int64))
        self.interior = InteriorFaces(cat(em), cat(sm), cat(ep), cat(sp))
        self.boundary = BoundaryFaces(cat(be), cat(bs), cat(bt))
        self.tag_names = list(TAG_NAMES[:2 * dim])


def build_box_mesh(extents, counts, grading=None, delta=1.0, periodic=None):
    return BoxMesh(extents, counts, grading, delta, periodic)


# ---------------------------------------------------------------------------
# geometry (reference geometry.py), Cartesian cells

class Geometry:
    """JxW, J^-T, normals, surface JxW at the points of one rule
    (geometry.py:29-87, affine axis-aligned cells)."""

    def __init__(self, mesh, n_q):
        dim = mesh.dim
        self.dim = dim
        self.n_q = n_q
        w = gauss_rule(n_q).weights
        ne = mesh.n_elements
        h = mesh.h
        det = np.prod(h / 2.0, axis=1)                       # (ne,)
        if not (det > 0).all():
            raise ValueError("non-positive mapping Jacobian")
        wt = 1.0
        for _ in range(dim):
            wt = np.multiply.outer(wt, w)
        self.jxw = det.reshape((ne,) + (1,) * dim) * wt      # (ne, q..)
        jit = np.zeros((dim, dim, ne) + (1,) * dim)
        for a in range(dim):
            jit[a, a] = (2.0 / h[:, a]).reshape((ne,) + (1,) * dim)
        self.jinvT = jit
        self.volumes = np.prod(h, axis=1)
        # faces: per slot normal (+-e_d), J^-T, surface JxW
        wf = 1.0
        for _ in range(dim - 1):
            wf = np.multiply.outer(wf, w)
        self.normal = np.zeros((dim, 2 * dim, ne) + (1,) * (dim - 1))
        self.sjxw = np.empty((2 * dim, ne) + (n_q,) * (dim - 1))
        self.face_areas = np.empty((2 * dim, ne))
        self.jinvT_f = jit[..., 0]                            # (dim, dim, ne, 1..)
        for d in range(dim):
            tang = [dd for dd in range(dim) if dd != d]
            fdet = np.prod(h[:, tang] / 2.0, axis=1)
            for s in (0, 1):
                self.normal[d, 2 * d + s] = 2.0 * s - 1.0
                self.sjxw[2 * d + s] = fdet.reshape((ne,) + (1,) * (dim - 1)) * wf
                self.face_areas[2 * d + s] = np.prod(h[:, tang], axis=1)
        self.xq = None


def compute_tau_ip(mesh, geom, k):
    """tau_e = (k+1)^2 (A_int/2 + A_bnd)/V; interior max; boundary own
    (geometry.py:90-108)."""
    ne = mesh.n_elements
    a_int = np.zeros(ne)
    a_bnd = np.zeros(ne)
    f = mesh.interior
    np.add.at(a_int, f.em, geom.face_areas[f.sm, f.em])
    np.add.at(a_int, f.ep, geom.face_areas[f.sp, f.ep])
    b = mesh.boundary
    np.add.at(a_bnd, b.elem, geom.face_areas[b.slot, b.elem])
    tau_e = (k + 1) ** 2 * (0.5 * a_int + a_bnd) / geom.volumes
    return tau_e, np.maximum(tau_e[f.em], tau_e[f.ep]), tau_e[b.elem]


# ---------------------------------------------------------------------------
# space + boundary conditions (reference spaces.py, operators.py:77-131)

class DgSpace:
    def __init__(self, mesh, k, n_q_over=None):
        if k < 1:
            raise ValueError(f"polynomial degree must be >= 1, got k={k}")
        self.mesh = mesh
        self.dim = mesh.dim
        self.k = k
        self.basis = get_basis(k, k + 1)
        self.geom = Geometry(mesh, k + 1)
        self.tau_e, self.tau_if, self.tau_bf = compute_tau_ip(mesh, self.geom, k)
        f = mesh.interior
        self.f_em, self.f_sm, self.f_ep, self.f_sp = f.em, f.sm, f.ep, f.sp
        b = mesh.boundary
        self.b_groups = {}
        for i, name in enumerate(mesh.tag_names):
            sel = b.tag == i
            if sel.any():
                self.b_groups[name] = (b.elem[sel], b.slot[sel])
        self._nq_over = n_q_over or convective_rule_points(k)
        self._over = None

    @property
    def n_local(self):
        return (self.k + 1) ** self.dim

    def field_shape(self, ncomp=None):
        s = (self.mesh.n_elements,) + (self.k + 1,) * self.dim
        return s if ncomp is None else (ncomp,) + s

    @property
    def basis_over(self):
        """Over-integration rule + geometry (spaces.py:117-122)."""
        if self._over is None:
            self._over = (get_basis(self.k, self._nq_over),
                          Geometry(self.mesh, self._nq_over))
        return self._over

    def node_coords(self):
        """Physical GLL node coordinates, (dim, ne, m..) (spaces.py:87-107)."""
        dim, m = self.dim, self.k + 1
        xi = self.basis.nodes
        out = []
        for d in range(dim):
            c = (self.mesh.lower[:, d][:, None] +
                 0.5 * (xi[None, :] + 1.0) * self.mesh.h[:, d][:, None])
            shape = [self.mesh.n_elements] + [1] * dim
            shape[_ax(dim, d)] = m
            out.append(np.broadcast_to(c.reshape(shape),
                                       self.field_shape()).copy())
        return np.stack(out)

    def gather_minus(self, A):
        return A[self.f_sm, self.f_em]

    def gather_plus(self, A):
        # Cartesian boxes: both sides enumerate face points identically
        return A[self.f_sp, self.f_ep]

    def scatter_faces(self, Vm, Vp, out):
        """Plain assignment, each (slot, elem) written once (spaces.py:151-163)."""
        out[self.f_sm, self.f_em] = Vm
        out[self.f_sp, self.f_ep] = Vp


@dataclass
class DirichletBC:
    g: Callable
    dg_dt: Optional[Callable] = None


@dataclass
class NeumannBC:
    h: Callable
    g_p: Callable


class BoundarySpec:
    def __init__(self, kinds):
        self.kinds = dict(kinds)

    def validate(self, mesh):
        present = {mesh.tag_names[t] for t in mesh.boundary.tag}
        missing = present - set(self.kinds)
        if missing:
            raise ValueError(f"boundary tags without a condition: {missing}")

    def resolve(self, space):
        return ResolvedBCs(space, self)


class ResolvedBCs:
    def __init__(self, space, spec):
        spec.validate(space.mesh)
        self.dirichlet, self.neumann = [], []
        for tag, (eb, sb) in space.b_groups.items():
            kind = spec.kinds[tag]
            if isinstance(kind, DirichletBC):
                self.dirichlet.append((eb, sb, kind))
            elif isinstance(kind, NeumannBC):
                self.neumann.append((eb, sb, kind))
            else:
                raise TypeError(f"unsupported boundary kind for tag {tag!r}")


def zero_dirichlet(dim):
    return DirichletBC(lambda x, t: np.zeros((dim,) + x.shape[1:]),
                       lambda x, t: np.zeros((dim,) + x.shape[1:]))


def zero_neumann(dim):
    return NeumannBC(lambda x, t: np.zeros((dim,) + x.shape[1:]),
                     lambda x, t: np.zeros(x.shape[1:]))


# ---------------------------------------------------------------------------
# operators (reference operators.py)

def _phys_grad(jit, g):
    """p_a = sum_b jinvT[a][b] g_b (operators.py:137-140, :150-153)."""
    dim = len(g)
    return [sum(jit[a, b] * g[b] for b in range(dim)) for a in range(dim)]


def _ref_test(jit, dphys):
    """r_b = sum_a jinvT[a][b] d_a (operators.py:143-147, :156-159)."""
    dim = len(dphys)
    return [sum(jit[a, b] * dphys[a] for a in range(dim)) for b in range(dim)]


def _face_jit(space, geom):
    return geom.jinvT_f[:, :, None]      # broadcast over slots


def mass_apply(space, u):
    """operators.py:167-173."""
    b, g, dim = space.basis, space.geom, space.dim
    if u.ndim == dim + 1:
        return apply_mass(u, b, g.jxw, dim)
    return np.stack([apply_mass(c, b, g.jxw, dim) for c in u])


def inverse_mass_apply(space, r):
    """operators.py:176-181."""
    b, g, dim = space.basis, space.geom, space.dim
    if r.ndim == dim + 1:
        return apply_inverse_mass(r, b, g.jxw, dim)
    return np.stack([apply_inverse_mass(c, b, g.jxw, dim) for c in r])


def _zeros_faces(space, n, q):
    shape = (2 * space.dim, space.mesh.n_elements) + (q,) * (space.dim - 1)
    return [np.zeros(shape) for _ in range(n)]


def apply_pressure_laplace(space, p, bcs, tau_scale=1.0):
    """SIP Laplacian (operators.py:187-238)."""
    b, g, dim = space.basis, space.geom, space.dim
    q = b.n_q
    grads = vol_gradients(p, b, dim)
    ph = _phys_grad(g.jinvT, grads)
    out = vol_integrate_gradients(_ref_test(g.jinvT, [c * g.jxw for c in ph]),
                                  b, dim)
    fv = face_values(p, b, dim)
    fg = face_gradients(p, b, dim)
    jf = _face_jit(space, g)
    pf = _phys_grad(jf, fg)
    gn = sum(g.normal[a] * pf[a] for a in range(dim))

    Vc, = _zeros_faces(space, 1, q)
    D = _zeros_faces(space, dim, q)
    sj = g.sjxw[space.f_sm, space.f_em]
    nrm = [g.normal[a][space.f_sm, space.f_em] for a in range(dim)]
    vm, vp = space.gather_minus(fv), space.gather_plus(fv)
    gnm, gnp = space.gather_minus(gn), space.gather_plus(gn)
    tau = tau_scale * space.tau_if.reshape((-1,) + (1,) * (dim - 1))
    jump = vm - vp
    avg_gn = 0.5 * (gnm - gnp)
    Vm = -(avg_gn - tau * jump) * sj
    space.scatter_faces(Vm, -Vm, Vc)
    for a in range(dim):
        G = -0.5 * jump * nrm[a] * sj
        space.scatter_faces(G, G, D[a])
    for eb, sb, _ in bcs.neumann:                          # :227-233
        sjb = g.sjxw[sb, eb]
        vb = fv[sb, eb]
        taub = tau_scale * space.tau_e[eb].reshape((-1,) + (1,) * (dim - 1))
        Vc[sb, eb] = -(gn[sb, eb] - 2.0 * taub * vb) * sjb
        for a in range(dim):
            D[a][sb, eb] = -vb * g.normal[a][sb, eb] * sjb
    rf = _ref_test(jf, D)
    face_lift_values(Vc, b, out, dim)
    face_lift_gradients(rf, b, out, dim)
    return out


def _laplace_block_apply(space, p, bcs, tau_scale):
    """Element-block part of the SIP Laplacian (operators.py:675-714)."""
    b, g, dim = space.basis, space.geom, space.dim
    q = b.n_q
    ph = _phys_grad(g.jinvT, vol_gradients(p, b, dim))
    out = vol_integrate_gradients(_ref_test(g.jinvT, [c * g.jxw for c in ph]),
                                  b, dim)
    fv = face_values(p, b, dim)
    jf = _face_jit(space, g)
    pf = _phys_grad(jf, face_gradients(p, b, dim))
    gn = sum(g.normal[a] * pf[a] for a in range(dim))
    Vc, = _zeros_faces(space, 1, q)
    D = _zeros_faces(space, dim, q)
    tau = tau_scale * space.tau_if.reshape((-1,) + (1,) * (dim - 1))
    for ee, ss in ((space.f_em, space.f_sm), (space.f_ep, space.f_sp)):
        sj = g.sjxw[ss, ee]
        v = fv[ss, ee]
        Vc[ss, ee] = -(0.5 * gn[ss, ee] - tau * v) * sj
        for a in range(dim):
            D[a][ss, ee] = -0.5 * v * g.normal[a][ss, ee] * sj
    for eb, sb, _ in bcs.neumann:
        sjb = g.sjxw[sb, eb]
        vb = fv[sb, eb]
        taub = tau_scale * space.tau_e[eb].reshape((-1,) + (1,) * (dim - 1))
        Vc[sb, eb] = -(gn[sb, eb] - 2.0 * taub * vb) * sjb
        for a in range(dim):
            D[a][sb, eb] = -vb * g.normal[a][sb, eb] * sjb
    face_lift_values(Vc, b, out, dim)
    face_lift_gradients(_ref_test(jf, D), b, out, dim)
    return out


def laplace_diagonal(space, bcs, tau_scale=1.0):
    """Exact Jacobi diagonal by unit-vector block applies (operators.py:717-730)."""
    shape = space.field_shape()
    diag = np.empty(shape)
    unit = np.zeros(shape)
    m = space.k + 1
    for loc in np.ndindex(*(m,) * space.dim):
        unit[...] = 0.0
        unit[(slice(None),) + loc] = 1.0
        out = _laplace_block_apply(space, unit, bcs, tau_scale)
        diag[(slice(None),) + loc] = out[(slice(None),) + loc]
    return diag


def apply_projection_operator(space, w, tau_d_e, tau_c_f):
    """M + tau_D div-div + tau_C interior jump (operators.py:372-412)."""
    b, g, dim = space.basis, space.geom, space.dim
    q = b.n_q
    out = np.empty_like(w)
    bshape = (-1,) + (1,) * dim
    if tau_d_e is None:
        for c in range(dim):
            out[c] = apply_mass(w[c], b, g.jxw, dim)
    else:
        div = 0.0
        for c in range(dim):
            ph = _phys_grad(g.jinvT, vol_gradients(w[c], b, dim))
            div = div + ph[c]
        s = (np.asarray(tau_d_e).reshape(bshape) * div) * g.jxw
        for c in range(dim):
            out[c] = vol_integrate_values(vol_values(w[c], b, dim) * g.jxw, b, dim)
            data = [s if a == c else np.zeros_like(s) for a in range(dim)]
            out[c] += vol_integrate_gradients(_ref_test(g.jinvT, data), b, dim)
    if tau_c_f is not None:
        sj = g.sjxw[space.f_sm, space.f_em]
        tc = np.asarray(tau_c_f).reshape((-1,) + (1,) * (dim - 1))
        for c in range(dim):
            f = face_values(w[c], b, dim)
            V, = _zeros_faces(space, 1, q)
            Vm = tc * (space.gather_minus(f) - space.gather_plus(f)) * sj
            space.scatter_faces(Vm, -Vm, V)
            face_lift_values(V, b, out[c], dim)
    return out


def apply_viscous_helmholtz(space, u, gamma0_dt, nu, bcs):
    """(gamma0/dt) M u + SIP of -div(2 nu eps(u)) (operators.py:418-491)."""
    b, g, dim = space.basis, space.geom, space.dim
    q = b.n_q
    grads = [_phys_grad(g.jinvT, vol_gradients(u[c], b, dim)) for c in range(dim)]
    out = np.empty_like(u)
    # T_ab = nu (du_a/dx_b + du_b/dx_a) = 2 nu eps_ab
    for a in range(dim):
        data = [nu * (grads[a][bb] + grads[bb][a]) * g.jxw for bb in range(dim)]
        out[a] = vol_integrate_gradients(_ref_test(g.jinvT, data), b, dim)
        out[a] += vol_integrate_values(gamma0_dt * vol_values(u[a], b, dim)
                                       * g.jxw, b, dim)
    if nu == 0.0:
        return out
    jf = _face_jit(space, g)
    fv = [face_values(u[c], b, dim) for c in range(dim)]
    fg = [_phys_grad(jf, face_gradients(u[c], b, dim)) for c in range(dim)]
    nrm_a = g.normal
    visc_n = [nu * sum((fg[a][bb] + fg[bb][a]) * nrm_a[bb] for bb in range(dim))
              for a in range(dim)]
    V = _zeros_faces(space, dim, q)
    Dd = [_zeros_faces(space, dim, q) for _ in range(dim)]
    sj = g.sjxw[space.f_sm, space.f_em]
    nrm = [nrm_a[a][space.f_sm, space.f_em] for a in range(dim)]
    tau = space.tau_if.reshape((-1,) + (1,) * (dim - 1)) * nu
    j = [space.gather_minus(fv[a]) - space.gather_plus(fv[a]) for a in range(dim)]
    for a in range(dim):
        avg = 0.5 * (space.gather_minus(visc_n[a]) - space.gather_plus(visc_n[a]))
        Vm = -(avg - tau * j[a]) * sj
        space.scatter_faces(Vm, -Vm, V[a])
        for bb in range(dim):
            G = -0.5 * nu * (j[a] * nrm[bb] + j[bb] * nrm[a]) * sj
            space.scatter_faces(G, G, Dd[a][bb])
    for eb, sb, _ in bcs.dirichlet:
        sjb = g.sjxw[sb, eb]
        nb = [nrm_a[a][sb, eb] for a in range(dim)]
        taub = space.tau_e[eb].reshape((-1,) + (1,) * (dim - 1)) * nu
        ub = [fv[a][sb, eb] for a in range(dim)]
        for a in range(dim):
            V[a][sb, eb] = -(visc_n[a][sb, eb] - 2.0 * taub * ub[a]) * sjb
            for bb in range(dim):
                Dd[a][bb][sb, eb] = -nu * (ub[a] * nb[bb] + ub[bb] * nb[a]) * sjb
    for a in range(dim):
        face_lift_values(V[a], b, out[a], dim)
        face_lift_gradients(_ref_test(jf, Dd[a]), b, out[a], dim)
    return out


def _lax_friedrichs(um, up, nrm):
    """F*(u).n^- per point (operators.py:597-604)."""
    unm = sum(um[a] * nrm[a] for a in range(len(um)))
    unp = sum(up[a] * nrm[a] for a in range(len(um)))
    lam = 2.0 * np.maximum(np.abs(unm), np.abs(unp))
    return [0.5 * (um[a] * unm + up[a] * unp) + 0.5 * lam * (um[a] - up[a])
            for a in range(len(um))]


def eval_convective_rhs(space, bcs, history, betas, times, t_np1,
                        body_force=None):
    """sum_i beta_i[(grad v, u u) - (v, F*.n)] + (v, f) on the over-integration
    rule (operators.py:533-594)."""
    b, g = space.basis_over
    dim = space.dim
    q = b.n_q
    out = np.zeros(space.field_shape(dim))
    sj = g.sjxw[space.f_sm, space.f_em]
    nrm = [g.normal[a][space.f_sm, space.f_em] for a in range(dim)]
    for beta, u, t_i in zip(betas, history, times):
        v = [vol_values(u[c], b, dim) for c in range(dim)]
        for a in range(dim):
            data = [v[a] * v[bb] * g.jxw for bb in range(dim)]
            out[a] += beta * vol_integrate_gradients(_ref_test(g.jinvT, data),
                                                     b, dim)
        f = [face_values(u[c], b, dim) for c in range(dim)]
        V = _zeros_faces(space, dim, q)
        um = [space.gather_minus(f[a]) for a in range(dim)]
        up = [space.gather_plus(f[a]) for a in range(dim)]
        F = _lax_friedrichs(um, up, nrm)
        for a in range(dim):
            Vm = -beta * F[a] * sj
            space.scatter_faces(Vm, -Vm, V[a])
        for eb, sb, bc in bcs.dirichlet:
            nb = [np.broadcast_to(g.normal[a][sb, eb], f[0][sb, eb].shape)
                  for a in range(dim)]
            ub = [f[a][sb, eb] for a in range(dim)]
            xb = _face_points(space, g, b, eb, sb)
            gu = bc.g(xb, t_i)
            Fb = _lax_friedrichs(ub, [2 * gu[a] - ub[a] for a in range(dim)], nb)
            for a in range(dim):
                V[a][sb, eb] = -beta * Fb[a] * g.sjxw[sb, eb]
        for eb, sb, _ in bcs.neumann:
            un = sum(f[a][sb, eb] * g.normal[a][sb, eb] for a in range(dim))
            for a in range(dim):
                V[a][sb, eb] = -beta * f[a][sb, eb] * un * g.sjxw[sb, eb]
        for a in range(dim):
            face_lift_values(V[a], b, out[a], dim)
    if body_force is not None:
        xq = _vol_points(space, b)
        fq = body_force(xq, t_np1)
        for a in range(dim):
            out[a] += vol_integrate_values(fq[a] * g.jxw, b, dim)
    return out


def _vol_points(space, b):
    """Physical coordinates of the tensor Gauss points, (dim, ne, q..)."""
    dim, mesh = space.dim, space.mesh
    q = b.n_q
    pts = b.rule.points
    out = []
    for d in range(dim):
        c = mesh.lower[:, d][:, None] + 0.5 * (pts[None] + 1.0) * mesh.h[:, d][:, None]
        shape = [mesh.n_elements] + [1] * dim
        shape[_ax(dim, d)] = q
        out.append(np.broadcast_to(c.reshape(shape), (mesh.n_elements,) + (q,) * dim))
    return np.stack(out)


def _face_points(space, g, b, eb, sb):
    """Physical coordinates of face points of boundary faces (eb, sb)."""
    dim, mesh = space.dim, space.mesh
    q = b.n_q
    pts = b.rule.points
    out = np.empty((dim, len(eb)) + (q,) * (dim - 1))
    for i, (e, s) in enumerate(zip(eb, sb)):
        d = s // 2
        tang = _tangential(dim, d)
        for a in range(dim):
            if a == d:
                out[a, i] = mesh.lower[e, a] + (s % 2) * mesh.h[e, a]
            else:
                c = mesh.lower[e, a] + 0.5 * (pts + 1.0) * mesh.h[e, a]
                shape = [1] * (dim - 1)
                shape[tang.index(a)] = q
                out[a, i] = np.broadcast_to(c.reshape(shape), (q,) * (dim - 1))
    return out


def compute_penalty_parameters(space, u, dt, cfl, zeta_d_star=1.0,
                               zeta_c_star=1.0, uses_divdiv=True,
                               uses_jump=True):
    """tau_D = zeta_D |u_mean| h dt, tau_C = zeta_C |u_mean| dt
    (operators.py:736-755); h = V^(1/dim)."""
    if cfl <= 0:
        raise ValueError(f"CFL must be positive, got {cfl}")
    b, g, dim = space.basis, space.geom, space.dim
    axes = tuple(range(1, dim + 1))
    means = [(vol_values(u[c], b, dim) * g.jxw).sum(axis=axes) for c in range(dim)]
    norm = np.sqrt(sum(m * m for m in means)) / g.volumes
    tau_d = tau_c = None
    if uses_divdiv:
        h = g.volumes ** (1.0 / dim)
        tau_d = (zeta_d_star / cfl) * norm * h * dt
    if uses_jump:
        tce = (zeta_c_star / cfl) * norm * dt
        tau_c = 0.5 * (tce[space.f_em] + tce[space.f_ep])
    return tau_d, tau_c


# ---------------------------------------------------------------------------
# once-per-step right-hand sides (reference operators.py:241-366, 494-527,
# 610-672), DIM-generic

def _bshape(space):
    return (-1,) + (1,) * (space.dim - 1)


def gp_dirichlet_rhs(space, bcs, t, tau_scale=1.0):
    """Pressure-Dirichlet data g_p on velocity-Neumann faces
    (operators.py:241-259)."""
    b, g, dim = space.basis, space.geom, space.dim
    q = b.n_q
    Vc, = _zeros_faces(space, 1, q)
    D = _zeros_faces(space, dim, q)
    for eb, sb, bc in bcs.neumann:
        gp = bc.g_p(_face_points(space, g, b, eb, sb), t)
        sjb = g.sjxw[sb, eb]
        taub = tau_scale * space.tau_e[eb].reshape(_bshape(space))
        Vc[sb, eb] = 2.0 * taub * gp * sjb
        for a in range(dim):
            D[a][sb, eb] = -gp * g.normal[a][sb, eb] * sjb
    out = np.zeros(space.field_shape())
    face_lift_values(Vc, b, out, dim)
    face_lift_gradients(_ref_test(_face_jit(space, g), D), b, out, dim)
    return out


def _divergence_at_q(space, u):
    b, g, dim = space.basis, space.geom, space.dim
    div = 0.0
    for c in range(dim):
        div = div + _phys_grad(g.jinvT, vol_gradients(u[c], b, dim))[c]
    return div


def eval_divergence_rhs(space, u, bcs, scale, form="standard"):
    """a(q, u) scaled: standard / weak (central flux) / strong
    (operators.py:265-316)."""
    b, g, dim = space.basis, space.geom, space.dim
    q = b.n_q
    if form == "standard":
        return vol_integrate_values(-scale * _divergence_at_q(space, u) * g.jxw,
                                    b, dim)
    if form not in ("weak", "strong"):
        raise ValueError(f"unknown divergence form {form!r}")
    f = [face_values(u[c], b, dim) for c in range(dim)]
    un = sum(g.normal[a] * f[a] for a in range(dim))
    Vc, = _zeros_faces(space, 1, q)
    sj = g.sjxw[space.f_sm, space.f_em]
    unm, unp = space.gather_minus(un), space.gather_plus(un)
    if form == "weak":
        data = [scale * vol_values(u[c], b, dim) * g.jxw for c in range(dim)]
        out = vol_integrate_gradients(_ref_test(g.jinvT, data), b, dim)
        Vm = -scale * 0.5 * (unm - unp) * sj
        space.scatter_faces(Vm, -Vm, Vc)
        for groups in (bcs.dirichlet, bcs.neumann):
            for eb, sb, _ in groups:
                Vc[sb, eb] = -scale * un[sb, eb] * g.sjxw[sb, eb]
        face_lift_values(Vc, b, out, dim)
        return out
    out = vol_integrate_values(-scale * _divergence_at_q(space, u) * g.jxw, b, dim)
    Vm = scale * 0.5 * (unm + unp) * sj
    space.scatter_faces(Vm, Vm, Vc)
    face_lift_values(Vc, b, out, dim)
    return out


def eval_pressure_gradient_rhs(space, p, bcs, scale, form="standard"):
    """b(v, p) scaled: standard -(v, scale grad p) or weak with central flux
    (operators.py:322-366)."""
    b, g, dim = space.basis, space.geom, space.dim
    q = b.n_q
    out = np.empty(space.field_shape(dim))
    if form == "standard":
        ph = _phys_grad(g.jinvT, vol_gradients(p, b, dim))
        for a in range(dim):
            out[a] = vol_integrate_values(-scale * ph[a] * g.jxw, b, dim)
        return out
    if form != "weak":
        raise ValueError(f"unknown pressure-gradient form {form!r}")
    s = scale * vol_values(p, b, dim) * g.jxw
    for a in range(dim):
        data = [s if c == a else np.zeros_like(s) for c in range(dim)]
        out[a] = vol_integrate_gradients(_ref_test(g.jinvT, data), b, dim)
    fv = face_values(p, b, dim)
    sj = g.sjxw[space.f_sm, space.f_em]
    avg = 0.5 * (space.gather_minus(fv) + space.gather_plus(fv))
    for a in range(dim):
        V, = _zeros_faces(space, 1, q)
        Vm = -scale * avg * g.normal[a][space.f_sm, space.f_em] * sj
        space.scatter_faces(Vm, -Vm, V)
        for groups in (bcs.dirichlet, bcs.neumann):
            for eb, sb, _ in groups:
                V[sb, eb] = -scale * fv[sb, eb] * g.normal[a][sb, eb] * g.sjxw[sb, eb]
        face_lift_values(V, b, out[a], dim)
    return out


def viscous_rhs_bc(space, bcs, t, nu):
    """Boundary-data terms of the viscous solve (operators.py:494-527)."""
    b, g, dim = space.basis, space.geom, space.dim
    q = b.n_q
    V = _zeros_faces(space, dim, q)
    Dd = [_zeros_faces(space, dim, q) for _ in range(dim)]
    for eb, sb, bc in bcs.dirichlet:
        gu = bc.g(_face_points(space, g, b, eb, sb), t)
        sjb = g.sjxw[sb, eb]
        nb = [g.normal[a][sb, eb] for a in range(dim)]
        taub = space.tau_e[eb].reshape(_bshape(space)) * nu
        for a in range(dim):
            V[a][sb, eb] = 2.0 * taub * gu[a] * sjb
            for c in range(dim):
                Dd[a][c][sb, eb] = -nu * (gu[a] * nb[c] + gu[c] * nb[a]) * sjb
    for eb, sb, bc in bcs.neumann:
        xb = _face_points(space, g, b, eb, sb)
        h, gp = bc.h(xb, t), bc.g_p(xb, t)
        sjb = g.sjxw[sb, eb]
        for a in range(dim):
            V[a][sb, eb] = (h[a] + gp * g.normal[a][sb, eb]) * sjb
    out = np.zeros(space.field_shape(dim))
    jf = _face_jit(space, g)
    for a in range(dim):
        face_lift_values(V[a], b, out[a], dim)
        face_lift_gradients(_ref_test(jf, Dd[a]), b, out[a], dim)
    return out


def _curl(grad):
    """curl from grad[c][a] = d u_c / d x_a: scalar in 2D, 3-vector in 3D."""
    if len(grad) == 2:
        return grad[1][0] - grad[0][1]
    return [grad[2][1] - grad[1][2], grad[0][2] - grad[2][0], grad[1][0] - grad[0][1]]


def compute_vorticity(space, u):
    """Element-local L2 projection of curl u (operators.py:610-618); a scalar
    field in 2D (the reference), the three curl components in 3D."""
    b, g, dim = space.basis, space.geom, space.dim
    grad = [_phys_grad(g.jinvT, vol_gradients(u[c], b, dim)) for c in range(dim)]
    w = _curl(grad)
    if dim == 2:
        return apply_inverse_mass(vol_integrate_values(w * g.jxw, b, dim), b, g.jxw, dim)
    return np.stack([apply_inverse_mass(vol_integrate_values(wc * g.jxw, b, dim),
                                        b, g.jxw, dim) for wc in w])


def eval_pressure_neumann_rhs(space, bcs, history, vorticity_history, betas, nu,
                              t_np1, body_force=None):
    """Consistent pressure Neumann data on velocity-Dirichlet faces:
    -(dg/dt + sum_i beta_i (div(u u) + nu curl w) - f) . n (operators.py:621-672).
    In 3D the vorticity is a 3-vector and curl w its vector curl."""
    b, g, dim = space.basis, space.geom, space.dim
    q = b.n_q
    out = np.zeros(space.field_shape())
    if not bcs.dirichlet:
        return out
    jf = _face_jit(space, g)
    hp = [0.0] * dim
    for beta, u, w in zip(betas, history, vorticity_history):
        f = [face_values(u[c], b, dim) for c in range(dim)]
        gr = [_phys_grad(jf, face_gradients(u[c], b, dim)) for c in range(dim)]
        div = sum(gr[c][c] for c in range(dim))
        conv = [f[a] * div + sum(f[c] * gr[a][c] for c in range(dim)) for a in range(dim)]
        if dim == 2:
            gw = _phys_grad(jf, face_gradients(w, b, dim))
            curlw = [gw[1], -gw[0]]
        else:
            curlw = _curl([_phys_grad(jf, face_gradients(w[c], b, dim)) for c in range(dim)])
        for a in range(dim):
            hp[a] = hp[a] + beta * (conv[a] + nu * curlw[a])
    Vc, = _zeros_faces(space, 1, q)
    for eb, sb, bc in bcs.dirichlet:
        xb = _face_points(space, g, b, eb, sb)
        if bc.dg_dt is not None:
            dgdt = bc.dg_dt(xb, t_np1)
        else:
            dgdt = np.zeros((dim,) + xb.shape[1:])
        h = [dgdt[a] + hp[a][sb, eb] for a in range(dim)]
        if body_force is not None:
            fb = body_force(xb, t_np1)
            h = [h[a] - fb[a] for a in range(dim)]
        hn = sum(h[a] * g.normal[a][sb, eb] for a in range(dim))
        Vc[sb, eb] = -hn * g.sjxw[sb, eb]
    face_lift_values(Vc, b, out, dim)
    return out


# ---------------------------------------------------------------------------
# solvers (reference solvers.py; dimension-agnostic)

@dataclass
class SolverStats:
    iterations: int
    residual: float
    converged: bool
    breakdown: bool = False
    history: Optional[list] = None


def pcg(op, prec, b, x0=None, rel_tol=1e-8, abs_tol=0.0, max_iter=1000):
    """Classical PCG, preconditioned-norm stopping (solvers.py:30-73).
    Records the residual history sqrt(r.z) per iteration."""
    prec = prec or (lambda v: v.copy())
    if x0 is None:
        x = np.zeros_like(b)
        r = b.copy()
    else:
        x = x0.copy()
        r = b - op(x)
    z = prec(r)
    rz = np.vdot(r, z).real
    if rz < 0:
        return x, SolverStats(0, np.sqrt(abs(rz)), False, True, [])
    norm0 = np.sqrt(rz)
    hist = [norm0]
    tol = max(rel_tol * norm0, abs_tol)
    if norm0 <= tol:
        return x, SolverStats(0, norm0, True, False, hist)
    p = z.copy()
    norm = norm0
    for it in range(1, max_iter + 1):
        Ap = op(p)
        pAp = np.vdot(p, Ap).real
        if pAp <= 0.0:
            return x, SolverStats(it, norm, False, True, hist)
        alpha = rz / pAp
        x += alpha * p
        r -= alpha * Ap
        z = prec(r)
        rz_new = np.vdot(r, z).real
        norm = np.sqrt(max(rz_new, 0.0))
        hist.append(norm)
        if norm <= tol:
            return x, SolverStats(it, norm, True, False, hist)
        if rz_new <= 0.0:
            return x, SolverStats(it, norm, False, True, hist)
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, SolverStats(max_iter, norm, False, False, hist)


@dataclass
class ChebyshevConfig:
    degree: int = 5
    smoothing_range: float = 20.0
    lambda_max: float = 1.0

    def __post_init__(self):
        if self.degree < 0:
            raise ValueError("Chebyshev degree must be >= 0")
        if self.smoothing_range <= 1.0:
            raise ValueError("smoothing range must exceed 1")


def chebyshev_smooth(op, diag, cfg, rhs, x=None, degree=None):
    """Chebyshev iteration on [lmax/range, lmax] (solvers.py:93-129)."""
    deg = cfg.degree if degree is None else degree
    if x is None:
        x = np.zeros_like(rhs)
        r = rhs.copy()
    else:
        x = x.copy()
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


def eigen_estimate_via_cg(op, prec_diag, b, n_iter=20):
    """Lanczos lambda estimates from CG coefficients (solvers.py:138-176)."""
    diag = prec_diag if prec_diag is not None else np.ones_like(b)
    x = np.zeros_like(b)
    r = b.copy()
    z = r / diag
    rz = np.vdot(r, z).real
    alphas, betas = [], []
    p = z.copy()
    for _ in range(n_iter):
        Ap = op(p)
        pAp = np.vdot(p, Ap).real
        if pAp <= 0 or rz <= 0:
            break
        alpha = rz / pAp
        alphas.append(alpha)
        x += alpha * p
        r -= alpha * Ap
        z = r / diag
        rz_new = np.vdot(r, z).real
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


def element_local_pcg(op_local, prec_local, b, rel_tol=1e-12, max_iter=200,
                      floor_factor=8.0):
    """Batched per-cell CG with per-cell stopping and the eps*lambda_max floor
    from the running Lanczos diagonal (solvers.py:201-256).  Layout
    (ncomp, ne, ...): the cell axis is axis 1 here (axis 2 in the reference's
    (ncomp, m, ne, m) kernel layout)."""
    ne = b.shape[1]
    red = (0,) + tuple(range(2, b.ndim))
    bc = (None, slice(None)) + (None,) * (b.ndim - 2)

    def edot(u, v):
        return (u * v).sum(axis=red)

    x = np.zeros_like(b)
    r = b.copy()
    z = prec_local(r)
    rz = edot(r, z)
    norm0 = np.sqrt(np.maximum(rz, 0.0))
    active = norm0 > rel_tol * norm0
    iters = np.zeros(ne, dtype=int)
    p = z.copy()
    eps = np.finfo(float).eps
    lan_max = np.ones(ne)
    alpha_prev = np.ones(ne)
    beta_prev = np.zeros(ne)
    for it in range(1, max_iter + 1):
        if not active.any():
            break
        Ap = op_local(p)
        pAp = edot(p, Ap)
        safe = np.where(active & (pAp > 0), pAp, 1.0)
        alpha = np.where(active, rz / safe, 1.0)
        lan_max = np.maximum(lan_max, 1.0 / alpha + beta_prev / alpha_prev)
        x += np.where(active, alpha, 0.0)[bc] * p
        r -= np.where(active, alpha, 0.0)[bc] * Ap
        z = prec_local(r)
        rz_new = edot(r, z)
        norm = np.sqrt(np.maximum(rz_new, 0.0))
        iters[active] = it
        tol = np.maximum(rel_tol, floor_factor * eps * lan_max) * norm0
        active = active & (norm > tol)
        beta = np.where(active, rz_new / np.where(rz > 0, rz, 1.0), 0.0)
        alpha_prev, beta_prev = alpha, beta
        p = z + beta[bc] * p
        rz = rz_new
    return x, iters, ~active


def zero_mean_project(space, p):
    """Subtract the L2 mean (solvers.py:179-184)."""
    g = space.geom
    vals = vol_values(p, space.basis, space.dim)
    return p - (vals * g.jxw).sum() / g.volumes.sum()


def dual_weights(space):
    """w_i = integral of l_i (solvers.py:196-197)."""
    return vol_integrate_values(np.ascontiguousarray(space.geom.jxw),
                                space.basis, space.dim)


def zero_mean_project_dual(space, b):
    """b - (sum b / |Omega|) w (solvers.py:187-198)."""
    return b - (b.sum() / space.geom.volumes.sum()) * dual_weights(space)


def chebyshev_from_lanczos(space, op, diag, degree=5, smoothing_range=20.0,
                           est_iters=20, safety=1.1, seed=987, project=None):
    """ChebyshevConfig as the reference builds it per MG level
    (multigrid.py:100-114): lambda_max = safety * Lanczos estimate on a
    seeded standard-normal start vector (projected on singular problems)."""
    rng = np.random.default_rng(seed)
    seed_vec = rng.standard_normal(diag.shape)
    est_op = op
    if project is not None:
        seed_vec = project(space, seed_vec)
        est_op = lambda v: project(space, op(v))
    lmax, _ = eigen_estimate_via_cg(est_op, diag, seed_vec, est_iters)
    return ChebyshevConfig(degree, smoothing_range, safety * lmax)
