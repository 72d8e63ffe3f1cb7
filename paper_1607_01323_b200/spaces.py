"""DgSpace: mesh + degree + device contexts (reference spaces.py:61-163).

A space owns one device context per boundary-kind assignment (the reference
passes ``bcs`` per operator call; the context bakes the per-tag kinds into
its face modes).  Contexts hold the Cartesian geometry (cell sizes per axis),
tau_e per cell (Eq. 18, geometry.py:90-108) and the 1D tables.

Device vectors are torch CUDA tensors in element-major order
(component, cell, [z,] y, x); ``to_device`` / ``to_host`` convert the
reference's 2D kernel layout (m, ne, m) (spaces.py:18-58).
"""

import ctypes

import numpy as np

from . import _lib
from .mesh import BoxMesh, TAG_NAMES, box_from_reference


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise _lib.DgError("no CUDA device: the DG operators run only on the GPU "
                           "(there is no CPU fallback)")
    return torch


class DeviceContext:
    """Owns one dg_ctx (include/dgmf.h)."""

    def __init__(self, mesh, k, bc_kinds, n_q_over=0, slab=None):
        _torch()
        L = _lib.lib()
        self._verts = [np.ascontiguousarray(v, dtype=np.float64)
                       for v in mesh.axis_vertices]
        desc = _lib.MeshDesc()
        desc.dim = mesh.dim
        desc.k = k
        desc.n_q_over = int(n_q_over or 0)
        for d in range(3):
            desc.counts[d] = mesh.counts[d] if d < mesh.dim else 1
            desc.periodic[d] = int(mesh.periodic[d]) if d < mesh.dim else 0
        for d in range(mesh.dim):
            desc.vertices[d] = self._verts[d].ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        for t in range(6):
            desc.bc_kind[t] = bc_kinds[t]
        desc.slab_begin, desc.slab_end = slab if slab is not None else (0, 0)
        h = ctypes.c_void_p()
        _lib.check(L.dg_ctx_create(ctypes.byref(desc), ctypes.byref(h)))
        self.handle = h
        nc, nd = ctypes.c_int64(), ctypes.c_int64()
        _lib.check(L.dg_ctx_sizes(h, ctypes.byref(nc), ctypes.byref(nd)))
        self.n_cells, self.n_dofs = nc.value, nd.value
        self._L = L

    def tau(self):
        out = np.empty(self.n_cells)
        _lib.check(self._L.dg_ctx_tau(self.handle, out.ctypes.data_as(
            ctypes.POINTER(ctypes.c_double))))
        return out

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self._L.dg_ctx_destroy(h)
            except Exception:
                pass
            self.handle = None


class DgSpace:
    """DG Q_k space (reference spaces.py:61-81) on a box mesh.

    Drop-in for the reference's ``DgSpace(mesh, k)``: ``mesh`` may be this
    package's BoxMesh or the reference's own ``Mesh`` object.  A reference
    mesh that is an axis-aligned box (build_box_mesh) becomes the Cartesian
    context (mesh.box_from_reference); any other reference mesh (curved,
    cylinder, refined hierarchies) yields the general-geometry space
    general.GeneralSpace2D, which the same operator calls dispatch on."""

    def __new__(cls, mesh, k: int, n_q_over=None):
        if not isinstance(mesh, BoxMesh) and hasattr(mesh, "elem_vertices"):
            if box_from_reference(mesh) is None:
                from .general import GeneralSpace2D
                return GeneralSpace2D(mesh, k)
        return super().__new__(cls)

    def __init__(self, mesh, k: int, n_q_over=None):
        if k < 1:
            raise ValueError(f"polynomial degree must be >= 1, got k={k}")
        if k > 7:
            raise ValueError("the device path supports k <= 7")
        if not isinstance(mesh, BoxMesh):
            box = box_from_reference(mesh)
            if box is None:
                raise ValueError("DgSpace: not a box mesh (use general.GeneralSpace2D)")
            mesh = box
        self.mesh = mesh
        self.dim = mesh.dim
        self.k = k
        self.n_q_over = n_q_over or ((3 * k) // 2 + 1)
        self._ctx = {}

    @property
    def n_local(self):
        return (self.k + 1) ** self.dim

    @property
    def n_dofs(self):
        return self.mesh.n_elements * self.n_local

    def field_shape(self, ncomp=None):
        s = (self.mesh.n_elements,) + (self.k + 1,) * self.dim
        return s if ncomp is None else (ncomp,) + s

    def ctx(self, bc_kinds=(0, 0, 0, 0, 0, 0), slab=None) -> DeviceContext:
        key = (tuple(bc_kinds), slab)
        if key not in self._ctx:
            self._ctx[key] = DeviceContext(self.mesh, self.k, bc_kinds,
                                           self.n_q_over, slab)
        return self._ctx[key]

    def default_kinds(self):
        """Velocity-Dirichlet on every boundary tag (any kind gives the same
        mass / inverse-mass / zero-mean result)."""
        kinds = [0] * 6
        for d in range(self.dim):
            if not self.mesh.periodic[d]:
                kinds[2 * d] = kinds[2 * d + 1] = _lib.BC_VELOCITY_DIRICHLET
        return tuple(kinds)

    def interior_faces(self):
        """Interior (incl. periodic) faces as (em, sm, ep, sp) arrays, the
        reference's InteriorFaces SoA (mesh.py:46-59): direction-major, the
        minus side is the lower cell with slot 2d+1, the plus side slot 2d."""
        if getattr(self, "_faces", None) is None:
            counts = self.mesh.counts
            e = np.arange(self.mesh.n_elements)
            idx, rem = [], e
            for d in range(self.dim):
                idx.append(rem % counts[d])
                rem = rem // counts[d]
            stride = np.cumprod((1,) + counts[:-1])
            em, sm, ep, sp = [], [], [], []
            for d in range(self.dim):
                n = counts[d]
                lo = e[idx[d] < n - 1]
                em.append(lo); sm.append(np.full(lo.size, 2 * d + 1))
                ep.append(lo + stride[d]); sp.append(np.full(lo.size, 2 * d))
                if self.mesh.periodic[d]:
                    last = e[idx[d] == n - 1]
                    em.append(last); sm.append(np.full(last.size, 2 * d + 1))
                    ep.append(last - (n - 1) * stride[d]); sp.append(np.full(last.size, 2 * d))
            self._faces = tuple(np.concatenate(a).astype(np.int64) for a in (em, sm, ep, sp))
        return self._faces

    def node_coords(self):
        """Physical GLL node coordinates, (dim, ne, [z,] y, x)."""
        from .basis import gll_nodes
        xi = gll_nodes(self.k)
        m = self.k + 1
        out = []
        idx = np.indices(self.mesh.counts[::-1]).reshape(self.dim, -1)[::-1]  # ix, iy, iz
        for d in range(self.dim):
            v = self.mesh.axis_vertices[d]
            lo = v[idx[d]]
            h = np.diff(v)[idx[d]]
            c = lo[:, None] + 0.5 * (xi[None, :] + 1.0) * h[:, None]
            shape = [self.mesh.n_elements] + [1] * self.dim
            shape[self.dim - d] = m
            out.append(np.broadcast_to(c.reshape(shape), self.field_shape()))
        return np.stack(out)

    def general_view(self):
        """The same 2D box as a general-geometry space (bilinear mapping,
        the box's own face lists and cell order): the general 2D kernels
        (csrc/gen2d.cuh) then run the vector operators, which they do faster
        than the per-cell quadrature-point kernel on small 2D cells."""
        if self.dim != 2:
            raise ValueError("general view: 2D spaces")
        if getattr(self, "_gview", None) is None:
            from types import SimpleNamespace
            from .general import GeneralSpace2D
            nx, ny = self.mesh.counts
            vx, vy = self.mesh.axis_vertices
            e = np.arange(self.mesh.n_elements)
            ix, iy = e % nx, e // nx
            geom = np.empty((2, 2, e.size, 2))
            geom[0] = np.stack([vx[ix], vx[ix + 1]], axis=1)[None, :, :]
            geom[1] = np.stack([vy[iy], vy[iy + 1]], axis=1).T[:, :, None]
            em, sm, ep, sp = self.interior_faces()
            names = list(TAG_NAMES[:4])
            bel, bsl, btg = [], [], []
            for side, sel in enumerate((ix == 0, ix == nx - 1, iy == 0, iy == ny - 1)):
                if self.mesh.periodic[side // 2]:
                    continue
                bel.append(e[sel]); bsl.append(np.full(int(sel.sum()), side))
                btg.append(np.full(int(sel.sum()), side))
            cat = lambda a: np.concatenate(a) if a else np.zeros(0, np.int64)
            view = SimpleNamespace(
                geom_degree=1, geom_nodes=geom, n_elements=e.size, tag_names=names,
                interior=SimpleNamespace(em=em, sm=sm, ep=ep, sp=sp, flip=np.zeros(em.size, bool)),
                boundary=SimpleNamespace(elem=cat(bel), slot=cat(bsl), tag=cat(btg)),
                parent=None, quadrant=None)
            self._gview = GeneralSpace2D(view, self.k)
        return self._gview

    def node_coords_reference(self):
        """Node coordinates in the reference layout: (2, m, ne, m) in 2D
        (spaces.py:86-105); element-major (3, ne, z, y, x) in 3D."""
        x = self.node_coords()
        if self.dim == 2:
            return np.ascontiguousarray(x.transpose(0, 2, 1, 3))
        return x

    def interpolate(self, fn, t: float, ncomp: int):
        """Nodal interpolant of fn(x, t) (spaces.py:107-113), x in the
        reference layout; returns fn's values in that layout."""
        x = self.node_coords_reference()
        vals = fn(x, t)
        if ncomp == 1 and np.asarray(vals).shape != (1,) + x.shape[1:]:
            vals = np.asarray(vals)[None]
        return np.ascontiguousarray(np.asarray(vals, dtype=float))

    # --- layout conversion (reference kernel layout <-> element-major) ---
    def is_reference_layout(self, a, ncomp):
        """2D reference kernel layout (m, ne, m) / (ncomp, m, ne, m)."""
        if self.dim != 2:
            return False
        m, ne = self.k + 1, self.mesh.n_elements
        want = (m, ne, m) if ncomp == 1 else (ncomp, m, ne, m)
        return tuple(a.shape) == want and (ne != m or ncomp != 1)

    def to_element_major(self, a, ncomp):
        a = np.asarray(a, dtype=np.float64)
        if self.dim == 2 and a.ndim == (3 if ncomp == 1 else 4) and \
                a.shape[-3:] == (self.k + 1, self.mesh.n_elements, self.k + 1):
            if ncomp == 1:
                return np.ascontiguousarray(a.transpose(1, 0, 2))
            return np.ascontiguousarray(a.transpose(0, 2, 1, 3))
        return np.ascontiguousarray(a.reshape(self.field_shape(None if ncomp == 1 else ncomp)))

    def from_element_major(self, a, ncomp, like_shape):
        if self.dim == 2 and len(like_shape) == (3 if ncomp == 1 else 4) and \
                tuple(like_shape[-3:]) == (self.k + 1, self.mesh.n_elements, self.k + 1):
            a = a.reshape(self.field_shape(None if ncomp == 1 else ncomp))
            if ncomp == 1:
                return np.ascontiguousarray(a.transpose(1, 0, 2))
            return np.ascontiguousarray(a.transpose(0, 2, 1, 3))
        return a.reshape(like_shape)


def tag_kinds_tuple(space, kinds_by_tag):
    out = [0] * 6
    for t, kind in kinds_by_tag.items():
        out[TAG_NAMES.index(t)] = kind
    return tuple(out)


class FieldVector:
    """DoF storage for one field (reference spaces.py:18-58): ``data`` in the
    reference layout ((ncomp, m, ne, m) in 2D, element-major in 3D), with the
    element-major serialisation (component, element, [z,] y, x) the device
    vectors use.  Works with DgSpace and the general 2D space."""

    def __init__(self, data: np.ndarray, k: int):
        self.data = data
        self.k = k

    @classmethod
    def zeros(cls, space, ncomp: int) -> "FieldVector":
        m = space.k + 1
        ne = space.n_elements if hasattr(space, "n_elements") else space.mesh.n_elements
        if space.dim == 2:
            return cls(np.zeros((ncomp, m, ne, m)), space.k)
        return cls(np.zeros((ncomp, ne, m, m, m)), space.k)

    @property
    def ncomp(self) -> int:
        return self.data.shape[0]

    @property
    def n_elements(self) -> int:
        return self.data.shape[2] if self.data.ndim == 4 else self.data.shape[1]

    def copy(self) -> "FieldVector":
        return FieldVector(self.data.copy(), self.k)

    def has_nan(self) -> bool:
        return bool(np.isnan(self.data).any())

    def element_major(self) -> np.ndarray:
        """Flat vector ordered (component, element, [z,] y-node, x-node)."""
        if self.data.ndim == 4:
            return np.ascontiguousarray(self.data.transpose(0, 2, 1, 3)).ravel()
        return np.ascontiguousarray(self.data).ravel()

    def to_device(self):
        """The element-major vector as a CUDA tensor (the device operators'
        input)."""
        return _torch().as_tensor(self.element_major()).to("cuda")

    @classmethod
    def from_element_major(cls, flat, space, ncomp: int) -> "FieldVector":
        if hasattr(flat, "detach"):
            flat = flat.detach().cpu().numpy()
        m = space.k + 1
        ne = space.n_elements if hasattr(space, "n_elements") else space.mesh.n_elements
        if space.dim == 2:
            a = np.asarray(flat).reshape(ncomp, ne, m, m)
            return cls(np.ascontiguousarray(a.transpose(0, 2, 1, 3)), space.k)
        return cls(np.asarray(flat).reshape(ncomp, ne, m, m, m).copy(), space.k)
