"""Structured box meshes (host setup for the device context).

Mirrors the reference builder ``build_box_mesh`` (pkg/src/dgins/mesh.py:
279-351) and ``grading_map`` (:32-43) for axis-aligned boxes in 2D and 3D:
per-axis vertex coordinates (optionally tanh-graded), cell numbering
e = ix + nx*(iy + ny*iz) (mesh.py:320-325), boundary tags xmin..zmax,
periodic axes turned into interior faces.  Only the data the device
context needs is kept: vertex coordinates per axis, counts, periodicity.
"""

import numpy as np

TAG_NAMES = ("xmin", "xmax", "ymin", "ymax", "zmin", "zmax")


def grading_map(s, gamma, delta=1.0):
    """delta * tanh(gamma (2s-1)) / tanh(gamma); gamma = 0 -> uniform
    (mesh.py:32-43)."""
    s = np.asarray(s, dtype=float)
    if gamma < 0:
        raise ValueError(f"grading parameter must be >= 0, got {gamma}")
    if gamma == 0.0:
        return delta * (2.0 * s - 1.0)
    return delta * np.tanh(gamma * (2.0 * s - 1.0)) / np.tanh(gamma)


class BoxMesh:
    """Tensor-product box: per-axis vertices, counts, periodic flags."""

    def __init__(self, extents, counts, grading=None, delta=1.0, periodic=None):
        dim = len(counts)
        if dim not in (2, 3) or len(extents) != dim:
            raise ValueError("box meshes have 2 or 3 axes")
        grading = tuple(grading) if grading is not None else (0.0,) * dim
        periodic = tuple(bool(p) for p in periodic) if periodic is not None else (False,) * dim
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
        self.extents = tuple((float(a), float(b)) for a, b in extents)
        self.grading = grading
        self.periodic = periodic
        self.delta = delta
        self.axis_vertices = []
        for d in range(dim):
            s = np.linspace(0.0, 1.0, self.counts[d] + 1)
            f = grading_map(s, grading[d], delta)
            lo, hi = self.extents[d]
            self.axis_vertices.append(np.ascontiguousarray(
                lo + (f - f[0]) / (f[-1] - f[0]) * (hi - lo)))
        self.tag_names = list(TAG_NAMES[:2 * dim])

    @classmethod
    def from_axis_vertices(cls, axis_vertices, periodic):
        """Box with the given per-axis vertex coordinates (strictly
        increasing) -- e.g. read off a reference Mesh (box_from_reference)."""
        verts = [np.ascontiguousarray(v, dtype=np.float64) for v in axis_vertices]
        dim = len(verts)
        m = cls(tuple((float(v[0]), float(v[-1])) for v in verts),
                tuple(len(v) - 1 for v in verts), periodic=periodic)
        for d in range(dim):
            if np.any(np.diff(verts[d]) <= 0):
                raise ValueError("non-positive mapping Jacobian (vertex coordinates must increase)")
        m.axis_vertices = verts
        return m

    @property
    def n_elements(self):
        return int(np.prod(self.counts))

    def boundary_tags(self):
        """Tags present on the boundary (non-periodic axes)."""
        return [TAG_NAMES[2 * d + s] for d in range(self.dim)
                if not self.periodic[d] for s in (0, 1)]

    def cell_sizes(self):
        return [np.diff(v) for v in self.axis_vertices]


def build_box_mesh(extents, counts, grading=None, delta=1.0, periodic=None,
                   k_geo=1, tag_prefix=None):
    """Reference-compatible signature (mesh.py:279-280); only straight-sided
    (k_geo = 1) boxes without tag prefixes are on the hot path."""
    if k_geo != 1:
        raise ValueError("the device path supports affine (k_geo = 1) boxes")
    if tag_prefix:
        raise ValueError("tag prefixes are not supported by the device path")
    return BoxMesh(extents, counts, grading, delta, periodic)


def box_from_reference(mesh, rtol=1e-13):
    """The reference's 2D ``Mesh`` (pkg/src/dgins/mesh.py:72-90, as built by
    build_box_mesh :279-351) -> BoxMesh, when it IS an axis-aligned
    tensor-product box in the reference's cell order e = iy * nx + ix (corners
    c0..c3 = (ix, iy), (ix+1, iy), (ix, iy+1), (ix+1, iy+1), mesh.py:316-325),
    affine geometry, unprefixed tags xmin..ymax and periodic axes given by
    ``periodic_spec``.  Returns None for anything else (curved, unstructured,
    prefixed tags): those run on the general-geometry path."""
    need = ("vertices", "elem_vertices", "geom_degree", "tag_names")
    if not all(hasattr(mesh, a) for a in need):
        return None
    if int(mesh.geom_degree) != 1 or getattr(mesh, "curved", None):
        return None
    if any(t not in TAG_NAMES[:4] for t in mesh.tag_names):
        return None
    v = np.asarray(mesh.vertices, dtype=np.float64)
    ev = np.asarray(mesh.elem_vertices)
    if v.ndim != 2 or v.shape[1] != 2 or ev.ndim != 2 or ev.shape[1] != 4:
        return None
    scale = max(np.ptp(v[:, 0]), np.ptp(v[:, 1]), 1.0)
    # build_box_mesh places vertices on a meshgrid of the axis nodes: the
    # distinct coordinates ARE the axis nodes (no rounding)
    xs, ys = np.unique(v[:, 0]), np.unique(v[:, 1])
    nx, ny = len(xs) - 1, len(ys) - 1
    if nx < 1 or ny < 1 or ev.shape[0] != nx * ny:
        return None
    e = np.arange(nx * ny)
    ix, iy = e % nx, e // nx
    want = np.stack([np.stack([xs[ix], ys[iy]], 1), np.stack([xs[ix + 1], ys[iy]], 1),
                     np.stack([xs[ix], ys[iy + 1]], 1), np.stack([xs[ix + 1], ys[iy + 1]], 1)], 1)
    if not np.allclose(v[ev], want, rtol=0.0, atol=rtol * scale):
        return None
    spec = getattr(mesh, "periodic_spec", {}) or {}
    per = (0 in spec, 1 in spec)
    box = BoxMesh.from_axis_vertices([xs, ys], per)
    box.source = mesh
    return box
