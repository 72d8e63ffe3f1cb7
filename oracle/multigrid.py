"""Geometric multigrid V-cycle -- TEST INFRASTRUCTURE (CPU oracle).

Restates the reference's pkg/src/dgins/multigrid.py (and the nested box
hierarchy of pkg/src/dgins/mesh.py:354-374) for DIM in {2, 3} on the
element-major layout of ``dg_oracle`` (cell axis 0 of a scalar field,
x fastest).  Same degree on every level; the transfer is the tensorial
polynomial embedding of a parent cell into its 2^dim children
(multigrid.py:33-73), restriction its transpose; smoother Chebyshev
(degree, range) over Jacobi with lambda_max = safety x the Lanczos estimate
of a CG run on a seeded standard-normal vector per level (multigrid.py:
100-114); coarsest level a fixed-count Chebyshev iteration whose count comes
from the classic bound reaching coarse_tol (multigrid.py:116-125).  The
reference's optional dense coarse block (multigrid.py:126-128) is a pure
speed measure with the same action up to roundoff and is not restated.
"""

import math
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from . import dg_oracle as O


def box_mesh_hierarchy(extents, base_counts, levels, grading=None, delta=1.0,
                       periodic=None):
    """Nested boxes with base_counts * 2^l cells per axis (mesh.py:354-374)."""
    dim = len(base_counts)
    return [O.build_box_mesh(extents, tuple(c * 2 ** l for c in base_counts),
                             grading=grading, delta=delta, periodic=periodic)
            for l in range(levels + 1)]


class Transfer:
    """Polynomial embedding coarse -> fine (multigrid.py:33-73)."""

    def __init__(self, coarse, fine):
        self.dim = fine.dim
        for d in range(self.dim):
            if fine.mesh.counts[d] != 2 * coarse.mesh.counts[d]:
                raise ValueError("fine mesh must refine the coarse one 2x per axis")
        nodes = O.gll_nodes(fine.k)
        self.E = [O.lagrange_values(nodes, 0.5 * (nodes - 1.0)),
                  O.lagrange_values(nodes, 0.5 * (nodes + 1.0))]
        self.coarse, self.fine = coarse, fine
        cf = np.asarray(fine.mesh.cell_index)               # (dim, ne_f)
        cc = np.asarray(coarse.mesh.counts)
        par = np.zeros(cf.shape[1], dtype=np.int64)
        stride = 1
        for d in range(self.dim):
            par += (cf[d] // 2) * stride
            stride *= cc[d]
        self.parent = par
        self.child = [cf[d] % 2 for d in range(self.dim)]  # per axis 0/1

    def _apply(self, x, mats_of_cell, transpose):
        """Apply per-cell tensor products of the 1D embeddings."""
        dim = self.dim
        out = x
        for d in range(dim):
            ax = O._ax(dim, d)       # array axis of direction d (cell axis 0)
            E = self.E
            res = np.empty_like(out)
            for c in (0, 1):
                sel = self.child[d] == c
                T = E[c].T if transpose else E[c]
                res[sel] = O._contract(out[sel], T, ax)
            out = res
        return out

    def prolong(self, xc):
        return self._apply(xc[self.parent], None, False)

    def restrict(self, xf):
        t = self._apply(xf, None, True)
        out = np.zeros(self.coarse.field_shape())
        np.add.at(out, self.parent, t)
        return out


@dataclass
class MgLevel:
    space: object
    op: Callable
    diag: np.ndarray
    cheb: O.ChebyshevConfig
    lmin: float = 0.0
    coarse_iters: Optional[int] = None
    coarse_range: Optional[float] = None


class MultigridHierarchy:
    """multigrid.py:76-151, DIM-generic.  ``seed_draw(rng, space)`` returns
    the level's Lanczos start vector in element-major layout (default: a
    standard-normal draw of the element-major field shape; the 2D golden
    tests pass the reference's kernel-layout draw)."""

    def __init__(self, spaces, bc_spec, tau_scale=1.0, degree=5, smoothing_range=20.0,
                 coarse_tol=1e-3, est_iters=20, safety=1.1, seed=987, project=None,
                 seed_draw=None):
        if len(spaces) < 1:
            raise ValueError("hierarchy needs at least one level")
        self.levels, self.transfers = [], []
        rng = np.random.default_rng(seed)
        for lvl, space in enumerate(spaces):
            bcs = bc_spec.resolve(space)
            op = (lambda s, b: lambda p: O.apply_pressure_laplace(s, p, b, tau_scale))(space, bcs)
            diag = O.laplace_diagonal(space, bcs, tau_scale)
            seed_vec = (seed_draw(rng, space) if seed_draw is not None
                        else rng.standard_normal(diag.shape))
            est_op = op
            if project is not None:
                seed_vec = project(space, seed_vec)
                est_op = (lambda o, s: lambda p: project(s, o(p)))(op, space)
            lmax, lmin = O.eigen_estimate_via_cg(est_op, diag, seed_vec, est_iters)
            level = MgLevel(space, op, diag,
                            O.ChebyshevConfig(degree, smoothing_range, safety * lmax), lmin)
            if lvl == 0:
                kappa = (safety * lmax) / max(lmin / safety, 1e-12 * lmax)
                q = (math.sqrt(kappa) - 1.0) / (math.sqrt(kappa) + 1.0)
                n = math.ceil(math.log(2.0 / coarse_tol) / -math.log(max(q, 1e-12)))
                level.coarse_iters = max(n, 1)
                level.coarse_range = kappa
            self.levels.append(level)
        for c, f in zip(self.levels[:-1], self.levels[1:]):
            self.transfers.append(Transfer(c.space, f.space))

    @property
    def n_levels(self):
        return len(self.levels)

    def vcycle(self, b):
        return self._cycle(b, self.n_levels - 1)

    def _cycle(self, b, lvl):
        level = self.levels[lvl]
        if lvl == 0:
            cfg = O.ChebyshevConfig(level.coarse_iters, max(level.coarse_range, 1.0 + 1e-8),
                                    level.cheb.lambda_max)
            return O.chebyshev_smooth(level.op, level.diag, cfg, b)
        x = O.chebyshev_smooth(level.op, level.diag, level.cheb, b)
        r = b - level.op(x)
        xc = self._cycle(self.transfers[lvl - 1].restrict(r), lvl - 1)
        x += self.transfers[lvl - 1].prolong(xc)
        return O.chebyshev_smooth(level.op, level.diag, level.cheb, b, x)
