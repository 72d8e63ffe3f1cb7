"""Geometric multigrid V-cycle preconditioner on the GPU (reference
pkg/src/dgins/multigrid.py, nested boxes of pkg/src/dgins/mesh.py:354-374).

Same names and semantics as the reference:

  box_mesh_hierarchy(extents, base_counts, levels, ...)     mesh.py:354
  Transfer(coarse, fine).prolong / .restrict               multigrid.py:33-73
  MultigridHierarchy(spaces, bc_spec, tau_scale, degree, smoothing_range,
                     coarse_tol, est_iters, safety, seed, project)
      .vcycle(b)                                            multigrid.py:76-151

The hierarchy setup (Jacobi diagonals, the seeded Lanczos estimates, the
coarse Chebyshev count) runs on the device through the generic solvers; the
V-cycle itself is one C call (dg_mg_vcycle): Chebyshev smoothing with fused
vmult epilogues, residual, restriction, recursion, prolongation -- all device
kernels, no host round trip.  ``laplace_pcg_mg`` runs the whole MG-PCG on the
device (dg_laplace_pcg_mg).
"""

import ctypes
import math
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from . import _lib
from .mesh import build_box_mesh
from .operators import _Arg, ctypes_ptr, _stream, laplace_diagonal, apply_pressure_laplace
from .solvers import SolverStats, eigen_estimate_via_cg, _to_dev
from .spaces import _torch


def box_mesh_hierarchy(extents, base_counts, levels, grading=None, delta=1.0,
                       periodic=None, k_geo=1):
    """Nested boxes with base_counts * 2^l cells per axis, l = 0..levels
    (mesh.py:354-374; grading applies to the uniform parameter, so coarse
    vertices are a subset of the fine ones)."""
    return [build_box_mesh(extents, tuple(c * 2 ** l for c in base_counts), grading=grading,
                           delta=delta, periodic=periodic, k_geo=k_geo)
            for l in range(levels + 1)]


class Transfer:
    """Polynomial embedding between a space and its 2x refinement
    (multigrid.py:33-73)."""

    def __init__(self, coarse, fine):
        for d in range(fine.dim):
            if fine.mesh.counts[d] != 2 * coarse.mesh.counts[d]:
                raise ValueError("fine mesh must refine the coarse one 2x per axis")
        if fine.k != coarse.k:
            raise ValueError("levels need the same polynomial degree")
        self.coarse, self.fine = coarse, fine

    def _ctx(self, space):
        return space.ctx(space.default_kinds())

    def prolong(self, xc, out=None, add=False):
        a = _Arg(self.coarse, xc, 1)
        torch = _torch()
        xf = out if out is not None else torch.empty(self.fine.n_dofs, dtype=torch.float64,
                                                      device="cuda")
        _lib.call("dg_mg_prolong", self._ctx(self.coarse).handle, self._ctx(self.fine).handle,
                  a.ptr(), ctypes_ptr(xf.data_ptr()), int(add), _stream())
        if a.is_torch:
            return xf
        return self.fine.from_element_major(xf.cpu().numpy(), 1, self._like(self.fine, a.shape))

    def restrict(self, xf):
        a = _Arg(self.fine, xf, 1)
        torch = _torch()
        xc = torch.empty(self.coarse.n_dofs, dtype=torch.float64, device="cuda")
        _lib.call("dg_mg_restrict", self._ctx(self.fine).handle, self._ctx(self.coarse).handle,
                  a.ptr(), ctypes_ptr(xc.data_ptr()), _stream())
        if a.is_torch:
            return xc
        return self.coarse.from_element_major(xc.cpu().numpy(), 1,
                                              self._like(self.coarse, a.shape))

    @staticmethod
    def _like(space, shape):
        m, ne = space.k + 1, space.mesh.n_elements
        if space.dim == 2 and len(shape) == 3 and shape[1] != m:
            return (m, ne, m)            # reference kernel layout
        return space.field_shape()


@dataclass
class MgLevel:
    space: object
    bcs: object
    diag: object              # device Jacobi diagonal
    lambda_max: float         # safety x Lanczos estimate
    lambda_min: float
    coarse_iters: Optional[int] = None
    coarse_range: Optional[float] = None


def reference_seed_draw(rng, space):
    """The reference draws each level's Lanczos start vector as
    rng.standard_normal(diag.shape): the 2D kernel layout (m, ne, m); in 3D
    (no reference) the element-major field shape.  Returned element-major."""
    m, ne = space.k + 1, space.mesh.n_elements
    if space.dim == 2:
        return np.ascontiguousarray(rng.standard_normal((m, ne, m)).transpose(1, 0, 2))
    return rng.standard_normal(space.field_shape())


class MultigridHierarchy:
    """Levels coarse (0) to fine (-1) plus transfers (multigrid.py:76-151)."""

    def __init__(self, spaces, bc_spec, tau_scale: float = 1.0, degree: int = 5,
                 smoothing_range: float = 20.0, coarse_tol: float = 1e-3, est_iters: int = 20,
                 safety: float = 1.1, seed: int = 987, project: Optional[Callable] = None,
                 dense_coarse_limit: int = 4096, seed_draw: Callable = reference_seed_draw,
                 precision: str = "fp64"):
        if len(spaces) < 1:
            raise ValueError("hierarchy needs at least one level")
        if degree < 0:
            raise ValueError("Chebyshev degree must be >= 0")
        if smoothing_range <= 1.0:
            raise ValueError("smoothing range must exceed 1")
        del dense_coarse_limit  # the reference's dense coarse block is a CPU speed measure
        rng = np.random.default_rng(seed)
        self.levels = []
        self.tau_scale, self.degree, self.smoothing_range = tau_scale, degree, smoothing_range
        for lvl, space in enumerate(spaces):
            bcs = bc_spec.resolve(space)
            diag = laplace_diagonal(space, bcs, tau_scale)
            seed_vec = _to_dev(seed_draw(rng, space)).reshape(-1)
            op = (lambda s, b: lambda p: apply_pressure_laplace(s, p, b, tau_scale))(space, bcs)
            est_op = op
            if project is not None:
                seed_vec = project(space, seed_vec)
                est_op = (lambda o, s: lambda p: project(s, o(p)))(op, space)
            lmax, lmin = eigen_estimate_via_cg(est_op, diag, seed_vec, est_iters)
            level = MgLevel(space, bcs, diag, safety * lmax, lmin)
            if lvl == 0:
                kappa = (safety * lmax) / max(lmin / safety, 1e-12 * lmax)
                q = (math.sqrt(kappa) - 1.0) / (math.sqrt(kappa) + 1.0)
                n = math.ceil(math.log(2.0 / coarse_tol) / -math.log(max(q, 1e-12)))
                level.coarse_iters = max(n, 1)
                level.coarse_range = kappa
            self.levels.append(level)
        self.transfers = [Transfer(c.space, f.space)
                          for c, f in zip(self.levels[:-1], self.levels[1:])]
        ctxs = [lv.space.ctx(lv.bcs.kinds) for lv in self.levels]
        nl = len(ctxs)
        self._ctxs = ctxs
        lev = (ctypes.c_void_p * nl)(*[c.handle.value for c in ctxs])
        dg = (ctypes.c_void_p * nl)(*[lv.diag.data_ptr() for lv in self.levels])
        lm = (ctypes.c_double * nl)(*[lv.lambda_max for lv in self.levels])
        h = ctypes.c_void_p()
        c0 = self.levels[0]
        _lib.call("dg_mg_create", ctypes.cast(lev, ctypes.c_void_p), nl,
                  ctypes.cast(dg, ctypes.c_void_p), ctypes.cast(lm, ctypes.c_void_p),
                  int(degree), float(smoothing_range), int(c0.coarse_iters),
                  float(c0.coarse_range), float(tau_scale), ctypes.byref(h))
        self._h = h
        if precision not in ("fp64", "fp32"):
            raise ValueError("precision must be 'fp64' or 'fp32'")
        self.precision = precision
        if precision == "fp32":
            # the paper's single-precision V-cycle; the outer
            # CG stays fp64
            _lib.call("dg_mg_set_precision", h, 32)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.lib().dg_mg_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def n_levels(self):
        return len(self.levels)

    @property
    def handle(self):
        return self._h

    def vcycle(self, b):
        """x = V(b) on the finest level (multigrid.py:133-151)."""
        top = self.levels[-1].space
        a = _Arg(top, b, 1)
        torch = _torch()
        x = torch.empty(top.n_dofs, dtype=torch.float64, device="cuda")
        _lib.call("dg_mg_vcycle", self._h, a.ptr(), ctypes_ptr(x.data_ptr()), _stream())
        return a.result(x)


def laplace_pcg_mg(mg: MultigridHierarchy, b, project_dual: bool = False,
                   rel_tol: float = 1e-8, abs_tol: float = 0.0, max_iter: int = 1000):
    """Fused device PCG on the finest level with the V-cycle as
    preconditioner: ``pcg(op, mg.vcycle, b)`` of the reference
    (solvers.py:30-73, pkg/tests/test_solvers_multigrid.py:254-288).
    Returns (x, SolverStats with the sqrt(r.z) history)."""
    torch = _torch()
    top = mg.levels[-1]
    a = _Arg(top.space, b, 1)
    x = torch.empty(top.space.n_dofs, dtype=torch.float64, device="cuda")
    prm = _lib.PcgParams()
    prm.tau_scale = mg.tau_scale
    prm.project_dual = int(project_dual)
    prm.cheb_degree, prm.cheb_range, prm.cheb_lambda_max = 0, 20.0, 1.0
    prm.rel_tol, prm.abs_tol, prm.max_iter = rel_tol, abs_tol, max_iter
    st = _lib.PcgStats()
    hist = np.zeros(max_iter + 1)
    _lib.call("dg_laplace_pcg_mg", mg._ctxs[-1].handle, mg.handle, a.ptr(),
              ctypes_ptr(x.data_ptr()), ctypes.byref(prm), ctypes.byref(st),
              hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), _stream())
    stats = SolverStats(st.iterations, st.residual, bool(st.converged), bool(st.breakdown),
                        list(hist[:st.iterations + 1]))
    return a.result(x), stats
