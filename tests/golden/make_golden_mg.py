"""Golden vectors for the geometric multigrid V-cycle, from the REAL reference
(pkg/src/dgins/multigrid.py, mesh.py:354-374) in 2D.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_mg.py

Writes tests/golden/ref2d_mg.npz (committed).  Cases follow
pkg/tests/test_solvers_multigrid.py:195-288 (transfer identities, V-cycle,
MG-preconditioned PCG on periodic and mixed-BC hierarchies).  Vectors are
element-major (element, y-node, x-node); the Lanczos seed draws of the
hierarchy happen inside the reference in its kernel layout (m, ne, m) --
consumers reproduce them with ``default_rng(987)`` draws of that shape.
"""

import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from dgins import operators as ops  # noqa: E402
from dgins import solvers as sol  # noqa: E402
from dgins.mesh import box_mesh_hierarchy  # noqa: E402
from dgins.multigrid import MultigridHierarchy, Transfer  # noqa: E402
from dgins.spaces import DgSpace, FieldVector  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref2d_mg.npz")


def em(space, a):
    return FieldVector(a[None] if a.ndim == 3 else a, space.k).element_major()


def unem(space, f):
    return FieldVector.from_element_major(f, space, 1).data[0]


def spaces_of(levels, k, periodic):
    meshes = box_mesh_hierarchy(((0, 1), (0, 1)), (2, 2), levels,
                                periodic=(periodic, periodic))
    return [DgSpace(m, k) for m in meshes]


def z2(x, t):
    return np.zeros((2,) + x.shape[1:])


def z1(x, t):
    return np.zeros(x.shape[1:])


MIXED = {"xmin": ops.DirichletBC(z2), "xmax": ops.NeumannBC(z2, z1),
         "ymin": ops.DirichletBC(z2), "ymax": ops.DirichletBC(z2)}

CASES = {
    # name: (levels, k, periodic)
    "per_l2_k3": (2, 3, True),
    "per_l3_k3": (3, 3, True),
    "per_l2_k5": (2, 5, True),
    "mix_l3_k3": (3, 3, False),
    "mix_l0_k2": (0, 2, False),
}


def main():
    out = {}
    rng = np.random.default_rng(20261020)
    # transfer (multigrid.py:33-73) on a 2 -> 4 hierarchy, k = 3
    sp = spaces_of(1, 3, False)
    tr = Transfer(sp[0], sp[1])
    xc = rng.standard_normal((4, 4, 4))
    yf = rng.standard_normal((4, 16, 4))
    out["tr_xc"] = em(sp[0], xc)
    out["tr_yf"] = em(sp[1], yf)
    out["tr_prolong"] = em(sp[1], tr.prolong(xc))
    out["tr_restrict"] = em(sp[0], tr.restrict(yf))
    for name, (levels, k, periodic) in CASES.items():
        spaces = spaces_of(levels, k, periodic)
        spec = ops.BoundarySpec({} if periodic else MIXED)
        proj = sol.zero_mean_project if periodic else None
        mg = MultigridHierarchy(spaces, spec, project=proj)
        out[f"{name}_lmax"] = np.array([lv.cheb.lambda_max for lv in mg.levels])
        out[f"{name}_coarse_iters"] = np.array(mg.levels[0].coarse_iters)
        out[f"{name}_coarse_range"] = np.array(mg.levels[0].coarse_range)
        space = spaces[-1]
        bcs = spec.resolve(space)
        m = k + 1
        shape = (m, space.mesh.n_elements, m)
        b = rng.standard_normal(shape)
        if periodic:
            b = sol.zero_mean_project(space, b)
        out[f"{name}_vb"] = em(space, b)
        out[f"{name}_vx"] = em(space, mg.vcycle(b))
        if levels == 0:
            continue
        b = rng.standard_normal(shape)
        if periodic:
            b = sol.zero_mean_project_dual(space, b)
            op = lambda p: sol.zero_mean_project_dual(
                space, ops.apply_pressure_laplace(space, p, bcs))
        else:
            op = lambda p: ops.apply_pressure_laplace(space, p, bcs)
        hist = []

        def prec(r, hist=hist):
            z = mg.vcycle(r)
            hist.append(np.sqrt(max(np.vdot(r, z).real, 0.0)))
            return z
        x, st = sol.pcg(op, prec, b, rel_tol=1e-8, max_iter=40)
        out[f"{name}_b"] = em(space, b)
        out[f"{name}_x"] = em(space, x)
        out[f"{name}_hist"] = np.array(hist)
        out[f"{name}_iters"] = np.array(st.iterations)
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, len(out), "arrays")


if __name__ == "__main__":
    main()
