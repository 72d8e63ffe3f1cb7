"""The multigrid oracle (oracle/multigrid.py) reproduces the REAL reference
V-cycle (pkg/src/dgins/multigrid.py) in 2D: transfer, per-level Lanczos
lambda_max, coarse iteration count, V-cycle action and MG-preconditioned PCG
(iterations and residual history; golden vectors tests/golden/ref2d_mg.npz),
plus DIM=3 structural checks (constant / polynomial reproduction,
restriction = prolongation^T, V-cycle linearity, PCG <= 15 iterations)."""

import os

import numpy as np
import pytest

from oracle import dg_oracle as O
from oracle import multigrid as MG
from tests.golden_setups import relerr

ZM = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref2d_mg.npz"))
CASES = {"per_l2_k3": (2, 3, True), "per_l3_k3": (3, 3, True), "per_l2_k5": (2, 5, True),
         "mix_l3_k3": (3, 3, False), "mix_l0_k2": (0, 2, False)}


def ref_layout_draw(rng, space):
    """The reference draws its Lanczos seeds in the 2D kernel layout (m, ne, m)."""
    m, ne = space.k + 1, space.mesh.n_elements
    return np.ascontiguousarray(rng.standard_normal((m, ne, m)).transpose(1, 0, 2))


def spaces_of(levels, k, periodic, dim=2):
    base = (2,) * dim
    meshes = MG.box_mesh_hierarchy(((0, 1),) * dim, base, levels, periodic=(periodic,) * dim)
    return [O.DgSpace(m, k) for m in meshes]


def spec_of(periodic, dim=2):
    if periodic:
        return O.BoundarySpec({})
    kinds = {"xmin": O.zero_dirichlet(dim), "xmax": O.zero_neumann(dim),
             "ymin": O.zero_dirichlet(dim), "ymax": O.zero_dirichlet(dim)}
    if dim == 3:
        kinds.update({"zmin": O.zero_dirichlet(dim), "zmax": O.zero_neumann(dim)})
    return O.BoundarySpec(kinds)


def test_transfer_matches_reference():
    sp = spaces_of(1, 3, False)
    tr = MG.Transfer(sp[0], sp[1])
    xc = ZM["tr_xc"].reshape(sp[0].field_shape())
    yf = ZM["tr_yf"].reshape(sp[1].field_shape())
    assert relerr(tr.prolong(xc).ravel(), ZM["tr_prolong"]) < 1e-14
    assert relerr(tr.restrict(yf).ravel(), ZM["tr_restrict"]) < 1e-14


@pytest.mark.parametrize("name", list(CASES))
def test_hierarchy_vcycle_pcg_match_reference(name):
    levels, k, periodic = CASES[name]
    spaces = spaces_of(levels, k, periodic)
    proj = O.zero_mean_project if periodic else None
    mg = MG.MultigridHierarchy(spaces, spec_of(periodic), project=proj, seed_draw=ref_layout_draw)
    lmax = np.array([lv.cheb.lambda_max for lv in mg.levels])
    np.testing.assert_allclose(lmax, ZM[f"{name}_lmax"], rtol=1e-11)
    assert mg.levels[0].coarse_iters == int(ZM[f"{name}_coarse_iters"])
    space = spaces[-1]
    b = ZM[f"{name}_vb"].reshape(space.field_shape())
    # the reference applies its coarse operator as a compiled dense block:
    # same action up to roundoff (multigrid.py:126-128)
    assert relerr(mg.vcycle(b).ravel(), ZM[f"{name}_vx"]) < 1e-10
    if levels == 0:
        return
    bcs = spec_of(periodic).resolve(space)
    b = ZM[f"{name}_b"].reshape(space.field_shape())
    if periodic:
        op = lambda p: O.zero_mean_project_dual(space, O.apply_pressure_laplace(space, p, bcs))
    else:
        op = lambda p: O.apply_pressure_laplace(space, p, bcs)
    x, st = O.pcg(op, mg.vcycle, b, rel_tol=1e-8, max_iter=40)
    assert st.converged and st.iterations == int(ZM[f"{name}_iters"])
    np.testing.assert_allclose(st.history, ZM[f"{name}_hist"], rtol=1e-8)
    assert relerr(x.ravel(), ZM[f"{name}_x"]) < 1e-8


def test_transfer_3d_identities(rng):
    sp = spaces_of(1, 3, False, dim=3)
    tr = MG.Transfer(sp[0], sp[1])
    np.testing.assert_allclose(tr.prolong(np.full(sp[0].field_shape(), 3.0)), 3.0, atol=1e-13)
    # degree-k polynomial reproduced exactly on the children
    f = lambda X: X[0] ** 3 + X[0] * X[1] ** 2 - 2 * X[1] * X[2] ** 2 + X[2]
    pc, pf = f(sp[0].node_coords()), f(sp[1].node_coords())
    np.testing.assert_allclose(tr.prolong(pc), pf, atol=1e-12)
    xc = rng.standard_normal(sp[0].field_shape())
    yf = rng.standard_normal(sp[1].field_shape())
    assert np.vdot(tr.prolong(xc), yf) == pytest.approx(np.vdot(xc, tr.restrict(yf)), rel=1e-13)


def test_vcycle_3d_linear_and_pcg_bound(rng):
    spaces = spaces_of(2, 2, False, dim=3)
    spec = spec_of(False, dim=3)
    mg = MG.MultigridHierarchy(spaces, spec)
    space = spaces[-1]
    b1, b2 = rng.standard_normal(space.field_shape()), rng.standard_normal(space.field_shape())
    lhs = mg.vcycle(0.7 * b1 - 1.9 * b2)
    rhs = 0.7 * mg.vcycle(b1) - 1.9 * mg.vcycle(b2)
    assert np.linalg.norm(lhs - rhs) <= 1e-12 * max(np.linalg.norm(rhs), 1.0)
    bcs = spec.resolve(space)
    x, st = O.pcg(lambda p: O.apply_pressure_laplace(space, p, bcs), mg.vcycle, b1,
                  rel_tol=1e-8, max_iter=40)
    assert st.converged and st.iterations <= 15
