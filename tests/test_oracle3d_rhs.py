"""Gate 2 for the once-per-step right-hand sides and the element-local PCG
(reference operators.py:241-366, 494-527, 610-672; solvers.py:201-256) in 3D.

1. Extrusion pin against the REAL reference (2D golden vectors) on a
   z-periodic extruded mesh with z-constant fields and z-free boundary data.
2. Sum factorisation == dense assembly for the divergence / pressure-gradient
   forms (restating pkg/src/dgins/oracle.py:244-348 in 3D), and the weak
   forms' negative-transpose identity (pkg/tests/test_operators.py:243-248).
3. Exactness: the vorticity of a rigid rotation, the pressure Neumann data of
   a polynomial field against its analytic face values, element-local PCG
   against a dense block solve (pkg/tests/test_solvers_multigrid.py:155-195).
"""

import numpy as np
import pytest

from oracle import dg_oracle as O
from oracle.dense import DenseOracle
from tests.golden_setups import (SETUPS, body_force, g_data, dgdt_data, gp_data,
                                 h_data, load_golden, oracle_bcs, relerr)
from tests.test_oracle3d import const3, extrude, lift3, zmass_row

Z = load_golden()


def _z0(f):
    """2D vector boundary data -> z-independent 3D data with zero z part."""
    def g(x, t):
        v = f(x[:2], t)
        return np.concatenate([v, np.zeros((1,) + v.shape[1:])])
    return g


def extrude_data(name, k, nz, hz):
    space, _, sp2, ne2 = extrude(name, k, nz, hz)
    kinds = SETUPS[name][4]
    dbc = O.DirichletBC(_z0(g_data), _z0(dgdt_data))
    nbc = O.NeumannBC(_z0(h_data), lambda x, t: gp_data(x[:2], t))
    spec = O.BoundarySpec({t: (dbc if v == "D" else nbc) for t, v in kinds.items()})
    zspec = O.BoundarySpec({t: (O.zero_dirichlet(3) if v == "D" else O.zero_neumann(3))
                            for t, v in kinds.items()})
    return space, spec.resolve(space), zspec.resolve(space), sp2, ne2


@pytest.mark.parametrize("name", list(SETUPS))
@pytest.mark.parametrize("k", (2, 3))
def test_extrusion_rhs_match_reference_2d(name, k):
    nz, hz = 2, 0.7
    space, bcd, bcs, sp2, ne2 = extrude_data(name, k, nz, hz)
    key = f"{name}_k{k}"
    m = k + 1
    zrow = zmass_row(space.basis, hz / nz)
    sh2 = sp2.field_shape()
    u2 = Z[key + "_u"].reshape(sp2.field_shape(2))
    v2 = Z[key + "_u2"].reshape(sp2.field_shape(2))
    u3 = np.stack([const3(u2[0], nz, m), const3(u2[1], nz, m), np.zeros(space.field_shape())])
    v3 = np.stack([const3(v2[0], nz, m), const3(v2[1], nz, m), np.zeros(space.field_shape())])
    p3 = const3(Z[key + "_p"].reshape(sh2), nz, m)

    def scal(suffix, got):
        want = lift3(Z[key + suffix].reshape(sh2), ne2, nz, zrow)
        if np.linalg.norm(want) == 0.0:
            assert np.abs(got).max() == 0.0, suffix
        else:
            assert relerr(got.ravel(), want.ravel()) < 1e-13, suffix

    def vec(suffix, got):
        want = Z[key + suffix].reshape(sp2.field_shape(2))
        if np.linalg.norm(want) == 0.0:
            assert np.abs(got).max() == 0.0, suffix
            return
        for c in range(2):
            assert relerr(got[c].ravel(), lift3(want[c], ne2, nz, zrow).ravel()) < 1e-13
        assert np.abs(got[2]).max() <= 1e-13 * np.abs(got[:2]).max()

    for form in ("standard", "weak", "strong"):
        scal(f"_div_{form}", O.eval_divergence_rhs(space, u3, bcd, 2.5, form))
    for form in ("standard", "weak"):
        vec(f"_grad_{form}", O.eval_pressure_gradient_rhs(space, p3, bcd, 1.7, form))
    w1 = O.compute_vorticity(space, u3)
    w2 = O.compute_vorticity(space, v3)
    assert np.abs(w1[:2]).max() < 1e-12 * np.abs(w1[2]).max()
    assert relerr(w1[2].ravel(), const3(Z[key + "_vort"].reshape(sh2), nz, m).ravel()) < 1e-13
    scal("_pn0", O.eval_pressure_neumann_rhs(space, bcs, [u3], [w1], (1.0,), 0.025, 0.4))
    bf3 = _z0(body_force)
    scal("_pn", O.eval_pressure_neumann_rhs(space, bcd, [u3, v3], [w1, w2], (2.0, -1.0),
                                            0.025, 0.4, body_force=bf3))
    scal("_gp", O.gp_dirichlet_rhs(space, bcd, 0.3))
    scal("_gp75", O.gp_dirichlet_rhs(space, bcd, 0.3, 7.5))
    vec("_vrb", O.viscous_rhs_bc(space, bcd, 0.3, 0.025))


def setup3d(kind, k, counts=(2, 2, 2), data=False):
    dbc, nbc = oracle_bcs(O, 3, data)
    if kind == "periodic":
        mesh = O.build_box_mesh(((0, 1), (0, 1), (0, 1)), counts, periodic=(True,) * 3)
        spec = O.BoundarySpec({})
    elif kind == "walls":
        mesh = O.build_box_mesh(((0, 1), (0, 2), (0, 1)), counts)
        spec = O.BoundarySpec({t: dbc for t in O.TAG_NAMES})
    else:
        mesh = O.build_box_mesh(((0, 1), (-1, 1), (0, 0.5)), counts,
                                grading=(0.0, 1.2, 0.0), periodic=(True, False, False))
        spec = O.BoundarySpec({"ymin": dbc, "ymax": nbc, "zmin": nbc, "zmax": dbc})
    space = O.DgSpace(mesh, k)
    return space, spec.resolve(space)


KINDS3 = ["periodic", "walls", "mixed"]


@pytest.mark.parametrize("kind", KINDS3)
@pytest.mark.parametrize("k", (1, 2))
def test_divergence_gradient_dense(kind, k, rng):
    space, bcs = setup3d(kind, k)
    dense = DenseOracle(space)
    u = rng.standard_normal(space.field_shape(3))
    p = rng.standard_normal(space.field_shape())
    for form in ("standard", "weak"):
        A = dense.divergence_form_matrix(bcs, 2.5, form)
        got = O.eval_divergence_rhs(space, u, bcs, 2.5, form).ravel()
        assert relerr(got, A @ u.ravel()) < 1e-12
        B = dense.pressure_gradient_matrix(bcs, 1.7, form)
        got = O.eval_pressure_gradient_rhs(space, p, bcs, 1.7, form).ravel()
        assert relerr(got, B @ p.ravel()) < 1e-12
    # weak == strong divergence (pkg/tests/test_operators.py:232-241)
    aw = O.eval_divergence_rhs(space, u, bcs, 1.3, "weak")
    st = O.eval_divergence_rhs(space, u, bcs, 1.3, "strong")
    assert np.linalg.norm(aw - st) <= 1e-12 * max(np.linalg.norm(aw), 1.0)
    if kind == "periodic":   # pkg/tests/test_operators.py:243-248
        A = dense.divergence_form_matrix(bcs, 1.0, "weak")
        B = dense.pressure_gradient_matrix(bcs, 1.0, "weak")
        assert relerr(B, -A.T) < 1e-12


def test_vorticity_known_fields():
    """pkg/tests/test_operators.py:285-301 in 3D: constant -> 0, rigid
    rotation w x r -> 2 w, gradient field -> 0."""
    space, _ = setup3d("mixed", 3, counts=(2, 3, 2))
    x, y, z = space.node_coords()
    u = np.stack([np.full_like(x, 1.5), np.full_like(x, -2.0), np.full_like(x, 0.3)])
    np.testing.assert_allclose(O.compute_vorticity(space, u), 0.0, atol=1e-12)
    om = np.array([0.4, -1.1, 2.0])
    u = np.stack([om[1] * z - om[2] * y, om[2] * x - om[0] * z, om[0] * y - om[1] * x])
    w = O.compute_vorticity(space, u)
    for c in range(3):
        np.testing.assert_allclose(w[c], 2.0 * om[c], atol=1e-11)
    u = np.stack([x, y, z])
    np.testing.assert_allclose(O.compute_vorticity(space, u), 0.0, atol=1e-11)


def test_pressure_neumann_rhs_polynomial_field():
    """Degree-2 velocity (exact at k=3): the lifted data must equal the face
    integral of the analytic -(div(u u) + nu curl curl u) . n."""
    k, nu = 3, 0.3
    space, bcs = setup3d("walls", k, counts=(2, 2, 2))
    x, y, z = space.node_coords()
    u = np.stack([x * y + z * z, 0.5 * x * x - y * z, x * z + y])
    w = O.compute_vorticity(space, u)
    got = O.eval_pressure_neumann_rhs(space, bcs, [u], [w], (1.0,), nu, 0.0)

    def h_exact(X):
        xx, yy, zz = X
        ux, uy, uz = xx * yy + zz * zz, 0.5 * xx * xx - yy * zz, xx * zz + yy
        # grad[c][a] = d u_c / d x_a
        gr = [[yy, xx, 2 * zz], [xx, -zz, -yy], [zz, 1.0 + 0 * xx, xx]]
        div = gr[0][0] + gr[1][1] + gr[2][2]
        uu = [ux, uy, uz]
        conv = [uu[a] * div + sum(uu[c] * gr[a][c] for c in range(3)) for a in range(3)]
        # curl curl u = grad div u - lap u ; div u = y - z + x, lap u = (2, 1, 0)
        cc = [1.0 - 2.0, 1.0 - 1.0, -1.0 - 0.0]
        return [conv[a] + nu * cc[a] for a in range(3)]

    b, g = space.basis, space.geom
    Vc, = O._zeros_faces(space, 1, b.n_q)
    for eb, sb, _ in bcs.dirichlet:
        xb = O._face_points(space, g, b, eb, sb)
        h = h_exact(xb)
        hn = sum(h[a] * g.normal[a][sb, eb] for a in range(3))
        Vc[sb, eb] = -hn * g.sjxw[sb, eb]
    want = np.zeros(space.field_shape())
    O.face_lift_values(Vc, b, want, 3)
    assert relerr(got.ravel(), want.ravel()) < 1e-12


@pytest.mark.parametrize("k", (2, 3))
def test_element_local_pcg_dense_block_solve(k, rng):
    """pkg/tests/test_solvers_multigrid.py:165-182 in 3D."""
    space, _ = setup3d("mixed", k, counts=(2, 2, 1))
    ne = space.mesh.n_elements
    tau_d = np.full(ne, 0.8)
    b = rng.standard_normal(space.field_shape(3))
    x, iters, conv = O.element_local_pcg(
        lambda v: O.apply_projection_operator(space, v, tau_d, None),
        lambda r: O.inverse_mass_apply(space, r), b, rel_tol=1e-13)
    assert conv.all()
    P = DenseOracle(space).projection_matrix(tau_d, None)
    np.testing.assert_allclose(x.ravel(), np.linalg.solve(P, b.ravel()), atol=1e-10)
    # tau = 0: one iteration, x = M^-1 b (test_solvers_multigrid.py:158-163)
    x, iters, conv = O.element_local_pcg(
        lambda v: O.apply_projection_operator(space, v, None, None),
        lambda r: O.inverse_mass_apply(space, r), b)
    assert conv.all() and (iters <= 1).all()
    np.testing.assert_allclose(x, O.inverse_mass_apply(space, b), atol=1e-11)
