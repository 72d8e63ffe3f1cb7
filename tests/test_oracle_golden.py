"""Gate 1: the numpy oracle at DIM=2 reproduces the REAL reference.

Golden vectors were produced by running the reference ``dgins`` package
(tests/golden/make_golden.py); every operator of the hot path is compared
at 1e-13 relative L2 (the reference's own dense-oracle tolerance is 1e-12,
pkg/tests/test_operators.py:85-178).
"""

import numpy as np
import pytest

from oracle import dg_oracle as O
from tests.golden_setups import (KS, SETUPS, body_force, load_golden,
                                 map_tau_c, oracle_setup, relerr)

Z = load_golden()
TOL = 1e-13


def flat(a):
    return np.ascontiguousarray(a).ravel()


@pytest.mark.parametrize("k", range(1, 8))
def test_tables_match_reference(k):
    for f in Z.files:
        if not f.startswith(f"tab_k{k}_q") or not f.endswith("_S"):
            continue
        nq = int(f.split("_q")[1].split("_")[0])
        b = O.get_basis(k, nq)
        key = f"tab_k{k}_q{nq}"
        np.testing.assert_allclose(b.S, Z[key + "_S"], atol=2e-15, rtol=0)
        np.testing.assert_allclose(b.D, Z[key + "_D"], atol=2e-13, rtol=1e-14)
        np.testing.assert_allclose(b.nodes, Z[key + "_nodes"], atol=1e-15)
        np.testing.assert_allclose(b.rule.points, Z[key + "_pts"], atol=1e-15)
        np.testing.assert_allclose(b.rule.weights, Z[key + "_w"], atol=1e-15)
        np.testing.assert_allclose(b.left_deriv, Z[key + "_ld"], rtol=1e-13)
        np.testing.assert_allclose(b.right_deriv, Z[key + "_rd"], rtol=1e-13)


@pytest.mark.parametrize("name", list(SETUPS))
@pytest.mark.parametrize("k", KS)
def test_operators_match_reference(name, k):
    space, bcs = oracle_setup(name, k)
    key = f"{name}_k{k}"
    sh1 = space.field_shape()
    sh2 = space.field_shape(2)
    np.testing.assert_allclose(space.tau_e, Z[key + "_tau_e"], rtol=1e-13)
    np.testing.assert_allclose(space.mesh.h, Z[key + "_h"], rtol=1e-13)
    p = Z[key + "_p"].reshape(sh1)
    u = Z[key + "_u"].reshape(sh2)
    u2 = Z[key + "_u2"].reshape(sh2)
    checks = {
        "_lap": O.apply_pressure_laplace(space, p, bcs),
        "_lap75": O.apply_pressure_laplace(space, p, bcs, tau_scale=7.5),
        "_diag": O.laplace_diagonal(space, bcs),
        "_diag75": O.laplace_diagonal(space, bcs, 7.5),
        "_mass": O.mass_apply(space, u),
        "_invmass": O.inverse_mass_apply(space, u),
        "_helm": O.apply_viscous_helmholtz(space, u, 3.6, 0.025, bcs),
        "_zm": O.zero_mean_project(space, p),
        "_zmd": O.zero_mean_project_dual(space, p),
        "_conv": O.eval_convective_rhs(space, bcs, [u, u2], (2.0, -1.0),
                                       (0.3, 0.2), 0.4, body_force=body_force),
        "_conv1": O.eval_convective_rhs(space, bcs, [u], (1.0,), (0.0,), 0.0),
    }
    tau_d = Z[key + "_tau_d"]
    tau_c = map_tau_c(space, Z, key)
    checks["_proj"] = O.apply_projection_operator(space, u, tau_d, tau_c)
    checks["_projD"] = O.apply_projection_operator(space, u, tau_d, None)
    for suffix, got in checks.items():
        err = relerr(flat(got), Z[key + suffix])
        assert err < TOL, (suffix, err)


@pytest.mark.parametrize("k,nx", [(3, 8), (4, 6)])
def test_solver_histories_match_reference(k, nx):
    """Chebyshev(5,20)-Jacobi and Jacobi PCG on the 2D pure-Neumann problem:
    identical iteration counts and residual histories (2D analogue of
    BASELINE config 2)."""
    mesh = O.build_box_mesh(((0, 1), (0, 1)), (nx, nx), periodic=(True, False))
    spec = O.BoundarySpec({"ymin": O.zero_dirichlet(2), "ymax": O.zero_dirichlet(2)})
    space = O.DgSpace(mesh, k)
    bcs = spec.resolve(space)
    key = f"cg_k{k}_n{nx}"
    sh = space.field_shape()
    L = lambda p: O.apply_pressure_laplace(space, p, bcs)
    op = lambda p: O.zero_mean_project_dual(space, L(p))
    diag = O.laplace_diagonal(space, bcs)
    seed = O.zero_mean_project(space, Z[key + "_seed"].reshape(sh))
    lmax, _ = O.eigen_estimate_via_cg(lambda v: O.zero_mean_project(space, L(v)),
                                      diag, seed, 20)
    assert abs(lmax - float(Z[key + "_lmax"])) < 1e-12 * lmax
    cfg = O.ChebyshevConfig(5, 20.0, 1.1 * lmax)
    b = Z[key + "_b"].reshape(sh)
    for pname, prec in (("cheb", lambda r: O.chebyshev_smooth(L, diag, cfg, r)),
                        ("jac", lambda r: r / diag)):
        x, st = O.pcg(op, prec, b, rel_tol=1e-10, max_iter=2000)
        assert st.converged
        assert st.iterations == int(Z[f"{key}_{pname}_iters"])
        ref_hist = Z[f"{key}_{pname}_hist"]
        got = np.array(st.history)
        n = len(ref_hist) if pname == "cheb" else 60
        np.testing.assert_allclose(got[:n], ref_hist[:n], rtol=1e-9)
        assert relerr(flat(x), Z[f"{key}_{pname}_x"]) < 1e-9


@pytest.mark.parametrize("name", list(SETUPS))
@pytest.mark.parametrize("k", KS)
def test_step_rhs_match_reference(name, k):
    """Once-per-step right-hand sides (operators.py:241-366, 494-527,
    610-672) with non-zero boundary data."""
    space, bcs = oracle_setup(name, k)
    _, bcd = oracle_setup(name, k, data=True)
    key = f"{name}_k{k}"
    p = Z[key + "_p"].reshape(space.field_shape())
    u = Z[key + "_u"].reshape(space.field_shape(2))
    u2 = Z[key + "_u2"].reshape(space.field_shape(2))
    w1 = O.compute_vorticity(space, u)
    w2 = O.compute_vorticity(space, u2)
    checks = {"_vort": w1,
              "_convd": O.eval_convective_rhs(space, bcd, [u, u2], (2.0, -1.0), (0.3, 0.2),
                                              0.4, body_force=body_force)}
    for form in ("standard", "weak", "strong"):
        checks[f"_div_{form}"] = O.eval_divergence_rhs(space, u, bcd, 2.5, form)
    for form in ("standard", "weak"):
        checks[f"_grad_{form}"] = O.eval_pressure_gradient_rhs(space, p, bcd, 1.7, form)
    checks["_pn"] = O.eval_pressure_neumann_rhs(space, bcd, [u, u2], [w1, w2],
                                                (2.0, -1.0), 0.025, 0.4,
                                                body_force=body_force)
    checks["_pn0"] = O.eval_pressure_neumann_rhs(space, bcs, [u], [w1], (1.0,),
                                                 0.025, 0.4)
    checks["_gp"] = O.gp_dirichlet_rhs(space, bcd, 0.3)
    checks["_gp75"] = O.gp_dirichlet_rhs(space, bcd, 0.3, 7.5)
    checks["_vrb"] = O.viscous_rhs_bc(space, bcd, 0.3, 0.025)
    for suffix, got in checks.items():
        want = Z[key + suffix]
        if np.linalg.norm(want) == 0.0:
            assert np.linalg.norm(flat(got)) == 0.0, suffix
            continue
        err = relerr(flat(got), want)
        assert err < TOL, (suffix, err)


@pytest.mark.parametrize("name", list(SETUPS))
@pytest.mark.parametrize("k", KS)
def test_element_local_pcg_matches_reference(name, k):
    """Per-cell CG on M + tau_D div-div with inverse-mass preconditioning:
    identical per-cell iteration counts (solvers.py:201-256)."""
    space, _ = oracle_setup(name, k)
    key = f"{name}_k{k}"
    u = Z[key + "_u"].reshape(space.field_shape(2))
    for tag, rtol, mit in (("el", 1e-8, 200), ("elx", 1e-8, 200),
                           ("el12", 1e-12, 200), ("el5", 1e-14, 5)):
        td = Z[f"{key}_{tag}_tau"]
        x, iters, conv = O.element_local_pcg(
            lambda w: O.apply_projection_operator(space, w, td, None),
            lambda r: O.inverse_mass_apply(space, r), u, rel_tol=rtol, max_iter=mit)
        want = Z[f"{key}_{tag}_iters"]
        np.testing.assert_array_equal(conv, Z[f"{key}_{tag}_conv"])
        if tag == "el5":    # fixed iteration count: the iterate itself agrees
            np.testing.assert_array_equal(iters, want)
            assert relerr(flat(x), Z[f"{key}_{tag}_x"]) < 1e-12
        else:               # converged solves: counts to +-2 (see make_golden)
            assert np.abs(iters - want).max() <= 2, (tag, iters, want)
            assert relerr(flat(x), Z[f"{key}_{tag}_x"]) < (1e-10 if tag == "el12" else 1e-6)


def test_field_vector_roundtrip():
    """FieldVector (reference spaces.py:18-58): zeros, element-major
    serialisation and back, in the 2D reference layout."""
    from types import SimpleNamespace
    from paper_1607_01323_b200.spaces import FieldVector
    space = SimpleNamespace(k=2, dim=2, n_elements=5)
    fv = FieldVector.zeros(space, 2)
    assert fv.data.shape == (2, 3, 5, 3) and fv.ncomp == 2 and fv.n_elements == 5
    fv.data[...] = np.random.default_rng(0).standard_normal(fv.data.shape)
    flat = fv.element_major()
    assert np.array_equal(flat.reshape(2, 5, 3, 3), fv.data.transpose(0, 2, 1, 3))
    back = FieldVector.from_element_major(flat, space, 2)
    assert np.array_equal(back.data, fv.data) and not back.has_nan()


def test_chebyshev_error_factor():
    """solvers.py:132-135: 2 q^n with q = (sqrt(k)-1)/(sqrt(k)+1)."""
    from paper_1607_01323_b200.solvers import chebyshev_error_factor
    assert abs(chebyshev_error_factor(9.0, 3) - 2.0 * 0.5 ** 3) < 1e-15
    assert chebyshev_error_factor(1.0, 5) == 0.0
