"""GPU parity of the once-per-step right-hand sides and the element-local PCG
(reference operators.py:241-366, 494-527, 533-604, 610-672;
solvers.py:201-256).

2D: against golden vectors from the real reference (rel L2 <= 1e-12; the
element-local solves: fixed-iteration iterates to 1e-12, converged solves to
+-2 iterations per cell -- the reference's own counts move by that much under
a change of summation order, see tests/golden/make_golden.py).
3D: against the numpy oracle with non-zero boundary data and body forces."""

import numpy as np
import pytest

from tests.golden_setups import (KS, SETUPS, body_force, body_force3, dgdt_data, dgdt_data3,
                                 g_data, g_data3, gp_data, gp_data3, h_data, h_data3,
                                 load_golden, oracle_bcs, relerr)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1607_01323_b200 import mesh as M  # noqa: E402
from paper_1607_01323_b200 import operators as ops  # noqa: E402
from paper_1607_01323_b200 import solvers as sol  # noqa: E402
from paper_1607_01323_b200.spaces import DgSpace  # noqa: E402
from oracle import dg_oracle as O  # noqa: E402

Z = load_golden()
TOL = 1e-12


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64).ravel(), device="cuda")


def host(t):
    return t.detach().cpu().numpy().ravel()


def check(got, want, tol=TOL, what=""):
    want = np.asarray(want).ravel()
    if np.linalg.norm(want) == 0.0:
        assert np.abs(got).max() == 0.0, what
    else:
        assert relerr(got, want) < tol, (what, relerr(got, want))


def gpu_space(ext, counts, k, per, kinds, grading=None, data=False, dim=2, n_q_over=None):
    mesh = M.build_box_mesh(ext, counts, grading=grading, periodic=per)
    space = DgSpace(mesh, k, n_q_over=n_q_over)
    if data:
        dbc = ops.DirichletBC(g_data if dim == 2 else g_data3,
                              dgdt_data if dim == 2 else dgdt_data3)
        nbc = ops.NeumannBC(h_data if dim == 2 else h_data3, gp_data if dim == 2 else gp_data3)
    else:
        dbc, nbc = ops.DirichletBC(None), ops.NeumannBC(None, None)
    spec = ops.BoundarySpec({t: (dbc if v == "D" else nbc) for t, v in kinds.items()})
    return space, spec.resolve(space)


@pytest.mark.parametrize("name", list(SETUPS))
@pytest.mark.parametrize("k", KS)
def test_2d_golden_rhs(name, k):
    ext, counts, grading, per, kinds = SETUPS[name]
    space, bcd = gpu_space(ext, counts, k, per, kinds, grading, data=True)
    _, bcs = gpu_space(ext, counts, k, per, kinds, grading)
    key = f"{name}_k{k}"
    u, u2, p = dev(Z[key + "_u"]), dev(Z[key + "_u2"]), dev(Z[key + "_p"])
    for form in ("standard", "weak", "strong"):
        check(host(ops.eval_divergence_rhs(space, u, bcd, 2.5, form)),
              Z[f"{key}_div_{form}"], what=form)
    for form in ("standard", "weak"):
        check(host(ops.eval_pressure_gradient_rhs(space, p, bcd, 1.7, form)),
              Z[f"{key}_grad_{form}"], what=form)
    w1 = ops.compute_vorticity(space, u)
    w2 = ops.compute_vorticity(space, u2)
    check(host(w1), Z[key + "_vort"], what="vort")
    check(host(ops.eval_pressure_neumann_rhs(space, bcd, [u, u2], [w1, w2], (2.0, -1.0),
                                             0.025, 0.4, body_force=body_force)),
          Z[key + "_pn"], what="pn")
    check(host(ops.eval_pressure_neumann_rhs(space, bcs, [u], [w1], (1.0,), 0.025, 0.4)),
          Z[key + "_pn0"], what="pn0")
    check(host(ops.gp_dirichlet_rhs(space, bcd, 0.3, like="device")), Z[key + "_gp"], what="gp")
    check(host(ops.gp_dirichlet_rhs(space, bcd, 0.3, 7.5, like="device")), Z[key + "_gp75"],
          what="gp75")
    check(host(ops.viscous_rhs_bc(space, bcd, 0.3, 0.025, like="device")), Z[key + "_vrb"],
          what="vrb")
    check(host(ops.eval_convective_rhs(space, bcd, [u, u2], (2.0, -1.0), (0.3, 0.2), 0.4,
                                       body_force=body_force)), Z[key + "_convd"], what="convd")


@pytest.mark.parametrize("name", list(SETUPS))
@pytest.mark.parametrize("k", KS)
def test_2d_golden_numpy_layout(name, k):
    """Reference-layout numpy in, numpy out (the drop-in call form)."""
    ext, counts, grading, per, kinds = SETUPS[name]
    space, bcd = gpu_space(ext, counts, k, per, kinds, grading, data=True)
    key = f"{name}_k{k}"
    m, ne = k + 1, space.mesh.n_elements
    u = Z[key + "_u"].reshape(2, ne, m, m).transpose(0, 2, 1, 3)     # (2, m, ne, m)
    got = ops.eval_divergence_rhs(space, u, bcd, 2.5, "weak")
    assert got.shape == (m, ne, m)
    check(got.transpose(1, 0, 2).ravel(), Z[f"{key}_div_weak"])
    got = ops.gp_dirichlet_rhs(space, bcd, 0.3)
    assert got.shape == (m, ne, m)
    check(got.transpose(1, 0, 2).ravel(), Z[key + "_gp"])


@pytest.mark.parametrize("name", list(SETUPS))
@pytest.mark.parametrize("k", KS)
def test_2d_golden_element_local_pcg(name, k):
    ext, counts, grading, per, kinds = SETUPS[name]
    space, _ = gpu_space(ext, counts, k, per, kinds, grading)
    key = f"{name}_k{k}"
    u = dev(Z[key + "_u"])
    for tag, rtol, mit in (("el", 1e-8, 200), ("elx", 1e-8, 200), ("el12", 1e-12, 200),
                           ("el5", 1e-14, 5)):
        td = Z[f"{key}_{tag}_tau"]
        x, iters, conv = sol.projection_element_pcg(space, u, td, rel_tol=rtol, max_iter=mit)
        want = Z[f"{key}_{tag}_iters"]
        assert np.array_equal(conv, Z[f"{key}_{tag}_conv"]), tag
        if tag == "el5":
            assert np.array_equal(iters, want)
            assert relerr(host(x), Z[f"{key}_{tag}_x"]) < 1e-12
        else:
            assert np.abs(iters - want).max() <= 2, (tag, iters, want)
            assert relerr(host(x), Z[f"{key}_{tag}_x"]) < (1e-10 if tag == "el12" else 1e-6)


CASES = [
    (((0, 1), (0, 1), (0, 1)), (3, 2, 4), (True, True, True), {}, None),
    (((0, 1), (0, 2), (0, 1)), (2, 3, 2), (False, False, False),
     {"xmin": "D", "xmax": "N", "ymin": "D", "ymax": "D", "zmin": "N", "zmax": "D"}, None),
    (((0, 2), (-1, 1), (0, 1)), (3, 4, 2), (True, False, True),
     {"ymin": "D", "ymax": "N"}, (0.0, 1.8, 0.0)),
]


def oracle_space(ext, counts, k, per, kinds, grading=None, data=False, n_q_over=None):
    om = O.build_box_mesh(ext, counts, grading=grading, periodic=per)
    osp = O.DgSpace(om, k, n_q_over=n_q_over)
    dbc, nbc = oracle_bcs(O, 3, data)
    spec = O.BoundarySpec({t: (dbc if v == "D" else nbc) for t, v in kinds.items()})
    return osp, spec.resolve(osp)


@pytest.mark.parametrize("case", range(len(CASES)))
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6, 7])
def test_3d_rhs_vs_oracle(case, k):
    ext, counts, per, kinds, grading = CASES[case]
    osp, obcs = oracle_space(ext, counts, k, per, kinds, grading, data=True)
    gsp, gbcs = gpu_space(ext, counts, k, per, kinds, grading, data=True, dim=3)
    rng = np.random.default_rng(300 + 10 * case + k)
    u = rng.standard_normal(osp.field_shape(3))
    u2 = rng.standard_normal(osp.field_shape(3))
    p = rng.standard_normal(osp.field_shape())
    for form in ("standard", "weak", "strong"):
        check(host(ops.eval_divergence_rhs(gsp, dev(u), gbcs, 2.5, form)),
              O.eval_divergence_rhs(osp, u, obcs, 2.5, form), what=form)
    for form in ("standard", "weak"):
        check(host(ops.eval_pressure_gradient_rhs(gsp, dev(p), gbcs, 1.7, form)),
              O.eval_pressure_gradient_rhs(osp, p, obcs, 1.7, form), what=form)
    w1, w2 = O.compute_vorticity(osp, u), O.compute_vorticity(osp, u2)
    gw1, gw2 = ops.compute_vorticity(gsp, dev(u)), ops.compute_vorticity(gsp, dev(u2))
    check(host(gw1), w1, what="vort")
    check(host(ops.eval_pressure_neumann_rhs(gsp, gbcs, [dev(u), dev(u2)], [gw1, gw2],
                                             (2.0, -1.0), 0.025, 0.4, body_force=body_force3)),
          O.eval_pressure_neumann_rhs(osp, obcs, [u, u2], [w1, w2], (2.0, -1.0), 0.025, 0.4,
                                      body_force=body_force3), what="pn")
    check(host(ops.gp_dirichlet_rhs(gsp, gbcs, 0.3, 7.5, like="device")),
          O.gp_dirichlet_rhs(osp, obcs, 0.3, 7.5), what="gp")
    check(host(ops.viscous_rhs_bc(gsp, gbcs, 0.3, 0.025, like="device")),
          O.viscous_rhs_bc(osp, obcs, 0.3, 0.025), what="vrb")


@pytest.mark.parametrize("case", range(len(CASES)))
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_3d_convective_with_data(case, k):
    ext, counts, per, kinds, grading = CASES[case]
    osp, obcs = oracle_space(ext, counts, k, per, kinds, grading, data=True)
    gsp, gbcs = gpu_space(ext, counts, k, per, kinds, grading, data=True, dim=3)
    rng = np.random.default_rng(400 + 10 * case + k)
    hist = [rng.standard_normal(osp.field_shape(3)) for _ in range(2)]
    want = O.eval_convective_rhs(osp, obcs, hist, (2.0, -1.0), (0.3, 0.2), 0.4,
                                 body_force=body_force3)
    got = ops.eval_convective_rhs(gsp, gbcs, [dev(h) for h in hist], (2.0, -1.0), (0.3, 0.2),
                                  0.4, body_force=body_force3)
    check(host(got), want)


@pytest.mark.parametrize("case", range(len(CASES)))
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6, 7])
def test_3d_element_local_pcg(case, k):
    ext, counts, per, kinds, grading = CASES[case]
    osp, _ = oracle_space(ext, counts, k, per, kinds, grading)
    gsp, _ = gpu_space(ext, counts, k, per, kinds, grading, dim=3)
    rng = np.random.default_rng(500 + 10 * case + k)
    b = rng.standard_normal(osp.field_shape(3))
    tau_d = np.abs(rng.standard_normal(osp.mesh.n_elements)) * 3.0
    op = lambda w: O.apply_projection_operator(osp, w, tau_d, None)
    prec = lambda r: O.inverse_mass_apply(osp, r)
    # fixed iteration count: iterates agree to rounding
    xo4, io4, co4 = O.element_local_pcg(op, prec, b, rel_tol=1e-14, max_iter=4)
    xg, ig, cg = sol.projection_element_pcg(gsp, dev(b), tau_d, rel_tol=1e-14, max_iter=4)
    assert np.array_equal(ig, io4) and np.array_equal(cg, co4)
    assert relerr(host(xg), xo4.ravel()) < 1e-12
    # converged: counts +-2, solution to the tolerance
    xo, io, co = O.element_local_pcg(op, prec, b, rel_tol=1e-8, max_iter=2000)
    xg, ig, cg = sol.projection_element_pcg(gsp, dev(b), tau_d, rel_tol=1e-8, max_iter=2000)
    assert co.all() and cg.all()
    assert np.abs(ig - io).max() <= 2
    assert relerr(host(xg), xo.ravel()) < 1e-6
    # generic callable version on the device == fused kernel
    gop = lambda w: ops.apply_projection_operator(gsp, w, tau_d, None)
    gprec = lambda r: ops.inverse_mass_apply(gsp, r)
    xt, it, ct = sol.element_local_pcg(gop, gprec, dev(b).view(osp.field_shape(3)),
                                       rel_tol=1e-14, max_iter=4)
    assert np.array_equal(it, io4) and np.array_equal(ct, co4)
    assert relerr(host(xt), xo4.ravel()) < 1e-12


def test_element_local_pcg_edge_cases():
    """tau = 0 -> one iteration, x = M^-1 b (test_solvers_multigrid.py:158-163);
    zero right-hand side -> no iteration, converged; invalid arguments."""
    ext, counts, per, kinds, grading = CASES[1]
    gsp, _ = gpu_space(ext, counts, 3, per, kinds, grading, dim=3)
    rng = np.random.default_rng(7)
    b = dev(rng.standard_normal(3 * gsp.n_dofs))
    x, iters, conv = sol.projection_element_pcg(gsp, b, None)
    assert conv.all() and (iters <= 1).all()
    assert relerr(host(x), host(ops.inverse_mass_apply(gsp, b))) < 1e-13
    x, iters, conv = sol.projection_element_pcg(gsp, torch.zeros_like(b), np.ones(12))
    assert conv.all() and (iters == 0).all() and host(x).max() == 0.0
    with pytest.raises(ValueError):
        sol.projection_element_pcg(gsp, b, np.ones(5))
