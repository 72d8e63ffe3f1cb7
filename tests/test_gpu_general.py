"""GPU: the general-geometry 2D path (csrc/gen2d.cuh via dg_g2_*) against
the reference's own outputs on curved iso-parametric meshes (warped k_geo=2
box; the cylinder mesh with k_geo = 4 and flipped faces; a graded periodic
box): mass and exact inverse mass (scalar and vector), the SIP pressure
Laplacian (tau_scale 1 and 2.5, pressure-Dirichlet sides included) and its
exact diagonal, through the reference-named operator entry points."""

import numpy as np
import pytest

from tests.general_setups import CASES, kinds, load, mesh, relerr

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1607_01323_b200 import operators as ops  # noqa: E402
from paper_1607_01323_b200 import solvers as sol  # noqa: E402
from paper_1607_01323_b200.general import GeneralSpace2D  # noqa: E402

TOL = 1e-12


def setup(name, k):
    Z = load()
    m = mesh(Z, name)
    space = GeneralSpace2D(m, k)
    spec = ops.BoundarySpec({t: (ops.DirichletBC(None) if v == "D" else ops.NeumannBC(None, None))
                             for t, v in kinds(Z, name).items()})
    return Z, space, spec.resolve(space)


@pytest.mark.parametrize("name,k", [(n, k) for n, ks in CASES.items() for k in ks])
def test_general_operators_match_reference(name, k):
    Z, space, bcs = setup(name, k)
    key = f"{name}_k{k}"
    p, u = Z[key + "_p"], Z[key + "_u"]
    assert relerr(ops.mass_apply(space, p), Z[key + "_mass_p"]) < TOL
    assert relerr(ops.mass_apply(space, u), Z[key + "_mass_u"]) < TOL
    assert relerr(ops.inverse_mass_apply(space, p), Z[key + "_imass_p"]) < TOL
    assert relerr(ops.inverse_mass_apply(space, u), Z[key + "_imass_u"]) < TOL
    assert relerr(ops.apply_pressure_laplace(space, p, bcs), Z[key + "_lap"]) < TOL
    assert relerr(ops.apply_pressure_laplace(space, p, bcs, 2.5), Z[key + "_lap25"]) < TOL
    assert relerr(ops.laplace_diagonal(space, bcs, like=p), Z[key + "_diag"]) < TOL


def test_general_device_tensors_and_solver():
    """Element-major CUDA tensors in and out; the Laplacian is symmetric and
    a Jacobi-PCG solve through the reference-form pcg converges."""
    Z, space, bcs = setup("cylinder", 3)
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.rand(space.n_dofs, dtype=torch.float64, device="cuda", generator=g)
    y = torch.rand(space.n_dofs, dtype=torch.float64, device="cuda", generator=g)
    Lx = ops.apply_pressure_laplace(space, x, bcs)
    Ly = ops.apply_pressure_laplace(space, y, bcs)
    assert Lx.is_cuda and Lx.shape == x.shape
    assert abs(float(y @ Lx - x @ Ly)) < 1e-11 * float(x.norm() * Ly.norm())
    diag = ops.laplace_diagonal(space, bcs)
    b = ops.mass_apply(space, y)
    xs, st = sol.pcg(lambda v: ops.apply_pressure_laplace(space, v, bcs), lambda r: r / diag, b,
                     rel_tol=1e-10, max_iter=2000)
    assert st.converged
    r = b - ops.apply_pressure_laplace(space, xs, bcs)
    assert float(r.norm()) < 1e-8 * float(b.norm())
    assert relerr(ops.inverse_mass_apply(space, ops.mass_apply(space, y)).cpu(), y.cpu()) < 1e-12


def g_data(x, t):
    return np.stack([np.sin(2.0 * x[0] + t) * np.cos(x[1]), 0.3 * np.cos(x[0] - 2.0 * t) + x[1]])


def force(x, t):
    return np.stack([0.2 + np.cos(x[1]) * np.sin(t), x[0] * x[1] - 0.1])


@pytest.mark.parametrize("name,k", [(n, k) for n, ks in CASES.items() for k in ks])
def test_general_vector_operators_match_reference(name, k):
    Z, space, bcs = setup(name, k)
    key = f"{name}_k{k}"
    p, u, u2 = Z[key + "_p"], Z[key + "_u"], Z[key + "_u2"]
    assert relerr(ops.apply_viscous_helmholtz(space, u, 3.0, 0.7, bcs), Z[key + "_helm"]) < TOL
    assert relerr(ops.apply_viscous_helmholtz(space, u, 3.0, 0.0, bcs), Z[key + "_helm0"]) < TOL
    td, tc = Z[key + "_tau_d"], Z[key + "_tau_c"]
    assert relerr(ops.apply_projection_operator(space, u, td, tc), Z[key + "_proj"]) < TOL
    assert relerr(ops.apply_projection_operator(space, u, td, None), Z[key + "_projD"]) < TOL
    assert relerr(ops.apply_projection_operator(space, u, None, tc), Z[key + "_projC"]) < TOL
    for form in ("standard", "weak", "strong"):
        assert relerr(ops.eval_divergence_rhs(space, u, bcs, 1.7, form),
                      Z[key + f"_div_{form}"]) < TOL, form
    for form in ("standard", "weak"):
        assert relerr(ops.eval_pressure_gradient_rhs(space, p, bcs, 0.9, form),
                      Z[key + f"_grad_{form}"]) < TOL, form
    assert relerr(ops.compute_vorticity(space, u), Z[key + "_vort"]) < TOL
    assert relerr(ops.eval_convective_rhs(space, bcs, [u], (1.0,), (0.0,), 0.0),
                  Z[key + "_conv1"]) < TOL
    spec_g = ops.BoundarySpec({t: (ops.DirichletBC(g_data) if v == "D" else ops.NeumannBC(None, None))
                               for t, v in kinds(Z, name).items()})
    bcs_g = spec_g.resolve(space)
    got = ops.eval_convective_rhs(space, bcs_g, [u, u2], (2.0, -1.0), (0.3, 0.2), 0.4,
                                  body_force=force)
    assert relerr(got, Z[key + "_conv2"]) < TOL


def dg_data(x, t):
    return np.stack([np.cos(2.0 * x[0] + t) * np.cos(x[1]), 0.6 * np.sin(x[0] - 2.0 * t)])


def h_data(x, t):
    return np.stack([0.4 * x[1] + np.sin(t), np.cos(3.0 * x[0]) * x[1]])


def gp_data(x, t):
    return 0.5 + np.sin(x[0] + 2.0 * x[1] + t)


@pytest.mark.parametrize("name,k", [(n, k) for n, ks in CASES.items() for k in ks])
def test_general_boundary_data_rhs_match_reference(name, k):
    Z, space, _ = setup(name, k)
    key = f"{name}_k{k}"
    spec = ops.BoundarySpec({t: (ops.DirichletBC(g_data, dg_data) if v == "D"
                                 else ops.NeumannBC(h_data, gp_data))
                             for t, v in kinds(Z, name).items()})
    bcs = spec.resolve(space)
    u, u2, w1, w2 = Z[key + "_u"], Z[key + "_u2"], Z[key + "_w1"], Z[key + "_w2"]
    assert relerr(ops.gp_dirichlet_rhs(space, bcs, 0.35, tau_scale=1.7), Z[key + "_gp"]) < TOL
    assert relerr(ops.viscous_rhs_bc(space, bcs, 0.35, 0.03), Z[key + "_vbc"]) < TOL
    got = ops.eval_pressure_neumann_rhs(space, bcs, [u, u2], [w1, w2], (2.0, -1.0), 0.03, 0.45,
                                        body_force=force)
    assert relerr(got, Z[key + "_pn"]) < TOL


@pytest.mark.parametrize("name,k", [(n, k) for n, ks in CASES.items() for k in ks])
def test_general_projections_and_penalties_match_reference(name, k):
    Z, space, _ = setup(name, k)
    key = f"{name}_k{k}"
    p, u = Z[key + "_p"], Z[key + "_u"]
    assert relerr(sol.zero_mean_project(space, p), Z[key + "_zm"]) < TOL
    assert relerr(sol.zero_mean_project_dual(space, p), Z[key + "_zmd"]) < TOL
    td, tc = ops.compute_penalty_parameters(space, torch.as_tensor(
        space.to_element_major(u, 2).ravel()).cuda(), 1e-3, 0.8, ops.VariantConfig("V4", 1.3, 0.7))
    assert relerr(td.cpu().numpy(), Z[key + "_pen_d"]) < TOL
    f = space.mesh.interior
    assert relerr(tc.cpu().numpy()[f.em, f.sm], Z[key + "_pen_c"]) < TOL
    assert relerr(tc.cpu().numpy()[f.ep, f.sp], Z[key + "_pen_c"]) < TOL


@pytest.mark.parametrize("mname", ["mgcyl", "mgcylN"])
def test_general_multigrid_matches_reference(mname):
    """Refined cylinder hierarchy (136 -> 544 curved cells, k = 2): per-level
    Lanczos lambda_max, the coarse Chebyshev count, one V-cycle and the
    MG-preconditioned CG (iterations and residual history) against the
    reference's MultigridHierarchy (multigrid.py:76-175)."""
    from paper_1607_01323_b200.general import GeneralMultigrid
    Z = load()
    k = 2
    spaces = [GeneralSpace2D(mesh(Z, f"{mname}_L{lvl}"), k) for lvl in range(2)]
    spec = ops.BoundarySpec({t: (ops.DirichletBC(None) if v == "D" else ops.NeumannBC(None, None))
                             for t, v in kinds(Z, f"{mname}_L0").items()})
    singular = mname == "mgcylN"
    mg = GeneralMultigrid(spaces, spec, project=sol.zero_mean_project if singular else None)
    lm = np.array([lv["lambda_max"] for lv in mg.levels])
    assert relerr(lm, Z[f"{mname}_lmax"]) < 1e-10
    assert mg.levels[0]["coarse_iters"] == int(Z[f"{mname}_coarse_iters"])
    top = spaces[-1]
    b = Z[f"{mname}_b"]
    assert relerr(mg.vcycle(b), Z[f"{mname}_vcycle"]) < 1e-9
    bcs = spec.resolve(top)
    bt = torch.as_tensor(top.to_element_major(b, 1).ravel()).cuda()
    if singular:
        op = lambda x: sol.zero_mean_project_dual(top, ops.apply_pressure_laplace(top, x, bcs))
    else:
        op = lambda x: ops.apply_pressure_laplace(top, x, bcs)
    x, st = sol.pcg(op, mg.vcycle, bt, rel_tol=1e-8, max_iter=100)
    assert st.iterations == int(Z[f"{mname}_pcg_iters"])
    hw = Z[f"{mname}_pcg_hist"][:st.iterations + 1]
    assert np.allclose(np.asarray(st.history), hw, rtol=1e-8, atol=0)
    assert relerr(top.from_element_major(x.cpu().numpy(), 1), Z[f"{mname}_pcg_x"]) < 1e-7


@pytest.mark.parametrize("name,k", [(n, k) for n, ks in CASES.items() for k in ks])
def test_general_node_coords_and_interpolate(name, k):
    Z, space, _ = setup(name, k)
    key = f"{name}_k{k}"
    assert relerr(space.node_coords(), Z[key + "_xn"]) < 1e-14
    f = space.interpolate(lambda x, t: np.stack([x[0] + t, x[0] * x[1]]), 0.5, 2)
    assert f.shape == (2,) + Z[key + "_xn"].shape[1:]
