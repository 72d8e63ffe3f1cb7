"""GPU parity of the vector-valued operators: viscous Helmholtz, projection
(div-div + continuity penalty) and the convective Lax-Friedrichs term.

2D: against golden vectors from the real reference (rel L2 <= 1e-12);
3D: against the numpy oracle; BASELINE config 3 shape (periodic [0,2pi]^3,
Taylor-Green + 1e-2 noise, Q5, both over-integration rules)."""

import numpy as np
import pytest

from tests.golden_setups import KS, SETUPS, load_golden, map_tau_c, oracle_setup, relerr

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1607_01323_b200 import mesh as M  # noqa: E402
from paper_1607_01323_b200 import operators as ops  # noqa: E402
from paper_1607_01323_b200.spaces import DgSpace  # noqa: E402
from oracle import dg_oracle as O  # noqa: E402

Z = load_golden()
TOL = 1e-12


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64).ravel(), device="cuda")


def host(t):
    return t.detach().cpu().numpy().ravel()


def gpu_space(ext, counts, k, per, kinds, grading=None, n_q_over=None):
    mesh = M.build_box_mesh(ext, counts, grading=grading, periodic=per)
    space = DgSpace(mesh, k, n_q_over=n_q_over)
    spec = ops.BoundarySpec({t: (ops.DirichletBC(None) if v == "D" else ops.NeumannBC(None, None))
                             for t, v in kinds.items()})
    return space, spec.resolve(space)


@pytest.mark.parametrize("name", list(SETUPS))
@pytest.mark.parametrize("k", KS)
def test_2d_golden_vector_ops(name, k):
    ext, counts, grading, per, kinds = SETUPS[name]
    space, bcs = gpu_space(ext, counts, k, per, kinds, grading)
    osp, _ = oracle_setup(name, k)
    key = f"{name}_k{k}"
    u = dev(Z[key + "_u"])
    got = ops.apply_viscous_helmholtz(space, u, 3.6, 0.025, bcs)
    assert relerr(host(got), Z[key + "_helm"]) < TOL
    tau_d = Z[key + "_tau_d"]
    tau_c = map_tau_c(osp, Z, key)  # reference faces -> our face order
    em, sm, _, _ = space.interior_faces()
    assert np.array_equal(em, osp.f_em) and np.array_equal(sm, osp.f_sm)
    got = ops.apply_projection_operator(space, u, tau_d, tau_c)
    assert relerr(host(got), Z[key + "_proj"]) < TOL
    got = ops.apply_projection_operator(space, u, tau_d, None)
    assert relerr(host(got), Z[key + "_projD"]) < TOL
    got = ops.eval_convective_rhs(space, bcs, [u], (1.0,), (0.0,), 0.0)
    assert relerr(host(got), Z[key + "_conv1"]) < TOL


CASES = [
    (((0, 1), (0, 1), (0, 1)), (3, 2, 4), (True, True, True), {}, None),
    (((0, 1), (0, 2), (0, 1)), (2, 3, 2), (False, False, False),
     {"xmin": "D", "xmax": "N", "ymin": "D", "ymax": "D", "zmin": "N", "zmax": "D"}, None),
    (((0, 2), (-1, 1), (0, 1)), (3, 4, 2), (True, False, True),
     {"ymin": "D", "ymax": "D"}, (0.0, 1.8, 0.0)),
    # one cell across a periodic axis: every x side is its own neighbour
    (((0, 1), (0, 1), (0, 2)), (1, 3, 2), (True, False, True),
     {"ymin": "D", "ymax": "N"}, (0.0, 0.6, 0.0)),
]


def oracle_space(ext, counts, k, per, kinds, grading=None, n_q_over=None):
    om = O.build_box_mesh(ext, counts, grading=grading, periodic=per)
    osp = O.DgSpace(om, k, n_q_over=n_q_over)
    spec = O.BoundarySpec({t: (O.zero_dirichlet(3) if v == "D" else O.zero_neumann(3))
                           for t, v in kinds.items()})
    return osp, spec.resolve(osp)


@pytest.mark.parametrize("case", range(len(CASES)))
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6, 7])
def test_3d_helmholtz_projection(case, k):
    ext, counts, per, kinds, grading = CASES[case]
    osp, obcs = oracle_space(ext, counts, k, per, kinds, grading)
    gsp, gbcs = gpu_space(ext, counts, k, per, kinds, grading)
    rng = np.random.default_rng(10 * case + k)
    u = rng.standard_normal(osp.field_shape(3))
    for g0, nu in ((3.6, 0.025), (1500.0, 1.0 / 180.0), (4.0, 0.0)):
        want = O.apply_viscous_helmholtz(osp, u, g0, nu, obcs).ravel()
        got = host(ops.apply_viscous_helmholtz(gsp, dev(u), g0, nu, gbcs))
        assert relerr(got, want) < TOL, (g0, nu, relerr(got, want))
    tau_d = np.abs(rng.standard_normal(osp.mesh.n_elements)) * 0.3
    tau_c = np.abs(rng.standard_normal(osp.f_em.size)) * 0.2
    want = O.apply_projection_operator(osp, u, tau_d, tau_c).ravel()
    got = host(ops.apply_projection_operator(gsp, dev(u), tau_d, tau_c))
    assert relerr(got, want) < TOL


@pytest.mark.parametrize("case", range(len(CASES)))
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("literal", [False, True])
def test_3d_convective(case, k, literal):
    ext, counts, per, kinds, grading = CASES[case]
    nq = (3 * (k + 1)) // 2 if literal else None
    osp, obcs = oracle_space(ext, counts, k, per, kinds, grading, nq)
    gsp, gbcs = gpu_space(ext, counts, k, per, kinds, grading, nq)
    rng = np.random.default_rng(100 + 10 * case + k)
    hist = [rng.standard_normal(osp.field_shape(3)) for _ in range(2)]
    want = O.eval_convective_rhs(osp, obcs, hist, (2.0, -1.0), (0.3, 0.2), 0.4).ravel()
    got = host(ops.eval_convective_rhs(gsp, gbcs, [dev(h) for h in hist], (2.0, -1.0),
                                       (0.3, 0.2), 0.4))
    assert relerr(got, want) < TOL


def taylor_green(space_nodes, seed):
    x, y, z = space_nodes
    u = np.stack([np.sin(x) * np.cos(y) * np.cos(z), -np.cos(x) * np.sin(y) * np.cos(z),
                  np.zeros_like(x)])
    return u + 1e-2 * np.random.default_rng(seed).uniform(-1, 1, u.shape)


@pytest.mark.parametrize("literal", [False, True])
def test_config3_shape_vs_oracle(literal):
    """BASELINE config 3 setup at 8^3 cells (oracle-sized): periodic
    [0,2pi]^3, Q5, Taylor-Green + 1e-2 uniform noise (seed 2)."""
    ext = ((0, 2 * np.pi),) * 3
    nq = 9 if literal else None
    osp, obcs = oracle_space(ext, (8, 8, 8), 5, (True,) * 3, {}, None, nq)
    gsp, gbcs = gpu_space(ext, (8, 8, 8), 5, (True,) * 3, {}, None, nq)
    u = taylor_green(osp.node_coords(), 2)
    want = O.eval_convective_rhs(osp, obcs, [u], (1.0,), (0.0,), 0.0).ravel()
    got = host(ops.eval_convective_rhs(gsp, gbcs, [dev(u)], (1.0,), (0.0,), 0.0))
    assert relerr(got, want) < TOL


def test_config3_full_size_properties():
    """32^3 Q5 (21.2M velocity DoFs): zero residual for a constant state
    (pkg/tests/test_operators.py:254-261) and linearity in beta."""
    ext = ((0, 2 * np.pi),) * 3
    gsp, gbcs = gpu_space(ext, (32, 32, 32), 5, (True,) * 3, {})
    n = gsp.n_dofs
    c = torch.cat([torch.full((n,), v, dtype=torch.float64, device="cuda")
                   for v in (0.7, -0.2, 0.4)])
    r = ops.eval_convective_rhs(gsp, gbcs, [c], (1.0,), (0.0,), 0.0)
    assert r.abs().max().item() < 1e-12
    g = torch.Generator(device="cuda").manual_seed(2)
    u = torch.rand(3 * n, dtype=torch.float64, device="cuda", generator=g) - 0.5
    r1 = ops.eval_convective_rhs(gsp, gbcs, [u], (1.0,), (0.0,), 0.0)
    r2 = ops.eval_convective_rhs(gsp, gbcs, [u, u], (1.5, 0.5), (0.0, 0.0), 0.0)
    assert ((r2 - 2.0 * r1).norm() / r1.norm()).item() < 1e-13


@pytest.mark.parametrize("k", [1, 2, 3, 5])
def test_2d_view_routing_matches_per_cell_kernel(k, monkeypatch):
    """2D Cartesian Helmholtz / projection / convective run on the general
    view (gen2d kernels); the per-cell quadrature-point kernel
    (DG_2D_GENERIC=1) gives the same results to rounding."""
    mesh = M.build_box_mesh(((0, 2), (-1, 1)), (5, 4), grading=(0.0, 1.3), periodic=(True, False))
    space = DgSpace(mesh, k)
    bcs = ops.BoundarySpec({"ymin": ops.DirichletBC(None), "ymax": ops.NeumannBC(None, None)}).resolve(space)
    g = torch.Generator(device="cuda").manual_seed(k)
    u = torch.rand(2 * space.n_dofs, dtype=torch.float64, device="cuda", generator=g) - 0.5
    ne = mesh.n_elements
    td = torch.rand(ne, dtype=torch.float64, device="cuda", generator=g)
    tc = torch.rand(2 * ne, dtype=torch.float64, device="cuda", generator=g)
    calls = (lambda: ops.apply_viscous_helmholtz(space, u, 3.0, 0.2, bcs),
             lambda: ops.apply_projection_operator(space, u, td, tc),
             lambda: ops.eval_convective_rhs(space, bcs, [u], (1.0,), (0.0,), 0.0))
    routed = [f().cpu().numpy() for f in calls]
    monkeypatch.setenv("DG_2D_GENERIC", "1")
    generic = [f().cpu().numpy() for f in calls]
    for a, b in zip(routed, generic):
        assert relerr(a, b) < 1e-12
