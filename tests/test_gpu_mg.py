"""GPU parity of the geometric multigrid V-cycle (reference
pkg/src/dgins/multigrid.py) -- transfers, hierarchy constants, V-cycle and
MG-preconditioned PCG against the real reference in 2D (golden vectors
tests/golden/ref2d_mg.npz) and against the oracle in 3D."""

import os

import numpy as np
import pytest

from tests.golden_setups import relerr

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1607_01323_b200 import multigrid as MG  # noqa: E402
from paper_1607_01323_b200 import operators as ops  # noqa: E402
from paper_1607_01323_b200 import solvers as sol  # noqa: E402
from paper_1607_01323_b200.spaces import DgSpace  # noqa: E402
from oracle import dg_oracle as O  # noqa: E402
from oracle import multigrid as OMG  # noqa: E402

ZM = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref2d_mg.npz"))
CASES = {"per_l2_k3": (2, 3, True), "per_l3_k3": (3, 3, True), "per_l2_k5": (2, 5, True),
         "mix_l3_k3": (3, 3, False), "mix_l0_k2": (0, 2, False)}


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64).ravel(), device="cuda")


def host(t):
    return t.detach().cpu().numpy().ravel()


def gpu_spaces(levels, k, periodic, dim=2):
    meshes = MG.box_mesh_hierarchy(((0, 1),) * dim, (2,) * dim, levels, periodic=(periodic,) * dim)
    return [DgSpace(m, k) for m in meshes]


def gpu_spec(periodic, dim=2):
    if periodic:
        return ops.BoundarySpec({})
    kinds = {"xmin": ops.DirichletBC(None), "xmax": ops.NeumannBC(None, None),
             "ymin": ops.DirichletBC(None), "ymax": ops.DirichletBC(None)}
    if dim == 3:
        kinds.update({"zmin": ops.DirichletBC(None), "zmax": ops.NeumannBC(None, None)})
    return ops.BoundarySpec(kinds)


def test_transfer_golden():
    sp = gpu_spaces(1, 3, False)
    tr = MG.Transfer(sp[0], sp[1])
    assert relerr(host(tr.prolong(dev(ZM["tr_xc"]))), ZM["tr_prolong"]) < 1e-13
    assert relerr(host(tr.restrict(dev(ZM["tr_yf"]))), ZM["tr_restrict"]) < 1e-13
    # accumulate mode
    base = dev(np.ones(sp[1].n_dofs))
    tr.prolong(dev(ZM["tr_xc"]), out=base, add=True)
    assert relerr(host(base) - 1.0, ZM["tr_prolong"]) < 1e-13


@pytest.mark.parametrize("name", list(CASES))
def test_hierarchy_vcycle_pcg_golden(name):
    levels, k, periodic = CASES[name]
    spaces = gpu_spaces(levels, k, periodic)
    proj = sol.zero_mean_project if periodic else None
    mg = MG.MultigridHierarchy(spaces, gpu_spec(periodic), project=proj)
    lmax = np.array([lv.lambda_max for lv in mg.levels])
    np.testing.assert_allclose(lmax, ZM[f"{name}_lmax"], rtol=1e-10)
    assert mg.levels[0].coarse_iters == int(ZM[f"{name}_coarse_iters"])
    x = mg.vcycle(dev(ZM[f"{name}_vb"]))
    assert relerr(host(x), ZM[f"{name}_vx"]) < 1e-9
    if levels == 0:
        return
    space = spaces[-1]
    bcs = gpu_spec(periodic).resolve(space)
    b = dev(ZM[f"{name}_b"])
    # generic device pcg with the V-cycle callable (the reference call form)
    if periodic:
        op = lambda p: sol.zero_mean_project_dual(space, ops.apply_pressure_laplace(space, p, bcs))
    else:
        op = lambda p: ops.apply_pressure_laplace(space, p, bcs)
    hist = []

    def prec(r):
        z = mg.vcycle(r)
        hist.append(float(np.sqrt(max(float((r * z).sum()), 0.0))))
        return z
    xg, st = sol.pcg(op, prec, b, rel_tol=1e-8, max_iter=40)
    assert st.converged and st.iterations == int(ZM[f"{name}_iters"])
    np.testing.assert_allclose(hist, ZM[f"{name}_hist"], rtol=1e-7)
    assert relerr(host(xg), ZM[f"{name}_x"]) < 1e-7
    # fused device MG-PCG
    xf, st2 = MG.laplace_pcg_mg(mg, b, project_dual=periodic, rel_tol=1e-8, max_iter=40)
    assert st2.converged and st2.iterations == int(ZM[f"{name}_iters"])
    np.testing.assert_allclose(st2.history, ZM[f"{name}_hist"], rtol=1e-7)
    assert relerr(host(xf), ZM[f"{name}_x"]) < 1e-7


@pytest.mark.parametrize("k", [2, 3, 4])
def test_3d_vcycle_vs_oracle(k):
    levels = 2
    spaces = gpu_spaces(levels, k, False, dim=3)
    mg = MG.MultigridHierarchy(spaces, gpu_spec(False, dim=3))
    ospaces = [O.DgSpace(m, k) for m in OMG.box_mesh_hierarchy(((0, 1),) * 3, (2, 2, 2), levels,
                                                              periodic=(False,) * 3)]
    okinds = {"xmin": O.zero_dirichlet(3), "xmax": O.zero_neumann(3), "ymin": O.zero_dirichlet(3),
              "ymax": O.zero_dirichlet(3), "zmin": O.zero_dirichlet(3), "zmax": O.zero_neumann(3)}
    omg = OMG.MultigridHierarchy(ospaces, O.BoundarySpec(okinds))
    np.testing.assert_allclose([lv.lambda_max for lv in mg.levels],
                               [lv.cheb.lambda_max for lv in omg.levels], rtol=1e-10)
    assert mg.levels[0].coarse_iters == omg.levels[0].coarse_iters
    rng = np.random.default_rng(k)
    b = rng.standard_normal(ospaces[-1].field_shape())
    assert relerr(host(mg.vcycle(dev(b))), omg.vcycle(b).ravel()) < 1e-9
    # linearity (pkg/tests/test_solvers_multigrid.py:241-251)
    b2 = rng.standard_normal(ospaces[-1].field_shape())
    lhs = host(mg.vcycle(dev(0.7 * b - 1.9 * b2)))
    rhs = 0.7 * host(mg.vcycle(dev(b))) - 1.9 * host(mg.vcycle(dev(b2)))
    assert np.linalg.norm(lhs - rhs) <= 1e-12 * max(np.linalg.norm(rhs), 1.0)
    x, st = MG.laplace_pcg_mg(mg, dev(b), rel_tol=1e-8, max_iter=40)
    assert st.converged and st.iterations <= 15


@pytest.mark.parametrize("k,singular", [(2, True), (3, False), (4, True), (5, False)])
def test_fp32_vcycle(k, singular):
    """The fp32 V-cycle (dg_mg_set_precision): one cycle
    agrees with the fp64 cycle to single-precision accuracy, and the fp64
    MG-PCG it preconditions reaches the same solution (rel_tol 1e-10) in at
    most two more iterations."""
    meshes = MG.box_mesh_hierarchy(((0, 1), (0, 2), (0, 1)), (2, 2, 2), 2, grading=(0.0, 1.2, 0.0),
                                   periodic=(True, False, True))
    spaces = [DgSpace(m, k) for m in meshes]
    spec = ops.BoundarySpec({"ymin": ops.DirichletBC(None),
                             "ymax": ops.DirichletBC(None) if singular else ops.NeumannBC(None, None)})
    proj = sol.zero_mean_project if singular else None
    mg64 = MG.MultigridHierarchy(spaces, spec, project=proj)
    mg32 = MG.MultigridHierarchy(spaces, spec, project=proj, precision="fp32")
    top = spaces[-1]
    g = torch.Generator(device="cuda").manual_seed(k)
    b = torch.rand(top.n_dofs, dtype=torch.float64, device="cuda", generator=g) - 0.5
    if singular:
        b = sol.zero_mean_project_dual(top, b)
    v64, v32 = mg64.vcycle(b), mg32.vcycle(b)
    assert relerr(v32.cpu().numpy(), v64.cpu().numpy()) < 1e-4
    x64, s64 = MG.laplace_pcg_mg(mg64, b, project_dual=singular, rel_tol=1e-10)
    x32, s32 = MG.laplace_pcg_mg(mg32, b, project_dual=singular, rel_tol=1e-10)
    assert s64.converged and s32.converged
    assert s32.iterations <= s64.iterations + 2
    if singular:
        x64, x32 = sol.zero_mean_project(top, x64), sol.zero_mean_project(top, x32)
    assert relerr(x32.cpu().numpy(), x64.cpu().numpy()) < 1e-8
    mg32_back = MG.MultigridHierarchy(spaces, spec, project=proj, precision="fp32")
    from paper_1607_01323_b200 import _lib
    _lib.call("dg_mg_set_precision", mg32_back.handle, 64)
    assert torch.equal(mg32_back.vcycle(b), v64)
