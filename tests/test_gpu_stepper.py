"""GPU parity of the dual-splitting time step (paper_1607_01323_b200/stepper.py)
against its CPU restatement (oracle/stepper.py): two BDF2 steps on small 3D
channels (graded walls, periodic x/z, BASELINE config-4 shape scaled down)
and on a box with an outflow boundary, non-zero Dirichlet data and a body
force.  Per-substep fields (u^, p, u^^, u, vorticity) and solver iteration
counts are compared."""

import numpy as np
import pytest

from tests.golden_setups import relerr

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1607_01323_b200 import multigrid as MG  # noqa: E402
from paper_1607_01323_b200 import operators as ops  # noqa: E402
from paper_1607_01323_b200 import stepper as S  # noqa: E402
from paper_1607_01323_b200.spaces import DgSpace  # noqa: E402
from oracle import dg_oracle as O  # noqa: E402
from oracle import multigrid as OMG  # noqa: E402
from oracle import stepper as OS  # noqa: E402


def g_in(x, t):   # inflow profile on xmin (velocity-Dirichlet data)
    return np.stack([(1 - x[1] ** 2) * (1 + 0.1 * np.sin(t)), 0.05 * x[2] + 0 * x[1], 0 * x[1]])


def dg_in(x, t):
    return np.stack([(1 - x[1] ** 2) * 0.1 * np.cos(t), 0 * x[1], 0 * x[1]])


def force(x, t):
    return np.stack([0.02 + 0 * x[0], 0.01 * np.sin(x[0]), 0 * x[2]])


CASES = {
    # name: (extents, base counts, levels, grading, periodic, kinds, k)
    "channel": (((0, 2 * np.pi), (-1, 1), (0, np.pi)), (2, 1, 1), 1, (0.0, 1.8, 0.0),
                (True, False, True), {"ymin": "W", "ymax": "W"}, 2),
    "channel_k3": (((0, 2 * np.pi), (-1, 1), (0, np.pi)), (2, 1, 1), 1, (0.0, 1.8, 0.0),
                   (True, False, True), {"ymin": "W", "ymax": "W"}, 3),
    "outflow": (((0, 2), (-1, 1), (0, 1)), (2, 1, 1), 1, (0.0, 0.0, 0.0),
                (False, False, True),
                {"xmin": "I", "xmax": "O", "ymin": "W", "ymax": "W"}, 2),
}


def setups(name):
    ext, base, levels, grading, per, kinds, k = CASES[name]
    om = OMG.box_mesh_hierarchy(ext, base, levels, grading=grading, periodic=per)
    gm = MG.box_mesh_hierarchy(ext, base, levels, grading=grading, periodic=per)
    osp = [O.DgSpace(m, k) for m in om]
    gsp = [DgSpace(m, k) for m in gm]

    def okind(v):
        if v == "W":
            return O.zero_dirichlet(3)
        if v == "I":
            return O.DirichletBC(g_in, dg_in)
        return O.zero_neumann(3)

    def gkind(v):
        if v == "W":
            return ops.DirichletBC(None)
        if v == "I":
            return ops.DirichletBC(g_in, dg_in)
        return ops.NeumannBC(None, None)
    ospec = O.BoundarySpec({t: okind(v) for t, v in kinds.items()})
    gspec = ops.BoundarySpec({t: gkind(v) for t, v in kinds.items()})
    return osp, ospec, gsp, gspec


def initial(space, seed=3):
    x, y, z = space.node_coords()
    rng = np.random.default_rng(seed)
    u = np.stack([1 - y ** 2, 0 * y, 0 * y]) + 0.1 * rng.uniform(-1, 1, (3,) + y.shape)
    return u


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64).ravel(), device="cuda")


def host(t):
    return t.detach().cpu().numpy().ravel()


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("variant", ["V3c", "V4", "VHW", "V2"])
@pytest.mark.parametrize("fused", [False, True])
def test_two_steps_match_oracle(name, variant, fused):
    osp, ospec, gsp, gspec = setups(name)
    bf = force if name == "outflow" else None
    ocfg = OS.StepConfig(dt=1e-3, nu=1 / 180, variant=OS.Variant(variant), body_force=bf)
    gcfg = S.StepConfig(dt=1e-3, nu=1 / 180, variant=ops.VariantConfig(variant), body_force=bf)
    ovc = OS.VelocityCorrection(osp, ospec, ocfg, seed_draw=lambda rng, sp: rng.standard_normal(
        sp.field_shape()))
    gvc = S.VelocityCorrection(gsp, gspec, gcfg, fused=fused)
    np.testing.assert_allclose([lv.lambda_max for lv in gvc.mg.levels],
                               [lv.cheb.lambda_max for lv in ovc.mg.levels], rtol=1e-10)
    u0 = initial(osp[-1])
    ow = O.compute_vorticity(osp[-1], u0)
    ou, op_, ow_h = [u0, u0], [], [ow, ow]
    gu, gp_, gw_h = [dev(u0), dev(u0)], [], [dev(ow), dev(ow)]
    # the fused path (device MG-PCG on the correction, device vector PCG)
    # keeps the exact counts and the plain path's bar (profiles/r02/step_counts.py)
    tol = 1e-9 if not fused else 1e-10
    for n in range(2):
        t = n * 1e-3
        ro = ovc.step(ou, op_, ow_h, t)
        rg = gvc.step(gu, gp_, gw_h, t)
        assert relerr(host(rg.uhat), ro.uhat.ravel()) < 1e-11, "uhat"
        assert rg.iters["pressure"] == ro.iters["pressure"]
        p_ref = ro.p.ravel()
        assert relerr(host(rg.p), p_ref) < tol, ("p", relerr(host(rg.p), p_ref))
        if variant == "V3c":
            assert abs(rg.iters["projection"] - ro.iters["projection"]) <= 2
        else:
            assert rg.iters["projection"] == ro.iters["projection"]
        assert relerr(host(rg.uhh), ro.uhh.ravel()) < tol, "uhh"
        assert rg.iters["viscous"] == ro.iters["viscous"]
        assert relerr(host(rg.u), ro.u.ravel()) < tol, "u"
        assert relerr(host(rg.w), ro.w.ravel()) < tol * 10, "w"
        ou, op_, ow_h = [ro.u, ou[0]], [ro.p] + op_[:1], [ro.w, ow_h[0]]
        gu, gp_, gw_h = [rg.u, gu[0]], [rg.p] + gp_[:1], [rg.w, gw_h[0]]
