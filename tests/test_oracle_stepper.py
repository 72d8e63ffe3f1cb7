"""The restated dual-splitting step (oracle/stepper.py) on small 3D channels:
BDF constants (SPEC.md bdf_ex_constants examples), zero state stays zero
(SPEC.md advance_step example), a laminar Poiseuille profile stays steady up
to the solver tolerance, and the step runs through every variant path."""

import numpy as np
import pytest

from oracle import dg_oracle as O
from oracle import multigrid as OMG
from oracle import stepper as S


def test_bdf_constants():
    for J in (1, 2, 3):
        g0, al, be = S.bdf_ex_constants(J)
        assert sum(al) == pytest.approx(g0, abs=1e-14)
        assert sum(be) == pytest.approx(1.0, abs=1e-14)
    assert S.bdf_ex_constants(2) == (1.5, (2.0, -0.5), (2.0, -1.0))
    with pytest.raises(ValueError):
        S.bdf_ex_constants(4)


def channel(k=2, levels=1, base=(2, 1, 1)):
    meshes = OMG.box_mesh_hierarchy(((0, 2 * np.pi), (-1, 1), (0, np.pi)), base, levels,
                                    grading=(0.0, 1.8, 0.0), periodic=(True, False, True))
    spaces = [O.DgSpace(m, k) for m in meshes]
    spec = O.BoundarySpec({"ymin": O.zero_dirichlet(3), "ymax": O.zero_dirichlet(3)})
    return spaces, spec


@pytest.mark.parametrize("variant", ["V3c", "V4", "VHW", "V2"])
def test_zero_state_stays_zero(variant):
    spaces, spec = channel()
    cfg = S.StepConfig(dt=1e-3, nu=1 / 180, variant=S.Variant(variant))
    vc = S.VelocityCorrection(spaces, spec, cfg)
    z = np.zeros(spaces[-1].field_shape(3))
    w = O.compute_vorticity(spaces[-1], z)
    r = vc.step([z, z], [], [w, w], 0.0)
    assert np.abs(r.u).max() == 0.0 and np.abs(r.p).max() == 0.0


@pytest.mark.parametrize("variant", ["V4", "V2"])
def test_poiseuille_is_steady_with_forcing(variant):
    """u = (1 - y^2, 0, 0) with f = (2 nu, 0, 0) is an exact steady solution
    (representable at k = 2); one step keeps it to the solver tolerance."""
    spaces, spec = channel(k=2)
    nu = 1 / 180
    force = lambda x, t: np.stack([np.full(x.shape[1:], 2 * nu), 0 * x[1], 0 * x[2]])
    cfg = S.StepConfig(dt=1e-3, nu=nu, variant=S.Variant(variant), body_force=force,
                       rel_tol_p=1e-12, rel_tol_v=1e-12)
    vc = S.VelocityCorrection(spaces, spec, cfg)
    sp = spaces[-1]
    x, y, zc = sp.node_coords()
    u = np.stack([1 - y ** 2, 0 * y, 0 * y])
    w = O.compute_vorticity(sp, u)
    r = vc.step([u, u], [], [w, w], 0.0)
    assert np.abs(r.u - u).max() < 1e-8
    assert np.abs(r.p - r.p.mean()).max() < 1e-7


def test_v2_same_uhat_pressure_rhs_drops_history_divergence():
    """V2 (Eqs. 26-28): u^ is the same as the standard scheme's; the
    Poisson solve sees div u^_dt only, so on a history with nonzero
    divergence the V2 pressure differs from the VHW one."""
    spaces, spec = channel(k=2)
    sp = spaces[-1]
    rng = np.random.default_rng(3)
    u = rng.standard_normal(sp.field_shape(3))
    w = O.compute_vorticity(sp, u)
    res = {}
    for v in ("VHW", "V2"):
        cfg = S.StepConfig(dt=1e-3, nu=1 / 180, variant=S.Variant(v), rel_tol_p=1e-12)
        res[v] = S.VelocityCorrection(spaces, spec, cfg).step([u, u], [], [w, w], 0.0)
    d = np.abs(res["V2"].uhat - res["VHW"].uhat).max() / np.abs(u).max()
    assert d < 1e-13
    assert np.abs(res["V2"].p - res["VHW"].p).max() > 1e-3 * np.abs(res["VHW"].p).max()
