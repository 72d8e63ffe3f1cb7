"""Gate 2: the 3D restatement is pinned (no 3D reference code exists).

1. Extrusion pin against the REAL reference: a z-periodic 3D mesh built by
   extruding each 2D golden setup, with tau injected from the 2D space, acting
   on a z-constant field (zero z-velocity) must reproduce the reference's
   2D golden output tensored with the z mass row  (S^T w) h_z/2.
2. Sum factorisation == dense naive assembly (oracle/dense.py, restating
   pkg/src/dgins/oracle.py) at 1e-12, the reference's own tolerance
   (pkg/tests/test_operators.py:85-178).
3. Algebraic structure: symmetry, PSD, constant nullspace
   (pkg/tests/test_operators.py:181-250).
"""

import numpy as np
import pytest

from oracle import dg_oracle as O
from oracle.dense import DenseOracle
from tests.golden_setups import (SETUPS, body_force, load_golden, map_tau_c,
                                 oracle_setup, relerr)

Z = load_golden()


def extrude(name, k, nz=2, hz=0.7):
    ext, counts, grading, per, kinds = SETUPS[name]
    mesh = O.build_box_mesh(tuple(ext) + ((0.0, hz),), tuple(counts) + (nz,),
                            grading=tuple(grading) + (0.0,),
                            periodic=tuple(per) + (True,))
    spec = O.BoundarySpec({t: (O.zero_dirichlet(3) if v == "D" else O.zero_neumann(3))
                           for t, v in kinds.items()})
    space = O.DgSpace(mesh, k)
    sp2, _ = oracle_setup(name, k)
    ne2 = sp2.mesh.n_elements
    # inject the 2D penalty: tau_e per column; interior faces by max
    space.tau_e = np.tile(sp2.tau_e, nz)
    space.tau_if = np.maximum(space.tau_e[space.f_em], space.tau_e[space.f_ep])
    return space, spec.resolve(space), sp2, ne2


def zmass_row(b, hz):
    return (b.S.T @ b.rule.weights) * (0.5 * hz)


def lift3(a2, ne2, nz, zrow):
    """(ne2, y, x) 2D data -> (ne2*nz, z, y, x) tensored with zrow."""
    m = len(zrow)
    out = np.empty((nz, ne2, m) + a2.shape[1:])
    for l in range(m):
        out[:, :, l] = zrow[l] * a2[None]
    return out.reshape((nz * ne2, m) + a2.shape[1:])


def const3(a2, nz, m):
    out = np.broadcast_to(a2[None, :, None], (nz,) + a2.shape[:1] + (m,) + a2.shape[1:])
    return np.ascontiguousarray(out).reshape((-1, m) + a2.shape[1:])


@pytest.mark.parametrize("name", list(SETUPS))
@pytest.mark.parametrize("k", (2, 3))
def test_extrusion_matches_reference_2d(name, k):
    nz, hz = 2, 0.7
    space, bcs, sp2, ne2 = extrude(name, k, nz, hz)
    key = f"{name}_k{k}"
    m = k + 1
    zrow = zmass_row(space.basis, hz / nz)
    p2 = Z[key + "_p"].reshape(sp2.field_shape())
    p3 = const3(p2, nz, m)
    got = O.apply_pressure_laplace(space, p3, bcs)
    want = lift3(Z[key + "_lap"].reshape(sp2.field_shape()), ne2, nz, zrow)
    assert relerr(got.ravel(), want.ravel()) < 1e-13
    got = O.apply_pressure_laplace(space, p3, bcs, tau_scale=7.5)
    want = lift3(Z[key + "_lap75"].reshape(sp2.field_shape()), ne2, nz, zrow)
    assert relerr(got.ravel(), want.ravel()) < 1e-13

    u2 = Z[key + "_u"].reshape(sp2.field_shape(2))
    v2 = Z[key + "_u2"].reshape(sp2.field_shape(2))
    u3 = np.stack([const3(u2[0], nz, m), const3(u2[1], nz, m),
                   np.zeros(space.field_shape())])
    v3 = np.stack([const3(v2[0], nz, m), const3(v2[1], nz, m),
                   np.zeros(space.field_shape())])

    def check(suffix, got3, z_zero=True):
        want2 = Z[key + suffix].reshape(sp2.field_shape(2))
        assert relerr(got3[0].ravel(), lift3(want2[0], ne2, nz, zrow).ravel()) < 1e-13
        assert relerr(got3[1].ravel(), lift3(want2[1], ne2, nz, zrow).ravel()) < 1e-13
        if z_zero:   # div-div couples w_z to div(w) even for z-constant w
            assert np.abs(got3[2]).max() < 1e-13 * np.abs(got3[:2]).max()

    check("_mass", O.mass_apply(space, u3))
    check("_helm", O.apply_viscous_helmholtz(space, u3, 3.6, 0.025, bcs))
    tau_d = np.tile(Z[key + "_tau_d"], nz)
    check("_projD", O.apply_projection_operator(space, u3, tau_d, None), False)
    # tau_C: 2D faces replicate per z layer; z faces get an arbitrary value
    tc2 = map_tau_c(sp2, Z, key)
    lut = {(int(e), int(s)): t for e, s, t in zip(sp2.f_em, sp2.f_sm, tc2)}
    tau_c = np.array([lut.get((int(e) % ne2, int(s)), 0.123)
                      for e, s in zip(space.f_em, space.f_sm)])
    check("_proj", O.apply_projection_operator(space, u3, tau_d, tau_c), False)
    # convective on the over-integration rule: z mass row of that rule
    zrow_o = zmass_row(space.basis_over[0], hz / nz)
    got = O.eval_convective_rhs(space, bcs, [u3, v3], (2.0, -1.0), (0.3, 0.2), 0.4,
                                body_force=lambda x, t: np.concatenate(
                                    [body_force(x, t), np.zeros((1,) + x.shape[1:])]))
    want2 = Z[key + "_conv"].reshape(sp2.field_shape(2))
    for c in range(2):
        assert relerr(got[c].ravel(), lift3(want2[c], ne2, nz, zrow_o).ravel()) < 1e-13


def setup3d(kind, k, counts=(2, 2, 2)):
    if kind == "periodic":
        mesh = O.build_box_mesh(((0, 1), (0, 1), (0, 1)), counts,
                                periodic=(True, True, True))
        spec = O.BoundarySpec({})
    elif kind == "walls":
        mesh = O.build_box_mesh(((0, 1), (0, 2), (0, 1)), counts)
        spec = O.BoundarySpec({t: O.zero_dirichlet(3) for t in O.TAG_NAMES})
    elif kind == "mixed":
        mesh = O.build_box_mesh(((0, 1), (-1, 1), (0, 0.5)), counts,
                                grading=(0.0, 1.2, 0.0), periodic=(True, False, False))
        spec = O.BoundarySpec({"ymin": O.zero_dirichlet(3), "ymax": O.zero_neumann(3),
                               "zmin": O.zero_neumann(3), "zmax": O.zero_dirichlet(3)})
    space = O.DgSpace(mesh, k)
    return space, spec.resolve(space)


KINDS3 = ["periodic", "walls", "mixed"]


@pytest.mark.parametrize("kind", KINDS3)
@pytest.mark.parametrize("k", (1, 2, 3))
def test_laplace_sumfact_equals_dense(kind, k, rng):
    space, bcs = setup3d(kind, k)
    dense = DenseOracle(space)
    for ts in (1.0, 7.5):
        L = dense.laplace_matrix(bcs, tau_scale=ts)
        p = rng.standard_normal(space.field_shape())
        got = O.apply_pressure_laplace(space, p, bcs, ts).ravel()
        assert relerr(got, L @ p.ravel()) < 1e-12
        diag = O.laplace_diagonal(space, bcs, ts).ravel()
        assert relerr(diag, np.diag(L)) < 1e-12
    # symmetry / PSD / nullspace
    assert np.abs(L - L.T).max() < 1e-12 * np.abs(L).max()
    assert np.linalg.eigvalsh(0.5 * (L + L.T)).min() > -1e-10 * np.abs(L).max()
    if kind == "periodic":
        one = np.ones(space.field_shape())
        assert np.abs(O.apply_pressure_laplace(space, one, bcs)).max() < 1e-11


@pytest.mark.parametrize("kind", KINDS3)
def test_mass_helmholtz_projection_dense(kind, rng):
    space, bcs = setup3d(kind, 2)
    dense = DenseOracle(space)
    u = rng.standard_normal(space.field_shape(3))
    M = dense.mass_matrix(ncomp=3)
    assert relerr(O.mass_apply(space, u).ravel(), M @ u.ravel()) < 1e-12
    back = O.inverse_mass_apply(space, O.mass_apply(space, u))
    assert relerr(back.ravel(), u.ravel()) < 1e-12
    H = dense.helmholtz_matrix(bcs, 3.6, 0.025)
    got = O.apply_viscous_helmholtz(space, u, 3.6, 0.025, bcs).ravel()
    assert relerr(got, H @ u.ravel()) < 1e-12
    assert np.abs(H - H.T).max() < 1e-12 * np.abs(H).max()
    ne = space.mesh.n_elements
    tau_d = np.abs(rng.standard_normal(ne)) * 0.3
    tau_c = np.abs(rng.standard_normal(space.f_em.size)) * 0.2
    P = dense.projection_matrix(tau_d, tau_c)
    got = O.apply_projection_operator(space, u, tau_d, tau_c).ravel()
    assert relerr(got, P @ u.ravel()) < 1e-12


@pytest.mark.parametrize("kind", KINDS3)
def test_convective_dense(kind, rng):
    space, bcs = setup3d(kind, 2)
    dense = DenseOracle(space)
    hist = [rng.standard_normal(space.field_shape(3)) for _ in range(2)]
    force = lambda x, t: np.stack([np.sin(x[0]) + t, x[1] ** 2, x[2] * x[0]])
    got = O.eval_convective_rhs(space, bcs, hist, (2.0, -1.0), (0.3, 0.2), 0.4,
                                body_force=force).ravel()
    want = dense.convective_residual(bcs, [u.ravel() for u in hist], (2.0, -1.0),
                                     (0.3, 0.2), 0.4, body_force=force)
    assert relerr(got, want) < 1e-12


def test_tau_known_answers_3d():
    """Eq. 18 in 3D for unit cubes, k=3: interior 3*16, one boundary face
    3.5*16, edge 4*16, corner 4.5*16 (2D analogues 32, 40 pinned by
    pkg/tests/test_mesh_geometry.py:171-191)."""
    mesh = O.build_box_mesh(((0, 3), (0, 3), (0, 3)), (3, 3, 3))
    space = O.DgSpace(mesh, 3)
    t = space.tau_e
    assert t[13] == pytest.approx(48.0, rel=1e-12)      # center
    assert t[4] == pytest.approx(56.0, rel=1e-12)       # z-face center
    assert t[1] == pytest.approx(64.0, rel=1e-12)       # edge
    assert t[0] == pytest.approx(72.0, rel=1e-12)       # corner


def test_constant_state_periodic_zero_convective():
    """pkg/tests/test_operators.py:254-261 in 3D."""
    space, bcs = setup3d("periodic", 3)
    u = np.zeros(space.field_shape(3))
    u[0], u[1], u[2] = 0.7, -0.2, 0.4
    out = O.eval_convective_rhs(space, bcs, [u], (1.0,), (0.0,), 0.1)
    assert np.abs(out).max() < 1e-12
