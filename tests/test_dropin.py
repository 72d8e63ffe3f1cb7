"""Drop-in with the reference's own objects: DgSpace(mesh, k) accepts the Mesh
that the reference's build_box_mesh returns (pkg/src/dgins/mesh.py:279-351,
spaces.py:61-81), and the unchanged call sites -- BoundarySpec(kinds)
.resolve(space), apply_pressure_laplace / laplace_diagonal / mass_apply /
inverse_mass_apply / zero_mean_project[_dual] / pcg -- reproduce the
reference's golden outputs.  The meshes are reference-built fixtures
(tests/golden/make_golden_meshes.py), the outputs tests/golden/ref2d.npz."""

import numpy as np
import pytest

from paper_1607_01323_b200.mesh import BoxMesh, box_from_reference, build_box_mesh
from tests.golden_setups import KS, SETUPS, load_golden, reference_mesh, relerr


@pytest.mark.parametrize("name", list(SETUPS))
def test_reference_box_mesh_is_recognised(name):
    ext, counts, grading, per, kinds = SETUPS[name]
    ref = reference_mesh(name)
    box = box_from_reference(ref)
    assert isinstance(box, BoxMesh) and box.source is ref
    assert box.counts == tuple(counts) and box.periodic == tuple(per)
    mine = build_box_mesh(ext, counts, grading=grading, periodic=per)
    for d in range(2):
        np.testing.assert_allclose(box.axis_vertices[d], mine.axis_vertices[d], rtol=0, atol=1e-15)
    assert set(box.boundary_tags()) == set(kinds)


def test_non_affine_reference_mesh_goes_general():
    assert box_from_reference(reference_mesh("kgeo2")) is None


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(SETUPS))
@pytest.mark.parametrize("k", KS)
def test_reference_mesh_through_unchanged_call_sites(name, k):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1607_01323_b200 import operators as ops, solvers as sol
    from paper_1607_01323_b200.spaces import DgSpace
    Z = load_golden()
    ext, counts, grading, per, kinds = SETUPS[name]
    space = DgSpace(reference_mesh(name), k)  # the reference's Mesh object
    assert isinstance(space, DgSpace)
    spec = ops.BoundarySpec({t: (ops.DirichletBC(None) if v == "D" else ops.NeumannBC(None, None))
                             for t, v in kinds.items()})
    bcs = spec.resolve(space)
    key = f"{name}_k{k}"
    np.testing.assert_allclose(space.ctx(bcs.kinds).tau(), Z[key + "_tau_e"], rtol=1e-13)
    dev = lambda a: torch.as_tensor(np.ascontiguousarray(a, np.float64).ravel(), device="cuda")
    host = lambda t: t.detach().cpu().numpy().ravel()
    p, u = dev(Z[key + "_p"]), dev(Z[key + "_u"])
    checks = {
        "_lap": ops.apply_pressure_laplace(space, p, bcs),
        "_lap75": ops.apply_pressure_laplace(space, p, bcs, tau_scale=7.5),
        "_diag": ops.laplace_diagonal(space, bcs),
        "_mass": ops.mass_apply(space, u),
        "_invmass": ops.inverse_mass_apply(space, u),
        "_zm": sol.zero_mean_project(space, p),
        "_zmd": sol.zero_mean_project_dual(space, p),
    }
    for suffix, got in checks.items():
        assert relerr(host(got), Z[key + suffix]) < 1e-12, suffix


@pytest.mark.gpu
def test_straight_kgeo2_reference_mesh_runs_general_path():
    """A reference mesh the Cartesian context cannot take (iso-parametric
    k_geo = 2, here still a straight box) gets the general-geometry space;
    on this straight box its Laplacian equals the Cartesian one."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1607_01323_b200 import operators as ops
    from paper_1607_01323_b200.general import GeneralSpace2D
    from paper_1607_01323_b200.spaces import DgSpace
    sp = DgSpace(reference_mesh("kgeo2"), 3)
    assert isinstance(sp, GeneralSpace2D)
    box = DgSpace(build_box_mesh(((0, 1), (0, 1)), (3, 2)), 3)
    kinds = {t: ops.DirichletBC(None) for t in ("xmin", "xmax", "ymin", "ymax")}
    p = torch.rand(box.n_dofs, dtype=torch.float64, device="cuda")
    a = ops.apply_pressure_laplace(sp, p, ops.BoundarySpec(kinds).resolve(sp))
    b = ops.apply_pressure_laplace(box, p, ops.BoundarySpec(kinds).resolve(box))
    assert relerr(a.reshape(-1).cpu().numpy(), b.reshape(-1).cpu().numpy()) < 1e-12
