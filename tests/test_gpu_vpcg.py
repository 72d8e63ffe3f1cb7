"""GPU: the device velocity-solve PCG (dg_vector_pcg: fast-path operator,
fused x/r update + exact inverse mass + r.z) against the reference-form
``pcg(op, inverse_mass_apply, b, x0)`` composition (solvers.py:30-73) on
the same device operators: iteration counts equal, residual histories and
solutions to 1e-10 (only the reduction order differs)."""

import numpy as np
import pytest

from tests.golden_setups import relerr

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1607_01323_b200 import mesh as M  # noqa: E402
from paper_1607_01323_b200 import operators as ops  # noqa: E402
from paper_1607_01323_b200 import solvers as sol  # noqa: E402
from paper_1607_01323_b200.spaces import DgSpace  # noqa: E402


def setup(k, kinds):
    mesh = M.build_box_mesh(((0, 2), (-1, 1), (0, 1)), (4, 3, 3), grading=(0.0, 1.5, 0.0),
                            periodic=(True, False, True))
    space = DgSpace(mesh, k)
    spec = {}
    for tag, v in kinds.items():
        spec[tag] = ops.DirichletBC(None) if v == "D" else ops.NeumannBC(None, None)
    return space, ops.BoundarySpec(spec).resolve(space)


def compare(got, want):
    """Iterations equal; histories to 1e-10 while the residual is above 1e-4
    of the initial one (later entries amplify the reduction-order rounding
    of long solves); solutions to 1e-6."""
    (xg, sg), (xw, sw) = got, want
    assert sg.iterations == sw.iterations and sg.converged == sw.converged
    hg, hw = np.asarray(sg.history), np.asarray(sw.history)
    early = hw >= 1e-4 * hw[0]
    assert np.allclose(hg[early], hw[early], rtol=1e-10, atol=0)
    assert relerr(xg.cpu().numpy(), xw.cpu().numpy()) < 1e-6


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("kinds", [{"ymin": "D", "ymax": "D"}, {"ymin": "D", "ymax": "N"}])
def test_helmholtz_pcg(k, kinds):
    space, bcs = setup(k, kinds)
    g = torch.Generator(device="cuda").manual_seed(k)
    b = torch.rand(3 * space.n_dofs, dtype=torch.float64, device="cuda", generator=g) - 0.5
    x0 = torch.rand(3 * space.n_dofs, dtype=torch.float64, device="cuda", generator=g) * 0.1
    for guess in (None, x0):
        want = sol.pcg(lambda v: ops.apply_viscous_helmholtz(space, v, 1500.0, 1 / 180, bcs),
                       lambda r: ops.inverse_mass_apply(space, r), b, x0=guess, rel_tol=1e-10)
        got = sol.helmholtz_pcg(space, bcs, b, 1500.0, 1 / 180, x0=guess, rel_tol=1e-10)
        compare(got, want)


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_projection_pcg(k):
    space, _ = setup(k, {"ymin": "D", "ymax": "D"})
    ne = space.mesh.n_elements
    g = torch.Generator(device="cuda").manual_seed(10 + k)
    b = torch.rand(3 * space.n_dofs, dtype=torch.float64, device="cuda", generator=g) - 0.5
    tau_d = torch.rand(ne, dtype=torch.float64, device="cuda", generator=g) * 0.01
    tau_c = torch.rand(3 * ne, dtype=torch.float64, device="cuda", generator=g) * 0.01
    for td, tc in ((tau_d, tau_c), (tau_d, None), (None, tau_c)):
        want = sol.pcg(lambda w: ops.apply_projection_operator(space, w, td, tc),
                       lambda r: ops.inverse_mass_apply(space, r), b, x0=b, rel_tol=1e-10)
        got = sol.projection_pcg(space, b, td, tc, x0=b, rel_tol=1e-10)
        compare(got, want)


def test_vector_pcg_validation():
    space, bcs = setup(2, {"ymin": "D", "ymax": "D"})
    with pytest.raises(ValueError):
        sol.helmholtz_pcg(space, bcs, torch.zeros(5, dtype=torch.float64, device="cuda"), 1.0, 1.0)
