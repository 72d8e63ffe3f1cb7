"""BASELINE config 2 in 3D: the fused Chebyshev(5,20)-Jacobi PCG against the
oracle's pcg (restated pkg/src/dgins/solvers.py:30-129): identical iteration
count and sqrt(r.z) history to 1e-10.

* 8^3 cells: the oracle solve runs inside the test (about 8 s on the host).
* 32^3 cells (the BASELINE size, 4.1M DoFs): against tests/golden/c2_32.npz,
  written by tests/golden/make_golden_c2.py (oracle run, ~30 min).
"""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1607_01323_b200 import mesh as M  # noqa: E402
from paper_1607_01323_b200 import operators as ops  # noqa: E402
from paper_1607_01323_b200 import solvers as sol  # noqa: E402
from paper_1607_01323_b200.spaces import DgSpace  # noqa: E402
from tests.golden.make_golden_c2 import c2_problem, sample_index, solve_c2  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def gpu_c2(cells):
    mesh = M.build_box_mesh(((0, 1),) * 3, (cells,) * 3, periodic=(True, False, True))
    space = DgSpace(mesh, 4)
    bcs = ops.BoundarySpec({"ymin": ops.DirichletBC(None),
                            "ymax": ops.DirichletBC(None)}).resolve(space)
    xn = space.node_coords()
    f = np.sin(2 * np.pi * xn[0]) * np.cos(np.pi * xn[1]) * np.sin(2 * np.pi * xn[2])
    f = f + 1e-3 * np.random.default_rng(1).standard_normal(f.shape)
    b = sol.zero_mean_project_dual(space, ops.mass_apply(
        space, torch.as_tensor(np.ascontiguousarray(f).ravel(), device="cuda")))
    diag = ops.laplace_diagonal(space, bcs)
    lmax = sol.lanczos_lambda_max(space, bcs, diag, project=True)
    cfg = sol.ChebyshevConfig(5, 20.0, lmax)
    x, st = sol.laplace_pcg(space, bcs, b, project_dual=True, cheb=cfg, diag=diag,
                            rel_tol=1e-10, max_iter=5000)
    return dict(b=b, diag=diag, lmax=lmax, x=x, stats=st)


def check(got, iterations, history, lmax, x_idx, x_sample, b_norm, diag_norm):
    assert abs(got["lmax"] - lmax) <= 1e-10 * lmax
    assert abs(got["b"].norm().item() - b_norm) <= 1e-12 * b_norm
    assert abs(got["diag"].norm().item() - diag_norm) <= 1e-12 * diag_norm
    st = got["stats"]
    assert st.converged
    assert st.iterations == iterations, (st.iterations, iterations)
    np.testing.assert_allclose(np.array(st.history), history, rtol=1e-10, atol=1e-13 * history[0])
    x = got["x"].reshape(-1).cpu().numpy()
    np.testing.assert_allclose(x[x_idx], x_sample, rtol=0, atol=1e-9 * np.abs(x_sample).max())


def test_c2_shape_8cubed_matches_oracle():
    want = solve_c2(8)
    x = want["x"].ravel()
    idx = sample_index(x.size)
    check(gpu_c2(8), want["stats"].iterations, np.array(want["stats"].history), want["lmax"],
          idx, x[idx], np.linalg.norm(want["b"]), np.linalg.norm(want["diag"]))


def test_c2_32cubed_matches_golden():
    path = os.path.join(GOLDEN, "c2_32.npz")
    if not os.path.exists(path):
        pytest.fail("tests/golden/c2_32.npz missing: run tests/golden/make_golden_c2.py")
    z = np.load(path)
    check(gpu_c2(32), int(z["iterations"]), z["history"], float(z["lmax"]), z["x_idx"],
          z["x_sample"], float(z["b_norm"]), float(z["diag_norm"]))


def test_c2_golden_rhs_matches_oracle_problem():
    """The right-hand side the GPU test builds is the oracle's (8^3)."""
    _, _, b = c2_problem(8)
    got = gpu_c2_rhs(8)
    assert np.linalg.norm(got - b.ravel()) <= 1e-13 * np.linalg.norm(b)


def gpu_c2_rhs(cells):
    mesh = M.build_box_mesh(((0, 1),) * 3, (cells,) * 3, periodic=(True, False, True))
    space = DgSpace(mesh, 4)
    xn = space.node_coords()
    f = np.sin(2 * np.pi * xn[0]) * np.cos(np.pi * xn[1]) * np.sin(2 * np.pi * xn[2])
    f = f + 1e-3 * np.random.default_rng(1).standard_normal(f.shape)
    b = sol.zero_mean_project_dual(space, ops.mass_apply(
        space, torch.as_tensor(np.ascontiguousarray(f).ravel(), device="cuda")))
    return b.reshape(-1).cpu().numpy()
