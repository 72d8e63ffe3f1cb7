"""Golden solve for BASELINE config 2, generated with the 3D oracle.

    PYTHONPATH=. python tests/golden/make_golden_c2.py [cells]

Config 2 (BASELINE.json configs[1]): unit cube, 32^3
Cartesian cells, periodic in x and z, velocity-Dirichlet walls in y (pure
Neumann Poisson problem), Q4.  Right-hand side b = zero_mean_project_dual(
M f) with f = sin(2 pi x) cos(pi y) sin(2 pi z) + 1e-3 standard_normal(seed
1) at the GLL nodes (element-major draw) -- the same construction bench.py
uses.  Operator: zero_mean_project_dual o L (reference pattern
pkg/tests/test_solvers_multigrid.py:264-288).  Preconditioner: Chebyshev
degree 5, smoothing range 20, over the exact Jacobi diagonal, lambda_max =
1.1 x the 20-step CG-Lanczos estimate on a projected default_rng(987)
standard-normal seed (pkg/src/dgins/multigrid.py:100-114).  Solver: the
reference pcg (pkg/src/dgins/solvers.py:30-73), rel_tol 1e-10 on the
preconditioned norm sqrt(r.z).

Stored (tests/golden/c2_<cells>.npz): iteration count, the full sqrt(r.z)
history, lambda_max, the diagonal's and the solution's norms, and the
solution sampled at 4096 seeded indices (the full 4.1M-DoF vector would be
33 MB).  The oracle is pinned to the real 2D reference by
tests/test_oracle_golden.py and to dense 3D assembly by
tests/test_oracle3d.py; this script only runs it.  Runtime at 32^3: about
30 minutes on 8 cores.
"""

import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import dg_oracle as O  # noqa: E402


def c2_problem(cells):
    ext = ((0, 1),) * 3
    om = O.build_box_mesh(ext, (cells,) * 3, periodic=(True, False, True))
    osp = O.DgSpace(om, 4)
    obcs = O.BoundarySpec({"ymin": O.zero_dirichlet(3),
                           "ymax": O.zero_dirichlet(3)}).resolve(osp)
    xn = osp.node_coords()
    f = np.sin(2 * np.pi * xn[0]) * np.cos(np.pi * xn[1]) * np.sin(2 * np.pi * xn[2])
    f = f + 1e-3 * np.random.default_rng(1).standard_normal(f.shape)
    b = O.zero_mean_project_dual(osp, O.mass_apply(osp, f))
    return osp, obcs, b


def solve_c2(cells, log=None):
    osp, obcs, b = c2_problem(cells)
    L = lambda v: O.apply_pressure_laplace(osp, v, obcs)
    t0 = time.time()
    diag = O.laplace_diagonal(osp, obcs)
    if log:
        log(f"diag {time.time() - t0:.1f}s")
    cfg = O.chebyshev_from_lanczos(osp, L, diag, project=O.zero_mean_project)
    if log:
        log(f"lambda_max {cfg.lambda_max!r} {time.time() - t0:.1f}s")
    op = lambda v: O.zero_mean_project_dual(osp, L(v))
    prec = lambda r: O.chebyshev_smooth(L, diag, cfg, r)
    x, st = O.pcg(op, prec, b, rel_tol=1e-10, max_iter=5000)
    if log:
        log(f"pcg {st.iterations} its converged={st.converged} {time.time() - t0:.1f}s")
    return dict(b=b, diag=diag, lmax=cfg.lambda_max, x=x, stats=st)


def sample_index(n):
    return np.sort(np.random.default_rng(2024).choice(n, size=min(n, 4096), replace=False))


def main():
    cells = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    r = solve_c2(cells, log=lambda s: print(s, flush=True))
    x = r["x"].ravel()
    idx = sample_index(x.size)
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"c2_{cells}.npz")
    np.savez_compressed(out, iterations=r["stats"].iterations,
                        converged=r["stats"].converged,
                        history=np.array(r["stats"].history), lmax=r["lmax"],
                        b_norm=np.linalg.norm(r["b"]), diag_norm=np.linalg.norm(r["diag"]),
                        x_norm=np.linalg.norm(x), x_idx=idx, x_sample=x[idx])
    print("wrote", out)


if __name__ == "__main__":
    main()
