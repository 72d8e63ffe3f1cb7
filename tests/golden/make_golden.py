"""Generate golden vectors by running the REAL reference (2D ``dgins``).

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The resulting ``tests/golden/ref2d.npz`` is committed; tests on the GPU box
read only the npz (the reference tree does not travel).  All vectors are
stored in element-major order (component, element, y-node, x-node), the
reference's own serialisation (pkg/src/dgins/spaces.py:49-58).

Setups mirror the reference test-suite's ``make_setup`` (pkg/tests/
test_operators.py:34-52: "periodic" and "mixed"; the "curved" case needs
general geometry, out of scope) plus one extra graded case with the other
assignment of boundary kinds, and the solver cases of
pkg/tests/test_solvers_multigrid.py (Chebyshev/Jacobi PCG on a pure-Neumann
problem, the 2D analogue of BASELINE config 2).
"""

import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from dgins import operators as ops  # noqa: E402
from dgins import solvers as sol  # noqa: E402
from dgins.basis import get_basis, convective_rule_points  # noqa: E402
from dgins.mesh import build_box_mesh  # noqa: E402
from dgins.spaces import DgSpace, FieldVector  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref2d.npz")


def z2(x, t):
    return np.zeros((2,) + x.shape[1:])


def z1(x, t):
    return np.zeros(x.shape[1:])


def dirichlet_zero():
    return ops.DirichletBC(z2, z2)


def neumann_zero():
    return ops.NeumannBC(z2, z1)


SETUPS = {
    # name: (extents, counts, grading, periodic, kinds per tag)
    "periodic": (((0, 1), (0, 1)), (3, 3), (0.0, 0.0), (True, True), {}),
    "mixed": (((0, 1), (0, 1)), (3, 3), (0.8, 0.0), (False, False),
              {"xmin": "D", "xmax": "N", "ymin": "D", "ymax": "D"}),
    "mixed2": (((0, 2), (-1, 1)), (4, 3), (0.0, 1.1), (True, False),
               {"ymin": "N", "ymax": "D"}),
    "walls": (((0, 1), (0, 1)), (3, 2), (0.0, 0.0), (False, False),
              {"xmin": "N", "xmax": "N", "ymin": "N", "ymax": "D"}),
}


# non-zero boundary data for the once-per-step right-hand sides
# (operators.py:241-259, 494-527, 621-672); the same formulas live in
# tests/golden_setups.py for the consumers of the fixture.
def g_data(x, t):
    return np.stack([np.sin(x[0] + t) * x[1], np.cos(2 * x[1]) - t * x[0]])


def dgdt_data(x, t):
    return np.stack([np.cos(x[0] + t) * x[1], -x[0] + 0 * x[1]])


def h_data(x, t):
    return np.stack([x[0] * x[1] + t, np.sin(3 * x[0]) - x[1]])


def gp_data(x, t):
    return np.cos(x[0] - 2 * x[1]) + t


def make(name, k, data=False):
    ext, counts, grading, per, kinds = SETUPS[name]
    mesh = build_box_mesh(ext, counts, grading=grading, periodic=per)
    if data:
        dbc, nbc = ops.DirichletBC(g_data, dgdt_data), ops.NeumannBC(h_data, gp_data)
    else:
        dbc, nbc = dirichlet_zero(), neumann_zero()
    spec = ops.BoundarySpec({t: (dbc if v == "D" else nbc)
                             for t, v in kinds.items()})
    space = DgSpace(mesh, k)
    return space, spec.resolve(space)


def em(space, a):
    """reference kernel layout -> element-major flat."""
    if a.ndim == 3:
        a = a[None]
    return FieldVector(a, space.k).element_major()


def unem(space, f, ncomp):
    d = FieldVector.from_element_major(f, space, ncomp).data
    return d[0] if ncomp == 1 else d


def body_force(x, t):
    return np.stack([np.sin(x[0]) + t, x[1] ** 2])


def main():
    out = {}
    # 1D tables for k = 1..7 on the linear and convective rules
    for k in range(1, 8):
        for nq in sorted({k + 1, convective_rule_points(k), (3 * (k + 1)) // 2}):
            b = get_basis(k, nq)
            key = f"tab_k{k}_q{nq}"
            out[key + "_S"] = b.S
            out[key + "_D"] = b.D
            out[key + "_nodes"] = b.nodes
            out[key + "_pts"] = b.rule.points
            out[key + "_w"] = b.rule.weights
            out[key + "_ld"] = b.left_deriv
            out[key + "_rd"] = b.right_deriv
    rng = np.random.default_rng(20261019)
    for name in SETUPS:
        for k in (2, 3, 5):
            space, bcs = make(name, k)
            ne = space.mesh.n_elements
            m = k + 1
            key = f"{name}_k{k}"
            out[key + "_tau_e"] = space.tau_e
            out[key + "_h"] = np.array([[np.ptp(space.mesh.corner_coords()[e, :, d])
                                         for d in range(2)] for e in range(ne)])
            p = rng.standard_normal(ne * m * m)
            u = rng.standard_normal(2 * ne * m * m)
            u2 = rng.standard_normal(2 * ne * m * m)
            out[key + "_p"] = p
            out[key + "_u"] = u
            out[key + "_u2"] = u2
            pr = unem(space, p, 1)
            ur = unem(space, u, 2)
            u2r = unem(space, u2, 2)
            out[key + "_lap"] = em(space, ops.apply_pressure_laplace(space, pr, bcs))
            out[key + "_lap75"] = em(space, ops.apply_pressure_laplace(
                space, pr, bcs, tau_scale=7.5))
            out[key + "_diag"] = em(space, ops.laplace_diagonal(space, bcs))
            out[key + "_diag75"] = em(space, ops.laplace_diagonal(space, bcs, 7.5))
            out[key + "_mass"] = em(space, ops.mass_apply(space, ur))
            out[key + "_invmass"] = em(space, ops.inverse_mass_apply(space, ur))
            out[key + "_helm"] = em(space, ops.apply_viscous_helmholtz(
                space, ur, 3.6, 0.025, bcs))
            tau_d = np.abs(rng.standard_normal(ne)) * 0.3
            tau_c = np.abs(rng.standard_normal(space.f_em.shape[0])) * 0.2
            out[key + "_tau_d"] = tau_d
            # tau_c is stored per (minus element, minus slot) so the
            # consumer can map it onto its own face enumeration
            out[key + "_tau_c"] = tau_c
            out[key + "_f_em"] = space.f_em
            out[key + "_f_sm"] = space.f_sm
            out[key + "_f_ep"] = space.f_ep
            out[key + "_f_sp"] = space.f_sp
            out[key + "_proj"] = em(space, ops.apply_projection_operator(
                space, ur, tau_d, tau_c))
            out[key + "_projD"] = em(space, ops.apply_projection_operator(
                space, ur, tau_d, None))
            out[key + "_conv"] = em(space, ops.eval_convective_rhs(
                space, bcs, [ur, u2r], (2.0, -1.0), (0.3, 0.2), 0.4,
                body_force=body_force))
            out[key + "_conv1"] = em(space, ops.eval_convective_rhs(
                space, bcs, [ur], (1.0,), (0.0,), 0.0))
            out[key + "_zm"] = em(space, sol.zero_mean_project(space, pr))
            out[key + "_zmd"] = em(space, sol.zero_mean_project_dual(space, pr))
            # once-per-step right-hand sides (operators.py:241-366, 494-527,
            # 610-672) with non-zero boundary data
            _, bcd = make(name, k, data=True)
            out[key + "_convd"] = em(space, ops.eval_convective_rhs(
                space, bcd, [ur, u2r], (2.0, -1.0), (0.3, 0.2), 0.4,
                body_force=body_force))
            for form in ("standard", "weak", "strong"):
                out[f"{key}_div_{form}"] = em(space, ops.eval_divergence_rhs(
                    space, ur, bcd, 2.5, form))
            for form in ("standard", "weak"):
                out[f"{key}_grad_{form}"] = em(space, ops.eval_pressure_gradient_rhs(
                    space, pr, bcd, 1.7, form))
            w1 = ops.compute_vorticity(space, ur)
            w2 = ops.compute_vorticity(space, u2r)
            out[key + "_vort"] = em(space, w1)
            out[key + "_pn"] = em(space, ops.eval_pressure_neumann_rhs(
                space, bcd, [ur, u2r], [w1, w2], (2.0, -1.0), 0.025, 0.4,
                body_force=body_force))
            out[key + "_pn0"] = em(space, ops.eval_pressure_neumann_rhs(
                space, bcs, [ur], [w1], (1.0,), 0.025, 0.4))
            out[key + "_gp"] = em(space, ops.gp_dirichlet_rhs(space, bcd, 0.3))
            out[key + "_gp75"] = em(space, ops.gp_dirichlet_rhs(space, bcd, 0.3, 7.5))
            out[key + "_vrb"] = em(space, ops.viscous_rhs_bc(space, bcd, 0.3, 0.025))
            # element-local PCG on the block-diagonal projection operator
            # with inverse-mass preconditioning (solvers.py:201-256; the
            # configuration of pkg/tests/test_solvers_multigrid.py:155-195)
            # Per-cell counts of long local solves (k=5: ~40 iterations on
            # 72 unknowns, well past the loss of orthogonality) move by +-2
            # under a change of summation order (measured against a permuted
            # restatement), so the fixture also holds a fixed 5-iteration
            # run ("el5") whose iterate is compared exactly.
            for tag, zeta, rtol, mit in (("el", None, 1e-8, 200), ("elx", 1e6, 1e-8, 200),
                                         ("el12", None, 1e-12, 200),
                                         ("el5", None, 1e-14, 5)):
                td = np.full(ne, zeta) if zeta else tau_d * 10.0
                x, iters, conv = sol.element_local_pcg(
                    lambda w: ops.apply_projection_operator(space, w, td, None),
                    lambda r: ops.inverse_mass_apply(space, r), ur, rel_tol=rtol,
                    max_iter=mit)
                out[f"{key}_{tag}_tau"] = td
                out[f"{key}_{tag}_x"] = em(space, x)
                out[f"{key}_{tag}_iters"] = iters
                out[f"{key}_{tag}_conv"] = conv

    # solver histories (2D analogue of config 2): pure-Neumann periodic-x,
    # wall-y Poisson, Chebyshev(5, 20) over Jacobi with the MG level's
    # Lanczos lambda (multigrid.py:100-114), and plain Jacobi PCG.
    for (k, nx) in ((3, 8), (4, 6)):
        mesh = build_box_mesh(((0, 1), (0, 1)), (nx, nx), periodic=(True, False))
        spec = ops.BoundarySpec({"ymin": dirichlet_zero(), "ymax": dirichlet_zero()})
        space = DgSpace(mesh, k)
        bcs = spec.resolve(space)
        key = f"cg_k{k}_n{nx}"
        L = lambda p: ops.apply_pressure_laplace(space, p, bcs)
        op = lambda p: sol.zero_mean_project_dual(space, L(p))
        diag = ops.laplace_diagonal(space, bcs)
        rng2 = np.random.default_rng(987)
        seed_vec = rng2.standard_normal(diag.shape)   # reference layout draw
        seed_vec = sol.zero_mean_project(space, seed_vec)
        # multigrid.py:106-113: est_op = project(L(p)), project = zero_mean_project
        lmax, _ = sol.eigen_estimate_via_cg(
            lambda v: sol.zero_mean_project(space, L(v)), diag, seed_vec, 20)
        cfg = sol.ChebyshevConfig(5, 20.0, 1.1 * lmax)
        out[key + "_seed"] = em(space, seed_vec)
        out[key + "_lmax"] = np.array(lmax)
        xn = space.node_coords()
        rhs = np.sin(2 * np.pi * xn[0]) * np.cos(np.pi * xn[1])
        rhs = rhs + 1e-3 * np.random.default_rng(1).standard_normal(rhs.shape)
        b = sol.zero_mean_project_dual(space, ops.mass_apply(space, rhs))
        out[key + "_b"] = em(space, b)
        for pname, prec in (
                ("cheb", lambda r: sol.chebyshev_smooth(L, diag, cfg, r)),
                ("jac", lambda r: r / diag)):
            hist = []

            def rec(r, prec=prec, hist=hist):
                z = prec(r)
                hist.append(np.sqrt(max(np.vdot(r, z).real, 0.0)))
                return z
            x, st = sol.pcg(op, rec, b, rel_tol=1e-10, max_iter=2000)
            out[f"{key}_{pname}_x"] = em(space, x)
            out[f"{key}_{pname}_hist"] = np.array(hist)
            out[f"{key}_{pname}_iters"] = np.array(st.iterations)
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, len(out), "arrays")


if __name__ == "__main__":
    main()
