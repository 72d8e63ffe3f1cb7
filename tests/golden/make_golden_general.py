"""Golden vectors of the reference's GENERAL 2D geometry path (curved
iso-parametric cells, unstructured connectivity with face flips), produced
by running the real reference (2D ``dgins``) in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_general.py

Writes ``tests/golden/ref2d_general.npz`` (committed; the GPU box reads only
the npz).  Per case: the mesh as the reference builds it (geom_nodes, face
lists, tags), the reference Geometry arrays and tau_e (to pin the host-side
geometry restatement), seeded inputs and the reference operator outputs, all
in the reference kernel layout (m, ne, m) / (c, m, ne, m).

Cases: a box mesh with k_geo = 2 warped by a smooth map of our own (the
reference test-suite's "curved" setting, pkg/tests/test_operators.py:45-50)
and the laminar cylinder mesh (pkg/src/dgins/cylinder.py, 136 cells, k_geo
4, curved boundary, 8 flipped interior faces), plus a graded box through
the same path.
"""

import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from dgins import operators as ops  # noqa: E402
from dgins import solvers as sol  # noqa: E402
from dgins.cylinder import build_cylinder_mesh, cylinder_mesh_hierarchy  # noqa: E402
from dgins.multigrid import MultigridHierarchy  # noqa: E402
from dgins.mesh import build_box_mesh  # noqa: E402
from dgins.spaces import DgSpace  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref2d_general.npz")


def z2(x, t):
    return np.zeros((2,) + x.shape[1:])


def z1(x, t):
    return np.zeros(x.shape[1:])


def g_data(x, t):
    """Smooth velocity-Dirichlet data (vector)."""
    return np.stack([np.sin(2.0 * x[0] + t) * np.cos(x[1]), 0.3 * np.cos(x[0] - 2.0 * t) + x[1]])


def dg_data(x, t):
    return np.stack([np.cos(2.0 * x[0] + t) * np.cos(x[1]), 0.6 * np.sin(x[0] - 2.0 * t)])


def h_data(x, t):
    return np.stack([0.4 * x[1] + np.sin(t), np.cos(3.0 * x[0]) * x[1]])


def gp_data(x, t):
    return 0.5 + np.sin(x[0] + 2.0 * x[1] + t)


def force(x, t):
    return np.stack([0.2 + np.cos(x[1]) * np.sin(t), x[0] * x[1] - 0.1])


def warp(xy):
    """A smooth non-affine map of the unit square onto itself."""
    x, y = xy[0], xy[1]
    s = np.sin(np.pi * x) * np.sin(np.pi * y)
    return x + 0.07 * s * (1.0 - y), y - 0.04 * s * (0.5 + x)


def curved_box(n):
    m = build_box_mesh(((0, 1), (0, 1)), (n, n), k_geo=2)
    m.geom_nodes = np.stack(warp(np.stack([m.geom_nodes[0], m.geom_nodes[1]])))
    m.vertices = np.stack(warp(m.vertices.T), axis=1)
    return m


CASES = {
    # name: (mesh builder, degrees, kinds per tag)
    "curved": (lambda: curved_box(3), (2, 3, 5),
               {"xmin": "D", "xmax": "N", "ymin": "D", "ymax": "D"}),
    "cylinder": (lambda: build_cylinder_mesh(level=0, k_geo=4), (3,),
                 {"inflow": "D", "outflow": "N", "wall": "D", "cylinder": "D"}),
    "graded": (lambda: build_box_mesh(((0, 2), (-1, 1)), (4, 3), grading=(0.0, 1.2),
                                      periodic=(True, False)), (3,),
               {"ymin": "D", "ymax": "N"}),
}


def main():
    rng = np.random.default_rng(20261019)
    out = {}
    for name, (build, degrees, kinds) in CASES.items():
        mesh = build()
        f, b = mesh.interior, mesh.boundary
        out[f"{name}_geom_degree"] = np.array(mesh.geom_degree)
        out[f"{name}_geom_nodes"] = mesh.geom_nodes
        for key in ("em", "sm", "ep", "sp", "flip"):
            out[f"{name}_{key}"] = np.asarray(getattr(f, key))
        out[f"{name}_belem"] = np.asarray(b.elem)
        out[f"{name}_bslot"] = np.asarray(b.slot)
        out[f"{name}_btag"] = np.asarray(b.tag)
        out[f"{name}_tags"] = np.array(mesh.tag_names)
        out[f"{name}_kinds"] = np.array([f"{t}:{kinds.get(t, '-')}" for t in mesh.tag_names])
        spec = ops.BoundarySpec({t: (ops.DirichletBC(z2, z2) if v == "D" else ops.NeumannBC(z2, z1))
                                 for t, v in kinds.items()})
        spec_g = ops.BoundarySpec({t: (ops.DirichletBC(g_data, z2) if v == "D"
                                       else ops.NeumannBC(z2, z1)) for t, v in kinds.items()})
        spec_d = ops.BoundarySpec({t: (ops.DirichletBC(g_data, dg_data) if v == "D"
                                       else ops.NeumannBC(h_data, gp_data))
                                   for t, v in kinds.items()})
        for k in degrees:
            space = DgSpace(mesh, k)
            bcs = spec.resolve(space)
            g = space.geom
            key = f"{name}_k{k}"
            out[key + "_jxw"] = g.jxw
            out[key + "_jinvT"] = g.jinvT
            out[key + "_normal"] = g.normal
            out[key + "_sjxw"] = g.sjxw
            out[key + "_jinvT_f"] = g.jinvT_f
            out[key + "_tau_e"] = space.tau_e
            m, ne = k + 1, mesh.n_elements
            p = rng.standard_normal((m, ne, m))
            u = rng.standard_normal((2, m, ne, m))
            out[key + "_p"] = p
            out[key + "_u"] = u
            out[key + "_mass_p"] = ops.mass_apply(space, p)
            out[key + "_mass_u"] = ops.mass_apply(space, u)
            out[key + "_imass_p"] = ops.inverse_mass_apply(space, p)
            out[key + "_imass_u"] = ops.inverse_mass_apply(space, u)
            out[key + "_lap"] = ops.apply_pressure_laplace(space, p, bcs)
            out[key + "_lap25"] = ops.apply_pressure_laplace(space, p, bcs, tau_scale=2.5)
            out[key + "_diag"] = ops.laplace_diagonal(space, bcs)
            u2 = rng.standard_normal((2, m, ne, m))
            out[key + "_u2"] = u2
            out[key + "_helm"] = ops.apply_viscous_helmholtz(space, u, 3.0, 0.7, bcs)
            out[key + "_helm0"] = ops.apply_viscous_helmholtz(space, u, 3.0, 0.0, bcs)
            td = rng.uniform(0.1, 0.5, ne)
            tc = rng.uniform(0.1, 0.5, mesh.interior.n)
            out[key + "_tau_d"] = td
            out[key + "_tau_c"] = tc
            out[key + "_proj"] = ops.apply_projection_operator(space, u, td, tc)
            out[key + "_projD"] = ops.apply_projection_operator(space, u, td, None)
            out[key + "_projC"] = ops.apply_projection_operator(space, u, None, tc)
            for form in ("standard", "weak", "strong"):
                out[key + f"_div_{form}"] = ops.eval_divergence_rhs(space, u, bcs, 1.7, form)
            for form in ("standard", "weak"):
                out[key + f"_grad_{form}"] = ops.eval_pressure_gradient_rhs(space, p, bcs, 0.9, form)
            out[key + "_vort"] = ops.compute_vorticity(space, u)
            bcs_g = spec_g.resolve(space)
            out[key + "_conv1"] = ops.eval_convective_rhs(space, bcs, [u], (1.0,), (0.0,), 0.0)
            out[key + "_conv2"] = ops.eval_convective_rhs(space, bcs_g, [u, u2], (2.0, -1.0),
                                                          (0.3, 0.2), 0.4, body_force=force)
            bcs_d = spec_d.resolve(space)
            w1 = rng.standard_normal((m, ne, m))
            w2 = rng.standard_normal((m, ne, m))
            out[key + "_w1"] = w1
            out[key + "_w2"] = w2
            out[key + "_gp"] = ops.gp_dirichlet_rhs(space, bcs_d, 0.35, tau_scale=1.7)
            out[key + "_vbc"] = ops.viscous_rhs_bc(space, bcs_d, 0.35, 0.03)
            out[key + "_pn"] = ops.eval_pressure_neumann_rhs(space, bcs_d, [u, u2], [w1, w2],
                                                             (2.0, -1.0), 0.03, 0.45,
                                                             body_force=force)
            out[key + "_xn"] = space.node_coords()
            out[key + "_zm"] = sol.zero_mean_project(space, p)
            out[key + "_zmd"] = sol.zero_mean_project_dual(space, p)
            td, tcf = ops.compute_penalty_parameters(space, u, 1e-3, 0.8,
                                                     ops.VariantConfig("V4", 1.3, 0.7))
            out[key + "_pen_d"] = td
            out[key + "_pen_c"] = tcf
            print(name, k, "ne", ne, "flips", int(np.sum(f.flip)))
    # multigrid on the refined cylinder hierarchy (multigrid.py:76-175):
    # pressure-Dirichlet outflow (non-singular) and all velocity-Dirichlet
    # sides (pure Neumann pressure: projected Lanczos, dual-projected rhs)
    for mname, kinds in (("mgcyl", {"inflow": "D", "outflow": "N", "wall": "D", "cylinder": "D"}),
                         ("mgcylN", {"inflow": "D", "outflow": "D", "wall": "D", "cylinder": "D"})):
        meshes = cylinder_mesh_hierarchy(1, k_geo=4)
        k = 2
        spaces = [DgSpace(m, k) for m in meshes]
        spec = ops.BoundarySpec({t: (ops.DirichletBC(z2, z2) if v == "D" else ops.NeumannBC(z2, z1))
                                 for t, v in kinds.items()})
        singular = mname == "mgcylN"
        mg = MultigridHierarchy(spaces, spec,
                                project=sol.zero_mean_project if singular else None)
        top = spaces[-1]
        bcs = spec.resolve(top)
        m, ne = k + 1, top.mesh.n_elements
        b = rng.standard_normal((m, ne, m))
        if singular:
            b = sol.zero_mean_project_dual(top, b)
        out[f"{mname}_b"] = b
        out[f"{mname}_lmax"] = np.array([lv.cheb.lambda_max for lv in mg.levels])
        out[f"{mname}_coarse_iters"] = np.array(mg.levels[0].coarse_iters)
        out[f"{mname}_vcycle"] = mg.vcycle(b)
        if singular:
            op = lambda x: sol.zero_mean_project_dual(top, ops.apply_pressure_laplace(top, x, bcs))
        else:
            op = lambda x: ops.apply_pressure_laplace(top, x, bcs)
        hist = []

        def rec(r):
            z = mg.vcycle(r)
            hist.append(np.sqrt(max(np.vdot(r, z).real, 0.0)))
            return z
        x, st = sol.pcg(op, rec, b, rel_tol=1e-8, max_iter=100)
        out[f"{mname}_pcg_iters"] = np.array(st.iterations)
        out[f"{mname}_pcg_hist"] = np.array(hist)
        out[f"{mname}_pcg_x"] = x
        for lvl, mm in enumerate(meshes):
            pre = f"{mname}_L{lvl}"
            f, bb = mm.interior, mm.boundary
            out[pre + "_geom_nodes"] = mm.geom_nodes
            out[pre + "_geom_degree"] = np.array(mm.geom_degree)
            for kk in ("em", "sm", "ep", "sp", "flip"):
                out[pre + "_" + kk] = np.asarray(getattr(f, kk))
            out[pre + "_belem"], out[pre + "_bslot"], out[pre + "_btag"] = bb.elem, bb.slot, bb.tag
            out[pre + "_tags"] = np.array(mm.tag_names)
            out[pre + "_kinds"] = np.array([f"{t}:{kinds.get(t, '-')}" for t in mm.tag_names])
            if mm.parent is not None:
                out[pre + "_parent"] = np.asarray(mm.parent)
                out[pre + "_quadrant"] = np.asarray(mm.quadrant)
        print(mname, "levels", len(meshes), "iters", st.iterations, "coarse", mg.levels[0].coarse_iters)
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
