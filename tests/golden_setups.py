"""Shared builders mirroring tests/golden/make_golden.py's SETUPS, for the
oracle (CPU) and for the CUDA path (GPU)."""

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                      "ref2d.npz")

SETUPS = {
    "periodic": (((0, 1), (0, 1)), (3, 3), (0.0, 0.0), (True, True), {}),
    "mixed": (((0, 1), (0, 1)), (3, 3), (0.8, 0.0), (False, False),
              {"xmin": "D", "xmax": "N", "ymin": "D", "ymax": "D"}),
    "mixed2": (((0, 2), (-1, 1)), (4, 3), (0.0, 1.1), (True, False),
               {"ymin": "N", "ymax": "D"}),
    "walls": (((0, 1), (0, 1)), (3, 2), (0.0, 0.0), (False, False),
              {"xmin": "N", "xmax": "N", "ymin": "N", "ymax": "D"}),
}
KS = (2, 3, 5)


def load_golden():
    return np.load(GOLDEN)


def body_force(x, t):
    return np.stack([np.sin(x[0]) + t, x[1] ** 2])


def relerr(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


# non-zero boundary data of tests/golden/make_golden.py (2D)
def g_data(x, t):
    return np.stack([np.sin(x[0] + t) * x[1], np.cos(2 * x[1]) - t * x[0]])


def dgdt_data(x, t):
    return np.stack([np.cos(x[0] + t) * x[1], -x[0] + 0 * x[1]])


def h_data(x, t):
    return np.stack([x[0] * x[1] + t, np.sin(3 * x[0]) - x[1]])


def gp_data(x, t):
    return np.cos(x[0] - 2 * x[1]) + t


# 3D analogues (no reference exists in 3D; used against the 3D oracle)
def g_data3(x, t):
    return np.stack([np.sin(x[0] + t) * x[1], np.cos(2 * x[1]) - t * x[2],
                     x[0] * x[2] + 0.5])


def dgdt_data3(x, t):
    return np.stack([np.cos(x[0] + t) * x[1], -x[2] + 0 * x[1], np.sin(x[1] * x[2])])


def h_data3(x, t):
    return np.stack([x[0] * x[1] + t, np.sin(3 * x[0]) - x[2], x[1] - x[2] ** 2])


def gp_data3(x, t):
    return np.cos(x[0] - 2 * x[1] + x[2]) + t


def body_force3(x, t):
    return np.stack([np.sin(x[0]) + t, x[1] ** 2, np.cos(x[2]) * x[0]])


def oracle_bcs(O, dim, data):
    if not data:
        return O.zero_dirichlet(dim), O.zero_neumann(dim)
    if dim == 2:
        return O.DirichletBC(g_data, dgdt_data), O.NeumannBC(h_data, gp_data)
    return O.DirichletBC(g_data3, dgdt_data3), O.NeumannBC(h_data3, gp_data3)


def oracle_setup(name, k, data=False):
    from oracle import dg_oracle as O
    ext, counts, grading, per, kinds = SETUPS[name]
    mesh = O.build_box_mesh(ext, counts, grading=grading, periodic=per)
    dbc, nbc = oracle_bcs(O, 2, data)
    spec = O.BoundarySpec({t: (dbc if v == "D" else nbc) for t, v in kinds.items()})
    space = O.DgSpace(mesh, k)
    return space, spec.resolve(space)


def map_tau_c(space, z, key):
    """Reference per-face tau_C -> the oracle/GPU face enumeration, keyed by
    (minus element, minus slot) with the minus side normalised to the
    lower slot index pair of the face."""
    lut = {}
    for em, sm, ep, sp, t in zip(z[key + "_f_em"], z[key + "_f_sm"],
                                 z[key + "_f_ep"], z[key + "_f_sp"],
                                 z[key + "_tau_c"]):
        lut[(int(em), int(sm))] = t
        lut[(int(ep), int(sp))] = t
    return np.array([lut[(int(e), int(s))] for e, s in zip(space.f_em, space.f_sm)])


MESHES = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref2d_meshes.npz")


def reference_mesh(name):
    """A reference-built Mesh (tests/golden/make_golden_meshes.py) as an
    object with the reference Mesh's attribute names (pkg/src/dgins/mesh.py:
    72-90): what a reference caller passes to DgSpace(mesh, k)."""
    from types import SimpleNamespace
    z = np.load(MESHES)
    g = lambda f: z[f"{name}_{f}"]
    return SimpleNamespace(
        vertices=g("vertices"), elem_vertices=g("elem_vertices"),
        geom_degree=int(g("geom_degree")), geom_nodes=g("geom_nodes"),
        interior=SimpleNamespace(em=g("if_em"), sm=g("if_sm"), ep=g("if_ep"), sp=g("if_sp"),
                                 flip=g("if_flip")),
        boundary=SimpleNamespace(elem=g("bf_elem"), slot=g("bf_slot"), tag=g("bf_tag")),
        tag_names=[str(t) for t in g("tag_names")],
        periodic_spec={int(a): None for a in g("periodic_axes")},
        periodic_pairs=[], curved={}, parent=None, quadrant=None, coarser=None,
        n_elements=int(g("elem_vertices").shape[0]))
