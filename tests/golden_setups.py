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


def oracle_setup(name, k):
    from oracle import dg_oracle as O
    ext, counts, grading, per, kinds = SETUPS[name]
    mesh = O.build_box_mesh(ext, counts, grading=grading, periodic=per)
    spec = O.BoundarySpec({t: (O.zero_dirichlet(2) if v == "D" else O.zero_neumann(2))
                           for t, v in kinds.items()})
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
