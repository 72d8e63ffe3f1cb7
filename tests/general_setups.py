"""Meshes of the general-geometry 2D golden cases (tests/golden/
ref2d_general.npz, made by tests/golden/make_golden_general.py from the
reference) rebuilt as plain objects with the reference Mesh fields the
general path reads (duck typing: no reference import on the GPU box)."""

import os
from types import SimpleNamespace

import numpy as np

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref2d_general.npz")
CASES = {"curved": (2, 3, 5), "cylinder": (3,), "graded": (3,)}


def load():
    return np.load(GOLD)


def mesh(Z, name):
    faces = SimpleNamespace(**{k: Z[f"{name}_{k}"] for k in ("em", "sm", "ep", "sp", "flip")})
    bnd = SimpleNamespace(elem=Z[f"{name}_belem"], slot=Z[f"{name}_bslot"], tag=Z[f"{name}_btag"])
    m = SimpleNamespace(geom_degree=int(Z[f"{name}_geom_degree"]),
                        geom_nodes=Z[f"{name}_geom_nodes"], interior=faces, boundary=bnd,
                        tag_names=[str(t) for t in Z[f"{name}_tags"]],
                        n_elements=Z[f"{name}_geom_nodes"].shape[2], parent=None, quadrant=None)
    if f"{name}_parent" in Z:
        m.parent, m.quadrant = Z[f"{name}_parent"], Z[f"{name}_quadrant"]
    return m


def kinds(Z, name):
    """tag -> 'D' / 'N' for the tags the case assigns."""
    out = {}
    for s in Z[f"{name}_kinds"]:
        t, v = str(s).split(":")
        if v != "-":
            out[t] = v
    return out


def relerr(a, b):
    a, b = np.asarray(a).ravel(), np.asarray(b).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
