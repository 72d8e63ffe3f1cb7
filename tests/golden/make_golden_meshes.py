"""Reference Mesh objects as fixtures, for the drop-in tests.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_meshes.py

Runs the REAL reference build_box_mesh (pkg/src/dgins/mesh.py:279-351) for
the golden setups of make_golden.py (and one curved mesh) and stores every
Mesh field the device path reads -- vertices, elem_vertices, geom_degree,
geom_nodes, interior / boundary face arrays, tag names, periodic axes -- in
tests/golden/ref2d_meshes.npz.  tests/golden_setups.reference_mesh() rebuilds
an object with the reference Mesh's attribute names from it, so the GPU box
(no reference tree) can feed reference-built meshes through the unchanged
call sites DgSpace(mesh, k) / BoundarySpec(...).resolve(space) / operators.
"""

import os
import sys

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import numpy as np  # noqa: E402

from dgins.mesh import build_box_mesh  # noqa: E402
from tests.golden_setups import SETUPS  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref2d_meshes.npz")


def dump(out, key, m):
    out[key + "_vertices"] = m.vertices
    out[key + "_elem_vertices"] = m.elem_vertices
    out[key + "_geom_degree"] = m.geom_degree
    out[key + "_geom_nodes"] = m.geom_nodes
    for f in ("em", "sm", "ep", "sp", "flip"):
        out[key + "_if_" + f] = getattr(m.interior, f)
    for f in ("elem", "slot", "tag"):
        out[key + "_bf_" + f] = getattr(m.boundary, f)
    out[key + "_tag_names"] = np.array(m.tag_names, dtype="U16")
    out[key + "_periodic_axes"] = np.array(sorted(m.periodic_spec), dtype=np.int64)


def main():
    out = {}
    for name, (ext, counts, grading, per, kinds) in SETUPS.items():
        dump(out, name, build_box_mesh(ext, counts, grading=grading, periodic=per))
    # an iso-parametric (k_geo = 2) box: straight, but not the affine box the
    # Cartesian context needs -> the general path
    dump(out, "kgeo2", build_box_mesh(((0, 1), (0, 1)), (3, 2), k_geo=2))
    np.savez_compressed(OUT, **out)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
