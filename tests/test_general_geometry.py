"""CPU: the host-side geometry restatement of the general 2D path
(paper_1607_01323_b200/general.py: Geometry2D, compute_tau_ip) against the
reference's Geometry arrays and tau_e (geometry.py:29-108) on a warped
k_geo = 2 box, the cylinder mesh (k_geo = 4, flipped faces) and a graded
periodic box (tests/golden/ref2d_general.npz)."""

import numpy as np
import pytest

from tests.general_setups import CASES, load, mesh, relerr

from paper_1607_01323_b200.general import Geometry2D, compute_tau_ip  # noqa: E402

TOL = 1e-13


@pytest.mark.parametrize("name,k", [(n, k) for n, ks in CASES.items() for k in ks])
def test_geometry_matches_reference(name, k):
    Z = load()
    m = mesh(Z, name)
    g = Geometry2D(m, k + 1)
    key = f"{name}_k{k}"
    for attr, ref in (("jxw", "jxw"), ("jinvT", "jinvT"), ("normal", "normal"),
                      ("sjxw", "sjxw"), ("jinvT_f", "jinvT_f")):
        assert relerr(getattr(g, attr), Z[f"{key}_{ref}"]) < TOL, attr
    assert relerr(compute_tau_ip(m, g, k), Z[f"{key}_tau_e"]) < TOL


def test_cylinder_has_flipped_faces():
    Z = load()
    assert int(np.sum(Z["cylinder_flip"])) > 0


def test_negative_jacobian_rejected():
    Z = load()
    m = mesh(Z, "graded")
    gn = m.geom_nodes.copy()
    gn[0] = -gn[0]  # mirror x: orientation flips, det < 0
    m.geom_nodes = gn
    with pytest.raises(ValueError):
        Geometry2D(m, 4)
