"""CPU-side checks of the C ABI: the library loads, exports every symbol the
header declares, host-side tables match the oracle (which is pinned to the
reference), and argument validation maps to the reference's exceptions."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_1607_01323_b200 import _lib
from paper_1607_01323_b200.basis import get_basis
from paper_1607_01323_b200.mesh import build_box_mesh
from oracle import dg_oracle as O

HEADER = os.path.join(_lib.ROOT, "include", "dgmf.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(dg_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def L():
    _lib.build()
    return _lib.lib()


def test_every_declared_symbol_is_exported(L):
    syms = declared_symbols()
    assert "dg_laplace_vmult" in syms and len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    for s in _lib.PROTOTYPES:
        assert s in syms, f"{s} bound in _lib but not declared in dgmf.h"


@pytest.mark.parametrize("k", range(1, 8))
def test_host_tables_match_oracle(L, k):
    for nq in sorted({k + 1, (3 * k) // 2 + 1, (3 * (k + 1)) // 2}):
        t = get_basis(k, nq)
        b = O.get_basis(k, nq)
        np.testing.assert_allclose(t.nodes, b.nodes, atol=1e-15, rtol=0)
        np.testing.assert_allclose(t.points, b.rule.points, atol=1e-15, rtol=0)
        np.testing.assert_allclose(t.weights, b.rule.weights, atol=1e-15, rtol=0)
        np.testing.assert_allclose(t.S, b.S, atol=2e-15, rtol=0)
        np.testing.assert_allclose(t.D, b.D, atol=1e-13, rtol=1e-14)
        np.testing.assert_allclose(t.left_deriv, b.left_deriv, rtol=1e-13)
        np.testing.assert_allclose(t.right_deriv, b.right_deriv, rtol=1e-13)


def test_invalid_degree_is_value_error(L):
    buf = np.empty(64)
    P = buf.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    with pytest.raises(ValueError):
        _lib.check(L.dg_basis_tables(0, 2, P, P, P, P, P, P, P))


def test_mesh_validation_matches_reference():
    # mesh.py:291-304
    with pytest.raises(ValueError):
        build_box_mesh(((0, 1), (0, 1)), (0, 2))
    with pytest.raises(ValueError):
        build_box_mesh(((0, 1), (1, 0)), (2, 2))
    with pytest.raises(ValueError):
        build_box_mesh(((0, 1), (0, 1)), (2, 2), grading=(0.5, 0.0),
                       periodic=(True, False))
    m = build_box_mesh(((0, 2), (-1, 1), (0, 1)), (4, 3, 2), grading=(0, 1.8, 0))
    om = O.build_box_mesh(((0, 2), (-1, 1), (0, 1)), (4, 3, 2), grading=(0, 1.8, 0))
    for d in range(3):
        np.testing.assert_allclose(m.axis_vertices[d], om.axis_vertices[d], rtol=0,
                                   atol=1e-15)
