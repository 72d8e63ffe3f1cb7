"""1D tables from the library (long-double host code in csrc/tables.cpp).

Mirrors reference quadrature.py / basis.py: ``gll_nodes(k)``,
``gauss_rule(n)`` and ``get_basis(k, n_q)`` with S, D, endpoint rows.
"""

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib


@dataclass(frozen=True)
class Tables1D:
    k: int
    n_q: int
    nodes: np.ndarray
    points: np.ndarray
    weights: np.ndarray
    S: np.ndarray
    D: np.ndarray
    left_deriv: np.ndarray
    right_deriv: np.ndarray


_cache = {}


def get_basis(k, n_q):
    key = (k, n_q)
    if key in _cache:
        return _cache[key]
    n = k + 1
    S = np.empty((n_q, n))
    D = np.empty((n_q, n))
    nodes = np.empty(n)
    pts = np.empty(n_q)
    w = np.empty(n_q)
    ld = np.empty(n)
    rd = np.empty(n)
    P = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    _lib.check(_lib.lib().dg_basis_tables(k, n_q, P(S), P(D), P(nodes), P(pts),
                                          P(w), P(ld), P(rd)))
    for a in (S, D, nodes, pts, w, ld, rd):
        a.flags.writeable = False
    t = Tables1D(k, n_q, nodes, pts, w, S, D, ld, rd)
    _cache[key] = t
    return t


def gll_nodes(k):
    return get_basis(k, k + 1).nodes


def gauss_rule(n):
    t = get_basis(1, n)
    return t.points, t.weights
