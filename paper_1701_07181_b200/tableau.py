"""Butcher tableaux consumed by the hot path as host scalars.

Only the quantities the linear solve needs: A^-1 (the s x s stage mixing of
the transformed operator), b^T A^-1, and the uncoupled-preconditioner
shifts alpha_i = sum_{j != i} |(A^-1)_{ji}| (column sums, reference
``tableaux.py:257-275``, shift at ``:274``).  Closed forms follow the
published Radau IIA (orders 3, 5) and Alexander's DIRK3 coefficients, the
same ones the reference ships (``tableaux.py:79-119``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Tableau:
    name: str
    A: np.ndarray
    b: np.ndarray
    c: np.ndarray
    kind: str  # "irk" | "dirk"

    @property
    def s(self) -> int:
        return len(self.b)


@dataclass(frozen=True)
class Derived:
    a_inv: np.ndarray
    bT_a_inv: np.ndarray
    shifts: np.ndarray


def _radau23() -> Tableau:
    A = np.array([[5.0 / 12.0, -1.0 / 12.0], [3.0 / 4.0, 1.0 / 4.0]])
    return Tableau("RADAU23", A, A[1].copy(), np.array([1.0 / 3.0, 1.0]), "irk")


def _radau35() -> Tableau:
    r6 = math.sqrt(6.0)
    A = np.array([
        [11.0 / 45.0 - 7.0 * r6 / 360.0, 37.0 / 225.0 - 169.0 * r6 / 1800.0,
         -2.0 / 225.0 + r6 / 75.0],
        [37.0 / 225.0 + 169.0 * r6 / 1800.0, 11.0 / 45.0 + 7.0 * r6 / 360.0,
         -2.0 / 225.0 - r6 / 75.0],
        [4.0 / 9.0 - r6 / 36.0, 4.0 / 9.0 + r6 / 36.0, 1.0 / 9.0],
    ])
    return Tableau("RADAU35", A, A[2].copy(),
                   np.array([0.4 - r6 / 10.0, 0.4 + r6 / 10.0, 1.0]), "irk")


def _dirk33() -> Tableau:
    phi = math.atan(math.sqrt(2.0) / 4.0) / 3.0
    g = 1.0 + math.sqrt(6.0) / 2.0 * math.sin(phi) - math.sqrt(2.0) / 2.0 * math.cos(phi)
    tau2 = (1.0 + g) / 2.0
    b1 = -(6.0 * g ** 2 - 16.0 * g + 1.0) / 4.0
    b2 = (6.0 * g ** 2 - 20.0 * g + 5.0) / 4.0
    A = np.array([[g, 0.0, 0.0], [tau2 - g, g, 0.0], [b1, b2, g]])
    return Tableau("DIRK33", A, np.array([b1, b2, g]), np.array([g, tau2, 1.0]), "dirk")


_BUILTIN = {"RADAU23": _radau23, "RADAU35": _radau35, "DIRK33": _dirk33}


def builtin_tableau(name: str) -> Tableau:
    try:
        return _BUILTIN[name.upper()]()
    except KeyError:
        raise ValueError(f"unknown scheme {name!r}; expected one of {sorted(_BUILTIN)}")


def derive(tab: Tableau) -> Derived:
    """A^-1 = solve(A, I); shifts = off-diagonal |A^-1| column sums."""
    A = tab.A
    s = A.shape[0]
    if abs(np.linalg.det(A)) < 1e-14:
        raise ValueError(f"{tab.name}: Butcher matrix is singular")
    a_inv = np.linalg.solve(A, np.eye(s))
    shifts = np.abs(a_inv).sum(axis=0) - np.abs(np.diag(a_inv))
    return Derived(a_inv=a_inv, bT_a_inv=tab.b @ a_inv, shifts=shifts)
