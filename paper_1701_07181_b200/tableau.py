"""Butcher tableaux consumed by the hot path as host scalars.

Only the quantities the linear solve needs: A^-1 (the s x s stage mixing of
the transformed operator), b^T A^-1, and the uncoupled-preconditioner
shifts alpha_i = sum_{j != i} |(A^-1)_{ji}| (column sums, reference
``tableaux.py:257-275``, shift at ``:274``).  Closed forms follow the
published Radau IIA (orders 3, 5), Alexander's DIRK3 and the 6-stage
ESDIRK5 coefficients, the same ones the reference ships
(``tableaux.py:79-137``); RADAU47 / RADAU59 (and any s <= 9) come from the
s-stage Radau IIA construction (``tableaux.py:155-254``): abscissae = roots of
P_s(2x-1) - P_{s-1}(2x-1), A_ik = integral_0^{c_i} of the k-th Lagrange basis
polynomial on the abscissae, b = last row of A (stiff accuracy).
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
    kind: str  # "irk" | "dirk" | "esdirk"
    order: int = 0

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
    return Tableau("RADAU23", A, A[1].copy(), np.array([1.0 / 3.0, 1.0]), "irk", 3)


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
                   np.array([0.4 - r6 / 10.0, 0.4 + r6 / 10.0, 1.0]), "irk", 5)


def _dirk33() -> Tableau:
    phi = math.atan(math.sqrt(2.0) / 4.0) / 3.0
    g = 1.0 + math.sqrt(6.0) / 2.0 * math.sin(phi) - math.sqrt(2.0) / 2.0 * math.cos(phi)
    tau2 = (1.0 + g) / 2.0
    b1 = -(6.0 * g ** 2 - 16.0 * g + 1.0) / 4.0
    b2 = (6.0 * g ** 2 - 20.0 * g + 5.0) / 4.0
    A = np.array([[g, 0.0, 0.0], [tau2 - g, g, 0.0], [b1, b2, g]])
    return Tableau("DIRK33", A, np.array([b1, b2, g]), np.array([g, tau2, 1.0]), "dirk", 3)


def _esdirk65() -> Tableau:
    # 6-stage, order-5, L-stable ESDIRK (explicit first stage, a_11 = 0); published
    # coefficients as the reference lists them (tableaux.py:120-137)
    g = 0.2780538411364465
    A = np.zeros((6, 6))
    A[1, :2] = [g, g]
    A[2, :3] = [0.3137405401502951, 0.4363327154020044, g]
    A[3, :4] = [0.2741986534107860, -0.0164268277321164, 0.0048197082596452, g]
    A[4, :5] = [-0.2441776975175844, -3.3203529439447852, 0.0477747285706825, 3.2974431145814931, g]
    A[5, :6] = [-0.2786732780227907, 1.8929947094010862, -0.1280948204262490, -1.3574693381380240,
                0.5931888860495311, g]
    c = np.array([0.0, 0.556107682272893, 1.028127096688746, 0.540645375074761,
                  0.058741042826253, 1.0])
    return Tableau("ESDIRK65", A, A[5].copy(), c, "esdirk", 5)


def radau_abscissae(s: int) -> np.ndarray:
    """Radau IIA nodes on (0, 1]: the s-1 interior roots of
    Q_s(x) = P_s(2x-1) - P_{s-1}(2x-1) (Legendre companion-matrix eigenvalues,
    polished by Newton steps on Q_s) followed by x = 1 exactly."""
    from numpy.polynomial import legendre as leg
    if s == 1:
        return np.array([1.0])
    q = np.zeros(s + 1)
    q[s], q[s - 1] = 1.0, -1.0
    dq = leg.legder(q)
    y = np.sort(np.real(leg.legroots(q)))
    y = y[np.abs(y - 1.0) > 1e-8]               # drop the root at y = 1 (x = 1)
    if len(y) != s - 1:
        raise RuntimeError(f"Radau IIA: found {len(y)} interior nodes for s={s}")
    for _ in range(4):
        y = y - leg.legval(y, q) / leg.legval(y, dq)
    return np.append(np.sort(0.5 * (y + 1.0)), 1.0)


def generate_radau_iia(s: int) -> Tableau:
    """s-stage Radau IIA (order 2s-1; reference tableaux.py:246-254):
    A_ik = integral_0^{c_i} l_k(x) dx with l_k the Lagrange basis polynomial on
    the nodes (degree s-1), by an (s+1)-point Gauss-Legendre rule on [0, c_i]
    (exact for that degree; l_k evaluated in product form)."""
    from numpy.polynomial import legendre as leg
    if not 1 <= s <= 9:
        raise ValueError(f"stage count {s} outside supported range [1, 9]")
    c = radau_abscissae(s)
    xg, wg = leg.leggauss(s + 1)
    A = np.empty((s, s))
    for i in range(s):
        x = 0.5 * c[i] * (xg + 1.0)
        w = 0.5 * c[i] * wg
        for k in range(s):
            ell = np.ones_like(x)
            for j in range(s):
                if j != k:
                    ell *= (x - c[j]) / (c[k] - c[j])
            A[i, k] = w @ ell
    return Tableau(f"RADAU{s}{2 * s - 1}", A, A[s - 1].copy(), c, "irk", 2 * s - 1)


_BUILTIN = {"RADAU23": _radau23, "RADAU35": _radau35, "RADAU47": lambda: generate_radau_iia(4),
            "RADAU59": lambda: generate_radau_iia(5), "DIRK33": _dirk33, "ESDIRK65": _esdirk65}
BUILTIN_NAMES = ("RADAU23", "RADAU35", "RADAU47", "RADAU59", "DIRK33", "ESDIRK65")


def builtin_tableau(name: str) -> Tableau:
    try:
        return _BUILTIN[name.upper()]()
    except KeyError:
        raise ValueError(f"unknown scheme {name!r}; expected one of {sorted(_BUILTIN)}")


def derive(tab: Tableau) -> Derived:
    """A^-1 = solve(A, I); shifts = off-diagonal |A^-1| column sums.  ESDIRK:
    the implicit trailing block A[1:, 1:] (reference tableaux.py:257-275)."""
    A, b = (tab.A[1:, 1:], tab.b[1:]) if tab.kind == "esdirk" else (tab.A, tab.b)
    s = A.shape[0]
    if abs(np.linalg.det(A)) < 1e-14:
        raise ValueError(f"{tab.name}: Butcher matrix is singular")
    a_inv = np.linalg.solve(A, np.eye(s))
    shifts = np.abs(a_inv).sum(axis=0) - np.abs(np.diag(a_inv))
    return Derived(a_inv=a_inv, bT_a_inv=b @ a_inv, shifts=shifts)
