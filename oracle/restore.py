"""Oracle: restoration of the FFT'ed operator from its compressed forms
(eqs. (8), (9), (11), (13), (14); Figs. 3-4 described at P:137-149).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Factors are used as
stored, without conjugation (the equations carry none).  Directions p are
0-based here.
"""
from __future__ import annotations

import numpy as np

from .tensor import contract_mode3, mode_product


# ------------------------------------------------------------------ dense forms
def tucker_full(core: np.ndarray, factors) -> np.ndarray:
    """Eqs. (8)/(9): T = C x_1 U^1 x_2 U^2 x_3 U^3 (x_4 U^4)."""
    t = core
    for i, u in enumerate(factors, start=1):
        t = mode_product(t, u, i)
    return t


def htucker_core(c12, c34, c1234) -> np.ndarray:
    """Eq. (11)'s bracket, explicit form (reading Q12b):
    core[a,b,c,d] = sum_{i,j} C12[a,b,i] C1234[i,j] C34[c,d,j]
    = C12 x_3^3 (C34 x_3 C1234), with x_3^3 of eq. (12)."""
    c34_root = mode_product(c34, c1234, 3)          # C34 x_3 C1234: [c,d,i] = sum_j C34[c,d,j] C1234[i,j]
    z = contract_mode3(c12, c34_root)               # [a,b,c,d] = sum_i C12[a,b,i] (..)[c,d,i]
    return z


def htucker_full(leaves, c12, c34, c1234) -> np.ndarray:
    """Eq. (11): T_4D = core x_1 U^1 x_2 U^2 x_3 U^3 x_4 U^4."""
    return tucker_full(htucker_core(c12, c34, c1234), leaves)


def tt3d_full(u1, c1, u3) -> np.ndarray:
    """Eq. (13): T_3D = C^1 x_1 U^1 x_3 U^3 (C^1: r1 x n2 x r2)."""
    return mode_product(mode_product(c1, u1, 1), u3, 3)


def tt4d_full(u1, c1, c2, u4) -> np.ndarray:
    """Eq. (14): T_4D = (C^1 x_1 U^1) x_3^1 (C^2 x_3 U^last):
    T[i,j,k,p] = sum_{a,b,c} U1[i,a] C1[a,j,b] C2[b,k,c] U4[p,c]."""
    left = mode_product(c1, u1, 1)                  # n1 x n2 x r2
    right = mode_product(c2, u4, 3)                 # r2 x n3 x n4
    return np.einsum("ijb,bkp->ijkp", left, right)


# ------------------------------------------------------------------ slice chains
def tucker3d_restore(core, u1, u2, u3) -> np.ndarray:
    """Fig. 3(a): C -> x U^1 -> reshape -> x U^2 -> x U^3 -> T_3D."""
    return tucker_full(core, [u1, u2, u3])


def tucker4d_slice(core, factors, p: int) -> np.ndarray:
    """Fig. 3(b): core (as r1 r2 r3 x r4 matrix) times the transpose of
    row p of U^4 -> 3D core -> Fig. 3(a)."""
    r = core.shape
    cmat = np.reshape(core, (r[0] * r[1] * r[2], r[3]), order="F")
    c3 = np.reshape(cmat @ factors[3][p, :], r[:3], order="F")
    return tucker3d_restore(c3, factors[0], factors[1], factors[2])


def htucker_slice(leaves, c12, c34, c1234, p: int) -> np.ndarray:
    """Fig. 3(c): C34 (as a matrix) times row p of U^4 -> M (r3 x r34);
    then times C1234 and C12 -> 3D core (r1 x r2 x r3) -> Fig. 3(a)."""
    r3, r4, r34 = c34.shape
    r1, r2, r12 = c12.shape
    m = np.einsum("cdj,d->cj", c34, leaves[3][p, :])         # r3 x r34
    nmat = c1234 @ m.T                                        # r12 x r3
    c3 = np.reshape(np.reshape(c12, (r1 * r2, r12), order="F") @ nmat,
                    (r1, r2, r3), order="F")
    return tucker3d_restore(c3, leaves[0], leaves[1], leaves[2])


def tt3d_restore(u1, c1, u3) -> np.ndarray:
    """Fig. 4(a): step 1 U^1 . C (C^1 as r1 x n2 r2) = T1; step 2 reshape
    T1 to (n1 n2 x r2) and multiply by U^3 transposed; step 3 fold."""
    r1, n2, r2 = c1.shape
    n1, n3 = u1.shape[0], u3.shape[0]
    t1 = u1 @ np.reshape(c1, (r1, n2 * r2), order="F")      # n1 x n2 r2
    t1 = np.reshape(t1, (n1 * n2, r2), order="F")
    return np.reshape(t1 @ u3.T, (n1, n2, n3), order="F")


def tt4d_t2(c2, u4) -> np.ndarray:
    """Fig. 4(b) step 1: T2 = C^2 (as r2 n3 x r3) times U^last transposed
    (r2 n3 x n4).  Independent of p, so callers may compute it once."""
    r2, n3, r3 = c2.shape
    return np.reshape(c2, (r2 * n3, r3), order="F") @ u4.T


def tt4d_slice(u1, c1, c2, u4, p: int, t2=None) -> np.ndarray:
    """Fig. 4(b): step 1 T2 = C^2 (as r2 n3 x r3) times U^last
    transposed; step 2 column p of T2, reshaped r2 x n3, left-multiplied by
    T1 (n1 n2 x r2) of Fig. 4(a) step 1; step 3 fold."""
    r1, n2, r2 = c1.shape
    _, n3, r3 = c2.shape
    n1 = u1.shape[0]
    if t2 is None:
        t2 = tt4d_t2(c2, u4)                                  # r2 n3 x n4
    col = np.reshape(t2[:, p], (r2, n3), order="F")
    t1 = np.reshape(u1 @ np.reshape(c1, (r1, n2 * r2), order="F"), (n1 * n2, r2), order="F")
    return np.reshape(t1 @ col, (n1, n2, n3), order="F")
