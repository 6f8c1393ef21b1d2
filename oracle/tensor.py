"""Oracle: dense tensor primitives (§II.B).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Linearisation is first-index-fastest everywhere: the mode-m
unfolding has the mode-m index as row and the remaining modes, in increasing
mode order with the lowest varying fastest, as column (the convention of
Alg. 1 step 5).
"""
from __future__ import annotations

import numpy as np


def unfold(t: np.ndarray, mode: int) -> np.ndarray:
    """Mode-`mode` unfolding (mode is 1-based as in the paper)."""
    m = mode - 1
    return np.reshape(np.moveaxis(t, m, 0), (t.shape[m], -1), order="F")


def fold(mat: np.ndarray, mode: int, shape) -> np.ndarray:
    """Inverse of `unfold`."""
    m = mode - 1
    shape = tuple(shape)
    moved = (shape[m],) + shape[:m] + shape[m + 1:]
    return np.moveaxis(np.reshape(mat, moved, order="F"), 0, m)


def mode_product(t: np.ndarray, u: np.ndarray, mode: int) -> np.ndarray:
    """i-mode product Y = T x_i U, eq. (10): Y[.., v_i, ..] =
    sum_{i'} T[.., i', ..] U[v_i, i'].  Computed as unfold -> matmul -> fold."""
    shape = list(t.shape)
    shape[mode - 1] = u.shape[0]
    return fold(u @ unfold(t, mode), mode, shape)


def contract_mode3(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """Z = X x_3^3 Y, eq. (12): Z[a,b,c,d] = sum_i X[a,b,i] Y[c,d,i]."""
    return np.einsum("abi,cdi->abcd", x, y)


def frob(t: np.ndarray) -> float:
    return float(np.sqrt(np.sum(np.abs(t) ** 2)))


def rel_err(ref: np.ndarray, got: np.ndarray) -> float:
    """||ref - got||_F / ||ref||_F (||got||_F if ref is zero)."""
    d = frob(np.asarray(ref) - np.asarray(got))
    n = frob(ref)
    return d / n if n > 0 else frob(got)
