"""Oracle: aggregation (eq. (4)) and disaggregation (eq. (6)) around the
translation of eq. (5) -- SURVEY.md §8(f) NEXT #3.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  FP64 / complex128.

Arrays (linear box index v = x + Nx (y + Ny z), x fastest, as the library's signature layout):
  P    far-field patterns P+[p, n, c], c = theta, phi components; P- = conj(P+)
  I    basis-function coefficients I_n
  box_ptr  basis functions of box v are n in [box_ptr[v], box_ptr[v+1])
  A, B signatures [p, c, v]
"""
from __future__ import annotations

import numpy as np

from . import translate


def aggregate(P: np.ndarray, I: np.ndarray, box_ptr: np.ndarray) -> np.ndarray:
    """Eq. (4): A_v(k_p) = sum_{n in B_v} P+(k_p, b_n) I_n, zero for an empty box.
    Returns A[p, c, v] (complex128)."""
    P = np.asarray(P, dtype=np.complex128)
    I = np.asarray(I, dtype=np.complex128)
    ndir, _, ncomp = P.shape
    K = len(box_ptr) - 1
    A = np.zeros((ndir, ncomp, K), dtype=np.complex128)
    for v in range(K):
        lo, hi = int(box_ptr[v]), int(box_ptr[v + 1])
        if hi > lo:
            A[:, :, v] = np.einsum("pnc,n->pc", P[:, lo:hi, :], I[lo:hi])
    return A


def disaggregate(P: np.ndarray, B: np.ndarray, w: np.ndarray, box_ptr: np.ndarray) -> np.ndarray:
    """Eq. (6): y_m = sum_p w_p P-(k_p, b_m) . B_{v(m)}(k_p), P- = conj(P+), the
    theta/phi components contracted.  B[p, c, v]; returns y[m] (complex128)."""
    P = np.asarray(P, dtype=np.complex128)
    B = np.asarray(B, dtype=np.complex128)
    w = np.asarray(w, dtype=np.float64)
    N = P.shape[1]
    K = len(box_ptr) - 1
    y = np.zeros(N, dtype=np.complex128)
    for v in range(K):
        lo, hi = int(box_ptr[v]), int(box_ptr[v + 1])
        if hi > lo:
            y[lo:hi] = np.einsum("p,pnc,pc->n", w, np.conj(P[:, lo:hi, :]), B[:, :, v])
    return y


def far_matvec(P, I, box_ptr, w, T_of_p, Nx: int, Ny: int, Nz: int) -> np.ndarray:
    """The far-field part of the matrix-vector product: eq. (4) -> eq. (5) for every direction
    and component (FP64 FFT path, translate.translate_fft) -> eq. (6).
    T_of_p(p) returns the FFT'ed operator slice T_p (2Nx, 2Ny, 2Nz) (dense or restored)."""
    A = aggregate(P, I, box_ptr)
    ndir, ncomp, K = A.shape
    B = np.empty_like(A)
    for p in range(ndir):
        t = T_of_p(p)
        for c in range(ncomp):
            a = A[p, c].reshape(Nz, Ny, Nx).transpose(2, 1, 0)          # [x, y, z]
            b = translate.translate_fft(t, a)
            B[p, c] = b.transpose(2, 1, 0).reshape(K)
    return disaggregate(P, B, w, box_ptr)
