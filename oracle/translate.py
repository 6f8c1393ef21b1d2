"""Oracle: the translation (eq. (5)) and the direction sum (eq. (6)).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Signatures are numpy arrays A[x, y, z] of shape (Nx, Ny, Nz) (math order).
The operator slice T_p is (2Nx, 2Ny, 2Nz).
"""
from __future__ import annotations

import numpy as np


def translate_fft(t_p: np.ndarray, a_p: np.ndarray) -> np.ndarray:
    """Eq. (5) by FP64 FFTs: B = F^{-1}(T_p (.) F(pad(A_p))), truncated to the
    first Nx x Ny x Nz entries (Toeplitz embedding in the 2N circulant grid)."""
    Nx, Ny, Nz = a_p.shape
    a = np.zeros(t_p.shape, dtype=np.complex128)
    a[:Nx, :Ny, :Nz] = a_p
    y = np.fft.ifftn(t_p * np.fft.fftn(a, axes=(0, 1, 2)), axes=(0, 1, 2))
    return y[:Nx, :Ny, :Nz]


def spatial_kernel(t_p: np.ndarray) -> np.ndarray:
    """t~'_p = F^{-1}(T_p): the circulant spatial kernel whose convolution the
    FFT path evaluates."""
    return np.fft.ifftn(t_p, axes=(0, 1, 2))


def translate_direct(tk_p: np.ndarray, a_p: np.ndarray, targets=None) -> np.ndarray:
    """Plain definition of eq. (5)'s result, brute force:
        B[v] = sum_{v' in [0,N)^3} t~[(v - v') mod 2N] A[v'],   v in [0,N)^3.
    `tk_p` is the spatial circulant kernel (2Nx, 2Ny, 2Nz).  With `targets`
    (an int array [m, 3] of v), returns only those m outputs."""
    Nx, Ny, Nz = a_p.shape
    n1, n2, n3 = tk_p.shape
    sx, sy, sz = np.meshgrid(np.arange(Nx), np.arange(Ny), np.arange(Nz), indexing="ij")
    sx, sy, sz = sx.ravel(), sy.ravel(), sz.ravel()
    src = a_p.ravel()                       # C-order ravel matches sx/sy/sz ravel
    if targets is None:
        tx, ty, tz = sx, sy, sz
    else:
        targets = np.asarray(targets)
        tx, ty, tz = targets[:, 0], targets[:, 1], targets[:, 2]
    out = np.empty(len(tx), dtype=np.complex128)
    for m in range(len(tx)):
        kern = tk_p[(tx[m] - sx) % n1, (ty[m] - sy) % n2, (tz[m] - sz) % n3]
        out[m] = np.sum(kern * src)
    if targets is None:
        return out.reshape(Nx, Ny, Nz)
    return out


def direction_sum(b: np.ndarray, w: np.ndarray) -> np.ndarray:
    """Eq. (6) with P^- = 1 (reading Q15): S[v] = sum_p w_p B_p[v].
    `b` is indexed [p, x, y, z]."""
    return np.tensordot(np.asarray(w, dtype=np.float64), b, axes=(0, 0))


def sig_to_math(buf: np.ndarray) -> np.ndarray:
    """Library layout [ndir][Nz][Ny][Nx] -> oracle order [p, x, y, z]."""
    return np.transpose(buf, (0, 3, 2, 1)).astype(np.complex128)


def math_to_sig(b: np.ndarray) -> np.ndarray:
    """Oracle order [p, x, y, z] -> library layout [ndir][Nz][Ny][Nx]."""
    return np.ascontiguousarray(np.transpose(b, (0, 3, 2, 1)))
