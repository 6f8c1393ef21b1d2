"""Test helpers: oracle formats -> library arrays (complex64, first-index-fastest),
and oracle restorations from the SAME rounded factors (so GPU and oracle see
identical compressed factors, as BASELINE.json's parity clause requires).

Direction of data flow is oracle -> library only: nothing here feeds a
library output back into the oracle.
"""
from __future__ import annotations

import functools

import numpy as np

from oracle import decomp, fmm, restore, translate
from synth import config


def f32(a):
    """Round to complex64 and back: the factors both sides use."""
    return np.asarray(a).astype(np.complex64).astype(np.complex128)


def flat(a):
    return np.asarray(a).ravel(order="F").astype(np.complex64)


@functools.lru_cache(maxsize=None)
def operator(cfg: int, ndir: int | None = None):
    """Oracle FFT'ed operator T_4D (n1, n2, n3, ndir) and the weights."""
    c = config(cfg)
    khat, w, _, _ = fmm.direction_grid(c.L, c.nphi)
    if ndir is not None:
        khat, w = khat[:ndir], w[:ndir]
    grid = fmm.OperatorGrid(c.Nx, c.Ny, c.Nz, c.edge, c.k, c.L)
    return fmm.fft_operator_4d(grid, khat), w, khat


class Compressed:
    """An oracle-compressed operator, rounded to complex64, with the library
    import arrays and an oracle restore of each slice from the rounded factors."""

    def __init__(self, fmt: str, T4: np.ndarray, tol: float):
        self.fmt = fmt
        n1, n2, n3, nd = T4.shape
        self.n = (n1, n2, n3)
        self.ndir = nd
        if fmt == "dense":
            self.ranks = None
            self.T = f32(T4)
            self.arrays = [flat(np.transpose(self.T, (0, 1, 2, 3)))]   # [p][k][j][i] == F-order of (i,j,k,p)
        elif fmt == "tucker3d":
            fs = [decomp.tucker_svd(T4[..., p], tol) for p in range(nd)]
            self.ranks = np.array([f.ranks for f in fs], dtype=np.int64)
            self.cores = [f32(f.core) for f in fs]
            self.U = [[f32(u) for u in f.factors] for f in fs]
            self.arrays = [np.concatenate([flat(c) for c in self.cores])] + [
                np.concatenate([flat(u[i]) for u in self.U]) for i in range(3)]
        elif fmt == "tt3d":
            fs = [decomp.tt_svd(T4[..., p], tol) for p in range(nd)]
            self.ranks = np.array([f.ranks for f in fs], dtype=np.int64)
            self.parts = [(f32(f.head), f32(f.cores[0]), f32(f.tail)) for f in fs]
            self.arrays = [np.concatenate([flat(pp[i]) for pp in self.parts]) for i in range(3)]
        elif fmt == "tucker4d":
            f = decomp.tucker_svd(T4, tol)
            self.ranks = np.array(f.ranks, dtype=np.int64)
            self.core = f32(f.core)
            self.U = [f32(u) for u in f.factors]
            self.arrays = [flat(self.core)] + [flat(u) for u in self.U]
        elif fmt == "htucker4d":
            h = decomp.htucker_svd(T4, tol)
            self.ranks = np.array(h.ranks, dtype=np.int64)
            self.leaves = [f32(u) for u in h.leaves]
            self.c12, self.c34, self.c1234 = f32(h.c12), f32(h.c34), f32(h.c1234)
            self.arrays = [flat(u) for u in self.leaves] + [flat(self.c12), flat(self.c34), flat(self.c1234)]
        elif fmt == "tt4d":
            g = decomp.tt_svd(T4, tol)
            self.ranks = np.array(g.ranks, dtype=np.int64)
            self.u1, self.c1, self.c2, self.ul = f32(g.head), f32(g.cores[0]), f32(g.cores[1]), f32(g.tail)
            self.arrays = [flat(self.u1), flat(self.c1), flat(self.c2), flat(self.ul)]
            self.t2 = restore.tt4d_t2(self.c2, self.ul)
        else:
            raise ValueError(fmt)

    def restore(self, p: int) -> np.ndarray:
        """Oracle restoration of slice p (Figs. 3-4 chains) from the rounded factors."""
        if self.fmt == "dense":
            return self.T[..., p]
        if self.fmt == "tucker3d":
            u = self.U[p]
            return restore.tucker3d_restore(self.cores[p], u[0], u[1], u[2])
        if self.fmt == "tt3d":
            return restore.tt3d_restore(*self.parts[p])
        if self.fmt == "tucker4d":
            return restore.tucker4d_slice(self.core, self.U, p)
        if self.fmt == "htucker4d":
            return restore.htucker_slice(self.leaves, self.c12, self.c34, self.c1234, p)
        if self.fmt == "tt4d":
            return restore.tt4d_slice(self.u1, self.c1, self.c2, self.ul, p, self.t2)
        raise ValueError(self.fmt)

    def translate(self, sig_math: np.ndarray, p: int) -> np.ndarray:
        """Oracle eq. (5) (FP64 FFT path) for direction p with the restored slice."""
        return translate.translate_fft(self.restore(p), sig_math[p])


def rel(a, b):
    a = np.asarray(a, dtype=np.complex128)
    b = np.asarray(b, dtype=np.complex128)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(a.ravel()), 1e-300))


def t_lib_to_math(buf: np.ndarray, n) -> np.ndarray:
    """Library operator slice layout [k][j][i] -> math (i, j, k)."""
    return np.reshape(np.asarray(buf).ravel(), n, order="F")


class FromArrays:
    """Factors given as the library's flat complex64 arrays (fmmt_op_import order and layout, e.g. from
    fmmt_op_export of a GPU-compressed op), unpacked into the oracle's matrices (complex128 copies of the
    same complex64 values) so that the oracle restores / translates from IDENTICAL factors
    (BASELINE.json north_star: "identical compressed factors").  The GPU compressor itself is checked
    separately against the oracle's T (error bound) and the oracle's ranks."""

    def __init__(self, fmt: str, n, ndir: int, ranks, arrays):
        self.fmt, self.n, self.ndir = fmt, tuple(n), ndir
        n1, n2, n3 = self.n
        a = [np.asarray(x).astype(np.complex128) for x in arrays]
        F = lambda v, shape: np.reshape(v, shape, order="F")
        rk = np.asarray(ranks, dtype=np.int64)
        if fmt == "dense":
            self.T = F(a[0], (n1, n2, n3, ndir))
        elif fmt in ("tucker3d", "tt3d"):
            rk = rk.reshape(ndir, -1)
            self.parts = []
            off = [0] * len(a)
            for p in range(ndir):
                if fmt == "tucker3d":
                    r1, r2, r3 = rk[p]
                    shapes = [(r1, r2, r3), (n1, r1), (n2, r2), (n3, r3)]
                else:
                    r1, r2 = rk[p]
                    shapes = [(n1, r1), (r1, n2, r2), (n3, r2)]
                part = []
                for i, sh in enumerate(shapes):
                    sz = int(np.prod(sh))
                    part.append(F(a[i][off[i]:off[i] + sz], sh))
                    off[i] += sz
                self.parts.append(part)
        elif fmt == "tucker4d":
            r1, r2, r3, r4 = rk
            self.core = F(a[0], (r1, r2, r3, r4))
            self.U = [F(a[1], (n1, r1)), F(a[2], (n2, r2)), F(a[3], (n3, r3)), F(a[4], (ndir, r4))]
        elif fmt == "htucker4d":
            r1, r2, r3, r4, r12, r34 = rk
            self.leaves = [F(a[0], (n1, r1)), F(a[1], (n2, r2)), F(a[2], (n3, r3)), F(a[3], (ndir, r4))]
            self.c12, self.c34, self.c1234 = F(a[4], (r1, r2, r12)), F(a[5], (r3, r4, r34)), F(a[6], (r12, r34))
        elif fmt == "tt4d":
            r1, r2, r3 = rk
            self.u1, self.c1, self.c2, self.ul = (F(a[0], (n1, r1)), F(a[1], (r1, n2, r2)), F(a[2], (r2, n3, r3)),
                                                  F(a[3], (ndir, r3)))
            self.t2 = restore.tt4d_t2(self.c2, self.ul)
        else:
            raise ValueError(fmt)
        self._cache = {}

    def restore(self, p: int) -> np.ndarray:
        if p not in self._cache:
            self._cache[p] = self._restore(p)
        return self._cache[p]

    def _restore(self, p: int) -> np.ndarray:
        if self.fmt == "dense":
            return self.T[..., p]
        if self.fmt == "tucker3d":
            c, u1, u2, u3 = self.parts[p]
            return restore.tucker3d_restore(c, u1, u2, u3)
        if self.fmt == "tt3d":
            return restore.tt3d_restore(*self.parts[p])
        if self.fmt == "tucker4d":
            return restore.tucker4d_slice(self.core, self.U, p)
        if self.fmt == "htucker4d":
            return restore.htucker_slice(self.leaves, self.c12, self.c34, self.c1234, p)
        return restore.tt4d_slice(self.u1, self.c1, self.c2, self.ul, p, self.t2)

    def translate(self, sig_math: np.ndarray, p: int, i: int | None = None) -> np.ndarray:
        """eq. (5) for direction p; sig_math row i (default p)."""
        return translate.translate_fft(self.restore(p), sig_math[p if i is None else i])


def rank_ok(gpu_r, ora_trunc, band=1e-9):
    """Identical integer ranks, except inside the tie band of reading Q18 (oracle margin < band: r or r+1)."""
    for g, tr in zip(gpu_r, ora_trunc):
        if g != tr.rank and not (tr.margin < band and abs(int(g) - tr.rank) == 1):
            return False
    return True


def lib_T(T4: np.ndarray) -> np.ndarray:
    """Oracle T_4D (n1, n2, n3, ndir) -> the library's complex128 [ndir][n3][n2][n1] input layout."""
    return np.ascontiguousarray(np.transpose(T4, (3, 2, 1, 0)))
