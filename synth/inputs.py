"""Workload configurations and seeded signatures (no method arithmetic here).

Configurations are BASELINE.json `configs[0..4]` (numbered 1..5 as in
SURVEY.md §8).  Each is a box grid Nx x Ny x Nz (padded operator grid
2Nx x 2Ny x 2Nz), a box edge in wavelengths (lambda = 1,
so k = 2*pi, free space), the multipole count L and the
direction grid (L+1) Gauss-Legendre theta x nphi phi (nphi = 2(L+1) in the
BASELINE configs; the paper's own grid uses 2L+1).

Signatures: complex64 A_p[v], layout [ndir][Nz][Ny][Nx] (x fastest), real and
imaginary parts i.i.d. N(0, 1/2) so E|A|^2 = 1, drawn from
numpy PCG64(seed) with seed = 2010_00520 + 1000*config + matvec_index
(SURVEY.md §8(d)).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

SEED_BASE = 2010_00520


@dataclasses.dataclass(frozen=True)
class Config:
    index: int
    Nx: int
    Ny: int
    Nz: int
    edge: float          # box edge in wavelengths
    L: int               # multipole count (stated by BASELINE.json)
    digits: int          # FMM accuracy digits used to state L
    nphi: int            # azimuth samples
    formats: tuple       # (format name, tol) pairs BASELINE.json lists
    ndir: int = 0

    @property
    def k(self) -> float:
        return 2.0 * math.pi          # lambda = 1 (300 MHz, free space)

    @property
    def ntheta(self) -> int:
        return self.L + 1

    @property
    def n(self) -> tuple:
        return (2 * self.Nx, 2 * self.Ny, 2 * self.Nz)

    @property
    def K(self) -> int:
        return self.Nx * self.Ny * self.Nz

    @property
    def npad(self) -> int:
        return 8 * self.K


def _mk(index, Nx, Ny, Nz, edge, L, digits, formats):
    nphi = 2 * (L + 1)
    return Config(index, Nx, Ny, Nz, edge, L, digits, nphi, tuple(formats),
                  ndir=(L + 1) * nphi)


_ALL5 = ("tucker3d", "tucker4d", "htucker4d", "tt3d", "tt4d")

CONFIGS = {
    1: _mk(1, 4, 4, 4, 0.5, 12, 3, [("tucker3d", 1e-4)]),
    2: _mk(2, 16, 16, 16, 0.5, 12, 3,
           [(f, t) for t in (1e-4, 1e-6) for f in _ALL5]),
    3: _mk(3, 128, 8, 8, 0.5, 12, 3, [("tucker3d", 1e-5), ("tt3d", 1e-5)]),
    4: _mk(4, 32, 32, 32, 1.0, 20, 4, [("tucker4d", 1e-4), ("htucker4d", 1e-4)]),
    5: _mk(5, 64, 64, 32, 1.0, 20, 4, [("tt4d", 1e-4), ("tucker3d", 1e-4)]),
}


def config(i: int) -> Config:
    return CONFIGS[int(i)]


def signature_seed(config_index: int, matvec: int = 0) -> int:
    return SEED_BASE + 1000 * int(config_index) + int(matvec)


def weights_seed(config_index: int) -> int:
    return SEED_BASE + 1000 * int(config_index) + 999


def signatures(seed: int, ndir: int, Nx: int, Ny: int, Nz: int) -> np.ndarray:
    """CN(0,1) complex64 array of shape (ndir, Nz, Ny, Nx) (C order => x fastest)."""
    rng = np.random.Generator(np.random.PCG64(int(seed)))
    shape = (int(ndir), int(Nz), int(Ny), int(Nx))
    re = rng.standard_normal(shape, dtype=np.float32)
    im = rng.standard_normal(shape, dtype=np.float32)
    s = np.float32(math.sqrt(0.5))
    out = np.empty(shape, dtype=np.complex64)
    out.real = re * s
    out.imag = im * s
    return out


# ---------------------------------------------------------------- basis functions
def basis_seed(config_index: int) -> int:
    return SEED_BASE + 1000 * int(config_index) + 777


@dataclasses.dataclass(frozen=True)
class Basis:
    """Synthetic stand-in for the RWG basis functions of P:41-61 around the translation stage.

    Boxes hold basis functions only where a sphere's surface crosses them (the paper's sphere
    workloads): box v (linear index x + Nx (y + Ny z), x fastest) is non-empty iff its
    centre lies within edge*sqrt(3)/2 of the sphere of diameter min(Nx,Ny,Nz)*edge - edge inscribed
    in the box grid.  A non-empty box holds between `per_box[0]` and `per_box[1]` basis functions
    (uniform draw; the paper's 32 lambda sphere averages ~55 RWG functions per non-empty 0.5 lambda
    box).  Basis functions are numbered box by box: box v holds [box_ptr[v], box_ptr[v+1]).
    `pos` are points in the box (for the point-source pin), in wavelengths, box v spanning
    [v*edge, (v+1)*edge) per axis."""
    Nx: int
    Ny: int
    Nz: int
    edge: float
    box_ptr: np.ndarray      # int64 [K+1]
    box_of: np.ndarray       # int64 [N]: linear box index of each basis function
    pos: np.ndarray          # float64 [N, 3]

    @property
    def N(self) -> int:
        return int(self.box_ptr[-1])

    @property
    def K(self) -> int:
        return self.Nx * self.Ny * self.Nz


def basis(seed: int, Nx: int, Ny: int, Nz: int, edge: float, per_box=(40, 70), shell=True) -> Basis:
    rng = np.random.Generator(np.random.PCG64(int(seed)))
    z, y, x = np.meshgrid(np.arange(Nz), np.arange(Ny), np.arange(Nx), indexing="ij")
    cx, cy, cz = (x.ravel() + 0.5) * edge, (y.ravel() + 0.5) * edge, (z.ravel() + 0.5) * edge
    if shell:
        c0 = np.array([Nx, Ny, Nz], dtype=np.float64) * edge / 2.0
        radius = (min(Nx, Ny, Nz) - 1) * edge / 2.0
        dist = np.sqrt((cx - c0[0]) ** 2 + (cy - c0[1]) ** 2 + (cz - c0[2]) ** 2)
        occupied = np.abs(dist - radius) <= edge * math.sqrt(3.0) / 2.0
    else:
        occupied = np.ones(cx.shape, dtype=bool)
    counts = np.where(occupied, rng.integers(per_box[0], per_box[1] + 1, size=cx.shape), 0).astype(np.int64)
    box_ptr = np.zeros(len(counts) + 1, dtype=np.int64)
    np.cumsum(counts, out=box_ptr[1:])
    box_of = np.repeat(np.arange(len(counts), dtype=np.int64), counts)
    lo = np.stack([x.ravel(), y.ravel(), z.ravel()], axis=1)[box_of] * edge
    pos = lo + rng.random((len(box_of), 3)) * edge
    return Basis(int(Nx), int(Ny), int(Nz), float(edge), box_ptr, box_of, pos)


def patterns(seed: int, ndir: int, nbasis: int, ncomp: int = 2) -> np.ndarray:
    """Synthetic far-field patterns P+[p][n][c] (theta, phi components), complex64
    CN(0,1), layout [ndir][N][ncomp] (c fastest)."""
    rng = np.random.Generator(np.random.PCG64(int(seed)))
    shape = (int(ndir), int(nbasis), int(ncomp))
    s = np.float32(math.sqrt(0.5))
    out = np.empty(shape, dtype=np.complex64)
    out.real = rng.standard_normal(shape, dtype=np.float32) * s
    out.imag = rng.standard_normal(shape, dtype=np.float32) * s
    return out


def currents(seed: int, nbasis: int) -> np.ndarray:
    """Synthetic basis-function coefficients I_n, complex64 CN(0,1)."""
    rng = np.random.Generator(np.random.PCG64(int(seed)))
    s = np.float32(math.sqrt(0.5))
    out = np.empty(int(nbasis), dtype=np.complex64)
    out.real = rng.standard_normal(int(nbasis), dtype=np.float32) * s
    out.imag = rng.standard_normal(int(nbasis), dtype=np.float32) * s
    return out
