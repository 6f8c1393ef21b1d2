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
