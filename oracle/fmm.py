"""Oracle: FMM-FFT geometry and the FFT'ed translation operator (§II.A).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  FP64 / complex128.

Array convention: mathematical index order.  A 3D operator slice is a numpy
array T[i1, i2, i3] of shape (n1, n2, n3) = (2Nx, 2Ny, 2Nz); a 4D operator is
T[i1, i2, i3, p] with the direction p as the 4th (slowest) mode.
Flattening to the library's memory layout is `ravel(order="F")` (first index
fastest).
"""
from __future__ import annotations

import math

import numpy as np
from scipy import special

KAPPA = 4  # P:55 "kappa = 4 in this study"


def enclosing_radius(edge: float) -> float:
    """R^s, radius of the sphere enclosing a cubic box of side `edge`."""
    return math.sqrt(3.0) / 2.0 * edge


def multipole_count(k_abs: float, edge: float, digits: float) -> int:
    """L from the excess-bandwidth formula (refs [32,33]).

    Reading: the printed "2 kappa R^s" is 2|k|R^s, and L is the
    floor of  x + 1.8 * digits^(2/3) * x^(1/3),  x = 2|k|R^s.
    """
    x = 2.0 * k_abs * enclosing_radius(edge)
    return int(math.floor(x + 1.8 * digits ** (2.0 / 3.0) * x ** (1.0 / 3.0)))


def ndir_paper(L: int) -> int:
    """N_dir = (L+1)(2L+1)."""
    return (L + 1) * (2 * L + 1)


def direction_grid(L: int, nphi: int | None = None):
    """Plane-wave directions k_p and quadrature weights w_p.

    Cartesian product of the L+1 Gauss-Legendre nodes in cos(theta) (ascending
    cos theta) and nphi uniform azimuths phi_j = 2 pi j / nphi.  Order
    p = i*nphi + j (theta outer).  w_p = w_GL,i * 2 pi / nphi.
    Paper grid: nphi = 2L+1; BASELINE configs: nphi = 2(L+1).

    Returns (khat [ndir,3], w [ndir], cos_theta [L+1], phi [nphi]).
    """
    if nphi is None:
        nphi = 2 * L + 1
    mu, wgl = np.polynomial.legendre.leggauss(L + 1)   # ascending nodes in [-1, 1]
    phi = 2.0 * np.pi * np.arange(nphi) / nphi
    sin_t = np.sqrt(1.0 - mu ** 2)
    kx = (sin_t[:, None] * np.cos(phi)[None, :]).ravel()
    ky = (sin_t[:, None] * np.sin(phi)[None, :]).ravel()
    kz = np.repeat(mu, nphi)
    khat = np.stack([kx, ky, kz], axis=1)
    w = np.repeat(wgl, nphi) * (2.0 * np.pi / nphi)
    return khat, w, mu, phi


def circulant_offsets(N: int):
    """Box offset u of circulant index m in [0, 2N).

    u = m for m < N, u = m - 2N for m > N; the m = N plane carries no offset
    (reading Q6: it is set to zero; it never reaches the truncated output).
    Returns (u [2N] int, valid [2N] bool).
    """
    m = np.arange(2 * N)
    u = np.where(m < N, m, m - 2 * N)
    valid = m != N
    return u, valid


def offset_grid(Nx: int, Ny: int, Nz: int):
    """Integer offsets (ux, uy, uz) on the padded grid and the far-field mask.

    Far iff R > kappa R^s, i.e. |u|^2 > 12 in integers because
    kappa R^s = 2 sqrt(3) edge; ties (|u|^2 = 12) are near (reading Q5).
    """
    ux, vx = circulant_offsets(Nx)
    uy, vy = circulant_offsets(Ny)
    uz, vz = circulant_offsets(Nz)
    UX, UY, UZ = np.meshgrid(ux, uy, uz, indexing="ij")
    V = vx[:, None, None] & vy[None, :, None] & vz[None, None, :]
    u2 = UX * UX + UY * UY + UZ * UZ
    far = V & (u2 > 12)
    return UX, UY, UZ, far


def sph_hankel2(l: int, z):
    """Spherical Hankel function of the second kind h_l^(2)(z) = j_l(z) - i y_l(z)
    (P:77).  e^{+j omega t} convention: h_0^(2)(z) = j e^{-jz} / z.

    Real z: SciPy's spherical Bessel functions (library primitive).
    Complex z (lossy media): the textbook terminating series
        h_l^(2)(z) = j^{l+1} e^{-jz}/z  sum_{k=0}^{l} (l+k)! / (k! (l-k)!) (-j / (2z))^k,
    which stays accurate when |Im z| is large (j_l and y_l then grow like
    e^{|Im z|} and their difference h^(2) cancels catastrophically)."""
    z = np.asarray(z)
    if not np.iscomplexobj(z) or not np.any(np.imag(z) != 0):
        return special.spherical_jn(l, np.real(z) if not np.iscomplexobj(z) else z) - 1j * special.spherical_yn(
            l, np.real(z) if not np.iscomplexobj(z) else z)
    acc = np.zeros(z.shape, dtype=np.complex128)
    for k in range(l + 1):
        coef = math.factorial(l + k) / (math.factorial(k) * math.factorial(l - k))
        acc = acc + coef * (-1j / (2.0 * z)) ** k
    return (1j ** (l + 1)) * np.exp(-1j * z) / z * acc


def legendre(l: int, x):
    """Legendre polynomial Phi_l(x), SciPy library primitive."""
    return special.eval_legendre(l, x)


def medium_wavenumber(eps_r: complex, k0: float = 2.0 * math.pi) -> complex:
    """k = k0 sqrt(eps_r) of a (lossy) medium, e^{+j omega t} convention: eps_r = eps' - j eps''
    gives Im k <= 0, so h_l^(2)(kR) ~ e^{-jkR} decays with R (Table IV)."""
    k = k0 * np.sqrt(complex(eps_r))
    return complex(k.real, -abs(k.imag))


class OperatorGrid:
    """Direction-independent part of eq. (7) on the circulant grid:
    R = edge*|u|, R_hat, far mask, and h_l^(2)(kR) for l = 0..L.
    k may be complex (lossy medium); L is then chosen from |k|."""

    def __init__(self, Nx, Ny, Nz, edge, k, L):
        self.Nx, self.Ny, self.Nz = int(Nx), int(Ny), int(Nz)
        self.edge, self.L = float(edge), int(L)
        kc = complex(k)
        self.k = kc.real if kc.imag == 0 else kc
        UX, UY, UZ, far = offset_grid(self.Nx, self.Ny, self.Nz)
        self.shape = far.shape
        self.far = far
        ux = UX[far].astype(np.float64)
        uy = UY[far].astype(np.float64)
        uz = UZ[far].astype(np.float64)
        rn = np.sqrt(ux * ux + uy * uy + uz * uz)
        self.R = edge * rn
        self.Rhat = np.stack([ux / rn, uy / rn, uz / rn], axis=1)
        kR = k * self.R
        # (-j)^l (2l+1) h_l^(2)(kR), l = 0..L  -- the radial factor of eq. (7)
        self.radial = np.stack([((-1j) ** l) * (2 * l + 1) * sph_hankel2(l, kR)
                                for l in range(self.L + 1)], axis=0)

    def spatial(self, khat_p) -> np.ndarray:
        """T~(k_p) on the padded circulant grid, eq. (7) with l = 0..L (reading
        Q1) and the prefactor -k^2 eta / 16 pi^2 omitted (reading Q2):
            T~[u] = sum_{l=0}^{L} (-j)^l (2l+1) Phi_l(R_hat . k_p) h_l^(2)(k R),
        zero for near offsets and on the m = N planes.  Shape (n1, n2, n3)."""
        c = self.Rhat @ np.asarray(khat_p, dtype=np.float64)
        acc = np.zeros(c.shape, dtype=np.complex128)
        for l in range(self.L + 1):
            acc += self.radial[l] * legendre(l, c)
        out = np.zeros(self.shape, dtype=np.complex128)
        out[self.far] = acc
        return out


def fft3(t: np.ndarray) -> np.ndarray:
    """Unnormalised forward 3D DFT, kernel e^{-j 2 pi m f / n}."""
    return np.fft.fftn(t, axes=(0, 1, 2))


def ifft3(t: np.ndarray) -> np.ndarray:
    """Inverse 3D DFT with 1/n scaling."""
    return np.fft.ifftn(t, axes=(0, 1, 2))


def fft_operator_3d(grid: OperatorGrid, khat_p) -> np.ndarray:
    """T_3D for one direction: T = F(T~)."""
    return fft3(grid.spatial(khat_p))


def fft_operator_4d(grid: OperatorGrid, khat) -> np.ndarray:
    """T_4D = stack over directions of T_3D, direction as mode 4."""
    n1, n2, n3 = grid.shape
    out = np.empty((n1, n2, n3, len(khat)), dtype=np.complex128)
    for p in range(len(khat)):
        out[..., p] = fft_operator_3d(grid, khat[p])
    return out
