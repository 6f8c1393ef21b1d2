"""Pins for oracle/fmm.py: direction grid, multipole count, special functions,
eq. (7) operator (§II.A).  Each pin is fixed by the paper's printed
integers or by mathematics independent of the code under test."""
import json
import math
import os

import numpy as np
import pytest
from scipy import special

from oracle import fmm, tensor
from synth import config


# ---------------------------------------------------------------- direction grid
@pytest.mark.parametrize("L,nphi", [(1, 3), (12, 26), (14, 29), (20, 42)])
def test_quadrature_closed_forms(L, nphi):
    khat, w, _, _ = fmm.direction_grid(L, nphi)
    assert len(w) == (L + 1) * nphi
    np.testing.assert_allclose(np.linalg.norm(khat, axis=1), 1.0, atol=1e-14)
    assert abs(w.sum() - 4 * np.pi) < 1e-12                      # int dOmega = 4 pi
    assert abs((w * khat[:, 2] ** 2).sum() - 4 * np.pi / 3) < 1e-12  # int cos^2 = 4pi/3
    assert abs((w * khat[:, 0] ** 2).sum() - 4 * np.pi / 3) < 1e-12


def test_quadrature_integrates_spherical_harmonics_exactly():
    """sum_p w_p Y_lm conj(Y_l'm') = delta_ll' delta_mm' for l, l' <= L."""
    L, nphi = 6, 14
    khat, w, _, _ = fmm.direction_grid(L, nphi)
    theta = np.arccos(np.clip(khat[:, 2], -1, 1))
    phi = np.arctan2(khat[:, 1], khat[:, 0])
    ys = []
    for l in range(L + 1):
        for m in range(-l, l + 1):
            ys.append(special.sph_harm_y(l, m, theta, phi))
    Y = np.array(ys)
    G = (Y * w) @ Y.conj().T
    np.testing.assert_allclose(G, np.eye(len(ys)), atol=1e-12)


def test_ndir_paper_integers(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "ndir.json")))
    for case in g["cases"]:
        eps = complex(*case["eps_r"])
        k_abs = abs(2 * np.pi * np.sqrt(eps))
        L = fmm.multipole_count(k_abs, case["edge"], case["digits"])
        assert fmm.ndir_paper(L) == case["ndir"], case["cite"]
    for case in g["baseline_L"]:
        assert fmm.multipole_count(2 * np.pi, case["edge"], case["digits"]) == case["L"]


def test_baseline_configs_direction_counts():
    assert config(2).ndir == 13 * 26 == 338
    assert config(4).ndir == 21 * 42 == 882


# ---------------------------------------------------------------- special functions
def test_hankel_closed_forms():
    z = np.array([0.7, np.pi, 5.3, 11.33, 22.6])
    h0 = 1j * np.exp(-1j * z) / z
    h1 = np.exp(-1j * z) * (1j - z) / z ** 2
    np.testing.assert_allclose(fmm.sph_hankel2(0, z), h0, rtol=1e-14)
    np.testing.assert_allclose(fmm.sph_hankel2(1, z), h1, rtol=1e-13)
    assert abs(fmm.sph_hankel2(0, np.pi) - (-1j / np.pi)) < 1e-15   # SPEC S:375 worked value
    # upward recurrence h_{l+1} = (2l+1)/z h_l - h_{l-1} (textbook identity)
    for l in range(1, 12):
        lhs = fmm.sph_hankel2(l + 1, z)
        rhs = (2 * l + 1) / z * fmm.sph_hankel2(l, z) - fmm.sph_hankel2(l - 1, z)
        np.testing.assert_allclose(lhs, rhs, rtol=1e-11)


def test_legendre_values():
    assert abs(fmm.legendre(2, 0.5) + 0.125) < 1e-15
    for l in range(51):
        assert abs(fmm.legendre(l, 1.0) - 1.0) < 1e-12
    x = 0.3
    coef = np.zeros(8); coef[7] = 1
    assert abs(fmm.legendre(7, x) - np.polynomial.legendre.legval(x, coef)) < 1e-14


# ---------------------------------------------------------------- eq. (7) operator
def _t_scalar(X, khat, k, L):
    R = np.linalg.norm(X)
    c = khat @ (X / R)
    return sum(((-1j) ** l) * (2 * l + 1) * fmm.sph_hankel2(l, k * R) * fmm.legendre(l, c)
               for l in range(L + 1))


@pytest.mark.parametrize("cfg", [2, 4])
def test_green_function_identity_pins_sign_convention(cfg):
    """sum_p w_p e^{-jk k_p.d} T~(X, k_p) = 4 pi h_0^(2)(k|X+d|) (Gegenbauer +
    plane-wave expansion), to the FMM accuracy 10^-digits.  The opposite
    exponent sign fails at O(1), pinning the e^{+j omega t} convention."""
    c = config(cfg)
    khat, w, _, _ = fmm.direction_grid(c.L, c.nphi)
    rng = np.random.default_rng(7)
    worst = 0.0
    for u in [(4, 0, 0), (3, 2, 0), (2, 2, 3), (5, 4, 1)]:
        X = np.array(u, float) * c.edge
        for _ in range(3):
            d = rng.uniform(-0.5, 0.5, 3) * c.edge
            t = _t_scalar(X, khat, c.k, c.L)
            lhs = np.sum(w * np.exp(-1j * c.k * (khat @ d)) * t)
            rhs = 4 * np.pi * 1j * np.exp(-1j * c.k * np.linalg.norm(X + d)) / (c.k * np.linalg.norm(X + d))
            worst = max(worst, abs(lhs - rhs) / abs(rhs))
            bad = np.sum(w * np.exp(+1j * c.k * (khat @ d)) * t)
            assert abs(bad - rhs) / abs(rhs) > 1e-2
    assert worst < 10 * 10.0 ** (-c.digits)


def test_operator_matches_addition_theorem():
    """Eq. (7) vs the independent spherical-harmonic form
    T~ = 4 pi sum_{l,m} (-j)^l h_l(kR) Y_lm(R^) conj(Y_lm(k^))."""
    c = config(1)
    grid = fmm.OperatorGrid(c.Nx, c.Ny, c.Nz, c.edge, c.k, c.L)
    khat, _, _, _ = fmm.direction_grid(c.L, c.nphi)
    p = 57
    T = grid.spatial(khat[p])
    UX, UY, UZ, far = fmm.offset_grid(c.Nx, c.Ny, c.Nz)
    idx = np.argwhere(far)[:12]
    th_k = np.arccos(khat[p, 2]); ph_k = np.arctan2(khat[p, 1], khat[p, 0])
    for (a, b, cc) in idx:
        X = np.array([UX[a, b, cc], UY[a, b, cc], UZ[a, b, cc]], float) * c.edge
        R = np.linalg.norm(X)
        th = np.arccos(X[2] / R); ph = np.arctan2(X[1], X[0])
        v = 0
        for l in range(c.L + 1):
            hl = fmm.sph_hankel2(l, c.k * R)
            for m in range(-l, l + 1):
                v += ((-1j) ** l) * hl * special.sph_harm_y(l, m, th, ph) * np.conj(special.sph_harm_y(l, m, th_k, ph_k))
        v *= 4 * np.pi
        assert abs(T[a, b, cc] - v) <= 1e-10 * abs(v)


def test_near_and_padding_entries_are_zero():
    c = config(1)
    grid = fmm.OperatorGrid(c.Nx, c.Ny, c.Nz, c.edge, c.k, c.L)
    khat, _, _, _ = fmm.direction_grid(c.L, c.nphi)
    T = grid.spatial(khat[3])
    n1 = 2 * c.Nx
    # m = N planes are zero (reading Q6), zero offset and |u|^2 <= 12 are zero
    assert np.all(T[c.Nx, :, :] == 0) and np.all(T[:, c.Ny, :] == 0) and np.all(T[:, :, c.Nz] == 0)
    assert T[0, 0, 0] == 0 and T[2, 2, 2] == 0 and T[n1 - 2, 2, 2] == 0   # |u|^2 = 12 is near
    assert T[3, 2, 0] != 0                                               # |u|^2 = 13 is far
    # brute-force count of far offsets in [-(N-1), N-1]^3
    cnt = sum(1 for x in range(-3, 4) for y in range(-3, 4) for z in range(-3, 4)
              if x * x + y * y + z * z > 12)
    assert np.count_nonzero(T) == cnt == np.count_nonzero(grid.far)


def test_antipodal_symmetry():
    """k_p' = -k_p  =>  T~_p'[m] = T~_p[(-m) mod 2N] and T_p'[f] = T_p[(-f) mod 2N]
    (P_l(-x) = (-1)^l P_l(x), R^ -> -R^)."""
    c = config(1)
    grid = fmm.OperatorGrid(c.Nx, c.Ny, c.Nz, c.edge, c.k, c.L)
    khat, _, _, _ = fmm.direction_grid(c.L, c.nphi)
    nphi = c.nphi
    for p in [0, 5, 100, 200]:
        i, j = divmod(p, nphi)
        q = (c.L - i) * nphi + (j + nphi // 2) % nphi
        np.testing.assert_allclose(khat[q], -khat[p], atol=1e-14)
        a, b = grid.spatial(khat[p]), grid.spatial(khat[q])
        neg = lambda t: np.roll(t[::-1, ::-1, ::-1], 1, axis=(0, 1, 2))
        np.testing.assert_allclose(b, neg(a), atol=1e-12 * np.abs(a).max())
        A, B = fmm.fft3(a), fmm.fft3(b)
        np.testing.assert_allclose(B, neg(A), atol=1e-12 * np.abs(A).max())


def test_fft_preserves_multilinear_spectrum():
    """Normalised mode-i singular values of T = F(T~) equal those of T~ (DFT is
    unitary up to sqrt(n) per mode)."""
    c = config(1)
    grid = fmm.OperatorGrid(c.Nx, c.Ny, c.Nz, c.edge, c.k, c.L)
    khat, _, _, _ = fmm.direction_grid(c.L, c.nphi)
    t = grid.spatial(khat[11]); T = fmm.fft3(t)
    for m in (1, 2, 3):
        s1 = np.linalg.svd(tensor.unfold(t, m), compute_uv=False)
        s2 = np.linalg.svd(tensor.unfold(T, m), compute_uv=False)
        np.testing.assert_allclose(s2 / s2[0], s1 / s1[0], atol=1e-12)


def test_direction_mode_rank_is_L_plus_1_squared():
    """T~(u, k) is a degree-L band-limited function of k, so the mode-4 rank of
    T_4D is (L+1)^2 = 169 at L = 12 (Table II prints r4 = 225 = 15^2 at L = 14)."""
    c = config(2)
    grid = fmm.OperatorGrid(c.Nx, c.Ny, c.Nz, c.edge, c.k, c.L)
    khat, _, _, _ = fmm.direction_grid(c.L, c.nphi)
    # spatial operator suffices (mode-4 rank is invariant under the spatial DFT)
    M = np.stack([grid.spatial(khat[p])[grid.far] for p in range(len(khat))], axis=0)
    s = np.linalg.svd(M, compute_uv=False)
    r = (c.L + 1) ** 2
    assert s[r - 1] / s[0] > 0.1
    assert s[r] / s[0] < 1e-12


# ---------------------------------------------------------------- lossy media
def test_medium_wavenumber_sign_and_lossless_limit():
    """k = k0 sqrt(eps_r), Im k <= 0 for eps_r = eps' - j eps'' (e^{+j omega t}); Table IV media."""
    k = fmm.medium_wavenumber(2 - 1j)
    assert k.imag < 0 and abs(k * k - (2 * np.pi) ** 2 * (2 - 1j)) < 1e-12
    assert abs(fmm.medium_wavenumber(1.0) - 2 * np.pi) < 1e-15
    # h^(2) decays with R in a lossy medium
    assert abs(fmm.sph_hankel2(0, k * 10.0)) < abs(fmm.sph_hankel2(0, k * 5.0)) * np.exp(-4.0)


def test_hankel_complex_argument():
    """Closed forms and the upward recurrence at complex z (lossy kR)."""
    z = np.array([0.7 - 0.1j, np.pi - 0.5j, 5.3 - 1.2j, 11.33 - 2.6j, 22.6 - 5.1j])
    np.testing.assert_allclose(fmm.sph_hankel2(0, z), 1j * np.exp(-1j * z) / z, rtol=1e-11)
    np.testing.assert_allclose(fmm.sph_hankel2(1, z), np.exp(-1j * z) * (1j - z) / z ** 2, rtol=1e-11)
    h = [1j * np.exp(-1j * z) / z, np.exp(-1j * z) * (1j - z) / z ** 2]
    for l in range(1, 20):
        h.append((2 * l + 1) / z * h[l] - h[l - 1])
        np.testing.assert_allclose(fmm.sph_hankel2(l + 1, z), h[l + 1], rtol=1e-9)
    # small losses: the series agrees with SciPy's j_l - i y_l (no cancellation there)
    from scipy import special as sp
    zs = np.array([3.0 - 0.01j, 7.5 - 0.05j, 15.0 - 0.1j])
    for l in range(0, 15):
        np.testing.assert_allclose(fmm.sph_hankel2(l, zs), sp.spherical_jn(l, zs) - 1j * sp.spherical_yn(l, zs),
                                   rtol=1e-10)
    # strong losses: |h_l^(2)(z)| decays like e^{Im z} (no e^{|Im z|} garbage)
    zl = 40.0 - 30.0j
    assert abs(fmm.sph_hankel2(10, zl)) < 10 * np.exp(-30.0)


@pytest.mark.parametrize("eps_r", [2 - 1j, 2 - 2j])
def test_green_function_identity_lossy(eps_r):
    """The plane-wave identity of eq. (5)-(7) with a complex wavenumber:
    sum_p w_p e^{-jk k_p.d} T~(X, k_p) = 4 pi h_0^(2)(k|X+d|), L from |k| (P:63, 5 digits)."""
    k = fmm.medium_wavenumber(eps_r)
    edge, digits = 0.5, 5
    L = fmm.multipole_count(abs(k), edge, digits)
    khat, w, _, _ = fmm.direction_grid(L, 2 * (L + 1))
    rng = np.random.default_rng(11)
    worst = 0.0
    for u in [(4, 0, 0), (3, 2, 0), (2, 2, 3)]:
        X = np.array(u, float) * edge
        for _ in range(3):
            d = rng.uniform(-0.3, 0.3, 3) * edge
            t = _t_scalar(X, khat, k, L)
            lhs = np.sum(w * np.exp(-1j * k * (khat @ d)) * t)
            r = np.linalg.norm(X + d)
            rhs = 4 * np.pi * 1j * np.exp(-1j * k * r) / (k * r)
            worst = max(worst, abs(lhs - rhs) / abs(rhs))
    assert worst < 10 * 10.0 ** (-digits)


def test_lossy_operator_grid_reduces_to_lossless():
    """OperatorGrid with Im k -> 0 equals the real-k operator; lossy FFT'ed operator has
    a lower numerical multilinear rank (Table IV: savings rise with loss)."""
    from oracle import decomp
    c = config(1)
    khat, _, _, _ = fmm.direction_grid(c.L, c.nphi)
    g0 = fmm.OperatorGrid(c.Nx, c.Ny, c.Nz, c.edge, c.k, c.L)
    g1 = fmm.OperatorGrid(c.Nx, c.Ny, c.Nz, c.edge, complex(c.k, -1e-14), c.L)
    assert np.max(np.abs(g0.spatial(khat[5]) - g1.spatial(khat[5]))) < 1e-12
    kl = fmm.medium_wavenumber(2 - 8j)
    gl = fmm.OperatorGrid(8, 8, 8, 0.5, kl, fmm.multipole_count(abs(kl), 0.5, 3))
    kk = fmm.medium_wavenumber(2.0)
    gk = fmm.OperatorGrid(8, 8, 8, 0.5, kk, fmm.multipole_count(abs(kk), 0.5, 3))
    rl = decomp.tucker_svd(fmm.fft_operator_3d(gl, khat[5]), 1e-4).ranks
    rk = decomp.tucker_svd(fmm.fft_operator_3d(gk, khat[5]), 1e-4).ranks
    assert sum(rl) < sum(rk)
