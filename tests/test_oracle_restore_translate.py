"""Pins for oracle/restore.py, oracle/translate.py, oracle/memory.py.

Restoration: slice chains of Figs. 3-4 vs the dense equations for every p
(brute force), identity / rank-1 cases.  Translation: the FFT path vs the
O(N^2) circular direct sum, delta kernel, linearity, Parseval, the m = N plane
invariance.  Memory: the rank formulas vs the actual array sizes."""
import numpy as np
import pytest

from oracle import decomp, fmm, memory, restore, tensor, translate
from synth import config, signatures

RNG = np.random.default_rng(520)


def crand(*shape):
    return RNG.standard_normal(shape) + 1j * RNG.standard_normal(shape)


# ---------------------------------------------------------------- restoration
def test_tucker4d_slice_vs_dense_all_p():
    core = crand(3, 2, 4, 5)
    fac = [crand(6, 3), crand(5, 2), crand(7, 4), crand(9, 5)]
    dense = restore.tucker_full(core, fac)
    for p in range(9):
        np.testing.assert_allclose(restore.tucker4d_slice(core, fac, p), dense[..., p],
                                   rtol=0, atol=1e-12 * np.abs(dense).max())


def test_htucker_slice_vs_dense_all_p():
    leaves = [crand(6, 3), crand(5, 2), crand(4, 3), crand(8, 4)]
    c12, c34, root = crand(3, 2, 5), crand(3, 4, 6), crand(5, 6)
    dense = restore.htucker_full(leaves, c12, c34, root)
    # explicit quadruple sum of eq. (11)'s bracket
    core = np.zeros((3, 2, 3, 4), complex)
    for a, b, c, d in np.ndindex(*core.shape):
        core[a, b, c, d] = sum(c12[a, b, i] * root[i, j] * c34[c, d, j]
                               for i in range(5) for j in range(6))
    np.testing.assert_allclose(restore.htucker_core(c12, c34, root), core, rtol=1e-12)
    for p in range(8):
        np.testing.assert_allclose(restore.htucker_slice(leaves, c12, c34, root, p), dense[..., p],
                                   rtol=0, atol=1e-12 * np.abs(dense).max())


def test_tt_chains_vs_dense():
    u1, c1, u3 = crand(5, 3), crand(3, 6, 4), crand(7, 4)
    dense = np.einsum("ia,ajb,kb->ijk", u1, c1, u3)
    np.testing.assert_allclose(restore.tt3d_full(u1, c1, u3), dense, rtol=1e-12)
    np.testing.assert_allclose(restore.tt3d_restore(u1, c1, u3), dense, rtol=1e-12)
    c2, u4 = crand(4, 7, 5), crand(9, 5)
    d4 = restore.tt4d_full(u1, c1, c2, u4)
    ref = np.einsum("ia,ajb,bkc,pc->ijkp", u1, c1, c2, u4)
    np.testing.assert_allclose(d4, ref, rtol=1e-12)
    for p in range(9):
        np.testing.assert_allclose(restore.tt4d_slice(u1, c1, c2, u4, p), d4[..., p],
                                   rtol=0, atol=1e-12 * np.abs(d4).max())


def test_identity_and_rank1_restorations():
    t = crand(4, 5, 3)
    assert np.array_equal(restore.tucker3d_restore(t, np.eye(4), np.eye(5), np.eye(3)), t)
    a, b, c = crand(4, 1), crand(5, 1), crand(3, 1)
    core = np.full((1, 1, 1), 2.0 + 0j)
    ref = 2.0 * np.einsum("i,j,k->ijk", a[:, 0], b[:, 0], c[:, 0])
    np.testing.assert_allclose(restore.tucker3d_restore(core, a, b, c), ref, rtol=1e-14)


# ---------------------------------------------------------------- translation
@pytest.mark.parametrize("N", [(2, 2, 2), (3, 3, 3), (4, 3, 2)])
def test_fft_path_equals_direct_sum_tiny(N):
    n = tuple(2 * x for x in N)
    T = crand(*n)
    A = crand(*N)
    b_fft = translate.translate_fft(T, A)
    b_dir = translate.translate_direct(translate.spatial_kernel(T), A)
    np.testing.assert_allclose(b_fft, b_dir, rtol=0, atol=1e-12 * np.abs(b_dir).max())


def test_fft_path_equals_direct_sum_config1():
    c = config(1)
    grid = fmm.OperatorGrid(c.Nx, c.Ny, c.Nz, c.edge, c.k, c.L)
    khat, w, _, _ = fmm.direction_grid(c.L, c.nphi)
    sig = translate.sig_to_math(signatures(1, 4, c.Nx, c.Ny, c.Nz))
    for q, p in enumerate([0, 101, 202, 337]):
        t = grid.spatial(khat[p])
        b_dir = translate.translate_direct(t, sig[q])           # exact spatial operator
        b_fft = translate.translate_fft(fmm.fft3(t), sig[q])
        assert tensor.rel_err(b_dir, b_fft) < 1e-13


def test_delta_kernel_and_linearity():
    N = (3, 4, 2)
    n = tuple(2 * x for x in N)
    A, A2 = crand(*N), crand(*N)
    np.testing.assert_allclose(translate.translate_fft(np.ones(n, complex), A), A, atol=1e-13)
    T = crand(*n)
    np.testing.assert_allclose(translate.translate_fft(T, A + 2j * A2),
                               translate.translate_fft(T, A) + 2j * translate.translate_fft(T, A2),
                               atol=1e-12 * np.abs(T).max())


def test_parseval_and_roundtrip():
    t = crand(8, 8, 8)
    T = fmm.fft3(t)
    assert abs(np.sum(np.abs(T) ** 2) - t.size * np.sum(np.abs(t) ** 2)) < 1e-9 * t.size * np.sum(np.abs(t) ** 2)
    np.testing.assert_allclose(fmm.ifft3(T), t, atol=1e-13)
    d = np.zeros((4, 4, 4), complex); d[0, 0, 0] = 1
    np.testing.assert_allclose(fmm.fft3(d), np.ones((4, 4, 4)), atol=0)


def test_m_equals_N_plane_never_reaches_output():
    N = (3, 3, 3)
    n = (6, 6, 6)
    t = crand(*n)
    A = crand(*N)
    b0 = translate.translate_direct(t, A)
    t2 = t.copy(); t2[3, :, :] = 99.0; t2[:, 3, :] = -7j; t2[:, :, 3] = 5.0
    np.testing.assert_allclose(translate.translate_direct(t2, A), b0, atol=1e-12)
    np.testing.assert_allclose(translate.translate_fft(fmm.fft3(t2), A), b0, atol=1e-11)


def test_direction_sum_shards():
    b = crand(10, 2, 3, 2)
    w = RNG.uniform(0, 1, 10)
    full = translate.direction_sum(b, w)
    part = translate.direction_sum(b[:4], w[:4]) + translate.direction_sum(b[4:], w[4:])
    np.testing.assert_allclose(part, full, atol=1e-13)
    ref = sum(w[p] * b[p] for p in range(10))
    np.testing.assert_allclose(full, ref, atol=1e-13)


def test_sig_layout_roundtrip():
    s = signatures(3, 2, 3, 4, 5)
    m = translate.sig_to_math(s)
    assert m.shape == (2, 3, 4, 5)
    assert m[1, 2, 3, 4] == s[1, 4, 3, 2]
    assert np.array_equal(translate.math_to_sig(m).astype(np.complex64), s)


def test_signature_statistics():
    s = signatures(2010_00520, 64, 8, 8, 8)
    assert s.dtype == np.complex64 and s.shape == (64, 8, 8, 8)
    assert abs(np.mean(np.abs(s) ** 2) - 1.0) < 0.02
    assert abs(np.mean(s.real * s.imag)) < 0.01
    assert np.array_equal(s, signatures(2010_00520, 64, 8, 8, 8))


# ---------------------------------------------------------------- memory count
def test_memory_counts_match_array_sizes():
    c = config(1)
    grid = fmm.OperatorGrid(c.Nx, c.Ny, c.Nz, c.edge, c.k, c.L)
    khat, _, _, _ = fmm.direction_grid(c.L, c.nphi)
    T4 = fmm.fft_operator_4d(grid, khat[:40])
    n = T4.shape[:3]
    tk = [decomp.tucker_svd(T4[..., p], 1e-4) for p in range(40)]
    assert memory.tucker3d_elems(n, [f.ranks for f in tk]) == sum(
        f.core.size + sum(u.size for u in f.factors) for f in tk)
    tt = [decomp.tt_svd(T4[..., p], 1e-4) for p in range(40)]
    assert memory.tt3d_elems(n, [g.ranks for g in tt]) == sum(
        g.head.size + g.cores[0].size + g.tail.size for g in tt)
    f4 = decomp.tucker_svd(T4, 1e-4)
    assert memory.tucker4d_elems(n, 40, f4.ranks) == f4.core.size + sum(u.size for u in f4.factors)
    h = decomp.htucker_svd(T4, 1e-4)
    assert memory.htucker_elems(n, 40, h.ranks) == (sum(u.size for u in h.leaves) + h.c12.size
                                                    + h.c34.size + h.c1234.size)
    g4 = decomp.tt_svd(T4, 1e-4)
    assert memory.tt4d_elems(n, 40, g4.ranks) == (g4.head.size + g4.cores[0].size
                                                  + g4.cores[1].size + g4.tail.size)
    # SPEC S:178 worked example: 2x2x2 core + three 4x2 factors = 32 elements
    assert memory.tucker3d_elems((4, 4, 4), [(2, 2, 2)]) == 32
    assert memory.saving_percent(1, 4) == 75.0
