"""Pins for oracle/aggregate.py (eqs. (4) and (6)).

* Point-source pin (physics, independent of the oracle's own arithmetic): with the far-field
  pattern of a point source, P+(k_p, b_n) = exp(+j k k_p.(r_n - r_v)) (eq. (3) for a delta
  basis function, one component), aggregation -> eq. (5) with the dense eq. (7) operator ->
  disaggregation with P- = conj(P+) must reproduce the far part of the free-space interaction
      y_m = sum_{n: box(n) far from box(m)} 4 pi h0^(2)(k |r_m - r_n|) I_n,
  h0^(2)(z) = j e^{-jz}/z, to the FMM accuracy 10^-digits.  The opposite phase convention fails
  at O(1), which pins the sign of eq. (3) against eq. (7).
* Unit current: aggregating I = e_n puts P+[:, n, :] into box(n) only (indexing of box_ptr).
* Adjoint identity between eq. (4) and eq. (6): sum_m I'_m y_m(B) = sum_{p,c,v} w_p B[p,c,v] A'[p,c,v]
  with A' = aggregate(conj(P+), I').
"""
import math

import numpy as np
import pytest

from oracle import aggregate, fmm
from synth import basis, currents, patterns


def _box_xyz(b):
    v = b.box_of
    return np.stack([v % b.Nx, (v // b.Nx) % b.Ny, v // (b.Nx * b.Ny)], axis=1)


def _point_source_case(digits, sign=+1.0):
    Nx = Ny = Nz = 4
    edge, k = 0.5, 2.0 * math.pi
    L = fmm.multipole_count(k, edge, digits)
    khat, w, _, _ = fmm.direction_grid(L, 2 * (L + 1))
    grid = fmm.OperatorGrid(Nx, Ny, Nz, edge, k, L)
    T = [fmm.fft_operator_3d(grid, khat[p]) for p in range(len(khat))]
    b = basis(5, Nx, Ny, Nz, edge, per_box=(2, 4), shell=False)
    I = currents(6, b.N).astype(np.complex128)
    bxyz = _box_xyz(b)
    cen = (bxyz + 0.5) * edge
    P = np.exp(sign * 1j * k * ((b.pos - cen) @ khat.T)).T[:, :, None]      # [p, n, 1]
    y = aggregate.far_matvec(P, I, b.box_ptr, w, lambda p: T[p], Nx, Ny, Nz)
    du = bxyz[:, None, :] - bxyz[None, :, :]
    far = (du ** 2).sum(-1) > 12                                              # P:55, reading Q5
    R = np.linalg.norm(b.pos[:, None, :] - b.pos[None, :, :], axis=-1)
    Rs = np.where(far, R, 1.0)
    G = np.where(far, 4.0 * math.pi * 1j * np.exp(-1j * k * Rs) / (k * Rs), 0.0)
    ref = G @ I
    return np.linalg.norm(y - ref) / np.linalg.norm(ref)


@pytest.mark.parametrize("digits", [3, 4])
def test_point_source_chain_reproduces_green_function(digits):
    assert _point_source_case(digits) <= 10.0 ** (-digits)


def test_point_source_wrong_phase_convention_fails():
    assert _point_source_case(3, sign=-1.0) > 0.1


def test_unit_current_lands_in_its_box():
    b = basis(11, 3, 2, 4, 0.5, per_box=(0, 3), shell=False)
    P = patterns(12, 5, b.N, 2)
    for n in [0, b.N // 2, b.N - 1]:
        I = np.zeros(b.N, dtype=np.complex128)
        I[n] = 1.0
        A = aggregate.aggregate(P, I, b.box_ptr)
        v = int(b.box_of[n])
        assert np.array_equal(A[:, :, v], P[:, n, :].astype(np.complex128))
        A[:, :, v] = 0
        assert not np.any(A)


def test_empty_boxes_aggregate_to_zero():
    b = basis(13, 6, 6, 6, 0.5)                       # sphere shell: interior boxes empty
    empty = np.diff(b.box_ptr) == 0
    assert empty.any() and (~empty).any()
    P = patterns(14, 3, b.N, 2)
    A = aggregate.aggregate(P, currents(15, b.N), b.box_ptr)
    assert not np.any(A[:, :, empty])


def test_disaggregation_is_the_weighted_adjoint_of_aggregation():
    b = basis(21, 3, 3, 3, 0.5, per_box=(1, 4), shell=False)
    ndir = 7
    P = patterns(22, ndir, b.N, 2)
    rng = np.random.default_rng(23)
    B = rng.standard_normal((ndir, 2, b.K)) + 1j * rng.standard_normal((ndir, 2, b.K))
    w = rng.random(ndir)
    Ip = currents(24, b.N).astype(np.complex128)
    y = aggregate.disaggregate(P, B, w, b.box_ptr)
    lhs = np.sum(Ip * y)
    Ap = aggregate.aggregate(np.conj(P), Ip, b.box_ptr)
    rhs = np.sum(w[:, None, None] * B * Ap)
    assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(rhs))
