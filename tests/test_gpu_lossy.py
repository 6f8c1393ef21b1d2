"""GPU: lossy media (complex wavenumber, Table IV).

The hot path is unchanged; the operator builder takes k = k_re + j k_im.
Checks: the GPU FP64 operator (eq. (7) with complex kR, then FFT) against the
oracle's; GPU compression ranks against the oracle's (Q18 tie rule); the
translate path on oracle-compressed lossy operators against the oracle's eq. (5).
"""
import numpy as np
import pytest

from oracle import decomp, fmm, translate
from synth import signature_seed, signatures

from tests._helpers import rank_ok, Compressed, rel

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def fm():
    from paper_2010_00520_b200 import build
    build.build()
    from paper_2010_00520_b200 import fmmt
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return fmmt


@pytest.fixture(scope="module")
def ctx(fm):
    c = fm.Context(0, torch.cuda.current_stream().cuda_stream)
    yield c
    c.close()


def lossy_setup(eps_r, N=(8, 8, 8), edge=0.5, digits=3, nd=24):
    k = fmm.medium_wavenumber(eps_r)
    L = fmm.multipole_count(abs(k), edge, digits)
    khat, w, _, _ = fmm.direction_grid(L, 2 * (L + 1))
    sel = np.linspace(0, len(khat) - 1, nd).astype(int)
    grid = fmm.OperatorGrid(*N, edge, k, L)
    T4 = np.stack([fmm.fft_operator_3d(grid, khat[p]) for p in sel], axis=-1)
    return k, L, khat[sel], w[sel], T4


@pytest.mark.parametrize("eps_r", [2 - 1j, 2 - 8j])
def test_gpu_lossy_operator_matches_oracle(fm, ctx, eps_r):
    N = (8, 8, 8)
    k, L, khat, _, T4 = lossy_setup(eps_r, N)
    n = tuple(2 * x for x in N)
    T = torch.empty((len(khat),) + n[::-1], dtype=torch.complex128, device="cuda")
    ctx.build_operator_lossy(*N, 0.5, k, L, khat, T)
    ctx.sync()
    got = T.cpu().numpy()
    for p in range(len(khat)):
        # FP64 complex upward recurrence (GPU) vs the terminating series (oracle)
        assert rel(T4[..., p], np.transpose(got[p], (2, 1, 0))) < 1e-9


@pytest.mark.parametrize("fmt", ["tucker3d", "tt3d", "tucker4d"])
def test_gpu_lossy_translate_and_ranks(fm, ctx, fmt):
    N = (8, 8, 8)
    tol = 1e-4
    k, L, khat, w, T4 = lossy_setup(2 - 1j, N)
    nd = T4.shape[-1]
    cp = Compressed(fmt, T4, tol)
    op = ctx.import_op(fmt, cp.n, nd, cp.ranks, cp.arrays)
    sig = signatures(signature_seed(9, 0), nd, *N)
    d_in = torch.from_numpy(sig).cuda()
    d_out = torch.empty_like(d_in)
    op.translate(d_in, d_out, nd, N)
    ctx.sync()
    sm, om = translate.sig_to_math(sig), translate.sig_to_math(d_out.cpu().numpy())
    for p in range(nd):
        assert rel(cp.translate(sm, p), om[p]) <= 1e-5
    op.close()
    # GPU FP64 compression of the same lossy operator: identical ranks (tie band of Q18)
    Td = torch.from_numpy(np.ascontiguousarray(np.transpose(T4, (3, 2, 1, 0)))).cuda()
    gop = ctx.compress(Td, cp.n, nd, fmt, tol)
    gr = gop.ranks()
    # identical integer ranks, up to the tie band of reading Q18 (oracle margin < 1e-9: r or r+1)
    if fmt in ("tucker3d", "tt3d"):
        gr = gr.reshape(nd, -1)
        for p in range(nd):
            o = decomp.tucker_svd(T4[..., p], tol) if fmt == "tucker3d" else decomp.tt_svd(T4[..., p], tol)
            assert rank_ok(gr[p], o.truncations), (p, gr[p], o.ranks)
    else:
        o = decomp.tucker_svd(T4, tol)
        assert rank_ok(gr, o.truncations), (gr, o.ranks)
    gop.close()
