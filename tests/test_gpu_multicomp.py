"""GPU: multi-component signatures.

The aggregated far fields of eq. (4) have a theta and a phi component;
both are translated by the same operator T_p, so one restoration serves both.
fmmt_translate_multi / fmmt_translate_sum_multi take [ndir][ncomp][Nz][Ny][Nx]
signatures.  Checked against the oracle's eq. (5) per component (relative L2
<= 1e-5 per direction and component), the per-component direction sum of
eq. (6), and bitwise against the single-component path.
"""
import numpy as np
import pytest

from oracle import translate
from synth import config, signature_seed, signatures

from tests._helpers import Compressed, operator, rel

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

TOL = 1e-5
ND = 24


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


_CACHE = {}


def comp(fmt, tol):
    if (fmt, tol) not in _CACHE:
        T4, w, _ = operator(2, ND)
        _CACHE[(fmt, tol)] = (Compressed(fmt, T4, tol), w)
    return _CACHE[(fmt, tol)]


@pytest.mark.parametrize("fmt,tol", [("tucker3d", 1e-4), ("tt4d", 1e-4), ("htucker4d", 1e-4), ("tucker4d", 1e-4),
                                     ("tt3d", 1e-4), ("dense", 0.0)])
@pytest.mark.parametrize("ncomp", [2, 3])
def test_multicomponent_matches_oracle(fm, ctx, fmt, tol, ncomp):
    c = config(2)
    cp, w = comp(fmt, tol)
    N = (c.Nx, c.Ny, c.Nz)
    sig = signatures(signature_seed(2, 7), ND * ncomp, *N).reshape(ND, ncomp, c.Nz, c.Ny, c.Nx)
    op = ctx.import_op(fmt, cp.n, cp.ndir, cp.ranks, cp.arrays)
    d_in = torch.from_numpy(np.ascontiguousarray(sig)).cuda()
    d_out = torch.empty_like(d_in)
    op.translate_multi(d_in, d_out, ND, ncomp, N)
    wd = torch.from_numpy(w.astype(np.float32)).cuda()
    d_sum = torch.empty((ncomp, c.Nz, c.Ny, c.Nx), dtype=torch.complex64, device="cuda")
    op.translate_sum_multi(d_in, None, wd, d_sum, ND, ncomp, N)
    # single-component path on component 0 must agree bitwise (same kernels, same arithmetic)
    d0 = torch.from_numpy(np.ascontiguousarray(sig[:, 0])).cuda()
    d0_out = torch.empty_like(d0)
    op.translate(d0, d0_out, ND, N)
    ctx.sync()
    out = d_out.cpu().numpy()
    assert np.array_equal(out[:, 0], d0_out.cpu().numpy())
    sums = np.zeros((ncomp, c.Nx, c.Ny, c.Nz), dtype=np.complex128)
    for k in range(ncomp):
        sm = translate.sig_to_math(np.ascontiguousarray(sig[:, k]))
        om = translate.sig_to_math(np.ascontiguousarray(out[:, k]))
        for p in range(ND):
            ref = cp.translate(sm, p)
            assert rel(ref, om[p]) <= TOL, (k, p)
            sums[k] += w[p] * ref
    got_sum = np.transpose(d_sum.cpu().numpy(), (0, 3, 2, 1))
    for k in range(ncomp):
        assert rel(sums[k], got_sum[k]) <= TOL
    op.close()
