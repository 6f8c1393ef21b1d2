"""GPU: aggregation (eq. (4)), disaggregation (eq. (6)) and the far-field matvec around the
translation against oracle/aggregate.py.

Synthetic basis functions (synth.basis: sphere-shell box occupancy, 40-70 per non-empty box),
CN(0,1) patterns P+ [ndir][N][2] and coefficients I.  Bars (FP32 accumulation against FP64):
relative L2 <= 1e-5 per direction and component for the aggregated signatures (empty boxes
exactly zero), relative L2 <= 1e-5 for y; far_matvec with identical (exported) compressed
factors <= 1e-5 (the translate bar).
"""
import numpy as np
import pytest

from oracle import aggregate
from synth import basis, basis_seed, config, currents, patterns

from tests._helpers import Compressed, operator, rel

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

TOL = 1e-5


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


def _case(cfg, ndir, ncomp=2, shell=True, per_box=(40, 70)):
    c = config(cfg)
    b = basis(basis_seed(cfg), c.Nx, c.Ny, c.Nz, c.edge, per_box=per_box, shell=shell)
    P = patterns(basis_seed(cfg) + 1, ndir, b.N, ncomp)
    I = currents(basis_seed(cfg) + 2, b.N)
    return c, b, P, I


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("cfg,ndir,ncomp,shell", [(1, 338, 2, True), (1, 17, 1, False), (1, 5, 4, False),
                                                  (2, 24, 2, True), (3, 9, 3, True)])
def test_aggregate_matches_oracle(ctx, cfg, ndir, ncomp, shell):
    _check_aggregate(ctx, *_case(cfg, ndir, ncomp, shell), ndir, ncomp)


@pytest.mark.parametrize("ncomp", [1, 2, 3])
def test_aggregate_large_boxes(ctx, ncomp):
    # boxes of 100-300 basis functions: the kernels' multi-pass paths (128 per pass, 64 per CTA)
    ndir = 21
    _check_aggregate(ctx, *_case(1, ndir, ncomp, shell=False, per_box=(100, 300)), ndir, ncomp)


@pytest.mark.parametrize("ncomp", [2, 3])
def test_disaggregate_large_boxes(ctx, ncomp):
    ndir = 37
    c, b, P, _ = _case(1, ndir, ncomp, shell=False, per_box=(100, 300))
    rng = np.random.default_rng(5)
    B = (rng.standard_normal((ndir, ncomp, b.K)) + 1j * rng.standard_normal((ndir, ncomp, b.K))).astype(np.complex64)
    w = rng.random(ndir).astype(np.float32)
    y = torch.full((b.N,), float("nan"), dtype=torch.complex64, device="cuda")
    ctx.disaggregate(_dev(P), _dev(B), _dev(w), _dev(b.box_ptr), ndir, b.N, ncomp, (c.Nx, c.Ny, c.Nz), y)
    ctx.sync()
    assert rel(aggregate.disaggregate(P, B, w.astype(np.float64), b.box_ptr), y.cpu().numpy()) <= TOL


def _check_aggregate(ctx, c, b, P, I, ndir, ncomp):
    sig = torch.full((ndir, ncomp, c.Nz, c.Ny, c.Nx), float("nan"), dtype=torch.complex64, device="cuda")
    ctx.aggregate(_dev(P), _dev(I), _dev(b.box_ptr), ndir, b.N, ncomp, (c.Nx, c.Ny, c.Nz), sig)
    ctx.sync()
    got = sig.cpu().numpy().reshape(ndir, ncomp, b.K)
    ref = aggregate.aggregate(P, I, b.box_ptr)
    empty = np.diff(b.box_ptr) == 0
    assert np.all(got[:, :, empty] == 0)
    for p in range(ndir):
        for k in range(ncomp):
            assert rel(ref[p, k], got[p, k]) <= TOL, (p, k)


@pytest.mark.parametrize("cfg,ndir,ncomp", [(1, 338, 2), (2, 24, 2), (2, 5, 1), (1, 40, 3), (1, 33, 4)])
def test_disaggregate_matches_oracle(ctx, cfg, ndir, ncomp):
    c, b, P, _ = _case(cfg, ndir, ncomp)
    rng = np.random.default_rng(cfg * 10 + ndir)
    B = (rng.standard_normal((ndir, ncomp, b.K)) + 1j * rng.standard_normal((ndir, ncomp, b.K))).astype(np.complex64)
    w = rng.random(ndir).astype(np.float32)
    y = torch.full((b.N,), float("nan"), dtype=torch.complex64, device="cuda")
    ctx.disaggregate(_dev(P), _dev(B), _dev(w), _dev(b.box_ptr), ndir, b.N, ncomp, (c.Nx, c.Ny, c.Nz), y)
    ctx.sync()
    ref = aggregate.disaggregate(P, B, w.astype(np.float64), b.box_ptr)
    assert rel(ref, y.cpu().numpy()) <= TOL


def test_zero_basis_functions(ctx):
    c = config(1)
    box_ptr = np.zeros(c.K + 1, dtype=np.int64)
    P = np.zeros((3, 1, 2), dtype=np.complex64)          # a dummy device allocation
    sig = torch.full((3, 2, c.Nz, c.Ny, c.Nx), 1.0, dtype=torch.complex64, device="cuda")
    ctx.aggregate(_dev(P), _dev(np.zeros(1, np.complex64)), _dev(box_ptr), 3, 0, 2, (c.Nx, c.Ny, c.Nz), sig)
    ctx.sync()
    assert not torch.any(sig != 0)


_CACHE = {}


@pytest.mark.parametrize("cfg,ndir,fmt,tol", [(1, 338, "dense", 0.0), (1, 338, "tucker3d", 1e-4),
                                              (2, 24, "tt4d", 1e-4), (2, 24, "tucker3d", 1e-6)])
def test_far_matvec_matches_oracle(fm, ctx, cfg, ndir, fmt, tol):
    c, b, P, I = _case(cfg, ndir, 2)
    if (cfg, ndir, fmt, tol) not in _CACHE:
        T4, w, _ = operator(cfg, ndir)
        _CACHE[(cfg, ndir, fmt, tol)] = (Compressed(fmt, T4, tol), w)
    cp, w = _CACHE[(cfg, ndir, fmt, tol)]
    op = ctx.import_op(fmt, cp.n, cp.ndir, cp.ranks, cp.arrays)
    dP, dI, dbox, dw = _dev(P), _dev(I), _dev(b.box_ptr), _dev(w.astype(np.float32))
    y = torch.empty((b.N,), dtype=torch.complex64, device="cuda")
    N = (c.Nx, c.Ny, c.Nz)
    for _ in range(3):                          # direct, capture, replay: the same result each time
        y.fill_(float("nan"))
        op.far_matvec(dP, dI, dbox, dw, ndir, b.N, 2, N, y)
        ctx.sync()
        got = y.cpu().numpy()
        ref = aggregate.far_matvec(P, I, b.box_ptr, w.astype(np.float32).astype(np.float64), cp.restore,
                                   c.Nx, c.Ny, c.Nz)
        assert rel(ref, got) <= TOL
    op.close()
