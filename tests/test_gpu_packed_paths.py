"""GPU: the pre-split operand paths of the tensor-core kernels against the oracle.

* TT-4D at n3 = 64 (k_tc_conv_z64: V_q pre-split per parity pass) with two signature components;
* the same operators with the pre-split B disabled (FMMT_PACKB=0, the per-thread conversion path), which
  must agree with the oracle too;
* 4D formats re-planned into several batches (fmmt_op_set_batch): per-batch M_q / V_q pre-splits, static
  slice-operand pre-splits per batch.
Bar: the translate bar, relative L2 <= 1e-5 per direction and component (BASELINE north_star).
"""
import math
import os

import numpy as np
import pytest

from oracle import fmm, translate
from synth import signatures

from tests._helpers import Compressed, operator, rel, t_lib_to_math

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


def _ctx(fm, packb: bool):
    old = os.environ.get("FMMT_PACKB")
    os.environ["FMMT_PACKB"] = "1" if packb else "0"
    try:
        return fm.Context(0, torch.cuda.current_stream().cuda_stream)   # the variable is read at creation
    finally:
        if old is None:
            del os.environ["FMMT_PACKB"]
        else:
            os.environ["FMMT_PACKB"] = old


_OPS = {}


def _n64_operator(fmt, tol, nd=20, nxy=4):
    """A small n3 = 64 grid (nxy x nxy x 32 boxes, edge 0.5, L = 12): the z-stage takes the two-pass path."""
    key = (fmt, tol, nd, nxy)
    if key not in _OPS:
        k = 2 * math.pi
        khat, w, _, _ = fmm.direction_grid(12, 26)
        khat, w = khat[:nd], w[:nd]
        grid = fmm.OperatorGrid(nxy, nxy, 32, 0.5, k, 12)
        _OPS[key] = (Compressed(fmt, fmm.fft_operator_4d(grid, khat), tol), w)
    return _OPS[key]


def _check_multi(ctx, cp, N, ncomp, seed):
    nd = cp.ndir
    sig = signatures(seed, nd * ncomp, *N).reshape(nd, ncomp, N[2], N[1], N[0])
    op = ctx.import_op(cp.fmt, cp.n, nd, cp.ranks, cp.arrays)
    d_in = torch.from_numpy(np.ascontiguousarray(sig)).cuda()
    d_out = torch.empty_like(d_in)
    op.translate_multi(d_in, d_out, nd, ncomp, N)
    ctx.sync()
    out = d_out.cpu().numpy()
    op.close()
    for c in range(ncomp):
        sm = translate.sig_to_math(np.ascontiguousarray(sig[:, c]))
        om = translate.sig_to_math(np.ascontiguousarray(out[:, c]))
        for p in range(nd):
            assert rel(cp.translate(sm, p), om[p]) <= TOL, (c, p)
    return out


@pytest.mark.parametrize("packb", [True, False])
@pytest.mark.parametrize("ncomp", [1, 2])
def test_tt4d_n3_64_matches_oracle(fm, packb, ncomp):
    cp, _ = _n64_operator("tt4d", 1e-4)
    ctx = _ctx(fm, packb)
    _check_multi(ctx, cp, (4, 4, 32), ncomp, 90 + ncomp)
    ctx.close()


def test_packed_and_unpacked_paths_agree(fm):
    cp, _ = _n64_operator("tt4d", 1e-4)
    outs = []
    for packb in (True, False):
        ctx = _ctx(fm, packb)
        outs.append(_check_multi(ctx, cp, (4, 4, 32), 2, 97))
        ctx.close()
    # same arithmetic (the pre-split is the split the threads do): identical up to FP32 summation order
    assert rel(outs[0], outs[1]) <= 1e-6


@pytest.mark.parametrize("fmt", ["tt4d", "htucker4d", "tucker4d"])
def test_several_batches_match_oracle(fm, fmt):
    nd = 24
    T4, _, _ = operator(2, nd)
    cp = Compressed(fmt, T4, 1e-4)
    ctx = _ctx(fm, True)
    op = ctx.import_op(fmt, cp.n, nd, cp.ranks, cp.arrays)
    op.set_batch(7)                                  # 4 batches of 7, 7, 7, 3 directions
    N = (16, 16, 16)
    sig = signatures(123, nd, *N)
    d_in = torch.from_numpy(sig).cuda()
    d_out = torch.empty_like(d_in)
    for _ in range(3):                               # direct, graph capture, replay
        d_out.fill_(float("nan"))
        op.translate(d_in, d_out, nd, N)
        ctx.sync()
        sm, om = translate.sig_to_math(sig), translate.sig_to_math(d_out.cpu().numpy())
        for p in range(nd):
            assert rel(cp.translate(sm, p), om[p]) <= TOL, p
    op.close()
    ctx.close()


def _ctx_env(fm, **env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: str(v) for k, v in env.items()})
    try:
        return fm.Context(0, torch.cuda.current_stream().cuda_stream)
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


@pytest.mark.parametrize("nxy", [4, 8])
@pytest.mark.parametrize("ncomp", [1, 3])
@pytest.mark.parametrize("fmt", ["tucker3d", "tt3d", "tucker4d", "htucker4d"])
def test_n3_64_per_direction_a_matches_oracle(fm, fmt, ncomp, nxy):
    """n3 = 64 z-stage with a per-direction A operand (k_pk_conv_z64, CL = 1): a partial m-tile (8 x 8 lines,
    nxy = 4) and two full m-tiles (16 x 16, nxy = 8), one and three signature components."""
    cp, _ = _n64_operator(fmt, 1e-4, nd=12, nxy=nxy)
    ctx = _ctx_env(fm)
    _check_multi(ctx, cp, (nxy, nxy, 32), ncomp, 300 + ncomp + nxy)
    ctx.close()


@pytest.mark.parametrize("fc", [4, 8, 16])
def test_tt4d_flush_group_lengths_agree(fm, fc):
    """TT-4D n3 = 64 z-stage with TMEM flush groups of 4, 8 and 16 K-chunks (FMMT_ZFC; 8 is the default for
    the shared-A stage): all match the oracle at the translate bar."""
    cp, _ = _n64_operator("tt4d", 1e-4)
    ctx = _ctx_env(fm, FMMT_ZFC=fc)
    _check_multi(ctx, cp, (4, 4, 32), 2, 500 + fc)
    ctx.close()


def _fused_operator(nx, nd=10):
    """Tucker-3D of a grid with n1 = 2 nx >= 128 and n3 = 64 (nx x 2 x 32 boxes): the fused mode-1 / mode-3
    z-stage (kernels_tcfuse.cuh) takes it."""
    key = ("fused", nx, nd)
    if key not in _OPS:
        khat, w, _, _ = fmm.direction_grid(12, 26)
        grid = fmm.OperatorGrid(nx, 2, 32, 0.5, 2 * math.pi, 12)
        _OPS[key] = (Compressed("tucker3d", fmm.fft_operator_4d(grid, khat[:nd]), 1e-4), w[:nd])
    return _OPS[key]


@pytest.mark.parametrize("nx", [64, 128])
@pytest.mark.parametrize("ncomp", [1, 2])
def test_tucker3d_fused_chain_matches_oracle(fm, nx, ncomp):
    """Fused Tucker-3D chain (restore_mode2x + k_tucker_zf: G in TMEM / shared memory only) with one and two
    i-blocks per y index (n1 = 128, 256), one and two components: translate vs the oracle, restore vs the
    oracle's restoration, and the unfused chain (FMMT_ZFUSE=0) agrees."""
    cp, _ = _fused_operator(nx)
    N = (nx, 2, 32)
    outs = []
    for fz in (1, 0):
        ctx = _ctx_env(fm, FMMT_ZFUSE=fz)
        outs.append(_check_multi(ctx, cp, N, ncomp, 400 + ncomp + nx))
        if fz:
            op = ctx.import_op("tucker3d", cp.n, cp.ndir, cp.ranks, cp.arrays)
            out = torch.empty(int(np.prod(cp.n)), dtype=torch.complex64, device="cuda")
            for p in (0, cp.ndir - 1):
                op.restore(p, out)
                ctx.sync()
                got = t_lib_to_math(out.cpu().numpy(), cp.n)
                assert rel(cp.restore(p), got) <= 1e-6, p
            op.close()
        ctx.close()
    assert rel(outs[0], outs[1]) <= 1e-6
