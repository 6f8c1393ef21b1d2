"""GPU: the restore-GEMM kernels (tcgen05 3xTF32 and FP32 FFMA) through the
C-ABI test hook fmmt_test_cgemm, against a complex128 numpy product.

These GEMMs are the contractions of Figs. 3-4; the bar is the
FP32-class accuracy the 1e-6 restore tolerance needs: relative
Frobenius error <= 1e-6 on CN(0,1) operands.  Shapes span several 128-row
tiles, ragged M/N/K tails, K < one stage, and both operand orders.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

TOL = 1e-6


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


def cn(rng, shape):
    return ((rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) * np.sqrt(0.5)).astype(np.complex64)


SHAPES = [(128, 64, 16), (300, 70, 45), (1, 1, 1), (129, 17, 17), (1024, 32, 27), (4096, 338, 169),
          (961, 130, 351), (32, 729, 27), (257, 33, 8), (1024, 64, 1201)]


@pytest.mark.parametrize("impl", ["tc", "ffma"])
@pytest.mark.parametrize("transA", [0, 1])
@pytest.mark.parametrize("transB", [0, 1])
@pytest.mark.parametrize("m,n,k", SHAPES)
def test_cgemm_matches_numpy(fm, ctx, impl, transA, transB, m, n, k):
    rng = np.random.default_rng(m * 7919 + n * 31 + k + 1000 * transA + 100 * transB)
    A = cn(rng, (m, k))
    B = cn(rng, (k, n))
    # column-major storage in the library's convention
    a_store = A.T if not transA else A            # transA=0: A(i,l) at i + m*l  (Fortran) == C-order of A.T
    b_store = B.T if not transB else B            # transB=0: B(l,j) at l + k*j
    lda = m if not transA else k
    ldb = k if not transB else n
    dA = torch.from_numpy(np.ascontiguousarray(a_store)).cuda()
    dB = torch.from_numpy(np.ascontiguousarray(b_store)).cuda()
    dC = torch.full((n, m), complex(np.nan, np.nan), dtype=torch.complex64, device="cuda")
    ctx.test_cgemm(impl, m, n, k, dA, lda, dB, ldb, dC, m, transA=transA, transB=transB)
    ctx.sync()
    got = dC.cpu().numpy().T
    ref = A.astype(np.complex128) @ B.astype(np.complex128)
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert np.isfinite(got).all()
    assert err <= TOL, f"{impl} rel err {err:.3e}"


@pytest.mark.parametrize("scale_a,scale_b", [(1e5, 1e-7), (1e-20, 1e20), (3e30, 1e-30)])
def test_cgemm_dynamic_range(fm, ctx, scale_a, scale_b):
    """The fp16 split scales each operand by a power of two from its max |Re|, |Im| (DESIGN 6.1):
    operands far outside the fp16 range and rows spanning 8 decades keep the FP32-class bar
    (relative Frobenius error <= 1e-6 of the complex128 product)."""
    m, n, k = 300, 70, 45
    rng = np.random.default_rng(5)
    rows = 10.0 ** rng.uniform(-4, 4, size=(m, 1))
    A = (cn(rng, (m, k)).astype(np.complex128) * rows * scale_a).astype(np.complex64)
    B = (cn(rng, (k, n)).astype(np.complex128) * scale_b).astype(np.complex64)
    dA = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
    dB = torch.from_numpy(np.ascontiguousarray(B.T)).cuda()
    dC = torch.empty((n, m), dtype=torch.complex64, device="cuda")
    ctx.test_cgemm("tc", m, n, k, dA, m, dB, k, dC, m)
    ctx.sync()
    got = dC.cpu().numpy().T
    ref = A.astype(np.complex128) @ B.astype(np.complex128)
    assert np.isfinite(got).all()
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= TOL
