"""Experiment: how does tcgen05 kind::tf32 treat the low 13 mantissa bits of FP32 operands?
impl 2: hi = rna(x), lo = rna(x - hi); impl 3: hi = x, lo = x - trunc13(x); impl 4: hi = x, lo = x - rna(x)."""
import numpy as np, torch
from paper_2010_00520_b200 import fmmt
ctx = fmmt.Context(0, torch.cuda.current_stream().cuda_stream)
rng = np.random.default_rng(1)
for (m, n, k) in [(1024, 64, 27), (4096, 338, 169), (1024, 64, 1201)]:
    A = ((rng.standard_normal((m, k)) + 1j * rng.standard_normal((m, k))) * 0.7).astype(np.complex64)
    B = ((rng.standard_normal((k, n)) + 1j * rng.standard_normal((k, n))) * 0.7).astype(np.complex64)
    ref = A.astype(np.complex128) @ B.astype(np.complex128)
    dA = torch.from_numpy(np.ascontiguousarray(A.T)).cuda(); dB = torch.from_numpy(np.ascontiguousarray(B.T)).cuda()
    out = {}
    for impl in (0, 1, 2, 3, 4):
        dC = torch.zeros((n, m), dtype=torch.complex64, device="cuda")
        fmmt._check(fmmt.fmmt_test_cgemm(ctx.h, impl, m, n, k, 0, 0, dA.data_ptr(), m, dB.data_ptr(), k, dC.data_ptr(), m), ctx.h, "t")
        ctx.sync()
        got = dC.cpu().numpy().T
        out[impl] = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
    print((m, n, k), {i: f"{e:.3e}" for i, e in out.items()}, flush=True)
