"""Repro helper: GPU-built, GPU-compressed config-2 operator, translate_sum_multi with ncomp."""
import sys, time
import numpy as np, torch
from paper_2010_00520_b200 import fmmt
from synth import config, signatures, signature_seed
fmt = sys.argv[1]; tol = float(sys.argv[2]); ncomp = int(sys.argv[3])
c = config(2)
ctx = fmmt.Context(0, torch.cuda.current_stream().cuda_stream)
khat, w = fmmt.direction_grid(c.L, c.nphi)
nd = len(khat); n = c.n
T = torch.empty((nd, n[2], n[1], n[0]), dtype=torch.complex128, device="cuda")
ctx.build_operator(c.Nx, c.Ny, c.Nz, c.edge, c.k, c.L, khat, T)
op = ctx.compress(T, n, nd, fmt, tol)
del T
N = (c.Nx, c.Ny, c.Nz)
sig = torch.from_numpy(signatures(1, nd * ncomp, *N).reshape(nd, ncomp, c.Nz, c.Ny, c.Nx)).cuda()
wd = torch.from_numpy(w.astype(np.float32)).cuda()
s = torch.empty((ncomp, c.Nz, c.Ny, c.Nx), dtype=torch.complex64, device="cuda")
for i in range(4):
    t0 = time.time()
    op.translate_sum_multi(sig, None, wd, s, nd, ncomp, N)
    ctx.sync()
    print(fmt, tol, ncomp, i, round(time.time() - t0, 4), flush=True)
