"""Time / profile the aggregation and disaggregation kernels alone at a config's size
(synthetic sphere-shell basis functions, patterns drawn on the device).
    PYTHONPATH=. python scripts/agg_probe.py [config] [reps]"""
import math
import sys

import numpy as np
import torch

from paper_2010_00520_b200 import fmmt
from synth import basis, basis_seed, config

cfg_i = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
c = config(cfg_i)
b = basis(basis_seed(cfg_i), c.Nx, c.Ny, c.Nz, c.edge)
nd, nb, nc = c.ndir, b.N, 2
ctx = fmmt.Context(0, torch.cuda.current_stream().cuda_stream)
g = torch.Generator(device="cuda")
g.manual_seed(1)
P = torch.view_as_complex(torch.randn((nd, nb, nc, 2), generator=g, device="cuda"))
I = torch.view_as_complex(torch.randn((nb, 2), generator=g, device="cuda"))
box = torch.from_numpy(b.box_ptr).cuda()
sig = torch.empty((nd, nc, c.Nz, c.Ny, c.Nx), dtype=torch.complex64, device="cuda")
w = torch.rand(nd, device="cuda")
y = torch.empty(nb, dtype=torch.complex64, device="cuda")
N = (c.Nx, c.Ny, c.Nz)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn in (("aggregate", lambda: ctx.aggregate(P, I, box, nd, nb, nc, N, sig)),
                 ("disaggregate", lambda: ctx.disaggregate(P, sig, w, box, nd, nb, nc, N, y))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    gb = (nd * nb * nc * 8) / (ms * 1e-3) / 1e9
    print(f"{name}: {ms * 1e3:.1f} us  P-stream {gb:.0f} GB/s  (N={nb}, ndir={nd}, boxes {int((np.diff(b.box_ptr) > 0).sum())}/{c.K})")
ctx.sync()
