"""Debug: tensor-core z-stage for n3 = 64 on a tiny random Tucker-3D op."""
import sys, time
import numpy as np, torch
from paper_2010_00520_b200 import fmmt
from oracle import restore, translate
from synth import signatures
ctx = fmmt.Context(0, torch.cuda.current_stream().cuda_stream)
rng = np.random.default_rng(0)
N = tuple(int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (4, 4, 32)
n = tuple(2 * x for x in N)
nd, r = 3, (5, 6, int(sys.argv[4]) if len(sys.argv) > 4 else 7)
def cn(shape): return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(np.complex64).astype(np.complex128)
cores = [cn(r) for _ in range(nd)]
Us = [[cn((n[i], r[i])) for i in range(3)] for _ in range(nd)]
fl = lambda a: np.asarray(a).ravel(order="F").astype(np.complex64)
arrays = [np.concatenate([fl(c) for c in cores])] + [np.concatenate([fl(u[i]) for u in Us]) for i in range(3)]
op = ctx.import_op("tucker3d", n, nd, np.array([r] * nd), arrays)
print("imported", flush=True)
out = torch.empty(int(np.prod(n)), dtype=torch.complex64, device="cuda")
t0 = time.time(); op.restore(1, out); ctx.sync(); print("restore ok", time.time() - t0, flush=True)
got = np.reshape(out.cpu().numpy(), n, order="F")
ref = restore.tucker3d_restore(cores[1], *Us[1])
print("restore rel", np.linalg.norm(got - ref) / np.linalg.norm(ref), flush=True)
sig = signatures(5, nd, *N)
d_in = torch.from_numpy(sig).cuda(); d_out = torch.empty_like(d_in)
t0 = time.time(); op.translate(d_in, d_out, nd, N); ctx.sync(); print("translate ok", time.time() - t0, flush=True)
sm, om = translate.sig_to_math(sig), translate.sig_to_math(d_out.cpu().numpy())
for p in range(nd):
    ref = translate.translate_fft(restore.tucker3d_restore(cores[p], *Us[p]), sm[p])
    print("translate rel", p, np.linalg.norm(om[p] - ref) / np.linalg.norm(ref), flush=True)
