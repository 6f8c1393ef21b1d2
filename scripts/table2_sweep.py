"""Paper sweep on the GPU compressor: the Table II setting of
PAPER.md (spheres 8λ/16λ/32λ -> padded grids n = 32/64/128, box 0.5λ, 5 digits ->
L = 14, paper direction grid (L+1)(2L+1) = 435, gamma = 1e-6).

The operator is built on the GPU in FP64 (eq. (7) + FFT, fmmt_build_operator) and compressed
on the GPU in FP64 (Alg. 1-3, fmmt_compress) for the five formats; the ranks and the memory
saving are printed next to the paper's Table II ranks (context: the paper's operators come from
its own sphere geometry and its rank rule; readings Q7/Q8 of DESIGN.md differ).

    python scripts/table2_sweep.py [--gamma G] [n ...]   (default gamma 1e-6, n = 32 64) -> one JSON line per n

n = 128 (32 lambda) is outside the translate path (n3 <= 64) and is not swept.
"""
import json
import math
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2010_00520_b200 import fmmt  # noqa: E402

PAPER = {  # Table II: TT-3D rmax, Tucker-3D rmax, TT-4D (r1, r2), Tucker-4D r, H-Tucker (leaves, r12)
    32: {"tt3d": 28, "tucker3d": 29, "tt4d": (27, 322), "tucker4d": 28, "htucker4d": (25, 327), "r4": 225},
    64: {"tt3d": 42, "tucker3d": 44, "tt4d": (42, 503), "tucker4d": 44, "htucker4d": (43, 511), "r4": 225},
    128: {"tt3d": 67, "tucker3d": 69, "tt4d": (67, 826), "tucker4d": 68, "htucker4d": (63, 836), "r4": 225},
}


def main():
    args = sys.argv[1:]
    gamma = 1e-6
    if args[:1] == ["--gamma"]:
        gamma, args = float(args[1]), args[2:]
    ns = [int(x) for x in args] or [32, 64]
    ctx = fmmt.Context(0, torch.cuda.current_stream().cuda_stream)
    edge, digits = 0.5, 5
    k = 2 * math.pi
    L = fmmt.multipole_count(k, edge, digits)
    khat, _ = fmmt.direction_grid(L, 2 * L + 1)
    nd = len(khat)
    for n in ns:
        N = n // 2
        t0 = time.time()
        T = torch.empty((nd, n, n, n), dtype=torch.complex128, device="cuda")
        ctx.build_operator(N, N, N, edge, k, L, khat, T)
        ctx.sync()
        rec = {"n": n, "L": L, "ndir": nd, "gamma": gamma, "build_s": round(time.time() - t0, 2), "formats": {}}
        for fmt in ("tucker3d", "tt3d", "tucker4d", "htucker4d", "tt4d"):
            t0 = time.time()
            try:
                op = ctx.compress(T, (n, n, n), nd, fmt, gamma)
                ctx.sync()
                info = op.info()
                rec["formats"][fmt] = {"rank_max": info["rank_max"],
                                       "rank_mean": [round(x, 2) for x in info["rank_mean"]],
                                       "saving_pct": round(100 * (1 - info["compressed_bytes"] / info["original_bytes"]), 3),
                                       "compress_s": round(time.time() - t0, 2)}
                op.close()
            except Exception as e:  # report, continue with the next format
                rec["formats"][fmt] = {"error": str(e)[:200]}
            torch.cuda.empty_cache()
        rec["paper_table2"] = PAPER.get(n)
        print(json.dumps(rec), flush=True)
        del T
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
