"""Time the DENSE operator's translate (the P:161 overhead denominator) alone, for ncu captures of its kernels.

    python scripts/dense_probe.py [--config 5] [--reps 5]

Builds the eq. (7) operator of the config on the GPU, stores it uncompressed ("dense"), and runs
translate_sum on the config's seeded signatures; prints one JSON line (mean ms per translate_sum, CUDA events,
L2 flushed between reps).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from synth import config as get_config, signature_seed, signatures  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch
    from paper_2010_00520_b200 import fmmt
    cfg = get_config(args.config)
    n, ndir = cfg.n, cfg.ndir
    N = (cfg.Nx, cfg.Ny, cfg.Nz)
    stream = torch.cuda.Stream()
    ctx = fmmt.Context(0, stream.cuda_stream)
    khat, w = fmmt.direction_grid(cfg.L, cfg.nphi)
    with torch.cuda.stream(stream):
        T = torch.empty((ndir,) + n[::-1], dtype=torch.complex128, device="cuda")
        ctx.build_operator(cfg.Nx, cfg.Ny, cfg.Nz, cfg.edge, cfg.k, cfg.L, khat, T)
        ctx.sync()
        dense = ctx.compress(T, n, ndir, "dense", 0.5)
        del T
        torch.cuda.empty_cache()
        sig = torch.from_numpy(signatures(signature_seed(args.config, 0), ndir, *N)).cuda()
        sig_out = torch.empty_like(sig)
        wd = torch.from_numpy(w.astype(np.float32)).cuda()
        sums = torch.empty((cfg.Nz, cfg.Ny, cfg.Nx), dtype=torch.complex64, device="cuda")
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        for _ in range(3):
            dense.translate_sum(sig, sig_out, wd, sums, ndir, N)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dts = []
        for s in range(args.reps):
            flush.fill_(s & 0xFF)
            e0.record(stream)
            dense.translate_sum(sig, sig_out, wd, sums, ndir, N)
            e1.record(stream)
            e1.synchronize()
            dts.append(e0.elapsed_time(e1))
    ms = float(np.mean(dts))
    byts = ndir * int(np.prod(n)) * 8 + 2 * ndir * int(np.prod(N)) * 8
    print(json.dumps({"config": args.config, "dense_ms": round(ms, 4), "gbs": round(byts / ms / 1e6, 1)}))
    dense.close()


if __name__ == "__main__":
    main()
