"""Paper sweeps on the GPU compressor (§III.A.1-4):
memory saving (and, where the translate path runs, the paper-style overhead) of the five formats on the
FFT'ed translation operators of a PEC-sphere-sized box grid, against

  E1  structure size  n = 32 ... 256 (8λ ... 64λ sphere, 0.5λ boxes, 5 digits -> L = 14, 435 directions),
      gamma = 1e-6 (Fig. 5, Tables I and II);
  E2  tolerance       gamma = 1e-3 ... 1e-6 on the 64λ case (Fig. 6);
  E3  box size        0.25λ ... 1λ on the 32λ sphere, 5 digits (Fig. 7, Table III: 256^3 x 231 ... 64^3 x 1035);
  E4  FMM accuracy    3 ... 6 digits, 0.5λ boxes (Fig. 8: 325 ... 496 directions).

Operators are built on the GPU in FP64 (eq. (7) + FFT, fmmt_build_operator; paper direction grid
(L+1)(2L+1)) and compressed on the GPU in FP64 (Alg. 1-3, fmmt_compress; the memory-bounded Gram
path above ~1/2.5 of free memory).  Shapes outside the translate path give storage-only ops (ranks and
bytes); the overhead t(format) / t(DENSE) - 1 is measured where the translate path runs (n3 <= 64).
Synthetic operators only: no mesh, no dataset (the operator depends only on the box grid).

    python scripts/paper_sweeps.py E1 [E2 E3 E4] [--max-n 256] [--out profiles/r02_sweeps.jsonl]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2010_00520_b200 import fmmt  # noqa: E402

FORMATS = ("tucker3d", "tt3d", "tucker4d", "htucker4d", "tt4d")
# PAPER.md Table II and Tables I / III: context only (different rank rule
# reading and geometry; Q7 / Q8)
PAPER_T2 = {32: {"tt3d": 28, "tucker3d": 29, "tt4d": (27, 322), "tucker4d": 28, "htucker4d": (25, 327)},
            64: {"tt3d": 42, "tucker3d": 44, "tt4d": (42, 503), "tucker4d": 44, "htucker4d": (43, 511)},
            128: {"tt3d": 67, "tucker3d": 69, "tt4d": (67, 826), "tucker4d": 68, "htucker4d": (63, 836)},
            256: {"tt3d": 114, "tucker3d": 115, "tt4d": (113, 1438), "tucker4d": 114, "htucker4d": (113, 1452)}}
PAPER_T1 = {"tt3d": (81.41, 0.36), "tucker3d": (91.41, 0.35), "tt4d": (98.29, 2.27), "tucker4d": (95.43, 0.77),
            "htucker4d": (99.21, 0.42)}
PAPER_T3 = {"tt3d": (93.02, 0.25), "tucker3d": (97.80, 0.21), "tt4d": (99.17, 0.89), "tucker4d": (98.84, 0.42),
            "htucker4d": (99.75, 0.18)}


def time_translate(ctx, op, n, nd, reps=5):
    """Device time of one translate (ms), signatures CN(0,1) on the device."""
    N = (n[0] // 2, n[1] // 2, n[2] // 2)
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    sig = torch.view_as_complex(torch.randn((nd, N[2], N[1], N[0], 2), generator=g, device="cuda")
                                .mul_(math.sqrt(0.5)))
    out = torch.empty_like(sig)
    for _ in range(3):
        op.translate(sig, out, nd, N)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        op.translate(sig, out, nd, N)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def one_setting(ctx, tag, n_box, edge, digits, gamma, formats=FORMATS, timing=True, T=None):
    k = 2 * math.pi
    L = fmmt.multipole_count(k, edge, digits)
    khat, _ = fmmt.direction_grid(L, 2 * L + 1)
    nd = len(khat)
    n = (2 * n_box, 2 * n_box, 2 * n_box)
    rec = {"sweep": tag, "n": n[0], "edge": edge, "digits": digits, "L": L, "ndir": nd, "gamma": gamma,
           "T_gb_fp64": round(n[0] ** 3 * nd * 16 / 1e9, 2), "formats": {}}
    t0 = time.time()
    if T is None:
        T = torch.empty((nd,) + n, dtype=torch.complex128, device="cuda")
        ctx.build_operator(n_box, n_box, n_box, edge, k, L, khat, T)
        ctx.sync()
    rec["build_s"] = round(time.time() - t0, 2)
    torch.cuda.empty_cache()
    rec["free_gb_after_build"] = round(torch.cuda.mem_get_info()[0] / 1e9, 1)
    dense_ms = None
    translatable = n[2] <= 64
    if timing and translatable:
        dop = ctx.compress(T, n, nd, "dense", 0.5)
        dense_ms = time_translate(ctx, dop, n, nd)
        dop.close()
        torch.cuda.empty_cache()
        rec["dense_ms"] = round(dense_ms, 4)
    for fmt in formats:
        t0 = time.time()
        try:
            op = ctx.compress(T, n, nd, fmt, gamma)
            ctx.sync()
            info = op.info()
            r = {"rank_max": info["rank_max"], "rank_mean": [round(x, 2) for x in info["rank_mean"]],
                 "saving_pct": round(100 * (1 - info["compressed_bytes"] / info["original_bytes"]), 3),
                 "compressed_gb": round(info["compressed_bytes"] / 1e9, 4), "compress_s": round(time.time() - t0, 1)}
            if timing and info["translatable"] and dense_ms:
                ms = time_translate(ctx, op, n, nd)
                r["translate_ms"] = round(ms, 4)
                r["overhead_vs_dense"] = round(ms / dense_ms - 1, 3)
            op.close()
        except Exception as e:  # report the format's failure (e.g. FP64 TT-4D memory at 256^3) and go on
            r = {"error": str(e)[:240]}
        rec["formats"][fmt] = r
        torch.cuda.empty_cache()
    return rec, T


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("sweeps", nargs="*", default=["E1"])
    ap.add_argument("--max-n", type=int, default=256)
    ap.add_argument("--min-n", type=int, default=0)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "paper_sweeps.jsonl"))
    ap.add_argument("--inproc", action="store_true", help="run in this process (default: one process per sweep "
                    "setting, so every setting starts with a clean device)")
    args = ap.parse_args()
    if not args.inproc:
        import subprocess
        units = []
        for sw in args.sweeps:
            if sw == "E1":
                units += [("E1", n) for n in (32, 64, 128, 256) if args.min_n <= n <= args.max_n]
            elif sw == "E3":
                units += [("E3", n) for n in (256, 192, 128, 96, 64) if args.min_n <= n <= args.max_n]
            else:
                units.append((sw, 0))
        rc = 0
        for sw, n in units:
            cmd = [sys.executable, os.path.abspath(__file__), sw, "--inproc", "--out", args.out, "--max-n",
                   str(n if n else args.max_n), "--min-n", str(n if n else args.min_n)]
            r = subprocess.run(cmd)
            rc = rc or r.returncode
        raise SystemExit(rc)
    ctx = fmmt.Context(0, torch.cuda.current_stream().cuda_stream)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    f = open(args.out, "a")

    def emit(rec):
        print(json.dumps(rec), flush=True)
        f.write(json.dumps(rec) + "\n")
        f.flush()

    big = args.max_n // 2   # boxes per side of the "64λ" case
    for sw in args.sweeps:
        if sw == "E1":        # Fig. 5, Tables I, II: 8λ ... 64λ sphere, 0.5λ boxes, 5 digits, gamma 1e-6
            for nb in (16, 32, 64, 128):
                if not args.min_n <= 2 * nb <= args.max_n:
                    continue
                rec, T = one_setting(ctx, "E1", nb, 0.5, 5, 1e-6)
                rec["paper_table2"] = PAPER_T2.get(2 * nb)
                if 2 * nb == 256:
                    rec["paper_table1"] = PAPER_T1
                emit(rec)
                del T
                torch.cuda.empty_cache()
        elif sw == "E2":      # Fig. 6: gamma 1e-3 ... 1e-6 on the 64λ case (one operator, four tolerances)
            T = None
            for g in (1e-3, 1e-4, 1e-5, 1e-6):
                rec, T = one_setting(ctx, "E2", big, 0.5, 5, g, T=T)
                emit(rec)
            del T
            torch.cuda.empty_cache()
        elif sw == "E3":      # Fig. 7, Table III: 32λ sphere, box 0.25λ ... 1λ, 5 digits
            for edge in (0.25, 1 / 3, 0.5, 2 / 3, 1.0):
                nb = int(round(32 / edge))
                if not args.min_n <= 2 * nb <= args.max_n:
                    continue
                rec, T = one_setting(ctx, "E3", nb, edge, 5, 1e-6)
                if abs(edge - 0.25) < 1e-9:
                    rec["paper_table3"] = PAPER_T3
                emit(rec)
                del T
                torch.cuda.empty_cache()
        elif sw == "E4":      # Fig. 8: FMM accuracy 3 ... 6 digits, 0.5λ boxes
            for digits in (3, 4, 5, 6):
                rec, T = one_setting(ctx, "E4", big, 0.5, digits, 1e-6)
                emit(rec)
                del T
                torch.cuda.empty_cache()
    f.close()
    ctx.close()


if __name__ == "__main__":
    main()
