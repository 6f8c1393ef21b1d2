#!/usr/bin/env python
"""Benchmark of the compressed FMM-FFT translation stage (arXiv 2010.00520) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]

One step = one matvec of the translation stage (restore + FFT convolution +
direction sum) for every (format, tol) operator the
BASELINE.json configuration lists; at the default config 2 that is the five
formats (Tucker-3D, Tucker-4D, H-Tucker-4D, TT-3D, TT-4D) at tol 1e-4 and 1e-6.

Metric (BASELINE.json): direction x padded-grid-points translated per second,
value = sum over ops of (ndir * n1 n2 n3) / device time of the step (max over
ranks), inputs resident in HBM.  The operators are built on the GPU from eq. (7)
(FP64) and compressed on the GPU (FP64 Alg. 1-3); signatures are seeded CN(0,1).

For N > 1 (torchrun) directions are sharded in contiguous blocks and the
direction-summed result is NCCL-allreduced inside fmmt_translate_sum.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import config as get_config, signature_seed, signatures  # noqa: E402

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}
# FP32 FFMA peak: 148 SMs x 128 FP32 lanes x 2 flop x 1.965 GHz (B200_PROFILING.md
# table: 148 SMs, clocks.max.sm 1965 MHz) -- the "alu" roofline of the FFMA kernels.
FFMA_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return d, "measured"
    except Exception:
        return PEAKS_FALLBACK, "fallback"


# ------------------------------------------------------------------ per-kernel algorithmic work
def kernel_work(info: dict, fmt: str, ranks: np.ndarray, ndir: int):
    """Algorithmic flops (or bytes) per matvec for each kernel class of one op.
    CMAC = complex multiply-add = 8 real flops.  DESIGN.md §Roofline gives the
    per-unit figures."""
    n1, n2, n3 = info["n"]
    n = n1 * n2 * n3
    n12 = n1 * n2
    K = n // 8
    w = {}
    lg3 = math.log2(n3)
    if fmt in ("tucker3d", "tt3d"):
        rr = ranks.reshape(ndir, -1).astype(np.float64)
    else:
        rr = np.tile(ranks.astype(np.float64), (ndir, 1))
    if fmt in ("tucker3d", "tucker4d"):
        r1, r2, r3 = rr[:, 0], rr[:, 1], rr[:, 2]
        w["restore_mode1"] = 8 * float(np.sum(n1 * r1 * r2 * r3))
        w["restore_mode2"] = 8 * float(np.sum(n12 * r2 * r3))
        rz = r3
    elif fmt == "tt3d":
        r1, r2 = rr[:, 0], rr[:, 1]
        w["restore_tt_head"] = 8 * float(np.sum(n1 * r1 * n2 * r2))
        rz = r2
    elif fmt == "tt4d":
        r2, r3 = rr[:, 1], rr[:, 2]
        w["slice_tt4d"] = 8 * float(np.sum(r2 * n3 * r3))
        rz = r2
    if fmt == "tucker4d":
        w["slice_tucker4d"] = 8 * float(np.sum(rr[:, 0] * rr[:, 1] * rr[:, 2] * rr[:, 3]))
    if fmt == "htucker4d":
        r1, r2, r3, r4, r12, r34 = [rr[:, i] for i in range(6)]
        w["slice_htucker_M"] = 8 * float(np.sum(r3 * r4 * r34))
        w["slice_htucker_G"] = 8 * float(np.sum(n12 * r34 * r3))
        rz = r3
    if fmt == "dense":
        w["conv_z_dense"] = float(ndir * n * 8)           # bytes: the operator read once
    else:
        # restore (8 r flop/pt) + Hadamard (6) + pruned z-DFT pair (5 log2 n3) per padded point
        w[f"restore_conv_z_{fmt}"] = float(np.sum(8.0 * n * rz)) + ndir * n * (6 + 5 * lg3)
    return w


# ------------------------------------------------------------------ clocks
class ClockSampler:
    def __init__(self, device_index: int):
        self.idx = device_index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def __enter__(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        try:
            rows = [l.strip().split(",") for l in open(self.path) if l.strip()]
        except Exception:
            rows = []
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
                for nm, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
            except Exception:
                continue
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def workload_str(cfg_index, formats):
    cfg = get_config(cfg_index)
    n = cfg.n
    return (f"config{cfg_index}: {cfg.Nx}x{cfg.Ny}x{cfg.Nz} boxes, padded {n[0]}x{n[1]}x{n[2]}, "
            f"{cfg.ndir} dirs, edge {cfg.edge} lambda, L={cfg.L}; ops " + ",".join(f"{f}@{t:g}" for f, t in formats))


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2010_00520_b200 import fmmt

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world and world > 1:
        raise SystemExit(f"--gpus {args.gpus} != WORLD_SIZE {world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.Stream()
    cfg = get_config(args.config)
    N = (cfg.Nx, cfg.Ny, cfg.Nz)
    n = cfg.n
    npad = int(np.prod(n))
    K = cfg.K
    ndir = cfg.ndir

    # context (NCCL communicator for world > 1, id bootstrapped over torch.distributed)
    if world > 1:
        idt = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(fmmt.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        ctx = fmmt.Context(local, stream.cuda_stream, rank, world, bytes(idt.cpu().numpy()))
    else:
        ctx = fmmt.Context(local, stream.cuda_stream)
    d0, dn = fmmt.shard_range(ndir, rank, world)
    ctx.set_gemm_impl(args.gemm)

    # setup (untimed): directions, FP64 operator on the GPU, GPU compression
    t_setup = time.time()
    khat, w = fmmt.direction_grid(cfg.L, cfg.nphi)
    with torch.cuda.stream(stream):
        T = torch.empty((ndir,) + n[::-1], dtype=torch.complex128, device="cuda")
        ctx.build_operator(cfg.Nx, cfg.Ny, cfg.Nz, cfg.edge, cfg.k, cfg.L, khat, T)
        ctx.sync()
        ops = []
        fmts = cfg.formats
        if args.formats:
            want = {(f.split("@")[0], float(f.split("@")[1])) for f in args.formats.split(",")}
            fmts = tuple(ft for ft in fmts if (ft[0], ft[1]) in want)
        for fmt, tol in fmts:
            if fmt in ("tucker3d", "tt3d"):
                op = ctx.compress(T[d0:d0 + dn].contiguous(), n, dn, fmt, tol)
            else:
                op = ctx.compress(T, n, ndir, fmt, tol, d0, dn)
            ops.append((fmt, tol, op))
        dense = ctx.compress(T[d0:d0 + dn].contiguous(), n, dn, "dense", 0.5)
        del T
        torch.cuda.empty_cache()
        sig = torch.from_numpy(signatures(signature_seed(args.config, 0), ndir, *N)[d0:d0 + dn]).cuda()
        sig_out = torch.empty_like(sig)
        wd = torch.from_numpy(w[d0:d0 + dn].astype(np.float32)).cuda()
        sums = torch.empty((cfg.Nz, cfg.Ny, cfg.Nx), dtype=torch.complex64, device="cuda")
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    t_setup = time.time() - t_setup

    def step(events=None):
        for i, (_, _, op) in enumerate(ops):
            if events is not None:
                events[i][0].record(stream)
            op.translate_sum(sig, sig_out, wd, sums, dn, N)
            if events is not None:
                events[i][1].record(stream)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
        barrier()
        ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in ops]
              for _ in range(args.steps)]
        l0 = ctx.launches
        with ClockSampler(local) as clk:
            barrier()
            for s in range(args.steps):
                flush.fill_(s & 0xFF)          # L2 flush (256 MiB write) between timed steps, outside the events
                step(ev[s])
            barrier()
        launches = ctx.launches - l0
        per_op = np.zeros(len(ops))
        for s in range(args.steps):
            for i in range(len(ops)):
                per_op[i] += ev[s][i][0].elapsed_time(ev[s][i][1])
        per_op /= args.steps                     # ms per matvec per op (this rank)
        t_step = float(per_op.sum())
        if world > 1:
            tt = torch.tensor([t_step] + list(per_op), dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_step = float(tt[0])
            per_op = tt[1:].cpu().numpy()

        if args.quick:   # profiling mode (ncu): the timed steps only
            print(json.dumps({"quick": True, "ms_per_step": t_step, "launches": int(launches)}), flush=True)
            return
        # DENSE (uncompressed) baseline for the overhead figure
        dense_ms = None
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(2):
            dense.translate_sum(sig, sig_out, wd, sums, dn, N)
        dts = []
        for s in range(max(3, args.steps)):
            flush.fill_(s & 0xFF)
            e0.record(stream)
            dense.translate_sum(sig, sig_out, wd, sums, dn, N)
            e1.record(stream)
            e1.synchronize()
            dts.append(e0.elapsed_time(e1))
        dense_ms = float(np.mean(dts))

        # per-kernel breakdown (separate profiled pass: events around every launch)
        ctx.set_profiling(True)
        ctx.prof_reset()
        kwork = {}
        PROF_STEPS = 3
        for _ in range(PROF_STEPS):
            step()
        prof = ctx.prof_read()
        ctx.set_profiling(False)
        for fmt, tol, op in ops:
            info = op.info()
            for kname, v in kernel_work(info, fmt, op.ranks(), dn).items():
                kwork[kname] = kwork.get(kname, 0.0) + v * PROF_STEPS

        # two-component signatures: theta and phi share one restore per direction
        sig2 = torch.from_numpy(np.ascontiguousarray(
            signatures(signature_seed(args.config, 2), 2 * ndir, *N).reshape(ndir, 2, cfg.Nz, cfg.Ny, cfg.Nx)[d0:d0 + dn])).cuda()
        sums2 = torch.empty((2, cfg.Nz, cfg.Ny, cfg.Nx), dtype=torch.complex64, device="cuda")
        for _ in range(3):
            for _, _, op in ops:
                op.translate_sum_multi(sig2, None, wd, sums2, dn, 2, N)
        ms2 = []
        for s in range(args.steps):
            flush.fill_(s & 0xFF)
            torch.cuda.synchronize()
            e0.record(stream)
            for _, _, op in ops:
                op.translate_sum_multi(sig2, None, wd, sums2, dn, 2, N)
            e1.record(stream)
            e1.synchronize()
            ms2.append(e0.elapsed_time(e1))
        two_comp_ms = float(np.mean(ms2))
        if world > 1:
            tt = torch.tensor([two_comp_ms], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            two_comp_ms = float(tt[0])
        del sig2

        # far-field matvec: eq. (4) aggregation -> eq. (5) with each op -> eq. (6)
        # disaggregation, one graph per op.  Synthetic basis functions (synth.basis: sphere-shell boxes,
        # 40-70 per non-empty box); the patterns' values do not affect timing, so they are drawn on the
        # device (seeded torch generator) instead of on the host.
        far = far_matvec_measure(ctx, ops, cfg, args, d0, dn, wd, N, flush, stream)

        # end-to-end through the C ABI with host buffers (pinned), per step:
        # H2D of the signatures + weights, the matvec, D2H of the summed result
        sig_h = torch.from_numpy(signatures(signature_seed(args.config, 1), ndir, *N)[d0:d0 + dn]).pin_memory()
        w_h = torch.from_numpy(w[d0:d0 + dn].astype(np.float32)).pin_memory()
        sum_h = torch.empty((cfg.Nz, cfg.Ny, cfg.Nx), dtype=torch.complex64).pin_memory()
        for _, _, op in ops:
            op.translate_sum_host(sig_h, w_h, sum_h, dn, N)
        barrier()
        e2e_ms = []
        for s in range(args.steps):
            flush.fill_(s & 0xFF)
            torch.cuda.synchronize()
            e0.record(stream)
            for _, _, op in ops:
                op.translate_sum_host(sig_h, w_h, sum_h, dn, N)
            e1.record(stream)
            e1.synchronize()
            e2e_ms.append(e0.elapsed_time(e1))
        e2e_t = float(np.mean(e2e_ms))
        if world > 1:
            tt = torch.tensor([e2e_t], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_t = float(tt[0])

    units_per_op = ndir * npad                  # all ranks together
    total_units = units_per_op * len(ops)
    value = total_units / (t_step * 1e-3) / 1e9
    e2e_value = total_units / (e2e_t * 1e-3) / 1e9

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    peaks, peak_src = load_peaks()
    # dominant kernel of the step (largest device time in the profiled pass)
    dom = max(prof.items(), key=lambda kv: kv[1][0])
    dname, (dms, dl) = dom[0], dom[1]
    if dname == "conv_z_dense":
        bound, unit, peak = "hbm", "GB/s", float(peaks["hbm_gbs"])
        achieved = kwork.get(dname, 0.0) / (dms * 1e-3) / 1e9
    elif dname in kwork and args.gemm in ("tc", "tc1"):
        # tcgen05 kind::tf32 with the 3xTF32 split: 3 tensor MMAs per useful MAC, so the
        # FP32-accurate tensor roofline is the TF32 dense peak / 3; TF32 = bf16 x 1/2 (guide's
        # nominal ratio), bf16 = measured sustained (kernel timed inside a long step).
        tf32 = 0.5 * float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops")))
        bound, unit, peak = "tensor", "TFLOP/s", tf32 / 3.0
        peak_src = f"{peak_src} bf16 sustained x 0.5 (TF32) / 3 (3xTF32 split) = {tf32 / 3:.1f}; raw TF32 {tf32:.1f}"
        achieved = kwork[dname] / (dms * 1e-3) / 1e12
    elif dname in kwork:
        bound, unit, peak = "alu", "TFLOP/s", FFMA_PEAK_TFLOPS
        peak_src = "derived FFMA (148 SM x 128 lanes x 2 x 1.965 GHz)"
        achieved = kwork[dname] / (dms * 1e-3) / 1e12
    else:
        bound, unit, peak, achieved = "hbm", "GB/s", float(peaks["hbm_gbs"]), None
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(dname)
        except Exception:
            traffic = None
    kernels = {k: {"ms_per_launch": v[0] / v[1], "launches_per_step": v[1] / PROF_STEPS,
                   "share": v[0] / sum(x[0] for x in prof.values()),
                   **({"achieved_tflops": kwork[k] / (v[0] * 1e-3) / 1e12} if k in kwork and k != "conv_z_dense" else {}),
                   **({"achieved_gbs": kwork[k] / (v[0] * 1e-3) / 1e9} if k == "conv_z_dense" else {})}
               for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0])}

    per_format = {}
    for i, (fmt, tol, op) in enumerate(ops):
        info = op.info()
        per_format[f"{fmt}@{tol:g}"] = {
            "ms": round(float(per_op[i]), 4),
            "gpt_s": round(units_per_op / (per_op[i] * 1e-3) / 1e9, 2),
            "rank_max": info["rank_max"],
            "saving_pct": round(100 * (1 - info["compressed_bytes"] / info["original_bytes"]), 2),
            "overhead_vs_dense": round(float(per_op[i]) / dense_ms - 1, 3),
            "restore_gflop": round(8 * info["restore_cmac"] / 1e9, 3),
        }

    line = {
        "metric": "direction*grid-points translated/s (restore+FFT conv)",
        "value": round(value, 3),
        "unit": "Gdir*pt/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(t_step, 4),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "c64",
        "data": "synthetic: eq.(7) operators built on GPU (FP64), GPU-compressed; CN(0,1) seeded signatures",
        "config": {"workload": workload_str(args.config, [(f, t) for f, t, _ in ops]),
                   "l2": "flushed between timed steps (256 MiB write outside the events)",
                   "parallelism": f"direction-shard x{world}",
                   "restore_gemm": {"tc": "tcgen05 kind::tf32, 3xTF32 split, FP32 accumulate", "tc1": "tcgen05 kind::tf32, 3xTF32 (first design)", "ffma": "FP32 FFMA"}[args.gemm]},
        "gpu_launches": int(launches),
        "roofline": {"bound": bound, "kernel": dname, "achieved": None if achieved is None else round(achieved, 3),
                     "peak": round(peak, 2), "unit": unit,
                     "frac": None if achieved is None else round(achieved / peak, 4),
                     "traffic": traffic,
                     "peak_source": peak_src},
        "e2e": {"value": round(e2e_value, 3), "unit": "Gdir*pt/s",
                "h2d_bytes_per_step": int(len(ops) * (ndir * K * 8 + ndir * 4)),
                "d2h_bytes_per_step": int(len(ops) * K * 8)},
        "per_box": {"value": round(value / 8, 3), "unit": "Gdir*box/s",
                    "note": "the same rate per box of the Nx*Ny*Nz grid (the padded grid point unit is 8 per box)"},
        "dense_ms": round(dense_ms, 4),
        "two_component": {"value": round(2 * total_units / (two_comp_ms * 1e-3) / 1e9, 3), "unit": "Gdir*pt/s",
                          "ms_per_step": round(two_comp_ms, 4),
                          "note": "theta+phi signatures [ndir][2][Nz][Ny][Nx], one restore per direction serves both "
                                  "(SURVEY 8(f) NEXT #1); units count both components"},
        "far_matvec": far,
        "per_format": per_format,
        "kernels": kernels,
        "setup_s": round(t_setup, 1),
    }
    line["clocks"] = clk.summary()
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.config, sample_dirs=args.cpu_sample)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def far_matvec_measure(ctx, ops, cfg, args, d0, dn, wd, N, flush, stream):
    """Time fmmt_far_matvec for every op of the step; profile the aggregation and disaggregation
    kernels against the HBM roofline (algorithmic bytes: P read once per kernel, plus the
    signatures / coefficients they read and write)."""
    import torch
    from synth import basis, basis_seed
    bas = basis(basis_seed(args.config), cfg.Nx, cfg.Ny, cfg.Nz, cfg.edge)
    K, nb, ncomp = cfg.K, bas.N, 2
    g = torch.Generator(device="cuda")
    g.manual_seed(basis_seed(args.config))
    P = torch.randn((dn, nb, ncomp, 2), generator=g, device="cuda", dtype=torch.float32).mul_(math.sqrt(0.5))
    P = torch.view_as_complex(P)
    I = torch.view_as_complex(torch.randn((nb, 2), generator=g, device="cuda", dtype=torch.float32))
    box = torch.from_numpy(bas.box_ptr).cuda()
    y = torch.empty((nb,), dtype=torch.complex64, device="cuda")
    for _ in range(3):
        for _, _, op in ops:
            op.far_matvec(P, I, box, wd, dn, nb, ncomp, N, y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = []
    for s in range(max(3, args.steps)):
        flush.fill_(s & 0xFF)
        torch.cuda.synchronize()
        e0.record(stream)
        for _, _, op in ops:
            op.far_matvec(P, I, box, wd, dn, nb, ncomp, N, y)
        e1.record(stream)
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    ctx.set_profiling(True)
    ctx.prof_reset()
    for _, _, op in ops:
        op.far_matvec(P, I, box, wd, dn, nb, ncomp, N, y)
    prof = ctx.prof_read()
    ctx.set_profiling(False)
    peaks, src = load_peaks()
    hbm = float(peaks["hbm_gbs"])
    pbytes = dn * nb * ncomp * 8
    kb = {"aggregate": pbytes + nb * 8 + dn * ncomp * K * 8,
          "disaggregate_partial": pbytes + dn * ncomp * K * 8 + dn * 4}
    kern = {}
    for k, b in kb.items():
        if k in prof:
            t = prof[k][0] / prof[k][1]
            gbs = b / (t * 1e-3) / 1e9
            kern[k] = {"ms_per_launch": round(t, 4), "bytes_per_launch": int(b), "achieved_gbs": round(gbs, 1),
                       "peak_gbs": hbm, "frac": round(gbs / hbm, 4)}
    t = float(np.mean(ms))
    del P, I
    return {"ms_per_step": round(t, 4), "ops": len(ops), "basis_functions": int(nb),
            "nonempty_boxes": int((np.diff(bas.box_ptr) > 0).sum()), "ncomp": ncomp,
            "value": round(len(ops) * dn * nb / (t * 1e-3) / 1e9, 3), "unit": "G basis-function*dir/s",
            "kernels": kern, "peak_source": src + " HBM copy bandwidth",
            "note": "eq.(4) aggregation + eq.(5) translate (both components) + eq.(6) disaggregation per op; "
                    "synthetic sphere-shell basis functions, CN(0,1) patterns drawn on the device"}


# ------------------------------------------------------------------ the oracle (cpu_baseline / reference arm)
def _oracle_ops(cfg_index, formats, sample):
    """Oracle operators (setup, untimed): operator build + compression."""
    from oracle import decomp, fmm, restore
    c = get_config(cfg_index)
    khat, w, _, _ = fmm.direction_grid(c.L, c.nphi)
    grid = fmm.OperatorGrid(c.Nx, c.Ny, c.Nz, c.edge, c.k, c.L)
    need4d = any(f in ("tucker4d", "htucker4d", "tt4d") for f, _ in formats)
    T4 = fmm.fft_operator_4d(grid, khat) if need4d else None
    ops = []
    for fmt, tol in formats:
        if fmt == "tucker3d":
            fs = {p: decomp.tucker_svd(T4[..., p] if T4 is not None else fmm.fft_operator_3d(grid, khat[p]), tol)
                  for p in sample}
            ops.append((fmt, tol, lambda p, fs=fs: restore.tucker3d_restore(fs[p].core, *fs[p].factors)))
        elif fmt == "tt3d":
            fs = {p: decomp.tt_svd(T4[..., p] if T4 is not None else fmm.fft_operator_3d(grid, khat[p]), tol)
                  for p in sample}
            ops.append((fmt, tol, lambda p, fs=fs: restore.tt3d_restore(fs[p].head, fs[p].cores[0], fs[p].tail)))
        elif fmt == "tucker4d":
            f = decomp.tucker_svd(T4, tol)
            ops.append((fmt, tol, lambda p, f=f: restore.tucker4d_slice(f.core, f.factors, p)))
        elif fmt == "htucker4d":
            h = decomp.htucker_svd(T4, tol)
            ops.append((fmt, tol, lambda p, h=h: restore.htucker_slice(h.leaves, h.c12, h.c34, h.c1234, p)))
        elif fmt == "tt4d":
            g = decomp.tt_svd(T4, tol)
            t2 = restore.tt4d_t2(g.cores[1], g.tail)
            ops.append((fmt, tol, lambda p, g=g, t2=t2: restore.tt4d_slice(g.head, g.cores[0], g.cores[1], g.tail, p, t2)))
    return c, w, ops


def _oracle_step(c, w, ops, sample, sig_math):
    from oracle import translate
    for _, _, rest in ops:
        B = [translate.translate_fft(rest(p), sig_math[p]) for p in sample]
        translate.direction_sum(np.stack(B), w[list(sample)])


def cpu_baseline(cfg_index, sample_dirs=24):
    """The oracle (FP64 CPU, as it stands) on a bounded sample: the 3D-format ops
    of the configuration on `sample_dirs` directions (the 4D formats' oracle
    compressions alone take minutes and are left to --impl reference)."""
    from oracle import translate
    c = get_config(cfg_index)
    formats = [(f, t) for f, t in c.formats if f in ("tucker3d", "tt3d")] or [("tucker3d", 1e-4)]
    sample = list(range(0, c.ndir, max(1, c.ndir // sample_dirs)))[:sample_dirs]
    c, w, ops = _oracle_ops(cfg_index, formats, sample)
    sig = translate.sig_to_math(signatures(signature_seed(cfg_index, 0), c.ndir, c.Nx, c.Ny, c.Nz))
    _oracle_step(c, w, ops, sample, sig)       # warm-up
    t0 = time.time()
    reps = 0
    while True:
        _oracle_step(c, w, ops, sample, sig)
        reps += 1
        if time.time() - t0 > 10.0 or reps >= 50:
            break
    dt = (time.time() - t0) / reps
    units = len(ops) * len(sample) * c.npad
    return {"value": round(units / dt / 1e9, 6), "unit": "Gdir*pt/s", "cores": os.cpu_count(), "kind": "oracle",
            "sample": f"config{cfg_index}: ops " + ",".join(f"{f}@{t:g}" for f, t, _ in ops)
                      + f" on {len(sample)} of {c.ndir} directions (restore + FP64 FFT conv + direction sum), "
                      f"mean of {reps} reps after 1 warm-up"}


def run_reference(args):
    """--impl reference: the oracle as it stands on the box's host cores, same
    config / metric / unit; each step a bounded sample of the workload."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import translate
    c = get_config(args.config)
    sample = list(range(0, c.ndir, max(1, c.ndir // args.ref_sample)))[:args.ref_sample]
    t0 = time.time()
    c, w, ops = _oracle_ops(args.config, list(c.formats), sample)
    setup = time.time() - t0
    sig = translate.sig_to_math(signatures(signature_seed(args.config, 0), c.ndir, c.Nx, c.Ny, c.Nz))
    for _ in range(args.warmup):
        _oracle_step(c, w, ops, sample, sig)
    t0 = time.time()
    for _ in range(args.steps):
        _oracle_step(c, w, ops, sample, sig)
    dt = (time.time() - t0) / args.steps
    units = len(ops) * len(sample) * c.npad
    v = units / dt / 1e9
    line = {
        "impl": "reference", "metric": "direction*grid-points translated/s (restore+FFT conv)",
        "value": round(v, 6), "unit": "Gdir*pt/s", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "c128", "data": "synthetic (oracle-built operators)",
        "config": {"workload": workload_str(args.config, list(c.formats)), "parallelism": "host cores",
                   "sample": f"{len(sample)} of {c.ndir} directions per op"},
        "cpu_baseline": {"value": round(v, 6), "unit": "Gdir*pt/s", "cores": os.cpu_count(), "kind": "oracle",
                         "sample": f"{len(sample)} of {c.ndir} directions per op, ops "
                                   + ",".join(f"{f}@{t:g}" for f, t, _ in ops) + f"; setup {setup:.0f}s untimed"},
        "e2e": {"value": round(v, 6), "unit": "Gdir*pt/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true", help="timed steps only (for ncu launch lists)")
    ap.add_argument("--gemm", default="tc", choices=["tc", "tc1", "ffma"], help="restore-GEMM kernel (A/B)")
    ap.add_argument("--formats", default=None, help="comma list fmt@tol restricting the config's ops")
    ap.add_argument("--cpu-sample", type=int, default=24)
    ap.add_argument("--ref-sample", type=int, default=8)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
