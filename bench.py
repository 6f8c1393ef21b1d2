#!/usr/bin/env python
"""Benchmark of the compressed FMM-FFT translation stage (arXiv 2010.00520) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]

One step = one matvec of the translation stage (restore + FFT convolution +
direction sum + allreduce) for every (format, tol)
operator the BASELINE.json configuration lists.  The headline is config 5
(BASELINE configs[4]: 64x64x32 boxes, 128x128x64 padded grid, 882 directions,
TT-4D and Tucker-3D at 1e-4): the largest configuration, the one north_star's
1 -> 8 GPU scaling target names.  At N = 1 the line also carries config 2 (all
five formats at 1e-4 and 1e-6) and config 4 (Tucker-4D, H-Tucker-4D) as extra
keys (`other_configs`).

Metric (BASELINE.json): direction x padded-grid-points translated per second,
value = sum over ops of (ndir * n1 n2 n3) / device time of the step (max over
ranks), inputs resident in HBM.  Operators are built on the GPU from eq. (7)
(FP64) and compressed on the GPU (FP64 Alg. 1-3); signatures are seeded CN(0,1).

--gpus N > 1 without WORLD_SIZE in the environment re-launches this script under
torch.distributed.run with N ranks (one per GPU).  Directions are sharded in
contiguous blocks; the direction-summed result is NCCL-allreduced inside
fmmt_translate_sum; the 4D formats are compressed on rank 0 and broadcast.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import config as get_config, signature_seed, signatures  # noqa: E402

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}
METRIC = "direction*grid-points translated/s (restore+FFT conv), 1-8 B200, % of roofline"
UNIT = "Gdir*pt/s"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return json.load(open(p)), "measured"
    except Exception:
        return PEAKS_FALLBACK, "fallback (B200_PROFILING.md)"


def restore_peak_tflops(peaks, burst=True, split="fp16"):
    """FP32-accurate restore peak of the tensor cores (SURVEY §8(d) P_restore: the best unit's
    FP32-accurate rate).  The restore contractions run 3 tensor MMAs per useful MAC (hi.hi + hi.lo +
    lo.hi of an 11 + 11-bit split): fp16 split (kind::f16, the product build) at the fp16 = bf16 dense
    rate, or TF32 split (kind::tf32, A/B build) at bf16 x 1/2 (the guide's nominal 1.1 / 2.25 PF).
    bf16 = the measured cuBLAS figure: burst (a pass timed at max clocks) or sustained."""
    bf16 = float(peaks.get("bf16_tflops") if burst else peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops")))
    return bf16 * (1.0 if split == "fp16" else 0.5) / 3.0


# ------------------------------------------------------------------ algorithmic work
def _tucker3_chain_cmac(n, r):
    """Cheapest order of core(r1 r2 r3) x1 U1 x2 U2 x3 U3 (all 6 mode orders)."""
    import itertools
    best = None
    for order in itertools.permutations(range(3)):
        dims = list(r)
        c = 0.0
        for m in order:
            c += float(np.prod(dims)) * n[m]    # (prod of other dims) * r_m * n_m
            dims[m] = n[m]
        best = c if best is None else min(best, c)
    return best


def restore_cmac_per_dir(fmt, n, r):
    """a3 + a4 complex MACs for one direction at ranks r, cheapest contraction order
    (direction-independent products such as TT-4D T1 = U1 C1 and H-Tucker E are per op)."""
    n1, n2, n3 = n
    if fmt == "dense":
        return 0.0
    if fmt == "tucker3d":
        return _tucker3_chain_cmac(n, r[:3])
    if fmt == "tucker4d":
        return float(np.prod(r[:4])) + _tucker3_chain_cmac(n, r[:3])
    if fmt == "htucker4d":
        r1, r2, r3, r4, r12, r34 = r
        m = r3 * r4 * r34                                                     # M_p = C34 x2 u_p
        e_order = m + n1 * n2 * r34 * r3 + n1 * n2 * n3 * r3                  # G_p = E M_p^T, then x3 U3
        chain = m + r12 * r34 * r3 + r1 * r2 * r12 * r3 + _tucker3_chain_cmac(n, (r1, r2, r3))
        return float(min(e_order, chain))
    if fmt == "tt3d":
        r1, r2 = r[:2]
        return float(min(n1 * r1 * n2 * r2 + n1 * n2 * n3 * r2, r1 * n2 * r2 * n3 + n1 * r1 * n2 * n3))
    if fmt == "tt4d":
        r1, r2, r3 = r[:3]
        a3 = r2 * n3 * r3
        return float(a3 + min(n1 * n2 * r2 * n3, r1 * n2 * r2 * n3 + n1 * r1 * n2 * n3))
    raise ValueError(fmt)


def op_roofline(fmt, info, ranks, ndir_local, peaks, burst=True, split="fp16"):
    """t_roof = max((B_sig + B_fac)/BW, F_restore/P_restore) for one matvec of one op,
    B_fft = 0 (the half-padded spectra of a batch stay in L2 / on chip by design)."""
    n = info["n"]
    K = n[0] * n[1] * n[2] // 8
    if fmt in ("tucker3d", "tt3d"):
        rr = ranks.reshape(ndir_local, -1)
        cmac = float(sum(restore_cmac_per_dir(fmt, n, tuple(int(x) for x in row)) for row in rr))
    else:
        cmac = ndir_local * restore_cmac_per_dir(fmt, n, tuple(int(x) for x in ranks)) if fmt != "dense" else 0.0
    b_sig = 16.0 * K * ndir_local
    b_fac = float(info["compressed_bytes"])
    bw = float(peaks["hbm_gbs"]) * 1e9
    p = restore_peak_tflops(peaks, burst, split) * 1e12
    t_hbm, t_fl = (b_sig + b_fac) / bw, 8.0 * cmac / p
    return {"t_roof_ms": 1e3 * max(t_hbm, t_fl), "t_hbm_ms": 1e3 * t_hbm, "t_restore_ms": 1e3 * t_fl,
            "bound": "tensor" if t_fl > t_hbm else "hbm", "restore_gflop": 8.0 * cmac / 1e9,
            "bytes": b_sig + b_fac}


def kernel_flops(fmt, info, ranks, ndir):
    """Algorithmic flops of each restore kernel class of one op per matvec: the contraction the
    kernel performs (8 flop per complex MAC).  The z-stage of TT-4D performs all of a4, so it is
    credited with the cheapest a4 order; FFT / Hadamard ALU work is not counted."""
    n1, n2, n3 = info["n"]
    n12, n = n1 * n2, n1 * n2 * n3
    w = {}
    if fmt in ("tucker3d", "tt3d"):
        rr = ranks.reshape(ndir, -1).astype(np.float64)
    else:
        rr = np.tile(ranks.astype(np.float64), (ndir, 1))
    if fmt in ("tucker3d", "tucker4d"):
        r1, r2, r3 = rr[:, 0], rr[:, 1], rr[:, 2]
        w["restore_mode1"] = 8 * float(np.sum(n1 * r1 * r2 * r3))
        w["restore_mode2"] = 8 * float(np.sum(n12 * r2 * r3))
        w[f"restore_conv_z_{fmt}"] = 8 * float(np.sum(n * r3))
    if fmt == "tucker3d":
        # fused chain (n1 % 128 == 0, n3 = 64): mode 2 first (restore_mode2x: r1 n2 r3 r2 per direction), then
        # modes 1 and 3 in one kernel (n1 n2 r3 r1 + n r3)
        w["restore_mode2x"] = 8 * float(np.sum(r1 * n2 * r3 * r2))
        w["restore_conv_z_tucker3d_fused"] = 8 * float(np.sum(n12 * r3 * r1 + n * r3))
    if fmt == "tucker4d":
        w["slice_tucker4d"] = 8 * float(np.sum(rr[:, 0] * rr[:, 1] * rr[:, 2] * rr[:, 3]))
    if fmt == "tt3d":
        r1, r2 = rr[:, 0], rr[:, 1]
        w["restore_tt_head"] = 8 * float(np.sum(n1 * r1 * n2 * r2))
        w["restore_conv_z_tt3d"] = 8 * float(np.sum(n * r2))
    if fmt == "htucker4d":
        r3, r4, r34 = rr[:, 2], rr[:, 3], rr[:, 5]
        w["slice_htucker_M"] = 8 * float(np.sum(r3 * r4 * r34))
        w["slice_htucker_G"] = 8 * float(np.sum(n12 * r34 * r3))
        w["restore_conv_z_htucker4d"] = 8 * float(np.sum(n * r3))
    if fmt == "tt4d":
        r1, r2, r3 = rr[:, 0], rr[:, 1], rr[:, 2]
        w["slice_tt4d"] = 8 * float(np.sum(r2 * n3 * r3))
        w["restore_conv_z_tt4d"] = 8 * float(np.sum(np.minimum(n12 * r2 * n3, r1 * n2 * r2 * n3 + n1 * r1 * n2 * n3)))
    if fmt == "dense":
        w["conv_z_dense"] = float(ndir * n * 8)       # BYTES: the stored operator read once
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
            rows = [line.strip().split(",") for line in open(self.path) if line.strip()]
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
class Runner:
    """One rank of the GPU arm: context, stream, process group."""

    def __init__(self, args):
        import torch
        import torch.distributed as dist
        from paper_2010_00520_b200 import fmmt
        self.torch, self.dist, self.fmmt, self.args = torch, dist, fmmt, args
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        if self.world > 1 and args.gpus != self.world:
            raise SystemExit(f"--gpus {args.gpus} != WORLD_SIZE {self.world}")
        torch.cuda.set_device(self.local)
        if self.world > 1:
            dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
        self.stream = torch.cuda.Stream()
        if self.world > 1:
            idt = torch.zeros(128, dtype=torch.uint8, device="cuda")
            if self.rank == 0:
                idt.copy_(torch.frombuffer(bytearray(fmmt.nccl_unique_id()), dtype=torch.uint8))
            dist.broadcast(idt, 0)
            self.ctx = fmmt.Context(self.local, self.stream.cuda_stream, self.rank, self.world, bytes(idt.cpu().numpy()))
            if self.rank == 0:
                print(f"[bench] libfmmt NCCL communicator up: world {self.world}, one rank per GPU", file=sys.stderr,
                      flush=True)
        else:
            self.ctx = fmmt.Context(self.local, self.stream.cuda_stream)
        self.ctx.set_gemm_impl(args.gemm)

    def barrier(self):
        self.torch.cuda.synchronize()
        if self.world > 1:
            self.dist.barrier()
        self.torch.cuda.synchronize()

    def max_over_ranks(self, vals):
        vals = [float(v) for v in vals]
        if self.world == 1:
            return vals
        t = self.torch.tensor(vals, dtype=self.torch.float64, device="cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return [float(x) for x in t.cpu()]

    # -------------------------------------------------------------- setup of one configuration
    def setup(self, cfg_index, formats):
        torch, fmmt = self.torch, self.fmmt
        cfg = get_config(cfg_index)
        n, ndir = cfg.n, cfg.ndir
        d0, dn = fmmt.shard_range(ndir, self.rank, self.world)
        khat, w = fmmt.direction_grid(cfg.L, cfg.nphi)
        need4d = any(f in ("tucker4d", "htucker4d", "tt4d") for f, _ in formats)
        t0 = time.time()
        ops = []
        with torch.cuda.stream(self.stream):
            # FP64 operator (eq. (7) + FFT) on the GPU: the whole T_4D on rank 0 when a 4D format is
            # compressed there (then broadcast), otherwise each rank builds only its own directions
            full = need4d and self.rank == 0
            b0, bn = (0, ndir) if full else (d0, dn)
            T = torch.empty((bn,) + n[::-1], dtype=torch.complex128, device="cuda")
            self.ctx.build_operator(cfg.Nx, cfg.Ny, cfg.Nz, cfg.edge, cfg.k, cfg.L, khat[b0:b0 + bn], T)
            self.ctx.sync()
            loc = T[d0 - b0:d0 - b0 + dn]
            for fmt, tol in formats:
                if fmt in ("tucker3d", "tt3d"):
                    op = self.ctx.compress(loc.contiguous() if b0 != d0 or bn != dn else T, n, dn, fmt, tol)
                elif self.world > 1:
                    op = self.ctx.compress(T if self.rank == 0 else None, n, ndir, fmt, tol, d0, dn)
                else:
                    op = self.ctx.compress(T, n, ndir, fmt, tol, d0, dn)
                ops.append((fmt, tol, op))
            dense = self.ctx.compress(loc.contiguous() if b0 != d0 or bn != dn else T, n, dn, "dense", 0.5)
            del T, loc
            torch.cuda.empty_cache()
        setup_s = time.time() - t0
        return cfg, (d0, dn), w, ops, dense, setup_s

    # -------------------------------------------------------------- timed steps of one configuration
    def measure(self, cfg_index, formats, steps, warmup, full=True):
        torch = self.torch
        cfg, (d0, dn), w, ops, dense, setup_s = self.setup(cfg_index, formats)
        N = (cfg.Nx, cfg.Ny, cfg.Nz)
        ndir, npad, K = cfg.ndir, cfg.npad, cfg.K
        stream = self.stream
        res = {"workload": workload_str(cfg_index, formats), "setup_s": round(setup_s, 1)}
        with torch.cuda.stream(stream):
            sig = torch.from_numpy(signatures(signature_seed(cfg_index, 0), ndir, *N)[d0:d0 + dn]).cuda()
            sig_out = torch.empty_like(sig)
            wd = torch.from_numpy(w[d0:d0 + dn].astype(np.float32)).cuda()
            sums = torch.empty((cfg.Nz, cfg.Ny, cfg.Nx), dtype=torch.complex64, device="cuda")
            flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

            def step(events=None):
                for i, (_, _, op) in enumerate(ops):
                    if events is not None:
                        events[i][0].record(stream)
                    op.translate_sum(sig, sig_out, wd, sums, dn, N)
                    if events is not None:
                        events[i][1].record(stream)

            for _ in range(warmup):
                step()
            self.barrier()
            ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in ops]
                  for _ in range(steps)]
            l0 = self.ctx.launches
            with ClockSampler(self.local) as clk:
                self.barrier()
                for s in range(steps):
                    flush.fill_(s & 0xFF)            # L2 flush (256 MiB write) between timed steps, outside the events
                    step(ev[s])
                self.barrier()
            launches = (self.ctx.launches - l0) // max(1, steps)
            per_op = np.zeros(len(ops))
            for s in range(steps):
                for i in range(len(ops)):
                    per_op[i] += ev[s][i][0].elapsed_time(ev[s][i][1])
            per_op /= steps
            mx = self.max_over_ranks([per_op.sum()] + list(per_op))
            t_step, per_op = mx[0], np.array(mx[1:])
            res.update(t_step=t_step, per_op=per_op, launches=int(launches), clocks=clk.summary())
            if self.args.quick:
                return res, ops, dense
            # DENSE (uncompressed operator, same FFT convolution): the compression-overhead denominator
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for _ in range(2):
                dense.translate_sum(sig, sig_out, wd, sums, dn, N)
            dts = []
            for s in range(max(3, min(steps, 10))):
                flush.fill_(s & 0xFF)
                e0.record(stream)
                dense.translate_sum(sig, sig_out, wd, sums, dn, N)
                e1.record(stream)
                e1.synchronize()
                dts.append(e0.elapsed_time(e1))
            res["dense_ms"] = self.max_over_ranks([float(np.mean(dts))])[0]
            # per-kernel breakdown: one profiled (graph-captured, events around every launch) pass
            self.ctx.set_profiling(True)
            self.ctx.prof_reset()
            PROF = 2
            for _ in range(PROF):
                step()
            dense.translate_sum(sig, sig_out, wd, sums, dn, N)
            prof = self.ctx.prof_read()
            self.ctx.set_profiling(False)
            kflops = {}
            for fmt, tol, op in ops + [("dense", 0.5, dense)]:
                reps = PROF if op is not dense else 1
                for kname, v in kernel_flops(fmt, op.info(), op.ranks(), dn).items():
                    kflops[kname] = kflops.get(kname, 0.0) + v * reps
            res.update(prof=prof, kflops=kflops, prof_steps=PROF)
            if full:
                res["two_component"] = self.two_component(cfg_index, cfg, ops, d0, dn, wd, N, flush, steps)
                res["far_matvec"] = far_matvec_measure(self, ops, cfg, cfg_index, d0, dn, wd, N, flush)
                res["e2e_t"] = self.e2e(cfg_index, cfg, ops, w, d0, dn, N, flush, steps)
        res["ops"] = [(fmt, tol, op.info(), op.ranks()) for fmt, tol, op in ops]
        res["dn"] = dn
        for _, _, op in ops:
            op.close()
        dense.close()
        del sig, sig_out, flush
        torch.cuda.empty_cache()
        return res, None, None

    def two_component(self, cfg_index, cfg, ops, d0, dn, wd, N, flush, steps):
        """theta and phi signatures share one restored T_p per direction."""
        torch, stream = self.torch, self.stream
        ndir = cfg.ndir
        sig2 = torch.from_numpy(np.ascontiguousarray(
            signatures(signature_seed(cfg_index, 2), 2 * ndir, *N).reshape(ndir, 2, cfg.Nz, cfg.Ny, cfg.Nx)[d0:d0 + dn])).cuda()
        sums2 = torch.empty((2, cfg.Nz, cfg.Ny, cfg.Nx), dtype=torch.complex64, device="cuda")
        for _ in range(3):
            for _, _, op in ops:
                op.translate_sum_multi(sig2, None, wd, sums2, dn, 2, N)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ms = []
        for s in range(max(3, min(steps, 10))):
            flush.fill_(s & 0xFF)
            torch.cuda.synchronize()
            e0.record(stream)
            for _, _, op in ops:
                op.translate_sum_multi(sig2, None, wd, sums2, dn, 2, N)
            e1.record(stream)
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
        t = self.max_over_ranks([float(np.mean(ms))])[0]
        del sig2
        units = 2 * len(ops) * ndir * cfg.npad
        return {"value": round(units / (t * 1e-3) / 1e9, 3), "unit": UNIT, "ms_per_step": round(t, 4),
                "note": "theta+phi signatures [ndir][2][Nz][Ny][Nx], one restore per direction serves both "
                        "(SURVEY 8(f) NEXT #1); units count both components"}

    def e2e(self, cfg_index, cfg, ops, w, d0, dn, N, flush, steps):
        """Through the C ABI with host buffers (pinned): per step and op, H2D of the signatures and
        weights, the matvec, D2H of the direction-summed result (fmmt_translate_sum_host)."""
        torch, stream = self.torch, self.stream
        sig_h = torch.from_numpy(signatures(signature_seed(cfg_index, 1), cfg.ndir, *N)[d0:d0 + dn]).pin_memory()
        w_h = torch.from_numpy(w[d0:d0 + dn].astype(np.float32)).pin_memory()
        sum_h = torch.empty((cfg.Nz, cfg.Ny, cfg.Nx), dtype=torch.complex64).pin_memory()
        for _, _, op in ops:
            op.translate_sum_host(sig_h, w_h, sum_h, dn, N)
        self.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ms = []
        for s in range(max(3, min(steps, 10))):
            flush.fill_(s & 0xFF)
            torch.cuda.synchronize()
            e0.record(stream)
            for _, _, op in ops:
                op.translate_sum_host(sig_h, w_h, sum_h, dn, N)
            e1.record(stream)
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
        return self.max_over_ranks([float(np.mean(ms))])[0]


def far_matvec_measure(run, ops, cfg, cfg_index, d0, dn, wd, N, flush):
    """Time fmmt_far_matvec (eq. (4) aggregation -> eq. (5) -> eq. (6) disaggregation, SURVEY §8(f)
    NEXT #3) for every op; aggregation / disaggregation kernels against the HBM roofline."""
    torch = run.torch
    from synth import basis, basis_seed
    bas = basis(basis_seed(cfg_index), cfg.Nx, cfg.Ny, cfg.Nz, cfg.edge)
    K, nb, ncomp = cfg.K, bas.N, 2
    g = torch.Generator(device="cuda")
    g.manual_seed(basis_seed(cfg_index))
    P = torch.view_as_complex(torch.randn((dn, nb, ncomp, 2), generator=g, device="cuda").mul_(math.sqrt(0.5)))
    I = torch.view_as_complex(torch.randn((nb, 2), generator=g, device="cuda"))
    box = torch.from_numpy(bas.box_ptr).cuda()
    y = torch.empty((nb,), dtype=torch.complex64, device="cuda")
    for _ in range(3):
        for _, _, op in ops:
            op.far_matvec(P, I, box, wd, dn, nb, ncomp, N, y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = []
    for s in range(3):
        flush.fill_(s & 0xFF)
        torch.cuda.synchronize()
        e0.record(run.stream)
        for _, _, op in ops:
            op.far_matvec(P, I, box, wd, dn, nb, ncomp, N, y)
        e1.record(run.stream)
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    run.ctx.set_profiling(True)
    run.ctx.prof_reset()
    for _, _, op in ops:
        op.far_matvec(P, I, box, wd, dn, nb, ncomp, N, y)
    prof = run.ctx.prof_read()
    run.ctx.set_profiling(False)
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
    t = run.max_over_ranks([float(np.mean(ms))])[0]
    del P, I
    return {"ms_per_step": round(t, 4), "ops": len(ops), "basis_functions": int(nb),
            "nonempty_boxes": int((np.diff(bas.box_ptr) > 0).sum()), "ncomp": ncomp,
            "value": round(len(ops) * cfg.ndir * nb / (t * 1e-3) / 1e9, 3), "unit": "G basis-function*dir/s",
            "kernels": kern, "peak_source": src + " HBM copy bandwidth",
            "note": "eq.(4) aggregation + eq.(5) translate (both components) + eq.(6) disaggregation per op; "
                    "synthetic sphere-shell basis functions, CN(0,1) patterns drawn on the device"}


def summarize(res, world, peaks, peak_src, split="fp16"):
    """Value, per-op and step-level roofline, dominant-kernel roofline."""
    cfg_ops = res["ops"]
    dn = res["dn"]
    ndir_total = get_config(int(res["workload"].split(":")[0].replace("config", ""))).ndir
    t_step = res["t_step"]
    units_per_op = None
    per_format, troof = {}, 0.0
    total_units = 0
    for i, (fmt, tol, info, ranks) in enumerate(cfg_ops):
        npad = info["n"][0] * info["n"][1] * info["n"][2]
        units = ndir_total * npad
        total_units += units
        rf = op_roofline(fmt, info, ranks, dn, peaks, burst=True, split=split)
        troof += rf["t_roof_ms"]
        ms = float(res["per_op"][i])
        d = {"ms": round(ms, 4), "gpt_s": round(units / (ms * 1e-3) / 1e9, 3), "rank_max": info["rank_max"],
             "saving_pct": round(100 * (1 - info["compressed_bytes"] / info["original_bytes"]), 2),
             "restore_gflop_cheapest": round(rf["restore_gflop"], 3), "t_roof_ms": round(rf["t_roof_ms"], 4),
             "roofline_frac": round(rf["t_roof_ms"] / ms, 4), "bound": rf["bound"]}
        if "dense_ms" in res:
            # paper-style overhead (decompression time / convolution time with the original tensor);
            # restore is fused with the convolution here, so decompression = t(op) - t(DENSE)
            d["overhead_vs_dense"] = round(ms / res["dense_ms"] - 1, 3)
        per_format[f"{fmt}@{tol:g}"] = d
        units_per_op = units
    value = total_units / (t_step * 1e-3) / 1e9
    out = {"value": round(value, 3), "ms_per_step": round(t_step, 4), "per_format": per_format,
           "step_roofline": {"t_roof_ms": round(troof, 4), "t_ms": round(t_step, 4), "frac": round(troof / t_step, 4),
                             "definition": "sum over ops of max((B_sig+B_fac)/BW, F_restore/P_restore), cheapest "
                                           "contraction order, P_restore = measured bf16 burst / 3 (3 fp16 MMAs per "
                                           "FP32-accurate MAC; x 0.5 for the TF32-split build), BW = measured HBM copy "
                                           "(SURVEY 8(d))",
                             "p_restore_tflops": round(restore_peak_tflops(peaks, True, split), 1)},
           "gpu_launches": res["launches"], "clocks": res["clocks"], "setup_s": res["setup_s"]}
    if "dense_ms" in res:
        dms = res["dense_ms"]
        # the dense operator (complex64, read once) + signatures in and out: HBM-bound by design
        nn = cfg_ops[0][2]["n"]
        npad = nn[0] * nn[1] * nn[2]
        dbytes = 8.0 * npad * dn + 16.0 * (npad // 8) * dn
        out["dense"] = {"ms": round(dms, 4), "gbs": round(dbytes / (dms * 1e-3) / 1e9, 1),
                        "frac_hbm": round(dbytes / (dms * 1e-3) / 1e9 / float(peaks["hbm_gbs"]), 4)}
    if "prof" in res:
        prof, kfl, reps = res["prof"], res["kflops"], res["prof_steps"]
        tot = sum(v[0] for v in prof.values())
        kernels = {}
        for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0]):
            e = {"ms_per_launch": round(v[0] / v[1], 5), "launches": int(v[1]), "share": round(v[0] / tot, 4)}
            if k in kfl and k != "conv_z_dense":
                e["achieved_tflops"] = round(kfl[k] / (v[0] * 1e-3) / 1e12, 2)
            if k == "conv_z_dense":
                e["achieved_gbs"] = round(kfl[k] / (v[0] * 1e-3) / 1e9, 1)
            kernels[k] = e
        out["kernels"] = kernels
        # dominant kernel of the compressed ops (largest device time, the DENSE pass excluded)
        cand = {k: v for k, v in prof.items() if k != "conv_z_dense" and k in kfl}
        if cand:
            dname, (dms, dl) = max(cand.items(), key=lambda kv: kv[1][0])
            ach = kfl[dname] / (dms * 1e-3) / 1e12
            pk = restore_peak_tflops(peaks, burst=True, split=split)
            pks = restore_peak_tflops(peaks, burst=False, split=split)
            traffic = None
            tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
            if os.path.exists(tp):
                try:
                    traffic = json.load(open(tp)).get(dname)
                except Exception:
                    traffic = None
            out["roofline"] = {"bound": "tensor", "kernel": dname, "achieved": round(ach, 3), "peak": round(pk, 2),
                               "unit": "TFLOP/s", "frac": round(ach / pk, 4), "traffic": traffic,
                               "frac_of_sustained": round(ach / pks, 4),
                               "peak_source": (f"{peak_src}: bf16 burst {peaks.get('bf16_tflops')} / 3 (3 fp16 MMAs per "
                                               f"FP32-accurate MAC; fp16 rate = bf16) = {pk:.1f} TFLOP/s") if split == "fp16"
                                              else (f"{peak_src}: bf16 burst {peaks.get('bf16_tflops')} x 0.5 (TF32, guide's "
                                                    f"nominal ratio) / 3 (3xTF32 split) = {pk:.1f} TFLOP/s"),
                               "work": "cheapest-order a4 contraction flops of the kernel (8 per complex MAC), "
                                       "FFT / Hadamard ALU work excluded; CUDA events on the launching stream"}
    return out


def run_ours(args):
    run = Runner(args)
    peaks, peak_src = load_peaks()
    cfg = get_config(args.config)
    formats = list(cfg.formats)
    if args.formats:
        want = {(f.split("@")[0], float(f.split("@")[1])) for f in args.formats.split(",")}
        formats = [ft for ft in formats if (ft[0], ft[1]) in want]
    res, _, _ = run.measure(args.config, formats, args.steps, args.warmup, full=not args.quick)
    if args.quick:
        if run.rank == 0:
            print(json.dumps({"quick": True, "ms_per_step": res["t_step"], "launches": res["launches"]}), flush=True)
        return
    split = run.fmmt.SPLIT
    head = summarize(res, run.world, peaks, peak_src, split)
    ndir = cfg.ndir
    total_units = sum(ndir * info["n"][0] * info["n"][1] * info["n"][2] for _, _, info, _ in res["ops"])
    e2e_value = total_units / (res["e2e_t"] * 1e-3) / 1e9
    K = cfg.K
    others = {}
    if run.world == 1 and not args.no_extra:
        for ci in [int(x) for x in args.extra_configs.split(",") if x.strip()]:
            if ci == args.config:
                continue
            c2 = get_config(ci)
            r2, _, _ = run.measure(ci, list(c2.formats), max(3, args.steps // 2), 3, full=False)
            s2 = summarize(r2, 1, peaks, peak_src, split)
            others[f"config{ci}"] = {"workload": r2["workload"], **{k: s2[k] for k in (
                "value", "ms_per_step", "step_roofline", "roofline", "per_format", "dense", "gpu_launches", "setup_s")
                if k in s2}, "unit": UNIT, "kernels_top": dict(list(s2.get("kernels", {}).items())[:8])}
    if run.rank != 0:
        if run.world > 1:
            run.dist.barrier()
            run.dist.destroy_process_group()
        return
    line = {
        "metric": METRIC,
        "value": head["value"],
        "unit": UNIT,
        "n_gpus": run.world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": head["ms_per_step"],
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "c64",
        "data": "synthetic: eq.(7) operators built on GPU (FP64), GPU-compressed (FP64 Alg. 1-3); CN(0,1) seeded "
                "signatures",
        "config": {"workload": res["workload"],
                   "l2": "flushed between timed steps (256 MiB write outside the events)",
                   "parallelism": f"direction-shard x{run.world}",
                   "restore_gemm": {"tc": f"tcgen05 kind::{'f16' if split == 'fp16' else 'tf32'}, 3-product "
                                          f"{split} hi/lo split, FP32 accumulation, packed-operand pipeline",
                                    "ffma": "FP32 FFMA"}[args.gemm]},
        "gpu_launches": head["gpu_launches"],
        "roofline": head.get("roofline"),
        "step_roofline": head["step_roofline"],
        "e2e": {"value": round(e2e_value, 3), "unit": UNIT,
                "h2d_bytes_per_step": int(len(res["ops"]) * (res["dn"] * K * 8 + res["dn"] * 4)),
                "d2h_bytes_per_step": int(len(res["ops"]) * K * 8),
                "note": "fmmt_translate_sum_host per op: pinned host signatures + weights in (chunked upload on a copy stream, overlapped with the matvec), direction sum out"},
        "per_box": {"value": round(head["value"] / 8, 3), "unit": "Gdir*box/s",
                    "note": "the same rate per box of the Nx*Ny*Nz grid (8 padded points per box)"},
        "dense": head.get("dense"),
        "per_format": head["per_format"],
        "two_component": res.get("two_component"),
        "far_matvec": res.get("far_matvec"),
        "kernels": head.get("kernels"),
        "other_configs": others,
        "setup_s": head["setup_s"],
        "clocks": head["clocks"],
    }
    if run.world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.config, res["ops"], sample_dirs=args.cpu_sample)
    print(json.dumps(line), flush=True)
    if run.world > 1:
        run.dist.barrier()
        run.dist.destroy_process_group()


# ------------------------------------------------------------------ the oracle (cpu_baseline / reference arm)
def synthetic_oracle_ops(cfg_index, ops_ranks, sample, seed=7):
    """Oracle restore closures for the sample directions from seeded random factors with the given
    ranks (restore cost depends only on the ranks; the oracle's own FP64 compression of a 4D
    operator of up to 14.8 GB is setup, not the timed path).  Factors are oracle-side numpy arrays."""
    from oracle import restore
    c = get_config(cfg_index)
    n1, n2, n3 = c.n
    rng = np.random.default_rng(seed)
    cn = lambda *s: (rng.standard_normal(s) + 1j * rng.standard_normal(s)) * math.sqrt(0.5)
    ops = []
    for fmt, tol, r in ops_ranks:
        r = [int(x) for x in r]
        if fmt == "tucker3d":
            fs = {p: (cn(*r[:3]), cn(n1, r[0]), cn(n2, r[1]), cn(n3, r[2])) for p in sample}
            ops.append((fmt, tol, lambda p, fs=fs: restore.tucker3d_restore(*fs[p])))
        elif fmt == "tt3d":
            fs = {p: (cn(n1, r[0]), cn(r[0], n2, r[1]), cn(n3, r[1])) for p in sample}
            ops.append((fmt, tol, lambda p, fs=fs: restore.tt3d_restore(*fs[p])))
        elif fmt == "tucker4d":
            core, U = cn(*r[:4]), [cn(n1, r[0]), cn(n2, r[1]), cn(n3, r[2]), cn(c.ndir, r[3])]
            ops.append((fmt, tol, lambda p, core=core, U=U: restore.tucker4d_slice(core, U, p)))
        elif fmt == "htucker4d":
            L = [cn(n1, r[0]), cn(n2, r[1]), cn(n3, r[2]), cn(c.ndir, r[3])]
            c12, c34, c1234 = cn(r[0], r[1], r[4]), cn(r[2], r[3], r[5]), cn(r[4], r[5])
            ops.append((fmt, tol, lambda p, a=(L, c12, c34, c1234): restore.htucker_slice(*a, p)))
        elif fmt == "tt4d":
            u1, c1, c2, ul = cn(n1, r[0]), cn(r[0], n2, r[1]), cn(r[1], n3, r[2]), cn(c.ndir, r[2])
            t2 = restore.tt4d_t2(c2, ul)
            ops.append((fmt, tol, lambda p, a=(u1, c1, c2, ul, t2): restore.tt4d_slice(*a[:4], p, a[4])))
    return c, ops


def oracle_step(ops, sample, sig_math, w):
    from oracle import translate
    for _, _, rest in ops:
        B = [translate.translate_fft(rest(p), sig_math[i]) for i, p in enumerate(sample)]
        translate.direction_sum(np.stack(B), w[list(sample)])


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def _bench_ranks(cfg_index):
    """Per-direction ranks recorded for the paper-shaped operators of each configuration (SURVEY.md
    Appendix [probe], GPU compressor in round 1): the reference arm runs on the host only."""
    return {1: {"tucker3d": (7, 7, 7)},
            2: {"tucker3d": (26, 25, 26), "tt3d": (26, 25), "tucker4d": (27, 27, 27, 169),
                "htucker4d": (27, 27, 27, 169, 286, 286), "tt4d": (27, 281, 169)},
            3: {"tucker3d": (32, 15, 15), "tt3d": (32, 15)},
            4: {"tucker4d": (57, 57, 57, 441), "htucker4d": (57, 57, 57, 441, 952, 952)},
            5: {"tt4d": (95, 1201, 441), "tucker3d": (92, 86, 60)}}[cfg_index]


def cpu_baseline(cfg_index, ops=None, sample_dirs=8, budget_s=20.0):
    """The oracle (FP64 NumPy/SciPy restore + FFT convolution + direction sum, as it stands) on a
    bounded direction sample of the configuration, factors of the GPU op's ranks (3D formats:
    the ranks of the sampled directions); best of >= 3 repetitions after one warm-up."""
    from oracle import translate
    c = get_config(cfg_index)
    sample = list(range(0, c.ndir, max(1, c.ndir // sample_dirs)))[:sample_dirs]
    if ops is not None:
        oranks = []
        for fmt, tol, info, ranks in ops:
            if fmt in ("tucker3d", "tt3d"):
                rr = ranks.reshape(-1, len(ranks) // max(1, info["ndir"]))
                oranks.append((fmt, tol, tuple(int(x) for x in np.round(rr.mean(axis=0)))))
            else:
                oranks.append((fmt, tol, tuple(int(x) for x in ranks)))
    else:
        oranks = [(f, t, _bench_ranks(cfg_index)[f]) for f, t in c.formats]
    c, oops = synthetic_oracle_ops(cfg_index, oranks, sample)
    from oracle import fmm
    _, w, _, _ = fmm.direction_grid(c.L, c.nphi)
    sig = translate.sig_to_math(signatures(signature_seed(cfg_index, 0), c.ndir, c.Nx, c.Ny, c.Nz)[sample])
    oracle_step(oops, sample, sig, w)            # warm-up
    times = []
    t_all = time.time()
    while len(times) < 3 or (time.time() - t_all < budget_s and len(times) < 20):
        t0 = time.time()
        oracle_step(oops, sample, sig, w)
        times.append(time.time() - t0)
    dt = min(times)
    units = len(oops) * len(sample) * c.npad
    return {"value": round(units / dt / 1e9, 6), "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle",
            "cpu": _cpu_model(),
            "sample": f"config{cfg_index}: ops " + ",".join(f"{f}@{t:g} r={r}" for f, t, r in oranks)
                      + f" on {len(sample)} of {c.ndir} directions (FP64 restore from seeded factors of these ranks + "
                        f"FP64 FFT convolution + direction sum), best of {len(times)} after 1 warm-up"}


def run_reference(args):
    """--impl reference: the oracle as it stands on the box's host cores, same config / metric /
    unit; each step a bounded direction sample of the workload (rank 0 only)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    from oracle import fmm, translate
    c = get_config(args.config)
    sample = list(range(0, c.ndir, max(1, c.ndir // args.ref_sample)))[:args.ref_sample]
    t0 = time.time()
    oranks = [(f, t, _bench_ranks(args.config)[f]) for f, t in c.formats]
    c, oops = synthetic_oracle_ops(args.config, oranks, sample)
    _, w, _, _ = fmm.direction_grid(c.L, c.nphi)
    sig = translate.sig_to_math(signatures(signature_seed(args.config, 0), c.ndir, c.Nx, c.Ny, c.Nz)[sample])
    setup = time.time() - t0
    for _ in range(args.warmup):
        oracle_step(oops, sample, sig, w)
    t0 = time.time()
    for _ in range(args.steps):
        oracle_step(oops, sample, sig, w)
    dt = (time.time() - t0) / args.steps
    units = len(oops) * len(sample) * c.npad
    v = units / dt / 1e9
    line = {
        "impl": "reference", "metric": METRIC,
        "value": round(v, 6), "unit": UNIT, "n_gpus": int(os.environ.get("WORLD_SIZE", str(args.gpus))),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded factors of the "
        "configuration's ranks; oracle FP64 restore + FFT convolution)",
        "config": {"workload": workload_str(args.config, list(c.formats)), "parallelism": "host cores",
                   "sample": f"{len(sample)} of {c.ndir} directions per op"},
        "cpu_baseline": {"value": round(v, 6), "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle",
                         "cpu": _cpu_model(),
                         "sample": f"{len(sample)} of {c.ndir} directions per op, ops "
                                   + ",".join(f"{f}@{t:g} r={r}" for f, t, r in oranks) + f"; setup {setup:.1f}s untimed"},
        "e2e": {"value": round(v, 6), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the other_configs measurements")
    ap.add_argument("--extra-configs", default="2,4")
    ap.add_argument("--quick", action="store_true", help="timed steps only (for ncu launch lists)")
    ap.add_argument("--gemm", default="tc", choices=["tc", "ffma"], help="restore-GEMM kernel (A/B)")
    ap.add_argument("--formats", default=None, help="comma list fmt@tol restricting the config's ops")
    ap.add_argument("--cpu-sample", type=int, default=8)
    ap.add_argument("--ref-sample", type=int, default=4)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # self-launch one rank per GPU (the driver's torchrun command line, on 127.0.0.1)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
        print(f"[bench] launching {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
        raise SystemExit(subprocess.call(cmd))
    run_ours(args)


if __name__ == "__main__":
    main()
