"""Build libfmmt.so in-tree with nvcc for sm_100a (no torch extension machinery).

    python -m paper_2010_00520_b200.build        # or build.build()

Two variants of the same sources: libfmmt.so (the product: restore contractions with the fp16
hi/lo split, FMMT_TC_F16=1) and libfmmt_tf32.so (the TF32 hi/lo split, FMMT_TC_F16=0), kept for
A/B measurement; the binding loads the second only when FMMT_LIB=tf32.
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libfmmt.so")
VARIANTS = {OUT: ["-DFMMT_TC_F16=1"], os.path.join(HERE, "libfmmt_tf32.so"): ["-DFMMT_TC_F16=0"]}
SOURCES = ["fmmt_api.cu", "fmmt_setup.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    try:
        import nvidia.nccl as nn   # the NCCL that ships with torch (2.28.x)
        base = list(nn.__path__)[0]
        return os.path.join(base, "include"), os.path.join(base, "lib")
    except Exception:
        return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def nvcc() -> str:
    for c in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if os.path.exists(c) or c == "nvcc":
            return c
    return "nvcc"


def _build_one(out: str, defs: list, verbose: bool, force: bool) -> subprocess.Popen | None:
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    deps.append(os.path.join(HERE, "..", "include", "fmmt.h"))
    deps.append(os.path.abspath(__file__))
    if not force and os.path.exists(out):
        t = os.path.getmtime(out)
        if all(os.path.getmtime(d) <= t for d in deps):
            return None
    inc, lib = _nccl_dirs()
    tag = os.path.basename(out).replace(".so", "")
    objs, procs = [], []
    for s in srcs:
        o = os.path.join(CSRC, tag + "_" + os.path.basename(s).replace(".cu", ".o"))
        cmd = [nvcc(), "-O3", "-std=c++17", "-lineinfo", *ARCH, *defs, "-Xcompiler", "-fPIC", "-Xptxas",
               "-v" if verbose else "-O3", "-I", inc, "-I", os.path.join(HERE, "..", "include"), "-c", s, "-o", o]
        procs.append((subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True), cmd))
        objs.append(o)
    return procs, objs, out, lib


def _finish(job, verbose):
    procs, objs, out, lib = job
    for p, cmd in procs:
        o, _ = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(o)
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
        if verbose:
            sys.stdout.write(o)
    tmp = out + ".tmp"
    link = [nvcc(), "-shared", *ARCH, *objs, "-o", tmp, "-L", lib, "-lnccl", "-lcublas", "-lcusolver", "-lcufft",
            "-Xlinker", "-rpath=" + lib]
    r = subprocess.run(link, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout)
        raise RuntimeError("link failed")
    os.replace(tmp, out)
    for o in objs:
        try:
            os.remove(o)
        except OSError:
            pass


def build(verbose: bool = False, force: bool = False) -> str:
    """Compile every variant that is out of date (in parallel); returns the product library path."""
    jobs = [j for j in (_build_one(out, defs, verbose, force) for out, defs in VARIANTS.items()) if j]
    for j in jobs:
        _finish(j, verbose)
    return OUT


def build_variant(tag: str, defs: list, verbose: bool = False) -> str:
    """An experimental A/B build libfmmt_<tag>.so with extra -D flags (loaded with FMMT_LIB=<tag>)."""
    out = os.path.join(HERE, f"libfmmt_{tag}.so")
    job = _build_one(out, ["-DFMMT_TC_F16=1", *defs], verbose, True)
    _finish(job, verbose)
    return out


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force=True))
