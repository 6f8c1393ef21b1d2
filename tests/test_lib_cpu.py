"""CPU-side checks of the C-ABI library: it loads, exports every symbol that
include/fmmt.h declares, and its pure-host entry points (multipole count,
direction grid, shard partition) agree with the paper / the oracle.  No GPU
compute is called here."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import fmm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2010_00520_b200 import build
    build.build()
    from paper_2010_00520_b200 import fmmt
    return fmmt


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "fmmt.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(fmmt_[a-z0-9_]+)\s*\(", txt)))


def test_header_symbols_exported(lib):
    syms = header_symbols()
    assert len(syms) >= 25
    so = ctypes.CDLL(lib.LIB_PATH)
    for s in syms:
        assert hasattr(so, s), s
    assert set(syms) == set(lib.EXPORTED)


def test_library_is_sm100a():
    import subprocess
    from paper_2010_00520_b200 import fmmt
    out = subprocess.run(["cuobjdump", "--list-elf", fmmt.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version(lib):
    assert lib.fmmt_version() == 100


def test_multipole_count_matches_paper(lib, golden_dir):
    import json
    g = json.load(open(os.path.join(golden_dir, "ndir.json")))
    for case in g["cases"]:
        eps = complex(*case["eps_r"])
        k_abs = abs(2 * np.pi * np.sqrt(eps))
        L = lib.multipole_count(k_abs, case["edge"], case["digits"])
        assert (L + 1) * (2 * L + 1) == case["ndir"], case["cite"]


@pytest.mark.parametrize("L,nphi", [(1, 3), (12, 26), (20, 42), (14, 29)])
def test_direction_grid_matches_oracle(lib, L, nphi):
    khat, w = lib.direction_grid(L, nphi)
    ok, ow, _, _ = fmm.direction_grid(L, nphi)
    np.testing.assert_allclose(khat, ok, atol=1e-14)
    np.testing.assert_allclose(w, ow, rtol=1e-13)
    assert abs(w.sum() - 4 * np.pi) < 1e-12


@pytest.mark.parametrize("ndir,world", [(338, 1), (338, 2), (338, 8), (882, 8), (5, 8), (1, 3)])
def test_shard_range_partition(lib, ndir, world):
    spans = [lib.shard_range(ndir, r, world) for r in range(world)]
    pos = 0
    for b, c in spans:
        assert b == pos
        pos += c
    assert pos == ndir
    cnts = [c for _, c in spans]
    assert max(cnts) - min(cnts) <= 1


def test_errors_without_gpu(lib):
    # invalid arguments are rejected before any device work
    with pytest.raises(lib.FmmtError):
        lib.multipole_count(-1.0, 0.5, 3)
    with pytest.raises(lib.FmmtError):
        lib.shard_range(10, 3, 2)


def test_null_handles_rejected_without_gpu(lib, tmp_path):
    # serialisation and the host-buffer matvec refuse null handles before touching a device or a file
    path = str(tmp_path / "x.fmmtop").encode()
    out = lib.vp()
    assert lib.fmmt_op_save(None, path) == 1            # FMMT_E_ARG
    assert lib.fmmt_op_load(None, path, lib.C.byref(out)) == 1
    assert not out.value
    assert not (tmp_path / "x.fmmtop").exists()
    assert lib.fmmt_translate_sum_host(None, None, None, None, 1, 1, 1, 1) == 1
