"""Thin ctypes binding of libfmmt (include/fmmt.h): argument marshalling only.

Every computation runs in the CUDA library; this module only converts Python
values and torch tensors (used for device memory and streams) into the C ABI's
plain pointers and sizes.  If the library is missing the import fails loudly:
there is no CPU fallback.

The module-level functions carry the C names (fmmt_init, fmmt_translate, ...);
`Context` and `Op` are small RAII conveniences over them.
"""
from __future__ import annotations

import ctypes as C
import os
import weakref

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# FMMT_LIB=tf32 selects the TF32-split build of the same sources (A/B measurement only); any other tag an
# experimental build libfmmt_<tag>.so made with build.build_variant(tag, defs)
_TAG = os.environ.get("FMMT_LIB")
LIB_PATH = os.path.join(_HERE, f"libfmmt_{_TAG}.so" if _TAG else "libfmmt.so")
# operand split of the loaded build's restore contractions (3 tensor MMAs per useful MAC either way)
SPLIT = "tf32" if os.environ.get("FMMT_LIB") == "tf32" else "fp16"

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"libfmmt.so not found at {LIB_PATH}: build it with `python -m paper_2010_00520_b200.build` "
        "(the translate path has no CPU fallback)")
_lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)

FMMT_DENSE, FMMT_TUCKER3D, FMMT_TUCKER4D, FMMT_HTUCKER4D, FMMT_TT3D, FMMT_TT4D = range(6)
FORMATS = {"dense": 0, "tucker3d": 1, "tucker4d": 2, "htucker4d": 3, "tt3d": 4, "tt4d": 5}
FORMAT_NAMES = {v: k for k, v in FORMATS.items()}
STATUS = {0: "FMMT_OK", 1: "FMMT_E_ARG", 2: "FMMT_E_SHAPE", 3: "FMMT_E_NOMEM", 4: "FMMT_E_CUDA",
          5: "FMMT_E_NCCL", 6: "FMMT_E_STATE", 7: "FMMT_E_UNSUPPORTED"}
NSLOTS = {0: 0, 1: 3, 2: 4, 3: 6, 4: 2, 5: 3}
NARRAYS = {0: 1, 1: 4, 2: 5, 3: 7, 4: 3, 5: 4}

vp = C.c_void_p
i64 = C.c_int64
i64p = C.POINTER(C.c_int64)


class fmmt_op_info_t(C.Structure):
    _fields_ = [("format", C.c_int32), ("n1", i64), ("n2", i64), ("n3", i64), ("ndir", i64),
                ("rank_max", i64 * 6), ("rank_mean", C.c_double * 6), ("nranks", i64),
                ("compressed_bytes", i64), ("original_bytes", i64), ("workspace_bytes", i64),
                ("batch", i64), ("restore_cmac", C.c_double), ("translatable", i64)]


def _sig(name, res, *args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


fmmt_version = _sig("fmmt_version", C.c_int)
fmmt_init = _sig("fmmt_init", C.c_int, C.c_int, vp, C.POINTER(vp))
fmmt_init_sharded = _sig("fmmt_init_sharded", C.c_int, C.c_int, vp, C.c_int, C.c_int, vp, C.POINTER(vp))
fmmt_nccl_unique_id = _sig("fmmt_nccl_unique_id", C.c_int, vp)
fmmt_destroy = _sig("fmmt_destroy", None, vp)
fmmt_sync = _sig("fmmt_sync", C.c_int, vp)
fmmt_last_error = _sig("fmmt_last_error", C.c_char_p, vp)
fmmt_shard_range = _sig("fmmt_shard_range", C.c_int, i64, C.c_int, C.c_int, i64p, i64p)
fmmt_set_profiling = _sig("fmmt_set_profiling", C.c_int, vp, C.c_int)
fmmt_prof_reset = _sig("fmmt_prof_reset", C.c_int, vp)
fmmt_prof_read = _sig("fmmt_prof_read", C.c_int, vp, C.POINTER(C.c_char_p), C.POINTER(C.c_double), i64p, i64, i64p)
fmmt_launch_count = _sig("fmmt_launch_count", i64, vp)
fmmt_multipole_count = _sig("fmmt_multipole_count", C.c_int, C.c_double, C.c_double, C.c_double, i64p)
fmmt_direction_grid = _sig("fmmt_direction_grid", C.c_int, i64, i64, vp, vp)
fmmt_build_operator = _sig("fmmt_build_operator", C.c_int, vp, i64, i64, i64, C.c_double, C.c_double, i64, vp, i64, vp)
fmmt_build_operator_lossy = _sig("fmmt_build_operator_lossy", C.c_int, vp, i64, i64, i64, C.c_double, C.c_double,
                                 C.c_double, i64, vp, i64, vp)
fmmt_compress = _sig("fmmt_compress", C.c_int, vp, vp, i64, i64, i64, i64, i64, i64, C.c_int, C.c_double, C.POINTER(vp))
fmmt_op_import = _sig("fmmt_op_import", C.c_int, vp, C.c_int, i64, i64, i64, i64, i64p, C.POINTER(vp), i64, C.POINTER(vp))
fmmt_op_destroy = _sig("fmmt_op_destroy", None, vp)
fmmt_op_save = _sig("fmmt_op_save", C.c_int, vp, C.c_char_p)
fmmt_op_load = _sig("fmmt_op_load", C.c_int, vp, C.c_char_p, C.POINTER(vp))
fmmt_op_info = _sig("fmmt_op_info", C.c_int, vp, C.POINTER(fmmt_op_info_t))
fmmt_op_ranks = _sig("fmmt_op_ranks", C.c_int, vp, i64p, i64, i64p)
fmmt_op_export = _sig("fmmt_op_export", C.c_int, vp, i64, vp, i64, i64p)
fmmt_op_set_batch = _sig("fmmt_op_set_batch", C.c_int, vp, i64)
fmmt_translate = _sig("fmmt_translate", C.c_int, vp, vp, vp, i64, i64, i64, i64)
fmmt_translate_sum = _sig("fmmt_translate_sum", C.c_int, vp, vp, vp, vp, vp, i64, i64, i64, i64)
fmmt_translate_sum_host = _sig("fmmt_translate_sum_host", C.c_int, vp, vp, vp, vp, i64, i64, i64, i64)
fmmt_restore = _sig("fmmt_restore", C.c_int, vp, i64, vp)
fmmt_translate_multi = _sig("fmmt_translate_multi", C.c_int, vp, vp, vp, i64, i64, i64, i64, i64)
fmmt_translate_sum_multi = _sig("fmmt_translate_sum_multi", C.c_int, vp, vp, vp, vp, vp, i64, i64, i64, i64, i64)
fmmt_set_gemm_impl = _sig("fmmt_set_gemm_impl", C.c_int, vp, C.c_int)
fmmt_aggregate = _sig("fmmt_aggregate", C.c_int, vp, vp, vp, vp, i64, i64, i64, i64, i64, i64, vp)
fmmt_disaggregate = _sig("fmmt_disaggregate", C.c_int, vp, vp, vp, vp, vp, i64, i64, i64, i64, i64, i64, vp)
fmmt_far_matvec = _sig("fmmt_far_matvec", C.c_int, vp, vp, vp, vp, vp, i64, i64, i64, i64, i64, i64, vp)
fmmt_test_cgemm = _sig("fmmt_test_cgemm", C.c_int, vp, C.c_int, i64, i64, i64, C.c_int, C.c_int, vp, i64, vp, i64, vp, i64)

EXPORTED = [
    "fmmt_version", "fmmt_init", "fmmt_init_sharded", "fmmt_nccl_unique_id", "fmmt_destroy", "fmmt_sync",
    "fmmt_last_error", "fmmt_shard_range", "fmmt_set_profiling", "fmmt_prof_reset", "fmmt_prof_read",
    "fmmt_launch_count", "fmmt_multipole_count", "fmmt_direction_grid", "fmmt_build_operator", "fmmt_compress",
    "fmmt_op_import", "fmmt_op_destroy", "fmmt_op_info", "fmmt_op_ranks", "fmmt_op_export", "fmmt_op_save", "fmmt_op_load", "fmmt_op_set_batch", "fmmt_translate",
    "fmmt_translate_sum", "fmmt_translate_sum_host", "fmmt_restore", "fmmt_set_gemm_impl", "fmmt_test_cgemm",
    "fmmt_translate_multi", "fmmt_translate_sum_multi", "fmmt_build_operator_lossy",
    "fmmt_aggregate", "fmmt_disaggregate", "fmmt_far_matvec",
]


class FmmtError(RuntimeError):
    pass


def _ptr(x):
    """Device or host pointer of a torch tensor / numpy array / int."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if isinstance(x, np.ndarray):
        assert x.flags["C_CONTIGUOUS"]
        return x.ctypes.data
    # torch tensor
    assert x.is_contiguous(), "tensor must be contiguous"
    return x.data_ptr()


def _check(st, ctx=None, what=""):
    if st != 0:
        msg = fmmt_last_error(ctx).decode() if ctx else ""
        raise FmmtError(f"{what}: {STATUS.get(st, st)} {msg}")


# ------------------------------------------------------------------ host helpers
def multipole_count(k_abs: float, edge: float, digits: float) -> int:
    L = C.c_int64()
    _check(fmmt_multipole_count(k_abs, edge, digits, C.byref(L)), what="fmmt_multipole_count")
    return L.value


def direction_grid(L: int, nphi: int):
    nd = (L + 1) * nphi
    khat = np.zeros((nd, 3), dtype=np.float64)
    w = np.zeros(nd, dtype=np.float64)
    _check(fmmt_direction_grid(L, nphi, khat.ctypes.data, w.ctypes.data), what="fmmt_direction_grid")
    return khat, w


def shard_range(ndir: int, rank: int, world: int):
    b, c = C.c_int64(), C.c_int64()
    _check(fmmt_shard_range(ndir, rank, world, C.byref(b), C.byref(c)), what="fmmt_shard_range")
    return b.value, c.value


def nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    _check(fmmt_nccl_unique_id(C.cast(buf, vp)), what="fmmt_nccl_unique_id")
    return bytes(buf)


# ------------------------------------------------------------------ context / op
class Context:
    def __init__(self, device: int = 0, stream: int | None = None, rank: int = 0, world: int = 1,
                 nccl_id: bytes | None = None):
        h = vp()
        if world == 1 and nccl_id is None:
            st = fmmt_init(device, stream, C.byref(h))
        else:
            idbuf = C.create_string_buffer(nccl_id, 128)
            st = fmmt_init_sharded(device, stream, rank, world, C.cast(idbuf, vp), C.byref(h))
        _check(st, None, "fmmt_init")
        self.h = h
        self.device, self.rank, self.world = device, rank, world
        self._ops = weakref.WeakSet()     # live ops: destroyed before the context (they reference it)

    def close(self):
        if self.h:
            for op in list(self._ops):
                op.close()
            fmmt_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sync(self):
        _check(fmmt_sync(self.h), self.h, "fmmt_sync")

    @property
    def launches(self) -> int:
        return fmmt_launch_count(self.h)

    def set_profiling(self, on: bool):
        _check(fmmt_set_profiling(self.h, 1 if on else 0), self.h, "fmmt_set_profiling")

    def prof_reset(self):
        _check(fmmt_prof_reset(self.h), self.h, "fmmt_prof_reset")

    def prof_read(self) -> dict:
        cnt = C.c_int64()
        names = (C.c_char_p * 64)()
        ms = (C.c_double * 64)()
        la = (C.c_int64 * 64)()
        _check(fmmt_prof_read(self.h, names, ms, la, 64, C.byref(cnt)), self.h, "fmmt_prof_read")
        return {names[i].decode(): (ms[i], la[i]) for i in range(min(64, cnt.value))}

    def set_gemm_impl(self, impl: str):
        _check(fmmt_set_gemm_impl(self.h, {"ffma": 0, "tc": 1}[impl]), self.h, "fmmt_set_gemm_impl")

    def test_cgemm(self, impl: str, m, n, k, A, lda, B, ldb, Cout, ldc, transA=0, transB=0):
        _check(fmmt_test_cgemm(self.h, {"ffma": 0, "tc": 1}[impl], m, n, k, transA, transB, _ptr(A), lda, _ptr(B), ldb,
                               _ptr(Cout), ldc), self.h, "fmmt_test_cgemm")

    def build_operator(self, Nx, Ny, Nz, edge, k, L, khat: np.ndarray, out):
        khat = np.ascontiguousarray(khat, dtype=np.float64)
        _check(fmmt_build_operator(self.h, Nx, Ny, Nz, edge, k, L, khat.ctypes.data, len(khat), _ptr(out)),
               self.h, "fmmt_build_operator")

    def build_operator_lossy(self, Nx, Ny, Nz, edge, k: complex, L, khat: np.ndarray, out):
        khat = np.ascontiguousarray(khat, dtype=np.float64)
        _check(fmmt_build_operator_lossy(self.h, Nx, Ny, Nz, edge, float(k.real), float(k.imag), L, khat.ctypes.data,
                                         len(khat), _ptr(out)), self.h, "fmmt_build_operator_lossy")

    def compress(self, T, n, ndir, fmt, tol, dir_begin=0, dir_count=None) -> "Op":
        """T: complex128 [ndir][n3][n2][n1] (host or device).  Sharded 4D formats (world > 1): rank 0
        passes the whole T_4D, the other ranks pass T=None (the factors are broadcast)."""
        fmt = FORMATS[fmt] if isinstance(fmt, str) else fmt
        dir_count = ndir - dir_begin if dir_count is None else dir_count
        h = vp()
        _check(fmmt_compress(self.h, _ptr(T), n[0], n[1], n[2], ndir, dir_begin, dir_count, fmt, tol, C.byref(h)),
               self.h, "fmmt_compress")
        return Op(self, h)

    def aggregate(self, P, I, box_ptr, ndir, N_basis, ncomp, N, sig):
        """eq. (4): sig[p][c][Nz][Ny][Nx] from patterns P [ndir][N_basis][ncomp] and coefficients I."""
        _check(fmmt_aggregate(self.h, _ptr(P), _ptr(I), _ptr(box_ptr), ndir, N_basis, ncomp, N[0], N[1], N[2],
                              _ptr(sig)), self.h, "fmmt_aggregate")

    def disaggregate(self, P, B, w, box_ptr, ndir, N_basis, ncomp, N, y):
        """eq. (6): y[m] = sum_p w_p sum_c conj(P[p][m][c]) B[p][c][v(m)]."""
        _check(fmmt_disaggregate(self.h, _ptr(P), _ptr(B), _ptr(w), _ptr(box_ptr), ndir, N_basis, ncomp,
                                 N[0], N[1], N[2], _ptr(y)), self.h, "fmmt_disaggregate")

    def import_op(self, fmt, n, ndir, ranks, arrays) -> "Op":
        """arrays: list of complex64 numpy arrays (flattened in library layout)."""
        fmt = FORMATS[fmt] if isinstance(fmt, str) else fmt
        arrs = [np.ascontiguousarray(a, dtype=np.complex64) for a in arrays]
        ptrs = (vp * len(arrs))(*[a.ctypes.data for a in arrs])
        rk = None
        if ranks is not None:
            rk_np = np.ascontiguousarray(np.asarray(ranks, dtype=np.int64).ravel())
            rk = rk_np.ctypes.data_as(i64p)
        h = vp()
        _check(fmmt_op_import(self.h, fmt, n[0], n[1], n[2], ndir, rk, ptrs, len(arrs), C.byref(h)),
               self.h, "fmmt_op_import")
        return Op(self, h)

    def load_op(self, path) -> "Op":
        h = vp()
        _check(fmmt_op_load(self.h, os.fsencode(path), C.byref(h)), self.h, "fmmt_op_load")
        return Op(self, h)


class Op:
    def __init__(self, ctx: Context, h):
        self.ctx, self.h = ctx, h
        ctx._ops.add(self)

    def close(self):
        if self.h:
            fmmt_op_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> dict:
        i = fmmt_op_info_t()
        _check(fmmt_op_info(self.h, C.byref(i)), self.ctx.h, "fmmt_op_info")
        nr = i.nranks
        return dict(format=FORMAT_NAMES[i.format], n=(i.n1, i.n2, i.n3), ndir=i.ndir,
                    rank_max=list(i.rank_max[:nr]), rank_mean=list(i.rank_mean[:nr]),
                    compressed_bytes=i.compressed_bytes, original_bytes=i.original_bytes,
                    workspace_bytes=i.workspace_bytes, batch=i.batch, restore_cmac=i.restore_cmac,
                    translatable=bool(i.translatable))

    def export(self) -> list:
        """The op's complex64 factor arrays, in fmmt_op_import order (flat, library layout)."""
        fmt = self.info()["format"]
        out = []
        for idx in range(NARRAYS[FORMATS[fmt]]):
            cnt = C.c_int64()
            _check(fmmt_op_export(self.h, idx, None, 0, C.byref(cnt)), self.ctx.h, "fmmt_op_export")
            a = np.zeros(max(1, cnt.value), dtype=np.complex64)
            _check(fmmt_op_export(self.h, idx, a.ctypes.data, len(a), C.byref(cnt)), self.ctx.h, "fmmt_op_export")
            out.append(a[:cnt.value])
        return out

    def save(self, path):
        _check(fmmt_op_save(self.h, os.fsencode(path)), self.ctx.h, "fmmt_op_save")

    def ranks(self) -> np.ndarray:
        cnt = C.c_int64()
        _check(fmmt_op_ranks(self.h, None, 0, C.byref(cnt)), self.ctx.h, "fmmt_op_ranks")
        out = np.zeros(max(1, cnt.value), dtype=np.int64)
        _check(fmmt_op_ranks(self.h, out.ctypes.data_as(i64p), len(out), C.byref(cnt)), self.ctx.h, "fmmt_op_ranks")
        return out[:cnt.value]

    def set_batch(self, dirs: int):
        _check(fmmt_op_set_batch(self.h, dirs), self.ctx.h, "fmmt_op_set_batch")

    def translate(self, sig_in, sig_out, ndir, N):
        _check(fmmt_translate(self.h, _ptr(sig_in), _ptr(sig_out), ndir, N[0], N[1], N[2]), self.ctx.h,
               "fmmt_translate")

    def translate_sum(self, sig_in, sig_out, w, sum_out, ndir, N):
        _check(fmmt_translate_sum(self.h, _ptr(sig_in), _ptr(sig_out), _ptr(w), _ptr(sum_out), ndir, N[0], N[1], N[2]),
               self.ctx.h, "fmmt_translate_sum")

    def translate_sum_host(self, sig_in_host, w_host, sum_out_host, ndir, N):
        _check(fmmt_translate_sum_host(self.h, _ptr(sig_in_host), _ptr(w_host), _ptr(sum_out_host), ndir,
                                       N[0], N[1], N[2]), self.ctx.h, "fmmt_translate_sum_host")

    def translate_multi(self, sig_in, sig_out, ndir, ncomp, N):
        _check(fmmt_translate_multi(self.h, _ptr(sig_in), _ptr(sig_out), ndir, ncomp, N[0], N[1], N[2]), self.ctx.h,
               "fmmt_translate_multi")

    def translate_sum_multi(self, sig_in, sig_out, w, sum_out, ndir, ncomp, N):
        _check(fmmt_translate_sum_multi(self.h, _ptr(sig_in), _ptr(sig_out), _ptr(w), _ptr(sum_out), ndir, ncomp,
                                        N[0], N[1], N[2]), self.ctx.h, "fmmt_translate_sum_multi")

    def far_matvec(self, P, I, box_ptr, w, ndir, N_basis, ncomp, N, y):
        """eq. (4) -> eq. (5) with this op -> eq. (6), one graph."""
        _check(fmmt_far_matvec(self.h, _ptr(P), _ptr(I), _ptr(box_ptr), _ptr(w), ndir, N_basis, ncomp,
                               N[0], N[1], N[2], _ptr(y)), self.ctx.h, "fmmt_far_matvec")

    def restore(self, p: int, out):
        _check(fmmt_restore(self.h, p, _ptr(out)), self.ctx.h, "fmmt_restore")
