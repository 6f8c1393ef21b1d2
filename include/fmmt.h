/*
 * fmmt.h -- C ABI of libfmmt, the B200 (sm_100a) implementation of the
 * FMM-FFT translation stage with compressed FFT'ed translation operators of
 * arXiv 2010.00520 (Qian & Yucel, "On the Compression of Translation Operator
 * Tensors in FMM-FFT-Accelerated SIE Simulators via Tensor Decompositions").
 *
 * Citations "P:n" are lines of the paper text.
 *
 * Conventions (all entry points)
 *   - Every function returns fmmt_status; nothing aborts, throws or prints.
 *     fmmt_last_error(ctx) returns a one-line description of the last failure
 *     on that context (the string is owned by the context).
 *   - Arrays are first-index-fastest ("Fortran order").  A 3D operator slice
 *     T_p is n1 x n2 x n3 = 2Nx x 2Ny x 2Nz, element (i1,i2,i3) at
 *     i1 + n1*(i2 + n2*i3).  A stack of directions puts p slowest:
 *     [ndir][n3][n2][n1].  Signatures are [ndir][Nz][Ny][Nx] (x fastest).
 *     Matrices n x r are column-major (element (i,a) at i + n*a).
 *   - Complex numbers are interleaved (re, im).  The hot path stores and
 *     computes in complex64 with FP32 accumulation; the setup path (operator
 *     build, compression) computes in complex128.
 *   - Device pointers must be on the context's device.  Kernels are launched
 *     asynchronously on the context's stream; fault reports surface at
 *     fmmt_sync().  Validation errors are returned synchronously.
 *   - Grid sizes: n1, n2, n3 must be powers of two in [4, 256] for the
 *     translate path (FMMT_E_UNSUPPORTED otherwise).
 *   - An op must not be used concurrently from two host threads (its
 *     workspace belongs to it).  The library owns ctx, op and all factor and
 *     workspace memory; the caller owns every buffer it passes in.
 */
#ifndef FMMT_H_
#define FMMT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FMMT_VERSION 100  /* 1.0.0 */

typedef struct { float re, im; } fmmt_c64;
typedef struct { double re, im; } fmmt_c128;

typedef struct fmmt_ctx fmmt_ctx;
typedef struct fmmt_op fmmt_op;

/* Compressed formats of the FFT'ed translation operator (eqs. (8)-(14)).
 * FMMT_DENSE is the uncompressed operator (the paper's "original tensors",
 * P:161), used as the overhead baseline.                                    */
typedef enum {
  FMMT_DENSE = 0,      /* T_p stored as is                                     */
  FMMT_TUCKER3D = 1,   /* eq. (8), per direction: C_p x1 U1_p x2 U2_p x3 U3_p  */
  FMMT_TUCKER4D = 2,   /* eq. (9): C x1 U1 x2 U2 x3 U3 x4 U4                  */
  FMMT_HTUCKER4D = 3,  /* eq. (11): leaves U1..U4, C12, C34, root C1234       */
  FMMT_TT3D = 4,       /* eq. (13), per direction: C1_p x1 U1_p x3 U3_p        */
  FMMT_TT4D = 5        /* eq. (14): (C1 x1 U1) x3^1 (C2 x3 U_last)            */
} fmmt_format;

typedef enum {
  FMMT_OK = 0,
  FMMT_E_ARG = 1,          /* null pointer, tol not in (0,1), bad enum, aliasing  */
  FMMT_E_SHAPE = 2,        /* n != 2N, ndir mismatch, rank/shape chain mismatch  */
  FMMT_E_NOMEM = 3,        /* device or host allocation failed                   */
  FMMT_E_CUDA = 4,         /* CUDA / cuBLAS / cuSOLVER error                     */
  FMMT_E_NCCL = 5,         /* NCCL error                                         */
  FMMT_E_STATE = 6,        /* wrong device, destroyed handle, not sharded        */
  FMMT_E_UNSUPPORTED = 7   /* valid input outside this build (e.g. non-pow2 n)   */
} fmmt_status;

/* ------------------------------------------------------------------ context */

/* Create a context on CUDA device `device`, launching on `cuda_stream`
 * (a cudaStream_t; NULL = the legacy default stream).                       */
fmmt_status fmmt_init(int device, void* cuda_stream, fmmt_ctx** ctx);

/* Create a context that is rank `rank` of `world` direction shards.  The
 * 128-byte NCCL unique id comes from fmmt_nccl_unique_id() on rank 0 and is
 * distributed by the caller (e.g. a torch.distributed broadcast).  All ranks
 * must call this collectively.  world == 1 needs no id (may be NULL); given
 * one, it creates a single-rank communicator and every collective of the
 * sharded path (the 4D setup broadcast, the per-matvec allreduce) still runs,
 * which is how the NCCL call sequence is exercised on a one-GPU box.        */
fmmt_status fmmt_init_sharded(int device, void* cuda_stream, int rank, int world,
                              const void* nccl_unique_id, fmmt_ctx** ctx);
fmmt_status fmmt_nccl_unique_id(void* out_128_bytes);

void fmmt_destroy(fmmt_ctx* ctx);
fmmt_status fmmt_sync(fmmt_ctx* ctx);
const char* fmmt_last_error(const fmmt_ctx* ctx);
int fmmt_version(void);

/* Contiguous block partition of `ndir` directions over `world` ranks
 * (each processor owns a set of directions).  Rank r gets
 * [*begin, *begin + *count).  Pure host arithmetic.                          */
fmmt_status fmmt_shard_range(int64_t ndir, int rank, int world, int64_t* begin, int64_t* count);

/* Profiling: when enabled, the library brackets every kernel launch with CUDA
 * events on its stream and accumulates per-kernel-class device time.
 * fmmt_prof_read fills up to `cap` entries (name is a static string).       */
fmmt_status fmmt_set_profiling(fmmt_ctx* ctx, int enable);
fmmt_status fmmt_prof_reset(fmmt_ctx* ctx);
fmmt_status fmmt_prof_read(fmmt_ctx* ctx, const char** names, double* ms, int64_t* launches,
                           int64_t cap, int64_t* count);
/* Number of kernels this context has launched since creation.               */
int64_t fmmt_launch_count(const fmmt_ctx* ctx);

/* Implementation of the restore GEMMs (Figs. 3-4 contractions): 1 = tcgen05
 * tensor cores, kind::tf32 with the 3xTF32 split and FP32 accumulation,
 * operands copied asynchronously into the UMMA layout (default); 2 = the first
 * tcgen05 design (register-staged operands); 0 = FP32 FFMA kernel.  2 and 0 are kept for A/B
 * measurement.  All are hand-written sm_100a kernels of this library; none is
 * a CPU path.                                                                */
fmmt_status fmmt_set_gemm_impl(fmmt_ctx* ctx, int impl);

/* Test hook (not the hot path): C = op(A) . op(B) for device complex64
 * column-major matrices through the restore-GEMM kernel `impl` (as above).
 * op(A) is m x k: transA = 0 reads A(i,l) at A[i + lda*l], 1 at A[l + lda*i].
 * op(B) is k x n: transB = 0 reads B(l,j) at B[l + ldb*j], 1 at B[j + ldb*l].
 * C(i,j) is written at C[i + ldc*j].  Asynchronous on the context stream.   */
fmmt_status fmmt_test_cgemm(fmmt_ctx* ctx, int impl, int64_t m, int64_t n, int64_t k, int transA, int transB,
                            const fmmt_c64* A, int64_t lda, const fmmt_c64* B, int64_t ldb,
                            fmmt_c64* C, int64_t ldc);

/* ------------------------------------------------------- setup: the operator */

/* Multipole count L = floor(x + 1.8 digits^(2/3) x^(1/3)), x = 2|k|R^s,
 * R^s = sqrt(3)/2 * edge (reading Q3 of DESIGN.md).                    */
fmmt_status fmmt_multipole_count(double k_abs, double edge, double digits, int64_t* L);

/* Direction grid: (L+1) Gauss-Legendre nodes in cos(theta), ascending,
 * times nphi uniform azimuths phi_j = 2 pi j / nphi; p = i*nphi + j.
 * khat: host [ndir][3] (x,y,z); w: host [ndir], w = w_GL * 2 pi / nphi.
 * ndir = (L+1)*nphi.  Either output may be NULL.                            */
fmmt_status fmmt_direction_grid(int64_t L, int64_t nphi, double* khat, double* w);

/* FFT'ed translation operator T_p = F(T~_p) on the 2Nx x 2Ny x 2Nz
 * circulant grid for ndir directions, written to the device buffer T
 * ([ndir][n3][n2][n1] complex128).  T~ is eq. (7) with l = 0..L and the
 * prefactor omitted (readings Q1, Q2); far iff |u|^2 > 12 (kappa = 4);
 * the m = N planes are zero (reading Q6).  k = wavenumber (2 pi / lambda).
 * khat: host [ndir][3].  Computed in FP64 on the device.                   */
fmmt_status fmmt_build_operator(fmmt_ctx* ctx, int64_t Nx, int64_t Ny, int64_t Nz,
                                double edge, double k, int64_t L,
                                const double* khat, int64_t ndir, fmmt_c128* T);

/* Lossy medium (Table IV): the same operator
 * with a complex wavenumber k = k_re + j k_im, k_im <= 0 (e^{+j omega t}:
 * eps_r = eps' - j eps'').  h_l^(2)(kR) by the upward recurrence from the closed
 * forms h_0, h_1 (FP64, complex).  Choose L from |k| (fmmt_multipole_count).
 * k_im = 0 is exactly fmmt_build_operator.  FMMT_E_ARG if k_im > 0.         */
fmmt_status fmmt_build_operator_lossy(fmmt_ctx* ctx, int64_t Nx, int64_t Ny, int64_t Nz, double edge, double k_re,
                                      double k_im, int64_t L, const double* khat, int64_t ndir, fmmt_c128* T);

/* ------------------------------------------------------- setup: compression */

/* Compress the FFT'ed operator (Alg. 1 / 2 / 3) to relative
 * Frobenius tolerance `tol` in (0,1).
 *   T: complex128 [ndir][n3][n2][n1], host or device memory (detected).
 *   3D formats compress each direction in [dir_begin, dir_begin+dir_count)
 *   separately (||T_p - T_p^||_F <= tol ||T_p||_F).  4D formats compress the
 *   whole T_4D (||T - T^|| <= tol ||T||, n4 = ndir) and keep the direction
 *   factor rows of [dir_begin, dir_begin+dir_count) (sharding).  DENSE rounds
 *   the selected slices to complex64.
 * Truncation: r = min{r >= 1 : ||sigma_{r+1:}||_2 <= tol/sqrt(m) ||T||_F},
 *   m = d (Tucker), d-1 (TT), 6 (H-Tucker; reading Q7/Q8).
 * Factors are computed in FP64 (complex128) and rounded to complex64.
 * The op translates dir_count directions.
 * Sharded 4D setup (context from fmmt_init_sharded, world > 1): collective over
 * the communicator.  Rank 0 passes the whole T_4D and compresses it; the other
 * ranks pass T = NULL.  Rank 0 broadcasts the ranks and factors (ncclBroadcast)
 * and every rank keeps the direction-factor rows of its own
 * [dir_begin, dir_begin+dir_count).  If rank 0 fails before the broadcast the
 * other ranks return FMMT_E_STATE.
 * Shapes outside the translate path (non-power-of-two n, n3 > 64, one xy plane
 * above 227 KB of shared memory) give a storage-only op: ranks, info and export
 * work, translate / restore return FMMT_E_UNSUPPORTED (paper sweeps).       */
fmmt_status fmmt_compress(fmmt_ctx* ctx, const fmmt_c128* T, int64_t n1, int64_t n2, int64_t n3,
                          int64_t ndir, int64_t dir_begin, int64_t dir_count,
                          fmmt_format format, double tol, fmmt_op** op);

/* Import factors computed elsewhere (host complex64 arrays; copied).
 * `ranks` and `arrays` per format (all matrices column-major, tensors
 * first-index-fastest, per-direction arrays concatenated over p):
 *   DENSE      ranks: NULL           arrays: T [ndir][n3][n2][n1]
 *   TUCKER3D   ranks: [ndir][3]      arrays: core_p (r1 r2 r3), U1_p (n1 x r1),
 *                                            U2_p (n2 x r2), U3_p (n3 x r3)
 *   TUCKER4D   ranks: r1 r2 r3 r4    arrays: C (r1 r2 r3 r4), U1, U2, U3, U4 (ndir x r4)
 *   HTUCKER4D  ranks: r1 r2 r3 r4 r12 r34
 *                                    arrays: U1, U2, U3, U4 (ndir x r4),
 *                                            C12 (r1 r2 r12), C34 (r3 r4 r34),
 *                                            C1234 (r12 x r34)
 *   TT3D       ranks: [ndir][2]      arrays: U1_p (n1 x r1), C1_p (r1 n2 r2), U3_p (n3 x r2)
 *   TT4D       ranks: r1 r2 r3       arrays: U1 (n1 x r1), C1 (r1 n2 r2), C2 (r2 n3 r3),
 *                                            U_last (ndir x r3)                   */
fmmt_status fmmt_op_import(fmmt_ctx* ctx, fmmt_format format, int64_t n1, int64_t n2, int64_t n3,
                           int64_t ndir, const int64_t* ranks, const fmmt_c64* const* arrays,
                           int64_t narrays, fmmt_op** op);

void fmmt_op_destroy(fmmt_op* op);

typedef struct {
  int32_t format;
  int64_t n1, n2, n3, ndir;
  int64_t rank_max[6];         /* max over directions of each rank slot            */
  double rank_mean[6];         /* mean over directions (3D formats), else = max    */
  int64_t nranks;              /* rank slots used by this format                   */
  int64_t compressed_bytes;    /* stored complex64 factor bytes (P:161 count)      */
  int64_t original_bytes;      /* 8 * n1 n2 n3 ndir                                */
  int64_t workspace_bytes;     /* device workspace owned by the op                 */
  int64_t batch;               /* directions per internal batch                    */
  double restore_cmac;         /* complex MACs of restore per matvec (a3 + a4)     */
  int64_t translatable;        /* 1: translate / restore run; 0: storage-only op   */
} fmmt_op_info_t;

fmmt_status fmmt_op_info(const fmmt_op* op, fmmt_op_info_t* info);

/* Export factor array `index` (0 <= index < the format's array count, the
 * fmmt_op_import order and layout) as complex64 into dst (host or device memory,
 * detected; cap elements).  *count = the array's element count; dst == NULL
 * only queries it.  Synchronises the context stream.  Sharded 4D ops export
 * their local direction-factor rows.  Parity hook: the GPU compressor's factors
 * go to the oracle.  Errors: FMMT_E_ARG (index, cap, null count),
 * FMMT_E_CUDA (copy).                                                            */
fmmt_status fmmt_op_export(const fmmt_op* op, int64_t index, fmmt_c64* dst, int64_t cap, int64_t* count);

/* Optional op serialisation (SURVEY.md §5 "checkpoint / resume": skip the
 * setup-time compression of Alg. 1-3, on later runs).
 * fmmt_op_save writes the op's ranks and complex64 factor arrays (exactly what
 * fmmt_op_ranks / fmmt_op_export return, so a sharded op saves its own shard)
 * to `path` (host file, overwritten); fmmt_op_load re-creates an op from such a
 * file on `ctx` as fmmt_op_import would (derived operands and plans are rebuilt;
 * shapes outside the translate path load as storage-only ops).  A loaded op's
 * translate / restore output is bit-identical to the saved op's.
 * Errors: FMMT_E_ARG (null), FMMT_E_STATE (I/O failure, not an op file,
 * truncated, checksum mismatch), otherwise as fmmt_op_export / fmmt_op_import. */
fmmt_status fmmt_op_save(const fmmt_op* op, const char* path);
fmmt_status fmmt_op_load(fmmt_ctx* ctx, const char* path, fmmt_op** op);

/* Ranks: 3D formats write [ndir][nslots] (per direction), 4D formats nslots.
 * *count = number of int64 written (fails with FMMT_E_ARG if cap is short). */
fmmt_status fmmt_op_ranks(const fmmt_op* op, int64_t* ranks, int64_t cap, int64_t* count);

/* Number of directions per internal batch (workspace and the per-plan pre-split
 * operand buffers are rebuilt).  0 = auto: batches whose rank-sized intermediates
 * fit ~48 MB (L2), enlarged for the 4D formats until the shared slice operand
 * streamed once per batch no longer dominates (<= 4 GB of intermediates). */
fmmt_status fmmt_op_set_batch(fmmt_op* op, int64_t dirs_per_batch);

/* ------------------------------------------------------------ the hot path */

/* Execution: the launches of one matvec (translate or translate_sum) are
 * replayed as a CUDA graph: the first call with a given set of buffers runs
 * directly, the second captures, later calls replay (one cudaGraphLaunch).
 * Not used on the legacy default stream, while profiling, or with the
 * environment variable FMMT_GRAPHS=0.  Call fmmt_set_gemm_impl before the
 * first translate of an op.                                                  */

/* Translation, eq. (5), for the op's ndir directions:
 *   sig_out[p] = truncate_{Nx,Ny,Nz}( F^{-1}( T_p (.) F( pad(sig_in[p]) ) ) )
 * with T_p restored from the compressed form on the fly (never stored in
 * HBM).  sig_in, sig_out: device complex64 [ndir][Nz][Ny][Nx]; must not
 * overlap.  Requires n1 = 2Nx, n2 = 2Ny, n3 = 2Nz and ndir = op's ndir.      */
fmmt_status fmmt_translate(fmmt_op* op, const fmmt_c64* sig_in, fmmt_c64* sig_out,
                           int64_t ndir, int64_t Nx, int64_t Ny, int64_t Nz);

/* Translation plus the direction sum of eq. (6) with P^- = 1:
 *   sum_out[v] = sum over ALL ranks' directions p of w[p] * sig_out[p][v]
 * (the local partial sum is NCCL-allreduced over the shards of a sharded
 * context).  w: device float [ndir] (this rank's directions).  sig_out may be
 * NULL (per-direction results are then kept in op workspace).  sum_out:
 * device complex64 [Nz][Ny][Nx].                                            */
fmmt_status fmmt_translate_sum(fmmt_op* op, const fmmt_c64* sig_in, fmmt_c64* sig_out,
                               const float* w, fmmt_c64* sum_out,
                               int64_t ndir, int64_t Nx, int64_t Ny, int64_t Nz);

/* Multi-component signatures (the aggregated far fields have a theta and
 * a phi component, both translated by the same operator).  One restoration of
 * T_p serves all ncomp components.
 *   sig_in, sig_out: device complex64 [ndir][ncomp][Nz][Ny][Nx], ncomp in [1, 16].
 *   fmmt_translate_sum_multi: sum_out [ncomp][Nz][Ny][Nx] (per-component direction
 *   sum, allreduced over shards); sig_out may be NULL.
 * ncomp = 1 is exactly fmmt_translate / fmmt_translate_sum.                  */
fmmt_status fmmt_translate_multi(fmmt_op* op, const fmmt_c64* sig_in, fmmt_c64* sig_out, int64_t ndir, int64_t ncomp,
                                 int64_t Nx, int64_t Ny, int64_t Nz);
fmmt_status fmmt_translate_sum_multi(fmmt_op* op, const fmmt_c64* sig_in, fmmt_c64* sig_out, const float* w,
                                     fmmt_c64* sum_out, int64_t ndir, int64_t ncomp, int64_t Nx, int64_t Ny,
                                     int64_t Nz);

/* End-to-end variant on HOST buffers: copies sig_in (host, [ndir][Nz][Ny][Nx])
 * and w (host) to the device, runs fmmt_translate_sum, copies the summed
 * result to sum_out (host [Nz][Ny][Nx]) and synchronises the stream.
 * Pinned host memory gives asynchronous copies: the signatures are uploaded
 * in chunks of directions on a copy stream and each chunk is awaited only by
 * the first kernel that reads it, so the upload overlaps the restore GEMMs
 * and the earlier sub-batches (FMMT_H2D_OVERLAP=0: one serial copy first).   */
fmmt_status fmmt_translate_sum_host(fmmt_op* op, const fmmt_c64* sig_in_host, const float* w_host,
                                    fmmt_c64* sum_out_host, int64_t ndir,
                                    int64_t Nx, int64_t Ny, int64_t Nz);

/* ------------------------------------------- around the translation
 *
 * Aggregation, eq. (4):  sig[p][c][v] = sum_{n in box v} P[p][n][c] * I[n],
 * zero for an empty box.  Disaggregation, eq. (6), with P- = conj(P+):
 *     y[m] = sum_p w[p] sum_c conj(P[p][m][c]) * B[p][c][v(m)].
 * Arguments (all device memory, caller-owned; the library only reads P, I, B, w, box_ptr):
 *   P        complex64 [ndir][N][ncomp]: far-field patterns P+(k_p, b_n), components
 *            (theta, phi, ...) fastest; ncomp in [1, 16]
 *   I        complex64 [N]: basis-function coefficients
 *   box_ptr  int64 [K+1], K = Nx Ny Nz: the basis functions of box v (linear index
 *            x + Nx (y + Ny z)) are n in [box_ptr[v], box_ptr[v+1]); box_ptr[0] = 0,
 *            nondecreasing, box_ptr[K] = N (basis functions numbered box by box)
 *   sig, B   complex64 [ndir][ncomp][Nz][Ny][Nx]: the layout fmmt_translate_multi uses
 *   w        float [ndir]: quadrature weights
 *   y        complex64 [N]
 * Sharded contexts: each rank passes its own direction block (P, B, w rows); y is summed
 * over ranks (ncclAllReduce).  FP32 accumulation.  Errors: FMMT_E_ARG (null or host
 * pointer, ncomp out of range), FMMT_E_SHAPE (sizes), FMMT_E_STATE (wrong device),
 * FMMT_E_NOMEM (workspace).  box_ptr contents are not validated (a malformed box_ptr is
 * undefined behaviour).  Asynchronous on the context stream.                      */
fmmt_status fmmt_aggregate(fmmt_ctx* ctx, const fmmt_c64* P, const fmmt_c64* I, const int64_t* box_ptr,
                           int64_t ndir, int64_t N, int64_t ncomp, int64_t Nx, int64_t Ny, int64_t Nz,
                           fmmt_c64* sig);
fmmt_status fmmt_disaggregate(fmmt_ctx* ctx, const fmmt_c64* P, const fmmt_c64* B, const float* w,
                              const int64_t* box_ptr, int64_t ndir, int64_t N, int64_t ncomp, int64_t Nx,
                              int64_t Ny, int64_t Nz, fmmt_c64* y);
/* The far-field part of one matrix-vector product: eq. (4) -> eq. (5) with this op's
 * compressed operators for every direction and component -> eq. (6), as one CUDA graph
 * (workspaces owned by the op).  ndir and the grid must match the op.             */
fmmt_status fmmt_far_matvec(fmmt_op* op, const fmmt_c64* P, const fmmt_c64* I, const int64_t* box_ptr,
                            const float* w, int64_t ndir, int64_t N, int64_t ncomp, int64_t Nx, int64_t Ny,
                            int64_t Nz, fmmt_c64* y);

/* Test hook (not the hot path): restore T_p (local direction index p) from
 * the compressed form into the device buffer T_p (complex64 [n3][n2][n1])
 * with the same restore kernels and arithmetic the translate path uses.     */
fmmt_status fmmt_restore(fmmt_op* op, int64_t p, fmmt_c64* T_p);

#ifdef __cplusplus
}
#endif

#endif /* FMMT_H_ */
