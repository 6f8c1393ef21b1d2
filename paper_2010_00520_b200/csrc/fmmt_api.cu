// fmmt_api.cu -- C ABI of libfmmt: contexts, ops, and the translate hot path
// (eq. (5) with on-the-fly restoration).
//
// Per matvec the op walks its directions in batches of PB (sized so the
// batch's intermediates stay L2-resident) and launches, per batch:
//   [a3]  direction-slice GEMMs (4D formats)              k_cgemm
//   [a4]  restore chain up to G_p = (C_p x1 U1 x2 U2)      k_cgemm
//   [a2]  pruned forward DFT along x, y                    k_fwd_xy
//   [a4,a5,a2,a6] last restore contraction fused with the z-DFT, the Hadamard
//         product and the truncated inverse z-DFT          k_conv_z
//   [a6]  truncated inverse DFT along y, x, 1/n scaling    k_inv_xy
// and, for translate_sum, the weighted direction sum (a7) + NCCL allreduce.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "fmmt_internal.h"
#include "kernels_agg.cuh"
#include "kernels_dense.cuh"
#include "kernels_fft.cuh"
#include "kernels_fft_big.cuh"
#include "kernels_gemm.cuh"
#include "kernels_tcgemm.cuh"
#include "kernels_tcpk.cuh"
#include "kernels_tcfuse.cuh"

using fmmt::GemmDesc;
using fmmt::ZArgs;

// ============================================================== errors
namespace fmmt_internal {
fmmt_status set_err(fmmt_ctx* ctx, fmmt_status st, const char* fmt, ...) {
  if (ctx) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    ctx->err = buf;
  }
  return st;
}
}  // namespace fmmt_internal
using fmmt_internal::set_err;

#define CHECK_ARG(ctx, cond, ...) \
  do {                            \
    if (!(cond)) return set_err((ctx), FMMT_E_ARG, __VA_ARGS__); \
  } while (0)
#define CHECK_SHAPE(ctx, cond, ...) \
  do {                              \
    if (!(cond)) return set_err((ctx), FMMT_E_SHAPE, __VA_ARGS__); \
  } while (0)

static bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }

// ============================================================== profiling / launches
static cudaEvent_t take_event(fmmt_ctx* ctx) {
  if (!ctx->event_pool.empty()) {
    cudaEvent_t e = ctx->event_pool.back();
    ctx->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

struct ProfScope {
  fmmt_ctx* ctx;
  const char* name;
  cudaEvent_t e0 = nullptr;
  ProfScope(fmmt_ctx* c, const char* n) : ctx(c), name(n) {
    ctx->launches++;
    nvtxRangePushA(n);   // host-side launch ranges (per-stage NVTX)
    if (ctx->profiling) {
      e0 = take_event(ctx);
      cudaEventRecordWithFlags(e0, ctx->stream, cudaEventRecordExternal);   // graph node when captured
    }
  }
  ~ProfScope() {
    nvtxRangePop();
    if (ctx->profiling) {
      cudaEvent_t e1 = take_event(ctx);
      cudaEventRecordWithFlags(e1, ctx->stream, cudaEventRecordExternal);
      ctx->pending.push_back({name, e0, e1});
    }
  }
};

static void prof_flush(fmmt_ctx* ctx) {
  if (ctx->pending.empty()) return;
  cudaStreamSynchronize(ctx->stream);
  for (auto ex : ctx->prof_execs) cudaGraphExecDestroy((cudaGraphExec_t)ex);
  ctx->prof_execs.clear();
  for (auto& pe : ctx->pending) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, pe.e0, pe.e1);
    bool found = false;
    for (auto& kv : ctx->prof)
      if (strcmp(kv.first, pe.name) == 0) {
        kv.second.first += ms;
        kv.second.second += 1;
        found = true;
        break;
      }
    if (!found) ctx->prof.push_back({pe.name, {ms, 1}});
    ctx->event_pool.push_back(pe.e0);
    ctx->event_pool.push_back(pe.e1);
  }
  ctx->pending.clear();
}

// ============================================================== kernel dispatch
// Raise a kernel's dynamic shared-memory limit once per process (not per launch:
// the call is host-side work on the launch path and must stay out of graph capture).
static cudaError_t set_smem_once(const void* fn, int bytes, bool max_carveout = false) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> done;
  std::lock_guard<std::mutex> lk(mu);
  auto it = done.find(fn);
  if (it != done.end() && it->second >= bytes) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  // the largest shared-memory carveout for kernels sized so that two CTAs share an SM
  if (e == cudaSuccess && max_carveout)
    e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (e == cudaSuccess) done[fn] = bytes;
  return e;
}

namespace {

bool xy_big_enabled = true;   // FMMT_XY_BIG=0: the chunked four-step kernels for every plane size (A/B)
bool xy_half_enabled = true;   // FMMT_XY_HALF=0: the full-plane kernels for the one-plane-per-CTA sizes (A/B)

struct XYKernels {
  void (*fwd)(const float2*, float2*, int, int) = nullptr;
  void (*inv)(const float2*, float2*, int, int, float) = nullptr;
  int plane_smem = 0;     // complex elements per plane
  int lines = 0;          // max concurrent line-items per plane (for planes-per-CTA)
  int big_pp = 0;         // > 0: whole-plane kernels (kernels_fft_big.cuh), big_pp planes per 512-thread CTA
  int big_smem = 0;       // their dynamic shared memory (bytes)
  int big_smem_fwd = 0;   // the forward kernel's when it differs (half-buffer kernel, one plane per CTA)
};

// planes per CTA of the whole-plane kernels: the most of {4, 2, 1} whose buffers fit ~210 KB (0: none fits)
template <int NX, int NY>
constexpr int xy_big_pp() {
  return (NX < 64 || NY < 64 || NX > FMMT_TW_NMAX || NY > FMMT_TW_NMAX) ? 0
         : (4 * NY * (NX + 1) + NX + NY) * 8 <= (210 << 10) ? 4
         : (2 * NY * (NX + 1) + NX + NY) * 8 <= (210 << 10) ? 2
         : (NY * (NX + 1) + NX + NY) * 8 <= (227 << 10) ? 1 : 0;
}

template <int NX, int NY>
XYKernels make_xy_big(XYKernels k) {
  constexpr int PP = xy_big_pp<NX, NY>();
  if constexpr (PP > 0) {
    k.fwd = fmmt::k_fwd_xy_big<NX, NY, PP>;
    k.inv = fmmt::k_inv_xy_big<NX, NY, PP>;
    k.big_pp = PP;
    k.big_smem = fmmt::XYBig<NX, NY, PP>::SMEM;
    k.big_smem_fwd = k.big_smem;
    if constexpr (PP == 1) {
      if (xy_half_enabled) {
        k.fwd = fmmt::k_fwd_xy_half<NX, NY>;
        k.big_smem_fwd = fmmt::XYHalf<NX, NY>::SMEM;
        k.inv = fmmt::k_inv_xy_half<NX, NY>;
        k.big_smem = fmmt::XYInvHalf<NX, NY>::SMEM;
      }
    }
  }
  return k;
}

template <int NX, int NY>
XYKernels make_xy() {
  using G = fmmt::XYGeom<NX, NY>;
  using SX = fmmt::Split<NX>;
  using SY = fmmt::Split<NY>;
  XYKernels k;
  k.fwd = fmmt::k_fwd_xy<NX, NY>;
  k.inv = fmmt::k_inv_xy<NX, NY>;
  k.plane_smem = G::PLANE_SMEM;
  int lx = SX::two_pass ? G::XR * std::max(SX::A, SX::B) : G::Ny;   // line items per pass (chunked four-step)
  int ly = SY::two_pass ? G::YC * std::max(SY::A, SY::B) : NX;
  k.lines = std::max(lx, ly);
  if (xy_big_enabled) k = make_xy_big<NX, NY>(k);
  return k;
}

template <int NX>
XYKernels make_xy_ny(int ny) {
  switch (ny) {
    case 4: return make_xy<NX, 4>();
    case 8: return make_xy<NX, 8>();
    case 16: return make_xy<NX, 16>();
    case 32: return make_xy<NX, 32>();
    case 64: return make_xy<NX, 64>();
    case 128: return make_xy<NX, 128>();
    case 256: return make_xy<NX, 256>();
  }
  return XYKernels{};
}

XYKernels get_xy(int nx, int ny) {
  switch (nx) {
    case 4: return make_xy_ny<4>(ny);
    case 8: return make_xy_ny<8>(ny);
    case 16: return make_xy_ny<16>(ny);
    case 32: return make_xy_ny<32>(ny);
    case 64: return make_xy_ny<64>(ny);
    case 128: return make_xy_ny<128>(ny);
    case 256: return make_xy_ny<256>(ny);
  }
  return XYKernels{};
}

using ZFn = void (*)(ZArgs);
struct ZKernel {
  ZFn fn = nullptr;
  int S = 1;
};

template <int N3>
ZKernel make_z(int mode) {
  constexpr int S = (N3 <= 32) ? 1 : 2;
  ZKernel k;
  k.S = S;
  if (mode == fmmt::Z_DENSE) {
    k.fn = fmmt::k_conv_z_dense<N3, S>;
  } else if (mode == fmmt::Z_LOWRANK) k.fn = fmmt::k_conv_z<N3, S, fmmt::Z_LOWRANK>;
  else k.fn = fmmt::k_conv_z<N3, S, fmmt::Z_RESTORE>;
  return k;
}

ZKernel get_z(int n3, int mode) {
  switch (n3) {
    case 4: return make_z<4>(mode);
    case 8: return make_z<8>(mode);
    case 16: return make_z<16>(mode);
    case 32: return make_z<32>(mode);
    case 64: return make_z<64>(mode);
  }
  return ZKernel{};
}

}  // namespace

// ============================================================== op
struct GemmLaunch {
  int first = 0;       // index into op->descs
  int ndesc = 0;
  int maxtiles = 0;    // FFMA kernel: for the chosen tile size
  int maxsub = 0;
  bool big = false;    // FFMA kernel: 64x64 tiles
  int tc_bn = 64;      // tensor-core kernel: complex columns per tile
  int tc_maxtiles = 0; // tensor-core kernel: tiles of 128 x tc_bn
  const char* name = "";
  // pre-split the (dynamic) B operand of descriptor `first` into pack_dst before the launch
  float* pack_dst = nullptr;
  // pre-split the (dynamic) A operands of the launch's descriptors into their Ap before the launch
  bool pack_a_dyn = false;
};

struct Batch {
  int q0 = 0, nq = 0;
  std::vector<GemmLaunch> gemms;
  int zp_first = -1, zp_n = 0;   // z-stage: descriptors packing this batch's G_q (k_pk_pack_a_multi)
};

struct fmmt_op {
  fmmt_ctx* ctx = nullptr;
  fmmt_format format = FMMT_DENSE;
  int64_t n1 = 0, n2 = 0, n3 = 0, ndir = 0;
  int nslots = 0;
  std::vector<int64_t> ranks;                  // [ndir][nslots] (3D) or [nslots]
  std::vector<float2*> arr;                    // device factor arrays (import order)
  std::vector<int64_t> arr_elems;
  std::vector<std::vector<int64_t>> off;       // per array, per direction offsets (3D formats)
  int64_t* d_voff = nullptr;                   // per direction offset of the z-stage V factor
  int* d_rank = nullptr;                       // per direction z-stage rank (3D formats)
  // fused Tucker-3D chain (kernels_tcfuse.cuh, fmmt_ctx::z_fuse): per batch one mode-2 GEMM into H' (op->H),
  // then k_tucker_zf per xy sub-batch
  bool zfused = false;
  int* d_rank3 = nullptr;                      // [ndir][3] Tucker-3D ranks
  float* u1pk = nullptr;                       // U1 of every direction packed as an A operand (n1 rows, K = r1)
  int64_t* d_u1p_off = nullptr;
  int64_t h_stride = 0;                        // H' elements per batch-local direction
  float2* tbar1 = nullptr;                     // TT-4D: T1 = U1 . C1 (Fig. 4(a) step 1), n1 n2 x r2
  float2* E = nullptr;                         // H-Tucker: (C12 . C1234) x1 U1 x2 U2, n1 n2 x r34
  float* tbar1_pk = nullptr;                   // T1 pre-split for the tensor-core z-stage (k_tc_pack_a)
  float* E_pk = nullptr;                       // E pre-split for the tensor-core G step
  int64_t w_ncomp = 1;                         // signature components W is allocated for
  // workspace
  int64_t PB = 0;
  int64_t sigtmp_elems = 0;
  float2 *W = nullptr, *H = nullptr, *Gw = nullptr, *Cw = nullptr, *Mw = nullptr, *Nw = nullptr,
         *Vw = nullptr, *sigtmp = nullptr, *partial = nullptr;
  // every device buffer the op owns (factors, derived/pre-split operands, workspaces), with its bytes and kind:
  // fmmt_op_info sums it, fmmt_op_destroy frees what is left
  std::unordered_map<const void*, std::pair<int64_t, int>> mem;
  int64_t r1max = 1, r2max = 1, r3max = 1, rGmax = 1;     // workspace rank bounds
  std::vector<GemmDesc> descs;
  GemmDesc* d_descs = nullptr;
  std::vector<Batch> batches;
  int64_t partial_elems = 0;
  // CUDA graphs of whole matvecs, keyed by the buffers they read / write
  struct GraphEntry {
    const void* key[6];
    int calls = 0;
    cudaGraphExec_t exec = nullptr;
    int64_t launches = 0;   // kernels inside the graph
  };
  std::vector<GraphEntry> graphs;
  int64_t SB = 1;                              // directions per xy sub-batch (ensure_w)
  bool translatable = true;                    // false: storage-only op (compress beyond the translate shapes)
  // fp16-split operand scales: device max(|Re|, |Im|) slots.  [0, 7) factor arrays, 7 TT-4D T1, 8 H-Tucker E
  // (set once per op); from SLOT_DYN on, 4 per batch for the intermediates its launches produce (reset to 0
  // at the start of every matvec; the producing GEMM folds its max |C| in, the consumer derives its scale)
  float* d_slots = nullptr;
  int64_t nslots_dyn = 0;
  // packed-operand pipeline (kernels_tcpk.cuh): dynamic A workspaces per launch position of a batch,
  // the z-stage's packed G_q (per batch-local q) and packed static V factors (per direction p)
  std::vector<float*> apk_dyn;
  float* gpk = nullptr;
  int64_t gp_stride = 0;
  float* vpk_static = nullptr;
  int64_t* d_vp_off = nullptr;
  int64_t vp_stride = 0;
  bool packed = false;                         // finalize_packs ran for the tensor-core pipeline
  fmmt::PkB* d_vitems = nullptr;               // TT-4D: pack items of the batch's V_q (per q [, parity])
  int64_t nvitems = 0;
  std::vector<std::pair<std::vector<int64_t>, float*>> pk_cache;   // static operand packs (key -> buffer)
  // host staging for translate_sum_host
  float2* d_in_host = nullptr;   // device buffer for e2e input
  float* d_w_host = nullptr;
  float2* d_sum_host = nullptr;
  // overlapped upload (fmmt_translate_sum_host): events of the chunks of h2d_chunk directions, waited on by
  // translate_impl just before the first kernel that reads a chunk's signatures
  const cudaEvent_t* h2d_ev = nullptr;
  int64_t h2d_chunk = 0;
  int h2d_nchunks = 0, h2d_waited = 0;
  // far-field matvec (fmmt_far_matvec): aggregated and translated signatures [ndir][ncomp][K]
  float* Vpk = nullptr;                         // TT-4D z-stage: pre-split V_q of a batch (k_tc_pack_b)
  int64_t vpk_floats = 0;
  float2 *fA = nullptr, *fB = nullptr, *fPart = nullptr;   // + disaggregation partials [nsplit][N]
  int64_t fAB_elems = 0, fPart_elems = 0;
};

static int64_t rk(const fmmt_op* op, int64_t p, int slot) {
  if (op->format == FMMT_TUCKER3D || op->format == FMMT_TT3D) return op->ranks[p * op->nslots + slot];
  return op->ranks[slot];
}

// Destroy the op's captured matvec graphs (they hold workspace pointers); waits for the stream.
static void drop_graphs(fmmt_op* op) {
  cudaStreamSynchronize(op->ctx->stream);
  for (auto& g : op->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  op->graphs.clear();
}

enum MemKind { MEM_FACTOR = 0, MEM_DERIVED = 1, MEM_WORKSPACE = 2 };

template <class T>
static fmmt_status dev_alloc(fmmt_op* op, T** p, int64_t bytes, int kind, const char* what) {
  *p = nullptr;
  void* q = nullptr;
  cudaError_t e = cudaMalloc(&q, (size_t)std::max<int64_t>(bytes, 16));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_err(op->ctx, FMMT_E_NOMEM, "%s: cudaMalloc(%lld B) failed: %s", what, (long long)bytes, cudaGetErrorString(e));
  }
  op->mem[q] = {std::max<int64_t>(bytes, 16), kind};
  *p = static_cast<T*>(q);
  return FMMT_OK;
}

template <class T>
static void dev_free(fmmt_op* op, T*& p) {
  if (!p) return;
  cudaFree((void*)p);
  op->mem.erase((const void*)p);
  p = nullptr;
}

static int64_t mem_bytes(const fmmt_op* op, int kind) {
  int64_t b = 0;
  for (auto& kv : op->mem)
    if (kv.second.second == kind) b += kv.second.first;
  return b;
}

static void free_workspace(fmmt_op* op) {
  float2** bufs[] = {&op->W, &op->H, &op->Gw, &op->Cw, &op->Mw, &op->Nw, &op->Vw, &op->sigtmp, &op->partial};
  for (auto b : bufs) dev_free(op, *b);
  op->partial_elems = 0;
  op->sigtmp_elems = 0;
  dev_free(op, op->d_descs);
}

void fmmt_op_destroy(fmmt_op* op) {
  if (!op) return;
  cudaSetDevice(op->ctx->device);
  cudaStreamSynchronize(op->ctx->stream);
  for (auto& g : op->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  for (auto& kv : op->mem) cudaFree((void*)kv.first);
  delete op;
}

constexpr int SLOT_T1 = 7, SLOT_E = 8, SLOT_DYN = 16, SLOTS_PER_BATCH = 4;
static const float* sslot(const fmmt_op* op, int i) { return op->d_slots + i; }
static float* dslot(const fmmt_op* op, int batch, int stage) {
  return op->d_slots + SLOT_DYN + (int64_t)batch * SLOTS_PER_BATCH + stage;
}

// per-direction workspace bytes for batch sizing: every buffer sized by the batch (PB directions)
static int64_t per_dir_ws(const fmmt_op* op) {
  const int64_t n12 = op->n1 * op->n2;
  int64_t e = 0;   // complex elements (W, the half-padded spectra, is allocated for all directions)
  switch (op->format) {
    case FMMT_DENSE: break;
    case FMMT_TUCKER3D:
      e += op->zfused ? op->n2 * fmmt::zf_hj_stride(op->r1max, op->r3max) : op->n1 * op->r2max * op->r3max + n12 * op->r3max;
      break;
    case FMMT_TUCKER4D: e += rk(op, 0, 0) * rk(op, 0, 1) * rk(op, 0, 2) + op->n1 * op->r2max * op->r3max + n12 * op->r3max; break;
    case FMMT_HTUCKER4D: e += rk(op, 0, 2) * rk(op, 0, 5) + n12 * op->r3max; break;
    case FMMT_TT3D: e += n12 * op->rGmax; break;
    case FMMT_TT4D: {
      e += rk(op, 0, 1) * op->n3;
      // pre-split V_q (pack_v): 4 floats per complex per B' row pair, padded to 8-complex K chunks
      const int64_t nkc = (rk(op, 0, 1) + 7) / 8;
      e += nkc * 8 * op->n3 * 2;
      break;
    }
  }
  return e * 8;
}

static fmmt_status cmalloc(fmmt_op* op, float2** p, int64_t elems) {
  return dev_alloc(op, p, std::max<int64_t>(elems, 1) * 8, MEM_WORKSPACE, "workspace");
}

// Fold max(|Re|, |Im|) of a flat complex64 array into a scale slot (asynchronous).
static fmmt_status absmax_ctx(fmmt_ctx* ctx, const float2* x, int64_t n, float* slot) {
  if (n <= 0) return FMMT_OK;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)ctx->num_sms * 8));
  fmmt::k_absmax<<<grid, 256, 0, ctx->stream>>>(x, n, slot);
  FMMT_CUDA(ctx, cudaGetLastError());
  return FMMT_OK;
}
static fmmt_status absmax(fmmt_op* op, const float2* x, int64_t n, float* slot) { return absmax_ctx(op->ctx, x, n, slot); }

// Reset the per-batch (dynamic) scale slots: at the start of every matvec / restore (a memset node when captured).
static fmmt_status reset_dyn_slots(fmmt_op* op) {
  if (!op->d_slots || op->nslots_dyn <= 0) return FMMT_OK;
  FMMT_CUDA(op->ctx, cudaMemsetAsync(op->d_slots + SLOT_DYN, 0, op->nslots_dyn * 4, op->ctx->stream));
  return FMMT_OK;
}

static void add_gemm(fmmt_op* op, Batch& b, const std::vector<GemmDesc>& ds, const char* name) {
  if (ds.empty()) return;
  GemmLaunch L;
  L.first = (int)op->descs.size();
  L.ndesc = (int)ds.size();
  L.name = name;
  int64_t mmin = 1 << 30, nmin = 1 << 30;
  for (auto& d : ds) {
    mmin = std::min<int64_t>(mmin, d.m);
    nmin = std::min<int64_t>(nmin, d.n);
  }
  L.big = (mmin >= 64 && nmin >= 64);
  const int bm = L.big ? 64 : 32, bn = L.big ? 64 : 32;
  L.tc_bn = nmin >= 32 ? 32 : 16;   // BN = 64 needs 512 TMEM columns (1 CTA / SM)
  for (auto& d : ds) {
    int tiles = ((d.m + bm - 1) / bm) * ((d.n + bn - 1) / bn);
    L.maxtiles = std::max(L.maxtiles, tiles);
    L.tc_maxtiles = std::max(L.tc_maxtiles, ((d.m + fmmt::TC_BM - 1) / fmmt::TC_BM) * ((d.n + L.tc_bn - 1) / L.tc_bn));
    L.maxsub = std::max(L.maxsub, d.batch);
    op->descs.push_back(d);
    op->descs.back().n_fast = d.m > d.n ? 1 : 0;   // stream the larger operand once (A: m x k, B: k x n)
  }
  b.gemms.push_back(L);
}

// Column-major helper: C (ldc) = A (m x k, lda) . op(B), op(B) = B (k x n, ldb) or
// B^T when B is stored n x k (transB).  Sub-batch strides sA, sB, sC.
static GemmDesc gd(const float2* A, const float2* B, float2* C, int64_t m, int64_t n, int64_t k, int transB,
                   int64_t lda, int64_t ldb, int64_t ldc, int batch = 1, int64_t sA = 0, int64_t sB = 0, int64_t sC = 0) {
  GemmDesc d;
  memset(&d, 0, sizeof(d));
  d.A = A; d.B = B; d.C = C;
  d.m = (int)m; d.n = (int)n; d.k = (int)k;
  d.batch = batch;
  d.a_s0 = 1; d.a_s1 = 0; d.a_div = 1 << 30; d.a_sk = lda;
  if (transB) { d.b_sk = ldb; d.b_sn = 1; } else { d.b_sk = 1; d.b_sn = ldb; }
  d.c_s0 = 1; d.c_s1 = 0; d.c_div = 1 << 30; d.c_sn = ldc;
  d.sA = sA; d.sB = sB; d.sC = sC;
  return d;
}

// General helper: A(i,l) = A[(i%a_div)*a_s0 + (i/a_div)*a_s1 + l*a_sk], B(l,j) = B[l*b_sk + j*b_sn],
// C(i,j) = C[(i%c_div)*c_s0 + (i/c_div)*c_s1 + j*c_sn].
static GemmDesc gdx(const float2* A, const float2* B, float2* C, int64_t m, int64_t n, int64_t k, int64_t a_s0,
                    int64_t a_s1, int64_t a_div, int64_t a_sk, int64_t b_sk, int64_t b_sn, int64_t c_s0, int64_t c_s1,
                    int64_t c_div, int64_t c_sn, int batch = 1, int64_t sA = 0, int64_t sB = 0, int64_t sC = 0) {
  GemmDesc d;
  memset(&d, 0, sizeof(d));
  d.A = A; d.B = B; d.C = C;
  d.m = (int)m; d.n = (int)n; d.k = (int)k;
  d.batch = batch;
  d.a_s0 = a_s0; d.a_s1 = a_s1; d.a_div = (int)std::min<int64_t>(a_div, 1 << 30); d.a_sk = a_sk;
  d.b_sk = b_sk; d.b_sn = b_sn;
  d.c_s0 = c_s0; d.c_s1 = c_s1; d.c_div = (int)std::min<int64_t>(c_div, 1 << 30); d.c_sn = c_sn;
  d.sA = sA; d.sB = sB; d.sC = sC;
  return d;
}
constexpr int64_t NODIV = 1 << 30;

static fmmt_status launch_gemm_group(fmmt_ctx* ctx, const GemmLaunch& L, const GemmDesc* d_descs, int impl);

// One GEMM outside any plan (setup-time derived factors, the test hook).  Asynchronous.
static fmmt_status run_one_gemm(fmmt_ctx* ctx, const GemmDesc& d, int impl, const char* name) {
  fmmt_op tmp;
  tmp.ctx = ctx;
  Batch b;
  add_gemm(&tmp, b, {d}, name);
  GemmDesc* dd = nullptr;
  FMMT_CUDA(ctx, cudaMallocAsync((void**)&dd, sizeof(GemmDesc), ctx->stream));
  FMMT_CUDA(ctx, cudaMemcpyAsync(dd, &d, sizeof(GemmDesc), cudaMemcpyHostToDevice, ctx->stream));
  fmmt_status st;
  {
    ProfScope ps(ctx, name);
    st = launch_gemm_group(ctx, b.gemms[0], dd, impl);
  }
  cudaFreeAsync(dd, ctx->stream);
  return st;
}

// Pre-split a static A operand for the tensor-core kernels (k_tc_pack_a).  Synchronous.
static fmmt_status pack_a(fmmt_op* op, const GemmDesc& d, float** out) {
  fmmt_ctx* ctx = op->ctx;
  const int64_t tiles_m = (d.m + fmmt::TC_BM - 1) / fmmt::TC_BM, nkc = (d.k + fmmt::TC_BK - 1) / fmmt::TC_BK;
  const int64_t floats = tiles_m * nkc * fmmt::TC_PACK_FLOATS;
  if (fmmt_status st = dev_alloc(op, out, floats * 4, MEM_DERIVED, "packed operand")) return st;
  const int64_t work = tiles_m * fmmt::TC_BM * nkc * (fmmt::TC_BK / 2);
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, (int64_t)ctx->num_sms * 16));
  {
    ProfScope ps(ctx, "pack_a");
    fmmt::k_tc_pack_a<<<blocks, 256, 0, ctx->stream>>>(d, *out);
  }
  FMMT_CUDA(ctx, cudaGetLastError());
  FMMT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return FMMT_OK;
}

// Tucker chain shared by the Tucker / H-Tucker formats: per batch-local q with
// 3D core at core_q, H_q = U1 . core_q(1), G_q[:,:,c] = H_q[:,:,c] . U2^T.
static fmmt_status tucker_chain(fmmt_op* op, Batch& b, int bi) {
  // Fig. 3(a) in the "tall" orientation so every GEMM has >= n1*r rows:
  //   mode 1:  H_q[(b + r2 c) + r2 r3 i] = sum_a core_q[a + r1 (b + r2 c)] U1[i + n1 a]
  //   mode 2:  G_q[i + n1 j + n12 c]     = sum_b H_q[b + r2 c + r2 r3 i] U2[j + n2 b]
  // G_q is [c][ij], the layout the fused z-stage reads (A(ij, c), K = r3).
  const int64_t n1 = op->n1, n2 = op->n2, n12 = n1 * n2;
  std::vector<GemmDesc> sa, sb;
  if (op->zfused) {
    // fused chain (kernels_tcfuse.cuh): mode 2 first, H'_q[c + r3 a + hj j] = sum_b core_q[a + r1 b + r1 r2 c] U2[j + n2 b]
    // (hj = r1 r3 rounded up to even: 16-byte aligned blocks for the kernel's bulk copies)
    // (rows (c, a): c = row % r3, a = row / r3); modes 1 and 3 run inside k_tucker_zf
    for (int q = 0; q < b.nq; ++q) {
      const int64_t p = b.q0 + q;
      const int64_t r1 = rk(op, p, 0), r2 = rk(op, p, 1), r3 = rk(op, p, 2);
      GemmDesc d = gdx(op->arr[0] + op->off[0][p], op->arr[2] + op->off[2][p], op->H + q * op->h_stride, r1 * r3, n2, r2,
                       r1 * r2, 1, r3, r1, n2, 1, 1, 0, NODIV, fmmt::zf_hj_stride(r1, r3));
      d.amax = sslot(op, 0);
      d.bmax = sslot(op, 2);
      d.cmax = dslot(op, bi, 0);
      sa.push_back(d);
    }
    add_gemm(op, b, sa, "restore_mode2x");
    return FMMT_OK;
  }
  if (op->format == FMMT_TUCKER3D) {
    for (int q = 0; q < b.nq; ++q) {
      const int64_t p = b.q0 + q;
      const int64_t r1 = rk(op, p, 0), r2 = rk(op, p, 1), r3 = rk(op, p, 2);
      const float2* core = op->arr[0] + op->off[0][p];
      const float2* U1 = op->arr[1] + op->off[1][p];
      const float2* U2 = op->arr[2] + op->off[2][p];
      float2* Hq = op->H + q * n1 * op->r2max * op->r3max;
      float2* Gq = op->Gw + q * n12 * op->rGmax;
      GemmDesc d1 = gdx(core, U1, Hq, r2 * r3, n1, r1, r1, 0, NODIV, 1, n1, 1, 1, 0, NODIV, r2 * r3);
      d1.amax = sslot(op, 0);
      d1.bmax = sslot(op, 1);
      d1.cmax = dslot(op, bi, 0);
      sa.push_back(d1);
      GemmDesc d2 = gdx(Hq, U2, Gq, n1 * r3, n2, r2, r2 * r3, r2, n1, 1, n2, 1, 1, n12, n1, n1);
      d2.amax = dslot(op, bi, 0);
      d2.bmax = sslot(op, 2);
      d2.cmax = dslot(op, bi, 1);
      sb.push_back(d2);
    }
  } else {
    const int64_t r1 = rk(op, 0, 0), r2 = rk(op, 0, 1), r3 = rk(op, 0, 2);
    const float2* U1 = op->arr[op->format == FMMT_TUCKER4D ? 1 : 0];
    const float2* U2 = op->arr[op->format == FMMT_TUCKER4D ? 2 : 1];
    // (Tucker-4D: the slice GEMM wrote C_q with max into stage 0)
    GemmDesc d1 = gdx(op->Cw, U1, op->H, r2 * r3, n1, r1, r1, 0, NODIV, 1, n1, 1, 1, 0, NODIV, r2 * r3, b.nq,
                      r1 * r2 * r3, 0, n1 * r2 * r3);
    d1.amax = dslot(op, bi, 0);
    d1.bmax = sslot(op, 1);
    d1.cmax = dslot(op, bi, 1);
    sa.push_back(d1);
    GemmDesc d2 = gdx(op->H, U2, op->Gw, n1 * r3, n2, r2, r2 * r3, r2, n1, 1, n2, 1, 1, n12, n1, n1, b.nq,
                      n1 * r2 * r3, 0, n12 * r3);
    d2.amax = dslot(op, bi, 1);
    d2.bmax = sslot(op, 2);
    d2.cmax = dslot(op, bi, 2);
    sb.push_back(d2);
  }
  add_gemm(op, b, sa, "restore_mode1");
  add_gemm(op, b, sb, "restore_mode2");
  return FMMT_OK;
}

static void fill_zargs(fmmt_op* op, ZArgs& a, int bi);

// ---------------------------------------------------------------- packed operands (kernels_tcpk.cuh)
// Every tensor-core contraction streams both operands pre-split (fp16 / TF32 hi + lo, UMMA layout):
//   static operands (factors, T1, E; the rows of the direction factor a batch uses) are packed once per
//   op at plan time, dynamic ones (intermediates a batch produces) by a pack launch right before their
//   consumer, into per-launch-position workspaces shared by all batches.
static bool in_mem(const fmmt_op* op, const void* p, int kind_a, int kind_b) {
  const char* c = (const char*)p;
  for (auto& kv : op->mem)
    if ((kv.second.second == kind_a || kv.second.second == kind_b) && c >= (const char*)kv.first &&
        c < (const char*)kv.first + kv.second.first)
      return true;
  return false;
}
static bool is_static_operand(const fmmt_op* op, const void* p) { return in_mem(op, p, MEM_FACTOR, MEM_DERIVED); }

static int64_t pk_a_floats_sub(const GemmDesc& d) {
  return ((d.m + fmmt::TC_BM - 1) / fmmt::TC_BM) * ((d.k + fmmt::TC_BK - 1) / fmmt::TC_BK) * fmmt::TC_PACK_FLOATS;
}
static int64_t pk_b_floats_sub(const GemmDesc& d, int bn) {
  return ((d.n + bn - 1) / bn) * ((d.k + fmmt::TC_BK - 1) / fmmt::TC_BK) * (64 * bn * fmmt::TC_ESZ / 4);
}

static fmmt_status launch_pack_a_multi(fmmt_ctx* ctx, const GemmDesc* d_descs, int ndesc, int64_t max_items) {
  if (ndesc <= 0) return FMMT_OK;
  const unsigned bx = (unsigned)std::max<int64_t>(1, std::min<int64_t>((max_items + 255) / 256, (int64_t)ctx->num_sms * 8));
  ProfScope ps(ctx, "pack_a");
  fmmt::k_pk_pack_a_multi<<<dim3(bx, (unsigned)ndesc), 256, 0, ctx->stream>>>(d_descs);
  FMMT_CUDA(ctx, cudaGetLastError());
  return FMMT_OK;
}

static fmmt_status launch_pack_b_bn(fmmt_ctx* ctx, const GemmDesc& d, int bn, float* out) {
  const int nb = d.sB == 0 ? 1 : d.batch;
  const int64_t items = (int64_t)nb * pk_b_floats_sub(d, bn) / (64 * bn * fmmt::TC_ESZ / 4) * bn * (fmmt::TC_BK / 2);
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((items + 255) / 256, (int64_t)ctx->num_sms * 16));
  ProfScope ps(ctx, "pack_b");
  if (bn == 32)
    fmmt::k_tc_pack_b<32><<<grid, 256, 0, ctx->stream>>>(d.B, d.sB, d.b_sk, d.b_sn, d.k, d.n, nb, out, d.bmax);
  else
    fmmt::k_tc_pack_b<16><<<grid, 256, 0, ctx->stream>>>(d.B, d.sB, d.b_sk, d.b_sn, d.k, d.n, nb, out, d.bmax);
  FMMT_CUDA(ctx, cudaGetLastError());
  return FMMT_OK;
}

// Static A of d: packed once (cached by operand addressing), d.Ap / a_nkc / a_pk_sub set.
static fmmt_status pack_static_a(fmmt_op* op, GemmDesc& d) {
  fmmt_ctx* ctx = op->ctx;
  const int nb = d.sA == 0 ? 1 : d.batch;
  std::vector<int64_t> key = {0, (int64_t)d.A, d.m, d.k, d.a_s0, d.a_s1, d.a_div, d.a_sk, d.sA, nb};
  float* buf = nullptr;
  for (auto& e : op->pk_cache)
    if (e.first == key) buf = e.second;
  const int64_t sub = pk_a_floats_sub(d);
  if (!buf) {
    if (fmmt_status st = dev_alloc(op, &buf, nb * sub * 4, MEM_DERIVED, "packed A")) return st;
    GemmDesc t = d;
    t.Ap = buf;
    t.a_pk_sub = sub;
    t.batch = nb;
    GemmDesc* dd = nullptr;
    FMMT_CUDA(ctx, cudaMallocAsync((void**)&dd, sizeof(GemmDesc), ctx->stream));
    FMMT_CUDA(ctx, cudaMemcpyAsync(dd, &t, sizeof(GemmDesc), cudaMemcpyHostToDevice, ctx->stream));
    fmmt_status st = launch_pack_a_multi(ctx, dd, 1, nb * sub / fmmt::TC_PACK_FLOATS * fmmt::TC_BM * (fmmt::TC_BK / 2));
    cudaFreeAsync(dd, ctx->stream);
    if (st) return st;
    op->pk_cache.push_back({key, buf});
  }
  d.Ap = buf;
  d.a_nkc = (int)((d.k + fmmt::TC_BK - 1) / fmmt::TC_BK);
  d.a_pk_sub = d.sA == 0 ? 0 : sub;
  return FMMT_OK;
}

// Static B of d for a launch with bn columns per tile: packed once (cached), d.Bp / b_pk_sub set.
static fmmt_status pack_static_b(fmmt_op* op, GemmDesc& d, int bn) {
  const int nb = d.sB == 0 ? 1 : d.batch;
  std::vector<int64_t> key = {1, (int64_t)d.B, d.n, d.k, d.b_sk, d.b_sn, d.sB, nb, bn};
  float* buf = nullptr;
  for (auto& e : op->pk_cache)
    if (e.first == key) buf = e.second;
  const int64_t sub = pk_b_floats_sub(d, bn);
  if (!buf) {
    if (fmmt_status st = dev_alloc(op, &buf, nb * sub * 4, MEM_DERIVED, "packed B")) return st;
    if (fmmt_status st = launch_pack_b_bn(op->ctx, d, bn, buf)) return st;
    op->pk_cache.push_back({key, buf});
  }
  d.Bp = buf;
  d.b_pk_sub = d.sB == 0 ? 0 : sub;
  return FMMT_OK;
}

// After the batches are planned: pack every static operand, give every dynamic one a workspace region
// (its launch packs it), and prepare the z-stage's packed G (dynamic) and V (static) operands.
static fmmt_status finalize_packs(fmmt_op* op) {
  fmmt_ctx* ctx = op->ctx;
  op->packed = false;
  if (ctx->gemm_impl != 1 || op->format == FMMT_DENSE) return FMMT_OK;
  fmmt_status st;
  // ---- GEMM launches
  size_t npos = 0;
  for (auto& b : op->batches) npos = std::max(npos, b.gemms.size());
  std::vector<int64_t> need(npos, 0), needb(npos, 0);
  for (auto& b : op->batches)
    for (size_t li = 0; li < b.gemms.size(); ++li) {
      const GemmLaunch& L = b.gemms[li];
      int64_t a = 0, bb = 0;
      for (int i = 0; i < L.ndesc; ++i) {
        const GemmDesc& d = op->descs[L.first + i];
        if (!d.Ap && !is_static_operand(op, d.A)) a += (d.sA == 0 ? 1 : d.batch) * pk_a_floats_sub(d);
        if (!d.Bp && !is_static_operand(op, d.B)) bb += (d.sB == 0 ? 1 : d.batch) * pk_b_floats_sub(d, L.tc_bn);
      }
      need[li] = std::max(need[li], a);
      needb[li] = std::max(needb[li], bb);
    }
  for (auto& p : op->apk_dyn) dev_free(op, p);
  op->apk_dyn.assign(2 * npos, nullptr);
  for (size_t li = 0; li < npos; ++li) {
    if (need[li] && (st = dev_alloc(op, &op->apk_dyn[li], need[li] * 4, MEM_WORKSPACE, "packed A workspace"))) return st;
    if (need[li]) FMMT_CUDA(ctx, cudaMemsetAsync(op->apk_dyn[li], 0, need[li] * 4, ctx->stream));   // padding stays 0
    if (needb[li] && (st = dev_alloc(op, &op->apk_dyn[npos + li], needb[li] * 4, MEM_WORKSPACE, "packed B workspace")))
      return st;
  }
  for (auto& b : op->batches)
    for (size_t li = 0; li < b.gemms.size(); ++li) {
      GemmLaunch& L = b.gemms[li];
      int64_t ao = 0, bo = 0;
      for (int i = 0; i < L.ndesc; ++i) {
        GemmDesc& d = op->descs[L.first + i];
        if (!d.Ap) {
          if (is_static_operand(op, d.A)) {
            if ((st = pack_static_a(op, d))) return st;
          } else {
            const int64_t sub = pk_a_floats_sub(d);
            d.Ap = op->apk_dyn[li] + ao;
            d.a_nkc = (int)((d.k + fmmt::TC_BK - 1) / fmmt::TC_BK);
            d.a_pk_sub = d.sA == 0 ? 0 : sub;
            ao += (d.sA == 0 ? 1 : d.batch) * sub;
            L.pack_a_dyn = true;
          }
        } else if (d.a_pk_sub == 0 && d.sA != 0 && d.batch > 1) {
          d.a_pk_sub = pk_a_floats_sub(d);
        }
        if (!d.Bp) {
          if (is_static_operand(op, d.B)) {
            if ((st = pack_static_b(op, d, L.tc_bn))) return st;
          } else {
            const int64_t sub = pk_b_floats_sub(d, L.tc_bn);
            d.Bp = op->apk_dyn[npos + li] + bo;
            d.b_pk_sub = d.sB == 0 ? 0 : sub;
            bo += (d.sB == 0 ? 1 : d.batch) * sub;
            if (L.ndesc != 1) return set_err(ctx, FMMT_E_STATE, "dynamic B in a multi-descriptor launch");
            L.pack_dst = const_cast<float*>(d.Bp);
          }
        } else if (d.b_pk_sub == 0 && d.sB != 0 && d.batch > 1) {
          d.b_pk_sub = pk_b_floats_sub(d, L.tc_bn);
        }
      }
    }
  // ---- z-stage operands
  const int64_t n12 = op->n1 * op->n2, n3 = op->n3;
  const int64_t tiles_m = (n12 + fmmt::TC_BM - 1) / fmmt::TC_BM;
  if (op->zfused) {
    // U1 of every direction as k_tucker_zf's GEMM1 A operand: A(i, a) = U1_p[i + n1 a], K = r1
    std::vector<GemmDesc> ds;
    std::vector<int64_t> off(op->ndir);
    int64_t tot = 0;
    for (int64_t p = 0; p < op->ndir; ++p) {
      const int64_t r1 = rk(op, p, 0);
      GemmDesc d = gdx(op->arr[1] + op->off[1][p], nullptr, nullptr, op->n1, 1, r1, 1, 0, NODIV, op->n1, 0, 0, 0, 0, NODIV, 0);
      d.amax = sslot(op, 1);
      d.a_nkc = (int)((r1 + fmmt::TC_BK - 1) / fmmt::TC_BK);
      off[p] = tot;
      tot += pk_a_floats_sub(d);
      ds.push_back(d);
    }
    dev_free(op, op->u1pk);
    if ((st = dev_alloc(op, &op->u1pk, tot * 4, MEM_DERIVED, "packed U1"))) return st;
    int64_t items = 1;
    for (int64_t p = 0; p < op->ndir; ++p) {
      ds[p].Ap = op->u1pk + off[p];
      items = std::max<int64_t>(items, pk_a_floats_sub(ds[p]) / fmmt::TC_PACK_FLOATS * fmmt::TC_BM * 2);
    }
    GemmDesc* dd = nullptr;
    FMMT_CUDA(ctx, cudaMallocAsync((void**)&dd, ds.size() * sizeof(GemmDesc), ctx->stream));
    FMMT_CUDA(ctx, cudaMemcpyAsync(dd, ds.data(), ds.size() * sizeof(GemmDesc), cudaMemcpyHostToDevice, ctx->stream));
    for (size_t i0 = 0; i0 < ds.size() && !st; i0 += 65535)
      st = launch_pack_a_multi(ctx, dd + i0, (int)std::min<size_t>(65535, ds.size() - i0), items);
    cudaFreeAsync(dd, ctx->stream);
    if (st) return st;
    dev_free(op, op->d_u1p_off);
    if ((st = dev_alloc(op, &op->d_u1p_off, op->ndir * 8, MEM_DERIVED, "packed U1 offsets"))) return st;
    FMMT_CUDA(ctx, cudaMemcpyAsync(op->d_u1p_off, off.data(), op->ndir * 8, cudaMemcpyHostToDevice, ctx->stream));
  }
  if (op->format != FMMT_TT4D) {
    // dynamic G_q: A(ij, c) = G[q g_stride + ij + n12 c], K = the direction's z rank (not for the fused chain)
    ZArgs za;
    fill_zargs(op, za, 0);
    int64_t rzmax = 1;
    for (int64_t p = 0; p < op->ndir; ++p) rzmax = std::max<int64_t>(rzmax, za.rank_p ? (op->format == FMMT_TUCKER3D ? rk(op, p, 2) : rk(op, p, 1)) : za.rank);
    op->gp_stride = tiles_m * ((rzmax + fmmt::TC_BK - 1) / fmmt::TC_BK) * fmmt::TC_PACK_FLOATS;
    dev_free(op, op->gpk);
    if (!op->zfused) {
      if ((st = dev_alloc(op, &op->gpk, op->PB * op->gp_stride * 4, MEM_WORKSPACE, "packed G"))) return st;
      FMMT_CUDA(ctx, cudaMemsetAsync(op->gpk, 0, op->PB * op->gp_stride * 4, ctx->stream));
    }
    for (int bi = 0; bi < (int)op->batches.size() && !op->zfused; ++bi) {
      Batch& b = op->batches[bi];
      ZArgs a;
      fill_zargs(op, a, bi);
      b.zp_first = (int)op->descs.size();
      const bool per_dir = a.rank_p != nullptr;
      for (int q = 0; q < (per_dir ? b.nq : 1); ++q) {
        const int64_t p = b.q0 + q;
        const int64_t k = per_dir ? (op->format == FMMT_TUCKER3D ? rk(op, p, 2) : rk(op, p, 1)) : a.rank;
        GemmDesc d = gdx(a.G + q * a.g_stride, nullptr, nullptr, n12, 1, k, 1, 0, NODIV, n12, 0, 0, 0, 0, NODIV, 0,
                         per_dir ? 1 : b.nq, a.g_stride, 0, 0);
        d.Ap = op->gpk + q * op->gp_stride;
        d.a_nkc = (int)((k + fmmt::TC_BK - 1) / fmmt::TC_BK);
        d.a_pk_sub = op->gp_stride;
        d.amax = a.amax;
        op->descs.push_back(d);
      }
      b.zp_n = (int)op->descs.size() - b.zp_first;
    }
    // static V: B(c, kz) = V[c n3 + kz] per direction (3D formats) or shared (4D): one pack of
    // BN = max(16, n3) columns; n3 = 64 with the columns ordered [kz even | kz odd] (kzperm)
    const int bn = n3 <= 16 ? 16 : (int)n3;
    const int64_t ncp = op->format == FMMT_TUCKER3D || op->format == FMMT_TT3D ? op->ndir : 1;
    std::vector<int64_t> off(ncp);
    std::vector<fmmt::PkB> items;
    int64_t tot = 0;
    for (int64_t p = 0; p < ncp; ++p) {
      const int64_t k = za.rank_p ? (op->format == FMMT_TUCKER3D ? rk(op, p, 2) : rk(op, p, 1)) : za.rank;
      const int64_t per = ((k + fmmt::TC_BK - 1) / fmmt::TC_BK) * (64 * bn * fmmt::TC_ESZ / 4);
      off[p] = tot;
      fmmt::PkB it;
      it.B = za.V + (za.v_off ? op->off[op->format == FMMT_TUCKER3D ? 3 : 2][p] : 0);
      it.b_sk = n3;
      it.b_sn = 1;
      it.k = (int)k;
      it.n = (int)n3;
      it.out = nullptr;
      it.bmax = za.bmax;
      it.kzperm = n3 == 64;
      items.push_back(it);
      tot += per;
    }
    dev_free(op, op->vpk_static);
    if ((st = dev_alloc(op, &op->vpk_static, tot * 4, MEM_DERIVED, "packed V"))) return st;
    {
      int64_t o = 0;
      for (auto& it : items) {
        it.out = op->vpk_static + o;
        o += ((it.k + fmmt::TC_BK - 1) / fmmt::TC_BK) * (64 * bn * fmmt::TC_ESZ / 4);
      }
    }
    fmmt::PkB* d_items = nullptr;
    FMMT_CUDA(ctx, cudaMallocAsync((void**)&d_items, items.size() * sizeof(fmmt::PkB), ctx->stream));
    FMMT_CUDA(ctx, cudaMemcpyAsync(d_items, items.data(), items.size() * sizeof(fmmt::PkB), cudaMemcpyHostToDevice, ctx->stream));
    for (size_t i0 = 0; i0 < items.size(); i0 += 65535) {
      const unsigned ny = (unsigned)std::min<size_t>(65535, items.size() - i0);
      if (bn == 64) fmmt::k_pk_pack_b_multi<64><<<dim3(8, ny), 256, 0, ctx->stream>>>(d_items + i0, nullptr);
      else if (bn == 32) fmmt::k_pk_pack_b_multi<32><<<dim3(8, ny), 256, 0, ctx->stream>>>(d_items + i0, nullptr);
      else fmmt::k_pk_pack_b_multi<16><<<dim3(8, ny), 256, 0, ctx->stream>>>(d_items + i0, nullptr);
      FMMT_CUDA(ctx, cudaGetLastError());
    }
    cudaFreeAsync(d_items, ctx->stream);
    dev_free(op, op->d_vp_off);
    if (ncp > 1) {
      if ((st = dev_alloc(op, &op->d_vp_off, ncp * 8, MEM_DERIVED, "packed V offsets"))) return st;
      FMMT_CUDA(ctx, cudaMemcpyAsync(op->d_vp_off, off.data(), ncp * 8, cudaMemcpyHostToDevice, ctx->stream));
    }
    op->vp_stride = 0;
  } else {
    // TT-4D: the batch's V_q (dynamic) is packed per batch: items per (q [, parity h])
    const int64_t r2 = rk(op, 0, 1);
    const int bn = n3 <= 16 ? 16 : (int)n3;
    const int64_t per = ((r2 + fmmt::TC_BK - 1) / fmmt::TC_BK) * (64 * bn * fmmt::TC_ESZ / 4);
    op->vp_stride = per;
    dev_free(op, op->Vpk);
    if ((st = dev_alloc(op, &op->Vpk, op->PB * op->vp_stride * 4, MEM_WORKSPACE, "packed V_q"))) return st;
    op->vpk_floats = op->PB * op->vp_stride;
    std::vector<fmmt::PkB> items;
    for (int64_t q = 0; q < op->PB; ++q) {
      fmmt::PkB it;   // V_q(c, kz) = Vw[q r2 n3 + c + r2 kz]
      it.B = op->Vw + q * r2 * n3;
      it.b_sk = 1;
      it.b_sn = r2;
      it.k = (int)r2;
      it.n = (int)n3;
      it.out = op->Vpk + q * op->vp_stride;
      it.bmax = nullptr;
      it.kzperm = n3 == 64;
      items.push_back(it);
    }
    dev_free(op, op->d_vitems);
    if ((st = dev_alloc(op, &op->d_vitems, (int64_t)(items.size() * sizeof(fmmt::PkB)), MEM_WORKSPACE, "V_q pack items")))
      return st;
    FMMT_CUDA(ctx, cudaMemcpyAsync(op->d_vitems, items.data(), items.size() * sizeof(fmmt::PkB), cudaMemcpyHostToDevice,
                                   ctx->stream));
    op->nvitems = (int64_t)items.size();
  }
  FMMT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  op->packed = true;
  return FMMT_OK;
}

static fmmt_status build_plans(fmmt_op* op) {
  free_workspace(op);
  op->descs.clear();
  op->batches.clear();
  for (auto& e : op->pk_cache) dev_free(op, e.second);   // static packs follow the batching (direction rows)
  op->pk_cache.clear();
  const int64_t n1 = op->n1, n2 = op->n2, n3 = op->n3, n12 = n1 * n2, Nz = n3 / 2;
  if (op->PB <= 0) {
    // batch size: the per-batch intermediates (raw and packed) within ctx->batch_mb (launch count and tail
    // waves against L2 residency; FMMT_BATCH_MB) ...
    const int64_t target = (int64_t)op->ctx->batch_mb << 20, pdw = std::max<int64_t>(1, 2 * per_dir_ws(op));
    int64_t pb = std::max<int64_t>(1, std::min<int64_t>(op->ndir, target / pdw));
    // ... unless the 4D formats' shared slice operand (streamed from HBM once per batch, pre-split = 16 B
    // per complex) outweighs them: then batches of shared / per-direction-workspace directions, up to
    // 4 GB of intermediates (measured: config 4 Tucker-4D re-streamed its 1.3 GB core every 10 directions)
    int64_t shared = 0;
    switch (op->format) {
      case FMMT_TUCKER4D: shared = rk(op, 0, 0) * rk(op, 0, 1) * rk(op, 0, 2) * rk(op, 0, 3); break;
      case FMMT_HTUCKER4D: shared = n12 * rk(op, 0, 5) + rk(op, 0, 2) * rk(op, 0, 3) * rk(op, 0, 5); break;
      case FMMT_TT4D: shared = rk(op, 0, 1) * n3 * rk(op, 0, 2); break;
      default: break;
    }
    if (shared > 0) pb = std::max(pb, std::min<int64_t>(shared * 16 / pdw, (4ll << 30) / pdw));
    op->PB = std::max<int64_t>(1, std::min<int64_t>(op->ndir, pb));
    // even batches
    int64_t nb = (op->ndir + op->PB - 1) / op->PB;
    op->PB = (op->ndir + nb - 1) / nb;
  }
  const int64_t PB = op->PB;
  fmmt_status st;
  // (W, the half-padded spectra of one xy sub-batch, is sized by ensure_w at the first translate)
  switch (op->format) {
    case FMMT_DENSE: break;
    case FMMT_TUCKER3D:
      if (op->zfused) {
        op->h_stride = n2 * fmmt::zf_hj_stride(op->r1max, op->r3max);
        if ((st = cmalloc(op, &op->H, PB * op->h_stride))) return st;
        break;
      }
      if ((st = cmalloc(op, &op->H, PB * n1 * op->r2max * op->r3max))) return st;
      if ((st = cmalloc(op, &op->Gw, PB * n12 * op->rGmax))) return st;
      break;
    case FMMT_TUCKER4D:
      if ((st = cmalloc(op, &op->Cw, PB * rk(op, 0, 0) * rk(op, 0, 1) * rk(op, 0, 2)))) return st;
      if ((st = cmalloc(op, &op->H, PB * n1 * op->r2max * op->r3max))) return st;
      if ((st = cmalloc(op, &op->Gw, PB * n12 * op->rGmax))) return st;
      break;
    case FMMT_HTUCKER4D:
      if ((st = cmalloc(op, &op->Mw, PB * rk(op, 0, 2) * rk(op, 0, 5)))) return st;
      if ((st = cmalloc(op, &op->Gw, PB * n12 * op->rGmax))) return st;
      break;
    case FMMT_TT3D:
      if ((st = cmalloc(op, &op->Gw, PB * n12 * op->rGmax))) return st;
      break;
    case FMMT_TT4D:
      if ((st = cmalloc(op, &op->Vw, PB * rk(op, 0, 1) * n3))) return st;
      break;
  }
  const int64_t nbatches = (op->ndir + PB - 1) / PB;
  if (op->nslots_dyn < nbatches * SLOTS_PER_BATCH) {   // scale slots (see fmmt_op::d_slots)
    float* ns = nullptr;
    if ((st = dev_alloc(op, &ns, (SLOT_DYN + nbatches * SLOTS_PER_BATCH) * 4, MEM_WORKSPACE, "scale slots"))) return st;
    FMMT_CUDA(op->ctx, cudaMemsetAsync(ns, 0, (SLOT_DYN + nbatches * SLOTS_PER_BATCH) * 4, op->ctx->stream));
    if (op->d_slots)
      FMMT_CUDA(op->ctx, cudaMemcpyAsync(ns, op->d_slots, SLOT_DYN * 4, cudaMemcpyDeviceToDevice, op->ctx->stream));
    dev_free(op, op->d_slots);
    op->d_slots = ns;
    op->nslots_dyn = nbatches * SLOTS_PER_BATCH;
  }
  for (int64_t q0 = 0; q0 < op->ndir; q0 += PB) {
    Batch b;
    const int bi = (int)(q0 / PB);
    b.q0 = (int)q0;
    b.nq = (int)std::min<int64_t>(PB, op->ndir - q0);
    switch (op->format) {
      case FMMT_DENSE: break;
      case FMMT_TUCKER3D:
        if ((st = tucker_chain(op, b, bi))) return st;
        break;
      case FMMT_TUCKER4D: {
        const int64_t r1 = rk(op, 0, 0), r2 = rk(op, 0, 1), r3 = rk(op, 0, 2), r4 = rk(op, 0, 3);
        // a3 (Fig. 3(b)): C_q = C(r1 r2 r3 x r4) . U4[p,:]^T
        GemmDesc ds = gd(op->arr[0], op->arr[4] + b.q0, op->Cw, r1 * r2 * r3, b.nq, r4, 1, r1 * r2 * r3, op->ndir, r1 * r2 * r3);
        ds.amax = sslot(op, 0);
        ds.bmax = sslot(op, 4);
        ds.cmax = dslot(op, bi, 0);
        add_gemm(op, b, {ds}, "slice_tucker4d");
        if ((st = tucker_chain(op, b, bi))) return st;
        break;
      }
      case FMMT_HTUCKER4D: {
        // Fig. 3(c) with the direction-independent part precomputed once per op
        // (E = (C12 . C1234) x1 U1 x2 U2, n1 n2 x r34; create_op):
        //   M_q[c, j] = sum_d C34[c + r3 d + r3 r4 j] U4[p, d]      (a3)  stored Mw[c + r3 q + r3 nq j]
        //   G_q[ij, c] = sum_j E[ij + n12 j] M_q[c, j]              (a4)  stored Gw[ij + n12 (c + r3 q)]
        const int64_t r3 = rk(op, 0, 2), r4 = rk(op, 0, 3), r34 = rk(op, 0, 5);
        const int64_t nq = b.nq;
        const float2 *U4 = op->arr[3], *C34 = op->arr[5];
        GemmDesc dm = gdx(C34, U4 + b.q0, op->Mw, r3 * r34, nq, r4, 1, r3 * r4, r3, r3, op->ndir, 1, 1, r3 * nq, r3, r3);
        dm.amax = sslot(op, 5);
        dm.bmax = sslot(op, 3);
        dm.cmax = dslot(op, bi, 0);
        add_gemm(op, b, {dm}, "slice_htucker_M");
        GemmDesc dg = gdx(op->E, op->Mw, op->Gw, n12, r3 * nq, r34, 1, 0, NODIV, n12, r3 * nq, 1, 1, 0, NODIV, n12);
        dg.amax = sslot(op, SLOT_E);
        dg.bmax = dslot(op, bi, 0);
        dg.cmax = dslot(op, bi, 1);
        dg.Ap = op->E_pk;
        dg.a_nkc = (int)((r34 + fmmt::TC_BK - 1) / fmmt::TC_BK);
        add_gemm(op, b, {dg}, "slice_htucker_G");   // (M_q is packed right before it: finalize_packs)
        break;
      }
      case FMMT_TT3D: {
        std::vector<GemmDesc> ds;
        // Fig. 4(a): G_q[i + n1 j + n12 b] = sum_a C1_q[a + r1 (j + n2 b)] U1_q[i + n1 a]
        // (rows (j, b), n2 r2 of them; G_q is [b][ij] for the z-stage)
        for (int q = 0; q < b.nq; ++q) {
          const int64_t p = b.q0 + q;
          const int64_t r1 = rk(op, p, 0), r2 = rk(op, p, 1);
          GemmDesc dh = gdx(op->arr[1] + op->off[1][p], op->arr[0] + op->off[0][p], op->Gw + q * n12 * op->rGmax,
                            n2 * r2, n1, r1, r1, 0, NODIV, 1, n1, 1, n1, n12, n2, 1);
          dh.amax = sslot(op, 1);
          dh.bmax = sslot(op, 0);
          dh.cmax = dslot(op, bi, 0);
          ds.push_back(dh);
        }
        add_gemm(op, b, ds, "restore_tt_head");
        break;
      }
      case FMMT_TT4D: {
        const int64_t r2 = rk(op, 0, 1), r3 = rk(op, 0, 2);
        // a3 (Fig. 4(b) step 1, columns of T2 for the batch): V_q = C2(r2 n3 x r3) . U_last[p,:]^T
        GemmDesc dv = gd(op->arr[2], op->arr[3] + b.q0, op->Vw, r2 * n3, b.nq, r3, 1, r2 * n3, op->ndir, r2 * n3);
        dv.amax = sslot(op, 2);
        dv.bmax = sslot(op, 3);
        dv.cmax = dslot(op, bi, 0);
        add_gemm(op, b, {dv}, "slice_tt4d");
        break;
      }
    }
    op->batches.push_back(b);
  }
  if ((st = finalize_packs(op))) return st;
  FMMT_CUDA(op->ctx, cudaStreamSynchronize(op->ctx->stream));   // static pre-splits done
  if (!op->descs.empty()) {
    if ((st = dev_alloc(op, &op->d_descs, (int64_t)(op->descs.size() * sizeof(GemmDesc)), MEM_WORKSPACE, "descriptors")))
      return st;
    FMMT_CUDA(op->ctx, cudaMemcpy(op->d_descs, op->descs.data(), op->descs.size() * sizeof(GemmDesc), cudaMemcpyHostToDevice));
  }
  return FMMT_OK;
}

// ============================================================== launches
constexpr int TC_G = 1;   // thread groups per tensor-core CTA (2 = 256 threads: measured slower)

constexpr int PK_NS = 8;   // operand ring stages of the packed-operand pipeline (12 KB each at BN = 32, fp16)

template <int BN>
static fmmt_status launch_pk_bn(fmmt_ctx* ctx, const GemmLaunch& L, const GemmDesc* d) {
  using Cfg = fmmt::PkCfg<BN, PK_NS>;
  FMMT_CUDA(ctx, set_smem_once((const void*)fmmt::k_pk_cgemm<BN, PK_NS>, Cfg::SMEM));
  const int64_t total = (int64_t)L.tc_maxtiles * L.maxsub * L.ndesc;
  const int64_t cap = (int64_t)ctx->num_sms * ctx->tc_ctas_per_sm;   // resident CTAs (TMEM, smem), each walks tiles
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(total, cap));
  fmmt::k_pk_cgemm<BN, PK_NS><<<grid, fmmt::PK_THREADS, Cfg::SMEM, ctx->stream>>>(d, L.tc_maxtiles, L.maxsub, (int)total);
  return FMMT_OK;
}

// Launch one descriptor group.  impl: 0 = FP32 FFMA kernel, 1 = tcgen05 3xTF32
// (cp.async / bulk copies into the UMMA layout, 2 MMAs per K-step).
static fmmt_status launch_gemm_group(fmmt_ctx* ctx, const GemmLaunch& L, const GemmDesc* d_descs, int impl) {
  if (L.maxsub > 65535) return set_err(ctx, FMMT_E_UNSUPPORTED, "gemm sub-batch %d too large", L.maxsub);
  fmmt_status st = FMMT_OK;
  if (impl == 1) {
    if (L.tc_bn == 32) st = launch_pk_bn<32>(ctx, L, d_descs + L.first);
    else st = launch_pk_bn<16>(ctx, L, d_descs + L.first);
  } else {
    dim3 grid((unsigned)L.maxtiles, (unsigned)L.maxsub, (unsigned)L.ndesc);
    if (L.big)
      fmmt::k_cgemm<64, 64, 16, 4, 4><<<grid, 256, 0, ctx->stream>>>(d_descs + L.first);
    else
      fmmt::k_cgemm<32, 32, 16, 4, 4><<<grid, 64, 0, ctx->stream>>>(d_descs + L.first);
  }
  if (st) return st;
  FMMT_CUDA(ctx, cudaGetLastError());
  return FMMT_OK;
}

static fmmt_status launch_gemm(fmmt_op* op, const GemmLaunch& L) {
  fmmt_ctx* ctx = op->ctx;
  if (ctx->gemm_impl == 1 && !op->packed)
    return set_err(ctx, FMMT_E_STATE, "op planned for the FFMA kernels: call fmmt_set_gemm_impl before creating it");
  ProfScope ps(ctx, L.name);
  return launch_gemm_group(ctx, L, op->d_descs, ctx->gemm_impl);
}

// Block shape of the xy FFT kernels: about one line per thread per pass, with
// small CTAs (>= 64 threads, 1-2 planes) so that many CTAs are resident per
// SM and the load / FFT / store phases of different CTAs overlap.
static void xy_shape(const XYKernels& k, int* threads, int* ppc) {
  int t = std::max(64, std::min(fmmt::XY_THREADS, ((k.lines + 31) / 32) * 32));
  int p = std::max(1, std::min(2, t / std::max(1, k.lines)));
  const int64_t cap = (220 << 10) / 8 - FMMT_TW_NMAX;
  while (p > 1 && (int64_t)p * k.plane_smem > cap) --p;
  *threads = t;
  *ppc = p;
}

static fmmt_status launch_xy(fmmt_op* op, bool fwd, const float2* in, float2* out, int nplanes, float scale) {
  fmmt_ctx* ctx = op->ctx;
  XYKernels k = get_xy((int)op->n1, (int)op->n2);
  if (!k.fwd) return set_err(ctx, FMMT_E_UNSUPPORTED, "no xy kernel for n1=%lld n2=%lld", (long long)op->n1, (long long)op->n2);
  int threads, ppc;
  xy_shape(k, &threads, &ppc);
  size_t smem = (size_t)(FMMT_TW_NMAX + (int64_t)ppc * k.plane_smem) * sizeof(float2);
  if (k.big_pp) {
    threads = fmmt::XYB_THREADS;
    ppc = k.big_pp;
    smem = (size_t)(fwd ? k.big_smem_fwd : k.big_smem);
  }
  const unsigned grid = (unsigned)((nplanes + ppc - 1) / ppc);
  ProfScope ps(ctx, fwd ? "fft_fwd_xy" : "fft_inv_xy");
  if (fwd) {
    FMMT_CUDA(ctx, set_smem_once((const void*)k.fwd, (int)smem, k.big_pp == 1));
    k.fwd<<<grid, threads, smem, ctx->stream>>>(in, out, nplanes, ppc);
  } else {
    FMMT_CUDA(ctx, set_smem_once((const void*)k.inv, (int)smem, k.big_pp == 1));
    k.inv<<<grid, threads, smem, ctx->stream>>>(in, out, nplanes, ppc, scale);
  }
  FMMT_CUDA(ctx, cudaGetLastError());
  return FMMT_OK;
}

static void fill_zargs(fmmt_op* op, ZArgs& a, int bi) {
  const int64_t n12 = op->n1 * op->n2;
  memset(&a, 0, sizeof(a));
  a.n12 = n12;
  switch (op->format) {
    case FMMT_DENSE: a.T = op->arr[0]; break;
    case FMMT_TUCKER3D:
      a.G = op->Gw; a.g_stride = n12 * op->rGmax;
      a.V = op->arr[3]; a.v_off = op->d_voff; a.v_sc = op->n3; a.v_sk = 1; a.rank_p = op->d_rank;
      a.amax = dslot(op, bi, 1); a.bmax = sslot(op, 3);
      break;
    case FMMT_TUCKER4D:
      a.G = op->Gw; a.g_stride = n12 * rk(op, 0, 2);
      a.V = op->arr[3]; a.v_stride = 0; a.v_sc = op->n3; a.v_sk = 1; a.rank = (int)rk(op, 0, 2);
      a.amax = dslot(op, bi, 2); a.bmax = sslot(op, 3);
      break;
    case FMMT_HTUCKER4D:
      a.G = op->Gw; a.g_stride = n12 * rk(op, 0, 2);
      a.V = op->arr[2]; a.v_stride = 0; a.v_sc = op->n3; a.v_sk = 1; a.rank = (int)rk(op, 0, 2);
      a.amax = dslot(op, bi, 1); a.bmax = sslot(op, 2);
      break;
    case FMMT_TT3D:
      a.amax = dslot(op, bi, 0); a.bmax = sslot(op, 2);
      a.G = op->Gw; a.g_stride = n12 * op->rGmax;
      a.V = op->arr[2]; a.v_off = op->d_voff; a.v_sc = op->n3; a.v_sk = 1; a.rank_p = op->d_rank;
      break;
    case FMMT_TT4D:
      a.G = op->tbar1; a.g_stride = 0; a.Gp = op->tbar1_pk;
      a.amax = sslot(op, SLOT_T1); a.bmax = dslot(op, bi, 0);
      // T1 pre-split = 16 B per complex: block the z-stage tiles by direction when it exceeds ~1/4 of L2
      a.z_blocked = n12 * rk(op, 0, 1) * 16 > (32ll << 20) ? 1 : 0;
      a.V = op->Vw; a.v_stride = rk(op, 0, 1) * op->n3; a.v_sc = 1; a.v_sk = rk(op, 0, 1); a.rank = (int)rk(op, 0, 1);
      break;
  }
}

template <int N3, int MODE>
static fmmt_status launch_pk_z(fmmt_ctx* ctx, const ZArgs& a, int nq) {
  const int64_t tiles_m = (a.n12 + fmmt::TC_BM - 1) / fmmt::TC_BM;
  if constexpr (N3 == 64) {
    // all 64 kz per tile, one CTA per SM (PkwCfg); shared A (TT-4D T1): 2-CTA clusters, each A chunk
    // streamed once per pair and multicast
    constexpr int SM = fmmt::PkwCfg<fmmt::PKW_NS>::SMEM;
    const bool sh = a.g_stride == 0 && a.gp_stride == 0;
    const bool cl = ctx->z_cluster && sh && nq > 1;
    const int CL = cl ? 2 : 1;
    const int64_t groups = tiles_m * (int64_t)((nq + CL - 1) / CL);
    const unsigned ncl = (unsigned)std::max<int64_t>(1, std::min<int64_t>(groups, (int64_t)ctx->num_sms / CL));
    // shared A (TT-4D T1, K = r2 up to 1201): flush groups of 2 TC_FC K-chunks (the MMA warp runs twice as far
    // ahead of the per-tile z-DFT epilogue; FMMT_ZFC=4 for TC_FC, 16 for 4 TC_FC)
    const int fcm = !sh ? 1 : ctx->z_fc >= 4 * fmmt::TC_FC ? 4 : ctx->z_fc >= 2 * fmmt::TC_FC ? 2 : 1;
    auto kfn = fcm == 4 ? (cl ? fmmt::k_pk_conv_z64<MODE, fmmt::PKW_NS, 2, 4 * fmmt::TC_FC>
                              : fmmt::k_pk_conv_z64<MODE, fmmt::PKW_NS, 1, 4 * fmmt::TC_FC>)
             : fcm == 2 ? (cl ? fmmt::k_pk_conv_z64<MODE, fmmt::PKW_NS, 2, 2 * fmmt::TC_FC>
                              : fmmt::k_pk_conv_z64<MODE, fmmt::PKW_NS, 1, 2 * fmmt::TC_FC>)
                        : (cl ? fmmt::k_pk_conv_z64<MODE, fmmt::PKW_NS, 2> : fmmt::k_pk_conv_z64<MODE, fmmt::PKW_NS, 1>);
    FMMT_CUDA(ctx, set_smem_once((const void*)kfn, SM));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CL * ncl);
    cfg.blockDim = dim3(fmmt::PKW_THREADS);
    cfg.dynamicSmemBytes = SM;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = cl ? 1 : 0;
    FMMT_CUDA(ctx, cudaLaunchKernelEx(&cfg, kfn, a, nq));
    return FMMT_OK;
  } else {
    constexpr int BN = N3 < 16 ? 16 : N3;
    using Cfg = fmmt::PkCfg<BN, PK_NS>;
    const int64_t total = tiles_m * (int64_t)nq;
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(total, (int64_t)ctx->num_sms * ctx->tc_ctas_z));
    FMMT_CUDA(ctx, set_smem_once((const void*)fmmt::k_pk_conv_z<N3, MODE, PK_NS>, Cfg::SMEM));
    fmmt::k_pk_conv_z<N3, MODE, PK_NS><<<grid, fmmt::PK_THREADS, Cfg::SMEM, ctx->stream>>>(a, nq);
  }
  FMMT_CUDA(ctx, cudaGetLastError());
  return FMMT_OK;
}

template <int MODE>
static fmmt_status launch_pk_z_n3(fmmt_ctx* ctx, int n3, const ZArgs& a, int nq) {
  switch (n3) {
    case 4: return launch_pk_z<4, MODE>(ctx, a, nq);
    case 8: return launch_pk_z<8, MODE>(ctx, a, nq);
    case 16: return launch_pk_z<16, MODE>(ctx, a, nq);
    case 32: return launch_pk_z<32, MODE>(ctx, a, nq);
    case 64: return launch_pk_z<64, MODE>(ctx, a, nq);
  }
  return set_err(ctx, FMMT_E_UNSUPPORTED, "no z kernel for n3=%d", n3);
}

// The fused z-stage of a batch (or of one direction qoff of it, nq = 1, restore hook): its dynamic
// operand was packed by run_batch_zpack.
static fmmt_status launch_z(fmmt_op* op, int mode, int p0, int qoff, int nq, float2* Tout, float2* Wb = nullptr,
                            int ncomp = 1) {
  fmmt_ctx* ctx = op->ctx;
  if (op->zfused && ctx->gemm_impl != 1)
    return set_err(ctx, FMMT_E_STATE, "op planned for the fused tensor-core chain: call fmmt_set_gemm_impl before creating it");
  if (op->zfused && mode != fmmt::Z_DENSE) {
    if (!op->packed) return set_err(ctx, FMMT_E_STATE, "fused Tucker-3D op not packed");
    fmmt::ZfArgs a;
    memset(&a, 0, sizeof(a));
    a.W = Wb;
    a.n12 = op->n1 * op->n2;
    a.ncomp = ncomp;
    a.p0 = p0;
    a.q0 = qoff;
    a.n1 = (int)op->n1;
    a.U1p = op->u1pk;
    a.u1p_off = op->d_u1p_off;
    a.H = op->H;
    a.h_stride = op->h_stride;
    a.Vp = op->vpk_static;
    a.vp_off = op->d_vp_off;
    a.rank = op->d_rank3;
    a.u1max = sslot(op, 1);
    a.hmax = dslot(op, (int)(p0 / std::max<int64_t>(1, op->PB)), 0);
    a.u3max = sslot(op, 3);
    a.Tout = Tout;
    const int64_t tiles = (a.n12 / fmmt::TC_BM) * nq;
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)ctx->num_sms));
    ProfScope ps(ctx, mode == fmmt::Z_RESTORE ? "restore_out" : "restore_conv_z_tucker3d_fused");
    if constexpr (fmmt::TC_F16) {
      if (mode == fmmt::Z_RESTORE) {
        FMMT_CUDA(ctx, set_smem_once((const void*)fmmt::k_tucker_zf<fmmt::Z_RESTORE>, fmmt::ZfCfg::SMEM));
        fmmt::k_tucker_zf<fmmt::Z_RESTORE><<<grid, fmmt::ZF_THREADS, fmmt::ZfCfg::SMEM, ctx->stream>>>(a, nq);
      } else {
        FMMT_CUDA(ctx, set_smem_once((const void*)fmmt::k_tucker_zf<fmmt::Z_LOWRANK>, fmmt::ZfCfg::SMEM));
        fmmt::k_tucker_zf<fmmt::Z_LOWRANK><<<grid, fmmt::ZF_THREADS, fmmt::ZfCfg::SMEM, ctx->stream>>>(a, nq);
      }
    }
    FMMT_CUDA(ctx, cudaGetLastError());
    return FMMT_OK;
  }
  if (ctx->gemm_impl == 1 && mode != fmmt::Z_DENSE) {
    if (!op->packed)
      return set_err(ctx, FMMT_E_STATE, "op planned for the FFMA kernels: call fmmt_set_gemm_impl before creating it");
    ZArgs a;
    fill_zargs(op, a, (int)(p0 / std::max<int64_t>(1, op->PB)));
    a.W = Wb;
    a.ncomp = ncomp;
    a.p0 = p0;
    a.Tout = Tout;
    if (op->format == FMMT_TT4D) {
      a.Gp = op->tbar1_pk;
      a.gp_stride = 0;
      a.Vp = op->Vpk + (int64_t)qoff * op->vp_stride;
      a.vp_stride = op->vp_stride;
      a.vp_off = nullptr;
    } else {
      a.Gp = op->gpk + (int64_t)qoff * op->gp_stride;
      a.gp_stride = op->gp_stride;
      a.Vp = op->vpk_static;
      a.vp_off = op->d_vp_off;
      a.vp_stride = 0;
    }
    if (!a.Gp || !a.Vp) return set_err(ctx, FMMT_E_STATE, "z-stage operands not packed");
    static const char* znames[] = {"restore_conv_z_dense", "restore_conv_z_tucker3d", "restore_conv_z_tucker4d",
                                   "restore_conv_z_htucker4d", "restore_conv_z_tt3d", "restore_conv_z_tt4d"};
    ProfScope ps(ctx, mode == fmmt::Z_RESTORE ? "restore_out" : znames[op->format]);
    if (mode == fmmt::Z_RESTORE) return launch_pk_z_n3<fmmt::Z_RESTORE>(ctx, (int)op->n3, a, nq);
    return launch_pk_z_n3<fmmt::Z_LOWRANK>(ctx, (int)op->n3, a, nq);
  }
  ZKernel k = get_z((int)op->n3, mode);
  if (!k.fn) return set_err(ctx, FMMT_E_UNSUPPORTED, "no z kernel for n3=%lld", (long long)op->n3);
  ZArgs a;
  fill_zargs(op, a, (int)(p0 / std::max<int64_t>(1, op->PB)));
  a.W = Wb;
  a.ncomp = ncomp;
  a.p0 = p0;
  a.G = a.G ? a.G + (int64_t)qoff * a.g_stride : nullptr;
  if (!a.v_off && a.V) a.V += (int64_t)qoff * a.v_stride;
  a.Tout = Tout;
  const int lpc = fmmt::Z_THREADS / k.S;
  dim3 grid((unsigned)((a.n12 + lpc - 1) / lpc), (unsigned)nq);
  ProfScope ps(ctx, mode == fmmt::Z_RESTORE ? "restore_out" : (mode == fmmt::Z_DENSE ? "conv_z_dense" : "restore_conv_z"));
  k.fn<<<grid, fmmt::Z_THREADS, 0, ctx->stream>>>(a);
  FMMT_CUDA(ctx, cudaGetLastError());
  return FMMT_OK;
}

static fmmt_status run_batch_prep(fmmt_op* op, const Batch& b) {
  const bool tc = op->ctx->gemm_impl == 1;
  for (auto& L : b.gemms) {
    if (tc && L.pack_a_dyn) {   // A produced by the previous launch: pre-split it now
      int64_t items = 1;
      for (int i = 0; i < L.ndesc; ++i) {
        const GemmDesc& d = op->descs[L.first + i];
        items = std::max<int64_t>(items, (int64_t)d.batch * pk_a_floats_sub(d) / fmmt::TC_PACK_FLOATS * fmmt::TC_BM * 2);
      }
      if (fmmt_status st = launch_pack_a_multi(op->ctx, op->d_descs + L.first, L.ndesc, items)) return st;
    }
    if (tc && L.pack_dst)   // B produced by the previous launch
      if (fmmt_status st = launch_pack_b_bn(op->ctx, op->descs[L.first], L.tc_bn, L.pack_dst)) return st;
    fmmt_status st = launch_gemm(op, L);
    if (st) return st;
  }
  return FMMT_OK;
}

// The z-stage's dynamic operand of batch b: G_q packed (3D / Tucker / H-Tucker) or V_q packed (TT-4D).
static fmmt_status run_batch_zpack(fmmt_op* op, int bi) {
  fmmt_ctx* ctx = op->ctx;
  if (ctx->gemm_impl != 1 || op->format == FMMT_DENSE || op->zfused) return FMMT_OK;
  const Batch& b = op->batches[bi];
  if (op->format == FMMT_TT4D) {
    const unsigned ny = (unsigned)b.nq;
    ProfScope ps(ctx, "pack_v");
    if (op->n3 <= 16) fmmt::k_pk_pack_b_multi<16><<<dim3(16, ny), 256, 0, ctx->stream>>>(op->d_vitems, dslot(op, bi, 0));
    else if (op->n3 == 32) fmmt::k_pk_pack_b_multi<32><<<dim3(16, ny), 256, 0, ctx->stream>>>(op->d_vitems, dslot(op, bi, 0));
    else fmmt::k_pk_pack_b_multi<64><<<dim3(16, ny), 256, 0, ctx->stream>>>(op->d_vitems, dslot(op, bi, 0));
    FMMT_CUDA(ctx, cudaGetLastError());
    return FMMT_OK;
  }
  const int64_t items = op->gp_stride / fmmt::TC_PACK_FLOATS * fmmt::TC_BM * 2 * (b.zp_n == 1 ? b.nq : 1);
  return launch_pack_a_multi(ctx, op->d_descs + b.zp_first, b.zp_n, items);
}

// W: the half-padded spectra of one xy sub-batch (SB directions x ncomp components), sized so that the
// forward xy FFT, the z-stage and the inverse xy FFT of a sub-batch meet in L2 (ctx->w_mb; TT-4D keeps
// sub-batches of >= ZQB directions so its shared T1 still streams once per direction block).
static fmmt_status ensure_w(fmmt_op* op, int64_t ncomp) {
  if (ncomp <= op->w_ncomp && op->W) return FMMT_OK;
  drop_graphs(op);
  op->w_ncomp = std::max<int64_t>(ncomp, op->w_ncomp);
  const int64_t per_dir = op->w_ncomp * (op->n3 / 2) * op->n1 * op->n2 * 8;
  int64_t sb = std::max<int64_t>(1, ((int64_t)op->ctx->w_mb << 20) / per_dir);
  if (op->format == FMMT_TT4D) sb = std::max<int64_t>(sb, fmmt::ZQB);
  op->SB = std::min<int64_t>(sb, std::max<int64_t>(1, op->PB));
  dev_free(op, op->W);
  fmmt_status st = cmalloc(op, &op->W, op->SB * per_dir / 8);
  return st;
}

static fmmt_status translate_impl(fmmt_op* op, const fmmt_c64* sig_in, fmmt_c64* sig_out, int ncomp = 1) {
  const int Nz = (int)(op->n3 / 2);
  const float scale = (float)(1.0 / ((double)op->n1 * (double)op->n2 * (double)op->n3));
  const float2* in = reinterpret_cast<const float2*>(sig_in);
  float2* out = reinterpret_cast<float2*>(sig_out);
  // a1-a2: pruned x/y DFTs of all directions' (and components') planes in one launch (W holds
  // every half-padded spectrum, layout [p][comp][z]); per L2-sized batch: restore chain + fused
  // z-stage (one restore of T_p serves all ncomp components); a6: one launch back.
  // per batch: the restore GEMMs; then per xy sub-batch of SB directions: forward xy FFT into W, the fused
  // z-stage on W, inverse xy FFT out of W (W stays in L2 between the three launches)
  fmmt_status st;
  const int64_t K = (op->n1 / 2) * (op->n2 / 2) * (op->n3 / 2);
  if ((st = reset_dyn_slots(op))) return st;
  const int mode = op->format == FMMT_DENSE ? fmmt::Z_DENSE : fmmt::Z_LOWRANK;
  for (int bi = 0; bi < (int)op->batches.size(); ++bi) {
    const Batch& b = op->batches[bi];
    if ((st = run_batch_prep(op, b))) return st;
    if ((st = run_batch_zpack(op, bi))) return st;
    for (int s0 = 0; s0 < b.nq; s0 += (int)op->SB) {
      const int sn = (int)std::min<int64_t>(op->SB, b.nq - s0);
      const int64_t p = b.q0 + s0;
      const int planes = sn * ncomp * Nz;
      if (op->h2d_ev) {   // host path: the upload of these directions' chunks must have landed
        const int c = (int)std::min<int64_t>((p + sn - 1) / op->h2d_chunk, op->h2d_nchunks - 1);
        for (; op->h2d_waited <= c; ++op->h2d_waited)
          FMMT_CUDA(op->ctx, cudaStreamWaitEvent(op->ctx->stream, op->h2d_ev[op->h2d_waited], 0));
      }
      if ((st = launch_xy(op, true, in + p * ncomp * K, op->W, planes, 1.f))) return st;
      if ((st = launch_z(op, mode, (int)p, s0, sn, nullptr, op->W, ncomp))) return st;
      if ((st = launch_xy(op, false, op->W, out + p * ncomp * K, planes, scale))) return st;
    }
  }
  return FMMT_OK;
}

static fmmt_status check_translate_args(fmmt_op* op, const void* in, const void* out, int64_t ndir, int64_t Nx,
                                        int64_t Ny, int64_t Nz, int64_t ncomp = 1) {
  if (!op) return FMMT_E_ARG;
  fmmt_ctx* ctx = op->ctx;
  if (!op->translatable) return set_err(ctx, FMMT_E_UNSUPPORTED, "storage-only op (shape outside the translate path)");
  CHECK_ARG(ctx, in && out, "null signature pointer");
  CHECK_SHAPE(ctx, ndir == op->ndir, "ndir %lld != op ndir %lld", (long long)ndir, (long long)op->ndir);
  CHECK_SHAPE(ctx, 2 * Nx == op->n1 && 2 * Ny == op->n2 && 2 * Nz == op->n3, "grid %lldx%lldx%lld does not match op n=%lldx%lldx%lld",
              (long long)Nx, (long long)Ny, (long long)Nz, (long long)op->n1, (long long)op->n2, (long long)op->n3);
  CHECK_ARG(ctx, ncomp >= 1 && ncomp <= 16, "ncomp %lld not in [1, 16]", (long long)ncomp);
  const int64_t bytes = ndir * ncomp * Nx * Ny * Nz * 8;
  const char* a = (const char*)in;
  const char* b = (const char*)out;
  CHECK_ARG(ctx, a + bytes <= b || b + bytes <= a, "sig_in and sig_out overlap");
  cudaPointerAttributes pa, pb;
  if (cudaPointerGetAttributes(&pa, in) != cudaSuccess || cudaPointerGetAttributes(&pb, out) != cudaSuccess) {
    cudaGetLastError();
    return set_err(ctx, FMMT_E_ARG, "signature pointers are not CUDA device pointers");
  }
  CHECK_ARG(ctx, (pa.type == cudaMemoryTypeDevice || pa.type == cudaMemoryTypeManaged) &&
                     (pb.type == cudaMemoryTypeDevice || pb.type == cudaMemoryTypeManaged),
            "signature pointers must be device memory");
  if (pa.type == cudaMemoryTypeDevice && pa.device != ctx->device)
    return set_err(ctx, FMMT_E_STATE, "sig_in is on device %d, context on %d", pa.device, ctx->device);
  return FMMT_OK;
}

// Run `body` (the launches of one matvec) through a CUDA graph: the second
// call with the same buffers captures it, later calls replay it with one
// cudaGraphLaunch (the hot path is otherwise bound by ~300 host-side kernel
// launches per matvec).  Direct launches when profiling (per-kernel events) or
// on the legacy default stream (not capturable).
struct NvtxRange {
  explicit NvtxRange(const char* n) { nvtxRangePushA(n); }
  ~NvtxRange() { nvtxRangePop(); }
};

template <class F>
static fmmt_status run_graphed(fmmt_op* op, const void* k0, const void* k1, const void* k2, const void* k3, int64_t k4,
                               F&& body, const void* k5 = nullptr) {
  fmmt_ctx* ctx = op->ctx;
  NvtxRange nr("fmmt_matvec");
  if (ctx->stream == nullptr || !ctx->use_graphs) return body();
  if (ctx->profiling) {
    // per-kernel profile: capture the matvec with its event-record nodes and run it as one
    // graph, so the events time the kernels back to back (not host launch gaps)
    cudaGraph_t graph = nullptr;
    FMMT_CUDA(ctx, cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeRelaxed));
    fmmt_status st = body();
    cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
    if (st) {
      if (graph) cudaGraphDestroy(graph);
      return st;
    }
    if (e != cudaSuccess) return set_err(ctx, FMMT_E_CUDA, "graph capture failed: %s", cudaGetErrorString(e));
    cudaGraphExec_t exec = nullptr;
    e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return set_err(ctx, FMMT_E_CUDA, "graph instantiate failed: %s", cudaGetErrorString(e));
    ctx->prof_execs.push_back(exec);
    FMMT_CUDA(ctx, cudaGraphLaunch(exec, ctx->stream));
    return FMMT_OK;
  }
  fmmt_op::GraphEntry* ge = nullptr;
  for (auto& g : op->graphs)
    if (g.key[0] == k0 && g.key[1] == k1 && g.key[2] == k2 && g.key[3] == k3 && g.key[4] == (const void*)k4 &&
        g.key[5] == k5)
      ge = &g;
  if (ge && ge->exec) {
    FMMT_CUDA(ctx, cudaGraphLaunch(ge->exec, ctx->stream));
    ctx->launches += ge->launches;
    return FMMT_OK;
  }
  if (!ge) {   // first call: run directly (allocates lazily sized workspaces), remember the key
    fmmt_op::GraphEntry e;
    e.key[0] = k0; e.key[1] = k1; e.key[2] = k2; e.key[3] = k3; e.key[4] = (const void*)k4; e.key[5] = k5;
    e.calls = 1;
    op->graphs.push_back(e);
    return body();
  }
  cudaGraph_t graph = nullptr;
  FMMT_CUDA(ctx, cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeRelaxed));
  const int64_t l0 = ctx->launches;
  fmmt_status st = body();
  cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
  if (st) {
    if (graph) cudaGraphDestroy(graph);
    return st;
  }
  if (e != cudaSuccess) return set_err(ctx, FMMT_E_CUDA, "graph capture failed: %s", cudaGetErrorString(e));
  cudaGraphExec_t exec = nullptr;
  e = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return set_err(ctx, FMMT_E_CUDA, "graph instantiate failed: %s", cudaGetErrorString(e));
  ge->exec = exec;
  ge->launches = ctx->launches - l0;
  FMMT_CUDA(ctx, cudaGraphLaunch(exec, ctx->stream));
  return FMMT_OK;
}

// ============================================================== C ABI
extern "C" {

int fmmt_version(void) { return FMMT_VERSION; }

fmmt_status fmmt_init(int device, void* cuda_stream, fmmt_ctx** out) {
  return fmmt_init_sharded(device, cuda_stream, 0, 1, nullptr, out);
}

fmmt_status fmmt_nccl_unique_id(void* out128) {
  if (!out128) return FMMT_E_ARG;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return FMMT_E_NCCL;
  memcpy(out128, &id, 128);
  return FMMT_OK;
}

fmmt_status fmmt_init_sharded(int device, void* cuda_stream, int rank, int world, const void* nccl_id, fmmt_ctx** out) {
  if (!out) return FMMT_E_ARG;
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world) return FMMT_E_ARG;
  if (world > 1 && !nccl_id) return FMMT_E_ARG;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    return FMMT_E_CUDA;
  }
  if (cudaSetDevice(device) != cudaSuccess) return FMMT_E_CUDA;
  fmmt_ctx* ctx = new fmmt_ctx();
  ctx->device = device;
  ctx->stream = (cudaStream_t)cuda_stream;
  ctx->rank = rank;
  ctx->world = world;
  if (const char* e = getenv("FMMT_GEMM")) ctx->gemm_impl = (strcmp(e, "ffma") == 0) ? 0 : 1;
  if (const char* e = getenv("FMMT_GRAPHS")) ctx->use_graphs = atoi(e) != 0;
  if (const char* e = getenv("FMMT_AGG_STAGED")) ctx->agg_staged = atoi(e) != 0;
  if (const char* e = getenv("FMMT_TC_CTAS")) ctx->tc_ctas_per_sm = std::max(1, atoi(e));
  if (const char* e = getenv("FMMT_BATCH_MB")) ctx->batch_mb = std::max(1, atoi(e));
  if (const char* e = getenv("FMMT_W_MB")) ctx->w_mb = std::max(1, atoi(e));
  if (const char* e = getenv("FMMT_ZCLUSTER")) ctx->z_cluster = atoi(e) != 0;
  if (const char* e = getenv("FMMT_XY_BIG")) xy_big_enabled = atoi(e) != 0;
  if (const char* e = getenv("FMMT_XY_HALF")) xy_half_enabled = atoi(e) != 0;
  if (const char* e = getenv("FMMT_ZFUSE")) ctx->z_fuse = atoi(e) != 0;
  if (const char* e = getenv("FMMT_ZFC")) ctx->z_fc = atoi(e);
  if (const char* e = getenv("FMMT_H2D_OVERLAP")) ctx->h2d_overlap = atoi(e) != 0;
  if (const char* e = getenv("FMMT_TC_CTAS_Z")) ctx->tc_ctas_z = std::max(1, atoi(e));
  cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (world > 1 || nccl_id) {   // world == 1 with an id: a single-rank communicator (the collective paths still run)
    ncclUniqueId id;
    memcpy(&id, nccl_id, 128);
    ncclComm_t comm;
    ncclResult_t r = ncclCommInitRank(&comm, world, id, rank);
    if (r != ncclSuccess) {
      delete ctx;
      return FMMT_E_NCCL;
    }
    ctx->nccl_comm = comm;
  }
  *out = ctx;
  return FMMT_OK;
}

void fmmt_destroy(fmmt_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (auto& pe : ctx->pending) {
    cudaEventDestroy(pe.e0);
    cudaEventDestroy(pe.e1);
  }
  for (auto e : ctx->event_pool) cudaEventDestroy(e);
  for (auto e : ctx->h2d_events) cudaEventDestroy(e);
  if (ctx->h2d_fence) cudaEventDestroy(ctx->h2d_fence);
  if (ctx->copy_stream) {
    cudaStreamSynchronize(ctx->copy_stream);
    cudaStreamDestroy(ctx->copy_stream);
  }
  if (ctx->nccl_comm) ncclCommDestroy((ncclComm_t)ctx->nccl_comm);
  if (ctx->agg_part) cudaFree(ctx->agg_part);
  fmmt_internal::setup_release(ctx);
  delete ctx;
}

fmmt_status fmmt_sync(fmmt_ctx* ctx) {
  if (!ctx) return FMMT_E_ARG;
  cudaSetDevice(ctx->device);
  FMMT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  FMMT_CUDA(ctx, cudaGetLastError());
  return FMMT_OK;
}

const char* fmmt_last_error(const fmmt_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

fmmt_status fmmt_shard_range(int64_t ndir, int rank, int world, int64_t* begin, int64_t* count) {
  if (!begin || !count || world < 1 || rank < 0 || rank >= world || ndir < 0) return FMMT_E_ARG;
  const int64_t base = ndir / world, rem = ndir % world;
  // the first `rem` ranks get one extra direction
  *begin = rank * base + std::min<int64_t>(rank, rem);
  *count = base + (rank < rem ? 1 : 0);
  return FMMT_OK;
}

fmmt_status fmmt_set_profiling(fmmt_ctx* ctx, int enable) {
  if (!ctx) return FMMT_E_ARG;
  ctx->profiling = enable != 0;
  return FMMT_OK;
}

fmmt_status fmmt_prof_reset(fmmt_ctx* ctx) {
  if (!ctx) return FMMT_E_ARG;
  prof_flush(ctx);
  ctx->prof.clear();
  return FMMT_OK;
}

fmmt_status fmmt_prof_read(fmmt_ctx* ctx, const char** names, double* ms, int64_t* launches, int64_t cap, int64_t* count) {
  if (!ctx || !count) return FMMT_E_ARG;
  prof_flush(ctx);
  *count = (int64_t)ctx->prof.size();
  for (int64_t i = 0; i < std::min<int64_t>(cap, *count); ++i) {
    if (names) names[i] = ctx->prof[i].first;
    if (ms) ms[i] = ctx->prof[i].second.first;
    if (launches) launches[i] = ctx->prof[i].second.second;
  }
  return FMMT_OK;
}

int64_t fmmt_launch_count(const fmmt_ctx* ctx) { return ctx ? ctx->launches : -1; }

fmmt_status fmmt_set_gemm_impl(fmmt_ctx* ctx, int impl) {
  if (!ctx || impl < 0 || impl > 1) return FMMT_E_ARG;
  ctx->gemm_impl = impl;
  return FMMT_OK;
}

fmmt_status fmmt_test_cgemm(fmmt_ctx* ctx, int impl, int64_t m, int64_t n, int64_t k, int transA, int transB,
                            const fmmt_c64* A, int64_t lda, const fmmt_c64* B, int64_t ldb, fmmt_c64* C, int64_t ldc) {
  if (!ctx) return FMMT_E_ARG;
  CHECK_ARG(ctx, impl >= 0 && impl <= 1, "impl must be 0 (FFMA) or 1 (tcgen05)");
  CHECK_ARG(ctx, A && B && C, "null matrix");
  CHECK_SHAPE(ctx, m >= 1 && n >= 1 && k >= 1 && m < (1 << 30) && n < (1 << 30) && k < (1 << 30), "bad gemm dims");
  cudaSetDevice(ctx->device);
  GemmDesc d = gd(reinterpret_cast<const float2*>(A), reinterpret_cast<const float2*>(B), reinterpret_cast<float2*>(C),
                  m, n, k, transB, lda, ldb, ldc);
  if (transA) { d.a_s0 = lda; d.a_sk = 1; }
  // operand scales of the fp16 split over the referenced extents
  float* sl = nullptr;
  FMMT_CUDA(ctx, cudaMallocAsync((void**)&sl, 8, ctx->stream));
  FMMT_CUDA(ctx, cudaMemsetAsync(sl, 0, 8, ctx->stream));
  fmmt_status st = absmax_ctx(ctx, d.A, (m - 1) * d.a_s0 + (k - 1) * d.a_sk + 1, sl);
  if (!st) st = absmax_ctx(ctx, d.B, (k - 1) * d.b_sk + (n - 1) * d.b_sn + 1, sl + 1);
  d.amax = sl;
  d.bmax = sl + 1;
  float *apk = nullptr, *bpk = nullptr;
  GemmDesc* dd = nullptr;
  if (!st && impl == 1) {   // the tensor-core pipeline streams both operands pre-split
    const int bn = n >= 32 ? 32 : 16;   // (add_gemm's choice for one descriptor)
    FMMT_CUDA(ctx, cudaMallocAsync((void**)&apk, pk_a_floats_sub(d) * 4, ctx->stream));
    FMMT_CUDA(ctx, cudaMallocAsync((void**)&bpk, pk_b_floats_sub(d, bn) * 4, ctx->stream));
    d.Ap = apk;
    d.a_nkc = (int)((k + fmmt::TC_BK - 1) / fmmt::TC_BK);
    d.Bp = bpk;
    FMMT_CUDA(ctx, cudaMallocAsync((void**)&dd, sizeof(GemmDesc), ctx->stream));
    FMMT_CUDA(ctx, cudaMemcpyAsync(dd, &d, sizeof(GemmDesc), cudaMemcpyHostToDevice, ctx->stream));
    st = launch_pack_a_multi(ctx, dd, 1, pk_a_floats_sub(d) / fmmt::TC_PACK_FLOATS * fmmt::TC_BM * 4);
    if (!st) st = launch_pack_b_bn(ctx, d, bn, bpk);
  }
  if (!st) st = run_one_gemm(ctx, d, impl, "test_cgemm");
  if (dd) cudaFreeAsync(dd, ctx->stream);
  if (apk) cudaFreeAsync(apk, ctx->stream);
  if (bpk) cudaFreeAsync(bpk, ctx->stream);
  cudaFreeAsync(sl, ctx->stream);
  return st;
}

fmmt_status fmmt_op_import(fmmt_ctx* ctx, fmmt_format format, int64_t n1, int64_t n2, int64_t n3, int64_t ndir,
                           const int64_t* ranks, const fmmt_c64* const* arrays, int64_t narrays, fmmt_op** op) {
  return fmmt_internal::create_op(ctx, format, n1, n2, n3, ndir, ranks, (const void* const*)arrays, narrays, op, false);
}

fmmt_status fmmt_op_info(const fmmt_op* op, fmmt_op_info_t* info) {
  if (!op || !info) return FMMT_E_ARG;
  memset(info, 0, sizeof(*info));
  info->format = op->format;
  info->n1 = op->n1; info->n2 = op->n2; info->n3 = op->n3; info->ndir = op->ndir;
  info->nranks = op->nslots;
  const bool per_dir = op->format == FMMT_TUCKER3D || op->format == FMMT_TT3D;
  for (int s = 0; s < op->nslots; ++s) {
    int64_t mx = 0;
    double mean = 0;
    const int64_t cnt = per_dir ? op->ndir : 1;
    for (int64_t p = 0; p < cnt; ++p) {
      int64_t r = rk(op, p, s);
      mx = std::max(mx, r);
      mean += (double)r;
    }
    info->rank_max[s] = mx;
    info->rank_mean[s] = mean / (double)cnt;
  }
  int64_t comp = 0;
  for (auto e : op->arr_elems) comp += e;
  info->compressed_bytes = comp * 8;
  info->original_bytes = op->n1 * op->n2 * op->n3 * op->ndir * 8;
  // everything else the op holds on the device: derived / pre-split operands (T1, E, packed factors) and
  // the matvec workspaces (mem registry; compressed_bytes counts the factors alone)
  info->workspace_bytes = mem_bytes(op, MEM_DERIVED) + mem_bytes(op, MEM_WORKSPACE);
  info->batch = op->PB;
  // restore complex MACs per matvec (a3 + a4), in the contraction order the kernels use
  const int64_t n1 = op->n1, n2 = op->n2, n3 = op->n3, n = n1 * n2 * n3;
  double cm = 0;
  for (int64_t p = 0; p < op->ndir; ++p) {
    switch (op->format) {
      case FMMT_DENSE: break;
      case FMMT_TUCKER3D: case FMMT_TUCKER4D: {
        const double r1 = rk(op, p, 0), r2 = rk(op, p, 1), r3 = rk(op, p, 2);
        cm += n1 * r1 * r2 * r3 + n1 * n2 * r2 * r3 + (double)n * r3;
        if (op->format == FMMT_TUCKER4D) cm += r1 * r2 * r3 * rk(op, 0, 3);
        break;
      }
      case FMMT_HTUCKER4D: {
        // M_p (r3 r4 r34) + G_p = E . M_p^T (n1 n2 r34 r3) + z-stage (n r3); E is per op
        const double r3 = rk(op, 0, 2), r4 = rk(op, 0, 3), r34 = rk(op, 0, 5);
        cm += r3 * r4 * r34 + (double)n1 * n2 * r34 * r3 + (double)n * r3;
        break;
      }
      case FMMT_TT3D: {
        const double r1 = rk(op, p, 0), r2 = rk(op, p, 1);
        cm += n1 * r1 * n2 * r2 + (double)n * r2;
        break;
      }
      case FMMT_TT4D: {
        const double r2 = rk(op, 0, 1), r3 = rk(op, 0, 2);
        cm += r2 * n3 * r3 + (double)n * r2;
        break;
      }
    }
  }
  info->restore_cmac = cm;
  info->translatable = op->translatable ? 1 : 0;
  return FMMT_OK;
}

fmmt_status fmmt_op_export(const fmmt_op* op, int64_t index, fmmt_c64* dst, int64_t cap, int64_t* count) {
  if (!op || !count) return FMMT_E_ARG;
  fmmt_ctx* ctx = op->ctx;
  CHECK_ARG(ctx, index >= 0 && index < (int64_t)op->arr.size(), "array index %lld not in [0, %lld)", (long long)index,
            (long long)op->arr.size());
  *count = op->arr_elems[index];
  if (!dst) return FMMT_OK;
  CHECK_ARG(ctx, cap >= *count, "export buffer too small (%lld < %lld)", (long long)cap, (long long)*count);
  cudaSetDevice(ctx->device);
  FMMT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  FMMT_CUDA(ctx, cudaMemcpy(dst, op->arr[index], *count * sizeof(float2), cudaMemcpyDefault));
  return FMMT_OK;
}

fmmt_status fmmt_op_ranks(const fmmt_op* op, int64_t* ranks, int64_t cap, int64_t* count) {
  if (!op || !count) return FMMT_E_ARG;
  *count = (int64_t)op->ranks.size();
  if (ranks) {
    if (cap < *count) return set_err(op->ctx, FMMT_E_ARG, "rank buffer too small (%lld < %lld)", (long long)cap, (long long)*count);
    for (int64_t i = 0; i < *count; ++i) ranks[i] = op->ranks[i];
  }
  return FMMT_OK;
}

// ---------------------------------------------------------------- op serialisation (skip re-compression)
// File: magic "FMMTOP\1\0", int64 {format, n1, n2, n3, ndir, nranks, narrays}, int64 ranks[nranks], then per
// array int64 count + count complex64 (the fmmt_op_import order and layout), then a uint64 checksum of the array
// payload.  Little-endian, as the host writes it.
static const char OP_MAGIC[8] = {'F', 'M', 'M', 'T', 'O', 'P', 1, 0};

static uint64_t payload_sum(uint64_t h, const void* data, size_t bytes) {
  const uint64_t* w = static_cast<const uint64_t*>(data);   // complex64 payloads: multiples of 8 bytes
  for (size_t i = 0; i < bytes / 8; ++i) h = ((h << 7) | (h >> 57)) ^ (w[i] * 0x9E3779B97F4A7C15ull);
  return h;
}

fmmt_status fmmt_op_save(const fmmt_op* op, const char* path) {
  if (!op) return FMMT_E_ARG;
  fmmt_ctx* ctx = op->ctx;
  CHECK_ARG(ctx, path && *path, "null path");
  FILE* f = fopen(path, "wb");
  if (!f) return set_err(ctx, FMMT_E_STATE, "cannot open %s for writing", path);
  const int64_t hdr[7] = {(int64_t)op->format, op->n1, op->n2, op->n3, op->ndir, (int64_t)op->ranks.size(),
                          (int64_t)op->arr.size()};
  bool ok = fwrite(OP_MAGIC, 1, 8, f) == 8 && fwrite(hdr, 8, 7, f) == 7 &&
            fwrite(op->ranks.data(), 8, op->ranks.size(), f) == op->ranks.size();
  uint64_t sum = 0;
  std::vector<float2> host;
  fmmt_status st = FMMT_OK;
  for (size_t i = 0; ok && !st && i < op->arr.size(); ++i) {
    int64_t cnt = 0;
    host.resize((size_t)std::max<int64_t>(1, op->arr_elems[i]));
    st = fmmt_op_export(op, (int64_t)i, reinterpret_cast<fmmt_c64*>(host.data()), (int64_t)host.size(), &cnt);
    if (st) break;
    ok = fwrite(&cnt, 8, 1, f) == 1 && fwrite(host.data(), 8, (size_t)cnt, f) == (size_t)cnt;
    sum = payload_sum(sum, host.data(), (size_t)cnt * 8);
  }
  ok = ok && !st && fwrite(&sum, 8, 1, f) == 1;
  ok = (fclose(f) == 0) && ok;
  if (st) return st;
  if (!ok) return set_err(ctx, FMMT_E_STATE, "short write to %s", path);
  return FMMT_OK;
}

fmmt_status fmmt_op_load(fmmt_ctx* ctx, const char* path, fmmt_op** out) {
  if (!ctx || !out) return FMMT_E_ARG;
  *out = nullptr;
  CHECK_ARG(ctx, path && *path, "null path");
  FILE* f = fopen(path, "rb");
  if (!f) return set_err(ctx, FMMT_E_STATE, "cannot open %s", path);
  struct Closer {
    FILE* f;
    ~Closer() { fclose(f); }
  } closer{f};
  char magic[8];
  int64_t hdr[7];
  if (fread(magic, 1, 8, f) != 8 || memcmp(magic, OP_MAGIC, 8) != 0 || fread(hdr, 8, 7, f) != 7)
    return set_err(ctx, FMMT_E_STATE, "%s is not an fmmt op file", path);
  const int64_t format = hdr[0], ndir = hdr[4], nranks = hdr[5], narr = hdr[6];
  if (format < FMMT_DENSE || format > FMMT_TT4D || ndir < 1 || nranks < 0 || nranks > 6 * ndir || narr < 1 || narr > 8)
    return set_err(ctx, FMMT_E_STATE, "%s: bad header", path);
  std::vector<int64_t> ranks((size_t)nranks);
  if (fread(ranks.data(), 8, (size_t)nranks, f) != (size_t)nranks) return set_err(ctx, FMMT_E_STATE, "%s: truncated", path);
  fseek(f, 0, SEEK_END);
  const int64_t fsize = (int64_t)ftell(f);
  fseek(f, 8 + 7 * 8 + nranks * 8, SEEK_SET);
  std::vector<std::vector<float2>> arrays((size_t)narr);
  std::vector<const void*> ptrs((size_t)narr);
  uint64_t sum = 0;
  for (int64_t i = 0; i < narr; ++i) {
    int64_t cnt = -1;
    if (fread(&cnt, 8, 1, f) != 1 || cnt < 0 || cnt * 8 > fsize) return set_err(ctx, FMMT_E_STATE, "%s: truncated", path);
    arrays[i].resize((size_t)std::max<int64_t>(1, cnt));
    if (fread(arrays[i].data(), 8, (size_t)cnt, f) != (size_t)cnt) return set_err(ctx, FMMT_E_STATE, "%s: truncated", path);
    sum = payload_sum(sum, arrays[i].data(), (size_t)cnt * 8);
    ptrs[i] = arrays[i].data();
  }
  uint64_t stored = 0;
  if (fread(&stored, 8, 1, f) != 1 || stored != sum) return set_err(ctx, FMMT_E_STATE, "%s: checksum mismatch", path);
  // shapes and the rank chain are validated by create_op exactly as for fmmt_op_import
  return fmmt_internal::create_op(ctx, (fmmt_format)format, hdr[1], hdr[2], hdr[3], ndir, nranks ? ranks.data() : nullptr,
                                  ptrs.data(), narr, out, true);
}

fmmt_status fmmt_op_set_batch(fmmt_op* op, int64_t dirs) {
  if (!op || dirs < 0) return FMMT_E_ARG;
  if (!op->translatable) return set_err(op->ctx, FMMT_E_UNSUPPORTED, "storage-only op");
  cudaSetDevice(op->ctx->device);
  drop_graphs(op);
  op->PB = std::min<int64_t>(dirs, op->ndir);
  return build_plans(op);
}

fmmt_status fmmt_translate(fmmt_op* op, const fmmt_c64* sig_in, fmmt_c64* sig_out, int64_t ndir, int64_t Nx, int64_t Ny,
                           int64_t Nz) {
  fmmt_status st = check_translate_args(op, sig_in, sig_out, ndir, Nx, Ny, Nz);
  if (st) return st;
  cudaSetDevice(op->ctx->device);
  if ((st = ensure_w(op, 1))) return st;
  return run_graphed(op, sig_in, sig_out, nullptr, nullptr, 1, [&] { return translate_impl(op, sig_in, sig_out, 1); });
}

fmmt_status fmmt_translate_multi(fmmt_op* op, const fmmt_c64* sig_in, fmmt_c64* sig_out, int64_t ndir, int64_t ncomp,
                                 int64_t Nx, int64_t Ny, int64_t Nz) {
  fmmt_status st = check_translate_args(op, sig_in, sig_out, ndir, Nx, Ny, Nz, ncomp);
  if (st) return st;
  cudaSetDevice(op->ctx->device);
  if ((st = ensure_w(op, ncomp))) return st;
  return run_graphed(op, sig_in, sig_out, nullptr, nullptr, ncomp,
                     [&] { return translate_impl(op, sig_in, sig_out, (int)ncomp); });
}

static fmmt_status dirsum_and_reduce(fmmt_op* op, const float2* sig, const float* w, float2* sum_out, int ncomp = 1) {
  fmmt_ctx* ctx = op->ctx;
  const int64_t K = (op->n1 / 2) * (op->n2 / 2) * (op->n3 / 2) * ncomp;   // [comp][Nz][Ny][Nx] per direction
  // direction splits: enough (K x nsplit) threads to fill the GPU, at most 64 (k_dirsum_final: a warp per output)
  const int nsplit = (int)std::max<int64_t>(
      1, std::min<int64_t>(std::min<int64_t>(op->ndir, 64), (int64_t)ctx->num_sms * 1024 / std::max<int64_t>(K, 1)));
  if (nsplit > 1 && (!op->partial || op->partial_elems < (int64_t)nsplit * K)) {
    // captured matvec graphs hold the old buffer: drop them first (this call is never captured: a new
    // graph key always runs once directly before it is captured, see run_graphed)
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(ctx->stream, &cs);
    if (cs != cudaStreamCaptureStatusNone) return set_err(ctx, FMMT_E_STATE, "direction-sum workspace grows during capture");
    drop_graphs(op);
    dev_free(op, op->partial);
    op->partial_elems = 0;
    fmmt_status st = cmalloc(op, &op->partial, (int64_t)nsplit * K);
    if (st) return st;
    op->partial_elems = (int64_t)nsplit * K;
  }
  {
    ProfScope ps(ctx, "dirsum_partial");
    dim3 grid((unsigned)((K + 127) / 128), (unsigned)nsplit);
    fmmt::k_dirsum_partial<<<grid, 128, 0, ctx->stream>>>(sig, w, nsplit > 1 ? op->partial : sum_out, K, (int)op->ndir,
                                                           nsplit);
    FMMT_CUDA(ctx, cudaGetLastError());
  }
  if (nsplit > 1) {
    ProfScope ps(ctx, "dirsum_final");
    fmmt::k_dirsum_final<<<(unsigned)((K + 7) / 8), 256, 0, ctx->stream>>>(op->partial, sum_out, K, nsplit);
    FMMT_CUDA(ctx, cudaGetLastError());
  }
  if (ctx->nccl_comm) {
    ncclResult_t r = ncclAllReduce(sum_out, sum_out, (size_t)(2 * K), ncclFloat, ncclSum, (ncclComm_t)ctx->nccl_comm, ctx->stream);
    if (r != ncclSuccess) return set_err(ctx, FMMT_E_NCCL, "ncclAllReduce: %s", ncclGetErrorString(r));
  }
  return FMMT_OK;
}

fmmt_status fmmt_translate_sum_multi(fmmt_op* op, const fmmt_c64* sig_in, fmmt_c64* sig_out, const float* w,
                                     fmmt_c64* sum_out, int64_t ndir, int64_t ncomp, int64_t Nx, int64_t Ny, int64_t Nz) {
  if (!op) return FMMT_E_ARG;
  fmmt_ctx* ctx = op->ctx;
  CHECK_ARG(ctx, w && sum_out, "null weight or sum pointer");
  CHECK_ARG(ctx, ncomp >= 1 && ncomp <= 16, "ncomp %lld not in [1, 16]", (long long)ncomp);
  cudaSetDevice(ctx->device);
  if (!sig_out) {
    const int64_t need = op->ndir * ncomp * (op->n1 / 2) * (op->n2 / 2) * (op->n3 / 2);
    if (!op->sigtmp || op->sigtmp_elems < need) {
      drop_graphs(op);
      dev_free(op, op->sigtmp);
      fmmt_status st = cmalloc(op, &op->sigtmp, need);
      if (st) return st;
      op->sigtmp_elems = need;
    }
    sig_out = reinterpret_cast<fmmt_c64*>(op->sigtmp);
  }
  fmmt_status st = check_translate_args(op, sig_in, sig_out, ndir, Nx, Ny, Nz, ncomp);
  if (st) return st;
  if ((st = ensure_w(op, ncomp))) return st;
  return run_graphed(op, sig_in, sig_out, w, sum_out, ncomp, [&] {
    fmmt_status s2 = translate_impl(op, sig_in, sig_out, (int)ncomp);
    if (s2) return s2;
    return dirsum_and_reduce(op, reinterpret_cast<const float2*>(sig_out), w, reinterpret_cast<float2*>(sum_out),
                             (int)ncomp);
  });
}

fmmt_status fmmt_translate_sum(fmmt_op* op, const fmmt_c64* sig_in, fmmt_c64* sig_out, const float* w, fmmt_c64* sum_out,
                               int64_t ndir, int64_t Nx, int64_t Ny, int64_t Nz) {
  return fmmt_translate_sum_multi(op, sig_in, sig_out, w, sum_out, ndir, 1, Nx, Ny, Nz);
}

fmmt_status fmmt_translate_sum_host(fmmt_op* op, const fmmt_c64* sig_in_host, const float* w_host, fmmt_c64* sum_out_host,
                                    int64_t ndir, int64_t Nx, int64_t Ny, int64_t Nz) {
  if (!op) return FMMT_E_ARG;
  fmmt_ctx* ctx = op->ctx;
  CHECK_ARG(ctx, sig_in_host && w_host && sum_out_host, "null host pointer");
  if (!op->translatable) return set_err(ctx, FMMT_E_UNSUPPORTED, "storage-only op");
  CHECK_SHAPE(ctx, ndir == op->ndir, "ndir %lld != op ndir %lld", (long long)ndir, (long long)op->ndir);
  // shape first: the staging buffers are sized from the op, never from the caller's arguments
  CHECK_SHAPE(ctx, 2 * Nx == op->n1 && 2 * Ny == op->n2 && 2 * Nz == op->n3, "grid %lldx%lldx%lld does not match op n=%lldx%lldx%lld",
              (long long)Nx, (long long)Ny, (long long)Nz, (long long)op->n1, (long long)op->n2, (long long)op->n3);
  cudaSetDevice(ctx->device);
  const int64_t K = (op->n1 / 2) * (op->n2 / 2) * (op->n3 / 2);
  if (!op->d_in_host) {
    fmmt_status st;
    if ((st = dev_alloc(op, &op->d_in_host, op->ndir * K * 8, MEM_WORKSPACE, "host staging")) ||
        (st = dev_alloc(op, &op->d_w_host, op->ndir * 4, MEM_WORKSPACE, "host staging")) ||
        (st = dev_alloc(op, &op->d_sum_host, K * 8, MEM_WORKSPACE, "host staging")))
      return st;
  }
  if (!ctx->h2d_overlap || ctx->stream == nullptr || ctx->profiling) {
    FMMT_CUDA(ctx, cudaMemcpyAsync(op->d_in_host, sig_in_host, ndir * K * sizeof(float2), cudaMemcpyHostToDevice, ctx->stream));
    FMMT_CUDA(ctx, cudaMemcpyAsync(op->d_w_host, w_host, ndir * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
    fmmt_status st = fmmt_translate_sum(op, reinterpret_cast<const fmmt_c64*>(op->d_in_host), nullptr, op->d_w_host,
                                        reinterpret_cast<fmmt_c64*>(op->d_sum_host), ndir, Nx, Ny, Nz);
    if (st) return st;
  } else {
    // Overlapped upload: the signatures go up in chunks of one xy sub-batch of directions on a copy stream, an
    // event after each; the matvec is launched directly (no graph) and waits for a chunk only before the first
    // kernel that reads it (the forward xy FFT of that sub-batch), so the restore GEMMs and the earlier
    // sub-batches run under the copy.
    fmmt_status st = ensure_w(op, 1);   // fixes op->SB, the xy sub-batch (the upload chunk)
    if (st) return st;
    if (!ctx->copy_stream) {
      FMMT_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
      FMMT_CUDA(ctx, cudaEventCreateWithFlags(&ctx->h2d_fence, cudaEventDisableTiming));
    }
    const int64_t chunk = std::max<int64_t>(std::max<int64_t>(1, op->SB), (ndir + 63) / 64);
    const int nchunks = (int)((ndir + chunk - 1) / chunk);
    while ((int)ctx->h2d_events.size() < nchunks) {
      cudaEvent_t ev;
      FMMT_CUDA(ctx, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      ctx->h2d_events.push_back(ev);
    }
    // the staging buffer's earlier readers are on ctx->stream
    FMMT_CUDA(ctx, cudaEventRecord(ctx->h2d_fence, ctx->stream));
    FMMT_CUDA(ctx, cudaStreamWaitEvent(ctx->copy_stream, ctx->h2d_fence, 0));
    for (int c = 0; c < nchunks; ++c) {
      const int64_t d0 = c * chunk, dn = std::min<int64_t>(chunk, ndir - d0);
      FMMT_CUDA(ctx, cudaMemcpyAsync(op->d_in_host + d0 * K, reinterpret_cast<const float2*>(sig_in_host) + d0 * K,
                                     dn * K * sizeof(float2), cudaMemcpyHostToDevice, ctx->copy_stream));
      FMMT_CUDA(ctx, cudaEventRecord(ctx->h2d_events[c], ctx->copy_stream));
    }
    FMMT_CUDA(ctx, cudaMemcpyAsync(op->d_w_host, w_host, ndir * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
    if (!op->sigtmp || op->sigtmp_elems < ndir * K) {
      drop_graphs(op);
      dev_free(op, op->sigtmp);
      if (!(st = cmalloc(op, &op->sigtmp, ndir * K))) op->sigtmp_elems = ndir * K;
    }
    if (!st) st = check_translate_args(op, op->d_in_host, op->sigtmp, ndir, Nx, Ny, Nz, 1);
    if (!st) {
      NvtxRange nr("fmmt_matvec_host");
      op->h2d_ev = ctx->h2d_events.data();
      op->h2d_chunk = chunk;
      op->h2d_nchunks = nchunks;
      op->h2d_waited = 0;
      st = translate_impl(op, reinterpret_cast<const fmmt_c64*>(op->d_in_host), reinterpret_cast<fmmt_c64*>(op->sigtmp), 1);
      // every chunk is waited on even if a sub-batch loop ended early: the next call reuses the staging buffer
      for (; op->h2d_waited < nchunks; ++op->h2d_waited) cudaStreamWaitEvent(ctx->stream, op->h2d_ev[op->h2d_waited], 0);
      op->h2d_ev = nullptr;
      if (!st) st = dirsum_and_reduce(op, op->sigtmp, op->d_w_host, op->d_sum_host, 1);
    }
    if (st) {
      cudaStreamSynchronize(ctx->copy_stream);
      return st;
    }
  }
  FMMT_CUDA(ctx, cudaMemcpyAsync(sum_out_host, op->d_sum_host, K * sizeof(float2), cudaMemcpyDeviceToHost, ctx->stream));
  FMMT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return FMMT_OK;
}

// ---------------------------------------------------------------- aggregation / disaggregation
static fmmt_status check_device_ptr(fmmt_ctx* ctx, const void* ptr, const char* what) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();
    return set_err(ctx, FMMT_E_ARG, "%s is not a CUDA device pointer", what);
  }
  if (!(a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged))
    return set_err(ctx, FMMT_E_ARG, "%s must be device memory", what);
  if (a.type == cudaMemoryTypeDevice && a.device != ctx->device)
    return set_err(ctx, FMMT_E_STATE, "%s is on device %d, context on %d", what, a.device, ctx->device);
  return FMMT_OK;
}

static fmmt_status check_agg_args(fmmt_ctx* ctx, const void* P, const void* box_ptr, int64_t ndir, int64_t N,
                                  int64_t ncomp, int64_t Nx, int64_t Ny, int64_t Nz) {
  CHECK_ARG(ctx, P && box_ptr, "null pointer");
  CHECK_SHAPE(ctx, ndir >= 1 && N >= 0 && Nx >= 1 && Ny >= 1 && Nz >= 1, "bad sizes ndir %lld N %lld grid %lldx%lldx%lld",
              (long long)ndir, (long long)N, (long long)Nx, (long long)Ny, (long long)Nz);
  CHECK_ARG(ctx, ncomp >= 1 && ncomp <= 16, "ncomp %lld not in [1, 16]", (long long)ncomp);
  fmmt_status st;
  if ((st = check_device_ptr(ctx, box_ptr, "box_ptr"))) return st;
  if (N > 0 && (st = check_device_ptr(ctx, P, "P"))) return st;
  return FMMT_OK;
}

static fmmt_status aggregate_impl(fmmt_ctx* ctx, const float2* P, const float2* I, const int64_t* box_ptr, int64_t ndir,
                                  int64_t N, int ncomp, int64_t K, float2* sig) {
  ProfScope ps(ctx, "aggregate");
  // a warp per (box, block of AGG_PD directions); the generic kernel: a warp per (box, direction)
  const dim3 grid((unsigned)((K + 7) / 8), (unsigned)((ndir + fmmt::AGG_PD - 1) / fmmt::AGG_PD));
  const dim3 grid_any((unsigned)((K + 7) / 8), (unsigned)std::min<int64_t>(ndir, 65535));
  const dim3 grid_s((unsigned)K, (unsigned)((ndir + 31) / 32));   // shared-memory staged: a CTA per (box, 32 dirs)
  const bool staged = ctx->agg_staged;
  switch (ncomp) {
    case 1:
      if (staged) fmmt::k_aggregate_smem<1><<<grid_s, 256, 0, ctx->stream>>>(P, I, box_ptr, ndir, N, K, sig);
      else fmmt::k_aggregate<1><<<grid, 256, 0, ctx->stream>>>(P, I, box_ptr, ndir, N, K, sig);
      break;
    case 2:
      if (staged) fmmt::k_aggregate_smem<2><<<grid_s, 256, 0, ctx->stream>>>(P, I, box_ptr, ndir, N, K, sig);
      else fmmt::k_aggregate<2><<<grid, 256, 0, ctx->stream>>>(P, I, box_ptr, ndir, N, K, sig);
      break;
    case 4:
      if (staged) fmmt::k_aggregate_smem<4><<<grid_s, 256, 0, ctx->stream>>>(P, I, box_ptr, ndir, N, K, sig);
      else fmmt::k_aggregate<4><<<grid, 256, 0, ctx->stream>>>(P, I, box_ptr, ndir, N, K, sig);
      break;
    default: fmmt::k_aggregate_any<<<grid_any, 256, 0, ctx->stream>>>(P, I, box_ptr, ndir, N, ncomp, K, sig);
  }
  FMMT_CUDA(ctx, cudaGetLastError());
  return FMMT_OK;
}

// direction blocks of the disaggregation: up to 16 (non-empty boxes x blocks fill the SMs; the partial
// sums add 16 N complex writes + reads against the ndir N ncomp complex pattern reads)
static int agg_nsplit(const fmmt_ctx* ctx, int64_t ndir, int64_t) {
  if (ctx->agg_staged) return (int)((ndir + 31) / 32);                  // k_disaggregate_smem: 32 per block
  return (int)std::max<int64_t>(1, std::min<int64_t>(16, ndir / 16));   // >= 16 directions per block
}

// part: nsplit x N complex64 workspace
static fmmt_status disaggregate_impl(fmmt_ctx* ctx, const float2* P, const float2* B, const float* w,
                                     const int64_t* box_ptr, int64_t ndir, int64_t N, int ncomp, int64_t K, float2* y,
                                     float2* part) {
  if (N == 0) return FMMT_OK;
  const int nsplit = agg_nsplit(ctx, ndir, K);
  {
    ProfScope ps(ctx, "disaggregate_partial");
    const dim3 grid((unsigned)K, (unsigned)nsplit);
    if (ctx->agg_staged && (ncomp == 1 || ncomp == 2 || ncomp == 4)) {   // nsplit = ceil(ndir / 32)
      if (ncomp == 1) fmmt::k_disaggregate_smem<1><<<grid, 256, 0, ctx->stream>>>(P, B, w, box_ptr, ndir, N, K, part);
      else if (ncomp == 2) fmmt::k_disaggregate_smem<2><<<grid, 256, 0, ctx->stream>>>(P, B, w, box_ptr, ndir, N, K, part);
      else fmmt::k_disaggregate_smem<4><<<grid, 256, 0, ctx->stream>>>(P, B, w, box_ptr, ndir, N, K, part);
    } else switch (ncomp) {
      case 1: fmmt::k_disaggregate_partial<1><<<grid, 64, 0, ctx->stream>>>(P, B, w, box_ptr, ndir, N, K, nsplit, part); break;
      case 2: fmmt::k_disaggregate_partial<2><<<grid, 64, 0, ctx->stream>>>(P, B, w, box_ptr, ndir, N, K, nsplit, part); break;
      case 4: fmmt::k_disaggregate_partial<4><<<grid, 64, 0, ctx->stream>>>(P, B, w, box_ptr, ndir, N, K, nsplit, part); break;
      default:
        fmmt::k_disaggregate_partial_any<<<grid, 64, 0, ctx->stream>>>(P, B, w, box_ptr, ndir, N, ncomp, K, nsplit, part);
    }
    FMMT_CUDA(ctx, cudaGetLastError());
  }
  {
    ProfScope ps(ctx, "disaggregate_final");
    fmmt::k_disaggregate_final<<<(unsigned)((N + 255) / 256), 256, 0, ctx->stream>>>(part, N, nsplit, y);
    FMMT_CUDA(ctx, cudaGetLastError());
  }
  if (ctx->nccl_comm) {
    ncclResult_t r = ncclAllReduce(y, y, (size_t)(2 * N), ncclFloat, ncclSum, (ncclComm_t)ctx->nccl_comm, ctx->stream);
    if (r != ncclSuccess) return set_err(ctx, FMMT_E_NCCL, "ncclAllReduce: %s", ncclGetErrorString(r));
  }
  return FMMT_OK;
}

fmmt_status fmmt_aggregate(fmmt_ctx* ctx, const fmmt_c64* P, const fmmt_c64* I, const int64_t* box_ptr, int64_t ndir,
                           int64_t N, int64_t ncomp, int64_t Nx, int64_t Ny, int64_t Nz, fmmt_c64* sig) {
  if (!ctx) return FMMT_E_ARG;
  CHECK_ARG(ctx, sig && (I || N == 0), "null pointer");
  fmmt_status st = check_agg_args(ctx, P ? P : (const void*)box_ptr, box_ptr, ndir, N, ncomp, Nx, Ny, Nz);
  if (st) return st;
  if ((st = check_device_ptr(ctx, sig, "sig"))) return st;
  cudaSetDevice(ctx->device);
  return aggregate_impl(ctx, reinterpret_cast<const float2*>(P), reinterpret_cast<const float2*>(I), box_ptr, ndir, N,
                        (int)ncomp, Nx * Ny * Nz, reinterpret_cast<float2*>(sig));
}

fmmt_status fmmt_disaggregate(fmmt_ctx* ctx, const fmmt_c64* P, const fmmt_c64* B, const float* w, const int64_t* box_ptr,
                              int64_t ndir, int64_t N, int64_t ncomp, int64_t Nx, int64_t Ny, int64_t Nz, fmmt_c64* y) {
  if (!ctx) return FMMT_E_ARG;
  CHECK_ARG(ctx, B && w && (y || N == 0), "null pointer");
  fmmt_status st = check_agg_args(ctx, P ? P : (const void*)box_ptr, box_ptr, ndir, N, ncomp, Nx, Ny, Nz);
  if (st) return st;
  if ((st = check_device_ptr(ctx, B, "B"))) return st;
  cudaSetDevice(ctx->device);
  const int64_t need = (int64_t)agg_nsplit(ctx, ndir, Nx * Ny * Nz) * N;
  if (ctx->agg_part_elems < need) {
    if (ctx->agg_part) {
      cudaStreamSynchronize(ctx->stream);
      cudaFree(ctx->agg_part);
    }
    ctx->agg_part = nullptr;
    ctx->agg_part_elems = 0;
    cudaError_t e = cudaMalloc(&ctx->agg_part, need * sizeof(float2));
    if (e != cudaSuccess) return set_err(ctx, FMMT_E_NOMEM, "disaggregation workspace: %s", cudaGetErrorString(e));
    ctx->agg_part_elems = need;
  }
  return disaggregate_impl(ctx, reinterpret_cast<const float2*>(P), reinterpret_cast<const float2*>(B), w, box_ptr, ndir,
                           N, (int)ncomp, Nx * Ny * Nz, reinterpret_cast<float2*>(y),
                           reinterpret_cast<float2*>(ctx->agg_part));
}

fmmt_status fmmt_far_matvec(fmmt_op* op, const fmmt_c64* P, const fmmt_c64* I, const int64_t* box_ptr, const float* w,
                            int64_t ndir, int64_t N, int64_t ncomp, int64_t Nx, int64_t Ny, int64_t Nz, fmmt_c64* y) {
  if (!op) return FMMT_E_ARG;
  fmmt_ctx* ctx = op->ctx;
  CHECK_ARG(ctx, I && w && y, "null pointer");
  if (!op->translatable) return set_err(ctx, FMMT_E_UNSUPPORTED, "storage-only op");
  fmmt_status st = check_agg_args(ctx, P, box_ptr, ndir, N, ncomp, Nx, Ny, Nz);
  if (st) return st;
  CHECK_SHAPE(ctx, ndir == op->ndir, "ndir %lld != op ndir %lld", (long long)ndir, (long long)op->ndir);
  CHECK_SHAPE(ctx, 2 * Nx == op->n1 && 2 * Ny == op->n2 && 2 * Nz == op->n3, "grid does not match the op");
  cudaSetDevice(ctx->device);
  const int64_t K = Nx * Ny * Nz, elems = ndir * ncomp * K;
  const int64_t pelems = std::max<int64_t>(1, (int64_t)agg_nsplit(ctx, ndir, K) * N);
  if (op->fAB_elems < elems || op->fPart_elems < pelems) {   // workspaces change: drop captured graphs
    drop_graphs(op);
    for (float2** b : {&op->fA, &op->fB, &op->fPart}) dev_free(op, *b);
    op->fAB_elems = op->fPart_elems = 0;
    if ((st = cmalloc(op, &op->fA, elems)) || (st = cmalloc(op, &op->fB, elems)) || (st = cmalloc(op, &op->fPart, pelems)))
      return st;
    op->fAB_elems = elems;
    op->fPart_elems = pelems;
  }
  if ((st = ensure_w(op, ncomp))) return st;
  return run_graphed(op, P, I, y, w, N * 16 + ncomp, [&] {
    fmmt_status s2 = aggregate_impl(ctx, reinterpret_cast<const float2*>(P), reinterpret_cast<const float2*>(I), box_ptr,
                                    ndir, N, (int)ncomp, K, op->fA);
    if (s2) return s2;
    if ((s2 = translate_impl(op, reinterpret_cast<const fmmt_c64*>(op->fA), reinterpret_cast<fmmt_c64*>(op->fB),
                             (int)ncomp)))
      return s2;
    return disaggregate_impl(ctx, reinterpret_cast<const float2*>(P), op->fB, w, box_ptr, ndir, N, (int)ncomp, K,
                             reinterpret_cast<float2*>(y), op->fPart);
  }, box_ptr);
}

fmmt_status fmmt_restore(fmmt_op* op, int64_t p, fmmt_c64* T_p) {
  if (!op) return FMMT_E_ARG;
  fmmt_ctx* ctx = op->ctx;
  CHECK_ARG(ctx, T_p, "null output");
  if (!op->translatable) return set_err(ctx, FMMT_E_UNSUPPORTED, "storage-only op (shape outside the translate path)");
  CHECK_ARG(ctx, p >= 0 && p < op->ndir, "direction %lld out of range", (long long)p);
  cudaSetDevice(ctx->device);
  const int64_t n = op->n1 * op->n2 * op->n3;
  if (op->format == FMMT_DENSE) {
    ProfScope ps(ctx, "restore_copy");
    FMMT_CUDA(ctx, cudaMemcpyAsync(T_p, op->arr[0] + p * n, n * sizeof(float2), cudaMemcpyDeviceToDevice, ctx->stream));
    return FMMT_OK;
  }
  if (fmmt_status st = reset_dyn_slots(op)) return st;
  for (int bi = 0; bi < (int)op->batches.size(); ++bi) {
    const Batch& b = op->batches[bi];
    if (p < b.q0 || p >= b.q0 + b.nq) continue;
    fmmt_status st = run_batch_prep(op, b);
    if (!st) st = run_batch_zpack(op, bi);
    if (st) return st;
    return launch_z(op, fmmt::Z_RESTORE, (int)p, (int)(p - b.q0), 1, reinterpret_cast<float2*>(T_p));
  }
  return set_err(ctx, FMMT_E_STATE, "no batch holds direction %lld", (long long)p);
}

}  // extern "C"

// ============================================================== op creation
namespace fmmt_internal {

fmmt_status create_op(fmmt_ctx* ctx, fmmt_format format, int64_t n1, int64_t n2, int64_t n3, int64_t ndir,
                      const int64_t* ranks, const void* const* arrays, int64_t narrays, fmmt_op** out,
                      bool storage_only_ok) {
  if (!ctx || !out) return FMMT_E_ARG;
  *out = nullptr;
  CHECK_ARG(ctx, format >= FMMT_DENSE && format <= FMMT_TT4D, "bad format %d", (int)format);
  CHECK_ARG(ctx, arrays != nullptr, "null arrays");
  CHECK_SHAPE(ctx, n1 >= 2 && n2 >= 2 && n3 >= 2 && ndir >= 1, "bad dims");
  CHECK_SHAPE(ctx, n1 % 2 == 0 && n2 % 2 == 0 && n3 % 2 == 0, "n must be even (n = 2N)");
  bool translatable = is_pow2(n1) && is_pow2(n2) && is_pow2(n3) && n1 >= 4 && n2 >= 4 && n3 >= 4 && n1 <= 256 &&
                      n2 <= 256 && n3 <= 64;
  if (translatable) {   // the xy FFT kernel holds one padded plane (plus twiddles) in shared memory
    const XYKernels xk = get_xy((int)n1, (int)n2);
    translatable = xk.fwd && (xk.big_pp > 0 || (int64_t)(FMMT_TW_NMAX + xk.plane_smem) * 8 <= 227 * 1024);
  }
  if (!translatable && !storage_only_ok)
    return set_err(ctx, FMMT_E_UNSUPPORTED,
                   "translate path supports power-of-two n1,n2 in [4,256] (one xy plane <= 227 KB of shared memory), "
                   "n3 in [4,64]; got %lldx%lldx%lld",
                   (long long)n1, (long long)n2, (long long)n3);
  static const int nslots_of[] = {0, 3, 4, 6, 2, 3};
  static const int narr_of[] = {1, 4, 5, 7, 3, 4};
  CHECK_ARG(ctx, narrays == narr_of[format], "format %d needs %d arrays, got %lld", (int)format, narr_of[format], (long long)narrays);
  for (int i = 0; i < narr_of[format]; ++i) CHECK_ARG(ctx, arrays[i] != nullptr, "array %d is null", i);
  cudaSetDevice(ctx->device);
  fmmt_op* op = new fmmt_op();
  op->ctx = ctx;
  op->format = format;
  op->n1 = n1; op->n2 = n2; op->n3 = n3; op->ndir = ndir;
  op->nslots = nslots_of[format];
  op->translatable = translatable;
  const bool per_dir = format == FMMT_TUCKER3D || format == FMMT_TT3D;
  if (op->nslots) {
    CHECK_ARG(ctx, ranks != nullptr, "null ranks");
    const int64_t cnt = per_dir ? ndir * op->nslots : op->nslots;
    op->ranks.assign(ranks, ranks + cnt);
    for (auto r : op->ranks)
      if (r < 1) {
        delete op;
        return set_err(ctx, FMMT_E_SHAPE, "ranks must be >= 1");
      }
  }
  // element counts per array (and per-direction offsets for 3D formats)
  std::vector<int64_t> elems;
  op->off.clear();
  auto R = [&](int64_t p, int s) { return rk(op, p, s); };
  switch (format) {
    case FMMT_DENSE: elems = {n1 * n2 * n3 * ndir}; break;
    case FMMT_TUCKER3D: {
      op->off.assign(4, std::vector<int64_t>(ndir));
      elems.assign(4, 0);
      for (int64_t p = 0; p < ndir; ++p) {
        const int64_t r1 = R(p, 0), r2 = R(p, 1), r3 = R(p, 2);
        if (r1 > n1 || r2 > n2 || r3 > n3) { delete op; return set_err(ctx, FMMT_E_SHAPE, "rank exceeds mode size"); }
        const int64_t sz[4] = {r1 * r2 * r3, n1 * r1, n2 * r2, n3 * r3};
        for (int i = 0; i < 4; ++i) { op->off[i][p] = elems[i]; elems[i] += sz[i]; }
        op->r1max = std::max(op->r1max, r1);
        op->r2max = std::max(op->r2max, r2);
        op->r3max = std::max(op->r3max, r3);
      }
      op->rGmax = op->r3max;
      // fused mode-1 / mode-3 chain (kernels_tcfuse.cuh): tensor-core fp16 build, n3 = 64, whole 128-line i-blocks,
      // H'_j within the shared-memory region, G within 64 TMEM columns
      op->zfused = ctx->z_fuse && ctx->gemm_impl == 1 && fmmt::TC_F16 && n3 == 64 && n1 % 128 == 0 &&
                   op->r1max <= fmmt::ZfCfg::MAX_R1 && op->r3max <= 64;
      break;
    }
    case FMMT_TUCKER4D: {
      const int64_t r1 = R(0, 0), r2 = R(0, 1), r3 = R(0, 2), r4 = R(0, 3);
      elems = {r1 * r2 * r3 * r4, n1 * r1, n2 * r2, n3 * r3, ndir * r4};
      op->r2max = r2; op->r3max = r3; op->rGmax = r3;
      break;
    }
    case FMMT_HTUCKER4D: {
      const int64_t r1 = R(0, 0), r2 = R(0, 1), r3 = R(0, 2), r4 = R(0, 3), r12 = R(0, 4), r34 = R(0, 5);
      elems = {n1 * r1, n2 * r2, n3 * r3, ndir * r4, r1 * r2 * r12, r3 * r4 * r34, r12 * r34};
      op->r2max = r2; op->r3max = r3; op->rGmax = r3;
      break;
    }
    case FMMT_TT3D: {
      op->off.assign(3, std::vector<int64_t>(ndir));
      elems.assign(3, 0);
      for (int64_t p = 0; p < ndir; ++p) {
        const int64_t r1 = R(p, 0), r2 = R(p, 1);
        const int64_t sz[3] = {n1 * r1, r1 * n2 * r2, n3 * r2};
        for (int i = 0; i < 3; ++i) { op->off[i][p] = elems[i]; elems[i] += sz[i]; }
        op->rGmax = std::max(op->rGmax, r2);
      }
      break;
    }
    case FMMT_TT4D: {
      const int64_t r1 = R(0, 0), r2 = R(0, 1), r3 = R(0, 2);
      elems = {n1 * r1, r1 * n2 * r2, r2 * n3 * r3, ndir * r3};
      break;
    }
  }
  op->arr_elems = elems;
  for (size_t i = 0; i < elems.size(); ++i) {
    float2* d = nullptr;
    if (fmmt_status st = dev_alloc(op, &d, std::max<int64_t>(1, elems[i]) * 8, MEM_FACTOR, "factor")) {
      fmmt_op_destroy(op);
      return st;
    }
    op->arr.push_back(d);
    cudaError_t e = cudaMemcpy(d, arrays[i], elems[i] * sizeof(float2), cudaMemcpyDefault);
    if (e != cudaSuccess) {
      fmmt_op_destroy(op);
      return set_err(ctx, FMMT_E_CUDA, "factor copy failed: %s", cudaGetErrorString(e));
    }
  }
  if (per_dir) {
    // z-stage V factor offsets and ranks per direction
    std::vector<int64_t> voff(ndir);
    std::vector<int> rz(ndir);
    const int vi = (format == FMMT_TUCKER3D) ? 3 : 2;
    for (int64_t p = 0; p < ndir; ++p) {
      voff[p] = op->off[vi][p];
      rz[p] = (int)(format == FMMT_TUCKER3D ? R(p, 2) : R(p, 1));
    }
    fmmt_status st;
    if ((st = dev_alloc(op, &op->d_voff, ndir * 8, MEM_DERIVED, "z-stage offsets")) ||
        (st = dev_alloc(op, &op->d_rank, ndir * 4, MEM_DERIVED, "z-stage ranks"))) {
      fmmt_op_destroy(op);
      return st;
    }
    cudaError_t e1 = cudaMemcpy(op->d_voff, voff.data(), ndir * sizeof(int64_t), cudaMemcpyHostToDevice);
    cudaError_t e2 = cudaMemcpy(op->d_rank, rz.data(), ndir * sizeof(int), cudaMemcpyHostToDevice);
    if (e1 != cudaSuccess || e2 != cudaSuccess) {
      fmmt_op_destroy(op);
      return set_err(ctx, FMMT_E_CUDA, "z-stage table copy failed: %s", cudaGetErrorString(e1 != cudaSuccess ? e1 : e2));
    }
    if (op->zfused) {
      std::vector<int> r3t(ndir * 3);
      for (int64_t p = 0; p < ndir; ++p)
        for (int s3 = 0; s3 < 3; ++s3) r3t[p * 3 + s3] = (int)R(p, s3);
      if ((st = dev_alloc(op, &op->d_rank3, ndir * 12, MEM_DERIVED, "Tucker-3D ranks"))) {
        fmmt_op_destroy(op);
        return st;
      }
      cudaError_t e3 = cudaMemcpy(op->d_rank3, r3t.data(), ndir * 12, cudaMemcpyHostToDevice);
      if (e3 != cudaSuccess) {
        fmmt_op_destroy(op);
        return set_err(ctx, FMMT_E_CUDA, "rank table copy failed: %s", cudaGetErrorString(e3));
      }
    }
  }
  if (!translatable) {   // storage-only: factors, ranks, info and export (no plans, no derived operands)
    *out = op;
    return FMMT_OK;
  }
  {  // fp16-split scale slots of the factor arrays (fmmt_op::d_slots)
    fmmt_status st = dev_alloc(op, &op->d_slots, SLOT_DYN * 4, MEM_WORKSPACE, "scale slots");
    if (!st && cudaMemsetAsync(op->d_slots, 0, SLOT_DYN * 4, ctx->stream) != cudaSuccess)
      st = set_err(ctx, FMMT_E_CUDA, "scale slot reset failed");
    for (size_t i = 0; !st && i < elems.size(); ++i) st = absmax(op, op->arr[i], elems[i], op->d_slots + i);
    if (st) {
      fmmt_op_destroy(op);
      return st;
    }
  }
  if (format == FMMT_HTUCKER4D) {
    // Direction-independent part of Fig. 3(c), once per op, in FP64 (setup):
    //   E[i + n1 jj + n12 j] = sum_{a,b} U1[i,a] U2[jj,b] (C12 . C1234)[a + r1 b, j]
    const int64_t r1 = R(0, 0), r2 = R(0, 1), r12 = R(0, 4), r34 = R(0, 5), n12 = n1 * n2;
    if (fmmt_status ast = dev_alloc(op, &op->E, n12 * r34 * 8, MEM_DERIVED, "H-Tucker E")) {
      fmmt_op_destroy(op);
      return ast;
    }
    fmmt_status st = fmmt_internal::htucker_E_fp64(ctx, op->arr[0], op->arr[1], op->arr[4], op->arr[6], n1, n2, r1, r2,
                                                   r12, r34, op->E);
    if (!st) st = absmax(op, op->E, n12 * r34, op->d_slots + SLOT_E);
    if (st) {
      fmmt_op_destroy(op);
      return st;
    }
    GemmDesc de = gdx(op->E, nullptr, nullptr, n12, 1, r34, 1, 0, NODIV, n12, 0, 0, 0, 0, NODIV, 0);
    de.amax = sslot(op, SLOT_E);
    if ((st = pack_a(op, de, &op->E_pk))) {
      fmmt_op_destroy(op);
      return st;
    }
  }
  fmmt_status st = build_plans(op);
  if (st) {
    fmmt_op_destroy(op);
    return st;
  }
  if (format == FMMT_TT4D) {
    // T1 = U1 . C1 (Fig. 4(a) step 1, reused by every direction of Fig. 4(b)), stored [b][ij], in FP64
    const int64_t r1 = R(0, 0), r2 = R(0, 1);
    if (fmmt_status ast = dev_alloc(op, &op->tbar1, n1 * n2 * r2 * 8, MEM_DERIVED, "TT-4D T1")) {
      fmmt_op_destroy(op);
      return ast;
    }
    fmmt_status tst = fmmt_internal::tt4d_T1_fp64(ctx, op->arr[0], op->arr[1], n1, r1, n2, r2, op->tbar1);
    const int64_t n12 = n1 * n2;
    if (!tst) tst = absmax(op, op->tbar1, n12 * r2, op->d_slots + SLOT_T1);
    if (tst) {
      fmmt_op_destroy(op);
      return tst;
    }
    GemmDesc dt = gdx(op->tbar1, nullptr, nullptr, n12, 1, r2, 1, 0, NODIV, n12, 0, 0, 0, 0, NODIV, 0);
    dt.amax = sslot(op, SLOT_T1);
    fmmt_status pst = pack_a(op, dt, &op->tbar1_pk);
    if (pst) {
      fmmt_op_destroy(op);
      return pst;
    }
  }
  *out = op;
  return FMMT_OK;
}

}  // namespace fmmt_internal
