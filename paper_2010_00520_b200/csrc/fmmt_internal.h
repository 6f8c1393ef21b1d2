// fmmt_internal.h -- library-private structures shared by the translation
// units of libfmmt (fmmt_api.cu: hot path + op management; fmmt_setup.cu:
// direction grid, FP64 operator builder, FP64 compressor).
#pragma once
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/fmmt.h"

struct fmmt_prof_entry {
  const char* name;
  cudaEvent_t e0, e1;
};

struct fmmt_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int rank = 0, world = 1;
  void* nccl_comm = nullptr;        // ncclComm_t when world > 1
  std::string err;
  int64_t launches = 0;
  bool profiling = false;
  int num_sms = 148;                // SM count of the device (persistent grids)
  int gemm_impl = 1;                // restore GEMMs: 1 = tcgen05 3xTF32 (default), 0 = FP32 FFMA, 2 = first tcgen05 design
  bool use_graphs = true;           // replay whole matvecs as CUDA graphs (see run_graphed)
  int tc_ctas_per_sm = 2;           // tensor-core GEMM grid: CTAs per SM = the resident count (each loops over tiles)
  int batch_mb = 2048;              // per-batch intermediate budget of the 3D formats (FMMT_BATCH_MB)
  int z_fc = 8;                     // shared-A n3 = 64 z-stage flush group in K-chunks (2 TC_FC; FMMT_ZFC=4: TC_FC)
  bool z_fuse = true;               // Tucker-3D at n3 = 64, n1 % 128 == 0: fused mode-1 / mode-3 z-stage (FMMT_ZFUSE)
  bool z_cluster = true;            // shared-A n3 = 64 z-stage in 2-CTA clusters with multicast A (FMMT_ZCLUSTER)
  int w_mb = 128;                   // half-padded spectra per xy sub-batch (FMMT_W_MB; 16-128 measured within 4 %)
  int tc_ctas_z = 4;                // tensor-core z-stage grid: CTAs per SM (two waves measured faster there)
  bool agg_staged = true;           // aggregation: shared-memory staged kernel (FMMT_AGG_STAGED=0: warp-per-box)
  void* agg_part = nullptr;         // disaggregation partial sums [nsplit][N] (complex64)
  int64_t agg_part_elems = 0;
  std::vector<fmmt_prof_entry> pending;
  std::vector<std::pair<const char*, std::pair<double, int64_t>>> prof;   // name -> (ms, launches)
  std::vector<cudaEvent_t> event_pool;
  std::vector<void*> prof_execs;    // cudaGraphExec_t of profiled matvecs (destroyed at flush)
  bool h2d_overlap = true;          // fmmt_translate_sum_host: chunked upload on copy_stream, overlapped with the matvec (FMMT_H2D_OVERLAP=0: serial)
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t h2d_fence = nullptr;
  std::vector<cudaEvent_t> h2d_events;   // one per uploaded chunk of directions
  void* blas = nullptr;             // cublasHandle_t (setup only)
  void* solver = nullptr;           // cusolverDnHandle_t (setup only)
};

namespace fmmt_internal {

fmmt_status set_err(fmmt_ctx* ctx, fmmt_status st, const char* fmt, ...);

// Create an op from complex64 arrays (host or device memory, copied).  storage_only_ok: shapes
// outside the translate path give a storage-only op (ranks / info / export; translate and restore
// return FMMT_E_UNSUPPORTED) instead of an error (the compressor's paper-sweep sizes).
fmmt_status create_op(fmmt_ctx* ctx, fmmt_format format, int64_t n1, int64_t n2, int64_t n3,
                      int64_t ndir, const int64_t* ranks, const void* const* arrays,
                      int64_t narrays, fmmt_op** out, bool storage_only_ok);

void setup_release(fmmt_ctx* ctx);   // free cuBLAS / cuSOLVER handles

// FP64 (cuBLAS ZGEMM) direction-independent restore operands, rounded once to complex64.
fmmt_status htucker_E_fp64(fmmt_ctx* ctx, const float2* U1, const float2* U2, const float2* C12, const float2* C1234,
                           int64_t n1, int64_t n2, int64_t r1, int64_t r2, int64_t r12, int64_t r34, float2* E);
fmmt_status tt4d_T1_fp64(fmmt_ctx* ctx, const float2* U1, const float2* C1, int64_t n1, int64_t r1, int64_t n2,
                         int64_t r2, float2* T1);

}  // namespace fmmt_internal

#define FMMT_CUDA(ctx, call)                                                                \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return fmmt_internal::set_err((ctx), FMMT_E_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, \
                                    #call, cudaGetErrorString(e_));                        \
  } while (0)
