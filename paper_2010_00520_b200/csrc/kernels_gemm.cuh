// kernels_gemm.cuh -- batched complex64 GEMM (FP32 accumulation) for the
// restore chains that precede the fused z-stage:
//   Tucker (Fig. 3(a)):  H_p = U1 . C_p(1),   G_p[:,:,c] = H_p[:,:,c] . U2^T
//   Tucker-4D (Fig. 3(b)):      C_p = C(1234 -> 123 x 4) . U4[p,:]^T   (a3)
//   H-Tucker (Fig. 3(c)):       M_p, N_p = C1234 . M_p^T, C_p = C12 . N_p (a3)
//   TT-3D (Fig. 4(a)):   G_p = U1_p . C1_p
//   TT-4D (Fig. 4(b)):   T2 columns  V_p = C2 . U_last[p,:]^T      (a3)
// Every call is C = A . B with general (two-level) strides; a descriptor list
// gives one (possibly strided-batched) GEMM per entry so that directions
// with different ranks (3D formats) run in one launch.
#pragma once
#include "common.cuh"

namespace fmmt {

struct GemmDesc {
  const float2* A;
  const float2* B;
  float2* C;
  int m, n, k;
  int batch;           // strided sub-batch count
  // A(i,l) = A[(i % a_div) * a_s0 + (i / a_div) * a_s1 + l * a_sk]   (two-level row index)
  int64_t a_s0, a_s1, a_sk;
  int a_div;
  // B(l,j) = B[l * b_sk + j * b_sn]
  int64_t b_sk, b_sn;
  // C(i,j) = C[(i % c_div) * c_s0 + (i / c_div) * c_s1 + j * c_sn]
  int64_t c_s0, c_s1, c_sn;
  int c_div;
  int64_t sA, sB, sC;  // sub-batch strides (elements)
  // optional pre-split A for the tensor-core kernel (kernels_tcgemm.cuh, k_tc_pack_a):
  // tile (m/128, k-chunk) at Ap + (tile_m * a_nkc + chunk) * TC_PACK_FLOATS; nullptr = none
  const float* Ap;
  int a_nkc;
  int b_eo;            // tensor-core z-stage: B columns taken in (even, odd) order
  // optional pre-split B (k_tc_pack_b) of this tile's columns: chunk c at Bp + c * TcGemmCfg::BP_FLOATS
  // (set per tile by the kernel); nullptr = none
  const float* Bp;
  // tensor-core tile order: 0 = m-tiles fastest (B tile shared by consecutive CTAs), 1 = n-tiles fastest
  // (A tile shared; chosen when A is the larger operand, so it streams from DRAM once)
  int n_fast;
  // fp16-split operand scales (kernels_tcgemm.cuh): device max(|Re|, |Im|) of A and B (the power-of-two
  // scale is derived from it; packed operands were split with the same value), and the slot into which
  // the kernel folds max |C| for the consumer of C; nullptr = none / unit scale
  const float* amax;
  const float* bmax;
  float* cmax;
  // packed-operand strides per sub-batch (floats): A at Ap + sub * a_pk_sub, B' at Bp + sub * b_pk_sub
  // (b_pk_sub = 0: one B shared by every sub-batch)
  int64_t a_pk_sub;
  int64_t b_pk_sub;
};

__device__ __forceinline__ int64_t a_row(const GemmDesc& d, int i) {
  return (int64_t)(i % d.a_div) * d.a_s0 + (int64_t)(i / d.a_div) * d.a_s1;
}
__device__ __forceinline__ int64_t c_row(const GemmDesc& d, int i) {
  return (int64_t)(i % d.c_div) * d.c_s0 + (int64_t)(i / d.c_div) * d.c_s1;
}

template <int BM, int BN, int BK, int TM, int TN>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
k_cgemm(const GemmDesc* __restrict__ descs) {
  constexpr int NT = (BM / TM) * (BN / TN);
  const GemmDesc d = descs[blockIdx.z];
  const int sub = blockIdx.y;
  if (sub >= d.batch) return;
  const int tiles_m = (d.m + BM - 1) / BM;
  const int tiles_n = (d.n + BN - 1) / BN;
  const int tile = blockIdx.x;
  if (tile >= tiles_m * tiles_n) return;
  const int m0 = (tile % tiles_m) * BM;
  const int n0 = (tile / tiles_m) * BN;
  const float2* A = d.A + (int64_t)sub * d.sA;
  const float2* B = d.B + (int64_t)sub * d.sB;
  float2* C = d.C + (int64_t)sub * d.sC;

  __shared__ __align__(16) float2 As[BK][BM + 2];
  __shared__ __align__(16) float2 Bs[BK][BN + 2];

  const int tid = threadIdx.x;
  const int tx = tid % (BN / TN);
  const int ty = tid / (BN / TN);
  float2 acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = make_float2(0.f, 0.f);

  for (int k0 = 0; k0 < d.k; k0 += BK) {
    // A tile: (BM x BK), coalesced along m
    for (int e = tid; e < BM * BK; e += NT) {
      const int i = e % BM, kk = e / BM;
      const int gm = m0 + i, gk = k0 + kk;
      As[kk][i] = (gm < d.m && gk < d.k) ? A[a_row(d, gm) + gk * d.a_sk] : make_float2(0.f, 0.f);
    }
    if (d.b_sk != 1) {
      for (int e = tid; e < BN * BK; e += NT) {
        const int j = e % BN, kk = e / BN;
        const int gn = n0 + j, gk = k0 + kk;
        Bs[kk][j] = (gn < d.n && gk < d.k) ? B[gn * d.b_sn + gk * d.b_sk] : make_float2(0.f, 0.f);
      }
    } else {
      for (int e = tid; e < BN * BK; e += NT) {
        const int kk = e % BK, j = e / BK;
        const int gn = n0 + j, gk = k0 + kk;
        Bs[kk][j] = (gn < d.n && gk < d.k) ? B[gk + d.b_sn * gn] : make_float2(0.f, 0.f);
      }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float2 av[TM], bv[TN];
#pragma unroll
      for (int i = 0; i < TM; i += 2) {
        float4 v = *reinterpret_cast<const float4*>(&As[kk][ty * TM + i]);
        av[i] = make_float2(v.x, v.y);
        av[i + 1] = make_float2(v.z, v.w);
      }
#pragma unroll
      for (int j = 0; j < TN; j += 2) {
        float4 v = *reinterpret_cast<const float4*>(&Bs[kk][tx * TN + j]);
        bv[j] = make_float2(v.x, v.y);
        bv[j + 1] = make_float2(v.z, v.w);
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) cmac(acc[i][j], av[i], bv[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int gm = m0 + ty * TM + i;
    if (gm >= d.m) continue;
    const int64_t cr = c_row(d, gm);
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int gn = n0 + tx * TN + j;
      if (gn < d.n) C[cr + d.c_sn * gn] = acc[i][j];
    }
  }
}

}  // namespace fmmt
