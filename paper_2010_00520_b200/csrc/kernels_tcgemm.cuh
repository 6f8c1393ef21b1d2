// kernels_tcgemm.cuh -- complex64 contractions on the sm_100a tensor cores
// (tcgen05.mma kind::tf32, 3xTF32 split, FP32 accumulation) for the restore
// steps of Figs. 3-4:
//   Tucker-4D slice   C_p = C(123 x 4) . U4[p,:]^T             (a3, Fig. 3(b))
//   H-Tucker slices   M_p, G_p = E . M_p^T                       (a3/a4, Fig. 3(c))
//   TT-4D slice       V_p = C2(r2 n3 x r3) . U_last[p,:]^T       (a3, Fig. 4(b))
//   Tucker mode-1/2   H_p = C_p(1)^T . U1^T, G_p = H_p x2 U2     (a4, Fig. 3(a))
//   TT-3D head        G_p = U1_p . C1_p                         (a4, Fig. 4(a))
//   z-stage           T_p[ij,:] = G_p[ij,:] . V_p  fused with the z-DFT,
//                     Hadamard product and inverse z-DFT          (a4-a6, eq. (5))
//
// One CTA = 128*G threads computes one 128-row x BN-column output tile; the G
// thread groups share the rows (thread = row tid % 128) and split the columns
// (group tid / 128 owns columns [g BN/G, (g+1) BN/G)), so the per-chunk work
// (operand conversion, TMEM drain) is spread over 4G warps.  Per K-chunk
// (TC_BK complex), double-buffered:
//   * cp.async copies the raw complex64 A elements straight into the canonical
//     K-major UMMA layout (or, for pre-split static operands, one bulk async
//     copy brings A_hi and A_lo), and the B elements into a raw staging area;
//   * the threads round A in place to A_hi = rna_tf32(x), write A_lo =
//     rna_tf32(x - A_hi) next to it, and build B' = [B^_hi ; B^_lo] (the
//     complex-embedding rows, hi rows then lo rows).  (The tensor core reads the
//     top 19 bits of an FP32 operand, i.e. truncates: measured with hi = x, lo =
//     x - rna(x) is wrong at 1e-3 and lo = x - trunc(x) is right; the truncated
//     split is, however, twice as coarse and failed the 1e-6 restore bar.)
//   * thread 0 issues 2 MMAs per K=8 step: A_hi x B' (N = 4*BN, giving hi.hi and
//     hi.lo side by side in TMEM) and A_lo x B^_hi accumulated onto hi.lo.
// Accumulation accuracy: see tc_flush.
#pragma once
#include "kernels_fft.cuh"
#include "kernels_gemm.cuh"
#include "tc.cuh"

namespace fmmt {

// z-stage tile order.  Tile t of tiles_m x nq (m-tile, direction q).  With a per-direction A (3D formats)
// q-major order keeps each direction's operands together.  With a shared A (TT-4D T1) too large to stay
// in L2 (ZArgs::z_blocked, set by the host) the directions are taken in blocks of ZQB: within a block the
// m-tile is the slow index, so consecutive CTAs share one A tile through L2 and the block's pre-split V_q
// stay L2-resident while the m-tiles sweep (T1 streams from HBM once per block, not once per direction).
constexpr int ZQB = 16;
__device__ __forceinline__ void z_tile(int t, int tiles_m, int nq, bool shared_a, int& q, int& mt) {
  if (!shared_a) {
    q = t / tiles_m;
    mt = t % tiles_m;
    return;
  }
  const int qb = t / (tiles_m * ZQB);
  const int r = t - qb * tiles_m * ZQB;
  const int qbs = min(ZQB, nq - qb * ZQB);
  mt = r / qbs;
  q = qb * ZQB + r % qbs;
}

// Operand split (FMMT_TC_F16, build-time): 1 = fp16 hi + lo with a power-of-two operand scale
// (kind::f16, 16 real K per MMA, twice the tf32 rate and half the operand bytes), 0 = TF32 hi + lo
// (kind::tf32, 8 real K per MMA).  Both keep 11 + 11 significant bits per operand and FP32
// accumulation; the products hi.hi + hi.lo + lo.hi (3 MMAs per useful MAC).
#ifndef FMMT_TC_F16
#define FMMT_TC_F16 1
#endif
#ifndef FMMT_TC_FC16
#define FMMT_TC_FC16 4
#endif
constexpr bool TC_F16 = FMMT_TC_F16 != 0;
constexpr int TC_ESZ = TC_F16 ? 2 : 4;   // bytes per split operand element in shared memory
constexpr int TC_KSTEP = TC_F16 ? 16 : 8;   // real K per MMA instruction
constexpr int TC_BM = 128;      // rows per tile (UMMA M)
constexpr int TC_BK = 8;        // complex K per chunk (16 real: 1 f16 / 2 tf32 UMMA K-steps)
constexpr int TC_PACK_FLOATS = 2 * TC_BM * 2 * TC_BK * TC_ESZ / 4;   // one packed A chunk (hi + lo), in floats
// chunks per TMEM flush group = MMAs chained into one accumulator before it is drained to FP32
// registers: tf32 4 K-steps (8 failed the 1e-6 restore bar), f16 FMMT_TC_FC16 K-steps
constexpr int TC_FC = TC_F16 ? FMMT_TC_FC16 : 2;

// Operand layout of one 128-row x BN-complex-column tile (the pack kernels' output, the shared-memory
// stage of kernels_tcpk.cuh): per 8-complex K-chunk A_hi, A_lo (128 rows x 16 real, K-major canonical
// UMMA layout: 8-row x 16-byte core matrices, SBO 128 B, K-adjacent core matrices LBO apart) and
// B' = [B^_hi ; B^_lo] (2 NR rows).
template <int BN, int G = 1>
struct TcGemmCfg {
  static constexpr int NR = 2 * BN;                 // real N of C (re, im interleaved)
  static constexpr int KR = 2 * TC_BK;              // real K per chunk
  static constexpr int A_BYTES = TC_BM * KR * TC_ESZ;   // one of hi / lo
  static constexpr int BP_ROWS = 2 * NR;            // B' = [B^_hi ; B^_lo]
  static constexpr int BP_BYTES = BP_ROWS * KR * TC_ESZ;
  static constexpr int BP_FLOATS = BP_BYTES / 4;      // one pre-split B' chunk (k_tc_pack_b), in floats
  static constexpr uint32_t LBO_A = TC_BM * 16;     // K-adjacent core matrices
  static constexpr uint32_t LBO_B = BP_ROWS * 16;
  static_assert(2 * NR <= 256, "UMMA N <= 256");
  static_assert(NR % 16 == 0, "TMEM drain granularity: 16 columns");
  static_assert(TC_BK == 8, "pack mappings assume 4 complex pairs per row and chunk");
};

// Accuracy of the tensor-core accumulation.  The tensor core adds each MMA's
// products into the FP32 accumulator with truncation, so the error of one
// accumulator grows with the number of MMAs chained into it (measured 2.4e-6
// relative at K = 169 with a single chain, ~3.8e-8 per chained MMA; the
// restore bound is 1e-6).  Each K-chunk (4 K-steps) therefore accumulates into
// a fresh TMEM slot, with the hi.hi products and the 2^-11-smaller cross terms
// in separate accumulators, and the chunk results are summed in FP32 registers
// (round-to-nearest).  Two slots alternate so chunk k+1's MMAs overlap the
// drain of chunk k.  A thread drains its row's columns [c0, c0 + NRG).
template <int NR, int NRG>
__device__ __forceinline__ void tc_flush(uint32_t tslot_addr, int c0, float (&acc)[NRG]) {
#pragma unroll
  for (int c = 0; c < NRG; c += 16) {
    float vm[16], vx[16];
    tc::tmem_ld16(tslot_addr + c0 + c, vm);
    tc::tmem_ld16(tslot_addr + NR + c0 + c, vx);
#pragma unroll
    for (int j = 0; j < 16; j += 2) {   // acc += (hi.hi + cross), two columns per FADD2
      const float2 t = cadd(make_float2(acc[c + j], acc[c + j + 1]),
                            cadd(make_float2(vm[j], vm[j + 1]), make_float2(vx[j], vx[j + 1])));
      acc[c + j] = t.x;
      acc[c + j + 1] = t.y;
    }
  }
}

// ---------------------------------------------------------------- k_tc_pack_a
// Pre-split a (static) A operand into the tensor-core kernel's operand layout:
// per (128-row tile, 8-complex K-chunk) one contiguous block of TC_PACK_FLOATS
// floats = A_hi then A_lo (round-to-nearest split; fp16 after the power-of-two
// scale of *d.amax, or TF32), each in the canonical K-major UMMA layout, zero-padded
// outside m x k.  The GEMM then streams A with one bulk async copy per chunk and no
// per-element work.  One thread per (row, complex pair).
__global__ void k_tc_pack_a(GemmDesc d, float* __restrict__ out) {
  const int nkc = (d.k + TC_BK - 1) / TC_BK;
  const int64_t tiles_m = (d.m + TC_BM - 1) / TC_BM;
  const int64_t total = tiles_m * TC_BM * nkc * (TC_BK / 2);
  const float s = (TC_F16 && d.amax) ? tc::f16_scale(*d.amax) : 1.f;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e % TC_BM);                       // row in tile (fastest: coalesced writes)
    int64_t t = e / TC_BM;
    const int kp = (int)(t % (TC_BK / 2));
    t /= (TC_BK / 2);
    const int kc = (int)(t % nkc);
    const int64_t tm = t / nkc;
    const int gm = (int)(tm * TC_BM + r);
    const int gk = kc * TC_BK + 2 * kp;
    float2 a0 = make_float2(0.f, 0.f), a1 = make_float2(0.f, 0.f);
    if (gm < d.m) {
      const int64_t row = a_row(d, gm);
      if (gk < d.k) a0 = d.A[row + (int64_t)gk * d.a_sk];
      if (gk + 1 < d.k) a1 = d.A[row + (int64_t)(gk + 1) * d.a_sk];
    }
    uint8_t* tile = reinterpret_cast<uint8_t*>(out + (tm * nkc + kc) * TC_PACK_FLOATS);
    if constexpr (TC_F16) {
      uint2 hi, lo;
      tc::split_f16x2(a0.x * s, a0.y * s, hi.x, lo.x);
      tc::split_f16x2(a1.x * s, a1.y * s, hi.y, lo.y);
      const int off = r * 16 + (kp >> 1) * (TC_BM * 16) + (kp & 1) * 8;   // bytes (fp16 core matrices)
      *reinterpret_cast<uint2*>(tile + off) = hi;
      *reinterpret_cast<uint2*>(tile + TC_PACK_FLOATS * 2 + off) = lo;
    } else {
      float4 hi, lo;
      tc::split_tf32(a0.x, hi.x, lo.x);
      tc::split_tf32(a0.y, hi.y, lo.y);
      tc::split_tf32(a1.x, hi.z, lo.z);
      tc::split_tf32(a1.y, hi.w, lo.w);
      const int off = r * 16 + kp * (TC_BM * 16);           // bytes: row r -> 16 B, K core matrix -> TC_BM*16 B
      *reinterpret_cast<float4*>(tile + off) = hi;
      *reinterpret_cast<float4*>(tile + TC_PACK_FLOATS * 2 + off) = lo;
    }
  }
}

// ---------------------------------------------------------------- k_tc_pack_b
// Pre-split B operands (one per batch-local q, columns [0, n)) into the B' chunks the tensor-core
// mainloop would build in shared memory: per (q, n-tile, 8-complex K-chunk) one contiguous block of
// BP_FLOATS = [B^_hi ; B^_lo] rows in the canonical K-major UMMA layout (rows 2j = [Re b, -Im b],
// 2j+1 = [Im b, Re b], round-to-nearest split, fp16 after the scale of *bmax or TF32), zero outside
// k x n.  The GEMM then streams B with one bulk async copy per chunk.  B(l, j) of batch q at
// B + q * b_stride + l * b_sk + j * b_sn.
template <int BN>
__global__ void k_tc_pack_b(const float2* __restrict__ B, int64_t b_stride, int64_t b_sk, int64_t b_sn, int k, int n,
                            int nq, float* __restrict__ out, const float* __restrict__ bmax) {
  using Cfg = TcGemmCfg<BN, 1>;
  constexpr int NR = Cfg::NR;
  const int nkc = (k + TC_BK - 1) / TC_BK;
  const int tiles_n = (n + BN - 1) / BN;
  const int64_t total = (int64_t)nq * tiles_n * nkc * BN * (TC_BK / 2);
  const float s = (TC_F16 && bmax) ? tc::f16_scale(*bmax) : 1.f;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(e % BN);                 // column in tile (fastest)
    int64_t t = e / BN;
    const int kp = (int)(t % (TC_BK / 2));
    t /= (TC_BK / 2);
    const int kc = (int)(t % nkc);
    t /= nkc;
    const int tn = (int)(t % tiles_n);
    const int64_t q = t / tiles_n;
    const int gn = tn * BN + j, gk = kc * TC_BK + 2 * kp;
    float2 b0 = make_float2(0.f, 0.f), b1 = make_float2(0.f, 0.f);
    if (gn < n) {
      const float2* Bq = B + q * b_stride + (int64_t)gn * b_sn;
      if (gk < k) b0 = Bq[(int64_t)gk * b_sk];
      if (gk + 1 < k) b1 = Bq[(int64_t)(gk + 1) * b_sk];
    }
    uint8_t* blk = reinterpret_cast<uint8_t*>(out + ((q * tiles_n + tn) * nkc + kc) * Cfg::BP_FLOATS);
    if constexpr (TC_F16) {
      uint2 h0, l0, h1, l1;
      tc::split_f16x2(b0.x * s, -b0.y * s, h0.x, l0.x);
      tc::split_f16x2(b1.x * s, -b1.y * s, h0.y, l0.y);
      tc::split_f16x2(b0.y * s, b0.x * s, h1.x, l1.x);
      tc::split_f16x2(b1.y * s, b1.x * s, h1.y, l1.y);
      const int off = (2 * j) * 16 + (kp >> 1) * Cfg::LBO_B + (kp & 1) * 8;   // bytes
      *reinterpret_cast<uint2*>(blk + off) = h0;
      *reinterpret_cast<uint2*>(blk + off + 16) = h1;
      *reinterpret_cast<uint2*>(blk + off + NR * 16) = l0;
      *reinterpret_cast<uint2*>(blk + off + NR * 16 + 16) = l1;
    } else {
      float4 h0, l0, h1, l1;
      tc::split_tf32(b0.x, h0.x, l0.x); tc::split_tf32(-b0.y, h0.y, l0.y);
      tc::split_tf32(b1.x, h0.z, l0.z); tc::split_tf32(-b1.y, h0.w, l0.w);
      tc::split_tf32(b0.y, h1.x, l1.x); tc::split_tf32(b0.x, h1.y, l1.y);
      tc::split_tf32(b1.y, h1.z, l1.z); tc::split_tf32(b1.x, h1.w, l1.w);
      const int off = (2 * j) * 16 + kp * Cfg::LBO_B;   // bytes (the shared-memory B' layout)
      *reinterpret_cast<float4*>(blk + off) = h0;
      *reinterpret_cast<float4*>(blk + off + 16) = h1;
      *reinterpret_cast<float4*>(blk + off + NR * 16) = l0;
      *reinterpret_cast<float4*>(blk + off + NR * 16 + 16) = l1;
    }
  }
}

// ---------------------------------------------------------------- k_absmax
// max(|Re x|, |Im x|) over a flat complex64 array, folded into *slot (the fp16 split's operand scale).
__global__ void k_absmax(const float2* __restrict__ x, int64_t n, float* __restrict__ slot) {
  float m = 0.f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float2 v = x[i];
    m = fmaxf(m, fmaxf(fabsf(v.x), fabsf(v.y)));
  }
  tc::warp_absmax_to(m, slot);
}

}  // namespace fmmt
