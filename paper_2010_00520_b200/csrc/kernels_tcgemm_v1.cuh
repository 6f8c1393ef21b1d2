// kernels_tcgemm_v1.cuh -- first tcgen05 design (non-persistent, 128 threads, register-staged
// operands, 2 CTAs/SM), kept for A/B measurement against kernels_tcgemm.cuh (impl 2).
// kernels_tcgemm.cuh -- batched complex64 GEMM on the sm_100a tensor cores
// (tcgen05.mma kind::tf32, 3xTF32 split, FP32 accumulation in TMEM) for the
// restore contractions of Figs. 3-4 that are dense GEMMs:
//   Tucker-4D slice   C_p = C(123 x 4) . U4[p,:]^T          (a3, Fig. 3(b))
//   H-Tucker slices   M_p, N_p, C_p                           (a3, Fig. 3(c))
//   TT-4D slice       V_p = C2(r2 n3 x r3) . U_last[p,:]^T    (a3, Fig. 4(b))
//   Tucker mode-1/2   H_p = U1 . C_p(1),  G_p = H_p x2 U2    (a4, Fig. 3(a))
//   TT-3D head        G_p = U1_p . C1_p                      (a4, Fig. 4(a))
// Same descriptor list as k_cgemm (kernels_gemm.cuh): C = A . B, general strides.
//
// One CTA = 128 threads = one 128-row x BN-column output tile.  All threads
// stage operands (global -> registers -> hi/lo split -> K-major smem, double
// buffered); thread 0 issues 3 MMAs per K=8 step and commits to the stage's
// mbarrier; the epilogue reads the accumulator with tcgen05.ld (thread = row).
#pragma once
#include "kernels_gemm.cuh"
#include "tc.cuh"

namespace fmmt {
namespace v1 {

constexpr int TC_BM = 128;   // rows per tile (UMMA M)
constexpr int TC_BK = 16;    // complex K per stage (32 real = 4 UMMA K-steps)

template <int BN>
struct TcGemmCfg {
  static constexpr int NR = 2 * BN;                 // real N of the UMMA
  static constexpr int KR = 2 * TC_BK;              // real K per stage
  static constexpr int A_BYTES = TC_BM * KR * 4;    // one of hi / lo
  static constexpr int B_BYTES = NR * KR * 4;
  static constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int SMEM = 2 * STAGE;
  // two accumulator slots (alternating K-chunks) x {main hi.hi, cross hi.lo + lo.hi}
  static constexpr int TMEM_COLS = 4 * NR < 32 ? 32 : 4 * NR;
  static constexpr uint32_t LBO_A = TC_BM * 16;     // K-adjacent core matrices
  static constexpr uint32_t LBO_B = NR * 16;
};

// SPLIT 0: hi = rna(x), lo = rna(x - hi).  Experiments (impl 3 / 4): hi = x as stored
// (the tensor core reads the TF32 part), lo = x - trunc13(x) (3) or x - rna(x) (4).
template <int SPLIT = 0>
__device__ __forceinline__ float split1(float x, float& lo) {
  if constexpr (SPLIT == 0) {
    float hi;
    tc::split_tf32(x, hi, lo);
    return hi;
  } else if constexpr (SPLIT == 1) {
    const float t = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
    lo = x - t;
    return x;
  } else {
    uint32_t h;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
    lo = x - __uint_as_float(h);
    return x;
  }
}
template <int SPLIT = 0>
__device__ __forceinline__ float4 split4_hi_lo(float a, float b, float c, float d, float4& lo) {
  float4 hi;
  hi.x = split1<SPLIT>(a, lo.x);
  hi.y = split1<SPLIT>(b, lo.y);
  hi.z = split1<SPLIT>(c, lo.z);
  hi.w = split1<SPLIT>(d, lo.w);
  return hi;
}

// Accuracy of the tensor-core accumulation.  The tensor core adds each MMA's
// products into the FP32 accumulator with truncation, so the error of one
// accumulator grows with the number of MMAs chained into it (measured 2.4e-6
// relative at K = 169 with a single chain; the restore bound is 1e-6).  Each
// K-chunk (TC_BK complex = 4 K-steps) therefore accumulates into a fresh TMEM
// slot, with the hi.hi products (4 MMAs) and the two 2^-11-smaller cross terms
// (8 MMAs) in separate accumulators, and the chunk results are summed by the
// threads in FP32 registers (round-to-nearest).  Two slots alternate so chunk
// k+1's MMAs overlap the flush of chunk k.
//
// Per thread (= row m0 + tid): acc[2*BN] floats, (re, im) interleaved.
template <int BN>
__device__ __forceinline__ void tc_flush(uint32_t tslot_addr, float (&acc)[2 * BN]) {
  constexpr int NR = 2 * BN;
#pragma unroll
  for (int c0 = 0; c0 < NR; c0 += 16) {
    float vm[16], vx[16];
    tc::tmem_ld16(tslot_addr + c0, vm);
    tc::tmem_ld16(tslot_addr + NR + c0, vx);
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[c0 + j] += vm[j] + vx[j];
  }
}

// acc[2BN] (registers, thread = row m0 + tid) = A[m0:m0+128, :] . B[:, n0:n0+BN]
// over all of K.  Called by all 128 threads.
template <int BN, int SPLIT = 0>
__device__ __forceinline__ void tc_mainloop(const GemmDesc& d, const float2* __restrict__ A,
                                            const float2* __restrict__ B, int m0, int n0, uint8_t* tcsm,
                                            uint64_t* bar, uint32_t tmem, float (&acc)[2 * BN]) {
  using Cfg = TcGemmCfg<BN>;
  constexpr int BM = TC_BM, BK = TC_BK, NR = Cfg::NR;
  const uint32_t sbase = tc::smem_u32(tcsm);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool a_kcontig = d.a_sk == 1;   // rows of A are contiguous in K
  const bool b_kcontig = d.b_sk == 1;
  // rows this thread loads: row-per-thread (row tid) or K-contiguous (4 rows)
  int64_t arow[4];
  bool okrow[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int r = a_kcontig ? (lane & 7) + 8 * (u + 4 * warp) : tid;
    okrow[u] = m0 + r < d.m;
    arow[u] = okrow[u] ? a_row(d, m0 + r) : 0;
  }
  constexpr uint32_t IDESC = tc::idesc_tf32(BM, NR);
#pragma unroll
  for (int j = 0; j < NR; ++j) acc[j] = 0.f;
  const uint32_t twarp = tmem + ((uint32_t)(warp * 32) << 16);   // this warp's TMEM lanes

  const int nk = (d.k + BK - 1) / BK;
  for (int kc = 0; kc < nk; ++kc) {
    const int s = kc & 1;
    const int k0 = kc * BK;
    // ---- global -> registers (zero outside the problem)
    float2 ra[2 * (BK / 2)];         // A: 8 pairs (row-per-thread) or 8 items of a pair
    if (!a_kcontig) {
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        const int gk = k0 + kk;
        ra[kk] = (okrow[0] && gk < d.k) ? A[arow[0] + gk * d.a_sk] : make_float2(0.f, 0.f);
      }
    } else {
#pragma unroll
      for (int i = 0; i < BK / 2; ++i) {
        const int kp = (lane >> 3) + 4 * (i & 1);
        const int gk = k0 + 2 * kp;
        const bool okm = okrow[i >> 1];
        ra[2 * i] = (okm && gk < d.k) ? A[arow[i >> 1] + gk] : make_float2(0.f, 0.f);
        ra[2 * i + 1] = (okm && gk + 1 < d.k) ? A[arow[i >> 1] + gk + 1] : make_float2(0.f, 0.f);
      }
    }
    constexpr int BITEMS = BN * (BK / 2) / 128 > 0 ? BN * (BK / 2) / 128 : 1;
    float2 rb[2 * BITEMS];
#pragma unroll
    for (int i = 0; i < BITEMS; ++i) {
      const int idx = tid + 128 * i;
      int j, kp;
      if (!b_kcontig) { j = idx % BN; kp = idx / BN; }    // n (not k) contiguous in memory
      else { kp = idx % (BK / 2); j = idx / (BK / 2); }   // k contiguous
      const bool ok = idx < BN * (BK / 2);
      const int gn = n0 + j, gk = k0 + 2 * kp;
      const bool okn = ok && gn < d.n;
      rb[2 * i] = (okn && gk < d.k) ? B[gk * d.b_sk + gn * d.b_sn] : make_float2(0.f, 0.f);
      rb[2 * i + 1] = (okn && gk + 1 < d.k) ? B[(gk + 1) * d.b_sk + gn * d.b_sn] : make_float2(0.f, 0.f);
    }
    // ---- wait until the MMAs that last read this stage are done
    if (kc >= 2) {
      tc::mbar_wait(&bar[s], ((kc >> 1) - 1) & 1);
      tc::fence_after_sync();
      v1::tc_flush<BN>(twarp + s * 2 * NR, acc);    // chunk kc-2 -> registers; slot s is free again
    }
    uint8_t* st = tcsm + s * Cfg::STAGE;
    uint8_t* aHi = st;
    uint8_t* aLo = st + Cfg::A_BYTES;
    uint8_t* bHi = st + 2 * Cfg::A_BYTES;
    uint8_t* bLo = bHi + Cfg::B_BYTES;
    // ---- registers -> smem (hi / lo), 16-byte rows of the core matrices
    if (!a_kcontig) {
#pragma unroll
      for (int kp = 0; kp < BK / 2; ++kp) {
        float4 lo;
        const float4 hi = split4_hi_lo<SPLIT>(ra[2 * kp].x, ra[2 * kp].y, ra[2 * kp + 1].x, ra[2 * kp + 1].y, lo);
        const uint32_t off = tid * 16 + kp * Cfg::LBO_A;
        *reinterpret_cast<float4*>(aHi + off) = hi;
        *reinterpret_cast<float4*>(aLo + off) = lo;
      }
    } else {
#pragma unroll
      for (int i = 0; i < BK / 2; ++i) {
        const int kp = (lane >> 3) + 4 * (i & 1);
        const int r = (lane & 7) + 8 * ((i >> 1) + 4 * warp);
        float4 lo;
        const float4 hi = split4_hi_lo<SPLIT>(ra[2 * i].x, ra[2 * i].y, ra[2 * i + 1].x, ra[2 * i + 1].y, lo);
        const uint32_t off = r * 16 + kp * Cfg::LBO_A;
        *reinterpret_cast<float4*>(aHi + off) = hi;
        *reinterpret_cast<float4*>(aLo + off) = lo;
      }
    }
#pragma unroll
    for (int i = 0; i < BITEMS; ++i) {
      const int idx = tid + 128 * i;
      if (idx >= BN * (BK / 2)) continue;
      int j, kp;
      if (!b_kcontig) { j = idx % BN; kp = idx / BN; }
      else { kp = idx % (BK / 2); j = idx / (BK / 2); }
      const float2 b0 = rb[2 * i], b1 = rb[2 * i + 1];
      float4 lo;
      // row 2j: [Re b, -Im b] ; row 2j+1: [Im b, Re b]
      float4 hi = split4_hi_lo<SPLIT>(b0.x, -b0.y, b1.x, -b1.y, lo);
      uint32_t off = (2 * j) * 16 + kp * Cfg::LBO_B;
      *reinterpret_cast<float4*>(bHi + off) = hi;
      *reinterpret_cast<float4*>(bLo + off) = lo;
      hi = split4_hi_lo<SPLIT>(b0.y, b0.x, b1.y, b1.x, lo);
      off += 16;
      *reinterpret_cast<float4*>(bHi + off) = hi;
      *reinterpret_cast<float4*>(bLo + off) = lo;
    }
    tc::fence_async_smem();
    tc::fence_before_sync();
    __syncthreads();
    if (tid == 0) {
      tc::fence_after_sync();
      const uint32_t sa_hi = sbase + s * Cfg::STAGE, sa_lo = sa_hi + Cfg::A_BYTES;
      const uint32_t sb_hi = sa_hi + 2 * Cfg::A_BYTES, sb_lo = sb_hi + Cfg::B_BYTES;
#pragma unroll
      for (int ks = 0; ks < Cfg::KR / 8; ++ks) {
        const uint64_t ah = tc::sdesc(sa_hi + ks * 2 * Cfg::LBO_A, Cfg::LBO_A, 128);
        const uint64_t al = tc::sdesc(sa_lo + ks * 2 * Cfg::LBO_A, Cfg::LBO_A, 128);
        const uint64_t bh = tc::sdesc(sb_hi + ks * 2 * Cfg::LBO_B, Cfg::LBO_B, 128);
        const uint64_t bl = tc::sdesc(sb_lo + ks * 2 * Cfg::LBO_B, Cfg::LBO_B, 128);
        const uint32_t tm = tmem + s * 2 * NR, tx = tm + NR;
        tc::mma_tf32(tx, al, bh, IDESC, ks != 0);
        tc::mma_tf32(tx, ah, bl, IDESC, 1);
        tc::mma_tf32(tm, ah, bh, IDESC, ks != 0);
      }
      tc::mma_commit(&bar[s]);
    }
  }
  // drain the (up to) two chunks still in TMEM
  for (int kc = (nk >= 2 ? nk - 2 : 0); kc < nk; ++kc) {
    tc::mbar_wait(&bar[kc & 1], (kc >> 1) & 1);
    tc::fence_after_sync();
    v1::tc_flush<BN>(twarp + (kc & 1) * 2 * NR, acc);
  }
}

// TMEM allocation + stage barriers (all threads call; warp 0 allocates).
template <int TMEM_COLS>
__device__ __forceinline__ uint32_t tc_setup(uint64_t* bar, uint32_t* tslot) {
  if ((threadIdx.x >> 5) == 0) tc::tmem_alloc<TMEM_COLS>(tslot);
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar[0], 1);
    tc::mbar_init(&bar[1], 1);
    tc::fence_barrier_init();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  return *tslot;
}

template <int TMEM_COLS>
__device__ __forceinline__ void tc_teardown(uint32_t tmem) {
  tc::fence_before_sync();
  __syncthreads();
  if ((threadIdx.x >> 5) == 0) tc::tmem_dealloc<TMEM_COLS>(tmem);
}

template <int BN, int SPLIT = 0>
__global__ void __launch_bounds__(128, 1) k_tc_cgemm(const GemmDesc* __restrict__ descs) {
  using Cfg = TcGemmCfg<BN>;
  constexpr int BM = TC_BM, NR = Cfg::NR;
  extern __shared__ __align__(1024) uint8_t tcsm[];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ uint32_t tslot;

  const GemmDesc d = descs[blockIdx.z];
  const int sub = blockIdx.y;
  if (sub >= d.batch) return;
  const int tiles_m = (d.m + BM - 1) / BM;
  const int tiles_n = (d.n + BN - 1) / BN;
  const int tile = blockIdx.x;
  if (tile >= tiles_m * tiles_n) return;
  const int m0 = (tile % tiles_m) * BM;
  const int n0 = (tile / tiles_m) * BN;
  const float2* __restrict__ A = d.A + (int64_t)sub * d.sA;
  const float2* __restrict__ B = d.B + (int64_t)sub * d.sB;
  float2* __restrict__ C = d.C + (int64_t)sub * d.sC;

  const uint32_t tmem = v1::tc_setup<Cfg::TMEM_COLS>(bar, &tslot);
  float acc[NR];
  v1::tc_mainloop<BN, SPLIT>(d, A, B, m0, n0, tcsm, bar, tmem, acc);

  // ---- epilogue: registers -> C (thread = row)
  const int gm = m0 + threadIdx.x;
  if (gm < d.m) {
    const int64_t crow = c_row(d, gm);
#pragma unroll
    for (int j = 0; j < BN; ++j) {
      const int gn = n0 + j;
      if (gn < d.n) C[crow + d.c_sn * (int64_t)gn] = make_float2(acc[2 * j], acc[2 * j + 1]);
    }
  }
  v1::tc_teardown<Cfg::TMEM_COLS>(tmem);
}

}  // namespace v1
}  // namespace fmmt

// ---------------------------------------------------------------- k_tc_conv_z
// Tensor-core version of k_conv_z (kernels_fft.cuh) for n3 <= 32: per batch
// direction q and 128 (kx,ky) lines ij, the last restore contraction
//     T_p[ij, kz] = sum_c G_q[c][ij] V_p(c, kz)        (a4: x3 U3 / TT tail)
// runs on tcgen05 (3xTF32) into TMEM (lane = line ij, columns = kz), and the
// epilogue thread that owns line ij does the pruned forward z-DFT of the
// half-padded spectrum W, the Hadamard product with T_p (a5) and the inverse
// z-DFT truncated to z < Nz (a6), in registers.  T_p never leaves the SM.
namespace fmmt {
namespace v1 {

template <int N3, int MODE>
__global__ void __launch_bounds__(128, 1) k_tc_conv_z(ZArgs a) {
  constexpr int BN = N3 < 16 ? 16 : N3;
  using Cfg = TcGemmCfg<BN>;
  constexpr int Nz = N3 / 2;
  extern __shared__ __align__(1024) uint8_t tcsm[];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ uint32_t tslot;

  const int q = blockIdx.y;
  const int p = a.p0 + q;
  const int m0 = blockIdx.x * TC_BM;
  GemmDesc d;
  d.m = (int)a.n12;
  d.n = N3;
  d.k = a.rank_p ? a.rank_p[p] : a.rank;
  d.batch = 1;
  d.a_s0 = 1; d.a_s1 = 0; d.a_div = 1 << 30; d.a_sk = a.n12;
  d.b_sk = a.v_sc; d.b_sn = a.v_sk;
  d.c_s0 = 0; d.c_s1 = 0; d.c_div = 1; d.c_sn = 0;
  d.sA = d.sB = d.sC = 0;
  const float2* A = a.G + (int64_t)q * a.g_stride;
  const float2* B = a.V + (a.v_off ? a.v_off[p] : (int64_t)q * a.v_stride);

  const uint32_t tmem = v1::tc_setup<Cfg::TMEM_COLS>(bar, &tslot);
  float acc[2 * BN];
  v1::tc_mainloop<BN>(d, A, B, m0, 0, tcsm, bar, tmem, acc);

  const int tid = threadIdx.x;
  const int64_t ij = m0 + tid;
  const bool valid = ij < a.n12;
  if constexpr (MODE == Z_RESTORE) {
    if (valid) {
#pragma unroll
      for (int kz = 0; kz < N3; ++kz) a.Tout[(int64_t)kz * a.n12 + ij] = make_float2(acc[2 * kz], acc[2 * kz + 1]);
    }
  } else {
    float2* Wl = a.W + (int64_t)q * Nz * a.n12 + (valid ? ij : 0);
    float2 f[N3];
#pragma unroll
    for (int z = 0; z < Nz; ++z) f[z] = valid ? Wl[(int64_t)z * a.n12] : make_float2(0.f, 0.f);
    fft_reg<N3, false, true>(f);
#pragma unroll
    for (int kz = 0; kz < N3; ++kz) f[kz] = cmul(make_float2(acc[2 * kz], acc[2 * kz + 1]), f[kz]);
    fft_reg<N3, true, false>(f);
    if (valid) {
#pragma unroll
      for (int z = 0; z < Nz; ++z) Wl[(int64_t)z * a.n12] = f[z];
    }
  }
  v1::tc_teardown<Cfg::TMEM_COLS>(tmem);
}

}  // namespace v1
}  // namespace fmmt
