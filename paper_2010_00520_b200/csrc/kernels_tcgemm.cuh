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
// Kernel structure (persistent, warp-specialised, 256 threads, 1 CTA / SM):
//   warps 0-3  producers: cp.async the raw complex64 A / B elements of a
//              K-chunk into a 3-deep raw ring, split them into TF32 hi / lo
//              parts in the canonical K-major UMMA layout (double-buffered),
//              and thread 0 issues the chunk's 12 MMAs into a TMEM slot and
//              commits them to the slot's mbarrier;
//   warps 4-7  accumulator / epilogue: wait for each chunk's commit, add the
//              slot into FP32 registers (thread = output row), release the
//              slot, and after the tile's last chunk run the epilogue (store,
//              or the z-convolution of eq. (5)) while the producers already
//              stream the next tile.
// Tiles are 128 rows x BN complex columns; a CTA walks tiles blockIdx.x,
// blockIdx.x + gridDim.x, ...
#pragma once
#include "kernels_fft.cuh"
#include "kernels_gemm.cuh"
#include "tc.cuh"

namespace fmmt {

constexpr int TC_BM = 128;      // rows per tile (UMMA M)
constexpr int TC_BK = 16;       // complex K per chunk (32 real = 4 UMMA K-steps)
constexpr int TC_NS = 3;        // raw cp.async ring (prefetch distance TC_NS - 1 chunks)
constexpr int TC_THREADS = 256; // 4 producer + 4 accumulator/epilogue warps

template <int BN>
struct TcGemmCfg {
  static constexpr int NR = 2 * BN;                 // real N of the UMMA
  static constexpr int KR = 2 * TC_BK;              // real K per chunk
  static constexpr int A_BYTES = TC_BM * KR * 4;    // one of hi / lo
  static constexpr int B_BYTES = NR * KR * 4;
  static constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;       // hi/lo operand buffer
  static constexpr int BITEMS = BN * (TC_BK / 2) / 128 > 0 ? BN * (TC_BK / 2) / 128 : 1;
  static constexpr int RAW_A = TC_BM * TC_BK * 8;                // raw complex64 staging
  static constexpr int RAW = RAW_A + BITEMS * 128 * 16;
  static constexpr int SMEM = 2 * STAGE + TC_NS * RAW;
  // two accumulator slots (alternating K-chunks) x {main hi.hi, cross hi.lo + lo.hi}
  static constexpr int TMEM_COLS = 4 * NR < 32 ? 32 : 4 * NR;
  static constexpr uint32_t LBO_A = TC_BM * 16;     // K-adjacent core matrices
  static constexpr uint32_t LBO_B = NR * 16;
};

// Pipeline barriers (static shared memory).
struct TcSync {
  uint64_t mma[2];    // tcgen05.commit of the chunk that used operand buffer / TMEM slot s
  uint64_t tfree[2];  // the 128 accumulator threads have drained TMEM slot s
  uint32_t tslot;     // TMEM base address
};

__device__ __forceinline__ float4 split4_hi_lo(float a, float b, float c, float d, float4& lo) {
  float4 hi;
  tc::split_tf32(a, hi.x, lo.x);
  tc::split_tf32(b, hi.y, lo.y);
  tc::split_tf32(c, hi.z, lo.z);
  tc::split_tf32(d, hi.w, lo.w);
  return hi;
}

__device__ __forceinline__ void producer_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// Accuracy of the tensor-core accumulation.  The tensor core adds each MMA's
// products into the FP32 accumulator with truncation, so the error of one
// accumulator grows with the number of MMAs chained into it (measured 2.4e-6
// relative at K = 169 with a single chain; the restore bound is 1e-6).  Each
// K-chunk (TC_BK complex = 4 K-steps) therefore accumulates into a fresh TMEM
// slot, with the hi.hi products (4 MMAs) and the two 2^-11-smaller cross terms
// (8 MMAs) in separate accumulators, and the chunk results are summed in FP32
// registers (round-to-nearest) by the accumulator warps.  Two slots alternate
// so chunk k+1's MMAs overlap the drain of chunk k.
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

// Producer side of one tile: A[m0:m0+128, :] . B[:, n0:n0+BN], all K-chunks.
// Called by the 128 producer threads (tid 0..127).  g = this CTA's running
// chunk counter (slot / buffer of chunk g is g & 1, its use index g >> 1).
template <int BN>
__device__ __forceinline__ void tc_produce(const GemmDesc& d, const float2* __restrict__ A,
                                           const float2* __restrict__ B, int m0, int n0, uint8_t* tcsm,
                                           TcSync& S, uint32_t tmem, uint32_t g) {
  using Cfg = TcGemmCfg<BN>;
  constexpr int BM = TC_BM, BK = TC_BK, NR = Cfg::NR, NS = TC_NS;
  constexpr int BITEMS = Cfg::BITEMS;
  const uint32_t sbase = tc::smem_u32(tcsm);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool a_kcontig = d.a_sk == 1;   // rows of A are contiguous in K
  const bool b_kcontig = d.b_sk == 1;
  // rows this thread copies: row-per-thread (row tid) or K-contiguous (4 rows)
  int64_t arow[4];
  bool okrow[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int r = a_kcontig ? (lane & 7) + 8 * (u + 4 * warp) : tid;
    okrow[u] = m0 + r < d.m;
    arow[u] = okrow[u] ? a_row(d, m0 + r) : 0;
  }
  constexpr uint32_t IDESC = tc::idesc_tf32(BM, NR);
  const uint32_t raw0 = sbase + 2 * Cfg::STAGE;

  const int nk = (d.k + BK - 1) / BK;
  // raw copies of chunk c into ring stage c % NS (zero-filled outside the problem); each
  // thread copies exactly the elements it converts later, so copy -> convert needs no barrier
  auto issue = [&](int c) {
    if (c < nk) {
      const int k0 = c * BK;
      const uint32_t ra = raw0 + (c % NS) * Cfg::RAW;
      if (!a_kcontig) {
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
          const int gk = k0 + kk;
          const bool ok = okrow[0] && gk < d.k;
          tc::cp_async8(ra + (kk * 128 + tid) * 8, ok ? (const void*)(A + arow[0] + gk * d.a_sk) : (const void*)A, ok);
        }
      } else {
#pragma unroll
        for (int i = 0; i < BK / 2; ++i) {
          const int gk = k0 + 2 * ((lane >> 3) + 4 * (i & 1));
          const bool ok0 = okrow[i >> 1] && gk < d.k, ok1 = okrow[i >> 1] && gk + 1 < d.k;
          const uint32_t dst = ra + (i * 128 + tid) * 16;
          tc::cp_async8(dst, ok0 ? (const void*)(A + arow[i >> 1] + gk) : (const void*)A, ok0);
          tc::cp_async8(dst + 8, ok1 ? (const void*)(A + arow[i >> 1] + gk + 1) : (const void*)A, ok1);
        }
      }
      const uint32_t rb = ra + Cfg::RAW_A;
#pragma unroll
      for (int i = 0; i < BITEMS; ++i) {
        const int idx = tid + 128 * i;
        int j, kp;
        if (!b_kcontig) { j = idx % BN; kp = idx / BN; }    // n (not k) contiguous in memory
        else { kp = idx % (BK / 2); j = idx / (BK / 2); }   // k contiguous
        const int gn = n0 + j, gk = k0 + 2 * kp;
        const bool okn = idx < BN * (BK / 2) && gn < d.n;
        const bool ok0 = okn && gk < d.k, ok1 = okn && gk + 1 < d.k;
        const uint32_t dst = rb + (i * 128 + tid) * 16;
        tc::cp_async8(dst, ok0 ? (const void*)(B + gk * d.b_sk + gn * d.b_sn) : (const void*)B, ok0);
        tc::cp_async8(dst + 8, ok1 ? (const void*)(B + (gk + 1) * d.b_sk + gn * d.b_sn) : (const void*)B, ok1);
      }
    }
    tc::cp_async_commit();   // (possibly empty) group per chunk keeps the group count uniform
  };
#pragma unroll
  for (int c = 0; c < NS - 1; ++c) issue(c);

  for (int kc = 0; kc < nk; ++kc) {
    const uint32_t gg = g + kc;
    const int s = gg & 1;
    issue(kc + NS - 1);
    tc::cp_async_wait<NS - 1>();                  // this thread's copies of chunk kc have landed
    const uint8_t* rawA = tcsm + 2 * Cfg::STAGE + (kc % NS) * Cfg::RAW;
    const uint8_t* rawB = rawA + Cfg::RAW_A;
    // operand buffer s is free once the MMAs of chunk gg-2 completed
    if (gg >= 2) tc::mbar_wait(&S.mma[s], ((gg >> 1) - 1) & 1);
    uint8_t* st = tcsm + s * Cfg::STAGE;
    uint8_t* aHi = st;
    uint8_t* aLo = st + Cfg::A_BYTES;
    uint8_t* bHi = st + 2 * Cfg::A_BYTES;
    uint8_t* bLo = bHi + Cfg::B_BYTES;
    // ---- raw -> hi / lo operand buffers, 16-byte rows of the core matrices
    if (!a_kcontig) {
#pragma unroll
      for (int kp = 0; kp < BK / 2; ++kp) {
        const float2 a0 = *reinterpret_cast<const float2*>(rawA + ((2 * kp) * 128 + tid) * 8);
        const float2 a1 = *reinterpret_cast<const float2*>(rawA + ((2 * kp + 1) * 128 + tid) * 8);
        float4 lo;
        const float4 hi = split4_hi_lo(a0.x, a0.y, a1.x, a1.y, lo);
        const uint32_t off = tid * 16 + kp * Cfg::LBO_A;
        *reinterpret_cast<float4*>(aHi + off) = hi;
        *reinterpret_cast<float4*>(aLo + off) = lo;
      }
    } else {
#pragma unroll
      for (int i = 0; i < BK / 2; ++i) {
        const int kp = (lane >> 3) + 4 * (i & 1);
        const int r = (lane & 7) + 8 * ((i >> 1) + 4 * warp);
        const float4 a = *reinterpret_cast<const float4*>(rawA + (i * 128 + tid) * 16);
        float4 lo;
        const float4 hi = split4_hi_lo(a.x, a.y, a.z, a.w, lo);
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
      const float4 bb = *reinterpret_cast<const float4*>(rawB + (i * 128 + tid) * 16);
      float4 lo;
      // row 2j: [Re b, -Im b] ; row 2j+1: [Im b, Re b]
      float4 hi = split4_hi_lo(bb.x, -bb.y, bb.z, -bb.w, lo);
      uint32_t off = (2 * j) * 16 + kp * Cfg::LBO_B;
      *reinterpret_cast<float4*>(bHi + off) = hi;
      *reinterpret_cast<float4*>(bLo + off) = lo;
      hi = split4_hi_lo(bb.y, bb.x, bb.w, bb.z, lo);
      off += 16;
      *reinterpret_cast<float4*>(bHi + off) = hi;
      *reinterpret_cast<float4*>(bLo + off) = lo;
    }
    tc::fence_async_smem();
    producer_bar();
    if (tid == 0) {
      // TMEM slot s is free once the accumulator warps drained chunk gg-2
      if (gg >= 2) tc::mbar_wait(&S.tfree[s], ((gg >> 1) - 1) & 1);
      tc::fence_after_sync();
      const uint32_t sa_hi = sbase + s * Cfg::STAGE, sa_lo = sa_hi + Cfg::A_BYTES;
      const uint32_t sb_hi = sa_hi + 2 * Cfg::A_BYTES, sb_lo = sb_hi + Cfg::B_BYTES;
      const uint32_t tm = tmem + s * 2 * NR, tx = tm + NR;
#pragma unroll
      for (int ks = 0; ks < Cfg::KR / 8; ++ks) {
        const uint64_t ah = tc::sdesc(sa_hi + ks * 2 * Cfg::LBO_A, Cfg::LBO_A, 128);
        const uint64_t al = tc::sdesc(sa_lo + ks * 2 * Cfg::LBO_A, Cfg::LBO_A, 128);
        const uint64_t bh = tc::sdesc(sb_hi + ks * 2 * Cfg::LBO_B, Cfg::LBO_B, 128);
        const uint64_t bl = tc::sdesc(sb_lo + ks * 2 * Cfg::LBO_B, Cfg::LBO_B, 128);
        tc::mma_tf32(tx, al, bh, IDESC, ks != 0);
        tc::mma_tf32(tx, ah, bl, IDESC, 1);
        tc::mma_tf32(tm, ah, bh, IDESC, ks != 0);
      }
      tc::mma_commit(&S.mma[s]);
    }
  }
  tc::cp_async_wait<0>();
}

// Accumulator side of one tile (the 128 threads of warps 4-7; thread = row):
// acc[2BN] (re, im interleaved) = sum over the tile's nk chunks.
template <int BN>
__device__ __forceinline__ void tc_accumulate(int nk, uint32_t g, TcSync& S, uint32_t tmem, float (&acc)[2 * BN]) {
  constexpr int NR = 2 * BN;
  const uint32_t twarp = tmem + ((uint32_t)(((threadIdx.x >> 5) & 3) * 32) << 16);   // this warp's lanes
#pragma unroll
  for (int j = 0; j < NR; ++j) acc[j] = 0.f;
  for (int kc = 0; kc < nk; ++kc) {
    const uint32_t gg = g + kc;
    const int s = gg & 1;
    tc::mbar_wait(&S.mma[s], (gg >> 1) & 1);
    tc::fence_after_sync();
    tc_flush<BN>(twarp + s * 2 * NR, acc);
    tc::fence_before_sync();
    tc::mbar_arrive(&S.tfree[s]);
  }
}

// TMEM allocation + pipeline barriers (all threads call; warp 0 allocates).
template <int TMEM_COLS>
__device__ __forceinline__ uint32_t tc_setup(TcSync& S) {
  if ((threadIdx.x >> 5) == 0) tc::tmem_alloc<TMEM_COLS>(&S.tslot);
  if (threadIdx.x == 0) {
    tc::mbar_init(&S.mma[0], 1);
    tc::mbar_init(&S.mma[1], 1);
    tc::mbar_init(&S.tfree[0], 128);
    tc::mbar_init(&S.tfree[1], 128);
    tc::fence_barrier_init();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  return S.tslot;
}

template <int TMEM_COLS>
__device__ __forceinline__ void tc_teardown(uint32_t tmem) {
  tc::fence_before_sync();
  __syncthreads();
  if ((threadIdx.x >> 5) == 0) tc::tmem_dealloc<TMEM_COLS>(tmem);
}

// Tile t of a descriptor-list launch -> (descriptor, sub-batch, m0, n0); false if empty.
template <int BN>
__device__ __forceinline__ bool tc_tile(const GemmDesc* __restrict__ descs, int t, int maxtiles, int maxsub,
                                        GemmDesc& d, int& sub, int& m0, int& n0) {
  const int x = t % maxtiles;
  const int y = (t / maxtiles) % maxsub;
  const int z = t / (maxtiles * maxsub);
  d = descs[z];
  sub = y;
  if (sub >= d.batch) return false;
  const int tiles_m = (d.m + TC_BM - 1) / TC_BM;
  const int tiles_n = (d.n + BN - 1) / BN;
  if (x >= tiles_m * tiles_n) return false;
  m0 = (x % tiles_m) * TC_BM;
  n0 = (x / tiles_m) * BN;
  return true;
}

template <int BN>
__global__ void __launch_bounds__(TC_THREADS, 1) k_tc_cgemm(const GemmDesc* __restrict__ descs, int maxtiles,
                                                             int maxsub, int ndesc) {
  using Cfg = TcGemmCfg<BN>;
  constexpr int NR = Cfg::NR;
  extern __shared__ __align__(1024) uint8_t tcsm[];
  __shared__ TcSync S;
  const uint32_t tmem = tc_setup<Cfg::TMEM_COLS>(S);
  const int total = maxtiles * maxsub * ndesc;
  uint32_t g = 0;
  if (threadIdx.x < 128) {
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      GemmDesc d;
      int sub, m0, n0;
      if (!tc_tile<BN>(descs, t, maxtiles, maxsub, d, sub, m0, n0)) continue;
      tc_produce<BN>(d, d.A + (int64_t)sub * d.sA, d.B + (int64_t)sub * d.sB, m0, n0, tcsm, S, tmem, g);
      g += (d.k + TC_BK - 1) / TC_BK;
    }
  } else {
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      GemmDesc d;
      int sub, m0, n0;
      if (!tc_tile<BN>(descs, t, maxtiles, maxsub, d, sub, m0, n0)) continue;
      const int nk = (d.k + TC_BK - 1) / TC_BK;
      float acc[NR];
      tc_accumulate<BN>(nk, g, S, tmem, acc);
      g += nk;
      float2* C = d.C + (int64_t)sub * d.sC;
      const int gm = m0 + (threadIdx.x - 128);
      if (gm < d.m) {
        const int64_t crow = c_row(d, gm);
#pragma unroll
        for (int j = 0; j < BN; ++j) {
          const int gn = n0 + j;
          if (gn < d.n) C[crow + d.c_sn * (int64_t)gn] = make_float2(acc[2 * j], acc[2 * j + 1]);
        }
      }
    }
  }
  tc_teardown<Cfg::TMEM_COLS>(tmem);
}

// ---------------------------------------------------------------- k_tc_conv_z
// Tensor-core version of k_conv_z (kernels_fft.cuh) for n3 <= 32.  Tile =
// (batch direction q, 128 (kx,ky) lines ij).  The last restore contraction
//     T_p[ij, kz] = sum_c G_q[c][ij] V_p(c, kz)        (a4: x3 U3 / TT tail)
// runs on tcgen05 (3xTF32); the accumulator thread that owns line ij then does
// the pruned forward z-DFT of the half-padded spectrum W, the Hadamard product
// with T_p (a5) and the inverse z-DFT truncated to z < Nz (a6), in registers.
// T_p never leaves the SM.
template <int N3>
__device__ __forceinline__ void z_desc(const ZArgs& a, int q, GemmDesc& d, const float2*& A, const float2*& B) {
  const int p = a.p0 + q;
  d.m = (int)a.n12;
  d.n = N3;
  d.k = a.rank_p ? a.rank_p[p] : a.rank;
  d.batch = 1;
  d.a_s0 = 1; d.a_s1 = 0; d.a_div = 1 << 30; d.a_sk = a.n12;
  d.b_sk = a.v_sc; d.b_sn = a.v_sk;
  d.c_s0 = 0; d.c_s1 = 0; d.c_div = 1; d.c_sn = 0;
  d.sA = d.sB = d.sC = 0;
  A = a.G + (int64_t)q * a.g_stride;
  B = a.V + (a.v_off ? a.v_off[p] : (int64_t)q * a.v_stride);
}

template <int N3, int MODE>
__global__ void __launch_bounds__(TC_THREADS, 1) k_tc_conv_z(ZArgs a, int nq) {
  constexpr int BN = N3 < 16 ? 16 : N3;
  using Cfg = TcGemmCfg<BN>;
  constexpr int Nz = N3 / 2;
  extern __shared__ __align__(1024) uint8_t tcsm[];
  __shared__ TcSync S;
  const uint32_t tmem = tc_setup<Cfg::TMEM_COLS>(S);
  const int tiles_m = (int)((a.n12 + TC_BM - 1) / TC_BM);
  const int total = tiles_m * nq;
  uint32_t g = 0;
  if (threadIdx.x < 128) {
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      GemmDesc d;
      const float2 *A, *B;
      z_desc<N3>(a, t / tiles_m, d, A, B);
      tc_produce<BN>(d, A, B, (t % tiles_m) * TC_BM, 0, tcsm, S, tmem, g);
      g += (d.k + TC_BK - 1) / TC_BK;
    }
  } else {
    const int e = threadIdx.x - 128;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      const int q = t / tiles_m;
      const int p = a.p0 + q;
      const int nk = ((a.rank_p ? a.rank_p[p] : a.rank) + TC_BK - 1) / TC_BK;
      const int64_t ij = (int64_t)(t % tiles_m) * TC_BM + e;
      const bool valid = ij < a.n12;
      float2* Wl = a.W + (int64_t)q * Nz * a.n12 + (valid ? ij : 0);
      float2 f[N3];
      if constexpr (MODE != Z_RESTORE) {
        // the half-padded spectrum line is loaded before the accumulator wait (latency overlap)
#pragma unroll
        for (int z = 0; z < Nz; ++z) f[z] = valid ? Wl[(int64_t)z * a.n12] : make_float2(0.f, 0.f);
      }
      float acc[2 * BN];
      tc_accumulate<BN>(nk, g, S, tmem, acc);
      g += nk;
      if constexpr (MODE == Z_RESTORE) {
        if (valid) {
#pragma unroll
          for (int kz = 0; kz < N3; ++kz) a.Tout[(int64_t)kz * a.n12 + ij] = make_float2(acc[2 * kz], acc[2 * kz + 1]);
        }
      } else {
        fft_reg<N3, false, true>(f);
#pragma unroll
        for (int kz = 0; kz < N3; ++kz) f[kz] = cmul(make_float2(acc[2 * kz], acc[2 * kz + 1]), f[kz]);
        fft_reg<N3, true, false>(f);
        if (valid) {
#pragma unroll
          for (int z = 0; z < Nz; ++z) Wl[(int64_t)z * a.n12] = f[z];
        }
      }
    }
  }
  tc_teardown<Cfg::TMEM_COLS>(tmem);
}

}  // namespace fmmt
