// kernels_tcws.cuh -- warp-specialised tensor-core restore kernels (one CTA per SM).
//
// Same arithmetic as kernels_tcgemm.cuh (complex embedding, 3xTF32 split, TMEM
// accumulators drained every 4 K-steps into FP32 registers), different schedule:
//   warps 0-3  producers: copy the K-chunks of the CTA's tiles into a TCW_NS-deep
//              shared-memory ring (cp.async straight into the UMMA layout, or one
//              bulk copy of a pre-split static A), split them into TF32 hi / lo,
//              and thread 0 issues the MMAs of each chunk (two per K=8 step) into
//              one of two TMEM slots, committing every chunk to the stage's
//              barrier and every flush group to the slot's barrier;
//   warps 4-7  consumers: drain each flush group's TMEM slot into FP32
//              registers (thread = output row) and release the slot; after a
//              tile's last group they run its epilogue (store C, or the z-DFT,
//              Hadamard and inverse z-DFT of eq. (5)) while the producers and
//              the tensor core already work on the next tile.
// Barriers (shared memory):
//   mmab[NS]  chunk's MMAs complete (tcgen05.commit)   -> stage may be refilled
//   abar[NS]  packed A copy landed (bulk copy tx)      -> producers convert/arrive
//   full[NS]  128 producer arrivals                    -> thread 0 issues MMAs
//   tfull[2]  flush group's MMAs complete (commit)     -> consumers drain the slot
//   tfree[2]  128 consumer arrivals                    -> thread 0 reuses the slot
// Phases: chunk c (CTA-wide count) uses stage c % NS, phase (c / NS) & 1; flush
// group g uses slot g & 1, phase (g / 2) & 1; both roles walk the same tiles.
#pragma once
#include "kernels_tcgemm.cuh"

namespace fmmt {

constexpr int TCW_NS = 8;          // ring stages (8 x 26 KB at BN = 32)
constexpr int TCW_D = TCW_NS - 2;  // copy prefetch distance (chunks)

template <int BN>
struct TcwCfg {
  using C = TcGemmCfg<BN, 1>;
  static constexpr int SMEM = TCW_NS * C::STAGE;
  static constexpr int NBAR = 3 * TCW_NS + 4;
};

struct TcwCursor {
  int c = 0;  // chunks issued (producers)
  int g = 0;  // flush groups (both roles)
};

// Producer side of one tile (tid < 128).
template <int BN>
__device__ __forceinline__ void tcw_produce(const GemmDesc& d, const float2* __restrict__ A,
                                            const float2* __restrict__ B, int m0, int n0, uint8_t* tcsm,
                                            uint64_t* bar, uint32_t tmem, TcwCursor& cur) {
  using Cfg = TcGemmCfg<BN, 1>;
  constexpr int BM = TC_BM, BK = TC_BK, NR = Cfg::NR, NS = TCW_NS, D = TCW_D;
  constexpr int BITEMS = BN * (BK / 2) / 128 > 0 ? BN * (BK / 2) / 128 : 1;
  static_assert(Cfg::BITEMS == BITEMS, "B items per producer thread");
  uint64_t* mmab = bar;
  uint64_t* abar = bar + NS;
  uint64_t* full = bar + 2 * NS;
  uint64_t* tfull = bar + 3 * NS;
  uint64_t* tfree = bar + 3 * NS + 2;
  const uint32_t sbase = tc::smem_u32(tcsm);
  const int tid = threadIdx.x, wrow = tid >> 5, lane = tid & 31;
  const bool a_kcontig = d.a_sk == 1;
  const bool b_kcontig = d.b_sk == 1;
  int64_t arow[4];
  bool okrow[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int r = a_kcontig ? (lane & 7) + 8 * (u + 4 * wrow) : tid;
    okrow[u] = m0 + r < d.m;
    arow[u] = okrow[u] ? a_row(d, m0 + r) : 0;
  }
  constexpr uint32_t IDESC_BP = tc::idesc_tf32(BM, 2 * NR);
  constexpr uint32_t IDESC_B = tc::idesc_tf32(BM, NR);
  const int nk = __shfl_sync(0xffffffffu, (d.k + BK - 1) / BK, 0);   // warp-uniform (see tc_mainloop)
  const int cur_c = __shfl_sync(0xffffffffu, cur.c, 0), cur_g = __shfl_sync(0xffffffffu, cur.g, 0);
  const int warp_u = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const uint32_t sbase_u = __shfl_sync(0xffffffffu, sbase, 0);
  const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem, 0);
  const uint32_t bar_u = __shfl_sync(0xffffffffu, tc::smem_u32(bar), 0);
  const uint64_t dAh = tc::sdesc(sbase_u, Cfg::LBO_A, 128), dAl = tc::sdesc(sbase_u + Cfg::A_BYTES, Cfg::LBO_A, 128);
  const uint64_t dBp = tc::sdesc(sbase_u + 2 * Cfg::A_BYTES, Cfg::LBO_B, 128);
  const bool apack = d.Ap != nullptr;
  const float* apk = apack ? d.Ap + (int64_t)(m0 / BM) * d.a_nkc * TC_PACK_FLOATS : nullptr;

  auto issue = [&](int c) {   // chunk c of this tile -> stage (cur.c + c) % NS, once that stage is free
    const int gc = cur.c + c;
    const int cs = gc % NS;
    if (gc >= NS) tc::mbar_wait(&mmab[cs], ((gc - NS) / NS) & 1);
    const int k0 = c * BK;
    const uint32_t st = sbase + cs * Cfg::STAGE;
    if (apack) {
      if (tid == 0) {
        tc::mbar_expect_tx(&abar[cs], 2 * Cfg::A_BYTES);
        tc::bulk_g2s(st, apk + (int64_t)c * TC_PACK_FLOATS, 2 * Cfg::A_BYTES, &abar[cs]);
      }
    } else if (!a_kcontig) {
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        const int gk = k0 + kk;
        const bool ok = okrow[0] && gk < d.k;
        tc::cp_async8(st + tid * 16 + (kk >> 1) * Cfg::LBO_A + (kk & 1) * 8,
                      ok ? (const void*)(A + arow[0] + gk * d.a_sk) : (const void*)A, ok);
      }
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int kp = lane >> 3;
        const int r = (lane & 7) + 8 * (u + 4 * wrow);
        const int gk = k0 + 2 * kp;
        const bool ok0 = okrow[u] && gk < d.k, ok1 = okrow[u] && gk + 1 < d.k;
        const uint32_t dst = st + r * 16 + kp * Cfg::LBO_A;
        tc::cp_async8(dst, ok0 ? (const void*)(A + arow[u] + gk) : (const void*)A, ok0);
        tc::cp_async8(dst + 8, ok1 ? (const void*)(A + arow[u] + gk + 1) : (const void*)A, ok1);
      }
    }
    const uint32_t rb = st + 2 * Cfg::A_BYTES + Cfg::BP_BYTES;
#pragma unroll
    for (int i = 0; i < BITEMS; ++i) {
      const int idx = tid + 128 * i;
      int j, kp;
      if (!b_kcontig) { j = idx % BN; kp = idx / BN; }
      else { kp = idx % (BK / 2); j = idx / (BK / 2); }
      const int gn = n0 + j, gk = k0 + 2 * kp;
      const bool okn = idx < BN * (BK / 2) && gn < d.n;
      const int gcol = d.b_eo ? (gn < d.n / 2 ? 2 * gn : 2 * (gn - d.n / 2) + 1) : gn;
      const bool ok0 = okn && gk < d.k, ok1 = okn && gk + 1 < d.k;
      const uint32_t dst = rb + (i * 128 + tid) * 16;
      tc::cp_async8(dst, ok0 ? (const void*)(B + gk * d.b_sk + gcol * d.b_sn) : (const void*)B, ok0);
      tc::cp_async8(dst + 8, ok1 ? (const void*)(B + (gk + 1) * d.b_sk + gcol * d.b_sn) : (const void*)B, ok1);
    }
    tc::cp_async_commit();
  };

#pragma unroll 1
  for (int c = 0; c < D; ++c) {
    if (c < nk) issue(c);
    else tc::cp_async_commit();
  }
  for (int kc = 0; kc < nk; ++kc) {
    const int gc = cur.c + kc;
    const int s = gc % NS;
    const uint32_t ph = (gc / NS) & 1;
    if (kc + D < nk) issue(kc + D);
    else tc::cp_async_commit();
    tc::cp_async_wait<D>();
    if (apack) tc::mbar_wait(&abar[s], ph);
    uint8_t* st = tcsm + s * Cfg::STAGE;
    uint8_t* aHi = st;
    uint8_t* aLo = st + Cfg::A_BYTES;
    uint8_t* bP = st + 2 * Cfg::A_BYTES;
    const uint8_t* bRaw = bP + Cfg::BP_BYTES;
    if (!apack) {
#pragma unroll
      for (int u = 0; u < BK / 2; ++u) {
        const uint32_t off = a_kcontig ? ((lane & 7) + 8 * (u + 4 * wrow)) * 16 + (lane >> 3) * Cfg::LBO_A
                                       : tid * 16 + u * Cfg::LBO_A;
        const float4 a = *reinterpret_cast<const float4*>(aHi + off);
        float4 hi, lo;
        tc::split_tf32(a.x, hi.x, lo.x);
        tc::split_tf32(a.y, hi.y, lo.y);
        tc::split_tf32(a.z, hi.z, lo.z);
        tc::split_tf32(a.w, hi.w, lo.w);
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
      const float4 bb = *reinterpret_cast<const float4*>(bRaw + (i * 128 + tid) * 16);
      const float4 r0 = make_float4(bb.x, -bb.y, bb.z, -bb.w);
      const float4 r1 = make_float4(bb.y, bb.x, bb.w, bb.z);
      const uint32_t off = (2 * j) * 16 + kp * Cfg::LBO_B;
      float4 h0, l0, h1, l1;
      tc::split_tf32(r0.x, h0.x, l0.x); tc::split_tf32(r0.y, h0.y, l0.y);
      tc::split_tf32(r0.z, h0.z, l0.z); tc::split_tf32(r0.w, h0.w, l0.w);
      tc::split_tf32(r1.x, h1.x, l1.x); tc::split_tf32(r1.y, h1.y, l1.y);
      tc::split_tf32(r1.z, h1.z, l1.z); tc::split_tf32(r1.w, h1.w, l1.w);
      *reinterpret_cast<float4*>(bP + off) = h0;
      *reinterpret_cast<float4*>(bP + off + 16) = h1;
      *reinterpret_cast<float4*>(bP + off + NR * 16) = l0;
      *reinterpret_cast<float4*>(bP + off + NR * 16 + 16) = l1;
    }
    tc::fence_async_smem();
    tc::mbar_arrive(&full[s]);
    if (warp_u == 0) {                                // warp 0 issues (elect.sync per tcgen05 op)
      __syncwarp();
      const int gcu = cur_c + kc;
      const int su = gcu % NS;
      tc::mbar_wait_addr(bar_u + (2 * NS + su) * 8, (gcu / NS) & 1);           // full[su]
      const int g = cur_g + kc / TC_FC;
      const bool fresh = kc % TC_FC == 0;
      if (fresh && g >= 2) tc::mbar_wait_addr(bar_u + (3 * NS + 2 + (g & 1)) * 8, ((g >> 1) - 1) & 1);   // tfree
      __syncwarp();
      tc::fence_after_sync();
      const uint64_t so = (uint64_t)((su * Cfg::STAGE) >> 4);
      const uint32_t tm = tmem_u + (g & 1) * 2 * NR, tx = tm + NR;
#pragma unroll
      for (int ks = 0; ks < Cfg::KR / 8; ++ks) {
        const uint64_t oa = so + ((ks * 2 * Cfg::LBO_A) >> 4), ob = so + ((ks * 2 * Cfg::LBO_B) >> 4);
        tc::mma_tf32_el(tm, dAh + oa, dBp + ob, IDESC_BP, !(fresh && ks == 0));
        tc::mma_tf32_el(tx, dAl + oa, dBp + ob, IDESC_B, 1);
      }
      tc::mma_commit_el(bar_u + su * 8);                                        // mmab[su]
      if (kc % TC_FC == TC_FC - 1 || kc == nk - 1) tc::mma_commit_el(bar_u + (3 * NS + (g & 1)) * 8);   // tfull
    }
  }
  tc::cp_async_wait<0>();
  cur.c += nk;
  cur.g += (nk + TC_FC - 1) / TC_FC;
}

// Consumer side of one tile (tid >= 128; thread = row tid - 128): acc = sum of the groups.
template <int BN>
__device__ __forceinline__ void tcw_consume(int nk, uint64_t* bar, uint32_t tmem, float (&acc)[2 * BN],
                                            TcwCursor& cur) {
  constexpr int NR = 2 * BN, NS = TCW_NS;
  uint64_t* tfull = bar + 3 * NS;
  uint64_t* tfree = bar + 3 * NS + 2;
  const uint32_t twarp = tmem + ((uint32_t)(((threadIdx.x >> 5) & 3) * 32) << 16);
#pragma unroll
  for (int j = 0; j < NR; ++j) acc[j] = 0.f;
  const int ng = (nk + TC_FC - 1) / TC_FC;
  for (int gl = 0; gl < ng; ++gl) {
    const int g = cur.g + gl;
    tc::mbar_wait(&tfull[g & 1], (g >> 1) & 1);
    tc::fence_after_sync();
    tc_flush<NR, NR>(twarp + (g & 1) * 2 * NR, 0, acc);
    tc::fence_before_sync();
    tc::mbar_arrive(&tfree[g & 1]);
  }
  cur.g += ng;
}

template <int BN>
__device__ __forceinline__ uint32_t tcw_setup(uint64_t* bar, uint32_t* tslot) {
  using Cfg = TcGemmCfg<BN, 1>;
  constexpr int NS = TCW_NS;
  if ((threadIdx.x >> 5) == 0) tc::tmem_alloc<Cfg::TMEM_COLS>(tslot);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2 * NS; ++i) tc::mbar_init(&bar[i], 1);            // mmab, abar
    for (int i = 2 * NS; i < 3 * NS; ++i) tc::mbar_init(&bar[i], 128);     // full
    tc::mbar_init(&bar[3 * NS], 1);                                        // tfull
    tc::mbar_init(&bar[3 * NS + 1], 1);
    tc::mbar_init(&bar[3 * NS + 2], 128);                                  // tfree
    tc::mbar_init(&bar[3 * NS + 3], 128);
    tc::fence_barrier_init();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  return *tslot;
}

// ---------------------------------------------------------------- GEMM
template <int BN>
__global__ void __launch_bounds__(256, 1) k_tcw_cgemm(const GemmDesc* __restrict__ descs, int maxtiles, int maxsub,
                                                      int total) {
  using Cfg = TcGemmCfg<BN, 1>;
  extern __shared__ __align__(1024) uint8_t tcsm[];
  __shared__ __align__(8) uint64_t bar[TcwCfg<BN>::NBAR];
  __shared__ uint32_t tslot;
  const uint32_t tmem = tcw_setup<BN>(bar, &tslot);
  TcwCursor cur;
  const bool producer = threadIdx.x < 128;
  for (int t = blockIdx.x; t < total; t += gridDim.x) {
    const int x = t % maxtiles;
    const int sub = (t / maxtiles) % maxsub;
    const GemmDesc d = descs[t / (maxtiles * maxsub)];
    if (sub >= d.batch) continue;
    const int tiles_m = (d.m + TC_BM - 1) / TC_BM;
    const int tiles_n = (d.n + BN - 1) / BN;
    if (x >= tiles_m * tiles_n) continue;
    const int m0 = (x % tiles_m) * TC_BM;
    const int n0 = (x / tiles_m) * BN;
    if (producer) {
      tcw_produce<BN>(d, d.A + (int64_t)sub * d.sA, d.B + (int64_t)sub * d.sB, m0, n0, tcsm, bar, tmem, cur);
    } else {
      float acc[2 * BN];
      tcw_consume<BN>((d.k + TC_BK - 1) / TC_BK, bar, tmem, acc, cur);
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

// ---------------------------------------------------------------- z-stage (n3 <= 32)
template <int N3, int MODE>
__global__ void __launch_bounds__(256, 1) k_tcw_conv_z(ZArgs a, int nq) {
  constexpr int BN = N3 < 16 ? 16 : N3;
  using Cfg = TcGemmCfg<BN, 1>;
  constexpr int Nz = N3 / 2;
  extern __shared__ __align__(1024) uint8_t tcsm[];
  __shared__ __align__(8) uint64_t bar[TcwCfg<BN>::NBAR];
  __shared__ uint32_t tslot;
  const int tiles_m = (int)((a.n12 + TC_BM - 1) / TC_BM);
  const int total = tiles_m * nq;
  const uint32_t tmem = tcw_setup<BN>(bar, &tslot);
  TcwCursor cur;
  const bool producer = threadIdx.x < 128;
  for (int t = blockIdx.x; t < total; t += gridDim.x) {
    const int q = t / tiles_m;
    const int p = a.p0 + q;
    const int m0 = (t % tiles_m) * TC_BM;
    const int rk = a.rank_p ? a.rank_p[p] : a.rank;
    if (producer) {
      GemmDesc d;
      d.m = (int)a.n12;
      d.n = N3;
      d.k = rk;
      d.batch = 1;
      d.a_s0 = 1; d.a_s1 = 0; d.a_div = 1 << 30; d.a_sk = a.n12;
      d.b_sk = a.v_sc; d.b_sn = a.v_sk;
      d.b_eo = 0;
      d.c_s0 = 0; d.c_s1 = 0; d.c_div = 1; d.c_sn = 0;
      d.sA = d.sB = d.sC = 0;
      d.Ap = a.Gp;
      d.Bp = nullptr;
      d.a_nkc = (rk + TC_BK - 1) / TC_BK;
      const float2* A = a.G + (int64_t)q * a.g_stride;
      const float2* B = a.V + (a.v_off ? a.v_off[p] : (int64_t)q * a.v_stride);
      tcw_produce<BN>(d, A, B, m0, 0, tcsm, bar, tmem, cur);
    } else {
      const int64_t ij = m0 + (threadIdx.x - 128);
      const bool valid = ij < a.n12;
      float acc[2 * BN];
      tcw_consume<BN>((rk + TC_BK - 1) / TC_BK, bar, tmem, acc, cur);
      if constexpr (MODE == Z_RESTORE) {
        if (valid) {
#pragma unroll
          for (int kz = 0; kz < N3; ++kz) a.Tout[(int64_t)kz * a.n12 + ij] = make_float2(acc[2 * kz], acc[2 * kz + 1]);
        }
      } else {
        for (int cc = 0; cc < a.ncomp; ++cc) {
          float2* Wl = a.W + ((int64_t)q * a.ncomp + cc) * Nz * a.n12 + (valid ? ij : 0);
          float2 f[N3];
#pragma unroll
          for (int z = 0; z < Nz; ++z) f[z] = valid ? Wl[(int64_t)z * a.n12] : make_float2(0.f, 0.f);
          fft_reg<N3, false, true>(f);
#pragma unroll
          for (int kz = 0; kz < N3; ++kz) f[kz] = cmul2(f[kz], make_float2(acc[2 * kz], acc[2 * kz + 1]));
          fft_reg<N3, true, false>(f);
          if (valid) {
#pragma unroll
            for (int z = 0; z < Nz; ++z) Wl[(int64_t)z * a.n12] = f[z];
          }
        }
      }
    }
  }
  tc_teardown<Cfg::TMEM_COLS>(tmem);
}

}  // namespace fmmt
