// kernels_tcfuse.cuh -- the Tucker-3D restore chain of Fig. 3(a) (eq. (8)) fused with the z-stage of
// eq. (5) for n3 = 64 and n1 a multiple of 128 (config 5's 128 x 128 x 64 grid).
//
// Per direction q the batch's restore_mode2x GEMM has produced H'_q = core_q x2 U2_q, stored
// H'[c + r3 a + hj j] (c the mode-3 rank index, a the mode-1 rank index, j the y index, hj = r1 r3 rounded
// up to even).  One tile of this
// kernel is (q, 128 lines ij = i + n1 j: an i-block at fixed j) and runs two tensor-core contractions:
//   GEMM1  G[i, c]  = sum_a U1_q[i, a] H'_q[a, c; j]     A: packed U1 (streamed), B: H'_j split into the fp16
//                                                         B' layout in shared memory by the epilogue warps
//   GEMM2  T[i, kz] = sum_c G[i, c] U3_q[kz, c]           A: G, drained from TMEM, scaled by the tile's own
//                                                         power of two, split and written to shared memory;
//                                                         B: packed U3 (streamed)
// then the z-stage epilogue of k_pk_conv_z64 (pruned forward z-DFT of the W line, Hadamard with T, inverse
// z-DFT; the odd-kz half handed over through shared memory).  G (n1 n2 r3 per direction, as large as T_p
// at config 5) never leaves the SM: the unfused chain wrote it, packed it and read it back through HBM.
//
// Warps: 0-7 epilogue (two groups of 128 threads = the 128 TMEM lanes; group h drains real columns
// [64h, 64h + 64) of each accumulator), 8 MMA issuer, 9 operand producer (6-stage ring of 8 KB chunks:
// U1 A-chunks of GEMM1, U3 B'-chunks of GEMM2, in tile order), 10 H' loader: bulk-copies the raw H'_j block
// of the next tile into a staging buffer as soon as the current one has been split (its HBM latency hides
// behind the tile's GEMMs and z-DFTs).  One shared-memory region holds H'_j (B' of GEMM1) and, once GEMM1 has
// completed, G (A of GEMM2); H'_{j+1} of the next tile is split into it (from the staging buffer) as soon as
// GEMM2 has completed, so GEMM1 of tile i+1 overlaps the z-DFT epilogue of tile i.
// TMEM: two 256-column slots (hi.hi | cross) alternating over the flush groups of both GEMMs (tc_flush).
// fp16-split build only (TC_F16).
#pragma once
#include "kernels_tcpk.cuh"

namespace fmmt {

struct ZfArgs {
  float2* W;                    // half-padded spectra of the xy sub-batch [q][comp][Nz][n12]
  int64_t n12;
  int ncomp;
  int p0;                       // op direction of launch-local q = 0 (the launch's first direction)
  int q0;                       // batch-local index of the launch's first direction (H' offset)
  int n1;
  const float* U1p;             // packed U1 of op direction p (A operand: n1 rows, K = r1) at U1p + u1p_off[p]
  const int64_t* u1p_off;
  const float2* H;              // H'_q at H + q h_stride (q batch-local); block j at + j hj_stride(q)
  int64_t h_stride;
  const float* Vp;              // packed U3 B' of op direction p (kz columns [even | odd]) at Vp + vp_off[p]
  const int64_t* vp_off;
  const int* rank;              // per op direction, [ndir][3]: r1, r2, r3
  const float* u1max;           // scale slots: U1 (static), H' (the batch's mode2x output), U3 (static)
  const float* hmax;
  const float* u3max;
  float2* Tout;                 // Z_RESTORE: T_p [kz][ij]
};

// H'_q block of one y index: r1 r3 complex padded to an even count (16-byte aligned bulk copies)
__host__ __device__ inline int64_t zf_hj_stride(int64_t r1, int64_t r3) { return (r1 * r3 + 1) & ~int64_t(1); }

constexpr int ZF_THREADS = 352;
constexpr int ZF_NS = 6;
struct ZfCfg {
  static constexpr int NR = 128;                     // 64 complex columns (c of GEMM1, kz of GEMM2)
  static constexpr int CHUNK = 8192;                 // one packed A chunk (hi + lo) = one B' chunk
  static constexpr int REGION_CHUNKS = 12;           // H'_j B' chunks: r1 <= 96;  G A chunks: r3 <= 64
  static constexpr int MAX_R1 = REGION_CHUNKS * TC_BK;
  static constexpr int HS = MAX_R1 * 64 * 8;         // raw H'_j staging (r1 <= 96, r3 <= 64)
  static constexpr int XB = TC_BM * 32 * 8;          // odd-kz hand-over of the z-DFT epilogue
  static constexpr int RING = ZF_NS * CHUNK;
  static constexpr int REGION = REGION_CHUNKS * CHUNK;
  static constexpr int SMEM = RING + REGION + HS + XB;
  static constexpr uint32_t LBO_A = TC_BM * 16;
  static constexpr uint32_t LBO_B = 2 * NR * 16;
};

template <int MODE>
__global__ void __launch_bounds__(ZF_THREADS, 1) k_tucker_zf(ZfArgs a, int nq) {
  if constexpr (!TC_F16) return;   // fp16-split build only (the host never plans it in the TF32 A/B build)
  constexpr int N3 = 64, H = 32, NR = ZfCfg::NR, NS = ZF_NS;
  constexpr uint32_t IDESC_BP = tc::idesc_f16(TC_BM, 2 * NR), IDESC_B = tc::idesc_f16(TC_BM, NR);
  extern __shared__ __align__(1024) uint8_t zfsm[];
  __shared__ __align__(8) uint64_t bar[2 * NS + 4 + 2 + 4];
  __shared__ uint32_t tslot;
  __shared__ float red[8];
  uint8_t* ring = zfsm;
  uint8_t* region = zfsm + ZfCfg::RING;
  const float2* hs = reinterpret_cast<const float2*>(zfsm + ZfCfg::RING + ZfCfg::REGION);
  float2* X = reinterpret_cast<float2*>(zfsm + ZfCfg::RING + ZfCfg::REGION + ZfCfg::HS);
  uint64_t* MMA = bar;                 // [NS] stage free
  uint64_t* DATA = bar + NS;           // [NS] chunk landed
  uint64_t* GDONE = bar + 2 * NS;      // [2]
  uint64_t* TFREE = bar + 2 * NS + 2;  // [2] (256 arrivals)
  uint64_t* B1FULL = bar + 2 * NS + 4; // H'_j split into the region
  uint64_t* A2FULL = bar + 2 * NS + 5; // G written into the region
  uint64_t* HFULL = bar + 2 * NS + 6;  // raw H'_j staged
  uint64_t* HFREE = bar + 2 * NS + 7;  // staging consumed (split into the region)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tc::tmem_alloc<512>(&tslot);
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) tc::mbar_init(&MMA[i], 1);
    for (int i = 0; i < NS; ++i) tc::mbar_init(&DATA[i], 1);
    tc::mbar_init(&GDONE[0], 1);
    tc::mbar_init(&GDONE[1], 1);
    tc::mbar_init(&TFREE[0], 256);
    tc::mbar_init(&TFREE[1], 256);
    tc::mbar_init(B1FULL, 1);
    tc::mbar_init(A2FULL, 1);
    tc::mbar_init(HFULL, 1);
    tc::mbar_init(HFREE, 1);
    tc::fence_barrier_init();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tslot;
  const int bpd = a.n1 / TC_BM;                         // i-blocks per y index
  const int tiles_m = (int)(a.n12 / TC_BM);
  const int total = tiles_m * nq;
  const int ntiles = total > (int)blockIdx.x ? (total - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
  // tile i of this CTA: direction q (launch-local), m-tile mt = j * bpd + mh (lines ij = mt * 128 + row)
  auto coords = [&](int i, int& q, int& mt) {
    const int t = (int)blockIdx.x + i * (int)gridDim.x;
    q = t / tiles_m;
    mt = t % tiles_m;
  };
  auto r_of = [&](int q, int s) { return a.rank[(int64_t)(a.p0 + q) * 3 + s]; };
  const uint32_t ring_u = tc::smem_u32(ring), region_u = tc::smem_u32(region);

  if (warp == 9) {   // --------------------------------------------------------------- producer
    int64_t c = 0;
    for (int i = 0; i < ntiles; ++i) {
      int q, mt;
      coords(i, q, mt);
      const int p = a.p0 + q;
      const int nkc1 = (r_of(q, 0) + TC_BK - 1) / TC_BK, nkc2 = (r_of(q, 2) + TC_BK - 1) / TC_BK;
      const float* u1 = a.U1p + a.u1p_off[p] + (int64_t)(mt % bpd) * nkc1 * TC_PACK_FLOATS;
      const float* u3 = a.Vp + a.vp_off[p];
      for (int k = 0; k < nkc1 + nkc2; ++k, ++c) {
        const int s = (int)(c % NS);
        if (c >= NS) tc::mbar_wait(&MMA[s], (uint32_t)(((c / NS) - 1) & 1));
        if (lane == 0) {
          tc::mbar_expect_tx(&DATA[s], ZfCfg::CHUNK);
          const float* src = k < nkc1 ? u1 + (int64_t)k * TC_PACK_FLOATS : u3 + (int64_t)(k - nkc1) * (ZfCfg::CHUNK / 4);
          tc::bulk_g2s(ring_u + s * ZfCfg::CHUNK, src, ZfCfg::CHUNK, &DATA[s]);
        }
        __syncwarp();
      }
    }
  } else if (warp == 8) {   // -------------------------------------------------------- MMA issuer
    int64_t c = 0;
    int g = 0;
    for (int i = 0; i < ntiles; ++i) {
      int q, mt;
      coords(i, q, mt);
      const int nk[2] = {(r_of(q, 0) + TC_BK - 1) / TC_BK, (r_of(q, 2) + TC_BK - 1) / TC_BK};
      for (int gm = 0; gm < 2; ++gm) {
        tc::mbar_wait(gm == 0 ? B1FULL : A2FULL, (uint32_t)(i & 1));   // the region holds this GEMM's operand
        for (int kc = 0; kc < nk[gm]; ++kc, ++c) {
          const int s = (int)(c % NS);
          tc::mbar_wait(&DATA[s], (uint32_t)((c / NS) & 1));
          const bool fresh = kc % TC_FC == 0;
          if (fresh && g >= 2) tc::mbar_wait(&TFREE[g & 1], (uint32_t)(((g >> 1) - 1) & 1));
          __syncwarp();
          tc::fence_after_sync();
          const uint32_t tm = tmem + (g & 1) * 2 * NR, tx = tm + NR;
          const uint32_t sa = gm == 0 ? ring_u + s * ZfCfg::CHUNK : region_u + kc * ZfCfg::CHUNK;
          const uint32_t sb = gm == 0 ? region_u + kc * ZfCfg::CHUNK : ring_u + s * ZfCfg::CHUNK;
          const uint64_t dAh = tc::sdesc(sa, ZfCfg::LBO_A, 128), dAl = tc::sdesc(sa + ZfCfg::CHUNK / 2, ZfCfg::LBO_A, 128);
          const uint64_t dBp = tc::sdesc(sb, ZfCfg::LBO_B, 128);
          tc::mma_f16_el(tm, dAh, dBp, IDESC_BP, fresh ? 0u : 1u);
          tc::mma_f16_el(tx, dAl, dBp, IDESC_B, 1u);
          tc::mma_commit_el(tc::smem_u32(&MMA[s]));
          if (kc % TC_FC == TC_FC - 1 || kc == nk[gm] - 1) {
            tc::mma_commit_el(tc::smem_u32(&GDONE[g & 1]));
            ++g;
          }
        }
      }
    }
  } else if (warp == 10) {   // ------------------------------------------------------ H' loader
    for (int i = 0; i < ntiles; ++i) {
      int q, mt;
      coords(i, q, mt);
      const int64_t hj = zf_hj_stride(r_of(q, 0), r_of(q, 2));
      if (i >= 1) tc::mbar_wait(HFREE, (uint32_t)((i - 1) & 1));
      if (lane == 0) {
        tc::mbar_expect_tx(HFULL, (uint32_t)(hj * 8));
        tc::bulk_g2s(tc::smem_u32(hs), a.H + (int64_t)(a.q0 + q) * a.h_stride + hj * (mt / bpd), (uint32_t)(hj * 8), HFULL);
      }
      __syncwarp();
    }
  } else if (warp < 8) {   // -------------------------------------------------------- epilogue
    const int h = warp >> 2;
    const int row = threadIdx.x & (TC_BM - 1);
    const int et = threadIdx.x;                          // 0..255
    const uint32_t twarp = tmem + ((uint32_t)((warp & 3) * 32) << 16);   // this warp's 32 TMEM lanes
    const float sU1 = tc::f16_scale(*a.u1max), sH = tc::f16_scale(*a.hmax), sU3 = tc::f16_scale(*a.u3max);
    // split H'_j of tile i into the region (B' layout of k_pk_pack_b_multi<64>: rows 2c = [Re, -Im],
    // 2c + 1 = [Im, Re] of column c, hi block then lo block, 16 real K per chunk)
    auto pack_h = [&](int i) {
      int q, mt;
      coords(i, q, mt);
      const int r1 = r_of(q, 0), r3 = r_of(q, 2);
      const int nkc1 = (r1 + TC_BK - 1) / TC_BK;
      const float2* Hj = hs;
      tc::mbar_wait(HFULL, (uint32_t)(i & 1));           // H'_j of tile i staged
      // item (B' row r = 2c + parity, K-chunk kc, K-half): 4 consecutive a -> one 16-byte row piece of hi and of lo;
      // consecutive threads take consecutive rows, so each quarter-warp stores 128 contiguous bytes
      const int items = nkc1 * 2 * NR;
      for (int e = et; e < items; e += 256) {
        const int r = e & (NR - 1), half = (e >> 7) & 1, kc = e >> 8;
        const int cc = r >> 1, par = r & 1;
        const int a0 = kc * TC_BK + 4 * half;
        float2 b[4];
#pragma unroll
        for (int t = 0; t < 4; ++t)
          b[t] = (cc < r3 && a0 + t < r1) ? Hj[cc + (int64_t)r3 * (a0 + t)] : make_float2(0.f, 0.f);
        uint4 hi, lo;
        uint32_t* hp = reinterpret_cast<uint32_t*>(&hi);
        uint32_t* lp = reinterpret_cast<uint32_t*>(&lo);
#pragma unroll
        for (int t = 0; t < 4; ++t) {   // row 2c: [Re, -Im], row 2c + 1: [Im, Re] (selects, no divergence)
          const float x0 = par ? b[t].y : b[t].x, x1 = par ? b[t].x : -b[t].y;
          tc::split_f16x2(x0 * sH, x1 * sH, hp[t], lp[t]);
        }
        uint8_t* blk = region + kc * ZfCfg::CHUNK + r * 16 + half * ZfCfg::LBO_B;
        *reinterpret_cast<uint4*>(blk) = hi;
        *reinterpret_cast<uint4*>(blk + NR * 16) = lo;
      }
      tc::fence_async_smem();
      tc::named_bar_sync(1, 256);
      if (et == 0) {
        tc::mbar_arrive(HFREE);                          // the staging buffer may take the next H'_j
        tc::mbar_arrive(B1FULL);
      }
    };
    auto drain = [&](int ngr, int& g, float (&acc)[64]) {
#pragma unroll
      for (int j = 0; j < 64; ++j) acc[j] = 0.f;
      for (int gq = 0; gq < ngr; ++gq, ++g) {
        tc::mbar_wait(&GDONE[g & 1], (uint32_t)((g >> 1) & 1));
        tc::fence_after_sync();
        tc_flush<NR, 64>(twarp + (g & 1) * 2 * NR, h * 64, acc);
        tc::fence_before_sync();
        tc::mbar_arrive(&TFREE[g & 1]);
      }
    };
    int g = 0;
    if (ntiles > 0) pack_h(0);
    for (int i = 0; i < ntiles; ++i) {
      int q, mt;
      coords(i, q, mt);
      const int nkc1 = (r_of(q, 0) + TC_BK - 1) / TC_BK, nkc2 = (r_of(q, 2) + TC_BK - 1) / TC_BK;
      float acc[64];
      // GEMM1 -> G (group h: complex columns c in [32h, 32h + 32))
      drain((nkc1 + TC_FC - 1) / TC_FC, g, acc);
      const float inv1 = 1.f / (sU1 * sH);
      float m = 0.f;
#pragma unroll
      for (int j = 0; j < 64; ++j) {
        acc[j] *= inv1;
        m = fmaxf(m, fabsf(acc[j]));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) red[warp] = m;
      tc::named_bar_sync(1, 256);
      float gmax = red[0];
#pragma unroll
      for (int w = 1; w < 8; ++w) gmax = fmaxf(gmax, red[w]);
      const float sG = tc::f16_scale(gmax);
      // G as GEMM2's A operand (k_pk_pack_a_multi layout): chunk kc2 = 4h + t, 4 complex K per 16 B row piece
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        uint8_t* tile = region + (4 * h + t) * ZfCfg::CHUNK;
#pragma unroll
        for (int kq = 0; kq < 2; ++kq) {
          const int c0 = 8 * t + 4 * kq;   // column within the group's 32
          uint4 hi, lo;
          tc::split_f16x2(acc[2 * c0] * sG, acc[2 * c0 + 1] * sG, hi.x, lo.x);
          tc::split_f16x2(acc[2 * c0 + 2] * sG, acc[2 * c0 + 3] * sG, hi.y, lo.y);
          tc::split_f16x2(acc[2 * c0 + 4] * sG, acc[2 * c0 + 5] * sG, hi.z, lo.z);
          tc::split_f16x2(acc[2 * c0 + 6] * sG, acc[2 * c0 + 7] * sG, hi.w, lo.w);
          const int off = row * 16 + kq * (TC_BM * 16);
          *reinterpret_cast<uint4*>(tile + off) = hi;
          *reinterpret_cast<uint4*>(tile + ZfCfg::CHUNK / 2 + off) = lo;
        }
      }
      tc::fence_async_smem();
      tc::named_bar_sync(1, 256);                        // (also: every thread has read red[])
      if (et == 0) tc::mbar_arrive(A2FULL);
      // GEMM2 -> T (group h: kz = 2m + h, m < 32)
      drain((nkc2 + TC_FC - 1) / TC_FC, g, acc);
      // the region is free (GEMM2 of this tile completed): the next tile's H'_j, so its GEMM1 overlaps the z-DFT
      if (i + 1 < ntiles) pack_h(i + 1);
      const float inv = 1.f / (sG * sU3);
      const int64_t ij = (int64_t)mt * TC_BM + row;
      if constexpr (MODE == Z_RESTORE) {
#pragma unroll
        for (int mm = 0; mm < H; ++mm)
          a.Tout[(int64_t)(2 * mm + h) * a.n12 + ij] = make_float2(acc[2 * mm] * inv, acc[2 * mm + 1] * inv);
      } else {
        for (int cc = 0; cc < a.ncomp; ++cc) {
          float2* Wl = a.W + ((int64_t)q * a.ncomp + cc) * H * a.n12 + ij;
          float2 f[H];
#pragma unroll
          for (int z = 0; z < H; ++z) f[z] = Wl[(int64_t)z * a.n12];
          if (h) {
#pragma unroll
            for (int z = 1; z < H; ++z) f[z] = cmul(f[z], twc<N3, false>(z));
          }
          fft_reg<H, false, false>(f);
#pragma unroll
          for (int mm = 0; mm < H; ++mm) f[mm] = cmul2(f[mm], make_float2(acc[2 * mm] * inv, acc[2 * mm + 1] * inv));
          fft_reg<H, true, false>(f);
          if (h) {
#pragma unroll
            for (int z = 0; z < H; ++z) X[z * TC_BM + row] = z ? cmul(f[z], twc<N3, true>(z)) : f[z];
          }
          tc::named_bar_sync(1, 256);                    // the odd half is in X (both groups read W)
          if (!h) {
#pragma unroll
            for (int z = 0; z < H; ++z) Wl[(int64_t)z * a.n12] = cadd(f[z], X[z * TC_BM + row]);
          }
          tc::named_bar_sync(1, 256);                    // X free for the next component / tile
        }
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

}  // namespace fmmt
