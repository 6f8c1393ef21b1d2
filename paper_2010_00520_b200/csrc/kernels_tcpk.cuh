// kernels_tcpk.cuh -- the restore contractions of Figs. 3-4 on the sm_100a tensor
// cores with BOTH operands pre-split in global memory (k_tc_pack_a / k_tc_pack_b layouts), as a
// persistent, tile-walking pipeline:
//
//   warp 0   one elected lane streams operand chunks with 1-D bulk async copies (TMA engine) into an
//            NS-stage shared-memory ring, up to NS - 2 chunks ahead of the MMAs and across tile
//            boundaries (the next tile's first chunks land during this tile's epilogue); the same
//            warp issues the chunk's tcgen05.mma pair (A_hi x [B_hi ; B_lo], A_lo x B_hi) and commits
//            them to the stage's barrier (stage free) and, at the end of each flush group, to the
//            group's barrier.
//   warps 0-3  drain each flush group's TMEM accumulators (hi.hi and cross terms, FP32, truncating
//            tensor-core adds) into round-to-nearest FP32 registers as soon as the group completes
//            (tc_flush; two TMEM slots alternate), then run the tile's epilogue (store, or the fused
//            z-DFT / Hadamard / inverse z-DFT of the translate z-stage).
//
// No thread converts operands: the pack kernels do it once per operand (static factors once per op,
// dynamic intermediates once per batch), so the mainloop has no per-chunk thread work, no
// cp.async, and no all-thread barrier per chunk.  Barriers: mma[NS] (stage free, waited by warp 0
// in chunk order), data[NS] (bulk copies landed), gdone[2] (a flush group's MMAs completed, waited
// by every thread), tfree[2] (128 arrivals: the group's TMEM slot drained).
#pragma once
#include "kernels_tcgemm.cuh"

namespace fmmt {

template <int BN, int NS>
struct PkCfg {
  static constexpr int NR = 2 * BN;                       // real columns of C (re, im interleaved)
  static constexpr int KR = 2 * TC_BK;                    // real K per chunk
  static constexpr int A_BYTES = TC_BM * KR * TC_ESZ;     // one of hi / lo
  static constexpr int BP_ROWS = 2 * NR;                  // B' = [B^_hi ; B^_lo]
  static constexpr int BP_BYTES = BP_ROWS * KR * TC_ESZ;
  static constexpr int BP_FLOATS = BP_BYTES / 4;          // == TcGemmCfg<BN>::BP_FLOATS (pack_b layout)
  static constexpr int STAGE = 2 * A_BYTES + BP_BYTES;
  static constexpr int SMEM = NS * STAGE;
  static constexpr int TMEM_COLS = 4 * NR < 32 ? 32 : 4 * NR;   // two slots x (hi.hi | cross)
  static constexpr uint32_t LBO_A = TC_BM * 16;
  static constexpr uint32_t LBO_B = BP_ROWS * 16;
  static constexpr int D = NS - 1;                        // chunks requested ahead of the next to issue
  static constexpr int NBAR = 2 * NS + 4;
  static_assert(BP_FLOATS == TcGemmCfg<BN, 1>::BP_FLOATS, "pack_b layout");
  static_assert(STAGE % 128 == 0, "stage alignment");
};

// One tile of the walk: packed A chunks (k-chunk c at apk + c * TC_PACK_FLOATS), packed B' chunks
// (at bpk + c * BP_FLOATS), chunk count; nk == 0: nothing to do for this tile.
struct PkTile {
  const float* apk;
  const float* bpk;
  int nk;
};

// CL = CTAs per cluster sharing the A operand (1, or 2: each CTA streams half of every A chunk and multicasts it
// to both; a stage is free once both CTAs' MMAs on it completed, so mma[s] counts CL commit arrivals).
// EG = drain/epilogue warpgroups (1: warps 0-3 drain all columns; 2: warps 0-3 the first NR / 2 and warps 4-7
// the second NR / 2 real columns of the same 128 TMEM lanes, MMA warp 8, producer warp 9).
template <int BN, int NS, int CL = 1, int EG = 1>
__device__ __forceinline__ uint32_t pk_setup(uint64_t* bar, uint32_t* tslot) {
  using Cfg = PkCfg<BN, NS>;
  if ((threadIdx.x >> 5) == 0) tc::tmem_alloc<Cfg::TMEM_COLS>(tslot);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NS; ++i) tc::mbar_init(&bar[i], CL);              // mma (stage free)
#pragma unroll
    for (int i = NS; i < 2 * NS + 2; ++i) tc::mbar_init(&bar[i], 1);      // data, gdone
#pragma unroll
    for (int i = 2 * NS + 2; i < 2 * NS + 4; ++i) tc::mbar_init(&bar[i], 128 * EG);   // tfree
    tc::fence_barrier_init();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if constexpr (CL > 1) tc::cluster_sync();   // the peer's multicast copies / commits target these barriers
  return *tslot;
}

// Walk `ntiles` tiles (this CTA's), tile i described by tile_of(i), with PK_THREADS = 192 threads in
// three roles:
//   warps 0-3  (the 128 TMEM lanes = tile rows): drain each flush group of the tile into FP32 registers,
//              then epi(i, acc) with acc = the tile's 128 x BN complex block (thread = row, re/im
//              interleaved, unscaled);
//   warp 4     MMA issuer: per chunk waits for its operands (data[s]) and, at a group start, for the
//              group's TMEM slot to be drained (tfree), issues the chunk's MMA pair, commits it to mma[s]
//              and, at a group end, to gdone;
//   warp 5     producer: streams chunks (bulk async copies) into the NS-stage ring as soon as a stage's
//              previous MMAs completed, across tile boundaries.
// The MMA warp therefore runs into tile i+1 (other TMEM slot) while warps 0-3 drain and finish tile i.
constexpr int PK_THREADS = 192;

template <int BN, int NS, class TileOf, class Epi, int CL = 1, int EG = 1, int FC = TC_FC>
__device__ __forceinline__ void pk_run(int ntiles, TileOf tile_of, Epi epi, uint8_t* sm, uint64_t* bar, uint32_t tmem) {
  using Cfg = PkCfg<BN, NS>;
  constexpr int NR = Cfg::NR;
  constexpr int NRG = NR / EG;   // real columns drained per epilogue warpgroup
  static_assert(NRG % 16 == 0, "drain granularity");
  constexpr uint32_t IDESC_BP = TC_F16 ? tc::idesc_f16(TC_BM, 2 * NR) : tc::idesc_tf32(TC_BM, 2 * NR);
  constexpr uint32_t IDESC_B = TC_F16 ? tc::idesc_f16(TC_BM, NR) : tc::idesc_tf32(TC_BM, NR);
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const uint32_t sbase = __shfl_sync(0xffffffffu, tc::smem_u32(sm), 0);
  const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem, 0);
  const uint32_t bar_u = __shfl_sync(0xffffffffu, tc::smem_u32(bar), 0);
  auto MMA = [&](int s) { return bar_u + s * 8; };
  auto DATA = [&](int s) { return bar_u + (NS + s) * 8; };
  auto GDONE = [&](int j) { return bar_u + (2 * NS + j) * 8; };
  auto TFREE = [&](int j) { return bar_u + (2 * NS + 2 + j) * 8; };

  if (warp == 4 * EG + 1) {   // ------------------------------------------------------- producer
    int64_t c = 0;
    const uint32_t crank = CL > 1 ? tc::cluster_rank() : 0;
    for (int i = 0; i < ntiles; ++i) {
      const PkTile t = tile_of(i);
      for (int k = 0; k < t.nk; ++k, ++c) {
        const int s = (int)(c % NS);
        if (c >= NS) tc::mbar_wait_addr(MMA(s), (uint32_t)(((c / NS) - 1) & 1));   // stage free (all CL CTAs)
        if (lane == 0) {
          uint64_t* db = bar + NS + s;
          tc::mbar_expect_tx(db, 2 * Cfg::A_BYTES + Cfg::BP_BYTES);
          const uint32_t st = sbase + s * Cfg::STAGE;
          const float* ach = t.apk + (int64_t)k * TC_PACK_FLOATS;
          if constexpr (CL == 1) {
            tc::bulk_g2s(st, ach, 2 * Cfg::A_BYTES, db);
          } else {   // this CTA's half of the A chunk (A_hi or A_lo) to both CTAs of the pair
            tc::bulk_g2s_mc(st + crank * Cfg::A_BYTES, ach + crank * (Cfg::A_BYTES / 4), Cfg::A_BYTES, DATA(s), 0x3);
          }
          tc::bulk_g2s(st + 2 * Cfg::A_BYTES, t.bpk + (int64_t)k * Cfg::BP_FLOATS, Cfg::BP_BYTES, db);
        }
        __syncwarp();
      }
    }
    if constexpr (CL > 1) {   // every stage's last commits (this CTA's and the peer's) have landed before exit
      for (int64_t e = c - NS < 0 ? 0 : c - NS; e < c; ++e)
        tc::mbar_wait_addr(MMA((int)(e % NS)), (uint32_t)((e / NS) & 1));
    }
  } else if (warp == 4 * EG) {   // ----------------------------------------------------- MMA issuer
    const uint64_t dAh = tc::sdesc(sbase, Cfg::LBO_A, 128), dAl = tc::sdesc(sbase + Cfg::A_BYTES, Cfg::LBO_A, 128);
    const uint64_t dBp = tc::sdesc(sbase + 2 * Cfg::A_BYTES, Cfg::LBO_B, 128);
    int64_t c = 0;
    int g = 0;
    for (int i = 0; i < ntiles; ++i) {
      const int nk = tile_of(i).nk;
      for (int kc = 0; kc < nk; ++kc, ++c) {
        const int s = (int)(c % NS);
        tc::mbar_wait_addr(DATA(s), (uint32_t)((c / NS) & 1));
        const bool fresh = kc % FC == 0;
        if (fresh && g >= 2) tc::mbar_wait_addr(TFREE(g & 1), (uint32_t)(((g >> 1) - 1) & 1));
        __syncwarp();
        tc::fence_after_sync();
        const uint64_t so = (uint64_t)((s * Cfg::STAGE) >> 4);
        const uint32_t tm = tmem_u + (g & 1) * 2 * NR, tx = tm + NR;
#pragma unroll
        for (int ks = 0; ks < Cfg::KR / TC_KSTEP; ++ks) {
          const uint64_t oa = so + ((ks * 2 * Cfg::LBO_A) >> 4), ob = so + ((ks * 2 * Cfg::LBO_B) >> 4);
          if constexpr (TC_F16) {
            tc::mma_f16_el(tm, dAh + oa, dBp + ob, IDESC_BP, !(fresh && ks == 0));
            tc::mma_f16_el(tx, dAl + oa, dBp + ob, IDESC_B, 1);
          } else {
            tc::mma_tf32_el(tm, dAh + oa, dBp + ob, IDESC_BP, !(fresh && ks == 0));
            tc::mma_tf32_el(tx, dAl + oa, dBp + ob, IDESC_B, 1);
          }
        }
        if constexpr (CL == 1) tc::mma_commit_el(MMA(s));
        else tc::mma_commit_mc_el(MMA(s), 0x3);            // frees the stage in both CTAs of the pair
        if (kc % FC == FC - 1 || kc == nk - 1) {   // group g closed
          tc::mma_commit_el(GDONE(g & 1));
          ++g;
        }
      }
    }
  } else if (warp < 4 * EG) {   // ------------------------------------ warps 0 .. 4 EG - 1: drain + epilogue
    const uint32_t twarp = tmem_u + ((uint32_t)((warp & 3) * 32) << 16);
    const int grp = warp >> 2;
    float acc[NRG];
    int g = 0;
    for (int i = 0; i < ntiles; ++i) {
      const int nk = tile_of(i).nk;
      if (nk <= 0) continue;
#pragma unroll
      for (int j = 0; j < NRG; ++j) acc[j] = 0.f;
      const int ngr = (nk + FC - 1) / FC;
      for (int q = 0; q < ngr; ++q, ++g) {
        tc::mbar_wait_addr(GDONE(g & 1), (uint32_t)((g >> 1) & 1));
        tc::fence_after_sync();
        tc_flush<NR, NRG>(twarp + (g & 1) * 2 * NR, grp * NRG, acc);
        tc::fence_before_sync();
        tc::mbar_arrive(&bar[2 * NS + 2 + (g & 1)]);
      }
      if constexpr (EG == 1) epi(i, acc);
      else epi(i, acc, grp);
    }
  }
}

template <int BN, int NS, int CL = 1, int EG = 1>
__device__ __forceinline__ void pk_teardown(uint32_t tmem) {
  tc::fence_before_sync();
  __syncthreads();
  if constexpr (CL > 1) tc::cluster_sync();
  if ((threadIdx.x >> 5) == 0) tc::tmem_dealloc<PkCfg<BN, NS>::TMEM_COLS>(tmem);
}

// ---------------------------------------------------------------- k_pk_cgemm
// Batched complex GEMMs C = A . B (descriptor list, as k_tc_cgemm) with both operands packed:
// A of descriptor d, sub-batch s, 128-row tile tm at d.Ap + s * d.a_pk_sub + tm * d.a_nkc * TC_PACK_FLOATS;
// B' of (s, n-tile tn) at d.Bp + (s * tiles_n + tn) * nkc * BP_FLOATS.  The epilogue undoes the operand
// scales and folds max |C| into d.cmax (the consumer's scale).
template <int BN, int NS>
__global__ void __launch_bounds__(PK_THREADS) k_pk_cgemm(const GemmDesc* __restrict__ descs, int maxtiles, int maxsub, int total) {
  using Cfg = PkCfg<BN, NS>;
  extern __shared__ __align__(1024) uint8_t pksm[];
  __shared__ __align__(8) uint64_t bar[Cfg::NBAR];
  __shared__ uint32_t tslot;
  const uint32_t tmem = pk_setup<BN, NS>(bar, &tslot);
  const int ntiles = total > (int)blockIdx.x ? (total - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
  auto geom = [&](int i, const GemmDesc*& d, int& sub, int& m0, int& n0) -> bool {
    const int t = blockIdx.x + i * gridDim.x;
    const int x = t % maxtiles;
    sub = (t / maxtiles) % maxsub;
    d = descs + t / (maxtiles * maxsub);
    if (sub >= d->batch) return false;
    const int tiles_m = (d->m + TC_BM - 1) / TC_BM, tiles_n = (d->n + BN - 1) / BN;
    if (x >= tiles_m * tiles_n) return false;
    m0 = (d->n_fast ? x / tiles_n : x % tiles_m) * TC_BM;
    n0 = (d->n_fast ? x % tiles_n : x / tiles_m) * BN;
    return true;
  };
  auto tile_of = [&](int i) -> PkTile {
    const GemmDesc* d;
    int sub, m0, n0;
    if (!geom(i, d, sub, m0, n0)) return PkTile{nullptr, nullptr, 0};
    const int nkc = (d->k + TC_BK - 1) / TC_BK, tiles_n = (d->n + BN - 1) / BN;
    PkTile t;
    t.apk = d->Ap + (int64_t)sub * d->a_pk_sub + (int64_t)(m0 / TC_BM) * d->a_nkc * TC_PACK_FLOATS;
    t.bpk = d->Bp + (int64_t)sub * d->b_pk_sub + (int64_t)(n0 / BN) * nkc * Cfg::BP_FLOATS;
    t.nk = nkc;
    return t;
  };
  auto epi = [&](int i, float (&acc)[Cfg::NR]) {
    const GemmDesc* d;
    int sub, m0, n0;
    geom(i, d, sub, m0, n0);
    const float sA = (TC_F16 && d->amax) ? tc::f16_scale(*d->amax) : 1.f;
    const float sB = (TC_F16 && d->bmax) ? tc::f16_scale(*d->bmax) : 1.f;
    const float inv = 1.f / (sA * sB);
    const int gm = m0 + (int)threadIdx.x;
    float2* __restrict__ C = d->C + (int64_t)sub * d->sC;
    float cm = 0.f;
    if (gm < d->m) {
      const int64_t crow = c_row(*d, gm);
#pragma unroll
      for (int j = 0; j < BN; ++j) {
        const int gn = n0 + j;
        if (gn < d->n) {
          const float2 v = make_float2(acc[2 * j] * inv, acc[2 * j + 1] * inv);
          C[crow + d->c_sn * (int64_t)gn] = v;
          cm = fmaxf(cm, fmaxf(fabsf(v.x), fabsf(v.y)));
        }
      }
    }
    if (d->cmax) tc::warp_absmax_to(cm, d->cmax);
  };
  pk_run<BN, NS>(ntiles, tile_of, epi, pksm, bar, tmem);
  pk_teardown<BN, NS>(tmem);
}

// ---------------------------------------------------------------- k_pk_conv_z (n3 <= 32)
// The fused z-stage of eq. (5) (a4, a5, a2, a6) with packed operands: per (direction q, 128 lines ij)
// the last restore contraction T_p[ij, kz] = sum_c G_q[c][ij] V_p(c, kz) on the tensor cores, then per
// line the pruned forward z-DFT of W, the Hadamard product and the truncated inverse z-DFT in
// registers.  Packed G of batch-local q at a.Gp + q * a.gp_stride (per m-tile: nkc(p) chunks); packed V
// of direction p at a.Vp + (a.vp_off ? a.vp_off[p] : q * a.vp_stride).
template <int N3, int MODE, int NS>
__global__ void __launch_bounds__(PK_THREADS, 2) k_pk_conv_z(ZArgs a, int nq) {
  constexpr int BN = N3 < 16 ? 16 : N3;
  using Cfg = PkCfg<BN, NS>;
  constexpr int Nz = N3 / 2;
  extern __shared__ __align__(1024) uint8_t pksm[];
  __shared__ __align__(8) uint64_t bar[Cfg::NBAR];
  __shared__ uint32_t tslot;
  const uint32_t tmem = pk_setup<BN, NS>(bar, &tslot);
  const int tiles_m = (int)((a.n12 + TC_BM - 1) / TC_BM);
  const int total = tiles_m * nq;
  const int ntiles = total > (int)blockIdx.x ? (total - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
  const bool shared_a = a.g_stride == 0 && a.gp_stride == 0;
  auto tile_of = [&](int i) -> PkTile {
    int q, mt;
    z_tile(blockIdx.x + i * gridDim.x, tiles_m, nq, shared_a && a.z_blocked, q, mt);
    const int p = a.p0 + q;
    const int k = a.rank_p ? a.rank_p[p] : a.rank;
    const int nkc = (k + TC_BK - 1) / TC_BK;
    PkTile t;
    t.apk = a.Gp + (int64_t)q * a.gp_stride + (int64_t)mt * nkc * TC_PACK_FLOATS;
    t.bpk = a.Vp + (a.vp_off ? a.vp_off[p] : (int64_t)q * a.vp_stride);
    t.nk = nkc;
    return t;
  };
  const float sB0 = (TC_F16 && a.bmax) ? tc::f16_scale(*a.bmax) : 1.f;
  const float sA0 = (TC_F16 && a.amax) ? tc::f16_scale(*a.amax) : 1.f;
  const float inv = 1.f / (sA0 * sB0);
  auto epi = [&](int i, float (&acc)[Cfg::NR]) {
    int q, mt;
    z_tile(blockIdx.x + i * gridDim.x, tiles_m, nq, shared_a && a.z_blocked, q, mt);
    const int64_t ij = (int64_t)mt * TC_BM + threadIdx.x;
    const bool valid = ij < a.n12;
    if constexpr (MODE == Z_RESTORE) {
      if (valid) {
#pragma unroll
        for (int kz = 0; kz < N3; ++kz)
          a.Tout[(int64_t)kz * a.n12 + ij] = make_float2(acc[2 * kz] * inv, acc[2 * kz + 1] * inv);
      }
    } else {
      for (int cc = 0; cc < a.ncomp; ++cc) {   // signature components share the restored line
        float2* Wl = a.W + ((int64_t)q * a.ncomp + cc) * Nz * a.n12 + (valid ? ij : 0);
        float2 f[N3];
#pragma unroll
        for (int z = 0; z < Nz; ++z) f[z] = valid ? Wl[(int64_t)z * a.n12] : make_float2(0.f, 0.f);
        fft_reg<N3, false, true>(f);
#pragma unroll
        for (int kz = 0; kz < N3; ++kz) f[kz] = cmul2(f[kz], make_float2(acc[2 * kz] * inv, acc[2 * kz + 1] * inv));
        fft_reg<N3, true, false>(f);
        if (valid) {
#pragma unroll
          for (int z = 0; z < Nz; ++z) Wl[(int64_t)z * a.n12] = f[z];
        }
      }
    }
  };
  pk_run<BN, NS>(ntiles, tile_of, epi, pksm, bar, tmem);
  pk_teardown<BN, NS>(tmem);
}

// ---------------------------------------------------------------- k_pk_conv_z64 (n3 = 64)
// One tile per (direction, m-tile) with all 64 kz columns: packed V columns ordered [kz even | kz odd]
// (k_pk_pack_b_multi kzperm), so the MMA runs at N = 256 (A_hi x [B_hi ; B_lo]) + 128 and each A chunk
// serves twice the columns of a 32-column pass.  Two epilogue warpgroups (EG = 2) share the tile's 128
// TMEM lanes: group h drains the parity-h half (32 complex kz = 2j + h) and runs its half of the
// decimated z-convolution (32-point forward DFT of the W line, twiddled for h = 1, Hadamard, inverse);
// group 1 hands its twiddled half to group 0 through shared memory and group 0 writes the sum back
// to W.  One CTA per SM (the two 256-column TMEM slots fill TMEM).
// CL = 2 (shared A only, launched with 2-CTA clusters): the two CTAs of a cluster take directions 2 qp and
// 2 qp + 1 of the same m-tile, each streaming half of every A chunk and multicasting it; with an odd
// direction count the last pair's second CTA repeats the first's direction and skips its epilogue.
constexpr int PKW_THREADS = 320;
constexpr int PKW_NS = 10;
template <int NS>
struct PkwCfg {
  using Cfg = PkCfg<64, NS>;
  static constexpr int X_BYTES = TC_BM * 32 * 8;   // group 1 -> group 0 hand-over (32 complex per row)
  static constexpr int SMEM = Cfg::SMEM + X_BYTES;
};

// FC: K-chunks per TMEM flush group (TC_FC; 2 TC_FC = FMMT_ZFC=8 for the long-K shared-A TT-4D stage lets the MMA
// warp run twice as far ahead of the per-tile z-DFT epilogue, at twice the chained truncating adds per group)
template <int MODE, int NS, int CL = 1, int FC = TC_FC>
__global__ void __launch_bounds__(PKW_THREADS, 1) k_pk_conv_z64(ZArgs a, int nq) {
  constexpr int N3 = 64, H = 32, BN = 64;
  using Cfg = PkCfg<BN, NS>;
  extern __shared__ __align__(1024) uint8_t pksm[];
  __shared__ __align__(8) uint64_t bar[Cfg::NBAR];
  __shared__ uint32_t tslot;
  float2* X = reinterpret_cast<float2*>(pksm + Cfg::SMEM);
  const uint32_t tmem = pk_setup<BN, NS, CL, 2>(bar, &tslot);
  const int tiles_m = (int)((a.n12 + TC_BM - 1) / TC_BM);
  const int nqc = (nq + CL - 1) / CL;                    // direction groups (pairs when CL = 2)
  const int total = tiles_m * nqc;
  const int cid = (int)blockIdx.x / CL, ncl = (int)gridDim.x / CL, crank = (int)blockIdx.x % CL;
  const int ntiles = total > cid ? (total - cid + ncl - 1) / ncl : 0;
  const bool shared_a = a.g_stride == 0 && a.gp_stride == 0;
  auto tile_of = [&](int i) -> PkTile {
    int q, mt;
    z_tile(cid + i * ncl, tiles_m, nqc, shared_a && a.z_blocked, q, mt);
    q = min(q * CL + crank, nq - 1);
    const int p = a.p0 + q;
    const int k = a.rank_p ? a.rank_p[p] : a.rank;
    const int nkc = (k + TC_BK - 1) / TC_BK;
    PkTile t;
    t.apk = a.Gp + (int64_t)q * a.gp_stride + (int64_t)mt * nkc * TC_PACK_FLOATS;
    t.bpk = a.Vp + (a.vp_off ? a.vp_off[p] : (int64_t)q * a.vp_stride);
    t.nk = nkc;
    return t;
  };
  const float sB0 = (TC_F16 && a.bmax) ? tc::f16_scale(*a.bmax) : 1.f;
  const float sA0 = (TC_F16 && a.amax) ? tc::f16_scale(*a.amax) : 1.f;
  const float inv = 1.f / (sA0 * sB0);
  auto epi = [&](int i, float (&acc)[Cfg::NR / 2], int h) {
    int q, mt;
    z_tile(cid + i * ncl, tiles_m, nqc, shared_a && a.z_blocked, q, mt);
    q = q * CL + crank;
    if (q >= nq) return;                                 // (CL = 2, odd nq: the ghost half of the last pair)
    const int row = threadIdx.x & (TC_BM - 1);
    const int64_t ij = (int64_t)mt * TC_BM + row;
    const bool valid = ij < a.n12;
    if constexpr (MODE == Z_RESTORE) {
      if (valid) {
#pragma unroll
        for (int m = 0; m < H; ++m)
          a.Tout[(int64_t)(2 * m + h) * a.n12 + ij] = make_float2(acc[2 * m] * inv, acc[2 * m + 1] * inv);
      }
    } else {
      for (int cc = 0; cc < a.ncomp; ++cc) {
        float2* Wl = a.W + ((int64_t)q * a.ncomp + cc) * H * a.n12 + (valid ? ij : 0);
        float2 f[H];
#pragma unroll
        for (int z = 0; z < H; ++z) f[z] = valid ? Wl[(int64_t)z * a.n12] : make_float2(0.f, 0.f);
        if (h) {
#pragma unroll
          for (int z = 1; z < H; ++z) f[z] = cmul(f[z], twc<N3, false>(z));
        }
        fft_reg<H, false, false>(f);
#pragma unroll
        for (int m = 0; m < H; ++m) f[m] = cmul2(f[m], make_float2(acc[2 * m] * inv, acc[2 * m + 1] * inv));
        fft_reg<H, true, false>(f);
        if (h) {
#pragma unroll
          for (int z = 0; z < H; ++z) X[z * TC_BM + row] = z ? cmul(f[z], twc<N3, true>(z)) : f[z];
        }
        tc::named_bar_sync(1, 256);                      // the odd half is in X (and both groups read W)
        if (!h && valid) {
#pragma unroll
          for (int z = 0; z < H; ++z) Wl[(int64_t)z * a.n12] = cadd(f[z], X[z * TC_BM + row]);
        }
        tc::named_bar_sync(1, 256);                      // X free for the next component / tile
      }
    }
  };
  pk_run<BN, NS, decltype(tile_of), decltype(epi), CL, 2, FC>(ntiles, tile_of, epi, pksm, bar, tmem);
  pk_teardown<BN, NS, CL, 2>(tmem);
}

// ---------------------------------------------------------------- multi-operand packs
// Pack the A operand of every descriptor of a list (blockIdx.y = descriptor), all sub-batches, into
// its d.Ap (sub-batch s at d.Ap + s * d.a_pk_sub), as k_tc_pack_a; the scale from *d.amax.  One item =
// one row and four consecutive complex K (16 B of hi, 16 B of lo in the fp16 layout: one core-matrix
// row), threads ordered along the operand's contiguous index so loads coalesce and each warp's
// stores cover whole 16-byte core rows.
__global__ void k_pk_pack_a_multi(const GemmDesc* __restrict__ descs) {
  const GemmDesc& d = descs[blockIdx.y];
  const int nkc = (d.k + TC_BK - 1) / TC_BK;
  const int64_t tiles_m = (d.m + TC_BM - 1) / TC_BM;
  constexpr int KQ = TC_BK / 4;                              // 4-complex groups per chunk
  const int64_t per = tiles_m * TC_BM * nkc * KQ;
  const int64_t total = per * d.batch;
  const float s = (TC_F16 && d.amax) ? tc::f16_scale(*d.amax) : 1.f;
  float* out = const_cast<float*>(d.Ap);
  const bool kfast = d.a_sk == 1 && d.a_s0 != 1;   // K contiguous in memory: K groups fastest
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t sub = e / per;
    int64_t t = e - sub * per;
    int r, kq;
    if (kfast) {
      kq = (int)(t % KQ);
      t /= KQ;
      r = (int)(t % TC_BM);
      t /= TC_BM;
    } else {
      r = (int)(t % TC_BM);
      t /= TC_BM;
      kq = (int)(t % KQ);
      t /= KQ;
    }
    const int kc = (int)(t % nkc);
    const int64_t tm = t / nkc;
    const int gm = (int)(tm * TC_BM + r);
    const int gk = kc * TC_BK + 4 * kq;
    const float2* A = d.A + sub * d.sA;
    float2 a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) a[u] = make_float2(0.f, 0.f);
    if (gm < d.m) {
      const int64_t row = a_row(d, gm);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (gk + u < d.k) a[u] = A[row + (int64_t)(gk + u) * d.a_sk];
    }
    uint8_t* tile = reinterpret_cast<uint8_t*>(out + sub * d.a_pk_sub + (tm * nkc + kc) * TC_PACK_FLOATS);
    if constexpr (TC_F16) {
      uint4 hi, lo;
      tc::split_f16x2(a[0].x * s, a[0].y * s, hi.x, lo.x);
      tc::split_f16x2(a[1].x * s, a[1].y * s, hi.y, lo.y);
      tc::split_f16x2(a[2].x * s, a[2].y * s, hi.z, lo.z);
      tc::split_f16x2(a[3].x * s, a[3].y * s, hi.w, lo.w);
      const int off = r * 16 + kq * (TC_BM * 16);          // 4 complex = 8 halves = one core-matrix row
      *reinterpret_cast<uint4*>(tile + off) = hi;
      *reinterpret_cast<uint4*>(tile + TC_PACK_FLOATS * 2 + off) = lo;
    } else {
#pragma unroll
      for (int h = 0; h < 2; ++h) {                        // tf32: 2 complex per 16-byte core row
        float4 hi, lo;
        tc::split_tf32(a[2 * h].x, hi.x, lo.x);
        tc::split_tf32(a[2 * h].y, hi.y, lo.y);
        tc::split_tf32(a[2 * h + 1].x, hi.z, lo.z);
        tc::split_tf32(a[2 * h + 1].y, hi.w, lo.w);
        const int off = r * 16 + (2 * kq + h) * (TC_BM * 16);
        *reinterpret_cast<float4*>(tile + off) = hi;
        *reinterpret_cast<float4*>(tile + TC_PACK_FLOATS * 2 + off) = lo;
      }
    }
  }
}

// B operands of a list (blockIdx.y = item): B(l, j) = B[l * b_sk + j * b_sn], l < k, j < n, packed as
// k_tc_pack_b<BN> (one n-tile per BN columns) into out; scale from *bmax.
struct PkB {
  const float2* B;
  int64_t b_sk, b_sn;
  int k, n;
  float* out;
  const float* bmax;
  int kzperm = 0;   // 1 (n = 64 z-stage V): column j holds kz = 2 (j % 32) + j / 32, i.e. [kz even | kz odd]
};

template <int BN>
__global__ void k_pk_pack_b_multi(const PkB* __restrict__ items, const float* __restrict__ bmax_all) {
  using Cfg = TcGemmCfg<BN, 1>;
  constexpr int NR = Cfg::NR;
  const PkB& it = items[blockIdx.y];
  const int nkc = (it.k + TC_BK - 1) / TC_BK;
  const int tiles_n = (it.n + BN - 1) / BN;
  const int64_t total = (int64_t)tiles_n * nkc * BN * (TC_BK / 2);
  const float* bm = bmax_all ? bmax_all : it.bmax;   // (a per-launch scale slot overrides the items')
  const float s = (TC_F16 && bm) ? tc::f16_scale(*bm) : 1.f;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(e % BN);
    int64_t t = e / BN;
    const int kp = (int)(t % (TC_BK / 2));
    t /= (TC_BK / 2);
    const int kc = (int)(t % nkc);
    const int tn = (int)(t / nkc);
    const int gn = tn * BN + j, gk = kc * TC_BK + 2 * kp;
    float2 b0 = make_float2(0.f, 0.f), b1 = make_float2(0.f, 0.f);
    if (gn < it.n) {
      const int col = it.kzperm ? 2 * (gn & 31) + (gn >> 5) : gn;
      const float2* Bq = it.B + (int64_t)col * it.b_sn;
      if (gk < it.k) b0 = Bq[(int64_t)gk * it.b_sk];
      if (gk + 1 < it.k) b1 = Bq[(int64_t)(gk + 1) * it.b_sk];
    }
    uint8_t* blk = reinterpret_cast<uint8_t*>(it.out + ((int64_t)tn * nkc + kc) * Cfg::BP_FLOATS);
    if constexpr (TC_F16) {
      uint2 h0, l0, h1, l1;
      tc::split_f16x2(b0.x * s, -b0.y * s, h0.x, l0.x);
      tc::split_f16x2(b1.x * s, -b1.y * s, h0.y, l0.y);
      tc::split_f16x2(b0.y * s, b0.x * s, h1.x, l1.x);
      tc::split_f16x2(b1.y * s, b1.x * s, h1.y, l1.y);
      const int off = (2 * j) * 16 + (kp >> 1) * Cfg::LBO_B + (kp & 1) * 8;
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
      const int off = (2 * j) * 16 + kp * Cfg::LBO_B;
      *reinterpret_cast<float4*>(blk + off) = h0;
      *reinterpret_cast<float4*>(blk + off + 16) = h1;
      *reinterpret_cast<float4*>(blk + off + NR * 16) = l0;
      *reinterpret_cast<float4*>(blk + off + NR * 16 + 16) = l1;
    }
  }
}

}  // namespace fmmt
