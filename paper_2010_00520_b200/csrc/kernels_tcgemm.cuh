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
constexpr int TC_NS = 4;        // operand ring stages: copies run 2 chunks ahead, MMAs of chunk k-1 overlap
                                // the conversion of chunk k
constexpr int TC_PACK_FLOATS = 2 * TC_BM * 2 * TC_BK * TC_ESZ / 4;   // one packed A chunk (hi + lo), in floats
// chunks per TMEM flush group = MMAs chained into one accumulator before it is drained to FP32
// registers: tf32 4 K-steps (8 failed the 1e-6 restore bar), f16 FMMT_TC_FC16 K-steps
constexpr int TC_FC = TC_F16 ? FMMT_TC_FC16 : 2;

template <int BN, int G = 1>
struct TcGemmCfg {
  static constexpr int NT = 128 * G;                // threads
  static constexpr int NR = 2 * BN;                 // real N of C (re, im interleaved)
  static constexpr int NRG = NR / G;                // real columns per thread group
  static constexpr int KR = 2 * TC_BK;              // real K per chunk
  static constexpr int A_BYTES = TC_BM * KR * TC_ESZ;   // one of hi / lo
  static constexpr int BP_ROWS = 2 * NR;            // B' = [B^_hi ; B^_lo]
  static constexpr int BP_BYTES = BP_ROWS * KR * TC_ESZ;
  static constexpr int BP_FLOATS = BP_BYTES / 4;      // one pre-split B' chunk (k_tc_pack_b), in floats
  static constexpr int BITEMS = BN * (TC_BK / 2) / NT > 0 ? BN * (TC_BK / 2) / NT : 1;
  static constexpr int BRAW = BITEMS * NT * 16;     // raw B staging
  static constexpr int ARAW = TC_F16 ? TC_BM * KR * 4 : 0;   // raw FP32 A staging (f16: split out of place)
  static constexpr int STAGE = 2 * A_BYTES + BP_BYTES + ARAW + BRAW;
  static constexpr int SMEM = TC_NS * STAGE;
  // two accumulator slots (alternating K-chunks) x {hi.hi, hi.lo + lo.hi}
  static constexpr int TMEM_COLS = 4 * NR < 32 ? 32 : 4 * NR;
  static constexpr uint32_t LBO_A = TC_BM * 16;     // K-adjacent core matrices
  static constexpr uint32_t LBO_B = BP_ROWS * 16;
  static_assert(2 * NR <= 256, "UMMA N <= 256");
  static_assert(NRG % 16 == 0, "TMEM drain granularity: 16 columns per thread group");
  static_assert(TC_BK == 8, "copy mappings below assume 4 complex pairs per row and chunk");
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
struct TcCursor {
  int c = 0;   // chunks issued by this CTA so far
  int g = 0;   // TMEM flush groups used by this CTA so far
};

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

// acc[NRG] (registers; thread = row m0 + tid % 128, columns [g NRG, (g+1) NRG) of
// the tile, re/im interleaved) = A[m0:m0+128, :] . B[:, n0:n0+BN] over all of K.
// Called by all 128 G threads.  bar[0..1]: MMA commits per stage; bar[2..3]:
// packed-A bulk copies per stage.
// Per-CTA pipeline position, continued across calls (several tiles per CTA, two passes of the
// n3 = 64 z-stage): c = chunks issued so far (ring stage c % NS, barrier phase (c / NS) & 1,
// exact - a gap would desynchronise the per-stage barrier phases), g = TMEM flush groups so far
// (slot g & 1, tfree phase (g / 2) & 1; every call starts a fresh group).
template <int BN, int G>
__device__ __forceinline__ void tc_mainloop(const GemmDesc& d, const float2* __restrict__ A,
                                           const float2* __restrict__ B, int m0, int n0, uint8_t* tcsm,
                                           uint64_t* bar, uint32_t tmem,
                                           float (&acc)[TcGemmCfg<BN, G>::NRG], TcCursor& cur, float sA = 1.f,
                                           float sB = 1.f) {
  using Cfg = TcGemmCfg<BN, G>;
  constexpr int BM = TC_BM, BK = TC_BK, NR = Cfg::NR, NRG = Cfg::NRG, NT = Cfg::NT;
  constexpr int BITEMS = Cfg::BITEMS;
  const uint32_t sbase = tc::smem_u32(tcsm);
  const int tid = threadIdx.x, row = tid & 127, grp = tid >> 7;
  const int wrow = row >> 5, lane = tid & 31;      // warp index within the group = TMEM lane quarter
  const bool a_kcontig = d.a_sk == 1;   // rows of A are contiguous in K
  const bool b_kcontig = d.b_sk == 1;
  // rows this thread copies: row-per-thread (row) or K-contiguous (4 rows)
  int64_t arow[4];
  bool okrow[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int r = a_kcontig ? (lane & 7) + 8 * (u + 4 * wrow) : row;
    okrow[u] = m0 + r < d.m;
    arow[u] = okrow[u] ? a_row(d, m0 + r) : 0;
  }
  constexpr uint32_t IDESC_BP = TC_F16 ? tc::idesc_f16(BM, 2 * NR) : tc::idesc_tf32(BM, 2 * NR);   // A_hi x [B_hi ; B_lo]
  constexpr uint32_t IDESC_B = TC_F16 ? tc::idesc_f16(BM, NR) : tc::idesc_tf32(BM, NR);            // A_lo x B_hi
#pragma unroll
  for (int j = 0; j < NRG; ++j) acc[j] = 0.f;
  const uint32_t twarp = tmem + ((uint32_t)(wrow * 32) << 16);   // this warp's TMEM lanes
  const int c0 = grp * NRG;                                      // this group's columns

  // warp-uniform copies (the MMA-issuing warp 0 keeps its operands in uniform registers)
  const int nk = __shfl_sync(0xffffffffu, (d.k + BK - 1) / BK, 0);
  const int cur_c = __shfl_sync(0xffffffffu, cur.c, 0), cur_g = __shfl_sync(0xffffffffu, cur.g, 0);
  const int warp_u = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const uint32_t sbase_u = __shfl_sync(0xffffffffu, sbase, 0);
  const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem, 0);
  const uint32_t bar_u = __shfl_sync(0xffffffffu, tc::smem_u32(bar), 0);
  const uint64_t dAh = tc::sdesc(sbase_u, Cfg::LBO_A, 128), dAl = tc::sdesc(sbase_u + Cfg::A_BYTES, Cfg::LBO_A, 128);
  const uint64_t dBp = tc::sdesc(sbase_u + 2 * Cfg::A_BYTES, Cfg::LBO_B, 128);
  const bool apack = d.Ap != nullptr;   // A pre-split into hi/lo tiles: one bulk copy per chunk
  const bool bpack = d.Bp != nullptr;   // B pre-split into B' chunks: one bulk copy per chunk
  const bool both_u = __shfl_sync(0xffffffffu, (int)(apack && bpack), 0);   // no per-thread operand work
  const float* apk = apack ? d.Ap + (int64_t)(m0 / BM) * d.a_nkc * TC_PACK_FLOATS : nullptr;
  // raw A lands in the canonical (TF32-layout) A_hi tile for the in-place tf32 split, in a staging
  // area for the out-of-place fp16 split; raw B always in its staging area
  constexpr int AR_OFF = TC_F16 ? 2 * Cfg::A_BYTES + Cfg::BP_BYTES : 0;
  constexpr int BR_OFF = 2 * Cfg::A_BYTES + Cfg::BP_BYTES + Cfg::ARAW;
  constexpr uint32_t LBO_AR = TC_BM * 16;   // raw FP32 A: K-adjacent 4-element groups
  // copies of chunk c into stage c % NS
  auto issue = [&](int c) {
    const int k0 = c * BK;
    const int cs = (cur.c + c) % TC_NS;
    const uint32_t st = sbase + cs * Cfg::STAGE;
    if ((apack || bpack) && tid == 0) {   // pre-split operands: bulk async copies on one transaction barrier
      tc::mbar_expect_tx(&bar[TC_NS + cs], (apack ? 2 * Cfg::A_BYTES : 0) + (bpack ? Cfg::BP_BYTES : 0));
      if (apack) tc::bulk_g2s(st, apk + (int64_t)c * TC_PACK_FLOATS, 2 * Cfg::A_BYTES, &bar[TC_NS + cs]);
      if (bpack)
        tc::bulk_g2s(st + 2 * Cfg::A_BYTES, d.Bp + (int64_t)c * Cfg::BP_FLOATS, Cfg::BP_BYTES, &bar[TC_NS + cs]);
    }
    if (apack) {
    } else if (!a_kcontig) {
      // row-per-thread: group g copies K elements [g BK/G, (g+1) BK/G) of its row
#pragma unroll
      for (int kq = 0; kq < BK / G; ++kq) {
        const int kk = grp * (BK / G) + kq;
        const int gk = k0 + kk;
        const bool ok = okrow[0] && gk < d.k;
        tc::cp_async8(st + AR_OFF + row * 16 + (kk >> 1) * LBO_AR + (kk & 1) * 8,
                      ok ? (const void*)(A + arow[0] + gk * d.a_sk) : (const void*)A, ok);
      }
    } else {
      // K-contiguous rows: lane -> (row low 3 bits, complex pair kp = lane / 8); item u = 0..3 -> row
      // group (u + 4 * warp); thread group g takes items u % G == g
#pragma unroll
      for (int uu = 0; uu < 4 / G; ++uu) {
        const int u = uu * G + grp;
        const int kp = lane >> 3;
        const int r = (lane & 7) + 8 * (u + 4 * wrow);
        const int gk = k0 + 2 * kp;
        const bool okr = (G == 1) ? okrow[uu] : (grp ? okrow[2 * uu + 1] : okrow[2 * uu]);
        const int64_t ar = (G == 1) ? arow[uu] : (grp ? arow[2 * uu + 1] : arow[2 * uu]);
        const bool ok0 = okr && gk < d.k, ok1 = okr && gk + 1 < d.k;
        const uint32_t dst = st + AR_OFF + r * 16 + kp * LBO_AR;
        tc::cp_async8(dst, ok0 ? (const void*)(A + ar + gk) : (const void*)A, ok0);
        tc::cp_async8(dst + 8, ok1 ? (const void*)(A + ar + gk + 1) : (const void*)A, ok1);
      }
    }
    const uint32_t rb = st + BR_OFF;
#pragma unroll
    for (int i = 0; i < BITEMS; ++i) {
      if (bpack) break;
      const int idx = tid + NT * i;
      int j, kp;
      if (!b_kcontig) { j = idx % BN; kp = idx / BN; }    // n (not k) contiguous in memory
      else { kp = idx % (BK / 2); j = idx / (BK / 2); }   // k contiguous
      const int gn = n0 + j, gk = k0 + 2 * kp;
      const bool okn = idx < BN * (BK / 2) && gn < d.n;
      const int gc = d.b_eo ? (gn < d.n / 2 ? 2 * gn : 2 * (gn - d.n / 2) + 1) : gn;   // even/odd column order
      const bool ok0 = okn && gk < d.k, ok1 = okn && gk + 1 < d.k;
      const uint32_t dst = rb + (i * NT + tid) * 16;
      tc::cp_async8(dst, ok0 ? (const void*)(B + gk * d.b_sk + gc * d.b_sn) : (const void*)B, ok0);
      tc::cp_async8(dst + 8, ok1 ? (const void*)(B + (gk + 1) * d.b_sk + gc * d.b_sn) : (const void*)B, ok1);
    }
    tc::cp_async_commit();
  };

  // Barrier-free pipeline (no __syncthreads in the K loop).  Every thread converts exactly the
  // shared-memory segments its own cp.async copied, fences them for the async proxy and arrives
  // on full[s]; warp 0 waits for the 128 arrivals, issues the chunk's MMAs and commits them to
  // mma[s]; a stage is refilled once mma[s] completed; TMEM slots are handed back through tfree.
  //   bar[0, NS) mma commits   bar[NS, 2NS) packed-A bulk copies   bar[2NS, 3NS) full (128)
  //   bar[3NS, 3NS+2) tfree (128), one per TMEM slot
  // Chunk c: stage c % NS, phase (c / NS) & 1; flush group g = c / FC: slot g & 1, phase (g / 2) & 1.
  static_assert(G == 1, "own-segment conversion mapping assumes one thread group");
  uint64_t* mmab = bar;
  uint64_t* abar = bar + TC_NS;
  uint64_t* full = bar + 2 * TC_NS;
  uint64_t* tfree = bar + 3 * TC_NS;
  int flushed = 0;                       // this call's flush groups already drained into acc
  auto drain_complete = [&](int done) {  // this call's chunks [0, done) have completed MMAs
    for (; (flushed + 1) * TC_FC <= done; ++flushed) {
      const int gid = cur.g + flushed;
      tc_flush<NR, NRG>(twarp + (gid & 1) * 2 * NR, c0, acc);
      tc::fence_before_sync();
      tc::mbar_arrive(&tfree[gid & 1]);
    }
  };
  constexpr int D = TC_NS - 2;           // copy prefetch distance (chunks)
#pragma unroll
  for (int c = 0; c < D; ++c) {
    if (c < nk) issue(c);
    else tc::cp_async_commit();
  }
  for (int kc = 0; kc < nk; ++kc) {
    const int gc = cur.c + kc;             // CTA-wide chunk number (stage, barrier phases)
    const int s = gc % TC_NS;
    const uint32_t ph = (gc / TC_NS) & 1;
    if (kc >= 2) {
      // MMAs of chunk kc-2 (and earlier) complete: stage (kc+2) % NS is free, closed groups drain
      // (for kc < 2 the stages were last used by a previous call, whose MMAs all completed)
      tc::mbar_wait(&mmab[(gc - 2) % TC_NS], ((gc - 2) / TC_NS) & 1);
      tc::fence_after_sync();
      drain_complete(kc - 1);
    }
    if (kc + D < nk) issue(kc + D);
    else tc::cp_async_commit();          // keep one group per iteration
    tc::cp_async_wait<D>();              // this thread's copies of chunk kc have landed
    if (apack || bpack) tc::mbar_wait(&abar[s], ph);
    uint8_t* st = tcsm + s * Cfg::STAGE;
    uint8_t* aHi = st;
    uint8_t* aLo = st + Cfg::A_BYTES;
    uint8_t* bP = st + 2 * Cfg::A_BYTES;
    const uint8_t* aRaw = st + AR_OFF;
    const uint8_t* bRaw = st + BR_OFF;
    // ---- split this thread's A segments: A_hi = rn(x), A_lo = rn(x - A_hi).  Round-to-nearest on
    //      both parts keeps |x - hi - lo| and the dropped lo.lo product at 2^-22 |x| (a truncated hi
    //      doubles both: measured restore errors up to 1.02e-6 against the 1e-6 bar).
    if (!apack) {
#pragma unroll
      for (int u = 0; u < BK / 2; ++u) {
        const int r = a_kcontig ? (lane & 7) + 8 * (u + 4 * wrow) : row;
        const int kp = a_kcontig ? (lane >> 3) : u;      // complex pair = reals [4 kp, 4 kp + 4)
        const float4 a = *reinterpret_cast<const float4*>(aRaw + r * 16 + kp * LBO_AR);
        if constexpr (TC_F16) {
          uint2 hi, lo;
          tc::split_f16x2(a.x * sA, a.y * sA, hi.x, lo.x);
          tc::split_f16x2(a.z * sA, a.w * sA, hi.y, lo.y);
          const uint32_t off = r * 16 + (kp >> 1) * Cfg::LBO_A + (kp & 1) * 8;
          *reinterpret_cast<uint2*>(aHi + off) = hi;
          *reinterpret_cast<uint2*>(aLo + off) = lo;
        } else {
          const uint32_t off = r * 16 + kp * Cfg::LBO_A;
          float4 hi, lo;
          tc::split_tf32(a.x, hi.x, lo.x);
          tc::split_tf32(a.y, hi.y, lo.y);
          tc::split_tf32(a.z, hi.z, lo.z);
          tc::split_tf32(a.w, hi.w, lo.w);
          *reinterpret_cast<float4*>(aHi + off) = hi;
          *reinterpret_cast<float4*>(aLo + off) = lo;
        }
      }
    }
    // ---- B' rows: [0, NR) = B^_hi, [NR, 2NR) = B^_lo;  row 2j = [Re b, -Im b], row 2j+1 = [Im b, Re b]
#pragma unroll
    for (int i = 0; i < BITEMS; ++i) {
      const int idx = tid + NT * i;
      if (bpack || idx >= BN * (BK / 2)) continue;
      int j, kp;
      if (!b_kcontig) { j = idx % BN; kp = idx / BN; }
      else { kp = idx % (BK / 2); j = idx / (BK / 2); }
      const float4 bb = *reinterpret_cast<const float4*>(bRaw + (i * NT + tid) * 16);
      if constexpr (TC_F16) {
        uint2 h0, l0, h1, l1;
        tc::split_f16x2(bb.x * sB, -bb.y * sB, h0.x, l0.x);
        tc::split_f16x2(bb.z * sB, -bb.w * sB, h0.y, l0.y);
        tc::split_f16x2(bb.y * sB, bb.x * sB, h1.x, l1.x);
        tc::split_f16x2(bb.w * sB, bb.z * sB, h1.y, l1.y);
        const uint32_t off = (2 * j) * 16 + (kp >> 1) * Cfg::LBO_B + (kp & 1) * 8;
        *reinterpret_cast<uint2*>(bP + off) = h0;
        *reinterpret_cast<uint2*>(bP + off + 16) = h1;
        *reinterpret_cast<uint2*>(bP + off + NR * 16) = l0;
        *reinterpret_cast<uint2*>(bP + off + NR * 16 + 16) = l1;
      } else {
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
    }
    if (!both_u) tc::fence_async_smem();              // this thread's converted operands -> async proxy
    // every thread arrives, also with two pre-split operands (nothing converted): the full[] barrier
    // keeps warp 0 from running more than one chunk ahead of the slowest warp, which the abar /
    // mmab parity waits need (a lead of NS chunks would alias their phases)
    tc::mbar_arrive(&full[s]);
    if (warp_u == 0) {                                // warp 0 issues; one elected lane per tcgen05 op
      __syncwarp();
      const int gcu = cur_c + kc;
      const int su = gcu % TC_NS;
      tc::mbar_wait_addr(bar_u + (2 * TC_NS + su) * 8, (gcu / TC_NS) & 1);   // chunk kc's operands in place
      const int g = cur_g + kc / TC_FC;               // CTA-wide flush group (TMEM slot, tfree phase)
      const bool fresh = kc % TC_FC == 0;             // first chunk of a flush group
      if (fresh && g >= 2) tc::mbar_wait_addr(bar_u + (3 * TC_NS + (g & 1)) * 8, ((g >> 1) - 1) & 1);   // g-2 drained
      __syncwarp();
      tc::fence_after_sync();
      const uint64_t so = (uint64_t)((su * Cfg::STAGE) >> 4);   // descriptor start-address units
      const uint32_t tm = tmem_u + (g & 1) * 2 * NR, tx = tm + NR;
#pragma unroll
      for (int ks = 0; ks < Cfg::KR / TC_KSTEP; ++ks) {   // one K-step = two K-adjacent core matrices
        const uint64_t oa = so + ((ks * 2 * Cfg::LBO_A) >> 4), ob = so + ((ks * 2 * Cfg::LBO_B) >> 4);
        if constexpr (TC_F16) {
          tc::mma_f16_el(tm, dAh + oa, dBp + ob, IDESC_BP, !(fresh && ks == 0));   // [hi.hi | hi.lo]
          tc::mma_f16_el(tx, dAl + oa, dBp + ob, IDESC_B, 1);                       // += lo.hi (rows [0, NR))
        } else {
          tc::mma_tf32_el(tm, dAh + oa, dBp + ob, IDESC_BP, !(fresh && ks == 0));   // [hi.hi | hi.lo]
          tc::mma_tf32_el(tx, dAl + oa, dBp + ob, IDESC_B, 1);                       // += lo.hi (rows [0, NR))
        }
      }
      tc::mma_commit_el(bar_u + su * 8);              // -> mmab[su]
    }
  }
  tc::cp_async_wait<0>();
  // drain the remaining flush groups (the last one possibly partial)
  tc::mbar_wait(&mmab[(cur.c + nk - 1) % TC_NS], ((cur.c + nk - 1) / TC_NS) & 1);
  tc::fence_after_sync();
  drain_complete(nk);
  if (flushed * TC_FC < nk) {                        // the last, partial group
    const int gid = cur.g + flushed;
    tc_flush<NR, NRG>(twarp + (gid & 1) * 2 * NR, c0, acc);
    tc::fence_before_sync();
    tc::mbar_arrive(&tfree[gid & 1]);                // (keeps tfree phases aligned for a next call)
    ++flushed;
  }
  cur.c += nk;
  cur.g += flushed;
  if constexpr (TC_F16) {                            // undo the operand scales (exact: powers of two)
    const float inv = 1.f / (sA * sB);
#pragma unroll
    for (int j = 0; j < NRG; ++j) acc[j] *= inv;
  }
}

// TMEM allocation + stage barriers (all threads call; warp 0 allocates).
template <int TMEM_COLS>
__device__ __forceinline__ uint32_t tc_setup(uint64_t* bar, uint32_t* tslot) {
  if ((threadIdx.x >> 5) == 0) tc::tmem_alloc<TMEM_COLS>(tslot);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < 2 * TC_NS; ++i) tc::mbar_init(&bar[i], 1);      // MMA commits, bulk copies
#pragma unroll
    for (int i = 2 * TC_NS; i < 3 * TC_NS + 2; ++i) tc::mbar_init(&bar[i], 128);   // full, tfree
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

// A CTA walks the launch's tiles t = blockIdx.x, blockIdx.x + gridDim.x, ... (flattened over
// (tile, sub-batch, descriptor)), reusing its TMEM allocation and barriers; the chunk numbering
// continues across tiles (TcCursor), so the ring and the TMEM slots stay consistent.
template <int BN, int G>
__global__ void __launch_bounds__(128 * G) k_tc_cgemm(const GemmDesc* __restrict__ descs, int maxtiles, int maxsub,
                                                      int total) {
  using Cfg = TcGemmCfg<BN, G>;
  constexpr int BM = TC_BM, NRG = Cfg::NRG;
  extern __shared__ __align__(1024) uint8_t tcsm[];
  __shared__ __align__(8) uint64_t bar[3 * TC_NS + 2];
  __shared__ uint32_t tslot;

  const uint32_t tmem = tc_setup<Cfg::TMEM_COLS>(bar, &tslot);
  TcCursor cur;
  for (int t = blockIdx.x; t < total; t += gridDim.x) {
    const int x = t % maxtiles;
    const int sub = (t / maxtiles) % maxsub;
    GemmDesc d = descs[t / (maxtiles * maxsub)];
    if (sub >= d.batch) continue;                      // uniform over the CTA
    const int tiles_m = (d.m + BM - 1) / BM;
    const int tiles_n = (d.n + BN - 1) / BN;
    if (x >= tiles_m * tiles_n) continue;
    const int m0 = (d.n_fast ? x / tiles_n : x % tiles_m) * BM;
    const int n0 = (d.n_fast ? x % tiles_n : x / tiles_m) * BN;
    if (d.Bp)   // pre-split B (k_tc_pack_b<BN>): this tile's chunks
      d.Bp += ((int64_t)sub * tiles_n + n0 / BN) * ((d.k + TC_BK - 1) / TC_BK) * Cfg::BP_FLOATS;
    const float2* __restrict__ A = d.A + (int64_t)sub * d.sA;
    const float2* __restrict__ B = d.B + (int64_t)sub * d.sB;
    float2* __restrict__ C = d.C + (int64_t)sub * d.sC;
    float acc[NRG];
    const float sA = (TC_F16 && d.amax) ? tc::f16_scale(*d.amax) : 1.f;
    const float sB = (TC_F16 && d.bmax) ? tc::f16_scale(*d.bmax) : 1.f;
    tc_mainloop<BN, G>(d, A, B, m0, n0, tcsm, bar, tmem, acc, cur, sA, sB);
    const int gm = m0 + (threadIdx.x & 127);
    const int nb = n0 + (threadIdx.x >> 7) * (BN / G);
    float cm = 0.f;
    if (gm < d.m) {
      const int64_t crow = c_row(d, gm);
#pragma unroll
      for (int j = 0; j < BN / G; ++j) {
        const int gn = nb + j;
        if (gn < d.n) {
          C[crow + d.c_sn * (int64_t)gn] = make_float2(acc[2 * j], acc[2 * j + 1]);
          cm = fmaxf(cm, fmaxf(fabsf(acc[2 * j]), fabsf(acc[2 * j + 1])));
        }
      }
    }
    if (d.cmax) tc::warp_absmax_to(cm, d.cmax);   // operand scale of the consumer of C
  }
  tc_teardown<Cfg::TMEM_COLS>(tmem);
}

// ---------------------------------------------------------------- k_tc_conv_z
// Tensor-core version of k_conv_z (kernels_fft.cuh) for n3 <= 32: per batch
// directions q0 .. q0+ND-1 and 128 (kx,ky) lines ij, the last restore contraction
//     T_p[ij, kz] = sum_c G_q[c][ij] V_p(c, kz)        (a4: x3 U3 / TT tail)
// runs on tcgen05 (3xTF32); the thread(s) owning line ij then do, per
// direction, the pruned forward z-DFT of the half-padded spectrum W, the
// Hadamard product with T_p (a5) and the inverse z-DFT truncated to z < Nz
// (a6), in registers.  T_p never leaves the SM.
//   The ncomp signature components of a direction share the restored line.
//   ND > 1 only when G is shared by all directions (TT-4D: G = T1 of Fig. 4(b))
//   and V_q is laid out [q][kz][c] (one tile's B = ND directions side by side).
template <int N3, int MODE, int ND, int G>
__global__ void __launch_bounds__(128 * G, 1) k_tc_conv_z(ZArgs a, int nq) {
  constexpr int BN0 = N3 * ND;
  constexpr int BN = BN0 < 16 ? 16 : BN0;
  using Cfg = TcGemmCfg<BN, G>;
  constexpr int Nz = N3 / 2;
  static_assert(ND == 1 || MODE != Z_RESTORE, "restore hook is per direction");
  static_assert(G == 1, "one thread group (thread = line ij)");
  extern __shared__ __align__(1024) uint8_t tcsm[];
  __shared__ __align__(8) uint64_t bar[3 * TC_NS + 2];
  __shared__ uint32_t tslot;

  const int tiles_m = (int)((a.n12 + TC_BM - 1) / TC_BM);
  const int total = tiles_m * ((nq + ND - 1) / ND);
  const int row = threadIdx.x & 127;
  const uint32_t tmem = tc_setup<Cfg::TMEM_COLS>(bar, &tslot);
  TcCursor cur;
  // tiles t = (m-tile, direction group), walked by this CTA with one TMEM allocation
  for (int t = blockIdx.x; t < total; t += gridDim.x) {
    int qg, mt;
    z_tile(t, tiles_m, (nq + ND - 1) / ND, ND == 1 && a.z_blocked, qg, mt);
    const int q0 = qg * ND;
    const int p0 = a.p0 + q0;
    const int nd = min(ND, nq - q0);
    const int m0 = mt * TC_BM;
    GemmDesc d;
    d.m = (int)a.n12;
    d.n = nd * N3;
    d.k = a.rank_p ? a.rank_p[p0] : a.rank;
    d.batch = 1;
    d.a_s0 = 1; d.a_s1 = 0; d.a_div = 1 << 30; d.a_sk = a.n12;
    d.b_sk = a.v_sc; d.b_sn = a.v_sk;     // ND > 1: v_stride == N3 * v_sk (checked on the host)
    d.b_eo = 0;
    d.c_s0 = 0; d.c_s1 = 0; d.c_div = 1; d.c_sn = 0;
    d.sA = d.sB = d.sC = 0;
    d.Ap = a.Gp;                          // pre-split shared G (TT-4D T1), or nullptr
    d.a_nkc = (d.k + TC_BK - 1) / TC_BK;
    d.Bp = (ND == 1 && a.Vp) ? a.Vp + (int64_t)q0 * a.vp_stride : nullptr;   // pre-split V_q, or nullptr
    const float2* A = a.G + (int64_t)q0 * a.g_stride;
    const float2* B = a.V + (a.v_off ? a.v_off[p0] : (int64_t)q0 * a.v_stride);
    const int64_t ij = m0 + row;
    const bool valid = ij < a.n12;

    float acc[Cfg::NRG];
    const float sA = (TC_F16 && a.amax) ? tc::f16_scale(*a.amax) : 1.f;
    const float sB = (TC_F16 && a.bmax) ? tc::f16_scale(*a.bmax) : 1.f;
    d.amax = d.bmax = nullptr;
    d.cmax = nullptr;
    tc_mainloop<BN, G>(d, A, B, m0, 0, tcsm, bar, tmem, acc, cur, sA, sB);

    if constexpr (MODE == Z_RESTORE) {
      if (valid) {
#pragma unroll
        for (int kz = 0; kz < N3; ++kz) a.Tout[(int64_t)kz * a.n12 + ij] = make_float2(acc[2 * kz], acc[2 * kz + 1]);
      }
    } else {
#pragma unroll
      for (int dq = 0; dq < ND; ++dq) {
        if (dq >= nd) continue;
        for (int cc = 0; cc < a.ncomp; ++cc) {   // signature components share the restored line
          float2* Wl = a.W + ((int64_t)(q0 + dq) * a.ncomp + cc) * Nz * a.n12 + (valid ? ij : 0);
          float2 f[N3];
#pragma unroll
          for (int z = 0; z < Nz; ++z) f[z] = valid ? Wl[(int64_t)z * a.n12] : make_float2(0.f, 0.f);
          fft_reg<N3, false, true>(f);
#pragma unroll
          for (int kz = 0; kz < N3; ++kz)
            f[kz] = cmul2(f[kz], make_float2(acc[2 * (dq * N3 + kz)], acc[2 * (dq * N3 + kz) + 1]));
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

// ---------------------------------------------------------------- k_tc_conv_z64
// z-stage for n3 = 64 (configs 4, 5) on the tensor cores.  A 64-column tile would need
// 512 TMEM columns and 128 accumulator registers per thread, so the kz range is split by
// parity (B columns in (even, odd) order) into two 32-column passes over the same rows:
//   A^[2m]   = DFT_32(x)[m],                A^[2m+1] = DFT_32(x[z] W_64^z)[m]      (x: z < 32)
//   y[z]     = IDFT_32(T_even A^_even)[z] + W_64^{-z} IDFT_32(T_odd A^_odd)[z]      (z < 32)
// (the unnormalised length-64 transforms of eq. (5), pruned input, truncated output).  The
// even-pass partial y goes to a scratch line S and is added in the odd pass.
template <int MODE>
__global__ void __launch_bounds__(128, 1) k_tc_conv_z64(ZArgs a, float2* __restrict__ S, int nq) {
  constexpr int N3 = 64, H = 32, BN = 32;
  using Cfg = TcGemmCfg<BN, 1>;
  extern __shared__ __align__(1024) uint8_t tcsm[];
  __shared__ __align__(8) uint64_t bar[3 * TC_NS + 2];
  __shared__ uint32_t tslot;

  const int tiles_m = (int)((a.n12 + TC_BM - 1) / TC_BM);
  const int total = tiles_m * nq;
  const uint32_t tmem = tc_setup<Cfg::TMEM_COLS>(bar, &tslot);
  TcCursor cur;
  for (int t = blockIdx.x; t < total; t += gridDim.x) {
  int q, mt;
  z_tile(t, tiles_m, nq, a.z_blocked, q, mt);
  const int p = a.p0 + q;
  const int m0 = mt * TC_BM;
  GemmDesc d;
  d.m = (int)a.n12;
  d.n = N3;
  d.k = a.rank_p ? a.rank_p[p] : a.rank;
  d.batch = 1;
  d.a_s0 = 1; d.a_s1 = 0; d.a_div = 1 << 30; d.a_sk = a.n12;
  d.b_sk = a.v_sc; d.b_sn = a.v_sk;
  d.b_eo = 1;                              // column j < 32 -> kz = 2j, j >= 32 -> kz = 2(j-32)+1
  d.c_s0 = 0; d.c_s1 = 0; d.c_div = 1; d.c_sn = 0;
  d.sA = d.sB = d.sC = 0;
  d.Ap = a.Gp;
  d.Bp = nullptr;
  d.a_nkc = (d.k + TC_BK - 1) / TC_BK;
  const float2* A = a.G + (int64_t)q * a.g_stride;
  const float2* B = a.V + (a.v_off ? a.v_off[p] : (int64_t)q * a.v_stride);

  const int row = threadIdx.x;
  const int64_t ij = m0 + row;
  const bool valid = ij < a.n12;

  float acc[2 * BN];
  const float sA = (TC_F16 && a.amax) ? tc::f16_scale(*a.amax) : 1.f;
  const float sB = (TC_F16 && a.bmax) ? tc::f16_scale(*a.bmax) : 1.f;
  d.amax = d.bmax = nullptr;
  d.cmax = nullptr;
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
    d.Bp = a.Vp ? a.Vp + ((int64_t)h * nq + q) * a.vp_stride : nullptr;   // pre-split V_q columns 2j + h
    tc_mainloop<BN, 1>(d, A, B, m0, h * H, tcsm, bar, tmem, acc, cur, sA, sB);   // T_p[ij, 2m + h]
    if constexpr (MODE == Z_RESTORE) {
      if (valid) {
#pragma unroll
        for (int m = 0; m < H; ++m) a.Tout[(int64_t)(2 * m + h) * a.n12 + ij] = make_float2(acc[2 * m], acc[2 * m + 1]);
      }
    } else {
      for (int cc = 0; cc < a.ncomp; ++cc) {
        const int64_t line = ((int64_t)q * a.ncomp + cc) * H * a.n12 + (valid ? ij : 0);
        float2* Wl = a.W + line;
        float2* Sl = S + line;
        float2 f[H];
#pragma unroll
        for (int z = 0; z < H; ++z) f[z] = valid ? Wl[(int64_t)z * a.n12] : make_float2(0.f, 0.f);
        if (h) {
#pragma unroll
          for (int z = 1; z < H; ++z) f[z] = cmul(f[z], twc<N3, false>(z));
        }
        fft_reg<H, false, false>(f);
#pragma unroll
        for (int m = 0; m < H; ++m) f[m] = cmul2(f[m], make_float2(acc[2 * m], acc[2 * m + 1]));
        fft_reg<H, true, false>(f);
        if (valid) {
          if (h == 0) {
#pragma unroll
            for (int z = 0; z < H; ++z) Sl[(int64_t)z * a.n12] = f[z];
          } else {
#pragma unroll
            for (int z = 0; z < H; ++z) {
              const float2 odd = z ? cmul(f[z], twc<N3, true>(z)) : f[z];
              Wl[(int64_t)z * a.n12] = cadd(Sl[(int64_t)z * a.n12], odd);
            }
          }
        }
      }
    }
  }
  }
  tc_teardown<Cfg::TMEM_COLS>(tmem);
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
