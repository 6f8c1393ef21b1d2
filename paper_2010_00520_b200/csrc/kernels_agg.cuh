// kernels_agg.cuh -- aggregation (eq. (4)) and disaggregation (eq. (6))
// around the translation stage.
//
// Basis functions are numbered box by box: box v (linear index x + Nx (y + Ny z)) holds
// n in [box_ptr[v], box_ptr[v+1]).  Far-field patterns P[p][n][c] (complex64, c = theta, phi
// components fastest), coefficients I[n], signatures [p][c][v] (the translate_multi layout).
// Both kernels stream P once (HBM-bound: 8 ncomp bytes per direction and basis function).
#pragma once
#include "common.cuh"

namespace fmmt {

// Loads of NC consecutive complex64 values (one basis function's components).
template <int NC>
__device__ __forceinline__ void ld_comp(const float2* __restrict__ src, float2 (&v)[NC]) {
  if constexpr (NC == 2) {
    const float4 t = __ldg(reinterpret_cast<const float4*>(src));
    v[0] = make_float2(t.x, t.y);
    v[1] = make_float2(t.z, t.w);
  } else {
#pragma unroll
    for (int c = 0; c < NC; ++c) v[c] = __ldg(src + c);
  }
}

// Aggregation: one warp per box v and block of AGG_PD directions (blockIdx.y); the 8 warps of a CTA
// take 8 consecutive boxes.  The lanes hold I[n] of up to 128 basis functions of the box (4 per lane)
// in registers and stream P[p][n][:] for two directions at a time (8 loads of NC complex per lane in
// flight) before the multiply-adds and the shuffle reduction over the box.  Empty boxes write 0.
constexpr int AGG_PD = 16;

// Sum of 8 per-lane values over the warp with 9 shuffles (instead of 8 x 5): each step halves the
// values a lane keeps and exchanges the other half with its partner.  Returns, in lane L, the warp
// sum of value q = ((L >> 4) & 1) * 4 + ((L >> 3) & 1) * 2 + ((L >> 2) & 1) (lanes 4q + {0..3} agree).
__device__ __forceinline__ float warp_reduce8(const float (&a)[8], int lane) {
  float b[4], c[2];
  const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float send = h16 ? a[i] : a[i + 4];
    const float keep = h16 ? a[i + 4] : a[i];
    b[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float send = h8 ? b[i] : b[i + 2];
    const float keep = h8 ? b[i + 2] : b[i];
    c[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  float d = (h4 ? c[1] : c[0]) + __shfl_xor_sync(0xffffffffu, h4 ? c[0] : c[1], 4);
  d += __shfl_xor_sync(0xffffffffu, d, 2);
  d += __shfl_xor_sync(0xffffffffu, d, 1);
  return d;
}

template <int NC>
__device__ __forceinline__ void agg_store(float2 (&acc)[NC], int lane, float2* __restrict__ sig, int64_t p, int64_t K,
                                          int64_t v) {
#pragma unroll
  for (int c = 0; c < NC; ++c) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      acc[c].x += __shfl_xor_sync(0xffffffffu, acc[c].x, o);
      acc[c].y += __shfl_xor_sync(0xffffffffu, acc[c].y, o);
    }
  }
  if (lane < NC) {                      // lane c writes component c
    float2 out = acc[0];
#pragma unroll
    for (int c = 1; c < NC; ++c)
      if (lane == c) out = acc[c];
    sig[(p * NC + lane) * K + v] = out;
  }
}

template <int NC>
__global__ void __launch_bounds__(256) k_aggregate(const float2* __restrict__ P, const float2* __restrict__ I,
                                                      const int64_t* __restrict__ box_ptr, int64_t ndir, int64_t N,
                                                      int64_t K, float2* __restrict__ sig) {
  constexpr int C = NC;
  const int lane = threadIdx.x & 31;
  const int64_t v = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (v >= K) return;
  const int64_t lo = box_ptr[v], hi = box_ptr[v + 1];
  const int64_t pa = (int64_t)blockIdx.y * AGG_PD, pe = min(ndir, pa + AGG_PD);
  for (int64_t base = lo; base < hi || base == lo; base += 128) {   // boxes of > 128: several passes
    const int64_t nb = hi < base + 128 ? hi : base + 128;
    float2 iv[4];
    bool ok[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t n = base + lane + 32 * j;
      ok[j] = n < nb;
      iv[j] = ok[j] ? __ldg(I + n) : make_float2(0.f, 0.f);
    }
    const float2* Pb = P + (pa * N + base + lane) * C;   // this lane's first element, direction pa
    const int64_t dstride = N * C;                         // one direction further
    for (int64_t p = pa; p < pe; p += 2, Pb += 2 * dstride) {
      const bool two = p + 1 < pe;
      float2 pv[2][4][C];
#pragma unroll
      for (int d = 0; d < 2; ++d)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (ok[j] && (d == 0 || two)) {
            ld_comp<C>(Pb + d * dstride + 32 * j * C, pv[d][j]);
          } else {
#pragma unroll
            for (int c = 0; c < C; ++c) pv[d][j][c] = make_float2(0.f, 0.f);
          }
        }
      if constexpr (C == 2) {
        if (base == lo && nb == hi) {   // whole box in one pass: both directions' sums in one transpose-reduction
          float a[8];                   // a[d * 4 + c * 2 + (re, im)]
#pragma unroll
          for (int d = 0; d < 2; ++d)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              float2 t = make_float2(0.f, 0.f);
#pragma unroll
              for (int j = 0; j < 4; ++j) cmac(t, pv[d][j][c], iv[j]);
              a[d * 4 + c * 2] = t.x;
              a[d * 4 + c * 2 + 1] = t.y;
            }
          const float r = warp_reduce8(a, lane);   // lane (4 q) holds the box sum of value q
          if ((lane & 3) == 0) {
            const int q = lane >> 2, d = q >> 2, c = (q >> 1) & 1;
            if (d == 0 || two) reinterpret_cast<float*>(sig + ((p + d) * C + c) * K + v)[q & 1] = r;
          }
          continue;
        }
      }
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        if (d == 1 && !two) break;
        float2 acc[C];
#pragma unroll
        for (int c = 0; c < C; ++c) acc[c] = make_float2(0.f, 0.f);
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int c = 0; c < C; ++c) cmac(acc[c], pv[d][j][c], iv[j]);
        if (base == lo && nb == hi) {
          agg_store<C>(acc, lane, sig, p + d, K, v);
        } else {                        // large box: accumulate the passes in sig (same warp, in order)
#pragma unroll
          for (int c = 0; c < C; ++c) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              acc[c].x += __shfl_xor_sync(0xffffffffu, acc[c].x, o);
              acc[c].y += __shfl_xor_sync(0xffffffffu, acc[c].y, o);
            }
          }
          if (lane < C) {
            float2 out = acc[0];
#pragma unroll
            for (int c = 1; c < C; ++c)
              if (lane == c) out = acc[c];
            float2* dst = sig + ((p + d) * C + lane) * K + v;
            if (base != lo) out = cadd(out, *dst);
            *dst = out;
          }
        }
      }
    }
    if (hi == lo) break;
  }
}

// Aggregation staged through shared memory: one CTA (256 threads) per box v and block of 32
// directions.  Per pass of up to AGS_F / NC basis functions the CTA copies the 32 directions' contiguous
// pattern rows P[p][n0:n1][:] into shared memory with coalesced 16-byte loads, then thread (np, c, d)
// (d = direction, lane-fastest; c = component; np = quarter of the pass) sums its quarter of
// P[d][n][c] I[n] from shared memory; the quarters are added through shared memory and lane d of the
// first NC warps writes sig[p][c][v].  No shuffles, few index operations per element.
constexpr int AGS_F = 128;   // staged float2 per direction row and pass (AGS_F / NC basis functions; boxes hold ~55)

template <int NC>
__global__ void __launch_bounds__(256) k_aggregate_smem(const float2* __restrict__ P, const float2* __restrict__ I,
                                                        const int64_t* __restrict__ box_ptr, int64_t ndir, int64_t N,
                                                        int64_t K, float2* __restrict__ sig) {
  static_assert(NC == 1 || NC == 2 || NC == 4, "components per basis function");
  constexpr int NP = 8 / NC;                     // n-parts: 32 directions x NC components x NP = 256 threads
  constexpr int AGS_N = AGS_F / NC;              // basis functions per pass
  constexpr int ROW = AGS_F + 1;                 // float2 per staged direction row (odd: no bank conflicts)
  __shared__ float2 sP[32 * ROW];
  __shared__ float2 sI[AGS_N];
  __shared__ float2 red[256];
  const int64_t v = blockIdx.x;
  const int64_t p0 = (int64_t)blockIdx.y * 32;
  const int tid = threadIdx.x;
  const int d = tid & 31, c = (tid >> 5) % NC, np = (tid >> 5) / NC;
  const int64_t lo = box_ptr[v], hi = box_ptr[v + 1];
  float2 acc = make_float2(0.f, 0.f);
  for (int64_t n0 = lo; n0 < hi; n0 += AGS_N) {
    const int m = (int)(hi - n0 < AGS_N ? hi - n0 : AGS_N);
    __syncthreads();                              // previous pass's reads done
    // stage: 32 rows of m * NC float2 (row r = direction p0 + r), coalesced along the row
    for (int e = tid; e < 32 * m * NC; e += 256) {
      const int r = e / (m * NC), o = e - r * (m * NC);
      const int64_t p = p0 + r;
      sP[r * ROW + o] = p < ndir ? __ldg(P + (p * N + n0) * NC + o) : make_float2(0.f, 0.f);
    }
    for (int e = tid; e < m; e += 256) sI[e] = __ldg(I + n0 + e);
    __syncthreads();
    // thread (np, c, d): n = np, np + NP, ... of this pass
    const float2* row = sP + d * ROW + c;
    for (int n = np; n < m; n += NP) cmac(acc, row[n * NC], sI[n]);
  }
  red[tid] = acc;
  __syncthreads();
  if (tid < 32 * NC) {                            // np == 0 threads: add the other quarters, write
    float2 t = red[tid];
#pragma unroll
    for (int q = 1; q < NP; ++q) t = cadd(t, red[tid + q * 32 * NC]);
    const int64_t p = p0 + d;
    if (p < ndir) sig[(p * NC + c) * K + v] = t;
  }
}

// Generic-ncomp aggregation (one component pass at a time): the fallback for ncomp not in {1, 2, 4}.
__global__ void __launch_bounds__(256) k_aggregate_any(const float2* __restrict__ P, const float2* __restrict__ I,
                                                       const int64_t* __restrict__ box_ptr, int64_t ndir, int64_t N,
                                                       int ncomp, int64_t K, float2* __restrict__ sig) {
  const int lane = threadIdx.x & 31;
  const int64_t v = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (v >= K) return;
  const int64_t lo = box_ptr[v], hi = box_ptr[v + 1];
  for (int64_t p = blockIdx.y; p < ndir; p += gridDim.y) {
    for (int c = 0; c < ncomp; ++c) {
      float2 acc = make_float2(0.f, 0.f);
      for (int64_t n = lo + lane; n < hi; n += 32) cmac(acc, __ldg(P + (p * N + n) * ncomp + c), __ldg(I + n));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
      }
      if (lane == 0) sig[(p * ncomp + c) * K + v] = acc;
    }
  }
}

// Partial disaggregation over the direction block s of nsplit: one CTA (64 threads) per box, a
// thread per basis function m of the box, 8 directions' loads in flight per thread:
//   part[s][m] = sum_{p in block s} w_p sum_c conj(P[p][m][c]) B[p][c][v].
// The box's B[p][:][v] and w_p are the same for all threads (broadcast loads).
template <int NC>
__global__ void __launch_bounds__(64) k_disaggregate_partial(const float2* __restrict__ P, const float2* __restrict__ B,
                                                             const float* __restrict__ w,
                                                             const int64_t* __restrict__ box_ptr, int64_t ndir,
                                                             int64_t N, int64_t K, int nsplit,
                                                             float2* __restrict__ part) {
  constexpr int C = NC;
  constexpr int U = 8;
  const int64_t v = blockIdx.x;
  const int s = blockIdx.y;
  const int64_t lo = box_ptr[v], hi = box_ptr[v + 1];
  const int64_t p0 = ndir * s / nsplit, p1 = ndir * (s + 1) / nsplit;
  for (int64_t m = lo + threadIdx.x; m < hi; m += blockDim.x) {
    float2 acc = make_float2(0.f, 0.f);
    for (int64_t pb = p0; pb < p1; pb += U) {
      float2 pv[U][C], bv[U][C];
      float wv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t p = pb + u;
        if (p < p1) {
          ld_comp<C>(P + (p * N + m) * C, pv[u]);
#pragma unroll
          for (int c = 0; c < C; ++c) bv[u][c] = __ldg(B + (p * C + c) * K + v);
          wv[u] = __ldg(w + p);
        } else {
#pragma unroll
          for (int c = 0; c < C; ++c) pv[u][c] = bv[u][c] = make_float2(0.f, 0.f);
          wv[u] = 0.f;
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        float2 t = make_float2(0.f, 0.f);
#pragma unroll
        for (int c = 0; c < C; ++c) cmac_conj(t, pv[u][c], bv[u][c]);   // conj(P) B
        acc.x = fmaf(wv[u], t.x, acc.x);
        acc.y = fmaf(wv[u], t.y, acc.y);
      }
    }
    part[(int64_t)s * N + m] = acc;
  }
}

// Partial disaggregation staged through shared memory: one CTA (256 threads) per box v and block s of
// 32 directions (nsplit = ceil(ndir / 32)).  Per pass of up to AGS_F / NC basis functions the CTA copies
// the 32 directions' pattern rows (coalesced) and w_p B[p][:][v] into shared memory; thread (dq, m)
// (m = basis function of the pass, fastest; dq = quarter of the 32 directions) sums
// w_p conj(P[p][m][c]) B[p][c][v] over its 8 directions; the quarters are added through shared memory:
//   part[s][m] = sum_{p in block s} w_p sum_c conj(P[p][m][c]) B[p][c][v].
template <int NC>
__global__ void __launch_bounds__(256) k_disaggregate_smem(const float2* __restrict__ P, const float2* __restrict__ B,
                                                           const float* __restrict__ w,
                                                           const int64_t* __restrict__ box_ptr, int64_t ndir,
                                                           int64_t N, int64_t K, float2* __restrict__ part) {
  static_assert(NC == 1 || NC == 2 || NC == 4, "components per basis function");
  constexpr int AGS_N = AGS_F / NC;              // basis functions per pass (64 for NC = 2)
  constexpr int ROW = AGS_F + 1;
  constexpr int MT = AGS_N < 64 ? AGS_N : 64;    // threads along m
  constexpr int DQ = 256 / MT;                   // direction parts
  __shared__ float2 sP[32 * ROW];
  __shared__ float2 sB[32 * NC];
  __shared__ float2 red[256];
  const int64_t v = blockIdx.x;
  const int s = blockIdx.y;
  const int64_t p0 = (int64_t)s * 32;
  const int tid = threadIdx.x;
  const int ml = tid % MT, dq = tid / MT;
  const int64_t lo = box_ptr[v], hi = box_ptr[v + 1];
  if (hi == lo) return;
  if (tid < 32 * NC) {                            // w_p B[p][c][v] of the block's directions
    const int r = tid / NC, c = tid % NC;
    const int64_t p = p0 + r;
    float2 b = make_float2(0.f, 0.f);
    if (p < ndir) {
      b = __ldg(B + (p * NC + c) * K + v);
      const float wp = __ldg(w + p);
      b.x *= wp;
      b.y *= wp;
    }
    sB[tid] = b;
  }
  for (int64_t n0 = lo; n0 < hi; n0 += AGS_N) {
    const int m = (int)(hi - n0 < AGS_N ? hi - n0 : AGS_N);
    __syncthreads();                              // previous pass's reads done (and sB written)
    for (int e = tid; e < 32 * m * NC; e += 256) {
      const int r = e / (m * NC), o = e - r * (m * NC);
      const int64_t p = p0 + r;
      sP[r * ROW + o] = p < ndir ? __ldg(P + (p * N + n0) * NC + o) : make_float2(0.f, 0.f);
    }
    __syncthreads();
    for (int mm0 = 0; mm0 < m; mm0 += MT) {      // uniform trip count (barriers inside)
      const int mm = mm0 + ml;
      float2 acc = make_float2(0.f, 0.f);
      if (mm < m) {
#pragma unroll 4
        for (int r = dq; r < 32; r += DQ)
#pragma unroll
          for (int c = 0; c < NC; ++c) cmac_conj(acc, sP[r * ROW + mm * NC + c], sB[r * NC + c]);
      }
      red[tid] = acc;
      __syncthreads();
      if (dq == 0 && mm < m) {
        float2 t = red[ml];
#pragma unroll
        for (int q = 1; q < DQ; ++q) t = cadd(t, red[ml + q * MT]);
        part[(int64_t)s * N + n0 + mm] = t;
      }
      __syncthreads();
    }
  }
}

// Generic-ncomp partial disaggregation (fallback for ncomp not in {1, 2, 4}).
__global__ void __launch_bounds__(64) k_disaggregate_partial_any(const float2* __restrict__ P,
                                                                 const float2* __restrict__ B,
                                                                 const float* __restrict__ w,
                                                                 const int64_t* __restrict__ box_ptr, int64_t ndir,
                                                                 int64_t N, int ncomp, int64_t K, int nsplit,
                                                                 float2* __restrict__ part) {
  const int64_t v = blockIdx.x;
  const int s = blockIdx.y;
  const int64_t lo = box_ptr[v], hi = box_ptr[v + 1];
  const int64_t p0 = ndir * s / nsplit, p1 = ndir * (s + 1) / nsplit;
  for (int64_t m = lo + threadIdx.x; m < hi; m += blockDim.x) {
    float2 acc = make_float2(0.f, 0.f);
    for (int64_t p = p0; p < p1; ++p) {
      float2 t = make_float2(0.f, 0.f);
      for (int c = 0; c < ncomp; ++c) cmac_conj(t, __ldg(P + (p * N + m) * ncomp + c), __ldg(B + (p * ncomp + c) * K + v));
      const float wp = __ldg(w + p);
      acc.x = fmaf(wp, t.x, acc.x);
      acc.y = fmaf(wp, t.y, acc.y);
    }
    part[(int64_t)s * N + m] = acc;
  }
}

__global__ void k_disaggregate_final(const float2* __restrict__ part, int64_t N, int nsplit, float2* __restrict__ y) {
  const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= N) return;
  float2 acc = part[m];
  for (int s = 1; s < nsplit; ++s) {
    const float2 t = part[(int64_t)s * N + m];
    acc.x += t.x;
    acc.y += t.y;
  }
  y[m] = acc;
}

}  // namespace fmmt
