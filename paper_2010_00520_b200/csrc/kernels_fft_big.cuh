// kernels_fft_big.cuh -- the xy FFT stages (a1, a2, a6 of eq. (5)) for planes of at least
// 64 x 64 padded points (configs 4 and 5).
//
// One CTA of 512 threads holds PP whole planes in shared memory (row pitch NX + 1: row-strided
// accesses are bank-conflict free) and runs each axis as a four-step DFT N = A * B in place:
//   pass 1, item (line, n2):  A-point DFT over n1 of x[B n1 + n2] (pruned: the zero-padded upper
//                             half, n1 >= A/2, is never read), times W_N^{n2 k1}, written back to the
//                             positions B k1 + n2 it was read from (read set within write set);
//   pass 2, item (line, k1):  B-point DFT over n2 of y[B k1 + n2] -> X[k1 + A k2] (natural order).
// Pass 2 reads and writes different positions, so every thread loads and transforms all its items
// before a barrier and stores after it, unless its output goes straight to global memory (forward y
// pass -> W, coalesced along kx).  Every pass has about one item per thread (the chunked four-step of
// k_fwd_xy / k_inv_xy ran 128-256 items per pass on 128 x 128 planes with 24 barriers per plane).
//   forward:  x pass on the Ny nonzero rows (input read from sig_in in pass 1), y pass on all NX
//             columns (pass 2 writes W[ky][kx]);
//   inverse:  y pass on all NX columns (pass 1 reads W), truncated to y < Ny; x pass on those rows,
//             truncated to x < Nx and scaled; coalesced copy to sig_out.
#pragma once
#include "kernels_fft.cuh"

namespace fmmt {

#ifndef FMMT_XYB_THREADS
#define FMMT_XYB_THREADS 512
#endif
constexpr int XYB_THREADS = FMMT_XYB_THREADS;

template <int NX, int NY, int PP>
struct XYBig {
  static_assert(NX >= 64 && NY >= 64 && NX <= FMMT_TW_NMAX && NY <= FMMT_TW_NMAX, "large planes only");
  static constexpr int Nx = NX / 2, Ny = NY / 2;
  static constexpr int PX = NX + 1;                 // row pitch (complex)
  static constexpr int PLANE = NY * PX;             // complex per plane buffer
  static constexpr int AX = Split<NX>::A, BX = Split<NX>::B;
  static constexpr int AY = Split<NY>::A, BY = Split<NY>::B;
  static constexpr int SMEM = (PP * PLANE + NX + NY) * 8;   // planes + the two four-step twiddle tables
};

// tw[k1 * B + n2] = W_N^{n2 k1} (forward sign) for the four-step split of N
template <int N>
__device__ __forceinline__ void load_fourstep_tw(float2* tw) {
  constexpr int B = Split<N>::B;
  for (int e = threadIdx.x; e < N; e += blockDim.x) {
    const int k1 = e / B, n2 = e % B;
    tw[e] = c_tw[(n2 * k1 * (FMMT_TW_NMAX / N)) & (FMMT_TW_NMAX - 1)];
  }
}

__device__ __forceinline__ float2 conjf2(float2 a) { return make_float2(a.x, -a.y); }

template <int NX, int NY, int PP>
__global__ void __launch_bounds__(XYB_THREADS, 1)
k_fwd_xy_big(const float2* __restrict__ sig_in, float2* __restrict__ W, int nplanes_total, int) {
  using G = XYBig<NX, NY, PP>;
  constexpr int Nx = G::Nx, Ny = G::Ny, PX = G::PX, AX = G::AX, BX = G::BX, AY = G::AY, BY = G::BY;
  extern __shared__ float2 smem[];
  float2* buf = smem;
  float2* twx = smem + PP * G::PLANE;
  float2* twy = twx + NX;
  const int g0 = blockIdx.x * PP;
  const int np = min(PP, nplanes_total - g0);
  if (np <= 0) return;
  load_fourstep_tw<NX>(twx);
  load_fourstep_tw<NY>(twy);
  __syncthreads();
  // x pass 1 (sig_in -> smem), item (j, y, n2), n2 fastest: each load instruction covers whole 64-byte
  // row segments
  for (int it = threadIdx.x; it < np * Ny * BX; it += XYB_THREADS) {
    const int n2 = it % BX, r = it / BX, y = r % Ny, j = r / Ny;
    const float2* row = sig_in + ((int64_t)(g0 + j) * Ny + y) * Nx;
    float2 v[AX];
#pragma unroll
    for (int n1 = 0; n1 < AX / 2; ++n1) v[n1] = row[BX * n1 + n2];
    fft_reg<AX, false, true>(v);
    float2* srow = buf + j * G::PLANE + y * PX;
#pragma unroll
    for (int k1 = 0; k1 < AX; ++k1) srow[BX * k1 + n2] = k1 ? cmul(v[k1], twx[k1 * BX + n2]) : v[k1];
  }
  __syncthreads();
  // x pass 2, item (j, y, k1), y fastest
  {
    constexpr int IPT = (PP * Ny * AX + XYB_THREADS - 1) / XYB_THREADS;
    float2 v[IPT][BX];
#pragma unroll
    for (int u = 0; u < IPT; ++u) {
      const int it = threadIdx.x + u * XYB_THREADS;
      if (it < np * Ny * AX) {
        const int y = it % Ny, r = it / Ny, k1 = r % AX, j = r / AX;
        const float2* srow = buf + j * G::PLANE + y * PX;
#pragma unroll
        for (int n2 = 0; n2 < BX; ++n2) v[u][n2] = srow[BX * k1 + n2];
        fft_reg<BX, false, false>(v[u]);
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < IPT; ++u) {
      const int it = threadIdx.x + u * XYB_THREADS;
      if (it < np * Ny * AX) {
        const int y = it % Ny, r = it / Ny, k1 = r % AX, j = r / AX;
        float2* srow = buf + j * G::PLANE + y * PX;
#pragma unroll
        for (int k2 = 0; k2 < BX; ++k2) srow[k1 + AX * k2] = v[u][k2];
      }
    }
  }
  __syncthreads();
  // y pass 1, item (j, x, n2), x fastest: rows BY n1 + n2 (n1 < AY / 2) -> rows BY k1 + n2
  for (int it = threadIdx.x; it < np * NX * BY; it += XYB_THREADS) {
    const int x = it % NX, r = it / NX, n2 = r % BY, j = r / BY;
    float2* col = buf + j * G::PLANE + x;
    float2 v[AY];
#pragma unroll
    for (int n1 = 0; n1 < AY / 2; ++n1) v[n1] = col[(BY * n1 + n2) * PX];
    fft_reg<AY, false, true>(v);
#pragma unroll
    for (int k1 = 0; k1 < AY; ++k1) col[(BY * k1 + n2) * PX] = k1 ? cmul(v[k1], twy[k1 * BY + n2]) : v[k1];
  }
  __syncthreads();
  // y pass 2 (smem -> W), item (j, x, k1), x fastest: W[ky = k1 + AY k2][x], coalesced along x
  for (int it = threadIdx.x; it < np * NX * AY; it += XYB_THREADS) {
    const int x = it % NX, r = it / NX, k1 = r % AY, j = r / AY;
    const float2* col = buf + j * G::PLANE + x;
    float2 v[BY];
#pragma unroll
    for (int n2 = 0; n2 < BY; ++n2) v[n2] = col[(BY * k1 + n2) * PX];
    fft_reg<BY, false, false>(v);
    float2* out = W + (int64_t)(g0 + j) * (NX * NY) + x;
#pragma unroll
    for (int k2 = 0; k2 < BY; ++k2) out[(int64_t)(k1 + AY * k2) * NX] = v[k2];
  }
}

// Half-buffer forward kernel for the one-plane-per-CTA sizes (128 x 128, 256 x 64, 64 x 256): the x pass only
// ever fills the Ny nonzero rows, and the y pass keeps in shared memory only the k1 < AY / 2 half of its
// intermediate (written back to exactly the rows it was read from); the other half waits in registers until the
// first half's pass 2 has gone out to W.  66 KB instead of 132 KB of shared memory -> two CTAs per SM, so one
// CTA's prologue, global loads and barrier tails run under the other's DFTs.
template <int NX, int NY>
struct XYHalf {
  static constexpr int PX = NX + 1;
  static constexpr int SMEM = ((NY / 2) * PX + NX + NY) * 8;
};

template <int NX, int NY>
__global__ void __launch_bounds__(XYB_THREADS, 2)
k_fwd_xy_half(const float2* __restrict__ sig_in, float2* __restrict__ W, int nplanes_total, int) {
  using G = XYBig<NX, NY, 1>;
  constexpr int Nx = G::Nx, Ny = G::Ny, PX = G::PX, AX = G::AX, BX = G::BX, AY = G::AY, BY = G::BY;
  extern __shared__ float2 smem[];
  float2* buf = smem;
  float2* twx = smem + Ny * PX;
  float2* twy = twx + NX;
  const int g = blockIdx.x;
  if (g >= nplanes_total) return;
  load_fourstep_tw<NX>(twx);
  load_fourstep_tw<NY>(twy);
  __syncthreads();
  // x pass 1 (sig_in -> smem), item (y, n2), n2 fastest
  for (int it = threadIdx.x; it < Ny * BX; it += XYB_THREADS) {
    const int n2 = it % BX, y = it / BX;
    const float2* row = sig_in + ((int64_t)g * Ny + y) * Nx;
    float2 v[AX];
#pragma unroll
    for (int n1 = 0; n1 < AX / 2; ++n1) v[n1] = row[BX * n1 + n2];
    fft_reg<AX, false, true>(v);
    float2* srow = buf + y * PX;
#pragma unroll
    for (int k1 = 0; k1 < AX; ++k1) srow[BX * k1 + n2] = k1 ? cmul(v[k1], twx[k1 * BX + n2]) : v[k1];
  }
  __syncthreads();
  // x pass 2, item (y, k1), y fastest
  {
    constexpr int IPT = (Ny * AX + XYB_THREADS - 1) / XYB_THREADS;
    float2 v[IPT][BX];
#pragma unroll
    for (int u = 0; u < IPT; ++u) {
      const int it = threadIdx.x + u * XYB_THREADS;
      if (it < Ny * AX) {
        const int y = it % Ny, k1 = it / Ny;
        const float2* srow = buf + y * PX;
#pragma unroll
        for (int n2 = 0; n2 < BX; ++n2) v[u][n2] = srow[BX * k1 + n2];
        fft_reg<BX, false, false>(v[u]);
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < IPT; ++u) {
      const int it = threadIdx.x + u * XYB_THREADS;
      if (it < Ny * AX) {
        const int y = it % Ny, k1 = it / Ny;
        float2* srow = buf + y * PX;
#pragma unroll
        for (int k2 = 0; k2 < BX; ++k2) srow[k1 + AX * k2] = v[u][k2];
      }
    }
  }
  __syncthreads();
  // y pass 1, item (x, n2), x fastest: rows BY n1 + n2 (n1 < AY / 2) -> the same rows for k1 < AY / 2, in place;
  // k1 >= AY / 2 held in registers
  constexpr int IPT1 = (NX * BY + XYB_THREADS - 1) / XYB_THREADS;
  float2 hold[IPT1][AY / 2];
#pragma unroll
  for (int u = 0; u < IPT1; ++u) {
    const int it = threadIdx.x + u * XYB_THREADS;
    if (it < NX * BY) {
      const int x = it % NX, n2 = it / NX;
      float2* col = buf + x;
      float2 v[AY];
#pragma unroll
      for (int n1 = 0; n1 < AY / 2; ++n1) v[n1] = col[(BY * n1 + n2) * PX];
      fft_reg<AY, false, true>(v);
#pragma unroll
      for (int k1 = 0; k1 < AY / 2; ++k1) col[(BY * k1 + n2) * PX] = k1 ? cmul(v[k1], twy[k1 * BY + n2]) : v[k1];
#pragma unroll
      for (int k1 = AY / 2; k1 < AY; ++k1) hold[u][k1 - AY / 2] = cmul(v[k1], twy[k1 * BY + n2]);
    }
  }
  __syncthreads();
  // y pass 2 (smem -> W), item (x, kk), x fastest, k1 = kk + h AY / 2: W[ky = k1 + AY k2][x]
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (h == 1) {
      __syncthreads();   // every read of the first half is done
#pragma unroll
      for (int u = 0; u < IPT1; ++u) {
        const int it = threadIdx.x + u * XYB_THREADS;
        if (it < NX * BY) {
          const int x = it % NX, n2 = it / NX;
          float2* col = buf + x;
#pragma unroll
          for (int kk = 0; kk < AY / 2; ++kk) col[(BY * kk + n2) * PX] = hold[u][kk];
        }
      }
      __syncthreads();
    }
    for (int it = threadIdx.x; it < NX * (AY / 2); it += XYB_THREADS) {
      const int x = it % NX, kk = it / NX, k1 = kk + h * (AY / 2);
      const float2* col = buf + x;
      float2 v[BY];
#pragma unroll
      for (int n2 = 0; n2 < BY; ++n2) v[n2] = col[(BY * kk + n2) * PX];
      fft_reg<BY, false, false>(v);
      float2* out = W + (int64_t)g * (NX * NY) + x;
#pragma unroll
      for (int k2 = 0; k2 < BY; ++k2) out[(int64_t)(k1 + AY * k2) * NX] = v[k2];
    }
  }
}


template <int NX, int NY, int PP>
__global__ void __launch_bounds__(XYB_THREADS, 1)
k_inv_xy_big(const float2* __restrict__ W, float2* __restrict__ sig_out, int nplanes_total, int, float scale) {
  using G = XYBig<NX, NY, PP>;
  constexpr int Nx = G::Nx, Ny = G::Ny, PX = G::PX, AX = G::AX, BX = G::BX, AY = G::AY, BY = G::BY;
  extern __shared__ float2 smem[];
  float2* buf = smem;
  float2* twx = smem + PP * G::PLANE;
  float2* twy = twx + NX;
  const int g0 = blockIdx.x * PP;
  const int np = min(PP, nplanes_total - g0);
  if (np <= 0) return;
  load_fourstep_tw<NX>(twx);
  load_fourstep_tw<NY>(twy);
  __syncthreads();
  // y pass 1 (W -> smem), item (j, x, n2), x fastest: all NY input rows
  for (int it = threadIdx.x; it < np * NX * BY; it += XYB_THREADS) {
    const int x = it % NX, r = it / NX, n2 = r % BY, j = r / BY;
    const float2* in = W + (int64_t)(g0 + j) * (NX * NY) + x;
    float2 v[AY];
#pragma unroll
    for (int n1 = 0; n1 < AY; ++n1) v[n1] = in[(int64_t)(BY * n1 + n2) * NX];
    fft_reg<AY, true, false>(v);
    float2* col = buf + j * G::PLANE + x;
#pragma unroll
    for (int k1 = 0; k1 < AY; ++k1) col[(BY * k1 + n2) * PX] = k1 ? cmul(v[k1], conjf2(twy[k1 * BY + n2])) : v[k1];
  }
  __syncthreads();
  // y pass 2, item (j, x, k1), x fastest: outputs y = k1 + AY k2 < Ny only (k2 < BY / 2)
  {
    constexpr int IPT = (PP * NX * AY + XYB_THREADS - 1) / XYB_THREADS;
    float2 o[IPT][BY / 2];
#pragma unroll
    for (int u = 0; u < IPT; ++u) {
      const int it = threadIdx.x + u * XYB_THREADS;
      if (it < np * NX * AY) {
        const int x = it % NX, r = it / NX, k1 = r % AY, j = r / AY;
        const float2* col = buf + j * G::PLANE + x;
        float2 v[BY];
#pragma unroll
        for (int n2 = 0; n2 < BY; ++n2) v[n2] = col[(BY * k1 + n2) * PX];
        fft_reg<BY, true, false>(v);
#pragma unroll
        for (int k2 = 0; k2 < BY / 2; ++k2) o[u][k2] = v[k2];
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < IPT; ++u) {
      const int it = threadIdx.x + u * XYB_THREADS;
      if (it < np * NX * AY) {
        const int x = it % NX, r = it / NX, k1 = r % AY, j = r / AY;
        float2* col = buf + j * G::PLANE + x;
#pragma unroll
        for (int k2 = 0; k2 < BY / 2; ++k2) col[(k1 + AY * k2) * PX] = o[u][k2];
      }
    }
  }
  __syncthreads();
  // x pass 1 on rows y < Ny, item (j, y, n2), y fastest: full input
  for (int it = threadIdx.x; it < np * Ny * BX; it += XYB_THREADS) {
    const int y = it % Ny, r = it / Ny, n2 = r % BX, j = r / BX;
    float2* srow = buf + j * G::PLANE + y * PX;
    float2 v[AX];
#pragma unroll
    for (int n1 = 0; n1 < AX; ++n1) v[n1] = srow[BX * n1 + n2];
    fft_reg<AX, true, false>(v);
#pragma unroll
    for (int k1 = 0; k1 < AX; ++k1) srow[BX * k1 + n2] = k1 ? cmul(v[k1], conjf2(twx[k1 * BX + n2])) : v[k1];
  }
  __syncthreads();
  // x pass 2, item (j, y, k1), y fastest: outputs x = k1 + AX k2 < Nx (k2 < BX / 2), scaled
  {
    constexpr int IPT = (PP * Ny * AX + XYB_THREADS - 1) / XYB_THREADS;
    float2 o[IPT][BX / 2];
#pragma unroll
    for (int u = 0; u < IPT; ++u) {
      const int it = threadIdx.x + u * XYB_THREADS;
      if (it < np * Ny * AX) {
        const int y = it % Ny, r = it / Ny, k1 = r % AX, j = r / AX;
        const float2* srow = buf + j * G::PLANE + y * PX;
        float2 v[BX];
#pragma unroll
        for (int n2 = 0; n2 < BX; ++n2) v[n2] = srow[BX * k1 + n2];
        fft_reg<BX, true, false>(v);
#pragma unroll
        for (int k2 = 0; k2 < BX / 2; ++k2) o[u][k2] = cscale(v[k2], scale);
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < IPT; ++u) {
      const int it = threadIdx.x + u * XYB_THREADS;
      if (it < np * Ny * AX) {
        const int y = it % Ny, r = it / Ny, k1 = r % AX, j = r / AX;
        float2* srow = buf + j * G::PLANE + y * PX;
#pragma unroll
        for (int k2 = 0; k2 < BX / 2; ++k2) srow[k1 + AX * k2] = o[u][k2];
      }
    }
  }
  __syncthreads();
  // store rows y < Ny, x < Nx (coalesced along x)
  {
    float2* dst = sig_out + (int64_t)g0 * (Nx * Ny);
    for (int e = threadIdx.x; e < np * Nx * Ny; e += XYB_THREADS) {
      const int x = e % Nx, r = e / Nx, y = r % Ny, j = r / Ny;
      dst[e] = buf[j * G::PLANE + y * PX + x];
    }
  }
}

// Three-quarter-buffer inverse kernel for the same sizes: the y pass keeps the k1 < AY / 2 half of its
// intermediate in NY / 2 rows (the other half in registers), writes that half's truncated outputs to an extra
// NY / 4 rows, then runs the second half through the same NY / 2 rows.  The Ny surviving rows end up permuted
// (row_of): the x pass works row by row, so only its row addressing and the final store see the permutation.
// The extra region starts 8 rows late so that 16 consecutive y still fall into 16 different bank pairs.
template <int NX, int NY>
struct XYInvHalf {
  static constexpr int PX = NX + 1;
  static constexpr int AY = Split<NY>::A, BY = Split<NY>::B;
  static constexpr int EXTRA = NY / 2 + 8;
  static constexpr int ROWS = EXTRA + NY / 4;
  static constexpr int SMEM = (ROWS * PX + NX + NY) * 8;
  __device__ static __forceinline__ int row_of(int y) {
    const int k1 = y % AY, k2 = y / AY;
    return k1 < AY / 2 ? EXTRA + k1 + (AY / 2) * k2 : (k1 - AY / 2) + (AY / 2) * k2;
  }
};

template <int NX, int NY>
__global__ void __launch_bounds__(XYB_THREADS, 2)
k_inv_xy_half(const float2* __restrict__ W, float2* __restrict__ sig_out, int nplanes_total, int, float scale) {
  using G = XYBig<NX, NY, 1>;
  using H = XYInvHalf<NX, NY>;
  constexpr int Nx = G::Nx, Ny = G::Ny, PX = G::PX, AX = G::AX, BX = G::BX, AY = G::AY, BY = G::BY;
  extern __shared__ float2 smem[];
  float2* buf = smem;
  float2* twx = smem + H::ROWS * PX;
  float2* twy = twx + NX;
  const int g = blockIdx.x;
  if (g >= nplanes_total) return;
  load_fourstep_tw<NX>(twx);
  load_fourstep_tw<NY>(twy);
  __syncthreads();
  // y pass 1 (W -> smem rows BY k1 + n2 for k1 < AY / 2, registers for the rest), item (x, n2), x fastest
  constexpr int IPT1 = (NX * BY + XYB_THREADS - 1) / XYB_THREADS;
  float2 hold[IPT1][AY / 2];
#pragma unroll
  for (int u = 0; u < IPT1; ++u) {
    const int it = threadIdx.x + u * XYB_THREADS;
    if (it < NX * BY) {
      const int x = it % NX, n2 = it / NX;
      const float2* in = W + (int64_t)g * (NX * NY) + x;
      float2 v[AY];
#pragma unroll
      for (int n1 = 0; n1 < AY; ++n1) v[n1] = in[(int64_t)(BY * n1 + n2) * NX];
      fft_reg<AY, true, false>(v);
      float2* col = buf + x;
#pragma unroll
      for (int k1 = 0; k1 < AY / 2; ++k1) col[(BY * k1 + n2) * PX] = k1 ? cmul(v[k1], conjf2(twy[k1 * BY + n2])) : v[k1];
#pragma unroll
      for (int k1 = AY / 2; k1 < AY; ++k1) hold[u][k1 - AY / 2] = cmul(v[k1], conjf2(twy[k1 * BY + n2]));
    }
  }
  __syncthreads();
  // y pass 2, first half: item (x, kk), outputs y = kk + AY k2 < Ny (k2 < BY / 2) go straight to the extra rows
  for (int it = threadIdx.x; it < NX * (AY / 2); it += XYB_THREADS) {
    const int x = it % NX, kk = it / NX;
    float2* col = buf + x;
    float2 v[BY];
#pragma unroll
    for (int n2 = 0; n2 < BY; ++n2) v[n2] = col[(BY * kk + n2) * PX];
    fft_reg<BY, true, false>(v);
#pragma unroll
    for (int k2 = 0; k2 < BY / 2; ++k2) col[(H::EXTRA + kk + (AY / 2) * k2) * PX] = v[k2];
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < IPT1; ++u) {
    const int it = threadIdx.x + u * XYB_THREADS;
    if (it < NX * BY) {
      const int x = it % NX, n2 = it / NX;
      float2* col = buf + x;
#pragma unroll
      for (int kk = 0; kk < AY / 2; ++kk) col[(BY * kk + n2) * PX] = hold[u][kk];
    }
  }
  __syncthreads();
  // second half (k1 = kk + AY / 2): outputs held over a barrier, then written to rows kk + (AY / 2) k2
  {
    constexpr int IPT2 = (NX * (AY / 2) + XYB_THREADS - 1) / XYB_THREADS;
    float2 o[IPT2][BY / 2];
#pragma unroll
    for (int u = 0; u < IPT2; ++u) {
      const int it = threadIdx.x + u * XYB_THREADS;
      if (it < NX * (AY / 2)) {
        const int x = it % NX, kk = it / NX;
        const float2* col = buf + x;
        float2 v[BY];
#pragma unroll
        for (int n2 = 0; n2 < BY; ++n2) v[n2] = col[(BY * kk + n2) * PX];
        fft_reg<BY, true, false>(v);
#pragma unroll
        for (int k2 = 0; k2 < BY / 2; ++k2) o[u][k2] = v[k2];
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < IPT2; ++u) {
      const int it = threadIdx.x + u * XYB_THREADS;
      if (it < NX * (AY / 2)) {
        const int x = it % NX, kk = it / NX;
        float2* col = buf + x;
#pragma unroll
        for (int k2 = 0; k2 < BY / 2; ++k2) col[(kk + (AY / 2) * k2) * PX] = o[u][k2];
      }
    }
  }
  __syncthreads();
  // x pass 1 on the Ny surviving rows, item (y, n2), y fastest: full input
  for (int it = threadIdx.x; it < Ny * BX; it += XYB_THREADS) {
    const int y = it % Ny, n2 = it / Ny;
    float2* srow = buf + H::row_of(y) * PX;
    float2 v[AX];
#pragma unroll
    for (int n1 = 0; n1 < AX; ++n1) v[n1] = srow[BX * n1 + n2];
    fft_reg<AX, true, false>(v);
#pragma unroll
    for (int k1 = 0; k1 < AX; ++k1) srow[BX * k1 + n2] = k1 ? cmul(v[k1], conjf2(twx[k1 * BX + n2])) : v[k1];
  }
  __syncthreads();
  // x pass 2, item (y, k1), y fastest: outputs x = k1 + AX k2 < Nx (k2 < BX / 2), scaled
  {
    constexpr int IPT = (Ny * AX + XYB_THREADS - 1) / XYB_THREADS;
    float2 o[IPT][BX / 2];
#pragma unroll
    for (int u = 0; u < IPT; ++u) {
      const int it = threadIdx.x + u * XYB_THREADS;
      if (it < Ny * AX) {
        const int y = it % Ny, k1 = it / Ny;
        const float2* srow = buf + H::row_of(y) * PX;
        float2 v[BX];
#pragma unroll
        for (int n2 = 0; n2 < BX; ++n2) v[n2] = srow[BX * k1 + n2];
        fft_reg<BX, true, false>(v);
#pragma unroll
        for (int k2 = 0; k2 < BX / 2; ++k2) o[u][k2] = cscale(v[k2], scale);
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < IPT; ++u) {
      const int it = threadIdx.x + u * XYB_THREADS;
      if (it < Ny * AX) {
        const int y = it % Ny, k1 = it / Ny;
        float2* srow = buf + H::row_of(y) * PX;
#pragma unroll
        for (int k2 = 0; k2 < BX / 2; ++k2) srow[k1 + AX * k2] = o[u][k2];
      }
    }
  }
  __syncthreads();
  // store rows y < Ny, x < Nx (coalesced along x)
  {
    float2* dst = sig_out + (int64_t)g * (Nx * Ny);
    for (int e = threadIdx.x; e < Nx * Ny; e += XYB_THREADS) {
      const int x = e % Nx, y = e / Nx;
      dst[e] = buf[H::row_of(y) * PX + x];
    }
  }
}


}  // namespace fmmt
