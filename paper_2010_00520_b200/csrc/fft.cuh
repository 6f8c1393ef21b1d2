// fft.cuh -- register-resident complex64 FFTs used by every translate stage.
//
// The 3D DFT of eq. (5) is separable; every stage of the hot path
// runs 1D DFTs of length <= 32 entirely in one thread's registers (radix-2
// DIT, fully unrolled, twiddles from constant memory at compile-time indices)
// and composes longer lines with the four-step factorisation N = A*B through
// shared memory (kernels_fft.cuh).  Forward kernel e^{-2 pi i m f / N},
// unnormalised; inverse e^{+...}, unnormalised (1/n applied once at the end).
#pragma once
#include "common.cuh"
#include "twiddles.cuh"

namespace fmmt {

// W_M^k = exp(-+ 2 pi i k / M) for compile-time M, k (after unrolling).
template <int M, bool INV>
__device__ __forceinline__ float2 twc(int k) {
  float2 w = c_tw[(k * (FMMT_TW_NMAX / M)) & (FMMT_TW_NMAX - 1)];
  return INV ? make_float2(w.x, -w.y) : w;
}

// Multiply b by W_SPAN^j with the trivial cases (j = 0, j = SPAN/4) free.
template <int SPAN, bool INV>
__device__ __forceinline__ float2 twmul(float2 b, int j) {
  if (j == 0) return b;
  if (SPAN >= 4 && 4 * j == SPAN) {
    // forward: * (-i) = (y, -x); inverse: * (+i) = (-y, x)
    return INV ? make_float2(-b.y, b.x) : make_float2(b.y, -b.x);
  }
  return cmul2(b, twc<SPAN, INV>(j));
}

// Radix-2 butterfly stages of span SPAN, 2 SPAN, ..., M (compile-time recursion, so
// every index and twiddle is a constant: no local-memory arrays).
template <int M, bool INV, int SPAN>
__device__ __forceinline__ void fft_stages(float2 (&y)[M]) {
  constexpr int half = SPAN / 2;
#pragma unroll
  for (int g = 0; g < M; g += SPAN) {
#pragma unroll
    for (int j = 0; j < half; ++j) {
      const float2 a = y[g + j];
      const float2 b = twmul<SPAN, INV>(y[g + j + half], j);
      y[g + j] = cadd(a, b);
      y[g + j + half] = csub(a, b);
    }
  }
  if constexpr (SPAN < M) fft_stages<M, INV, 2 * SPAN>(y);
}

// In-place M-point DFT of x (natural order in and out).
// PRUNED: x[M/2 .. M) are known to be zero and are not read (the zero-padded
// upper half of eq. (5)'s Toeplitz embedding).
template <int M, bool INV, bool PRUNED = false>
__device__ __forceinline__ void fft_reg(float2 (&x)[M]) {
  if constexpr (M > 1) {
    constexpr int LG = ILog2<M>::value;
    float2 y[M];
    // bit-reversed load; odd positions hold x[>= M/2]
#pragma unroll
    for (int i = 0; i < M; ++i) {
      if (!PRUNED || (i % 2) == 0) y[i] = x[bitrev(i, LG)];
    }
    // stage span 2 (twiddle 1)
#pragma unroll
    for (int t = 0; t < M / 2; ++t) {
      float2 a = y[2 * t];
      if (PRUNED) {
        y[2 * t + 1] = a;
      } else {
        float2 b = y[2 * t + 1];
        y[2 * t] = cadd(a, b);
        y[2 * t + 1] = csub(a, b);
      }
    }
    if constexpr (M >= 4) fft_stages<M, INV, 4>(y);
#pragma unroll
    for (int i = 0; i < M; ++i) x[i] = y[i];
  }
}

// Twiddle W_N^e for runtime e from a shared-memory copy of c_tw.
template <int N, bool INV>
__device__ __forceinline__ float2 tws(const float2* __restrict__ stw, int e) {
  float2 w = stw[(e * (FMMT_TW_NMAX / N)) & (FMMT_TW_NMAX - 1)];
  return INV ? make_float2(w.x, -w.y) : w;
}

// Four-step split N = A * B used for lines longer than 32 points.
template <int N> struct Split {
  static constexpr int A = (N <= 32) ? N : (N == 64 ? 8 : 16);   // first-pass DFT length
  static constexpr int B = N / A;                                // second-pass DFT length
  static constexpr bool two_pass = (N > 32);
};

}  // namespace fmmt
