// common.cuh -- shared device helpers of libfmmt (product side only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace fmmt {

// Packed FP32 pair arithmetic (sm_100: one FADD2 per complex add/sub).
__device__ __forceinline__ uint64_t pk2(float2 a) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
  return r;
}
__device__ __forceinline__ float2 upk2(uint64_t r) {
  float2 a;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
  return a;
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk2(a)), "l"(pk2(b)));
  return upk2(d);
}
__device__ __forceinline__ float2 csub(float2 a, float2 b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk2(a)), "l"(pk2(b)));
  return upk2(d);
}
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
// b * w = b.x (w.x, w.y) + b.y (-w.y, w.x): one FMUL2 + one FFMA2 (w a compile-time twiddle,
// so (-w.y, w.x) is a constant pair; for variable w the negation costs one FADD).
__device__ __forceinline__ float2 cmul2(float2 b, float2 w) {
  uint64_t t, r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(pk2(make_float2(b.x, b.x))), "l"(pk2(w)));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk2(make_float2(b.y, b.y))), "l"(pk2(make_float2(-w.y, w.x))),
      "l"(t));
  return upk2(r);
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
// acc += a * b  (4 FFMA)
__device__ __forceinline__ void cmac(float2& acc, float2 a, float2 b) {
  acc.x = fmaf(a.x, b.x, acc.x);
  acc.x = fmaf(-a.y, b.y, acc.x);
  acc.y = fmaf(a.x, b.y, acc.y);
  acc.y = fmaf(a.y, b.x, acc.y);
}

// acc += conj(a) * b  (4 FFMA)
__device__ __forceinline__ void cmac_conj(float2& acc, float2 a, float2 b) {
  acc.x = fmaf(a.x, b.x, acc.x);
  acc.x = fmaf(a.y, b.y, acc.x);
  acc.y = fmaf(a.x, b.y, acc.y);
  acc.y = fmaf(-a.y, b.x, acc.y);
}

__device__ __forceinline__ double2 zadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 zmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

template <int N> struct ILog2 { static constexpr int value = 1 + ILog2<N / 2>::value; };
template <> struct ILog2<1> { static constexpr int value = 0; };

__host__ __device__ constexpr int bitrev(int i, int bits) {
  int r = 0;
#pragma unroll
  for (int b = 0; b < 8; ++b)
    if (b < bits) r = (r << 1) | ((i >> b) & 1);
  return r;
}

}  // namespace fmmt
