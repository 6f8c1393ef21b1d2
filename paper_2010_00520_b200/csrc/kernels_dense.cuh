// kernels_dense.cuh -- the z-stage of the DENSE (uncompressed) FFT'ed operator: the baseline against which
// the paper states every overhead (Table I).
//
// Per (kx,ky) line of direction p: forward z-DFT of the half-padded spectrum W_p (a2), Hadamard with the
// stored T_p[kx,ky,:] (a5), inverse z-DFT truncated to z < Nz (a6) -- the same arithmetic as the low-rank
// z-stages, with T_p read from HBM instead of restored.  The op is bound by streaming T (16 B per padded grid
// point per direction; W stays in L2 between the xy FFTs and this kernel), so T does not go through registers:
// one thread issues the CTA's whole T tile ([N3][LPC] complex, 32 KB) as 1-D bulk async copies (TMA engine,
// L2 evict-first so the stream does not push W out of L2) at kernel start; the forward z-DFTs of the CTA's W
// lines run while the tile lands, and the Hadamard reads it from shared memory.  With the operator out of the
// register file three to four CTAs (12-16 warps, 96-128 KB of T in flight) fit on an SM.
#pragma once
#include "kernels_fft.cuh"
#include "tc.cuh"

namespace fmmt {

__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void bulk_g2s_hint(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(tc::smem_u32(bar)), "l"(pol)
      : "memory");
}

// Grid (ceil(n12 / LPC), nq), Z_THREADS threads, S threads per line (outputs k = S*m + h), LPC = Z_THREADS/S
// lines per CTA.  Requires n12 even (16-byte aligned rows of T; n1, n2 are powers of two >= 4).
template <int N3, int S>
__global__ void __launch_bounds__(Z_THREADS, (N3 >= 64 ? 3 : 4)) k_conv_z_dense(ZArgs a) {
  constexpr int M = N3 / S;
  constexpr int Nz = N3 / 2;
  constexpr int LPC = Z_THREADS / S;
  static_assert(S == 1 || S == 2, "z-line split must be 1 or 2");
  __shared__ __align__(128) float2 sT[N3 * LPC];
  __shared__ __align__(8) uint64_t bar;

  const int tid = threadIdx.x;
  const int h = (S == 1) ? 0 : (tid & (S - 1));
  const int l = tid / S;
  const int64_t ij0 = (int64_t)blockIdx.x * LPC;
  const int64_t ij = ij0 + l;
  const bool valid = ij < a.n12;
  const int q = blockIdx.y;
  const int p = a.p0 + q;

  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_barrier_init();
  }
  __syncthreads();
  if (tid == 0) {
    const int64_t nl = a.n12 - ij0 < LPC ? a.n12 - ij0 : (int64_t)LPC;
    const uint32_t bytes = (uint32_t)(nl * 8);
    const uint64_t pol = l2_evict_first_policy();
    tc::mbar_expect_tx(&bar, bytes * N3);
    const float2* src = a.T + (int64_t)p * N3 * a.n12 + ij0;
#pragma unroll 4
    for (int k = 0; k < N3; ++k) bulk_g2s_hint(tc::smem_u32(sT + k * LPC), src + (int64_t)k * a.n12, bytes, &bar, pol);
  }

  const int n12 = (int)a.n12;   // <= 2^16 lines: 32-bit line offsets (cheap to rematerialise, no spills)
  for (int cc = 0; cc < a.ncomp; ++cc) {
    float2* Wl = a.W + ((int64_t)q * a.ncomp + cc) * Nz * a.n12 + (valid ? ij : 0);
    float2 f[M];
    if constexpr (S == 1) {
#pragma unroll
      for (int z = 0; z < Nz; ++z) f[z] = valid ? Wl[z * n12] : make_float2(0.f, 0.f);
      fft_reg<N3, false, true>(f);
    } else {
      // X[2m + h] = DFT_M( a[z0] * W_N3^{h z0} )[m], z0 < M = Nz
#pragma unroll
      for (int z = 0; z < M; ++z) {
        float2 v = valid ? Wl[z * n12] : make_float2(0.f, 0.f);
        f[z] = (h && z) ? cmul(v, twc<N3, false>(z)) : v;
      }
      fft_reg<M, false, false>(f);
    }
    if (cc == 0) tc::mbar_wait(&bar, 0);
    // Hadamard (a5) with the stored operator line
#pragma unroll
    for (int m = 0; m < M; ++m) f[m] = cmul(sT[(S * m + h) * LPC + l], f[m]);
    fft_reg<M, true, false>(f);
    if constexpr (S == 1) {
      if (valid) {
#pragma unroll
        for (int z = 0; z < Nz; ++z) Wl[z * n12] = f[z];
      }
    } else {
      // y[z] = c_0[z] + W_N3^{-z} c_1[z], z < M; thread h keeps z in [h*M/2, (h+1)*M/2)
#pragma unroll
      for (int z = 1; z < M; ++z)
        if (h) f[z] = cmul(f[z], twc<N3, true>(z));
      float2 out[M / 2];
#pragma unroll
      for (int j = 0; j < M / 2; ++j) {
        float2 send = h ? f[j] : f[M / 2 + j];
        float2 mine = h ? f[M / 2 + j] : f[j];
        float2 recv;
        recv.x = __shfl_xor_sync(0xffffffffu, send.x, 1);
        recv.y = __shfl_xor_sync(0xffffffffu, send.y, 1);
        out[j] = cadd(mine, recv);
      }
      if (valid) {
#pragma unroll
        for (int j = 0; j < M / 2; ++j) Wl[(h * (M / 2) + j) * n12] = out[j];
      }
    }
  }
}


}  // namespace fmmt
