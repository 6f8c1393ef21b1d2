// mma_probe.cu -- microbenchmark of the tcgen05 kind::tf32 issue pattern of tc_mainloop
// (no global loads, no conversion): cycles per K-chunk (2 K-steps) for a given MMA mix,
// completion-wait depth and CTAs per SM.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
//   -O3 -std=c++17 -o mma_probe scripts/mma_probe.cu ; run: ./mma_probe
#include <cstdio>
#include <vector>
#include "../paper_2010_00520_b200/csrc/tc.cuh"

using namespace fmmt;

__device__ __forceinline__ void mma_el(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync r|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit_el(uint64_t* bar) {
  asm volatile("{\n\t.reg .pred e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\t"
               "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(tc::smem_u32(bar))
               : "memory");
}

// mix 0: A_hi x [B_hi;B_lo] (N=2NR) + A_lo x B_hi (N=NR)     (2 MMAs / K-step, current design v7)
// mix 1: three N=NR MMAs                                      (3 MMAs / K-step)
// mix 2: one N=NR MMA                                         (plain TF32, lower bound)
__global__ void __launch_bounds__(128, 1) probe(int rounds, int depth, int NR, int mix, int ce, int wi, int flags, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[8];
  __shared__ uint32_t slot;
  if ((threadIdx.x >> 5) == 0) tc::tmem_alloc<256>(&slot);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) tc::mbar_init(&bar[i], 1);
    tc::fence_barrier_init();
  }
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = __shfl_sync(0xffffffffu, slot, 0);                 // warp-uniform for the compiler
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const uint32_t sa = __shfl_sync(0xffffffffu, tc::smem_u32(sm), 0), sl = sa + 8192, sb = sa + 16384;
  if (wi ? warp == 0 : threadIdx.x == 0) {
    const uint32_t LBO_A = 128 * 16, LBO_B = 2 * NR * 16;
    const uint32_t id2 = tc::idesc_tf32(128, 2 * NR), id1 = tc::idesc_tf32(128, NR);
    auto MMA = [&](uint32_t t, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
      if (wi) mma_el(t, a, b, id, acc); else tc::mma_tf32(t, a, b, id, acc);
    };
    long long t0 = clock64();
    for (int c = 0; c < rounds; ++c) {
      if (!(flags & 1) && c % ce == 0 && c / ce >= depth) {
        const int w = c / ce - depth;
        tc::mbar_wait(&bar[w & 7], (w >> 3) & 1);
      }
      if (!(flags & 2)) tc::fence_after_sync();
      const uint32_t tm = tmem + (mix == 4 ? 0 : mix == 5 ? (c & 1) * NR : (4 * NR <= 256 ? (c & 1) * 2 * NR : 0));
      for (int ks = 0; ks < 2; ++ks) {
        const uint64_t ah = tc::sdesc(sa + ks * 2 * LBO_A, LBO_A, 128);
        const uint64_t al = tc::sdesc(sl + ks * 2 * LBO_A, LBO_A, 128);
        const uint64_t bh = tc::sdesc(sb + ks * 2 * LBO_B, LBO_B, 128);
        const uint64_t bl = tc::sdesc(sb + ks * 2 * LBO_B + NR * 16, LBO_B, 128);
        if (mix == 0) {
          MMA(tm, ah, bh, id2, ks);
          MMA(tm + NR, al, bh, id1, 1);
        } else if (mix == 1) {
          MMA(tm, ah, bh, id1, ks);
          MMA(tm + NR, ah, bl, id1, ks);
          MMA(tm + NR, al, bh, id1, 1);
        } else if (mix == 2) {
          MMA(tm, ah, bh, id1, ks);
        } else if (mix == 3) {                       // two independent N=NR chains, interleaved
          MMA(tm, ah, bh, id1, ks);
          MMA(tm + NR, al, bh, id1, ks);
        } else if (mix == 5) {                       // 3 independent chains: hh (slot), hl, lh (own blocks)
          MMA(tm, ah, bh, id1, ks);
          MMA(tmem + 2 * NR, ah, bl, id1, ks | (c > 0));
          MMA(tmem + 3 * NR, al, bh, id1, ks | (c > 0));
        } else {                                     // mix 0 twice on independent accumulators
          MMA(tm, ah, bh, id2, ks);
          MMA(tm + 4 * NR, ah, bh, id2, ks);
          MMA(tm + NR, al, bh, id1, 1);
          MMA(tm + 5 * NR, al, bh, id1, 1);
        }
      }
      if (c % ce == ce - 1) { if (wi) commit_el(&bar[(c / ce) & 7]); else tc::mma_commit(&bar[(c / ce) & 7]); }
    }
    const int last = rounds / ce - 1;
    tc::mbar_wait(&bar[last & 7], (last >> 3) & 1);
    if ((threadIdx.x & 31) == 0) out[blockIdx.x] = clock64() - t0;
  }
  tc::fence_before_sync();
  __syncthreads();
  if ((threadIdx.x >> 5) == 0) tc::tmem_dealloc<256>(tmem);
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  long long* d;
  cudaMalloc(&d, 4096 * sizeof(long long));
  const int rounds = 4000;
  setvbuf(stdout, nullptr, _IONBF, 0);
  printf("mix NR depth ctas/SM commit-every | cycles/chunk/CTA  cycles/chunk/SM  tf32-TFLOP/s(chip, 1.9GHz)\n");
  for (int flags : {0})
  for (int wi : {0, 1})
  for (int mix : {0, 1, 2, 5})
    for (int NR : {32, 64})
      for (int cps : {1, 2})
        for (int ce : {1})
        for (int depth : {2}) {
          if (mix == 4 && NR != 32) continue;   // N = 256 is the UMMA max: NR = 128 -> 2NR = 256 ok, but TMEM 4NR > 256
          const int smem = cps == 1 ? 200 * 1024 : 100 * 1024;
          cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
          const int grid = nsm * cps;
          probe<<<grid, 128, smem>>>(rounds, depth, NR, mix, ce, wi, flags, d);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
          std::vector<long long> h(grid);
          cudaMemcpy(h.data(), d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
          double mx = 0;
          for (auto v : h) mx = v > mx ? v : mx;
          const double cpc = mx / rounds;
          const int nmma_cols = mix == 0 ? 3 * NR : mix == 1 ? 3 * NR : mix == 2 ? NR : mix == 3 ? 2 * NR : mix == 5 ? 3 * NR : 6 * NR;   // total N per K-step
          const double flop_chunk = 2.0 * 128 * nmma_cols * 8 * 2;          // 2 K-steps of K=8
          const double tf = flop_chunk * rounds * grid / (mx / 1.9e9) / 1e12;
          printf("flags=%d wi=%d %d %3d %d %d ce=%d | %8.1f %8.1f %8.1f\n", flags, wi, mix, NR, depth, cps, ce, cpc, cpc / cps, tf);
        }
  return 0;
}
