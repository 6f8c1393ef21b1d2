// mma_probe2.cu -- lean tcgen05 issue loop (compile-time MMA mix, descriptors precomputed, issued by a
// warp-uniform warp 0 with elect.sync inside the asm): how close one CTA gets to the tcgen05 floor.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_probe2 scripts/mma_probe2.cu
#include <cstdio>
#include <vector>
#include "../paper_2010_00520_b200/csrc/tc.cuh"

using namespace fmmt;

__device__ __forceinline__ void mma_el(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync r|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit_el(uint32_t bar) {
  asm volatile("{\n\t.reg .pred e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\t"
               "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void wait_parity(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\tbra WAIT_%=;\n\tDONE_%=:\n\t}\n" ::"r"(bar), "r"(parity));
}

// MIX 0: per K-step A_hi x [B_hi;B_lo] (N = 2NR) + A_lo x B_hi (N = NR)  (the design's mix)
// MIX 2: one N = NR MMA per K-step
// MIX 6: per K-step 3 N = NR MMAs into 3 independent accumulators
template <int MIX, int NR, int DEPTH>
__global__ void __launch_bounds__(128, 1) probe(int rounds, long long* out) {
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
  const uint32_t tmem = __shfl_sync(0xffffffffu, slot, 0);
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const uint32_t sa = __shfl_sync(0xffffffffu, tc::smem_u32(sm), 0);
  const uint32_t bar0 = __shfl_sync(0xffffffffu, tc::smem_u32(bar), 0);
  constexpr uint32_t LBO_A = 128 * 16, LBO_B = 2 * NR * 16;
  constexpr uint32_t ID2 = tc::idesc_tf32(128, 2 * NR), ID1 = tc::idesc_tf32(128, NR);
  if (warp == 0) {
    const uint64_t dah = tc::sdesc(sa, LBO_A, 128), dal = tc::sdesc(sa + 8192, LBO_A, 128);
    const uint64_t dbh = tc::sdesc(sa + 16384, LBO_B, 128), dbl = tc::sdesc(sa + 16384 + NR * 16, LBO_B, 128);
    long long t0 = clock64();
    for (int c = 0; c < rounds; ++c) {
      if (c >= DEPTH) wait_parity(bar0 + ((c - DEPTH) & 7) * 8, ((c - DEPTH) >> 3) & 1);
      tc::fence_after_sync();
      const uint32_t tm = tmem + (c & 1) * (MIX == 6 ? NR : 2 * NR);
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const uint64_t oa = (ks * 2 * LBO_A) >> 4, ob = (ks * 2 * LBO_B) >> 4;
        if constexpr (MIX == 0) {
          mma_el(tm, dah + oa, dbh + ob, ID2, ks);
          mma_el(tm + NR, dal + oa, dbh + ob, ID1, 1);
        } else if constexpr (MIX == 2) {
          mma_el(tm, dah + oa, dbh + ob, ID1, ks);
        } else {
          mma_el(tm, dah + oa, dbh + ob, ID1, ks);
          mma_el(tmem + 2 * NR, dah + oa, dbl + ob, ID1, ks | (c > 0));
          mma_el(tmem + 3 * NR, dal + oa, dbh + ob, ID1, ks | (c > 0));
        }
      }
      commit_el(bar0 + (c & 7) * 8);
    }
    const int last = rounds - 1;
    wait_parity(bar0 + (last & 7) * 8, (last >> 3) & 1);
    if ((threadIdx.x & 31) == 0) out[blockIdx.x] = clock64() - t0;
  }
  tc::fence_before_sync();
  __syncthreads();
  if ((threadIdx.x >> 5) == 0) tc::tmem_dealloc<256>(tmem);
}

template <int MIX, int NR, int DEPTH>
void run(int nsm, long long* d, int cps) {
  const int rounds = 4000;
  const int smem = cps == 1 ? 200 * 1024 : 100 * 1024;
  cudaFuncSetAttribute(probe<MIX, NR, DEPTH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int grid = nsm * cps;
  probe<MIX, NR, DEPTH><<<grid, 128, smem>>>(rounds, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); exit(1); }
  std::vector<long long> h(grid);
  cudaMemcpy(h.data(), d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
  double mx = 0;
  for (auto v : h) mx = v > mx ? v : mx;
  const double cpc = mx / rounds;
  const int cols = MIX == 0 ? 3 * NR : MIX == 2 ? NR : 3 * NR;
  const double flop_chunk = 2.0 * 128 * cols * 8 * 2;
  const double tf = flop_chunk * rounds * grid / (mx / 1.9e9) / 1e12;
  const double floor = 2.0 * cols / 2.0;   // 128 x N x 8 tf32: N/2 cycles per MMA, 2 K-steps
  printf("mix %d NR %3d depth %d ctas/SM %d | %7.1f cyc/chunk/CTA %7.1f cyc/chunk/SM (floor %5.1f) %7.1f TF/s raw\n",
         MIX, NR, DEPTH, cps, cpc, cpc / cps, floor, tf);
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  long long* d;
  cudaMalloc(&d, 4096 * sizeof(long long));
  for (int cps : {1, 2}) {
    run<0, 64, 2>(nsm, d, cps);
    run<0, 64, 4>(nsm, d, cps);
    run<0, 32, 2>(nsm, d, cps);
    run<2, 64, 2>(nsm, d, cps);
    run<6, 64, 2>(nsm, d, cps);
    run<6, 32, 2>(nsm, d, cps);
  }
  return 0;
}
