// kernels_fft.cuh -- the FFT stages of the translate hot path (eq. (5)).
//
// Per matvec and direction p the translation computes
//     B_p = trunc( F^{-1}( T_p (.) F( pad(A_p) ) ) )
// on the 2Nx x 2Ny x 2Nz circulant grid.  It is split into three stages whose
// intermediate is the "half-padded" spectrum W_p[z][ky][kx] (z < Nz, all kx,
// ky): 4K complex per direction, kept L2-resident by direction batching.
//   k_fwd_xy : pruned forward DFT along x (Nx nonzero of 2Nx) then along y
//              (Ny nonzero of 2Ny) of each input z-plane.            (a1, a2)
//   k_conv_z : per (kx,ky) line: restore T_p[kx,ky,:] in registers (a4), DFT
//              along z (pruned), Hadamard (a5), inverse DFT along z
//              truncated to z < Nz.  The restored operator never leaves the
//              thread's registers.                               (a2, a4, a5, a6)
//   k_inv_xy : inverse DFT along y then x, truncated to y < Ny, x < Nx,
//              scaled by 1/(n1 n2 n3), written to sig_out.           (a6)
#pragma once
#include "fft.cuh"

namespace fmmt {

constexpr int XY_THREADS = 256;
constexpr int Z_THREADS = 128;

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ void load_tw_smem(float2* stw) {
  for (int i = threadIdx.x; i < FMMT_TW_NMAX; i += blockDim.x) stw[i] = c_tw[i];
}

template <int NX, int NY> struct XYGeom {
  static constexpr int Nx = NX / 2, Ny = NY / 2;
  using SX = Split<NX>;
  using SY = Split<NY>;
  static constexpr int PA = NX + 1;                                  // row pitch of bufA
  static constexpr int XT = SX::two_pass ? SX::A * (SX::B + 1) : 0;  // padded x-pass-1 row pitch
  static constexpr int BUFA = Ny * PA;
  // the four-step scratch holds XR rows (x pass) / YC columns (y pass) at a time, so a 128 x 128 plane needs
  // 84 KB of shared memory (two CTAs per SM) instead of 197 KB
  static constexpr int XR = Ny < 16 ? Ny : 16;
  static constexpr int YC = NX < 16 ? NX : 16;
  static constexpr int BUFB_X = SX::two_pass ? XR * XT : 0;
  static constexpr int BUFB_Y = SY::two_pass ? NY * YC : 0;
  static constexpr int BUFB = BUFB_X > BUFB_Y ? BUFB_X : BUFB_Y;
  static constexpr int PLANE_SMEM = BUFA + BUFB;                     // complex elements per plane
};

// x-direction DFT of `rows` rows of a plane group held in bufA (row pitch PA).
// FWD: pruned input (x < Nx), full output (NX).  INV: full input, output x < Nx.
template <int NX, int NY, bool INV>
__device__ __forceinline__ void x_pass(float2* bufA, float2* bufB, const float2* stw, int nplanes,
                                       float scale) {
  using G = XYGeom<NX, NY>;
  using S = typename G::SX;
  constexpr int Ny = G::Ny, PA = G::PA;
  const int tid = threadIdx.x;
  if constexpr (!S::two_pass) {
    const int items = nplanes * Ny;
    for (int it = tid; it < items; it += blockDim.x) {
      const int j = it / Ny, y = it % Ny;
      float2* row = bufA + j * G::BUFA + y * PA;
      float2 v[NX];
      if (!INV) {
#pragma unroll
        for (int n = 0; n < NX / 2; ++n) v[n] = row[n];
        fft_reg<NX, false, true>(v);
#pragma unroll
        for (int k = 0; k < NX; ++k) row[k] = v[k];
      } else {
#pragma unroll
        for (int n = 0; n < NX; ++n) v[n] = row[n];
        fft_reg<NX, true, false>(v);
#pragma unroll
        for (int k = 0; k < NX / 2; ++k) row[k] = cscale(v[k], scale);
      }
    }
    __syncthreads();
  } else {
    constexpr int A = S::A, B = S::B, XT = G::XT, XR = G::XR;
    for (int y0 = 0; y0 < Ny; y0 += XR) {   // rows in chunks of XR (the scratch holds XR rows)
      // pass 1: item (row, n2), n2 fastest.  inputs n = B*n1 + n2.
      {
        const int items = nplanes * XR * B;
        for (int it = tid; it < items; it += blockDim.x) {
          const int n2 = it % B;
          const int r = it / B;
          const int j = r / XR, yl = r % XR;
          const float2* row = bufA + j * G::BUFA + (y0 + yl) * PA;
          float2* trow = bufB + j * G::BUFB + yl * XT;
          float2 v[A];
          if (!INV) {
#pragma unroll
            for (int n1 = 0; n1 < A / 2; ++n1) v[n1] = row[B * n1 + n2];
            fft_reg<A, false, true>(v);
          } else {
#pragma unroll
            for (int n1 = 0; n1 < A; ++n1) v[n1] = row[B * n1 + n2];
            fft_reg<A, true, false>(v);
          }
#pragma unroll
          for (int k1 = 0; k1 < A; ++k1) {
            float2 t = (k1 == 0) ? v[k1] : cmul(v[k1], tws<NX, INV>(stw, n2 * k1));
            trow[k1 * (B + 1) + n2] = t;
          }
        }
      }
      __syncthreads();
      // pass 2: item (row, k1), k1 fastest.  outputs k = k1 + A*k2.
      {
        const int items = nplanes * XR * A;
        for (int it = tid; it < items; it += blockDim.x) {
          const int k1 = it % A;
          const int r = it / A;
          const int j = r / XR, yl = r % XR;
          float2* row = bufA + j * G::BUFA + (y0 + yl) * PA;
          const float2* trow = bufB + j * G::BUFB + yl * XT;
          float2 v[B];
#pragma unroll
          for (int n2 = 0; n2 < B; ++n2) v[n2] = trow[k1 * (B + 1) + n2];
          fft_reg<B, INV, false>(v);
          if (!INV) {
#pragma unroll
            for (int k2 = 0; k2 < B; ++k2) row[k1 + A * k2] = v[k2];
          } else {
#pragma unroll
            for (int k2 = 0; k2 < B / 2; ++k2) row[k1 + A * k2] = cscale(v[k2], scale);
          }
        }
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------- k_fwd_xy
// grid.x = ceil(nplanes_total / ppc); plane g -> (q = g / Nz, z = g % Nz).
// in : sig_in + (q) * K  (already offset to the batch's first direction)
// out: W[q][z][ky][kx], n12 = NX*NY per plane.
template <int NX, int NY>
__global__ void __launch_bounds__(XY_THREADS)
k_fwd_xy(const float2* __restrict__ sig_in, float2* __restrict__ W, int nplanes_total, int ppc) {
  using G = XYGeom<NX, NY>;
  using SY = typename G::SY;
  constexpr int Nx = G::Nx, Ny = G::Ny, PA = G::PA;
  extern __shared__ float2 smem[];
  float2* stw = smem;
  float2* bufA = smem + FMMT_TW_NMAX;
  float2* bufB = bufA + ppc * G::BUFA;
  const int g0 = blockIdx.x * ppc;
  const int np = min(ppc, nplanes_total - g0);
  if (np <= 0) return;
  load_tw_smem(stw);
  // load input planes (coalesced along x)
  {
    const int per = Nx * Ny;
    const float2* src = sig_in + (int64_t)g0 * per;
    for (int e = threadIdx.x; e < np * per; e += blockDim.x) {
      const int j = e / per, r = e % per;
      const int y = r / Nx, x = r % Nx;
      bufA[j * G::BUFA + y * PA + x] = src[e];
    }
  }
  __syncthreads();
  x_pass<NX, NY, false>(bufA, bufB, stw, np, 1.0f);
  // y-direction: lines are columns kx of bufA (Ny nonzero rows), output NY rows to W.
  constexpr int n12 = NX * NY;
  float2* dst0 = W + (int64_t)g0 * n12;
  if constexpr (!SY::two_pass) {
    const int items = np * NX;
    for (int it = threadIdx.x; it < items; it += blockDim.x) {
      const int j = it / NX, x = it % NX;
      const float2* col = bufA + j * G::BUFA + x;
      float2 v[NY];
#pragma unroll
      for (int n = 0; n < NY / 2; ++n) v[n] = col[n * PA];
      fft_reg<NY, false, true>(v);
      float2* out = dst0 + (int64_t)j * n12 + x;
#pragma unroll
      for (int k = 0; k < NY; ++k) out[k * NX] = v[k];
    }
  } else {
    constexpr int A = SY::A, B = SY::B, YC = G::YC;
    for (int x0 = 0; x0 < NX; x0 += YC) {   // columns in chunks of YC (the scratch holds YC columns)
      {
        const int items = np * B * YC;
        for (int it = threadIdx.x; it < items; it += blockDim.x) {
          const int xl = it % YC;
          const int r = it / YC;
          const int n2 = r % B, j = r / B;
          const float2* col = bufA + j * G::BUFA + x0 + xl;
          float2* tcol = bufB + j * G::BUFB + xl;
          float2 v[A];
#pragma unroll
          for (int n1 = 0; n1 < A / 2; ++n1) v[n1] = col[(B * n1 + n2) * PA];
          fft_reg<A, false, true>(v);
#pragma unroll
          for (int k1 = 0; k1 < A; ++k1) {
            float2 t = (k1 == 0) ? v[k1] : cmul(v[k1], tws<NY, false>(stw, n2 * k1));
            tcol[(k1 * B + n2) * YC] = t;
          }
        }
      }
      __syncthreads();
      {
        const int items = np * A * YC;
        for (int it = threadIdx.x; it < items; it += blockDim.x) {
          const int xl = it % YC;
          const int r = it / YC;
          const int k1 = r % A, j = r / A;
          const float2* tcol = bufB + j * G::BUFB + xl;
          float2 v[B];
#pragma unroll
          for (int n2 = 0; n2 < B; ++n2) v[n2] = tcol[(k1 * B + n2) * YC];
          fft_reg<B, false, false>(v);
          float2* out = dst0 + (int64_t)j * n12 + x0 + xl;
#pragma unroll
          for (int k2 = 0; k2 < B; ++k2) out[(k1 + A * k2) * NX] = v[k2];
        }
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------- k_inv_xy
// in : W[q][z][ky][kx]; out: sig_out + (g) * K  planes [y][x], scaled.
template <int NX, int NY>
__global__ void __launch_bounds__(XY_THREADS)
k_inv_xy(const float2* __restrict__ W, float2* __restrict__ sig_out, int nplanes_total, int ppc,
         float scale) {
  using G = XYGeom<NX, NY>;
  using SY = typename G::SY;
  constexpr int Nx = G::Nx, Ny = G::Ny, PA = G::PA;
  constexpr int n12 = NX * NY;
  extern __shared__ float2 smem[];
  float2* stw = smem;
  float2* bufA = smem + FMMT_TW_NMAX;
  float2* bufB = bufA + ppc * G::BUFA;
  const int g0 = blockIdx.x * ppc;
  const int np = min(ppc, nplanes_total - g0);
  if (np <= 0) return;
  load_tw_smem(stw);
  __syncthreads();
  const float2* src0 = W + (int64_t)g0 * n12;
  // y-direction inverse: columns kx, full NY input rows, output rows y < Ny into bufA.
  if constexpr (!SY::two_pass) {
    const int items = np * NX;
    for (int it = threadIdx.x; it < items; it += blockDim.x) {
      const int j = it / NX, x = it % NX;
      const float2* in = src0 + (int64_t)j * n12 + x;
      float2 v[NY];
#pragma unroll
      for (int k = 0; k < NY; ++k) v[k] = in[k * NX];
      fft_reg<NY, true, false>(v);
      float2* col = bufA + j * G::BUFA + x;
#pragma unroll
      for (int y = 0; y < Ny; ++y) col[y * PA] = v[y];
    }
  } else {
    constexpr int A = SY::A, B = SY::B, YC = G::YC;
    for (int x0 = 0; x0 < NX; x0 += YC) {   // columns in chunks of YC
      {
        const int items = np * B * YC;
        for (int it = threadIdx.x; it < items; it += blockDim.x) {
          const int xl = it % YC;
          const int r = it / YC;
          const int n2 = r % B, j = r / B;
          const float2* in = src0 + (int64_t)j * n12 + x0 + xl;
          float2* tcol = bufB + j * G::BUFB + xl;
          float2 v[A];
#pragma unroll
          for (int n1 = 0; n1 < A; ++n1) v[n1] = in[(B * n1 + n2) * NX];
          fft_reg<A, true, false>(v);
#pragma unroll
          for (int k1 = 0; k1 < A; ++k1) {
            float2 t = (k1 == 0) ? v[k1] : cmul(v[k1], tws<NY, true>(stw, n2 * k1));
            tcol[(k1 * B + n2) * YC] = t;
          }
        }
      }
      __syncthreads();
      {
        const int items = np * A * YC;
        for (int it = threadIdx.x; it < items; it += blockDim.x) {
          const int xl = it % YC;
          const int r = it / YC;
          const int k1 = r % A, j = r / A;
          const float2* tcol = bufB + j * G::BUFB + xl;
          float2 v[B];
#pragma unroll
          for (int n2 = 0; n2 < B; ++n2) v[n2] = tcol[(k1 * B + n2) * YC];
          fft_reg<B, true, false>(v);
          float2* col = bufA + j * G::BUFA + x0 + xl;
#pragma unroll
          for (int k2 = 0; k2 < B / 2; ++k2) col[(k1 + A * k2) * PA] = v[k2];
        }
      }
      __syncthreads();
    }
  }
  __syncthreads();
  x_pass<NX, NY, true>(bufA, bufB, stw, np, scale);
  // store (coalesced along x)
  {
    const int per = Nx * Ny;
    float2* dst = sig_out + (int64_t)g0 * per;
    for (int e = threadIdx.x; e < np * per; e += blockDim.x) {
      const int j = e / per, r = e % per;
      const int y = r / Nx, x = r % Nx;
      dst[e] = bufA[j * G::BUFA + y * PA + x];
    }
  }
}

// ---------------------------------------------------------------- k_conv_z
enum ZMode { Z_DENSE = 0, Z_LOWRANK = 1, Z_RESTORE = 2 };

struct ZArgs {
  float2* W;                 // half-padded spectra [q][comp][Nz][n12] (from the batch's first direction)
  int64_t n12;
  int ncomp;                 // signature components sharing one restored T_p (theta, phi)
  int p0;                    // op-local index of the batch's first direction
  // low-rank factors: T_p[ij, k] = sum_c G_p[c][ij] * V_p(c, k)
  const float2* G;           // base
  const float* Gp;           // G pre-split for the tensor-core kernel (shared G only), or nullptr
  int64_t g_stride;          // per batch-local q (0 = shared G)
  const float2* V;           // base
  const int64_t* v_off;      // per op direction p (elements) or nullptr
  int64_t v_stride;          // per batch-local q when v_off == nullptr
  int64_t v_sc, v_sk;        // element (c, k) at V + off + c*v_sc + k*v_sk
  const int* rank_p;         // per op direction, or nullptr
  int rank;                  // uniform rank when rank_p == nullptr
  const float* Vp;           // V pre-split for the tensor-core kernel (k_tc_pack_b), or nullptr
  int64_t vp_stride;         // floats per batch-local q
  int z_blocked;             // tensor-core z-stage: direction-blocked tile order (shared A larger than L2 share)
  const float* amax;         // fp16-split scales: device max |G| (A) and max |V| (B); nullptr = unit scale
  const float* bmax;
  int64_t gp_stride;         // packed G (Gp) floats per batch-local q (0 = shared G)
  const int64_t* vp_off;     // packed V of op direction p at Vp + vp_off[p] (static per-direction factors), or nullptr
  // dense operator: T[p][k][ij]
  const float2* T;
  // restore output [k][ij]
  float2* Tout;
};

constexpr int Z_CH = 16;     // ranks staged per V chunk

template <int N3, int S, int MODE>
__global__ void __launch_bounds__(Z_THREADS)
k_conv_z(ZArgs a) {
  constexpr int M = N3 / S;          // DFT outputs owned per thread (k = S*m + h)
  constexpr int Nz = N3 / 2;
  constexpr int LPC = Z_THREADS / S; // lines per CTA
  constexpr int VP = M + 2;          // padded row of the staged V chunk
  static_assert(S == 1 || S == 2, "z-line split must be 1 or 2");
  __shared__ __align__(16) float2 sV[(MODE == Z_LOWRANK || MODE == Z_RESTORE) ? Z_CH * S * VP : 1];

  const int tid = threadIdx.x;
  const int h = (S == 1) ? 0 : (tid & (S - 1));
  const int64_t ij = (int64_t)blockIdx.x * LPC + tid / S;
  const bool valid = ij < a.n12;
  const int q = blockIdx.y;
  const int p = a.p0 + q;

  float2 t[M];   // restored T_p[ij, S*m + h]
  if constexpr (MODE == Z_DENSE) {
    const float2* Tp = a.T + (int64_t)p * N3 * a.n12;
#pragma unroll
    for (int m = 0; m < M; ++m) t[m] = valid ? Tp[(int64_t)(S * m + h) * a.n12 + ij] : make_float2(0.f, 0.f);
  } else {
#pragma unroll
    for (int m = 0; m < M; ++m) t[m] = make_float2(0.f, 0.f);
    const int r = a.rank_p ? a.rank_p[p] : a.rank;
    const float2* Gp = a.G + (int64_t)q * a.g_stride;
    const float2* Vp = a.V + (a.v_off ? a.v_off[p] : (int64_t)q * a.v_stride);
    const int64_t ijc = valid ? ij : 0;
    for (int c0 = 0; c0 < r; c0 += Z_CH) {
      __syncthreads();
      for (int e = tid; e < Z_CH * N3; e += Z_THREADS) {
        const int c = e / N3, k = e % N3;
        float2 v = make_float2(0.f, 0.f);
        if (c0 + c < r) v = Vp[(int64_t)(c0 + c) * a.v_sc + (int64_t)k * a.v_sk];
        sV[c * S * VP + (k % S) * VP + (k / S)] = v;
      }
      __syncthreads();
      float2 g[Z_CH];
#pragma unroll
      for (int c = 0; c < Z_CH; ++c) {
        const int cc = min(c0 + c, r - 1);
        g[c] = Gp[(int64_t)cc * a.n12 + ijc];
      }
#pragma unroll
      for (int c = 0; c < Z_CH; ++c) {
        const float4* vrow = reinterpret_cast<const float4*>(sV + c * S * VP + h * VP);
#pragma unroll
        for (int m2 = 0; m2 < M / 2; ++m2) {
          float4 vv = vrow[m2];
          cmac(t[2 * m2], g[c], make_float2(vv.x, vv.y));
          cmac(t[2 * m2 + 1], g[c], make_float2(vv.z, vv.w));
        }
      }
    }
  }

  if constexpr (MODE == Z_RESTORE) {
    if (valid) {
#pragma unroll
      for (int m = 0; m < M; ++m) a.Tout[(int64_t)(S * m + h) * a.n12 + ij] = t[m];
    }
    return;
  }

  // per signature component: forward z-DFT of this line of the half-padded spectrum
  // (z < Nz nonzero), Hadamard with the restored line t, inverse z-DFT truncated
  for (int cc = 0; cc < a.ncomp; ++cc) {
    float2* Wl = a.W + ((int64_t)q * a.ncomp + cc) * Nz * a.n12 + (valid ? ij : 0);
    float2 f[M];
    if constexpr (S == 1) {
#pragma unroll
      for (int z = 0; z < Nz; ++z) f[z] = valid ? Wl[(int64_t)z * a.n12] : make_float2(0.f, 0.f);
      fft_reg<N3, false, true>(f);
    } else {
      // X[2m + h] = DFT_M( a[z0] * W_N3^{h z0} )[m], z0 < M = Nz
#pragma unroll
      for (int z = 0; z < M; ++z) {
        float2 v = valid ? Wl[(int64_t)z * a.n12] : make_float2(0.f, 0.f);
        f[z] = (h && z) ? cmul(v, twc<N3, false>(z)) : v;
      }
      fft_reg<M, false, false>(f);
    }
    // Hadamard (a5): Y = T (.) A^
#pragma unroll
    for (int m = 0; m < M; ++m) f[m] = cmul(t[m], f[m]);
    // inverse z-DFT, truncated to z < Nz
    fft_reg<M, true, false>(f);
    if constexpr (S == 1) {
      if (valid) {
#pragma unroll
        for (int z = 0; z < Nz; ++z) Wl[(int64_t)z * a.n12] = f[z];
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
        for (int j = 0; j < M / 2; ++j) Wl[(int64_t)(h * (M / 2) + j) * a.n12] = out[j];
      }
    }
  }
}

// ---------------------------------------------------------------- direction sum
// partial[s][v] = sum_{p in split s} w[p] * sig[p][v]     (eq. (6) with P^- = 1)
__global__ void k_dirsum_partial(const float2* __restrict__ sig, const float* __restrict__ w,
                                 float2* __restrict__ partial, int64_t K, int ndir, int nsplit) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int s = blockIdx.y;
  if (v >= K) return;
  const int per = (ndir + nsplit - 1) / nsplit;
  const int pb = s * per, pe = min(ndir, pb + per);
  float2 acc = make_float2(0.f, 0.f);
  for (int p = pb; p < pe; ++p) {
    float2 b = sig[(int64_t)p * K + v];
    float ww = w[p];
    acc.x = fmaf(ww, b.x, acc.x);
    acc.y = fmaf(ww, b.y, acc.y);
  }
  partial[(int64_t)s * K + v] = acc;
}

// One warp per output element: lane s adds partials s, s + 32, ... (nsplit <= 64), then a
// shuffle reduction (the split count, not K, sets the parallelism when K is small).
__global__ void k_dirsum_final(const float2* __restrict__ partial, float2* __restrict__ out,
                               int64_t K, int nsplit) {
  const int64_t v = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (v >= K) return;
  float2 acc = make_float2(0.f, 0.f);
  for (int s = lane; s < nsplit; s += 32) acc = cadd(acc, partial[(int64_t)s * K + v]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
  }
  if (lane == 0) out[v] = acc;
}

}  // namespace fmmt
