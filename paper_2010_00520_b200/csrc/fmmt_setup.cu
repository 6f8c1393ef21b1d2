// fmmt_setup.cu -- setup-time stages of libfmmt (not the per-matvec hot path):
//   * multipole count and direction grid,
//   * the FP64 FFT'ed translation operator on the circulant grid (eq. (7)),
//   * the FP64 compressors of the Appendix (Alg. 1 Tucker-SVD, Alg. 2 H-Tucker-SVD,
//     Alg. 3 TT-SVD) on the GPU with cuBLAS / cuSOLVER / cuFFT.
// The paper notes compression runs once in the setup stage; library
// routines are used here for the dense FP64 factorizations.
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cufft.h>
#include <cusolverDn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "fmmt_internal.h"

using fmmt_internal::set_err;
typedef cuDoubleComplex zc;

#define SETUP_CUBLAS(ctx, call)                                                                     \
  do {                                                                                             \
    cublasStatus_t s_ = (call);                                                                    \
    if (s_ != CUBLAS_STATUS_SUCCESS)                                                               \
      return set_err((ctx), FMMT_E_CUDA, "%s:%d cuBLAS %s -> %d", __FILE__, __LINE__, #call, (int)s_); \
  } while (0)
#define SETUP_CUSOLVER(ctx, call)                                                                     \
  do {                                                                                               \
    cusolverStatus_t s_ = (call);                                                                    \
    if (s_ != CUSOLVER_STATUS_SUCCESS)                                                               \
      return set_err((ctx), FMMT_E_CUDA, "%s:%d cuSOLVER %s -> %d", __FILE__, __LINE__, #call, (int)s_); \
  } while (0)
#define SETUP_TRY(expr)              \
  do {                               \
    fmmt_status st_ = (expr);        \
    if (st_ != FMMT_OK) return st_;  \
  } while (0)

void fmmt_internal::setup_release(fmmt_ctx* ctx) {
  if (ctx->blas) cublasDestroy((cublasHandle_t)ctx->blas);
  if (ctx->solver) cusolverDnDestroy((cusolverDnHandle_t)ctx->solver);
  ctx->blas = ctx->solver = nullptr;
}

static fmmt_status handles(fmmt_ctx* ctx, cublasHandle_t* b, cusolverDnHandle_t* s) {
  if (!ctx->blas) {
    cublasHandle_t h;
    if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) return set_err(ctx, FMMT_E_CUDA, "cublasCreate failed");
    ctx->blas = h;
  }
  if (!ctx->solver) {
    cusolverDnHandle_t h;
    if (cusolverDnCreate(&h) != CUSOLVER_STATUS_SUCCESS) return set_err(ctx, FMMT_E_CUDA, "cusolverDnCreate failed");
    ctx->solver = h;
  }
  *b = (cublasHandle_t)ctx->blas;
  *s = (cusolverDnHandle_t)ctx->solver;
  cublasSetStream(*b, ctx->stream);
  cusolverDnSetStream(*s, ctx->stream);
  return FMMT_OK;
}

// ============================================================== direction grid (host)
// Gauss-Legendre nodes/weights on [-1,1] by Newton iteration on P_{n}.
static void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& w) {
  x.assign(n, 0.0);
  w.assign(n, 0.0);
  for (int i = 0; i < n; ++i) {
    double z = std::cos(M_PI * (i + 0.75) / (n + 0.5));
    double dp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = z;
      for (int l = 2; l <= n; ++l) {
        double p2 = ((2.0 * l - 1.0) * z * p1 - (l - 1.0) * p0) / l;
        p0 = p1;
        p1 = p2;
      }
      if (n == 1) { p1 = z; p0 = 1.0; }
      dp = n * (z * p1 - p0) / (z * z - 1.0);
      double dz = p1 / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-16) break;
    }
    // recompute derivative at the converged node
    double p0 = 1.0, p1 = z;
    for (int l = 2; l <= n; ++l) {
      double p2 = ((2.0 * l - 1.0) * z * p1 - (l - 1.0) * p0) / l;
      p0 = p1;
      p1 = p2;
    }
    if (n == 1) { p1 = z; p0 = 1.0; }
    dp = n * (z * p1 - p0) / (z * z - 1.0);
    x[i] = z;
    w[i] = 2.0 / ((1.0 - z * z) * dp * dp);
  }
  // ascending order
  std::vector<int> idx(n);
  for (int i = 0; i < n; ++i) idx[i] = i;
  std::sort(idx.begin(), idx.end(), [&](int a, int b) { return x[a] < x[b]; });
  std::vector<double> xs(n), ws(n);
  for (int i = 0; i < n; ++i) { xs[i] = x[idx[i]]; ws[i] = w[idx[i]]; }
  x = xs;
  w = ws;
}

extern "C" fmmt_status fmmt_multipole_count(double k_abs, double edge, double digits, int64_t* L) {
  if (!L || !(k_abs > 0) || !(edge > 0) || !(digits > 0)) return FMMT_E_ARG;
  const double Rs = std::sqrt(3.0) / 2.0 * edge;     // P:55 enclosing-sphere radius
  const double x = 2.0 * k_abs * Rs;
  *L = (int64_t)std::floor(x + 1.8 * std::pow(digits, 2.0 / 3.0) * std::cbrt(x));
  if (*L < 1) *L = 1;
  return FMMT_OK;
}

extern "C" fmmt_status fmmt_direction_grid(int64_t L, int64_t nphi, double* khat, double* w) {
  if (L < 0 || nphi < 1) return FMMT_E_ARG;
  std::vector<double> x, wg;
  gauss_legendre((int)L + 1, x, wg);
  for (int64_t i = 0; i <= L; ++i) {
    const double st = std::sqrt(std::max(0.0, 1.0 - x[i] * x[i]));
    for (int64_t j = 0; j < nphi; ++j) {
      const int64_t p = i * nphi + j;
      const double phi = 2.0 * M_PI * (double)j / (double)nphi;
      if (khat) {
        khat[3 * p + 0] = st * std::cos(phi);
        khat[3 * p + 1] = st * std::sin(phi);
        khat[3 * p + 2] = x[i];
      }
      if (w) w[p] = wg[i] * 2.0 * M_PI / (double)nphi;
    }
  }
  return FMMT_OK;
}

// ============================================================== operator builder
constexpr int LMAX = 160;

// T~_p[m] of eq. (7) (l = 0..L, prefactor omitted) at every circulant index of
// the padded grid for directions [0, nd).  One thread per (point, direction).
__global__ void k_spatial_operator(double2* __restrict__ out, int n1, int n2, int n3, double edge, double k, int L,
                                   const double* __restrict__ khat, int nd) {
  const int64_t n = (int64_t)n1 * n2 * n3;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int p = blockIdx.y;
  if (idx >= n || p >= nd) return;
  const int i1 = (int)(idx % n1), i2 = (int)((idx / n1) % n2), i3 = (int)(idx / ((int64_t)n1 * n2));
  const int N1 = n1 / 2, N2 = n2 / 2, N3 = n3 / 2;
  double2 res = make_double2(0.0, 0.0);
  // circulant offsets; the m = N planes carry no offset (zero)
  const bool onplane = (i1 == N1) || (i2 == N2) || (i3 == N3);
  const int ux = i1 < N1 ? i1 : i1 - n1;
  const int uy = i2 < N2 ? i2 : i2 - n2;
  const int uz = i3 < N3 ? i3 : i3 - n3;
  const int u2 = ux * ux + uy * uy + uz * uz;
  if (!onplane && u2 > 12) {   // far iff R > kappa R^s = 2 sqrt(3) edge  <=>  |u|^2 > 12
    const double un = sqrt((double)u2);
    const double R = edge * un;
    const double c = (ux * khat[3 * p] + uy * khat[3 * p + 1] + uz * khat[3 * p + 2]) / un;
    const double z = k * R;
    double sz, cz;
    sincos(z, &sz, &cz);
    // spherical Bessel j_l: upward if z > L, else Miller downward normalised by j_0
    double jl[LMAX + 2];
    const double j0x = sz / z, j1x = sz / (z * z) - cz / z;
    if (z > L + 1) {
      jl[0] = j0x;
      jl[1] = j1x;
      for (int l = 1; l < L; ++l) jl[l + 1] = (2 * l + 1) / z * jl[l] - jl[l - 1];
    } else {
      // Miller: downward from ls with j_{ls+1} = 0, j_ls = 1, rescaled against overflow
      const int ls = L + 40 + (int)z;
      const int Ls = L < 1 ? 1 : L;
      double jp1 = 0.0, jc = 1.0;
      for (int l = ls; l >= 1; --l) {
        if (l <= Ls) jl[l] = jc;
        const double jm1 = (2 * l + 1) / z * jc - jp1;
        jp1 = jc;
        jc = jm1;
        if (fabs(jc) > 1e200) {
          jc *= 1e-200;
          jp1 *= 1e-200;
          for (int t = l; t <= Ls; ++t) jl[t] *= 1e-200;
        }
      }
      jl[0] = jc;
      const double scale = (fabs(j0x) >= fabs(j1x)) ? j0x / jl[0] : j1x / jl[1];
      for (int l = 0; l <= Ls; ++l) jl[l] *= scale;
    }
    // y_l upward (stable), Legendre upward
    double ym1 = -cz / z;                      // y_0
    double y0 = -cz / (z * z) - sz / z;        // y_1
    double Pm1 = 1.0, P0 = c;
    for (int l = 0; l <= L; ++l) {
      double yl, Pl;
      if (l == 0) { yl = ym1; Pl = 1.0; }
      else if (l == 1) { yl = y0; Pl = c; }
      else {
        const double yn = (2 * l - 1) / z * y0 - ym1;
        ym1 = y0; y0 = yn; yl = yn;
        const double Pn = ((2 * l - 1) * c * P0 - (l - 1) * Pm1) / l;
        Pm1 = P0; P0 = Pn; Pl = Pn;
      }
      // (-j)^l (2l+1) h_l^(2)(z) P_l(c),  h^(2) = j_l - i y_l
      const double hr = jl[l], hi = -yl;
      const double f = (2 * l + 1) * Pl;
      double tr, ti;
      switch (l & 3) {
        case 0: tr = hr; ti = hi; break;          // 1
        case 1: tr = hi; ti = -hr; break;         // -i
        case 2: tr = -hr; ti = -hi; break;        // -1
        default: tr = -hi; ti = hr; break;        // +i
      }
      res.x += f * tr;
      res.y += f * ti;
    }
  }
  out[(int64_t)p * n + idx] = res;
}

// Lossy medium (complex k): h_l^(2)(z) for complex z = kR by the upward
// recurrence h_{l+1} = (2l+1)/z h_l - h_{l-1} from h_0 = j e^{-jz}/z, h_1 = e^{-jz}(j - z)/z^2
// (h^(2) is the dominant solution, so the upward recurrence is stable).
__device__ __forceinline__ double2 zdiv(double2 a, double2 b) {
  const double den = b.x * b.x + b.y * b.y;
  return make_double2((a.x * b.x + a.y * b.y) / den, (a.y * b.x - a.x * b.y) / den);
}

__global__ void k_spatial_operator_c(double2* __restrict__ out, int n1, int n2, int n3, double edge, double kr,
                                     double ki, int L, const double* __restrict__ khat, int nd) {
  const int64_t n = (int64_t)n1 * n2 * n3;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int p = blockIdx.y;
  if (idx >= n || p >= nd) return;
  const int i1 = (int)(idx % n1), i2 = (int)((idx / n1) % n2), i3 = (int)(idx / ((int64_t)n1 * n2));
  const int N1 = n1 / 2, N2 = n2 / 2, N3 = n3 / 2;
  double2 res = make_double2(0.0, 0.0);
  const bool onplane = (i1 == N1) || (i2 == N2) || (i3 == N3);
  const int ux = i1 < N1 ? i1 : i1 - n1;
  const int uy = i2 < N2 ? i2 : i2 - n2;
  const int uz = i3 < N3 ? i3 : i3 - n3;
  const int u2 = ux * ux + uy * uy + uz * uz;
  if (!onplane && u2 > 12) {   // far iff |u|^2 > 12 (kappa = 4)
    const double un = sqrt((double)u2);
    const double R = edge * un;
    const double c = (ux * khat[3 * p] + uy * khat[3 * p + 1] + uz * khat[3 * p + 2]) / un;
    const double2 z = make_double2(kr * R, ki * R);
    // e^{-jz} = e^{Im z} (cos Re z - j sin Re z)
    double sr, cr;
    sincos(z.x, &sr, &cr);
    const double ea = exp(z.y);
    const double2 emj = make_double2(ea * cr, -ea * sr);
    const double2 h0 = zdiv(make_double2(-emj.y, emj.x), z);                        // j e^{-jz} / z
    const double2 z2 = fmmt::zmul(z, z);
    const double2 h1 = zdiv(fmmt::zmul(emj, make_double2(-z.x, 1.0 - z.y)), z2);         // e^{-jz} (j - z) / z^2
    double2 hm1 = h0, hc = h1;
    double Pm1 = 1.0, P0 = c;
    for (int l = 0; l <= L; ++l) {
      double2 hl;
      double Pl;
      if (l == 0) { hl = h0; Pl = 1.0; }
      else if (l == 1) { hl = h1; Pl = c; }
      else {
        const double2 t = zdiv(make_double2((2 * l - 1) * hc.x, (2 * l - 1) * hc.y), z);
        const double2 hn = make_double2(t.x - hm1.x, t.y - hm1.y);
        hm1 = hc; hc = hn; hl = hn;
        const double Pn = ((2 * l - 1) * c * P0 - (l - 1) * Pm1) / l;
        Pm1 = P0; P0 = Pn; Pl = Pn;
      }
      const double f = (2 * l + 1) * Pl;
      double tr, ti;
      switch (l & 3) {                  // (-j)^l h_l
        case 0: tr = hl.x; ti = hl.y; break;
        case 1: tr = hl.y; ti = -hl.x; break;
        case 2: tr = -hl.x; ti = -hl.y; break;
        default: tr = -hl.y; ti = hl.x; break;
      }
      res.x += f * tr;
      res.y += f * ti;
    }
  }
  out[(int64_t)p * n + idx] = res;
}

static fmmt_status build_operator_impl(fmmt_ctx* ctx, int64_t Nx, int64_t Ny, int64_t Nz, double edge, double k,
                                       double k_im, int64_t L, const double* khat, int64_t ndir, fmmt_c128* T) {
  if (!ctx) return FMMT_E_ARG;
  if (!khat || !T) return set_err(ctx, FMMT_E_ARG, "null pointer");
  if (Nx < 1 || Ny < 1 || Nz < 1 || ndir < 1 || L < 0 || L > LMAX - 1 || !(edge > 0) || !(k > 0) || k_im > 0)
    return set_err(ctx, FMMT_E_ARG, "bad operator parameters");
  cudaSetDevice(ctx->device);
  const int n1 = (int)(2 * Nx), n2 = (int)(2 * Ny), n3 = (int)(2 * Nz);
  const int64_t n = (int64_t)n1 * n2 * n3;
  double* dk = nullptr;
  FMMT_CUDA(ctx, cudaMalloc(&dk, ndir * 3 * sizeof(double)));
  FMMT_CUDA(ctx, cudaMemcpyAsync(dk, khat, ndir * 3 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  const int64_t chunk = 16384;
  for (int64_t p0 = 0; p0 < ndir; p0 += chunk) {
    const int nd = (int)std::min<int64_t>(chunk, ndir - p0);
    dim3 grid((unsigned)((n + 127) / 128), (unsigned)nd);
    if (k_im == 0.0)
      k_spatial_operator<<<grid, 128, 0, ctx->stream>>>(reinterpret_cast<double2*>(T) + p0 * n, n1, n2, n3, edge, k,
                                                        (int)L, dk + 3 * p0, nd);
    else
      k_spatial_operator_c<<<grid, 128, 0, ctx->stream>>>(reinterpret_cast<double2*>(T) + p0 * n, n1, n2, n3, edge, k,
                                                          k_im, (int)L, dk + 3 * p0, nd);
    FMMT_CUDA(ctx, cudaGetLastError());
  }
  // T = F(T~): unnormalised forward 3D DFT, batched over directions
  cufftHandle plan;
  int dims[3] = {n3, n2, n1};   // cuFFT row-major: last dim fastest
  // batches of <= 2^28 points (4 GB of complex128) so that cuFFT's work area stays small next to the
  // operator (the 256^3 x 435 sweep operator alone is 117 GB)
  const int64_t maxb = std::max<int64_t>(1, std::min<int64_t>(ndir, (int64_t)(1ll << 28) / n));
  if (cufftPlanMany(&plan, 3, dims, nullptr, 1, (int)n, nullptr, 1, (int)n, CUFFT_Z2Z, (int)maxb) != CUFFT_SUCCESS) {
    cudaFree(dk);
    return set_err(ctx, FMMT_E_CUDA, "cufftPlanMany failed");
  }
  cufftSetStream(plan, ctx->stream);
  for (int64_t p0 = 0; p0 + maxb <= ndir; p0 += maxb) {
    cufftDoubleComplex* ptr = reinterpret_cast<cufftDoubleComplex*>(T) + p0 * n;
    if (cufftExecZ2Z(plan, ptr, ptr, CUFFT_FORWARD) != CUFFT_SUCCESS) {
      cufftDestroy(plan);
      cudaFree(dk);
      return set_err(ctx, FMMT_E_CUDA, "cufftExecZ2Z failed");
    }
  }
  cufftDestroy(plan);
  const int64_t rem = ndir % maxb;
  if (rem) {
    if (cufftPlanMany(&plan, 3, dims, nullptr, 1, (int)n, nullptr, 1, (int)n, CUFFT_Z2Z, (int)rem) != CUFFT_SUCCESS) {
      cudaFree(dk);
      return set_err(ctx, FMMT_E_CUDA, "cufftPlanMany failed");
    }
    cufftSetStream(plan, ctx->stream);
    cufftDoubleComplex* ptr = reinterpret_cast<cufftDoubleComplex*>(T) + (ndir - rem) * n;
    cufftExecZ2Z(plan, ptr, ptr, CUFFT_FORWARD);
    cufftDestroy(plan);
  }
  FMMT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  cudaFree(dk);
  return FMMT_OK;
}

extern "C" fmmt_status fmmt_build_operator(fmmt_ctx* ctx, int64_t Nx, int64_t Ny, int64_t Nz, double edge, double k,
                                           int64_t L, const double* khat, int64_t ndir, fmmt_c128* T) {
  return build_operator_impl(ctx, Nx, Ny, Nz, edge, k, 0.0, L, khat, ndir, T);
}

extern "C" fmmt_status fmmt_build_operator_lossy(fmmt_ctx* ctx, int64_t Nx, int64_t Ny, int64_t Nz, double edge,
                                                 double k_re, double k_im, int64_t L, const double* khat,
                                                 int64_t ndir, fmmt_c128* T) {
  return build_operator_impl(ctx, Nx, Ny, Nz, edge, k_re, k_im, L, khat, ndir, T);
}

// ============================================================== FP64 helpers
// At[(l + L r), i] = conj(T[l + L (i + n r)]): conjugate transpose of the
// mode unfolding (mode size n, L = product of earlier modes, R = later modes).
__global__ void k_unfold_h(const double2* __restrict__ T, double2* __restrict__ At, int64_t L, int64_t n, int64_t R) {
  const int64_t total = L * n * R;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = e % L;
    const int64_t i = (e / L) % n;
    const int64_t r = e / (L * n);
    const double2 v = T[e];
    At[(l + L * r) + L * R * i] = make_double2(v.x, -v.y);
  }
}

__global__ void k_conj(const double2* __restrict__ a, double2* __restrict__ b, int64_t n) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    b[e] = make_double2(a[e].x, -a[e].y);
}

// copy the upper triangle of the leading n x n block of A (lda) into R (n x n), zero below
__global__ void k_upper(const double2* __restrict__ A, int64_t lda, double2* __restrict__ R, int64_t n) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % n, j = e / n;
    R[e] = (i <= j) ? A[i + lda * j] : make_double2(0.0, 0.0);
  }
}

__global__ void k_z2c(const double2* __restrict__ a, float2* __restrict__ b, int64_t n) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    b[e] = make_float2((float)a[e].x, (float)a[e].y);
}

static unsigned nblk(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 32)); }

// RAII device buffer
struct DBuf {
  void* p = nullptr;
  ~DBuf() { if (p) cudaFree(p); }
  template <class T> T* as() { return reinterpret_cast<T*>(p); }
};
static fmmt_status dalloc(fmmt_ctx* ctx, DBuf& b, int64_t bytes) {
  if (b.p) { cudaFree(b.p); b.p = nullptr; }
  cudaError_t e = cudaMalloc(&b.p, std::max<int64_t>(bytes, 16));
  if (e != cudaSuccess) return set_err(ctx, FMMT_E_NOMEM, "setup cudaMalloc(%lld) failed: %s", (long long)bytes, cudaGetErrorString(e));
  return FMMT_OK;
}

// Truncation (reading Q7): r = min{r >= 1 : ||sigma[r:]||_2 <= delta}.
static int64_t tail_rank(const std::vector<double>& s, double delta) {
  const int64_t n = (int64_t)s.size();
  std::vector<double> tail(n + 1, 0.0);
  for (int64_t i = n - 1; i >= 0; --i) tail[i] = tail[i + 1] + s[i] * s[i];
  for (int64_t r = 1; r <= n; ++r)
    if (std::sqrt(tail[r]) <= delta) return r;
  return std::max<int64_t>(n, 1);
}

struct Setup {
  fmmt_ctx* ctx;
  cublasHandle_t blas;
  cusolverDnHandle_t sol;
};

// Left singular vectors and singular values of A (rows x cols, col-major,
// given as its conjugate transpose At = A^H, cols x rows, ld = cols).
// Uses Householder QR of At (backward stable: sigma accurate to eps*||A||)
// then the SVD of the triangular factor.  U: rows x rows (device, ld rows),
// sigma: host, length rows (zero-padded when cols < rows).
static fmmt_status left_svd_from_AH(Setup& S, double2* At, int64_t rows, int64_t cols, DBuf& U, std::vector<double>& sigma) {
  fmmt_ctx* ctx = S.ctx;
  sigma.assign(rows, 0.0);
  // U: rows x min(rows, cols) left singular vectors (economy: a tall unfolding never needs a square U)
  SETUP_TRY(dalloc(ctx, U, rows * std::min(rows, cols) * 16));
  DBuf info, work, rwork, Sd;
  SETUP_TRY(dalloc(ctx, info, 16));
  if (cols >= rows) {
    // QR of At (cols x rows)
    DBuf tau, Rm, VT;
    SETUP_TRY(dalloc(ctx, tau, rows * 16));
    int lwork = 0;
    SETUP_CUSOLVER(ctx, cusolverDnZgeqrf_bufferSize(S.sol, (int)cols, (int)rows, (zc*)At, (int)cols, &lwork));
    SETUP_TRY(dalloc(ctx, work, (int64_t)lwork * 16));
    SETUP_CUSOLVER(ctx, cusolverDnZgeqrf(S.sol, (int)cols, (int)rows, (zc*)At, (int)cols, tau.as<zc>(), work.as<zc>(), lwork, info.as<int>()));
    SETUP_TRY(dalloc(ctx, Rm, rows * rows * 16));
    k_upper<<<nblk(rows * rows), 256, 0, ctx->stream>>>(At, cols, Rm.as<double2>(), rows);
    // R = Z S W^H  =>  A = R^H Q^H = W S Z^H Q^H : U = W = VT^H
    SETUP_TRY(dalloc(ctx, VT, rows * rows * 16));
    SETUP_TRY(dalloc(ctx, Sd, rows * 8));
    SETUP_TRY(dalloc(ctx, rwork, rows * 8 + 8));
    int lw2 = 0;
    SETUP_CUSOLVER(ctx, cusolverDnZgesvd_bufferSize(S.sol, (int)rows, (int)rows, &lw2));
    SETUP_TRY(dalloc(ctx, work, (int64_t)lw2 * 16));
    SETUP_CUSOLVER(ctx, cusolverDnZgesvd(S.sol, 'N', 'A', (int)rows, (int)rows, Rm.as<zc>(), (int)rows, Sd.as<double>(), nullptr, (int)rows,
                                         VT.as<zc>(), (int)rows, work.as<zc>(), lw2, rwork.as<double>(), info.as<int>()));
    const zc one = make_cuDoubleComplex(1, 0), zero = make_cuDoubleComplex(0, 0);
    SETUP_CUBLAS(ctx, cublasZgeam(S.blas, CUBLAS_OP_C, CUBLAS_OP_N, (int)rows, (int)rows, &one, VT.as<zc>(), (int)rows, &zero,
                                  VT.as<zc>(), (int)rows, U.as<zc>(), (int)rows));
    std::vector<double> s(rows);
    FMMT_CUDA(ctx, cudaMemcpyAsync(s.data(), Sd.p, rows * 8, cudaMemcpyDeviceToHost, ctx->stream));
    FMMT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    sigma = s;
  } else {
    // A = At^H (rows x cols), rows > cols: direct SVD
    DBuf A;
    SETUP_TRY(dalloc(ctx, A, rows * cols * 16));
    const zc one = make_cuDoubleComplex(1, 0), zero = make_cuDoubleComplex(0, 0);
    SETUP_CUBLAS(ctx, cublasZgeam(S.blas, CUBLAS_OP_C, CUBLAS_OP_N, (int)rows, (int)cols, &one, (zc*)At, (int)cols, &zero,
                                  A.as<zc>(), (int)rows, A.as<zc>(), (int)rows));
    SETUP_TRY(dalloc(ctx, Sd, cols * 8));
    SETUP_TRY(dalloc(ctx, rwork, cols * 8 + 8));
    int lw2 = 0;
    SETUP_CUSOLVER(ctx, cusolverDnZgesvd_bufferSize(S.sol, (int)rows, (int)cols, &lw2));
    SETUP_TRY(dalloc(ctx, work, (int64_t)lw2 * 16));
    FMMT_CUDA(ctx, cudaMemsetAsync(U.p, 0, rows * cols * 16, ctx->stream));
    SETUP_CUSOLVER(ctx, cusolverDnZgesvd(S.sol, 'S', 'N', (int)rows, (int)cols, A.as<zc>(), (int)rows, Sd.as<double>(), U.as<zc>(),
                                         (int)rows, nullptr, (int)cols, work.as<zc>(), lw2, rwork.as<double>(), info.as<int>()));
    std::vector<double> s(cols);
    FMMT_CUDA(ctx, cudaMemcpyAsync(s.data(), Sd.p, cols * 8, cudaMemcpyDeviceToHost, ctx->stream));
    FMMT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    for (int64_t i = 0; i < cols; ++i) sigma[i] = s[i];
  }
  int hinfo = 0;
  FMMT_CUDA(ctx, cudaMemcpy(&hinfo, info.p, sizeof(int), cudaMemcpyDeviceToHost));
  if (hinfo != 0) return set_err(ctx, FMMT_E_CUDA, "cuSOLVER info = %d", hinfo);
  return FMMT_OK;
}

static double fro_norm(Setup& S, const double2* T, int64_t n) {
  double acc = 0.0;
  const int64_t chunk = 1ll << 30;
  for (int64_t o = 0; o < n; o += chunk) {
    double v = 0.0;
    cublasDznrm2(S.blas, (int)std::min<int64_t>(chunk, n - o), (const zc*)(T + o), 1, &v);
    acc += v * v;
  }
  return std::sqrt(acc);
}

// Y = T x_m M  (M: p x n_m, column-major); T dims d[0..nd), mode m (0-based).
// conjM: use conj(M)^T ... here we always pass the matrix as op(M) applied.
// Computes Y_(m) = op(M) T_(m) where op = conjugate transpose when `herm`.
static fmmt_status mode_product(Setup& S, const double2* T, const std::vector<int64_t>& d, int m, const double2* Mat,
                                int64_t p, bool herm, DBuf& Y) {
  fmmt_ctx* ctx = S.ctx;
  int64_t L = 1, R = 1;
  for (int i = 0; i < m; ++i) L *= d[i];
  for (size_t i = m + 1; i < d.size(); ++i) R *= d[i];
  const int64_t n = d[m];
  SETUP_TRY(dalloc(ctx, Y, L * p * R * 16));
  const zc one = make_cuDoubleComplex(1, 0), zero = make_cuDoubleComplex(0, 0);
  // op(M) is p x n: herm -> M stored n x p (ld n), op = ^H; else M stored p x n (ld p)
  if (L == 1) {
    // Y (p x R) = op(M) (p x n) * T (n x R)
    SETUP_CUBLAS(ctx, cublasZgemm(S.blas, herm ? CUBLAS_OP_C : CUBLAS_OP_N, CUBLAS_OP_N, (int)p, (int)R, (int)n, &one, (const zc*)Mat,
                                  herm ? (int)n : (int)p, (const zc*)T, (int)n, &zero, Y.as<zc>(), (int)p));
  } else {
    // for each r: Y_r (L x p) = T_r (L x n) * op(M)^T ; op(M)^T = conj(M) (n x p) when herm, else M^T
    DBuf Mc;
    const double2* B = Mat;
    cublasOperation_t opB = CUBLAS_OP_T;
    int ldb = (int)p;
    if (herm) {
      SETUP_TRY(dalloc(ctx, Mc, n * p * 16));
      k_conj<<<nblk(n * p), 256, 0, ctx->stream>>>(Mat, Mc.as<double2>(), n * p);
      B = Mc.as<double2>();
      opB = CUBLAS_OP_N;
      ldb = (int)n;
    }
    SETUP_CUBLAS(ctx, cublasZgemmStridedBatched(S.blas, CUBLAS_OP_N, opB, (int)L, (int)p, (int)n, &one, (const zc*)T, (int)L, L * n,
                                                (const zc*)B, ldb, 0, &zero, Y.as<zc>(), (int)L, L * p, (int)R));
  }
  return FMMT_OK;
}

// Left singular vectors / singular values of the mode-m unfolding of T (dims d) from its Gram matrix
// G = T_(m) T_(m)^H (n_m x n_m; cuBLAS ZHERK over chunks of the later modes, each chunk unfolded into a
// bounded buffer, so T is never copied whole) and its eigen-decomposition (cuSOLVER ZHEEVD):
// sigma_i = sqrt(lambda_i) descending, U = the eigenvectors in that order.  The memory-bounded path for
// operators too large to unfold (the paper's 256^3 x 435 sweep sizes); sigma loses relative accuracy
// below ~1e-8 sigma_max, far beneath every truncation threshold used (gamma >= 1e-7).
static fmmt_status gram_eig(Setup& S, DBuf& U, int64_t n, bool conj_vectors, std::vector<double>& sigma);

static fmmt_status gram_left_svd(Setup& S, const double2* T, const std::vector<int64_t>& d, int m, DBuf& U,
                                 std::vector<double>& sigma) {
  fmmt_ctx* ctx = S.ctx;
  const int nd = (int)d.size();
  int64_t L = 1, R = 1;
  for (int i = 0; i < m; ++i) L *= d[i];
  for (int i = m + 1; i < nd; ++i) R *= d[i];
  const int64_t n = d[m];
  const double one = 1.0;
  SETUP_TRY(dalloc(ctx, U, n * n * 16));
  FMMT_CUDA(ctx, cudaMemsetAsync(U.p, 0, n * n * 16, ctx->stream));
  const int64_t kmax = 1ll << 30;   // ZHERK inner-dimension chunk (int32 arguments)
  if (L == 1) {
    // first mode: T_(1) is T itself (n x R, column-major): G = sum over column chunks of T_c T_c^H
    for (int64_t r0 = 0; r0 < R; r0 += kmax) {
      const int64_t rn = std::min<int64_t>(kmax, R - r0);
      SETUP_CUBLAS(ctx, cublasZherk(S.blas, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, (int)n, (int)rn, &one,
                                    (const zc*)(T + r0 * n), (int)n, &one, U.as<zc>(), (int)n));
    }
    return gram_eig(S, U, n, false, sigma);
  }
  if (R == 1 && L < (1ll << 31)) {
    // last mode: T is X = L x n (column-major) with T_(m) = X^T, so X^H X = conj(T_(m) T_(m)^H): accumulate
    // it over row chunks of X (no copy) and conjugate the eigenvectors
    for (int64_t l0 = 0; l0 < L; l0 += kmax) {
      const int64_t ln = std::min<int64_t>(kmax, L - l0);
      SETUP_CUBLAS(ctx, cublasZherk(S.blas, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_C, (int)n, (int)ln, &one,
                                    (const zc*)(T + l0), (int)L, &one, U.as<zc>(), (int)n));
    }
    return gram_eig(S, U, n, true, sigma);
  }
  const int64_t budget = 1ll << 31;   // bytes of one unfolded chunk
  const int64_t rc = std::max<int64_t>(1, std::min<int64_t>(R, budget / std::max<int64_t>(1, L * n * 16)));
  DBuf At;
  SETUP_TRY(dalloc(ctx, At, L * rc * n * 16));
  for (int64_t r0 = 0; r0 < R; r0 += rc) {
    const int64_t rn = std::min<int64_t>(rc, R - r0);
    k_unfold_h<<<nblk(L * n * rn), 256, 0, ctx->stream>>>(T + r0 * L * n, At.as<double2>(), L, n, rn);
    FMMT_CUDA(ctx, cudaGetLastError());
    // G += At^H At  (At: (L rn) x n, the chunk's unfolding conjugate-transposed)
    SETUP_CUBLAS(ctx, cublasZherk(S.blas, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_C, (int)n, (int)(L * rn), &one,
                                  (const zc*)At.as<double2>(), (int)(L * rn), &one, U.as<zc>(), (int)n));
  }
  return gram_eig(S, U, n, false, sigma);
}

// Eigen-decomposition of the Hermitian Gram matrix held (upper triangle) in U (n x n): on return U holds the
// eigenvectors in descending eigenvalue order (conjugated if conj_vectors) and sigma_i = sqrt(lambda_i).
static fmmt_status gram_eig(Setup& S, DBuf& U, int64_t n, bool conj_vectors, std::vector<double>& sigma) {
  fmmt_ctx* ctx = S.ctx;
  DBuf W, work, info;
  SETUP_TRY(dalloc(ctx, W, n * 8));
  SETUP_TRY(dalloc(ctx, info, 16));
  int lwork = 0;
  SETUP_CUSOLVER(ctx, cusolverDnZheevd_bufferSize(S.sol, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, (int)n, U.as<zc>(),
                                                   (int)n, W.as<double>(), &lwork));
  SETUP_TRY(dalloc(ctx, work, (int64_t)lwork * 16));
  SETUP_CUSOLVER(ctx, cusolverDnZheevd(S.sol, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, (int)n, U.as<zc>(), (int)n,
                                        W.as<double>(), work.as<zc>(), lwork, info.as<int>()));
  std::vector<double> lam(n);
  FMMT_CUDA(ctx, cudaMemcpyAsync(lam.data(), W.p, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  int hinfo = 0;
  FMMT_CUDA(ctx, cudaMemcpyAsync(&hinfo, info.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  FMMT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if (hinfo != 0) return set_err(ctx, FMMT_E_CUDA, "cuSOLVER zheevd info = %d", hinfo);
  // ascending eigenpairs -> descending singular triplets: reverse the columns
  DBuf Ur;
  SETUP_TRY(dalloc(ctx, Ur, n * n * 16));
  for (int64_t i = 0; i < n; ++i)
    FMMT_CUDA(ctx, cudaMemcpyAsync(Ur.as<double2>() + i * n, U.as<double2>() + (n - 1 - i) * n, n * 16,
                                   cudaMemcpyDeviceToDevice, ctx->stream));
  if (conj_vectors) {
    k_conj<<<nblk(n * n), 256, 0, ctx->stream>>>(Ur.as<double2>(), U.as<double2>(), n * n);
    FMMT_CUDA(ctx, cudaGetLastError());
  } else {
    std::swap(U.p, Ur.p);
  }
  sigma.assign(n, 0.0);
  for (int64_t i = 0; i < n; ++i) sigma[i] = std::sqrt(std::max(0.0, lam[n - 1 - i]));
  return FMMT_OK;
}

// Whether unfolding T (one more copy of `total` complex128) fits the device with headroom; else the Gram path.
static bool unfold_fits(fmmt_ctx* ctx, int64_t total) {
  if (const char* e = getenv("FMMT_COMPRESS_GRAM")) return atoi(e) == 0;
  size_t fr = 0, tot = 0;
  if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return (double)total * 16.0 * 2.5 < (double)fr;
}

// Alg. 1: classical HOSVD of T (dims d), delta = gamma / sqrt(n_trunc) * norm.
// Returns factors U_i (n_i x r_i, device) and the projected core (device).
struct TuckerOut {
  std::vector<DBuf> U;
  std::vector<int64_t> r;
  DBuf core;
};

static fmmt_status tucker_svd(Setup& S, const double2* T, const std::vector<int64_t>& d, double gamma, double n_trunc, double norm,
                              TuckerOut& out) {
  fmmt_ctx* ctx = S.ctx;
  const int nd = (int)d.size();
  int64_t total = 1;
  for (auto v : d) total *= v;
  const double delta = gamma / std::sqrt(n_trunc) * norm;
  out.U.clear();
  out.U.resize(nd);
  out.r.assign(nd, 1);
  const bool gram = !unfold_fits(ctx, total);
  DBuf At;
  if (!gram) SETUP_TRY(dalloc(ctx, At, total * 16));
  for (int m = 0; m < nd; ++m) {
    int64_t L = 1, R = 1;
    for (int i = 0; i < m; ++i) L *= d[i];
    for (int i = m + 1; i < nd; ++i) R *= d[i];
    std::vector<double> sigma;
    DBuf Ufull;
    if (gram) {
      SETUP_TRY(gram_left_svd(S, T, d, m, Ufull, sigma));
    } else {
      k_unfold_h<<<nblk(total), 256, 0, ctx->stream>>>(T, At.as<double2>(), L, d[m], R);
      FMMT_CUDA(ctx, cudaGetLastError());
      SETUP_TRY(left_svd_from_AH(S, At.as<double2>(), d[m], L * R, Ufull, sigma));
    }
    const int64_t r = tail_rank(sigma, delta);
    out.r[m] = r;
    SETUP_TRY(dalloc(ctx, out.U[m], d[m] * r * 16));
    FMMT_CUDA(ctx, cudaMemcpyAsync(out.U[m].p, Ufull.p, d[m] * r * 16, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  At = DBuf();
  if (gram && nd == 4) {
    // core = T x_1 U1^H x_2 U2^H x_3 U3^H x_4 U4^H in chunks of the last mode (bounded temporaries):
    // W[:, p] = (T[:, :, :, p] x_1 U1^H x_2 U2^H x_3 U3^H), then W x_4 U4^H
    const int64_t r123 = out.r[0] * out.r[1] * out.r[2], n123 = d[0] * d[1] * d[2];
    DBuf Wc;
    SETUP_TRY(dalloc(ctx, Wc, r123 * d[3] * 16));
    const int64_t pc = std::max<int64_t>(1, std::min<int64_t>(d[3], (1ll << 31) / (n123 * 16)));
    for (int64_t p0 = 0; p0 < d[3]; p0 += pc) {
      const int64_t pn = std::min<int64_t>(pc, d[3] - p0);
      std::vector<int64_t> cur = {d[0], d[1], d[2], pn};
      DBuf a, b;
      const double2* src = T + p0 * n123;
      for (int m = 0; m < 3; ++m) {
        DBuf& dst = (m % 2 == 0) ? a : b;
        SETUP_TRY(mode_product(S, src, cur, m, out.U[m].as<double2>(), out.r[m], true, dst));
        cur[m] = out.r[m];
        src = dst.as<double2>();
      }
      FMMT_CUDA(ctx, cudaMemcpyAsync(Wc.as<double2>() + p0 * r123, a.p, r123 * pn * 16, cudaMemcpyDeviceToDevice,
                                     ctx->stream));   // (after 3 products the result is in `a`)
    }
    std::vector<int64_t> cur = {out.r[0], out.r[1], out.r[2], d[3]};
    SETUP_TRY(mode_product(S, Wc.as<double2>(), cur, 3, out.U[3].as<double2>(), out.r[3], true, out.core));
    return FMMT_OK;
  }
  // core = T x_1 U1^H x_2 ... (step 8)
  std::vector<int64_t> cur = d;
  DBuf a, b;
  const double2* src = T;
  for (int m = 0; m < nd; ++m) {
    DBuf& dst = (m % 2 == 0) ? a : b;
    SETUP_TRY(mode_product(S, src, cur, m, out.U[m].as<double2>(), out.r[m], true, dst));
    cur[m] = out.r[m];
    src = dst.as<double2>();
  }
  DBuf& last = (nd % 2 == 1) ? a : b;
  out.core.p = last.p;
  last.p = nullptr;
  return FMMT_OK;
}

// Alg. 3: TT-SVD. cores[0] = U^1 (n1 x r1), cores[1..d-2] = C^i
// (r_{i-1} x n_i x r_i), tail = n_d x r_{d-1}.
struct TTOut {
  std::vector<DBuf> cores;
  DBuf tail;
  std::vector<int64_t> r;
};

static fmmt_status tt_svd(Setup& S, const double2* T, const std::vector<int64_t>& d, double gamma, TTOut& out) {
  fmmt_ctx* ctx = S.ctx;
  const int nd = (int)d.size();
  int64_t total = 1;
  for (auto v : d) total *= v;
  const double delta = gamma / std::sqrt((double)(nd - 1)) * fro_norm(S, T, total);
  out.cores.clear();
  out.cores.resize(nd - 1);
  out.r.assign(nd - 1, 1);
  // the remainder starts as T itself (read in place, never copied); each step's left factor comes from the
  // unfolding's SVD when a copy of it fits, else from its Gram matrix (memory-bounded, gram_left_svd)
  DBuf C;
  const double2* Cp = T;
  int64_t rprev = 1, cols = total;
  const zc one = make_cuDoubleComplex(1, 0), zero = make_cuDoubleComplex(0, 0);
  for (int i = 0; i < nd - 1; ++i) {
    const int64_t rows = rprev * d[i];
    cols = cols / d[i];
    // C is rows x cols (col-major)
    std::vector<double> sigma;
    DBuf Ufull;
    if (unfold_fits(ctx, rows * cols)) {
      DBuf At;   // At = C^H
      SETUP_TRY(dalloc(ctx, At, rows * cols * 16));
      k_unfold_h<<<nblk(rows * cols), 256, 0, ctx->stream>>>(Cp, At.as<double2>(), 1, rows, cols);
      FMMT_CUDA(ctx, cudaGetLastError());
      SETUP_TRY(left_svd_from_AH(S, At.as<double2>(), rows, cols, Ufull, sigma));
    } else {
      SETUP_TRY(gram_left_svd(S, Cp, {rows, cols}, 0, Ufull, sigma));
    }
    const int64_t r = tail_rank(sigma, delta);
    out.r[i] = r;
    SETUP_TRY(dalloc(ctx, out.cores[i], rows * r * 16));
    FMMT_CUDA(ctx, cudaMemcpyAsync(out.cores[i].p, Ufull.p, rows * r * 16, cudaMemcpyDeviceToDevice, ctx->stream));
    // remainder Sigma V^H = U_r^H C  (r x cols)
    DBuf Cn;
    SETUP_TRY(dalloc(ctx, Cn, r * cols * 16));
    SETUP_CUBLAS(ctx, cublasZgemm(S.blas, CUBLAS_OP_C, CUBLAS_OP_N, (int)r, (int)cols, (int)rows, &one, Ufull.as<zc>(), (int)rows,
                                  (const zc*)Cp, (int)rows, &zero, Cn.as<zc>(), (int)r));
    std::swap(C.p, Cn.p);
    Cp = C.as<double2>();
    rprev = r;
  }
  // tail = C^T (n_d x r_{d-1})
  SETUP_TRY(dalloc(ctx, out.tail, cols * rprev * 16));
  SETUP_CUBLAS(ctx, cublasZgeam(S.blas, CUBLAS_OP_T, CUBLAS_OP_N, (int)cols, (int)rprev, &one, C.as<zc>(), (int)rprev, &zero,
                                out.tail.as<zc>(), (int)cols, out.tail.as<zc>(), (int)cols));
  return FMMT_OK;
}

static fmmt_status to_c64(Setup& S, const double2* a, int64_t n, float2* dst) {
  k_z2c<<<nblk(n), 256, 0, S.ctx->stream>>>(a, dst, n);
  FMMT_CUDA(S.ctx, cudaGetLastError());
  return FMMT_OK;
}

// ---------------------------------------------------------------- sharded 4D setup (NCCL broadcast)
// Element counts of a 4D format's arrays (import order) for `rows` direction-factor rows, and which
// array is the direction factor (rows x r, column-major) with its rank slot.
static std::vector<int64_t> arrays4d(fmmt_format f, int64_t n1, int64_t n2, int64_t n3, int64_t rows, const int64_t* r,
                                     int* dir_arr) {
  switch (f) {
    case FMMT_TUCKER4D: *dir_arr = 4; return {r[0] * r[1] * r[2] * r[3], n1 * r[0], n2 * r[1], n3 * r[2], rows * r[3]};
    case FMMT_HTUCKER4D:
      *dir_arr = 3;
      return {n1 * r[0], n2 * r[1], n3 * r[2], rows * r[3], r[0] * r[1] * r[4], r[2] * r[3] * r[5], r[4] * r[5]};
    default: *dir_arr = 3; return {n1 * r[0], r[0] * n2 * r[1], r[1] * n3 * r[2], rows * r[2]};
  }
}
static int dir_rank_slot(fmmt_format f) { return f == FMMT_TT4D ? 2 : 3; }

// Broadcast ranks + all arrays (every direction row) from rank 0 over the context's communicator, then
// keep rows [b, b + c) of the direction factor and create the local op.  `full` (root only) are the arrays
// with all ndir rows; receivers pass an empty vector and get them.
static fmmt_status bcast_and_create(fmmt_ctx* ctx, int64_t n1, int64_t n2, int64_t n3, int64_t ndir, int64_t b, int64_t c,
                                    fmmt_format format, std::vector<int64_t> ranks, std::vector<const void*> full,
                                    fmmt_op** op) {
  ncclComm_t comm = (ncclComm_t)ctx->nccl_comm;
  if (!comm) return set_err(ctx, FMMT_E_STATE, "sharded compress needs a communicator (fmmt_init_sharded)");
  const bool root = ctx->rank == 0;
  // 1. ranks (6 int64 slots)
  DBuf hdr;
  SETUP_TRY(dalloc(ctx, hdr, 6 * 8));
  int64_t h[6] = {0, 0, 0, 0, 0, 0};
  if (root)
    for (size_t i = 0; i < ranks.size() && i < 6; ++i) h[i] = ranks[i];
  FMMT_CUDA(ctx, cudaMemcpyAsync(hdr.p, h, sizeof(h), cudaMemcpyHostToDevice, ctx->stream));
  ncclResult_t nr = ncclBroadcast(hdr.p, hdr.p, 6, ncclInt64, 0, comm, ctx->stream);
  if (nr != ncclSuccess) return set_err(ctx, FMMT_E_NCCL, "ncclBroadcast(ranks): %s", ncclGetErrorString(nr));
  FMMT_CUDA(ctx, cudaMemcpyAsync(h, hdr.p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  FMMT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  static const int nslots_of[] = {0, 3, 4, 6, 2, 3};
  ranks.assign(h, h + nslots_of[format]);
  for (auto r : ranks)
    if (r < 1) return set_err(ctx, FMMT_E_STATE, "broadcast ranks invalid (root failed?)");
  // 2. one payload buffer holding every array back to back (complex64)
  int dir_arr = 0;
  const std::vector<int64_t> el = arrays4d(format, n1, n2, n3, ndir, ranks.data(), &dir_arr);
  std::vector<int64_t> off(el.size() + 1, 0);
  for (size_t i = 0; i < el.size(); ++i) off[i + 1] = off[i] + el[i];
  DBuf pay;
  SETUP_TRY(dalloc(ctx, pay, off.back() * 8));
  float2* P = pay.as<float2>();
  if (root)
    for (size_t i = 0; i < el.size(); ++i)
      FMMT_CUDA(ctx, cudaMemcpyAsync(P + off[i], full[i], el[i] * 8, cudaMemcpyDeviceToDevice, ctx->stream));
  // (2 floats per complex; NCCL counts are size_t)
  nr = ncclBroadcast(P, P, (size_t)(2 * off.back()), ncclFloat, 0, comm, ctx->stream);
  if (nr != ncclSuccess) return set_err(ctx, FMMT_E_NCCL, "ncclBroadcast(factors): %s", ncclGetErrorString(nr));
  // 3. this rank's direction rows
  const int64_t r = ranks[dir_rank_slot(format)];
  DBuf loc;
  SETUP_TRY(dalloc(ctx, loc, c * r * 8));
  FMMT_CUDA(ctx, cudaMemcpy2DAsync(loc.p, c * 8, P + off[dir_arr] + b, ndir * 8, c * 8, r, cudaMemcpyDeviceToDevice,
                                   ctx->stream));
  FMMT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  std::vector<const void*> arrs;
  for (size_t i = 0; i < el.size(); ++i) arrs.push_back((int)i == dir_arr ? loc.p : (const void*)(P + off[i]));
  return fmmt_internal::create_op(ctx, format, n1, n2, n3, c, ranks.data(), arrs.data(), (int64_t)arrs.size(), op, true);
}

static fmmt_status compress_receive(fmmt_ctx* ctx, int64_t n1, int64_t n2, int64_t n3, int64_t ndir, int64_t b, int64_t c,
                                    fmmt_format format, fmmt_op** op) {
  return bcast_and_create(ctx, n1, n2, n3, ndir, b, c, format, {}, {}, op);
}

static fmmt_status compress_send(fmmt_ctx* ctx, int64_t n1, int64_t n2, int64_t n3, int64_t ndir, int64_t b, int64_t c,
                                 fmmt_format format, const std::vector<int64_t>& ranks, const std::vector<const void*>& full,
                                 fmmt_op** op) {
  return bcast_and_create(ctx, n1, n2, n3, ndir, b, c, format, ranks, full, op);
}

static fmmt_status compress_impl(fmmt_ctx* ctx, const fmmt_c128* T, int64_t n1, int64_t n2, int64_t n3, int64_t ndir,
                                 int64_t dir_begin, int64_t dir_count, fmmt_format format, double tol, fmmt_op** op,
                                 bool* sent) {
  if (!ctx || !op) return FMMT_E_ARG;
  *op = nullptr;
  const bool is4d = format == FMMT_TUCKER4D || format == FMMT_HTUCKER4D || format == FMMT_TT4D;
  // sharded 4D setup: rank 0 compresses the whole T_4D and broadcasts the shared factors and
  // the direction factor; every rank keeps the rows of its own directions.  Other ranks pass T = NULL.
  const bool bcast = is4d && ctx->nccl_comm != nullptr;
  const bool receiver = bcast && ctx->rank != 0;
  if (!T && !receiver) return set_err(ctx, FMMT_E_ARG, "null T");
  if (!(tol > 0 && tol < 1)) return set_err(ctx, FMMT_E_ARG, "tol must be in (0,1)");
  if (format < FMMT_DENSE || format > FMMT_TT4D) return set_err(ctx, FMMT_E_ARG, "bad format");
  if (n1 < 2 || n2 < 2 || n3 < 2 || ndir < 1 || dir_begin < 0 || dir_count < 1 || dir_begin + dir_count > ndir)
    return set_err(ctx, FMMT_E_SHAPE, "bad compress shape");
  const int64_t shard_begin = dir_begin, shard_count = dir_count;
  cudaSetDevice(ctx->device);
  if (receiver) return compress_receive(ctx, n1, n2, n3, ndir, dir_begin, dir_count, format, op);
  Setup S;
  S.ctx = ctx;
  SETUP_TRY(handles(ctx, &S.blas, &S.sol));
  const int64_t n = n1 * n2 * n3;
  if (bcast) {   // the root keeps every direction row until the broadcast; sliced below
    dir_begin = 0;
    dir_count = ndir;
  }
  // T may be host or device memory
  cudaPointerAttributes pa;
  const double2* Td = nullptr;
  DBuf Tcopy;
  if (cudaPointerGetAttributes(&pa, T) == cudaSuccess && (pa.type == cudaMemoryTypeDevice || pa.type == cudaMemoryTypeManaged)) {
    Td = reinterpret_cast<const double2*>(T);
  } else {
    cudaGetLastError();
    SETUP_TRY(dalloc(ctx, Tcopy, ndir * n * 16));
    FMMT_CUDA(ctx, cudaMemcpy(Tcopy.p, T, ndir * n * 16, cudaMemcpyHostToDevice));
    Td = Tcopy.as<double2>();
  }
  const std::vector<int64_t> d3 = {n1, n2, n3};
  std::vector<DBuf> outs;
  std::vector<int64_t> ranks;
  std::vector<const void*> arrs;
  auto alloc_out = [&](int64_t elems) -> float2* {
    outs.emplace_back();
    if (dalloc(ctx, outs.back(), elems * 8) != FMMT_OK) return nullptr;
    return outs.back().as<float2>();
  };
  // outs may reallocate; reserve
  outs.reserve(16);
  switch (format) {
    case FMMT_DENSE: {
      float2* t = alloc_out(dir_count * n);
      if (!t) return FMMT_E_NOMEM;
      SETUP_TRY(to_c64(S, Td + dir_begin * n, dir_count * n, t));
      arrs = {t};
      break;
    }
    case FMMT_TUCKER3D:
    case FMMT_TT3D: {
      const bool tuck = format == FMMT_TUCKER3D;
      // per-direction factors, concatenated (host-side sizes first pass)
      std::vector<std::vector<float2*>> parts;
      std::vector<std::vector<int64_t>> sizes;
      std::vector<DBuf> keep;
      keep.reserve(dir_count * 4 + 4);
      const int na = tuck ? 4 : 3;
      std::vector<int64_t> tot(na, 0);
      std::vector<std::vector<std::pair<void*, int64_t>>> items(na);
      for (int64_t p = dir_begin; p < dir_begin + dir_count; ++p) {
        const double2* Tp = Td + p * n;
        if (tuck) {
          TuckerOut to;
          SETUP_TRY(tucker_svd(S, Tp, d3, tol, 3.0, fro_norm(S, Tp, n), to));
          ranks.insert(ranks.end(), to.r.begin(), to.r.end());
          const int64_t sz[4] = {to.r[0] * to.r[1] * to.r[2], n1 * to.r[0], n2 * to.r[1], n3 * to.r[2]};
          DBuf* srcs[4] = {&to.core, &to.U[0], &to.U[1], &to.U[2]};
          for (int i = 0; i < 4; ++i) {
            keep.emplace_back();
            SETUP_TRY(dalloc(ctx, keep.back(), sz[i] * 8));
            SETUP_TRY(to_c64(S, srcs[i]->as<double2>(), sz[i], keep.back().as<float2>()));
            items[i].push_back({keep.back().p, sz[i]});
            tot[i] += sz[i];
          }
        } else {
          TTOut to;
          SETUP_TRY(tt_svd(S, Tp, d3, tol, to));
          ranks.insert(ranks.end(), to.r.begin(), to.r.end());
          const int64_t sz[3] = {n1 * to.r[0], to.r[0] * n2 * to.r[1], n3 * to.r[1]};
          DBuf* srcs[3] = {&to.cores[0], &to.cores[1], &to.tail};
          for (int i = 0; i < 3; ++i) {
            keep.emplace_back();
            SETUP_TRY(dalloc(ctx, keep.back(), sz[i] * 8));
            SETUP_TRY(to_c64(S, srcs[i]->as<double2>(), sz[i], keep.back().as<float2>()));
            items[i].push_back({keep.back().p, sz[i]});
            tot[i] += sz[i];
          }
        }
      }
      for (int i = 0; i < na; ++i) {
        float2* dst = alloc_out(tot[i]);
        if (!dst) return FMMT_E_NOMEM;
        int64_t o = 0;
        for (auto& it : items[i]) {
          FMMT_CUDA(ctx, cudaMemcpyAsync(dst + o, it.first, it.second * 8, cudaMemcpyDeviceToDevice, ctx->stream));
          o += it.second;
        }
        arrs.push_back(dst);
      }
      break;
    }
    case FMMT_TUCKER4D: {
      const std::vector<int64_t> d4 = {n1, n2, n3, ndir};
      TuckerOut to;
      SETUP_TRY(tucker_svd(S, Td, d4, tol, 4.0, fro_norm(S, Td, n * ndir), to));
      ranks = to.r;
      const int64_t r1 = to.r[0], r2 = to.r[1], r3 = to.r[2], r4 = to.r[3];
      float2* c = alloc_out(r1 * r2 * r3 * r4);
      float2* u1 = alloc_out(n1 * r1);
      float2* u2 = alloc_out(n2 * r2);
      float2* u3 = alloc_out(n3 * r3);
      float2* u4 = alloc_out(dir_count * r4);
      if (!c || !u1 || !u2 || !u3 || !u4) return FMMT_E_NOMEM;
      SETUP_TRY(to_c64(S, to.core.as<double2>(), r1 * r2 * r3 * r4, c));
      SETUP_TRY(to_c64(S, to.U[0].as<double2>(), n1 * r1, u1));
      SETUP_TRY(to_c64(S, to.U[1].as<double2>(), n2 * r2, u2));
      SETUP_TRY(to_c64(S, to.U[2].as<double2>(), n3 * r3, u3));
      // rows [dir_begin, dir_begin + dir_count) of U4 (ndir x r4, column-major)
      DBuf u4l;
      SETUP_TRY(dalloc(ctx, u4l, dir_count * r4 * 16));
      FMMT_CUDA(ctx, cudaMemcpy2DAsync(u4l.p, dir_count * 16, to.U[3].as<double2>() + dir_begin, ndir * 16, dir_count * 16, r4,
                                       cudaMemcpyDeviceToDevice, ctx->stream));
      SETUP_TRY(to_c64(S, u4l.as<double2>(), dir_count * r4, u4));
      arrs = {c, u1, u2, u3, u4};
      break;
    }
    case FMMT_HTUCKER4D: {
      const std::vector<int64_t> d4 = {n1, n2, n3, ndir};
      const double nrm = fro_norm(S, Td, n * ndir);
      TuckerOut to;
      SETUP_TRY(tucker_svd(S, Td, d4, tol, 6.0, nrm, to));   // leaves with gamma/sqrt(6) (reading Q8)
      const int64_t r1 = to.r[0], r2 = to.r[1], r3 = to.r[2], r4 = to.r[3];
      const double delta = tol / std::sqrt(6.0) * nrm;
      const double2* W12 = to.core.as<double2>();           // (r1 r2) x (r3 r4)
      DBuf At, U12, U34, W34, tmp, root, c34c;
      std::vector<double> s12, s34;
      // C12: left singular vectors of W12
      SETUP_TRY(dalloc(ctx, At, r1 * r2 * r3 * r4 * 16));
      k_unfold_h<<<nblk(r1 * r2 * r3 * r4), 256, 0, ctx->stream>>>(W12, At.as<double2>(), 1, r1 * r2, r3 * r4);
      SETUP_TRY(left_svd_from_AH(S, At.as<double2>(), r1 * r2, r3 * r4, U12, s12));
      const int64_t r12 = tail_rank(s12, delta);
      // C34: left singular vectors of W34 = W12^T
      const zc one = make_cuDoubleComplex(1, 0), zero = make_cuDoubleComplex(0, 0);
      SETUP_TRY(dalloc(ctx, W34, r1 * r2 * r3 * r4 * 16));
      SETUP_CUBLAS(ctx, cublasZgeam(S.blas, CUBLAS_OP_T, CUBLAS_OP_N, (int)(r3 * r4), (int)(r1 * r2), &one, (const zc*)W12, (int)(r1 * r2),
                                    &zero, W34.as<zc>(), (int)(r3 * r4), W34.as<zc>(), (int)(r3 * r4)));
      k_unfold_h<<<nblk(r1 * r2 * r3 * r4), 256, 0, ctx->stream>>>(W34.as<double2>(), At.as<double2>(), 1, r3 * r4, r1 * r2);
      SETUP_TRY(left_svd_from_AH(S, At.as<double2>(), r3 * r4, r1 * r2, U34, s34));
      const int64_t r34 = tail_rank(s34, delta);
      // root C1234 = C12^H W12 conj(C34)   (reading Q10)
      SETUP_TRY(dalloc(ctx, c34c, r3 * r4 * r34 * 16));
      k_conj<<<nblk(r3 * r4 * r34), 256, 0, ctx->stream>>>(U34.as<double2>(), c34c.as<double2>(), r3 * r4 * r34);
      SETUP_TRY(dalloc(ctx, tmp, r1 * r2 * r34 * 16));
      SETUP_CUBLAS(ctx, cublasZgemm(S.blas, CUBLAS_OP_N, CUBLAS_OP_N, (int)(r1 * r2), (int)r34, (int)(r3 * r4), &one, (const zc*)W12,
                                    (int)(r1 * r2), c34c.as<zc>(), (int)(r3 * r4), &zero, tmp.as<zc>(), (int)(r1 * r2)));
      SETUP_TRY(dalloc(ctx, root, r12 * r34 * 16));
      SETUP_CUBLAS(ctx, cublasZgemm(S.blas, CUBLAS_OP_C, CUBLAS_OP_N, (int)r12, (int)r34, (int)(r1 * r2), &one, U12.as<zc>(), (int)(r1 * r2),
                                    tmp.as<zc>(), (int)(r1 * r2), &zero, root.as<zc>(), (int)r12));
      ranks = {r1, r2, r3, r4, r12, r34};
      float2* u1 = alloc_out(n1 * r1);
      float2* u2 = alloc_out(n2 * r2);
      float2* u3 = alloc_out(n3 * r3);
      float2* u4 = alloc_out(dir_count * r4);
      float2* c12 = alloc_out(r1 * r2 * r12);
      float2* c34 = alloc_out(r3 * r4 * r34);
      float2* c1234 = alloc_out(r12 * r34);
      if (!u1 || !u2 || !u3 || !u4 || !c12 || !c34 || !c1234) return FMMT_E_NOMEM;
      SETUP_TRY(to_c64(S, to.U[0].as<double2>(), n1 * r1, u1));
      SETUP_TRY(to_c64(S, to.U[1].as<double2>(), n2 * r2, u2));
      SETUP_TRY(to_c64(S, to.U[2].as<double2>(), n3 * r3, u3));
      DBuf u4l;
      SETUP_TRY(dalloc(ctx, u4l, dir_count * r4 * 16));
      FMMT_CUDA(ctx, cudaMemcpy2DAsync(u4l.p, dir_count * 16, to.U[3].as<double2>() + dir_begin, ndir * 16, dir_count * 16, r4,
                                       cudaMemcpyDeviceToDevice, ctx->stream));
      SETUP_TRY(to_c64(S, u4l.as<double2>(), dir_count * r4, u4));
      SETUP_TRY(to_c64(S, U12.as<double2>(), r1 * r2 * r12, c12));
      SETUP_TRY(to_c64(S, U34.as<double2>(), r3 * r4 * r34, c34));
      SETUP_TRY(to_c64(S, root.as<double2>(), r12 * r34, c1234));
      arrs = {u1, u2, u3, u4, c12, c34, c1234};
      break;
    }
    case FMMT_TT4D: {
      const std::vector<int64_t> d4 = {n1, n2, n3, ndir};
      TTOut to;
      SETUP_TRY(tt_svd(S, Td, d4, tol, to));
      ranks = to.r;
      const int64_t r1 = to.r[0], r2 = to.r[1], r3 = to.r[2];
      float2* u1 = alloc_out(n1 * r1);
      float2* c1 = alloc_out(r1 * n2 * r2);
      float2* c2 = alloc_out(r2 * n3 * r3);
      float2* ul = alloc_out(dir_count * r3);
      if (!u1 || !c1 || !c2 || !ul) return FMMT_E_NOMEM;
      SETUP_TRY(to_c64(S, to.cores[0].as<double2>(), n1 * r1, u1));
      SETUP_TRY(to_c64(S, to.cores[1].as<double2>(), r1 * n2 * r2, c1));
      SETUP_TRY(to_c64(S, to.cores[2].as<double2>(), r2 * n3 * r3, c2));
      DBuf ull;
      SETUP_TRY(dalloc(ctx, ull, dir_count * r3 * 16));
      FMMT_CUDA(ctx, cudaMemcpy2DAsync(ull.p, dir_count * 16, to.tail.as<double2>() + dir_begin, ndir * 16, dir_count * 16, r3,
                                       cudaMemcpyDeviceToDevice, ctx->stream));
      SETUP_TRY(to_c64(S, ull.as<double2>(), dir_count * r3, ul));
      arrs = {u1, c1, c2, ul};
      break;
    }
  }
  FMMT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  static const int narr_of[] = {1, 4, 5, 7, 3, 4};
  if (bcast) {
    *sent = true;
    return compress_send(ctx, n1, n2, n3, ndir, shard_begin, shard_count, format, ranks, arrs, op);
  }
  return fmmt_internal::create_op(ctx, format, n1, n2, n3, dir_count, ranks.empty() ? nullptr : ranks.data(), arrs.data(),
                                  narr_of[format], op, true);
}

extern "C" fmmt_status fmmt_compress(fmmt_ctx* ctx, const fmmt_c128* T, int64_t n1, int64_t n2, int64_t n3, int64_t ndir,
                                     int64_t dir_begin, int64_t dir_count, fmmt_format format, double tol, fmmt_op** op) {
  bool sent = false;
  fmmt_status st = compress_impl(ctx, T, n1, n2, n3, ndir, dir_begin, dir_count, format, tol, op, &sent);
  const bool is4d = format == FMMT_TUCKER4D || format == FMMT_HTUCKER4D || format == FMMT_TT4D;
  if (st != FMMT_OK && !sent && ctx && ctx->rank == 0 && is4d && ctx->nccl_comm) {
    // the root failed before its broadcast: send an all-zero rank header so the other ranks return
    // FMMT_E_STATE instead of waiting forever (the root keeps its own error message)
    std::string err = ctx->err;
    DBuf hdr;
    if (dalloc(ctx, hdr, 6 * 8) == FMMT_OK && cudaMemsetAsync(hdr.p, 0, 48, ctx->stream) == cudaSuccess &&
        ncclBroadcast(hdr.p, hdr.p, 6, ncclInt64, 0, (ncclComm_t)ctx->nccl_comm, ctx->stream) == ncclSuccess)
      cudaStreamSynchronize(ctx->stream);
    ctx->err = err;
  }
  return st;
}

// ============================================================== FP64 derived operands (setup)
// The direction-independent products the hot path reuses every matvec are
// computed here in complex128 (cuBLAS ZGEMM) from the complex64 factors and
// rounded once to complex64, so they add one rounding (6e-8) instead of the
// 3xTF32 GEMM error to the restore chain:
//   H-Tucker (Fig. 3(c)):  E = (C12 . C1234) x1 U1 x2 U2        stored E[i + n1 j + n1 n2 jj]
//   TT-4D (Fig. 4(b) step 1 of Fig. 4(a)):  T1 = U1 . C1          stored T1[i + n1 (j + n2 b)]
__global__ void k_c2z(const float2* __restrict__ a, double2* __restrict__ b, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = make_double2(a[i].x, a[i].y);
}

namespace {
struct ZBuf {
  double2* p = nullptr;
  ~ZBuf() { if (p) cudaFree(p); }
};
fmmt_status zalloc_from(fmmt_ctx* ctx, ZBuf& b, const float2* src, int64_t n) {
  if (cudaMalloc(&b.p, std::max<int64_t>(1, n) * sizeof(double2)) != cudaSuccess) {
    cudaGetLastError();
    return set_err(ctx, FMMT_E_NOMEM, "setup allocation (%lld B) failed", (long long)(n * 16));
  }
  if (src) k_c2z<<<nblk(n), 256, 0, ctx->stream>>>(src, b.p, n);
  return FMMT_OK;
}
}  // namespace

fmmt_status fmmt_internal::htucker_E_fp64(fmmt_ctx* ctx, const float2* U1, const float2* U2, const float2* C12,
                                          const float2* C1234, int64_t n1, int64_t n2, int64_t r1, int64_t r2,
                                          int64_t r12, int64_t r34, float2* E) {
  cublasHandle_t blas;
  cusolverDnHandle_t sol;
  SETUP_TRY(handles(ctx, &blas, &sol));
  ZBuf u1, u2, c12, c1234, D, E1, Ez;
  SETUP_TRY(zalloc_from(ctx, u1, U1, n1 * r1));
  SETUP_TRY(zalloc_from(ctx, u2, U2, n2 * r2));
  SETUP_TRY(zalloc_from(ctx, c12, C12, r1 * r2 * r12));
  SETUP_TRY(zalloc_from(ctx, c1234, C1234, r12 * r34));
  SETUP_TRY(zalloc_from(ctx, D, nullptr, r1 * r2 * r34));
  SETUP_TRY(zalloc_from(ctx, E1, nullptr, n1 * r2 * r34));
  SETUP_TRY(zalloc_from(ctx, Ez, nullptr, n1 * n2 * r34));
  const zc one = make_cuDoubleComplex(1, 0), zero = make_cuDoubleComplex(0, 0);
  // D (r1 r2 x r34) = C12 (r1 r2 x r12) . C1234 (r12 x r34)
  SETUP_CUBLAS(ctx, cublasZgemm(blas, CUBLAS_OP_N, CUBLAS_OP_N, (int)(r1 * r2), (int)r34, (int)r12, &one, (const zc*)c12.p,
                                (int)(r1 * r2), (const zc*)c1234.p, (int)r12, &zero, (zc*)D.p, (int)(r1 * r2)));
  // E1 (n1 x r2 r34) = U1 (n1 x r1) . D (r1 x r2 r34)
  SETUP_CUBLAS(ctx, cublasZgemm(blas, CUBLAS_OP_N, CUBLAS_OP_N, (int)n1, (int)(r2 * r34), (int)r1, &one, (const zc*)u1.p,
                                (int)n1, (const zc*)D.p, (int)r1, &zero, (zc*)E1.p, (int)n1));
  // E(:,:,j) (n1 x n2) = E1(:,:,j) (n1 x r2) . U2^T (r2 x n2), for every j < r34
  SETUP_CUBLAS(ctx, cublasZgemmStridedBatched(blas, CUBLAS_OP_N, CUBLAS_OP_T, (int)n1, (int)n2, (int)r2, &one,
                                              (const zc*)E1.p, (int)n1, n1 * r2, (const zc*)u2.p, (int)n2, 0, &zero,
                                              (zc*)Ez.p, (int)n1, n1 * n2, (int)r34));
  k_z2c<<<nblk(n1 * n2 * r34), 256, 0, ctx->stream>>>(Ez.p, E, n1 * n2 * r34);
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return set_err(ctx, FMMT_E_CUDA, "H-Tucker E (FP64) failed");
  return FMMT_OK;
}

fmmt_status fmmt_internal::tt4d_T1_fp64(fmmt_ctx* ctx, const float2* U1, const float2* C1, int64_t n1, int64_t r1,
                                        int64_t n2, int64_t r2, float2* T1) {
  cublasHandle_t blas;
  cusolverDnHandle_t sol;
  SETUP_TRY(handles(ctx, &blas, &sol));
  ZBuf u1, c1, t1;
  SETUP_TRY(zalloc_from(ctx, u1, U1, n1 * r1));
  SETUP_TRY(zalloc_from(ctx, c1, C1, r1 * n2 * r2));
  SETUP_TRY(zalloc_from(ctx, t1, nullptr, n1 * n2 * r2));
  const zc one = make_cuDoubleComplex(1, 0), zero = make_cuDoubleComplex(0, 0);
  // T1 (n1 x n2 r2) = U1 (n1 x r1) . C1 (r1 x n2 r2)
  SETUP_CUBLAS(ctx, cublasZgemm(blas, CUBLAS_OP_N, CUBLAS_OP_N, (int)n1, (int)(n2 * r2), (int)r1, &one, (const zc*)u1.p,
                                (int)n1, (const zc*)c1.p, (int)r1, &zero, (zc*)t1.p, (int)n1));
  k_z2c<<<nblk(n1 * n2 * r2), 256, 0, ctx->stream>>>(t1.p, T1, n1 * n2 * r2);
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return set_err(ctx, FMMT_E_CUDA, "TT-4D T1 (FP64) failed");
  return FMMT_OK;
}
