// Thin SVD of a very tall matrix through its Gram (configs 4 and 5b: init,
// refresh and oracle, linalg.py:84-109 / engine.py:89,173 / metrics.py:56-64).
//
// The blocked Jacobi of dense_svd.cu parallelises over column-block pairs,
// which starves the GPU when one matrix has 4M rows and 1024 columns (32 CTAs
// each streaming 1 GB per round).  For m >= 4n and m*n >= kGramMinElems:
//
//   G = A^T A                                   (DMMA Gram, tall.cu)
//   G = L L^T, L V' = Vg diag(sigma)            (blocked Cholesky on DMMA, then
//                                                dense Jacobi on L's columns;
//                                                singular G: eig of G itself)
//   B = A Vg[:, :w']                            (DMMA GEMM, tall.cu)
//   B = Q R, R = Ur S Vr^T, twice               (CholeskyQR + core SVD = the
//                                                reortho guard, guard.cu)
//   U = Q Ur, V = Vg[:, :w'] Vr, sigma = S
//
// The leading w' triplets come out of a Rayleigh-Ritz step on A itself, so
// sigma and U carry the accuracy of a QR-based SVD of B; the subspace is
// Vg's, accurate to eps * sigma_1^2 / (sigma_w'^2 - sigma_w'+1^2).  w' is the
// numerical rank of G within the requested w (lambda_i > kGramRankTol *
// lambda_0, i.e. sigma_i > 1e-7 sigma_0 -- the Gram cannot resolve smaller
// singular values); the remaining columns get sigma = 0 and are completed
// by the caller (engine.py:33-70).  The tail of the spectrum (index >= w)
// is sqrt(lambda_i), good to eps * sigma_0^2 / sigma_i absolute.
#include <algorithm>
#include <cmath>
#include <vector>
#include "common.cuh"
#include "core_svd.cuh"
#include "dense_svd.cuh"
#include "guard.cuh"
#include "tall.cuh"
#include "../../include/isvd.h"

namespace isvd {

namespace {

constexpr double kGramRankTol = 1e-14;

__global__ void fill_kernel(int n, double* __restrict__ p, double v) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = v;
}

// s_w[0:w] snapped in place; s_all = [s_w, sqrt(lambda[w:nc])] snapped
// (linalg.py:88-90); is_sigma: lam already holds singular values
__global__ void gram_spectrum_kernel(int w, int nc, double* __restrict__ s_w,
                                     const double* __restrict__ lam, double* __restrict__ s_all,
                                     int is_sigma) {
  auto sv = [&](int i) { return is_sigma ? lam[i] : sqrt(fmax(lam[i], 0.0)); };
  const double s0 = w > 0 ? s_w[0] : sv(0);
  auto snap = [&](double x) { return (s0 > 0.0 && x < kZeroSvRtol * s0) ? 0.0 : x; };
  __syncthreads();
  for (int i = threadIdx.x; i < nc; i += blockDim.x) {
    const double x = i < w ? s_w[i] : sv(i);
    if (s_all) s_all[i] = snap(x);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < w; i += blockDim.x) s_w[i] = snap(s_w[i]);
}


// ---- Blocked lower Cholesky G = L L^T in place (row-major n x n, lower
// triangle read and written), 32-column panels, right-looking:
//   potrf of the diagonal block (one CTA), the panel below by forward
//   substitution (thread per row), the trailing lower triangle updated by
//   the panel's outer product on DMMA (64 x 64 tiles).
// *fail is set when a pivot is not positive (numerically singular Gram).
constexpr int kCb = 32;

__global__ void __launch_bounds__(1024) chol_potrf_kernel(int n, double* __restrict__ G, int k,
                                                          int* __restrict__ fail) {
  __shared__ double Ab[kCb][kCb + 1];
  const int nb = min(kCb, n - k);
  const int i = threadIdx.x >> 5, j = threadIdx.x & 31;
  if (i < nb && j <= i) Ab[i][j] = G[(int64_t)(k + i) * n + k + j];
  __syncthreads();
  for (int c = 0; c < nb; ++c) {
    if (threadIdx.x == 0) {
      const double d = Ab[c][c];
      if (!(d > 0.0)) *fail = 1;
      Ab[c][c] = d > 0.0 ? sqrt(d) : 1.0;
    }
    __syncthreads();
    if (j == c && i > c && i < nb) Ab[i][c] /= Ab[c][c];
    __syncthreads();
    if (i > c && i < nb && j > c && j <= i) Ab[i][j] -= Ab[i][c] * Ab[j][c];
    __syncthreads();
  }
  if (i < nb && j <= i) G[(int64_t)(k + i) * n + k + j] = Ab[i][j];
}

// rows k + nb ... n - 1 of the panel: x L_kk^T = g  (forward substitution)
__global__ void __launch_bounds__(128) chol_trsm_kernel(int n, double* __restrict__ G, int k) {
  __shared__ double Lk[kCb][kCb + 1];
  const int nb = min(kCb, n - k);
  for (int idx = threadIdx.x; idx < kCb * kCb; idx += blockDim.x) {
    const int a = idx / kCb, c = idx % kCb;
    Lk[a][c] = (a < nb && c <= a) ? G[(int64_t)(k + a) * n + k + c] : 0.0;
  }
  __syncthreads();
  const int row = k + nb + blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  double* gr = G + (int64_t)row * n + k;
  double x[kCb];
#pragma unroll
  for (int c = 0; c < kCb; ++c) x[c] = c < nb ? gr[c] : 0.0;
#pragma unroll
  for (int c = 0; c < kCb; ++c) {
    if (c < nb) {
      double v = x[c];
#pragma unroll
      for (int l = 0; l < c; ++l) v = fma(-x[l], Lk[c][l], v);
      x[c] = v / Lk[c][c];
    }
  }
#pragma unroll
  for (int c = 0; c < kCb; ++c)
    if (c < nb) gr[c] = x[c];
}

// trailing lower triangle: T[a][b] -= sum_c P[a][c] P[b][c], P = L[k+nb:, k:k+nb]
__global__ void __launch_bounds__(256) chol_syrk_kernel(int n, double* __restrict__ G, int k, int ntb) {
  __shared__ __align__(16) double Pa[64][kCb + 4];
  __shared__ __align__(16) double Pb[64][kCb + 4];
  const int nb = min(kCb, n - k);
  const int t0 = k + nb, m = n - t0;
  // lower-triangular tile enumeration: row ti holds tiles 0..ti
  int ti = 0, left = blockIdx.x;
  while (left > ti) {
    left -= ti + 1;
    ++ti;
  }
  const int tj = left;
  (void)ntb;
  const int a0 = ti * 64, b0 = tj * 64;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int mt0 = (warp >> 1) * 2, nt0 = (warp & 1) * 4;
  for (int idx = tid; idx < 64 * kCb; idx += 256) {
    const int rr = idx >> 5, cc = idx & 31;
    const bool cin = cc < nb;
    Pa[rr][cc] = (cin && a0 + rr < m) ? G[(int64_t)(t0 + a0 + rr) * n + k + cc] : 0.0;
    Pb[rr][cc] = (cin && b0 + rr < m) ? G[(int64_t)(t0 + b0 + rr) * n + k + cc] : 0.0;
  }
  __syncthreads();
  double acc[2][4][2];
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[t][u][0] = acc[t][u][1] = 0.0;
#pragma unroll
  for (int kk = 0; kk < kCb / 4; ++kk) {
    const int kc = kk * 4 + q;
    double av[2], bv[4];
#pragma unroll
    for (int t = 0; t < 2; ++t) av[t] = Pa[(mt0 + t) * 8 + g][kc];
#pragma unroll
    for (int u = 0; u < 4; ++u) bv[u] = Pb[(nt0 + u) * 8 + g][kc];
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
      for (int u = 0; u < 4; ++u) dmma_8x8x4(acc[t][u][0], acc[t][u][1], av[t], bv[u]);
  }
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int a = a0 + (mt0 + t) * 8 + g, bcol = b0 + (nt0 + u) * 8 + 2 * q + e;
        if (a < m && bcol <= a) {
          double* c = G + (int64_t)(t0 + a) * n + t0 + bcol;
          *c -= acc[t][u][e];
        }
      }
}

__global__ void chol_zero_upper_kernel(int n, double* __restrict__ G) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)n * n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(idx / n), j = (int)(idx % n);
    if (j > i) G[idx] = 0.0;
  }
}

// G -> its lower Cholesky factor in place; *fail (device) set on breakdown
int cholesky_lower(int n, double* G, int* fail, cudaStream_t st) {
  for (int k = 0; k < n; k += kCb) {
    chol_potrf_kernel<<<1, 1024, 0, st>>>(n, G, k, fail);
    ISVD_LAUNCHED();
    const int nb = std::min(kCb, n - k), m = n - k - nb;
    if (m <= 0) break;
    chol_trsm_kernel<<<ceil_div(m, 128), 128, 0, st>>>(n, G, k);
    ISVD_LAUNCHED();
    const int tn = ceil_div(m, 64);
    chol_syrk_kernel<<<tn * (tn + 1) / 2, 256, 0, st>>>(n, G, k, tn);
    ISVD_LAUNCHED();
  }
  chol_zero_upper_kernel<<<std::min(ceil_div((int64_t)n * n, 256), 4096), 256, 0, st>>>(n, G);
  ISVD_LAUNCHED();
  return ISVD_OK;
}

}  // namespace

bool use_gram_path(int m, int n, int w) {
  return (int64_t)m >= 4 * (int64_t)n && n >= 16 && (int64_t)m * n >= kGramMinElems &&
         w <= kGramMaxW;
}

int gram_svd_run(int m, int n, const double* a, int lda, int w, Mat u, Mat v, double* s_w,
                 double* s_all, cudaStream_t st, const Allreducer* ar) {
  w = std::max(0, std::min(w, n));
  const int ldq = round_up(std::max(w, 1), 8);
  const int64_t np = gram_part_elems(1, m, n, n);
  DenseSvdPlan P = dense_svd_plan(n, n, w);
  const int S = std::max(w, 1);
  double *G = nullptr, *part = nullptr, *x = nullptr, *jac = nullptr, *Vq = nullptr,
         *lam = nullptr, *swi = nullptr, *core = nullptr, *uk = nullptr, *vk = nullptr,
         *sv = nullptr, *vscr = nullptr, *s_tmp = nullptr;
  int* flags = nullptr;
  std::vector<int> hflags(1, 0);
  int rc = ISVD_OK;
  auto T = [&](int v2) { if (rc == ISVD_OK) rc = v2; };
  auto M = [&](double** p, int64_t elems) {
    if (rc == ISVD_OK && cudaMallocAsync((void**)p, sizeof(double) * std::max<int64_t>(elems, 1), st) != cudaSuccess) {
      set_error("gram_svd: device allocation failed");
      rc = ISVD_ENODEV;
    }
  };
  M(&G, (int64_t)n * n);
  M(&part, np);
  M(&x, P.x_elems());
  M(&jac, P.j_elems());
  M(&Vq, (int64_t)n * ldq);
  M(&lam, n);
  M(&swi, ldq);
  M(&core, (int64_t)S * S);
  M(&uk, (int64_t)S * S);
  M(&vk, (int64_t)S * S);
  M(&sv, S);
  M(&vscr, (int64_t)S * (S | 1));
  M(&s_tmp, S);
  if (rc == ISVD_OK && cudaMallocAsync((void**)&flags, sizeof(int), st) != cudaSuccess) rc = ISVD_ENODEV;
  Mat Am{const_cast<double*>(a), 0, lda};
  Mat Gm{G, 0, n};
  Mat Vqm{Vq, 0, ldq};
  T(launch_gram_tiles(1, m, n, n, Am, Am, 1, part, G, st));
  if (ar) T((*ar)(G, (int64_t)n * n));  // A^T A over all row shards
  // Preconditioned: L = chol(A^T A) (lower, = R^T of A = QR) and one-sided
  // Jacobi on the columns of L: L V' = U' S gives S = sigma(A) and U' = the
  // right singular vectors of A (normalised side).  The columns of L are as
  // well conditioned as A's, so the blocked Jacobi needs far fewer sweeps
  // than on the columns of A^T A (whose Gram squares kappa again: 24 sweeps
  // at 25000 x 6000).  A numerically singular Gram (pivot <= 0) falls back
  // to the eigenvectors of A^T A itself.
  bool sigma_out = false;
  {
    double* L = nullptr;
    int* cf = nullptr;
    M(&L, (int64_t)n * n);
    if (rc == ISVD_OK && cudaMallocAsync((void**)&cf, sizeof(int), st) != cudaSuccess) rc = ISVD_ENODEV;
    int hcf = 1;
    if (rc == ISVD_OK) {
      T(cudaMemsetAsync(cf, 0, sizeof(int), st) == cudaSuccess ? ISVD_OK : ISVD_ENODEV);
      T(cudaMemcpyAsync(L, G, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, st) == cudaSuccess
            ? ISVD_OK : ISVD_ENODEV);
      T(cholesky_lower(n, L, cf, st));
      T(cudaMemcpyAsync(&hcf, cf, sizeof(int), cudaMemcpyDeviceToHost, st) == cudaSuccess
            ? ISVD_OK : ISVD_ENODEV);
      T(cudaStreamSynchronize(st) == cudaSuccess ? ISVD_OK : ISVD_ENODEV);
    }
    if (rc == ISVD_OK && hcf == 0) {
      T(dense_svd_run(1, n, n, L, (int64_t)n * n, n, w, Vqm, Mat{nullptr, 0, 0}, swi, ldq, lam, n, x,
                      jac, flags, hflags.data(), st, nullptr));
      sigma_out = true;
    }
    if (L) cudaFreeAsync(L, st);
    if (cf) cudaFreeAsync(cf, st);
  }
  // eigenvectors of the PSD Gram = its right singular vectors (rotation side)
  if (!sigma_out)
    T(dense_svd_run(1, n, n, G, (int64_t)n * n, n, w, Mat{nullptr, 0, 0}, Vqm, swi, ldq, lam, n, x,
                    jac, flags, hflags.data(), st, nullptr));
  std::vector<double> hl(n, 0.0);
  if (rc == ISVD_OK) {
    if (cudaMemcpyAsync(hl.data(), lam, sizeof(double) * n, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
      set_error("gram_svd: device failure");
      rc = ISVD_ENODEV;
    }
  }
  int we = 0;
  if (rc == ISVD_OK && hl[0] > 0.0)
    while (we < w && (sigma_out ? hl[we] * hl[we] > kGramRankTol * hl[0] * hl[0]
                                : hl[we] > kGramRankTol * hl[0]))
      ++we;
  if (rc == ISVD_OK && w > 0) {
    // V[:, :w] = Vg[:, :w]; U[:, we:w] = 0, sigma[we:w] = 0
    T(launch_copy_rows(1, n, w, Vq, 0, ldq, v.p, 0, v.ld, st));
    T(cudaMemset2DAsync(u.p, sizeof(double) * u.ld, 0, sizeof(double) * w, m, st) == cudaSuccess
          ? ISVD_OK : ISVD_ENODEV);
    T(cudaMemsetAsync(s_w, 0, sizeof(double) * w, st) == cudaSuccess ? ISVD_OK : ISVD_ENODEV);
  }
  if (rc == ISVD_OK && we > 0) {
    T(launch_gemm_tall(1, m, n, we, Am, Vqm, u, st));
    fill_kernel<<<1, 128, 0, st>>>(we, s_w, 1.0);
    ISVD_LAUNCHED();
    // two CholeskyQR + core-SVD passes (CholeskyQR2): B = Q R, R = Ur S Vr^T
    for (int pass = 0; pass < 2 && rc == ISVD_OK; ++pass)
      T(reortho_apply(1, we, u, m, v, n, s_w, S, core, uk, vk, (int64_t)S * S, S, sv, vscr, st, ar));
  }
  if (rc == ISVD_OK) {
    gram_spectrum_kernel<<<1, 256, 0, st>>>(w, std::min(m, n), s_w, lam, s_all, sigma_out ? 1 : 0);
    ISVD_LAUNCHED();
  }
  for (double* p : {G, part, x, jac, Vq, lam, swi, core, uk, vk, sv, vscr, s_tmp})
    if (p) cudaFreeAsync(p, st);
  if (flags) cudaFreeAsync(flags, st);
  return rc;
}

}  // namespace isvd
