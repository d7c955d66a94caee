// Thin SVD of a very tall matrix through its Gram (configs 4 and 5b: init,
// refresh and oracle, linalg.py:84-109 / engine.py:89,173 / metrics.py:56-64).
//
// The blocked Jacobi of dense_svd.cu parallelises over column-block pairs,
// which starves the GPU when one matrix has 4M rows and 1024 columns (32 CTAs
// each streaming 1 GB per round).  For m >= 4n and m*n >= kGramMinElems:
//
//   G = A^T A                                   (DMMA Gram, tall.cu)
//   G = Vg diag(lambda) Vg^T                    (dense Jacobi on n x n)
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

// s_w[0:w] snapped in place; s_all = [s_w, sqrt(lambda[w:nc])] snapped (linalg.py:88-90)
__global__ void gram_spectrum_kernel(int w, int nc, double* __restrict__ s_w,
                                     const double* __restrict__ lam, double* __restrict__ s_all) {
  const double s0 = w > 0 ? s_w[0] : sqrt(fmax(lam[0], 0.0));
  auto snap = [&](double x) { return (s0 > 0.0 && x < kZeroSvRtol * s0) ? 0.0 : x; };
  __syncthreads();
  for (int i = threadIdx.x; i < nc; i += blockDim.x) {
    const double x = i < w ? s_w[i] : sqrt(fmax(lam[i], 0.0));
    if (s_all) s_all[i] = snap(x);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < w; i += blockDim.x) s_w[i] = snap(s_w[i]);
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
  // eigenvectors of the PSD Gram = its right singular vectors (rotation side)
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
    while (we < w && hl[we] > kGramRankTol * hl[0]) ++we;
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
    gram_spectrum_kernel<<<1, 256, 0, st>>>(w, std::min(m, n), s_w, lam, s_all);
    ISVD_LAUNCHED();
  }
  for (double* p : {G, part, x, jac, Vq, lam, swi, core, uk, vk, sv, vscr, s_tmp})
    if (p) cudaFreeAsync(p, st);
  if (flags) cudaFreeAsync(flags, st);
  return rc;
}

}  // namespace isvd
