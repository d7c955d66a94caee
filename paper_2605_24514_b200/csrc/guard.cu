// a7 -- the optional re-orthonormalisation guard (engine.py:210-217).
//
// Reference: if max(||U^T U - I||_F, ||V^T V - I||_F) > REORTHO_THRESHOLD,
// QR(U) = Qu Ru, QR(V) = Qv Rv, core_svd((Ru diag s) Rv^T) = Uk s' Vk^T,
// U <- Qu Uk, V <- Qv Vk.  Here the QR is CholeskyQR (Gram on the device,
// Cholesky of the w x w Gram, R upper with positive diagonal; Householder
// QR differs only by column signs, which the core SVD absorbs), and
// Qu Uk = U (Ru^{-1} Uk) is applied with the rotation kernel, so U is read
// and written once.
#include <vector>
#include "common.cuh"
#include "core_svd.cuh"
#include "guard.cuh"
#include "metrics.cuh"
#include "../../include/isvd.h"

namespace isvd {

namespace {

// in-place upper Cholesky of each w x w Gram (G = R^T R), one CTA per stream
__global__ void chol_kernel(int w, double* __restrict__ G) {
  double* g = G + (int64_t)blockIdx.x * w * w;
  for (int k = 0; k < w; ++k) {
    if (threadIdx.x == 0) g[k * w + k] = sqrt(fmax(g[k * w + k], 1e-300));
    __syncthreads();
    const double d = g[k * w + k];
    for (int j = k + 1 + threadIdx.x; j < w; j += blockDim.x) g[k * w + j] /= d;
    __syncthreads();
    const int rem = w - k - 1;
    for (int idx = threadIdx.x; idx < rem * rem; idx += blockDim.x) {
      const int i = k + 1 + idx / rem, j = k + 1 + idx % rem;
      if (j >= i) g[i * w + j] -= g[k * w + i] * g[k * w + j];
    }
    __syncthreads();
  }
}

// core[i][j] = sum_{k >= max(i,j)} Ru[i][k] s[k] Rv[j][k]
__global__ void guard_core_kernel(int w, const double* __restrict__ Ru,
                                  const double* __restrict__ Rv, const double* __restrict__ s,
                                  int lds, double* __restrict__ core, int64_t core_stride,
                                  int ldc) {
  const int b = blockIdx.x;
  const double* ru = Ru + (int64_t)b * w * w;
  const double* rv = Rv + (int64_t)b * w * w;
  const double* sb = s + (int64_t)b * lds;
  double* C = core + b * core_stride;
  for (int idx = threadIdx.x; idx < w * w; idx += blockDim.x) {
    const int i = idx / w, j = idx % w;
    double acc = 0.0;
    for (int k = max(i, j); k < w; ++k) acc = fma(ru[i * w + k] * sb[k], rv[j * w + k], acc);
    C[i * ldc + j] = acc;
  }
}

// M = R^{-1} Q (R upper, w x w); one thread per column of Q (pitch ldq),
// result written back into Q's storage.
__global__ void trsm_upper_kernel(int w, const double* __restrict__ R, double* __restrict__ Q,
                                  int64_t q_stride, int ldq) {
  const int b = blockIdx.x;
  const double* r = R + (int64_t)b * w * w;
  double* q = Q + b * q_stride;
  for (int c = threadIdx.x; c < w; c += blockDim.x) {
    for (int i = w - 1; i >= 0; --i) {
      double acc = q[i * ldq + c];
      for (int k = i + 1; k < w; ++k) acc -= r[i * w + k] * q[k * ldq + c];
      q[i * ldq + c] = acc / r[i * w + i];
    }
  }
}

}  // namespace

int reortho_defects(int batch, int w, Mat U, int m, Mat V, int n, double* host_du, double* host_dv,
                    cudaStream_t st, const Allreducer* ar) {
  const int rows = m > n ? m : n;
  const size_t np = (size_t)gram_part_elems(batch, rows, w, w);
  double *part = nullptr, *G = nullptr, *d = nullptr;
  ISVD_CUDA(cudaMallocAsync((void**)&part, sizeof(double) * np, st));
  ISVD_CUDA(cudaMallocAsync((void**)&G, sizeof(double) * batch * w * w, st));
  ISVD_CUDA(cudaMallocAsync((void**)&d, sizeof(double) * batch * 2, st));
  int rc = launch_gram(batch, m, w, w, U, U, part, G, st);
  if (rc == ISVD_OK && ar) rc = (*ar)(G, (int64_t)batch * w * w);
  if (rc == ISVD_OK) rc = launch_defect(batch, w, G, d, st);
  if (rc == ISVD_OK) rc = launch_gram(batch, n, w, w, V, V, part, G, st);
  if (rc == ISVD_OK) rc = launch_defect(batch, w, G, d + batch, st);
  if (rc == ISVD_OK) {
    cudaMemcpyAsync(host_du, d, sizeof(double) * batch, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(host_dv, d + batch, sizeof(double) * batch, cudaMemcpyDeviceToHost, st);
  }
  cudaFreeAsync(part, st);
  cudaFreeAsync(G, st);
  cudaFreeAsync(d, st);
  ISVD_CUDA(cudaStreamSynchronize(st));
  return rc;
}

int reortho_apply(int batch, int w, Mat U, int m, Mat V, int n, double* s, int lds, double* core,
                  double* uk, double* vk, int64_t cstride, int S, double* sv, double* vscr,
                  cudaStream_t st, const Allreducer* ar) {
  if (w < 1) return ISVD_OK;
  const int rows = m > n ? m : n;
  const size_t np = (size_t)gram_part_elems(batch, rows, w, w);
  double *part = nullptr, *Ru = nullptr, *Rv = nullptr;
  ISVD_CUDA(cudaMallocAsync((void**)&part, sizeof(double) * np, st));
  ISVD_CUDA(cudaMallocAsync((void**)&Ru, sizeof(double) * batch * w * w, st));
  ISVD_CUDA(cudaMallocAsync((void**)&Rv, sizeof(double) * batch * w * w, st));
  int rc = launch_gram(batch, m, w, w, U, U, part, Ru, st);
  if (rc == ISVD_OK && ar) rc = (*ar)(Ru, (int64_t)batch * w * w);  // U^T U over all shards
  if (rc == ISVD_OK) rc = launch_gram(batch, n, w, w, V, V, part, Rv, st);
  if (rc == ISVD_OK) {
    chol_kernel<<<batch, 128, 0, st>>>(w, Ru);
    ISVD_LAUNCHED();
    chol_kernel<<<batch, 128, 0, st>>>(w, Rv);
    ISVD_LAUNCHED();
    guard_core_kernel<<<batch, 128, 0, st>>>(w, Ru, Rv, s, lds, core, cstride, S);
    ISVD_LAUNCHED();
    rc = launch_core_svd(batch, w, core, cstride, S, uk, vk, cstride, S, sv, S, vscr, nullptr, st);
  }
  if (rc == ISVD_OK) {
    // Uk <- Ru^{-1} Uk, Vk <- Rv^{-1} Vk, then U <- U Uk, V <- V Vk
    trsm_upper_kernel<<<batch, 128, 0, st>>>(w, Ru, uk, cstride, S);
    ISVD_LAUNCHED();
    trsm_upper_kernel<<<batch, 128, 0, st>>>(w, Rv, vk, cstride, S);
    ISVD_LAUNCHED();
    RotJob ju{U, m, uk, cstride, S, nullptr, 0, nullptr, 0};
    RotJob jv{V, n, vk, cstride, S, nullptr, 0, nullptr, 0};
    rc = launch_rotate(batch, w, w, ju, &jv, st);
  }
  if (rc == ISVD_OK)
    rc = cudaMemcpy2DAsync(s, sizeof(double) * lds, sv, sizeof(double) * S, sizeof(double) * w,
                           batch, cudaMemcpyDeviceToDevice, st) == cudaSuccess
             ? ISVD_OK
             : ISVD_ENODEV;
  cudaFreeAsync(part, st);
  cudaFreeAsync(Ru, st);
  cudaFreeAsync(Rv, st);
  return rc;
}

}  // namespace isvd
