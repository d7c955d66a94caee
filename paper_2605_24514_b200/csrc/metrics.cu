// K8 -- metrics kernels (metrics.py:74-119, linalg.py:126-153).
// All reductions are two-stage with a fixed order, so repeated runs are
// bit-identical (tests/test_stream.py:204-215 compares runs exactly).
#include "common.cuh"
#include "metrics.cuh"
#include "tall.cuh"
#include "../../include/isvd.h"

namespace isvd {

namespace {

constexpr int kFrobRows = 32;   // rows per CTA
constexpr int kFrobCols = 64;   // V rows staged per chunk
constexpr int kWMax = 160;

// ||A - U diag(s) V^T||_F^2 partial sums over a 32-row slab.
__global__ void __launch_bounds__(256) frob_partial_kernel(int m, int n, int w, const double* A,
                                                          int64_t a_stride, int lda, Mat U,
                                                          const double* s, int lds, Mat V,
                                                          double* partial, int nblk) {
  extern __shared__ double sm[];
  double* us = sm;                          // [kFrobRows][w+1]
  double* vs = sm + kFrobRows * (w + 1);    // [kFrobCols][w+1]
  __shared__ double red[32];
  const int b = blockIdx.y, blk = blockIdx.x;
  const int row0 = blk * kFrobRows;
  const double* Ab = A ? A + b * a_stride : nullptr;
  const double* Ub = U.p + b * U.stride;
  const double* Vb = V.p + b * V.stride;
  const double* sb = s + (int64_t)b * lds;
  const int W1 = w + 1;
  for (int idx = threadIdx.x; idx < kFrobRows * w; idx += blockDim.x) {
    int i = idx / w, t = idx % w;
    int row = row0 + i;
    us[i * W1 + t] = row < m ? Ub[(int64_t)row * U.ld + t] * sb[t] : 0.0;
  }
  double acc = 0.0;
  for (int c0 = 0; c0 < n; c0 += kFrobCols) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < kFrobCols * w; idx += blockDim.x) {
      int j = idx / w, t = idx % w;
      int col = c0 + j;
      vs[j * W1 + t] = col < n ? Vb[(int64_t)col * V.ld + t] : 0.0;
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < kFrobRows * kFrobCols; idx += blockDim.x) {
      int i = idx / kFrobCols, j = idx % kFrobCols;
      int row = row0 + i, col = c0 + j;
      if (row < m && col < n) {
        double rec = 0.0;
        for (int t = 0; t < w; ++t) rec = fma(us[i * W1 + t], vs[j * W1 + t], rec);
        double d = Ab[(int64_t)row * lda + col] - rec;
        acc = fma(d, d, acc);
      }
    }
  }
  double tot = block_sum(acc, red);
  if (threadIdx.x == 0) partial[(int64_t)b * nblk + blk] = tot;
}

// out[b] = sum_k partial[b][k] (fixed order: per-thread strided then tree)
__global__ void reduce_partials_kernel(const double* partial, int nblk, int width, double* out) {
  __shared__ double red[32];
  const int b = blockIdx.y, e = blockIdx.x;  // e: element within width
  double acc = 0.0;
  for (int k = threadIdx.x; k < nblk; k += blockDim.x)
    acc += partial[((int64_t)b * nblk + k) * width + e];
  double tot = block_sum(acc, red);
  if (threadIdx.x == 0) out[(int64_t)b * width + e] = tot;
}

// defect[b] = ||G[b] - I||_F for square w x w Gram matrices.
__global__ void defect_kernel(int w, const double* G, double* out) {
  __shared__ double red[32];
  const int b = blockIdx.x;
  const double* g = G + (int64_t)b * w * w;
  double acc = 0.0;
  for (int e = threadIdx.x; e < w * w; e += blockDim.x) {
    double d = g[e] - ((e / w == e % w) ? 1.0 : 0.0);
    acc = fma(d, d, acc);
  }
  double tot = block_sum(acc, red);
  if (threadIdx.x == 0) out[b] = sqrt(tot);
}

}  // namespace

int frob_nblk(int m) { return ceil_div(m, kFrobRows); }

int launch_frob_error_sq(int batch, int m, int n, int w, const double* A, int64_t a_stride, int lda,
                         Mat U, const double* s, int lds, Mat V, double* partial, double* out,
                         cudaStream_t st) {
  if (w > kWMax) {
    set_error("frob_error: width too large");
    return ISVD_EINVAL;
  }
  int nblk = frob_nblk(m);
  size_t smem = sizeof(double) * (kFrobRows + kFrobCols) * (w + 1);
  static bool attr = false;
  if (!attr) {
    ISVD_CUDA(cudaFuncSetAttribute(frob_partial_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   200 * 1024));
    attr = true;
  }
  frob_partial_kernel<<<dim3(nblk, batch), 256, smem, st>>>(m, n, w, A, a_stride, lda, U, s, lds, V,
                                                            partial, nblk);
  ISVD_LAUNCHED();
  reduce_partials_kernel<<<dim3(1, batch), 256, 0, st>>>(partial, nblk, 1, out);
  ISVD_LAUNCHED();
  return ISVD_OK;
}

int launch_gram(int batch, int rows, int wa, int wb, Mat Xa, Mat Xb, double* partial, double* out,
                cudaStream_t st) {
  const bool sym = Xa.p == Xb.p && Xa.ld == Xb.ld && Xa.stride == Xb.stride && wa == wb;
  return launch_gram_tiles(batch, rows, wa, wb, Xa, Xb, sym ? 1 : 0, partial, out, st);
}

// ---- a13: per-tick risk of BASELINE config 3 (finance.py:326-364).
// cov = V diag(s^2) V^T / (t-1), symmetrised as the reference does;
// D_j = max(0, sum_i A_ij^2 / (t-1) - cov_jj) (the diagonal term BASELINE
// asks for over the mean-centred returns); per portfolio p:
// out[p] = {sqrt(max(0, w'cov w)), sqrt(max(0, w'(cov + D)w)), z99 * that,
// w'cov w} (the last lets the host raise the reference's not-PSD error).
__global__ void risk_kernel(int n, int r, Mat V, const double* __restrict__ s, int lds,
                            const double* __restrict__ A, int64_t a_stride, int lda, int m,
                            double inv_t1, const double* __restrict__ w, int P,
                            double* __restrict__ cov, double* __restrict__ diag,
                            double* __restrict__ out) {
  extern __shared__ double rsm[];
  double* c = rsm;            // [n][n]
  double* dd = rsm + n * n;   // [n]
  __shared__ double red[32];
  const int b = blockIdx.x;
  const double* Vb = V.p + b * V.stride;
  const double* sb = s + (int64_t)b * lds;
  const double* Ab = A ? A + b * a_stride : nullptr;
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
    const int i = idx / n, j = idx % n;
    double cij = 0.0, cji = 0.0;
    for (int l = 0; l < r; ++l) {
      const double s2 = sb[l] * sb[l];
      cij = fma(Vb[i * V.ld + l] * s2, Vb[j * V.ld + l], cij);
      cji = fma(Vb[j * V.ld + l] * s2, Vb[i * V.ld + l], cji);
    }
    // no FMA contraction, so c_ij and c_ji round identically (bit-symmetric)
    c[idx] = 0.5 * __dadd_rn(__dmul_rn(cij, inv_t1), __dmul_rn(cji, inv_t1));
  }
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double acc = 0.0;
    if (A)
      for (int i = 0; i < m; ++i) acc = fma(Ab[(int64_t)i * lda + j], Ab[(int64_t)i * lda + j], acc);
    dd[j] = fmax(0.0, acc * inv_t1 - c[j * n + j]);
  }
  __syncthreads();
  if (cov)
    for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) cov[(int64_t)b * n * n + idx] = c[idx];
  if (diag)
    for (int j = threadIdx.x; j < n; j += blockDim.x) diag[(int64_t)b * n + j] = dd[j];
  for (int p = 0; p < P; ++p) {
    const double* wp = w + (int64_t)p * n;
    double q = 0.0, qd = 0.0;
    for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
      const int i = idx / n, j = idx % n;
      q = fma(wp[i] * c[idx], wp[j], q);
    }
    for (int j = threadIdx.x; j < n; j += blockDim.x) qd = fma(wp[j] * wp[j], dd[j], qd);
    q = block_sum(q, red);
    qd = block_sum(qd, red);
    if (threadIdx.x == 0) {
      const double z99 = 2.3263478740408408;  // Phi^{-1}(0.99)
      const double vd = sqrt(fmax(0.0, q + qd));
      double* o = out + ((int64_t)b * P + p) * 4;
      o[0] = sqrt(fmax(0.0, q));
      o[1] = vd;
      o[2] = z99 * vd;
      o[3] = q;
    }
  }
}

int launch_risk(int batch, int n, int r, Mat V, const double* s, int lds, const double* A,
                int64_t a_stride, int lda, int m, double inv_t1, const double* w, int P,
                double* cov, double* diag, double* out, cudaStream_t st) {
  const size_t smem = sizeof(double) * ((size_t)n * n + n);
  if (smem > 200 * 1024) {
    set_error("risk: too many assets for the on-chip covariance");
    return ISVD_EINVAL;
  }
  static bool attr = false;
  if (!attr) {
    ISVD_CUDA(cudaFuncSetAttribute(risk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   200 * 1024));
    attr = true;
  }
  risk_kernel<<<batch, 256, smem, st>>>(n, r, V, s, lds, A, a_stride, lda, m, inv_t1, w, P, cov,
                                        diag, out);
  ISVD_LAUNCHED();
  return ISVD_OK;
}

int launch_defect(int batch, int w, const double* G, double* out, cudaStream_t st) {
  defect_kernel<<<batch, 256, 0, st>>>(w, G, out);
  ISVD_LAUNCHED();
  return ISVD_OK;
}

}  // namespace isvd
