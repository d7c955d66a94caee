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
  const double* Ab = A + b * a_stride;
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

int launch_defect(int batch, int w, const double* G, double* out, cudaStream_t st) {
  defect_kernel<<<batch, 256, 0, st>>>(w, G, out);
  ISVD_LAUNCHED();
  return ISVD_OK;
}

}  // namespace isvd
