// K8 -- metrics kernels (metrics.py:74-119, linalg.py:126-153).
// All reductions are two-stage with a fixed order, so repeated runs are
// bit-identical (tests/test_stream.py:204-215 compares runs exactly).
#include "common.cuh"
#include "metrics.cuh"
#include "tall.cuh"
#include "../../include/isvd.h"

namespace isvd {

namespace {

constexpr int kFT = 64;        // output tile edge (rows of A x columns of A)
constexpr int kFC = 32;        // contraction chunk (singular triplets)
constexpr int kFLd = kFC + 4;  // [kFT][kFLd] staging: conflict-free fragment loads and row stores
constexpr int kWMax = 160;

// ||A - U diag(s) V^T||_F^2 over one 64 x 64 tile of A (metrics.py:74-76):
// the reconstruction tile (U diag s) V^T is contracted on the FP64 tensor
// path (DMMA.8x8x4, 8 warps x (16 x 32) sub-tiles, 32-triplet chunks staged
// in shared memory with a register prefetch of the next chunk), the tile of
// A is loaded into registers before the contraction, and the epilogue
// squares the residual in the accumulator layout.  One partial per tile,
// summed in a fixed order by reduce_partials_kernel (deterministic).
__global__ void __launch_bounds__(256) frob_tile_kernel(int m, int n, int w, const double* A,
                                                       int64_t a_stride, int lda, Mat U,
                                                       const double* s, int lds, Mat V,
                                                       double* partial, int nblk) {
  __shared__ __align__(16) double Xs[kFT][kFLd];  // (U diag s) rows
  __shared__ __align__(16) double Vs[kFT][kFLd];  // V rows
  __shared__ double red[32];
  const int b = blockIdx.z;
  const int row0 = blockIdx.x * kFT, col0 = blockIdx.y * kFT;
  const double* Ab = A + b * a_stride;
  const double* Ub = U.p + b * U.stride;
  const double* Vb = V.p + b * V.stride;
  const double* sb = s + (int64_t)b * lds;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int mt0 = (warp >> 1) * 2, nt0 = (warp & 1) * 4;
  // the A entries this thread's accumulators cover, loaded up front
  double av[2][4][2];
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = row0 + (mt0 + t) * 8 + g, j = col0 + (nt0 + u) * 8 + 2 * q + e;
        av[t][u][e] = (i < m && j < n) ? Ab[(int64_t)i * lda + j] : 0.0;
      }
  // loader: element k of thread tid -> (row = idx / 32, triplet = idx % 32)
  double vx[8], vv[8];
  auto fetch = [&](int c0) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int idx = tid + k * 256;
      const int rr = idx >> 5, cc = idx & 31, t = c0 + cc;
      const bool tin = t < w;
      vx[k] = (tin && row0 + rr < m) ? Ub[(int64_t)(row0 + rr) * U.ld + t] * sb[t] : 0.0;
      vv[k] = (tin && col0 + rr < n) ? Vb[(int64_t)(col0 + rr) * V.ld + t] : 0.0;
    }
  };
  double acc[2][4][2];
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[t][u][0] = acc[t][u][1] = 0.0;
  fetch(0);
  for (int c0 = 0; c0 < w; c0 += kFC) {
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int idx = tid + k * 256;
      Xs[idx >> 5][idx & 31] = vx[k];
      Vs[idx >> 5][idx & 31] = vv[k];
    }
    __syncthreads();
    if (c0 + kFC < w) fetch(c0 + kFC);
#pragma unroll
    for (int kk = 0; kk < kFC / 4; ++kk) {
      const int kc = kk * 4 + q;
      double a[2], bf[4];
#pragma unroll
      for (int t = 0; t < 2; ++t) a[t] = Xs[(mt0 + t) * 8 + g][kc];
#pragma unroll
      for (int u = 0; u < 4; ++u) bf[u] = Vs[(nt0 + u) * 8 + g][kc];
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int u = 0; u < 4; ++u) dmma_8x8x4(acc[t][u][0], acc[t][u][1], a[t], bf[u]);
    }
  }
  double sq = 0.0;
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double d = av[t][u][e] - acc[t][u][e];  // out-of-range entries: 0 - 0
        sq = fma(d, d, sq);
      }
  const double tot = block_sum(sq, red);
  if (tid == 0) partial[(int64_t)b * nblk + (int64_t)blockIdx.y * gridDim.x + blockIdx.x] = tot;
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

int frob_nblk(int m, int n) { return ceil_div(m, kFT) * ceil_div(n, kFT); }

int launch_frob_error_sq(int batch, int m, int n, int w, const double* A, int64_t a_stride, int lda,
                         Mat U, const double* s, int lds, Mat V, double* partial, double* out,
                         cudaStream_t st) {
  if (w > kWMax) {
    set_error("frob_error: width too large");
    return ISVD_EINVAL;
  }
  if (batch == 0) return ISVD_OK;
  const int gx = ceil_div(m, kFT), gy = ceil_div(n, kFT);
  if (gy > 65535 || batch > 65535) {
    set_error("frob_error: matrix too wide");
    return ISVD_EINVAL;
  }
  const int nblk = gx * gy;
  frob_tile_kernel<<<dim3(gx, gy, batch), 256, 0, st>>>(m, n, w, A, a_stride, lda, U, s, lds, V,
                                                        partial, nblk);
  ISVD_LAUNCHED();
  reduce_partials_kernel<<<dim3(1, batch), 1024, 0, st>>>(partial, nblk, 1, out);
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
