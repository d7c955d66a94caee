// Tall-skinny contractions on the FP64 tensor path (DMMA.8x8x4):
//
//   Gram   C = Xa^T Xb        (rows x wa)^T (rows x wb), rows up to 2^22+
//   GEMM   C = X Q            (rows x n) (n x wc)
//
// These are the only dense contractions of the path (BASELINE north_star
// item 5): the Gram feeds the CholeskyQR of the re-orthonormalisation guard
// (engine.py:210-217), the orthonormality / angle metrics (linalg.py:126-153)
// and the Gram-based thin SVD of very tall matrices (init / refresh /
// oracle of configs 4 and 5b, linalg.py:84-109); the GEMM projects the
// tracked matrix onto the Gram eigenbasis.
//
// Gram: one CTA per 64 x 64 output tile and row split; 32-row chunks of both
// operands are staged in shared memory (register prefetch of the next chunk
// overlaps the DMMA work), 8 warps x (16 x 32) sub-tiles.  Each split writes
// its partial tile; a second kernel sums the splits in a fixed order, so the
// result is deterministic for a given shape.  Symmetric Grams compute only
// the tiles on and above the diagonal.
#include <algorithm>
#include "common.cuh"
#include "tall.cuh"
#include "../../include/isvd.h"

namespace isvd {

namespace {

constexpr int kT = 64;          // output tile edge
constexpr int kC = 32;          // contraction chunk
constexpr int kLd = kT + 4;     // [kC][kLd] staging: conflict-free fragment loads
constexpr int kLdx = kC + 4;    // [kT][kLdx] staging of the GEMM's X tile
constexpr int kThreads = 256;

__device__ __forceinline__ void tile_of(int t, int ntb, int sym, int& ti, int& tj) {
  if (!sym) {
    ti = t / ntb;
    tj = t % ntb;
    return;
  }
  // upper-triangular enumeration: row ti holds tiles ti..ntb-1
  int i = 0, left = t;
  while (left >= ntb - i) {
    left -= ntb - i;
    ++i;
  }
  ti = i;
  tj = i + left;
}

__global__ void __launch_bounds__(kThreads) gram_tile_kernel(int rows, int wa, int wb, Mat Xa,
                                                             Mat Xb, int sym, int ntb, int chunk,
                                                             int S, double* __restrict__ part) {
  __shared__ __align__(16) double As[kC][kLd];
  __shared__ __align__(16) double Bs[kC][kLd];
  const int b = blockIdx.z, split = blockIdx.y;
  int ti, tj;
  tile_of(blockIdx.x, ntb, sym, ti, tj);
  const int i0 = ti * kT, j0 = tj * kT;
  const int r_begin = split * chunk;
  const int r_end = min(rows, r_begin + chunk);
  const double* A = Xa.p + b * Xa.stride;
  const double* Bm = Xb.p + b * Xb.stride;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int mt0 = (warp >> 1) * 2, nt0 = (warp & 1) * 4;
  // loader: element q of thread tid -> (row = idx / 64, col = idx % 64)
  double va[8], vb[8];
  auto fetch = [&](int r0) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int idx = tid + q * kThreads;
      const int rr = idx >> 6, cc = idx & 63;
      const int row = r0 + rr;
      const bool in = row < r_end;
      va[q] = (in && i0 + cc < wa) ? A[(int64_t)row * Xa.ld + i0 + cc] : 0.0;
      vb[q] = (in && j0 + cc < wb) ? Bm[(int64_t)row * Xb.ld + j0 + cc] : 0.0;
    }
  };
  double acc[2][4][2];
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[t][u][0] = acc[t][u][1] = 0.0;
  if (r_begin < r_end) fetch(r_begin);
  for (int r0 = r_begin; r0 < r_end; r0 += kC) {
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int idx = tid + q * kThreads;
      As[idx >> 6][idx & 63] = va[q];
      Bs[idx >> 6][idx & 63] = vb[q];
    }
    __syncthreads();
    if (r0 + kC < r_end) fetch(r0 + kC);
#pragma unroll
    for (int kk = 0; kk < kC / 4; ++kk) {
      const int kr = kk * 4 + (lane & 3);
      double a[2], bf[4];
#pragma unroll
      for (int t = 0; t < 2; ++t) a[t] = As[kr][(mt0 + t) * 8 + (lane >> 2)];
#pragma unroll
      for (int u = 0; u < 4; ++u) bf[u] = Bs[kr][(nt0 + u) * 8 + (lane >> 2)];
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int u = 0; u < 4; ++u) dmma_8x8x4(acc[t][u][0], acc[t][u][1], a[t], bf[u]);
    }
  }
  double* P = part + ((int64_t)b * S + split) * wa * wb;
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + (mt0 + t) * 8 + (lane >> 2);
      const int j = j0 + (nt0 + u) * 8 + 2 * (lane & 3);
      if (i < wa) {
        if (j < wb) P[(int64_t)i * wb + j] = acc[t][u][0];
        if (j + 1 < wb) P[(int64_t)i * wb + j + 1] = acc[t][u][1];
      }
    }
}

// out[b][i][j] = sum_s part[b][s][i][j] (fixed order); for symmetric Grams the
// lower tiles are mirrored from the upper ones.
__global__ void gram_reduce_kernel(int wa, int wb, int S, int sym, const double* __restrict__ part,
                                   double* __restrict__ out) {
  const int b = blockIdx.y;
  const int64_t total = (int64_t)wa * wb;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(e / wb), j = (int)(e % wb);
    if (sym && (i / kT) > (j / kT)) {
      const int t = i;
      i = j;
      j = t;
    }
    const double* p = part + (int64_t)b * S * total + (int64_t)i * wb + j;
    double acc = 0.0;
    for (int s = 0; s < S; ++s) acc += p[(int64_t)s * total];
    out[(int64_t)b * total + e] = acc;
  }
}

// C[b] (rows x wc, pitch C.ld) = X[b] (rows x n) . Q[b] (n x wc)
__global__ void __launch_bounds__(kThreads) gemm_tile_kernel(int rows, int n, int wc, Mat X, Mat Q,
                                                             Mat C) {
  __shared__ __align__(16) double Xs[kT][kLdx];
  __shared__ __align__(16) double Qs[kC][kLd];
  const int b = blockIdx.z;
  const int row0 = blockIdx.x * kT, j0 = blockIdx.y * kT;
  const double* Xb = X.p + b * X.stride;
  const double* Qb = Q.p + b * Q.stride;
  double* Cb = C.p + b * C.stride;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int mt0 = (warp >> 1) * 2, nt0 = (warp & 1) * 4;
  double vx[8], vq[8];
  auto fetch = [&](int c0) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int idx = tid + q * kThreads;
      {
        const int rr = idx >> 5, cc = idx & 31;  // X tile: 64 rows x 32 cols
        const int row = row0 + rr, col = c0 + cc;
        vx[q] = (row < rows && col < n) ? Xb[(int64_t)row * X.ld + col] : 0.0;
      }
      {
        const int rr = idx >> 6, cc = idx & 63;  // Q tile: 32 rows x 64 cols
        const int row = c0 + rr, col = j0 + cc;
        vq[q] = (row < n && col < wc) ? Qb[(int64_t)row * Q.ld + col] : 0.0;
      }
    }
  };
  double acc[2][4][2];
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[t][u][0] = acc[t][u][1] = 0.0;
  fetch(0);
  for (int c0 = 0; c0 < n; c0 += kC) {
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int idx = tid + q * kThreads;
      Xs[idx >> 5][idx & 31] = vx[q];
      Qs[idx >> 6][idx & 63] = vq[q];
    }
    __syncthreads();
    if (c0 + kC < n) fetch(c0 + kC);
#pragma unroll
    for (int kk = 0; kk < kC / 4; ++kk) {
      const int kc = kk * 4 + (lane & 3);
      double a[2], bf[4];
#pragma unroll
      for (int t = 0; t < 2; ++t) a[t] = Xs[(mt0 + t) * 8 + (lane >> 2)][kc];
#pragma unroll
      for (int u = 0; u < 4; ++u) bf[u] = Qs[kc][(nt0 + u) * 8 + (lane >> 2)];
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int u = 0; u < 4; ++u) dmma_8x8x4(acc[t][u][0], acc[t][u][1], a[t], bf[u]);
    }
  }
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = row0 + (mt0 + t) * 8 + (lane >> 2);
      const int j = j0 + (nt0 + u) * 8 + 2 * (lane & 3);
      if (i < rows) {
        if (j < wc) Cb[(int64_t)i * C.ld + j] = acc[t][u][0];
        if (j + 1 < wc) Cb[(int64_t)i * C.ld + j + 1] = acc[t][u][1];
      }
    }
}

}  // namespace

int gram_splits(int batch, int rows, int wa, int wb) {
  const int ta = ceil_div(wa, kT), tb = ceil_div(wb, kT);
  const int64_t tiles = (int64_t)ta * tb * batch;
  int S = (int)std::max<int64_t>(1, (4 * 148 + tiles - 1) / tiles);
  S = std::min(S, std::max(1, rows / 256));
  const int64_t cap = (int64_t)(1u << 30) / (8 * (int64_t)wa * wb * batch);
  S = (int)std::max<int64_t>(1, std::min<int64_t>(S, cap));
  return std::min(S, 256);
}

int64_t gram_part_elems(int batch, int rows, int wa, int wb) {
  return (int64_t)gram_splits(batch, rows, wa, wb) * wa * wb * batch;
}

int launch_gram_tiles(int batch, int rows, int wa, int wb, Mat Xa, Mat Xb, int sym, double* part,
                      double* out, cudaStream_t st) {
  if (batch == 0 || wa == 0 || wb == 0) return ISVD_OK;
  if (sym && wa != wb) {
    set_error("gram: symmetric Gram needs wa == wb");
    return ISVD_EINVAL;
  }
  const int S = gram_splits(batch, rows, wa, wb);
  const int chunk = round_up(std::max(1, ceil_div(rows, S)), kC);
  const int ta = ceil_div(wa, kT), tb = ceil_div(wb, kT);
  const int tiles = sym ? ta * (ta + 1) / 2 : ta * tb;
  gram_tile_kernel<<<dim3(tiles, S, batch), kThreads, 0, st>>>(rows, wa, wb, Xa, Xb, sym, tb, chunk,
                                                              S, part);
  ISVD_LAUNCHED();
  const int64_t total = (int64_t)wa * wb;
  const int gx = (int)std::min<int64_t>((total + 255) / 256, 4096);
  gram_reduce_kernel<<<dim3(gx, batch), 256, 0, st>>>(wa, wb, S, sym, part, out);
  ISVD_LAUNCHED();
  return ISVD_OK;
}

int launch_gemm_tall(int batch, int rows, int n, int wc, Mat X, Mat Q, Mat C, cudaStream_t st) {
  if (batch == 0 || rows == 0 || wc == 0) return ISVD_OK;
  if ((int64_t)ceil_div(rows, kT) > 0x7fffffff) {
    set_error("gemm_tall: too many rows");
    return ISVD_EINVAL;
  }
  gemm_tile_kernel<<<dim3(ceil_div(rows, kT), ceil_div(wc, kT), batch), kThreads, 0, st>>>(
      rows, n, wc, X, Q, C);
  ISVD_LAUNCHED();
  return ISVD_OK;
}

}  // namespace isvd
