// One-warp basis rotations and zero-sigma completion for the fused tick
// epilogues (core kernels that already hold the core's Uk / Vk on chip).
//
// warp_rotate: X[0:rows, :] <- X[0:rows, 0:r] . Q[0:r, 0:keep] in place on
// the FP64 tensor path (DMMA.8x8x4, eight row groups of 8 at a time per
// warp), Q read through a functor q(k, n); columns >= keep come out 0.  With
// new_row, row `rows` becomes scale * Q[r, 0:keep] (the row-append form
// [X 0; 0 1] Q, _kernels.pyx:168-175).  r, keep <= 32.
//
// warp_complete_zero: engine.py:33-70 (_install) for one stream, one warp:
// columns of zero singular value whose norm is not 1 are replaced by the
// orthonormal completion (existing direction projected off the others, then
// e_0, e_1, ...), on both sides; with a deferred right basis V is
// materialised first (tick.cu vdefer_materialise, warp form).
#pragma once
#include "common.cuh"
#include "tick.cuh"

namespace isvd {

template <class QF>
__device__ __forceinline__ void warp_rotate(double* X, int ld, int rows, int r, int keep, QF q,
                                            bool new_row, double scale) {
  const int lane = threadIdx.x & 31, g = lane >> 2, qd = lane & 3;
  double bq[8][4];
#pragma unroll
  for (int kk = 0; kk < 8; ++kk)
#pragma unroll
    for (int nn = 0; nn < 4; ++nn) {
      const int k = kk * 4 + qd, n = nn * 8 + g;
      bq[kk][nn] = (k < r && n < keep) ? q(k, n) : 0.0;
    }
  // the next row group's operands are loaded before this group's results
  // are stored (the stores may alias the loads as far as the compiler
  // knows, which would otherwise serialise one memory latency per group)
  auto load_a = [&](double (&a)[8], int row0) {
    const int row = row0 + g;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const int k = kk * 4 + qd;
      a[kk] = (row < rows && k < r) ? X[(int64_t)row * ld + k] : 0.0;
    }
  };
  double a[8];
  load_a(a, 0);
  for (int row0 = 0; row0 < rows; row0 += 8) {
    const int row = row0 + g;
    double an[8];
    if (row0 + 8 < rows) load_a(an, row0 + 8);
    double d[4][2];
#pragma unroll
    for (int nn = 0; nn < 4; ++nn) d[nn][0] = d[nn][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk)
#pragma unroll
      for (int nn = 0; nn < 4; ++nn) dmma_8x8x4(d[nn][0], d[nn][1], a[kk], bq[kk][nn]);
    if (row < rows) {
#pragma unroll
      for (int nn = 0; nn < 4; ++nn) {
        const int c0 = nn * 8 + 2 * qd;
        if (c0 < ld) *reinterpret_cast<double2*>(X + (int64_t)row * ld + c0) = make_double2(d[nn][0], d[nn][1]);
      }
    }
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) a[kk] = an[kk];
  }
  if (new_row)
    for (int c = lane; c < ld; c += 32) X[(int64_t)rows * ld + c] = c < keep ? scale * q(r, c) : 0.0;
}

// one warp, one stream: X (rows x ld) column t completed against columns != t
__device__ inline void warp_complete_column(double* X, int64_t ld, int rows, int w, int t,
                                            double* coef) {
  const int lane = threadIdx.x & 31;
  for (int c = 0; c < w; ++c) {
    double acc = 0.0;
    if (c != t)
      for (int i = lane; i < rows; i += 32) acc = fma(X[i * ld + c], X[i * ld + t], acc);
    acc = warp_sum(acc);
    if (lane == 0) coef[c] = (c != t) ? acc : 0.0;
  }
  __syncwarp();
  double nn = 0.0;
  for (int i = lane; i < rows; i += 32) {
    double v = X[i * ld + t];
    for (int c = 0; c < w; ++c)
      if (c != t) v -= X[i * ld + c] * coef[c];
    nn = fma(v, v, nn);
  }
  const double nrm = sqrt(warp_sum(nn));
  if (nrm > 0.5) {
    for (int i = lane; i < rows; i += 32) {
      double v = X[i * ld + t];
      for (int c = 0; c < w; ++c)
        if (c != t) v -= X[i * ld + c] * coef[c];
      X[i * ld + t] = v / nrm;
    }
    __syncwarp();
    return;
  }
  for (int axis = 0; axis < rows; ++axis) {
    double cn = 0.0;
    for (int i = lane; i < rows; i += 32) {
      double v = (i == axis) ? 1.0 : 0.0;
      for (int c = 0; c < w; ++c)
        if (c != t) v -= X[i * ld + c] * X[axis * ld + c];
      cn = fma(v, v, cn);
    }
    const double cnrm = sqrt(warp_sum(cn));
    if (cnrm > 0.5) {
      if (lane < w) coef[lane] = X[axis * ld + lane];
      __syncwarp();
      for (int i = lane; i < rows; i += 32) {
        double v = (i == axis) ? 1.0 : 0.0;
        for (int c = 0; c < w; ++c)
          if (c != t) v -= X[i * ld + c] * coef[c];
        X[i * ld + t] = v / cnrm;
      }
      __syncwarp();
      return;
    }
  }
}

// the per-stream engine completion (complete_zero_stream) with one warp;
// U, V, vd already offset to this stream (vd.G / vd.Z per-stream pointers)
__device__ inline void warp_complete_zero(int w, const double* sb, Mat U, int m, Mat V, int n,
                                          VDefer vd, double* coef) {
  const int lane = threadIdx.x & 31;
  bool any_zero = false;
  for (int t = lane; t < w; t += 32) any_zero |= sb[t] == 0.0;
  if (!__any_sync(0xffffffffu, any_zero)) return;
  if (vd.G) {
    // V <- [V(:, :fw) | Z^T] G, G <- [I; 0] (lane = output column)
    double* Gb = const_cast<double*>(vd.G);
    for (int c = 0; c < n; ++c) {
      double* vr = V.p + (int64_t)c * V.ld;
      double acc = 0.0;
      if (lane < w) {
        for (int l = 0; l < vd.fw; ++l) acc = fma(vr[l], Gb[l * vd.ldg + lane], acc);
        for (int t = 0; t < vd.nz; ++t)
          acc = fma(vd.Z[(int64_t)t * vd.ldz + c], Gb[(vd.fw + t) * vd.ldg + lane], acc);
      }
      __syncwarp();
      if (lane < vd.fw || lane < w) vr[lane] = lane < w ? acc : 0.0;
      __syncwarp();
    }
    for (int idx = lane; idx < (vd.fw + vd.nz) * w; idx += 32) {
      const int l = idx / w, q = idx % w;
      Gb[l * vd.ldg + q] = (l == q) ? 1.0 : 0.0;
    }
    __syncwarp();
  }
  for (int t = 0; t < w; ++t) {
    if (sb[t] != 0.0) continue;
    for (int side = 0; side < 2; ++side) {
      double* X = side == 0 ? U.p : V.p;
      const int64_t ld = side == 0 ? U.ld : V.ld;
      const int rows = side == 0 ? m : n;
      double nn = 0.0;
      for (int i = lane; i < rows; i += 32) nn = fma(X[i * ld + t], X[i * ld + t], nn);
      if (fabs(warp_sum(nn) - 1.0) > 1e-6) warp_complete_column(X, ld, rows, w, t, coef);
    }
  }
}

}  // namespace isvd
