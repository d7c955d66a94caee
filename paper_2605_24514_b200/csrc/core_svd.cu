// K2 -- batched one-sided Jacobi SVD of the small Brand core.
//
// Semantics follow the reference's compiled backend, _kernels.pyx:22-109:
//   * one-sided Jacobi on the columns of G = K, accumulating V;
//     a pair (p, q) is rotated iff |a_pq| > 1e-14 sqrt(a_pp a_qq), the
//     rotation angle uses the same zeta/t/c/s formulas (:29-57);
//   * sigma_raw = column norms of G, stable descending sort (:94-97);
//   * snap sigma < 1e-12 sigma_0 to exactly 0 (:98-101);
//   * U[:, live] = G / sigma_raw; dead columns completed over e_0, e_1, ...
//     (_complete_basis, :62-79).
// The sweep uses a parallel (round-robin tournament) pair ordering instead of
// the cyclic-by-rows order, so rounding differs from the Cython kernel at the
// 1e-15 level -- the same kind of difference the reference's LAPACK backend
// already has.
//
// Layout: one CTA per core.  G and V live in shared memory, column-major with
// an odd pitch (bank-conflict-free column walks).  Each warp owns a pair per
// round; lanes stride over rows; three warp-shuffle reductions give
// a_pp, a_qq, a_pq.  For s > kSmemMaxS, V is kept in a global scratch.
#include "common.cuh"
#include "core_svd.cuh"
#include "../../include/isvd.h"

namespace isvd {

namespace {

__device__ __forceinline__ int tour_slot(int j, int round, int ne) {
  // circle method: slot 0 fixed, slots 1..ne-1 rotate by `round`.
  return j == 0 ? 0 : 1 + (j - 1 + round) % (ne - 1);
}

__global__ void jacobi_core_kernel(int s, const double* __restrict__ core, int64_t core_stride,
                                   int ldcore, double* __restrict__ uk, double* __restrict__ vk,
                                   int64_t out_stride, int ldo, double* __restrict__ sv,
                                   int64_t sv_stride, double* __restrict__ vscratch,
                                   const int* __restrict__ active) {
  extern __shared__ double smem[];
  const int b = blockIdx.x;
  if (active && !active[b]) return;
  const int ps = s | 1;
  double* G = smem;
  double* V = vscratch ? vscratch + (int64_t)b * s * ps : smem + s * ps;
  __shared__ int rotated;
  __shared__ double raw[kCoreMaxS];
  __shared__ int order[kCoreMaxS];

  const double* K = core + b * core_stride;
  for (int idx = threadIdx.x; idx < s * s; idx += blockDim.x) {
    int i = idx / s, j = idx % s;
    G[j * ps + i] = K[i * ldcore + j];
    V[j * ps + i] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int ne = s + (s & 1);
  const int npairs = ne / 2;
  for (int sweep = 0; sweep < kMaxSweeps; ++sweep) {
    if (threadIdx.x == 0) rotated = 0;
    __syncthreads();
    for (int round = 0; round < ne - 1; ++round) {
      for (int k = warp; k < npairs; k += nw) {
        int a = tour_slot(k, round, ne), c = tour_slot(ne - 1 - k, round, ne);
        int p = min(a, c), q = max(a, c);
        if (q >= s) continue;
        double* gp = G + p * ps;
        double* gq = G + q * ps;
        double app = 0, aqq = 0, apq = 0;
        for (int i = lane; i < s; i += 32) {
          double x = gp[i], y = gq[i];
          app = fma(x, x, app);
          aqq = fma(y, y, aqq);
          apq = fma(x, y, apq);
        }
        app = warp_sum(app);
        aqq = warp_sum(aqq);
        apq = warp_sum(apq);
        if (fabs(apq) <= kOrthoEps * sqrt(app * aqq)) continue;
        double zeta = (aqq - app) / (2.0 * apq);
        double t = zeta >= 0.0 ? 1.0 / (zeta + sqrt(1.0 + zeta * zeta))
                               : -1.0 / (-zeta + sqrt(1.0 + zeta * zeta));
        double cs = 1.0 / sqrt(1.0 + t * t);
        double sn = t * cs;
        for (int i = lane; i < s; i += 32) {
          double x = gp[i], y = gq[i];
          gp[i] = cs * x - sn * y;
          gq[i] = sn * x + cs * y;
        }
        double* vp = V + p * ps;
        double* vq = V + q * ps;
        for (int i = lane; i < s; i += 32) {
          double x = vp[i], y = vq[i];
          vp[i] = cs * x - sn * y;
          vq[i] = sn * x + cs * y;
        }
        if (lane == 0) rotated = 1;
      }
      __syncthreads();
    }
    if (!rotated) break;
    __syncthreads();
  }

  // column norms
  for (int j = warp; j < s; j += nw) {
    double acc = 0;
    for (int i = lane; i < s; i += 32) acc = fma(G[j * ps + i], G[j * ps + i], acc);
    acc = warp_sum(acc);
    if (lane == 0) raw[j] = sqrt(acc);
  }
  __syncthreads();
  // stable descending order: rank(j) = #{i : raw_i > raw_j} + #{i < j : raw_i == raw_j}
  for (int j = threadIdx.x; j < s; j += blockDim.x) {
    double rj = raw[j];
    int rank = 0;
    for (int i = 0; i < s; ++i) {
      double ri = raw[i];
      rank += (ri > rj) || (ri == rj && i < j);
    }
    order[rank] = j;
  }
  __syncthreads();
  const double s0 = raw[order[0]];
  double* U = uk + b * out_stride;
  double* W = vk + b * out_stride;
  double* S = sv + b * sv_stride;
  for (int idx = threadIdx.x; idx < s * s; idx += blockDim.x) {
    int i = idx / s, t = idx % s;
    int j = order[t];
    double r = raw[j];
    bool live = !(s0 > 0.0 && r < kZeroSvRtol * s0) && r > 0.0;
    U[i * ldo + t] = live ? G[j * ps + i] / r : 0.0;
    W[i * ldo + t] = V[j * ps + i];
  }
  for (int t = threadIdx.x; t < s; t += blockDim.x) {
    double r = raw[order[t]];
    bool snapped = s0 > 0.0 && r < kZeroSvRtol * s0;
    S[t] = snapped ? 0.0 : r;
  }
  __syncthreads();
  // dead-column completion (_kernels.pyx:62-79): rare; one warp, in order.
  if (warp == 0) {
    for (int t = 0; t < s; ++t) {
      double r = raw[order[t]];
      bool live = !(s0 > 0.0 && r < kZeroSvRtol * s0) && r > 0.0;
      if (live) continue;
      bool done = false;
      for (int axis = 0; axis < s && !done; ++axis) {
        // cand = e_axis - sum_{c != t} U[:, c] U[axis, c]
        double nrm2 = 0;
        for (int i = lane; i < s; i += 32) {
          double v = (i == axis) ? 1.0 : 0.0;
          for (int c = 0; c < s; ++c)
            if (c != t) v -= U[i * ldo + c] * U[axis * ldo + c];
          nrm2 = fma(v, v, nrm2);
        }
        nrm2 = warp_sum(nrm2);
        double nrm = sqrt(nrm2);
        if (nrm > 0.5) {
          // recompute and store (all lanes read U[axis, c] before any write
          // to column t; column t itself is excluded from the sum)
          double vals[(kCoreMaxS + 31) / 32];
          int cnt = 0;
          for (int i = lane; i < s; i += 32) {
            double v = (i == axis) ? 1.0 : 0.0;
            for (int c = 0; c < s; ++c)
              if (c != t) v -= U[i * ldo + c] * U[axis * ldo + c];
            vals[cnt++] = v / nrm;
          }
          __syncwarp();
          cnt = 0;
          for (int i = lane; i < s; i += 32) U[i * ldo + t] = vals[cnt++];
          __syncwarp();
          done = true;
        }
      }
    }
  }
}

}  // namespace

size_t core_svd_smem_bytes(int s, bool v_in_smem) {
  int ps = s | 1;
  return sizeof(double) * (size_t)s * ps * (v_in_smem ? 2 : 1);
}

int launch_core_svd(int batch, int s, const double* core, int64_t core_stride, int ldcore,
                    double* uk, double* vk, int64_t out_stride, int ldo, double* sv,
                    int64_t sv_stride, double* vscratch, const int* active, cudaStream_t st) {
  if (s < 1 || s > kCoreMaxS) {
    set_error("core size out of range (1.." + std::to_string(kCoreMaxS) + ")");
    return ISVD_EINVAL;
  }
  if (batch == 0) return ISVD_OK;
  bool v_in_smem = s <= kSmemMaxS;
  if (!v_in_smem && !vscratch) {
    set_error("core_svd: s > smem limit needs a V scratch buffer");
    return ISVD_EINVAL;
  }
  size_t smem = core_svd_smem_bytes(s, v_in_smem);
  static bool attr_set = false;
  if (!attr_set) {
    ISVD_CUDA(cudaFuncSetAttribute(jacobi_core_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   200 * 1024));
    attr_set = true;
  }
  int ne = s + (s & 1);
  int warps = ne / 2;
  if (warps > 16) warps = 16;
  if (warps < 1) warps = 1;
  jacobi_core_kernel<<<batch, 32 * warps, smem, st>>>(
      s, core, core_stride, ldcore, uk, vk, out_stride, ldo, sv, sv_stride,
      v_in_smem ? nullptr : vscratch, active);
  ISVD_LAUNCHED();
  return ISVD_OK;
}

}  // namespace isvd
