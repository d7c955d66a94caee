// K7 -- dense thin SVD on the device (init, refresh, oracle).
//
// Reference semantics: linalg.py:84-109 (np.linalg.svd -> LAPACK gesdd,
// snapped below 1e-12 s0, sign-canonical), used by SvdEngine.__init__
// (engine.py:89), refresh (engine.py:173) and compute_oracle (metrics.py:56-64).
//
// Algorithm: blocked one-sided Jacobi (Hestenes) on the columns of
// X = A (m >= n) or X = A^T (m < n).  Columns are grouped into blocks of 16;
// a round-robin tournament pairs blocks; for each block pair the 32 x 32 Gram
// matrix is formed on the FP64 tensor path (DMMA.8x8x4), diagonalised by a
// parallel two-sided Jacobi in shared memory (same rotation formulas as
// _kernels.pyx:38-44), and the resulting 32 x 32 rotation is applied to the
// 32 long columns and to the accumulated right rotation, again with DMMA.
// Convergence: a sweep in which no block pair's fresh Gram has an
// off-diagonal above tol * sqrt(M_pp M_qq).  sigma = column norms, so the
// result has one-sided-Jacobi (high relative) accuracy.
#include <algorithm>
#include <vector>
#include "common.cuh"
#include "dense_svd.cuh"
#include "metrics.cuh"
#include "../../include/isvd.h"

namespace isvd {

namespace {

constexpr int BW = 16;
constexpr int PW = 2 * BW;
constexpr int kThreads = 256;

__device__ __forceinline__ int tslot(int j, int round, int ne) {
  return j == 0 ? 0 : 1 + (j - 1 + round) % (ne - 1);
}

__global__ void dsvd_prep_kernel(int m, int n, int ldx, int ncp, const double* __restrict__ a,
                                 int64_t a_stride, int lda, double* __restrict__ X,
                                 int64_t x_stride, double* __restrict__ Jm, int64_t j_stride) {
  const int b = blockIdx.y;
  const double* ab = a + b * a_stride;
  double* xb = X + b * x_stride;
  double* jb = Jm + b * j_stride;
  const bool tall = m >= n;
  const int64_t total = (int64_t)ncp * ldx;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int j = (int)(idx / ldx), i = (int)(idx % ldx);
    double v = 0.0;
    if (tall) {
      if (i < m && j < n) v = ab[(int64_t)i * lda + j];
    } else {
      if (j < m && i < n) v = ab[(int64_t)j * lda + i];
    }
    xb[idx] = v;
  }
  const int64_t jt = (int64_t)ncp * ncp;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < jt;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int j = (int)(idx / ncp), i = (int)(idx % ncp);
    jb[idx] = (i == j) ? 1.0 : 0.0;
  }
}

__global__ void __launch_bounds__(kThreads) dsvd_round_kernel(int ldx, int ncp, int nbe, int round,
                                                               double* __restrict__ X,
                                                               int64_t x_stride,
                                                               double* __restrict__ Jm,
                                                               int64_t j_stride, int* flags,
                                                               double tol) {
  __shared__ double M[PW][PW + 1];
  __shared__ double Q[PW][PW + 1];
  __shared__ double rc[PW / 2], rs[PW / 2];
  __shared__ int rp[PW / 2], rq[PW / 2];
  __shared__ int any, rot;
  const int b = blockIdx.y;
  if (flags[b] & 2) return;  // stream already converged
  const int pi = blockIdx.x;
  const int I = tslot(pi, round, nbe), Jb = tslot(nbe - 1 - pi, round, nbe);
  double* xb = X + b * x_stride;
  double* jb = Jm + b * j_stride;
  auto col = [&](int c) { return c < BW ? I * BW + c : Jb * BW + (c - BW); };

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = kThreads / 32;
  const int g = lane >> 2, q = lane & 3;
  for (int idx = tid; idx < PW * (PW + 1); idx += kThreads) {
    (&M[0][0])[idx] = 0.0;
    (&Q[0][0])[idx] = 0.0;
  }
  __syncthreads();

  // ---- Gram of the 32 selected columns (DMMA); four 4-row chunks of loads
  // in flight per warp before their DMMAs
  {
    double acc[10][2];
#pragma unroll
    for (int t = 0; t < 10; ++t) acc[t][0] = acc[t][1] = 0.0;
    const double* cp[4];
#pragma unroll
    for (int cg = 0; cg < 4; ++cg) cp[cg] = xb + (int64_t)col(cg * 8 + g) * ldx + q;
    constexpr int U = 4;
    for (int k0 = warp * 4; k0 < ldx; k0 += nw * 4 * U) {
      double a[U][4];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int kk = k0 + u * nw * 4;
#pragma unroll
        for (int cg = 0; cg < 4; ++cg) a[u][cg] = kk < ldx ? cp[cg][kk] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        int t = 0;
#pragma unroll
        for (int c1 = 0; c1 < 4; ++c1)
#pragma unroll
          for (int c2 = c1; c2 < 4; ++c2) {
            dmma_8x8x4(acc[t][0], acc[t][1], a[u][c1], a[u][c2]);
            ++t;
          }
      }
    }
    // warps add their partial Grams in a fixed order (bit-reproducible runs)
    for (int w = 0; w < nw; ++w) {
      if (warp == w) {
        int t = 0;
#pragma unroll
        for (int c1 = 0; c1 < 4; ++c1)
#pragma unroll
          for (int c2 = c1; c2 < 4; ++c2) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              int row = c1 * 8 + g, cc = c2 * 8 + 2 * q + e;
              M[row][cc] += acc[t][e];
              if (c1 != c2) M[cc][row] += acc[t][e];
            }
            ++t;
          }
      }
      __syncthreads();
    }
  }
  if (tid == 0) any = 0;
  __syncthreads();
  for (int idx = tid; idx < PW * PW; idx += kThreads) {
    int p = idx / PW, qq = idx % PW;
    if (p < qq && fabs(M[p][qq]) > tol * sqrt(M[p][p] * M[qq][qq])) any = 1;
  }
  __syncthreads();
  if (!any) return;
  if (tid == 0) atomicOr(&flags[b], 1);
  for (int i = tid; i < PW; i += kThreads) Q[i][i] = 1.0;
  __syncthreads();

  // ---- parallel two-sided Jacobi on M (symmetric PSD), Q accumulates
  for (int sweep = 0; sweep < 12; ++sweep) {
    if (tid == 0) rot = 0;
    __syncthreads();
    for (int r2 = 0; r2 < PW - 1; ++r2) {
      if (tid < PW / 2) {
        int a0 = tslot(tid, r2, PW), a1 = tslot(PW - 1 - tid, r2, PW);
        int p = min(a0, a1), qq = max(a0, a1);
        double app = M[p][p], aqq = M[qq][qq], apq = M[p][qq];
        double c = 1.0, s = 0.0;
        if (fabs(apq) > tol * sqrt(app * aqq) && apq != 0.0) {
          double zeta = (aqq - app) / (2.0 * apq);
          double t = zeta >= 0.0 ? 1.0 / (zeta + sqrt(1.0 + zeta * zeta))
                                 : -1.0 / (-zeta + sqrt(1.0 + zeta * zeta));
          c = 1.0 / sqrt(1.0 + t * t);
          s = t * c;
          rot = 1;
        }
        rp[tid] = p;
        rq[tid] = qq;
        rc[tid] = c;
        rs[tid] = s;
      }
      __syncthreads();
      // M <- J^T M J and Q <- Q J in one pass: thread (pa, pb) owns the 2 x 2
      // block of rows {p_a, q_a} and columns {p_b, q_b} (the column rotation,
      // then the row rotation: the same arithmetic as two separate passes)
      {
        const int pa = tid >> 4, pb = tid & 15;
        const double ca = rc[pa], sa = rs[pa], cb = rc[pb], sb = rs[pb];
        if (sa != 0.0 || sb != 0.0) {
          const int ra = rp[pa], qa = rq[pa], kb = rp[pb], qb = rq[pb];
          double m00 = M[ra][kb], m01 = M[ra][qb], m10 = M[qa][kb], m11 = M[qa][qb];
          if (sb != 0.0) {
            const double n00 = cb * m00 - sb * m01, n01 = sb * m00 + cb * m01;
            const double n10 = cb * m10 - sb * m11, n11 = sb * m10 + cb * m11;
            m00 = n00; m01 = n01; m10 = n10; m11 = n11;
          }
          if (sa != 0.0) {
            const double n00 = ca * m00 - sa * m10, n10 = sa * m00 + ca * m10;
            const double n01 = ca * m01 - sa * m11, n11 = sa * m01 + ca * m11;
            m00 = n00; m01 = n01; m10 = n10; m11 = n11;
          }
          M[ra][kb] = m00; M[ra][qb] = m01; M[qa][kb] = m10; M[qa][qb] = m11;
        }
      }
      for (int task = tid; task < (PW / 2) * PW; task += kThreads) {
        int pr = task / PW, i = task % PW;
        double s = rs[pr];
        if (s == 0.0) continue;
        double c = rc[pr];
        int p = rp[pr], qq = rq[pr];
        double qp = Q[i][p], qv = Q[i][qq];
        Q[i][p] = c * qp - s * qv;
        Q[i][qq] = s * qp + c * qv;
      }
      __syncthreads();
    }
    // every thread reads the flag before thread 0 clears it for the next
    // sweep (without this barrier a late warp could see the cleared flag,
    // leave the loop alone and desynchronise the CTA)
    const int more = rot;
    __syncthreads();
    if (!more) break;
  }

  // ---- apply X[:, cols] <- X[:, cols] Q and J[:, cols] <- J[:, cols] Q (DMMA)
  double bq[8][4];
#pragma unroll
  for (int kk = 0; kk < 8; ++kk)
#pragma unroll
    for (int nn = 0; nn < 4; ++nn) bq[kk][nn] = Q[kk * 4 + q][nn * 8 + g];
  for (int target = 0; target < 2; ++target) {
    double* T = target == 0 ? xb : jb;
    const int ld = target == 0 ? ldx : ncp;
    // the next 8-row group's operands are loaded before this group's stores
    auto load = [&](double (&a)[8], int r0) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) a[kk] = T[(int64_t)col(kk * 4 + q) * ld + r0 + g];
    };
    double a[8];
    if (warp * 8 < ld) load(a, warp * 8);
    for (int r0 = warp * 8; r0 < ld; r0 += nw * 8) {
      double an[8];
      if (r0 + nw * 8 < ld) load(an, r0 + nw * 8);
#pragma unroll
      for (int nn = 0; nn < 4; ++nn) {
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) dmma_8x8x4(d0, d1, a[kk], bq[kk][nn]);
        T[(int64_t)col(nn * 8 + 2 * q) * ld + r0 + g] = d0;
        T[(int64_t)col(nn * 8 + 2 * q + 1) * ld + r0 + g] = d1;
      }
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) a[kk] = an[kk];
    }
  }
}

__global__ void dsvd_finalize_kernel(int m, int n, int nc, int ldx, int ncp,
                                     const double* __restrict__ X, int64_t x_stride,
                                     const double* __restrict__ Jm, int64_t j_stride, int w, Mat U,
                                     Mat V, double* s_w, int64_t s_w_stride, double* s_all,
                                     int64_t s_all_stride) {
  extern __shared__ double dsm[];
  double* raw = dsm;
  int* order = reinterpret_cast<int*>(dsm + nc);
  const int b = blockIdx.x;
  const double* xb = X + b * x_stride;
  const double* jb = Jm + b * j_stride;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = warp; j < nc; j += nw) {
    const double* c = xb + (int64_t)j * ldx;
    double acc = 0.0;
    for (int i = lane; i < ldx; i += 32) acc = fma(c[i], c[i], acc);
    acc = warp_sum(acc);
    if (lane == 0) raw[j] = sqrt(acc);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < nc; j += blockDim.x) {
    double rj = raw[j];
    int rank = 0;
    for (int i = 0; i < nc; ++i) {
      double ri = raw[i];
      rank += (ri > rj) || (ri == rj && i < j);
    }
    order[rank] = j;
  }
  __syncthreads();
  const double s0 = raw[order[0]];
  auto snapped = [&](int t) {
    double r = raw[order[t]];
    return (s0 > 0.0 && r < kZeroSvRtol * s0) ? 0.0 : r;
  };
  if (s_all)
    for (int t = threadIdx.x; t < nc; t += blockDim.x) s_all[b * s_all_stride + t] = snapped(t);
  if (s_w)
    for (int t = threadIdx.x; t < w; t += blockDim.x) s_w[b * s_w_stride + t] = snapped(t);
  const bool tall = m >= n;
  const int len = tall ? m : n;
  // normalized side (len rows) and rotation side (nc rows)
  double* Nb = tall ? (U.p ? U.p + b * U.stride : nullptr) : (V.p ? V.p + b * V.stride : nullptr);
  const int ldn = tall ? U.ld : V.ld;
  double* Rb = tall ? (V.p ? V.p + b * V.stride : nullptr) : (U.p ? U.p + b * U.stride : nullptr);
  const int ldr = tall ? V.ld : U.ld;
  for (int t = warp; t < w; t += nw) {
    const int j = order[t];
    const double r = raw[j];
    const bool live = snapped(t) > 0.0;
    const double inv = live ? 1.0 / r : 0.0;
    if (Nb) {
      const double* c = xb + (int64_t)j * ldx;
      for (int i = lane; i < len; i += 32) Nb[(int64_t)i * ldn + t] = live ? c[i] * inv : 0.0;
    }
    if (Rb) {
      const double* c = jb + (int64_t)j * ncp;
      for (int i = lane; i < nc; i += 32) Rb[(int64_t)i * ldr + t] = c[i];
    }
  }
}

// ---- orthonormality polish of the normalised side (one CholeskyQR step):
// Jacobi leaves the live columns orthogonal to ~tol; U <- U R^{-1} with
// U^T U = R^T R restores orthonormality to rounding while moving each
// vector by O(tol) only.  Dead (zero) columns are completed afterwards.
__global__ void polish_chol_kernel(int w, double* __restrict__ G, const double* __restrict__ s,
                                   int64_t s_stride, int* __restrict__ live) {
  const int b = blockIdx.x;
  double* g = G + (int64_t)b * w * w;
  const double* sb = s + b * s_stride;
  __shared__ int wl;
  if (threadIdx.x == 0) {
    int c = 0;
    while (c < w && sb[c] > 0.0) ++c;
    wl = c;
  }
  __syncthreads();
  const int L = wl;
  for (int k = 0; k < L; ++k) {
    if (threadIdx.x == 0) g[k * w + k] = sqrt(fmax(g[k * w + k], 1e-300));
    __syncthreads();
    const double d = g[k * w + k];
    for (int j = k + 1 + threadIdx.x; j < L; j += blockDim.x) g[k * w + j] /= d;
    __syncthreads();
    const int rem = L - k - 1;
    for (int idx = threadIdx.x; idx < rem * rem; idx += blockDim.x) {
      const int i = k + 1 + idx / rem, j = k + 1 + idx % rem;
      if (j >= i) g[i * w + j] -= g[k * w + i] * g[k * w + j];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) live[b] = L;
}

__global__ void polish_trsm_kernel(int rows, int w, Mat X, const double* __restrict__ G,
                                   const int* __restrict__ live) {
  const int b = blockIdx.y;
  const int L = live[b];
  const double* R = G + (int64_t)b * w * w;
  double* xb = X.p + b * X.stride;
  for (int row = blockIdx.x * blockDim.x + threadIdx.x; row < rows; row += gridDim.x * blockDim.x) {
    double* xr = xb + (int64_t)row * X.ld;
    for (int j = 0; j < L; ++j) {
      double acc = xr[j];
      for (int i = 0; i < j; ++i) acc -= xr[i] * R[i * w + j];
      xr[j] = acc / R[j * w + j];
    }
  }
}

}  // namespace

DenseSvdPlan dense_svd_plan(int m, int n, int w) {
  DenseSvdPlan p;
  p.m = m;
  p.n = n;
  p.nc = std::min(m, n);
  p.len = std::max(m, n);
  int nb = ceil_div(p.nc, BW);
  if (nb % 2) ++nb;
  p.nb = nb;
  p.ncp = nb * BW;
  p.ldx = round_up(p.len, 8);
  if (use_gram_path(m, n, w)) p.ldx = p.ncp = 1;  // gram_svd_run allocates its own
  return p;
}

int dense_svd_run(int batch, int m, int n, const double* a, int64_t a_stride, int lda, int w,
                  Mat u, Mat v, double* s_w, int64_t s_w_stride, double* s_all,
                  int64_t s_all_stride, double* x, double* jac, int* flags, int* flags_host,
                  cudaStream_t st, int* sweeps_out) {
  if (batch == 0) return ISVD_OK;
  if (use_gram_path(m, n, w)) {
    for (int b = 0; b < batch; ++b) {
      Mat ub{u.p ? u.p + b * u.stride : nullptr, u.stride, u.ld};
      Mat vb{v.p ? v.p + b * v.stride : nullptr, v.stride, v.ld};
      if (!ub.p || !vb.p || !s_w) {
        set_error("dense_svd: the Gram path needs U, V and s outputs");
        return ISVD_EINVAL;
      }
      ISVD_TRY(gram_svd_run(m, n, a + b * a_stride, lda, w, ub, vb, s_w + b * s_w_stride,
                            s_all ? s_all + b * s_all_stride : nullptr, st));
    }
    if (sweeps_out) *sweeps_out = 0;
    return ISVD_OK;
  }
  DenseSvdPlan P = dense_svd_plan(m, n, w);
  const int64_t xs = P.x_elems(), js = P.j_elems();
  {
    int64_t total = std::max(xs, js);
    int gx = (int)std::min<int64_t>((total + 255) / 256, 2048);
    dsvd_prep_kernel<<<dim3(gx, batch), 256, 0, st>>>(m, n, P.ldx, P.ncp, a, a_stride, lda, x, xs,
                                                      jac, js);
    ISVD_LAUNCHED();
  }
  ISVD_CUDA(cudaMemsetAsync(flags, 0, sizeof(int) * batch, st));
  const double eps = 2.220446049250313e-16;
  // Stop when every block-pair Gram has |M_pq| <= tol sqrt(M_pp M_qq): sigma is then
  // accurate to O(tol^2) relative and the vectors to O(tol / relative gap).  1e-12
  // also stays above the rounding floor of the Gram-based inner rotations
  // (eps sqrt(M_pp / M_qq) for strongly graded pairs), so the sweep count stays low.
  const double tol = std::max(1e-12, 16.0 * std::sqrt((double)P.len) * eps);
  std::vector<int> fl(batch, 0);
  int sweep = 0;
  const int kMaxOuter = 40;
  for (; sweep < kMaxOuter; ++sweep) {
    for (int round = 0; round < P.nb - 1; ++round) {
      dsvd_round_kernel<<<dim3(P.nb / 2, batch), kThreads, 0, st>>>(P.ldx, P.ncp, P.nb, round, x,
                                                                    xs, jac, js, flags, tol);
      ISVD_LAUNCHED();
    }
    ISVD_CUDA(cudaMemcpyAsync(flags_host, flags, sizeof(int) * batch, cudaMemcpyDeviceToHost, st));
    ISVD_CUDA(cudaStreamSynchronize(st));
    bool all_done = true;
    for (int b = 0; b < batch; ++b) {
      int f = flags_host[b];
      if (f & 2) continue;
      if (f & 1)
        all_done = false, f = 0;
      else
        f = 2;
      flags_host[b] = f;
    }
    if (all_done) break;
    ISVD_CUDA(cudaMemcpyAsync(flags, flags_host, sizeof(int) * batch, cudaMemcpyHostToDevice, st));
  }
  if (sweeps_out) *sweeps_out = sweep + 1;
  {
    size_t smem = sizeof(double) * P.nc + sizeof(int) * P.nc;
    static bool attr = false;
    if (!attr) {
      ISVD_CUDA(cudaFuncSetAttribute(dsvd_finalize_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      attr = true;
    }
    if (smem > 200 * 1024) {
      set_error("dense_svd: min(m, n) too large for the finalize kernel");
      return ISVD_EINVAL;
    }
    dsvd_finalize_kernel<<<batch, 256, smem, st>>>(m, n, P.nc, P.ldx, P.ncp, x, xs, jac, js, w, u,
                                                   v, s_w, s_w_stride, s_all, s_all_stride);
    ISVD_LAUNCHED();
  }
  // orthonormality polish of the normalised side (U if m >= n, else V)
  const bool tall = m >= n;
  Mat ns = tall ? u : v;
  const int rows = tall ? m : n;
  if (ns.p && s_w && w > 0 && w <= 160) {
    double *part = nullptr, *G = nullptr;
    int* live = nullptr;
    const size_t np = (size_t)gram_part_elems(batch, rows, w, w);
    ISVD_CUDA(cudaMallocAsync((void**)&part, sizeof(double) * np, st));
    ISVD_CUDA(cudaMallocAsync((void**)&G, sizeof(double) * batch * w * w, st));
    ISVD_CUDA(cudaMallocAsync((void**)&live, sizeof(int) * batch, st));
    int rc = launch_gram(batch, rows, w, w, ns, ns, part, G, st);
    if (rc == ISVD_OK) {
      polish_chol_kernel<<<batch, 256, 0, st>>>(w, G, s_w, s_w_stride, live);
      ISVD_LAUNCHED();
      const int gx = std::min(ceil_div(rows, 128), 1024);
      polish_trsm_kernel<<<dim3(gx, batch), 128, 0, st>>>(rows, w, ns, G, live);
      ISVD_LAUNCHED();
    }
    cudaFreeAsync(part, st);
    cudaFreeAsync(G, st);
    cudaFreeAsync(live, st);
    if (rc != ISVD_OK) return rc;
  }
  return ISVD_OK;
}

}  // namespace isvd
