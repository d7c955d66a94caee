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
#include <algorithm>
#include <vector>
#include <cstdlib>
#include "common.cuh"
#include "core_svd.cuh"
#include "tick.cuh"
#include "warp_rot.cuh"
#include "../../include/isvd.h"

namespace isvd {

// profiling counters: [0] jacobi32 sweeps, [1] jacobi32 cores (isvd_debug_counters)
__device__ unsigned long long g_debug_counters[8];
// rank-1 core phase timestamps (ISVD_R1_TRACE builds): [core][phase]
__device__ long long g_r1_trace[4096][10];
#ifdef ISVD_R1_TRACE
#define R1_MARK(k)                                                   \
  do {                                                               \
    if (threadIdx.x == 0 && b < 4096) g_r1_trace[b][k] = clock64();  \
  } while (0)
#else
#define R1_MARK(k) \
  do {             \
  } while (0)
#endif

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

// ---------------------------------------------------------------------------
// Warp-per-core variant for s <= 32 (the rank-1 core of a k <= 32 stream).
// Ordering: odd-even transposition -- rounds alternate pairs (2k, 2k+1) and
// (2k+1, 2k+2) and every rotated pair swaps places, so each pair of columns
// meets exactly once per sweep of 32 rounds and all register indices are
// compile-time; after a sweep the column order is reversed (tracked for the
// stable sort).  Rotation formulas and threshold as _kernels.pyx:38-57.  V
// is rotated once per sweep from a shared-memory (c, s) log (row layout).
constexpr int kJ32Warps = 4;
// Rank-1 sweep exit: once every rotation of a sweep had |a_pq| <= kConvRel
// sqrt(a_pp a_qq), the off-diagonal left is O(kConvRel^2) relative (cyclic
// Jacobi converges quadratically) and one first-order simultaneous step
// (j32_step) takes it below the reference's 1e-14 stop; Brand rank-1
// cores diag(s) + delta a b^T start with off-diagonals ~1e-5 relative, so
// one sweep suffices.  Generic cores (functional core_svd, angles, guard)
// sweep until a sweep makes no rotation, as _kernels.pyx:38-59.
constexpr double kConvRel = 1e-6;

// 1/sqrt(x) to ~1 ulp: MUFU.RSQ64H seed + two Newton steps (x > 0, normal)
__device__ __forceinline__ double j32_rsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  return y * fma(-hx * y, y, 1.5);
}

// 1/x to ~1e-12 relative (seed + one Newton step): enough for a rotation
// angle that only has to be right to first order
__device__ __forceinline__ double j32_rcp1(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return fma(r, fma(-x, r, 1.0), r);
}

__device__ __forceinline__ double j32_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// Replays the logged rotations of one sweep (32 rounds) on a row of V.
__device__ __forceinline__ void j32_apply_v(double (&v)[32], const double2* log) {
  for (int rr = 0; rr < 16; ++rr) {
    const double2* ev = log + (2 * rr) * 16;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const double2 r = ev[k];
      const double vp = v[2 * k], vq = v[2 * k + 1];
      v[2 * k] = r.y * vp + r.x * vq;
      v[2 * k + 1] = r.x * vp - r.y * vq;
    }
    const double2* od = log + (2 * rr + 1) * 16;
#pragma unroll
    for (int k = 0; k < 15; ++k) {
      const double2 r = od[k];
      const double vp = v[2 * k + 1], vq = v[2 * k + 2];
      v[2 * k + 1] = r.y * vp + r.x * vq;
      v[2 * k + 2] = r.x * vp - r.y * vq;
    }
  }
}

// Simultaneous Jacobi step on the FP64 tensor path.  With the Gram
// M = G^T G of the current columns, the rotation each pair (p, q) would get
// is, to first order, theta_pq = M_pq / (M_qq - M_pp); all of them are
// applied at once, G <- G J with Theta skew and
//   J = I + Theta + Theta^2 / 2   (J^T J = I + Theta^4 / 4), or
//   J = I + Theta                 when every |theta| <= 1e-8 (J^T J = I - Theta^2,
//                                 below rounding),
// which leaves off-diagonals O(theta^2) (quadratic convergence while the
// columns' norms are well separated).  Products on DMMA.8x8x4: 80 for the
// upper half of M, 128 for Theta^2, 128 for G (J - I); theta is formed in
// the accumulator layout, so shared memory carries only the staged G (gs,
// XOR-swizzled rows) and -- once the step is known to apply -- Theta,
// J - I and G (J - I) between layouts (ws).  Uses:
//  * the finishing step after one Jacobi sweep of small rotations (cap
//    1e-7): the sweep leaves O(1e-12) relative off-diagonals, the reference
//    stops at 1e-14 (_kernels.pyx:38-57: one more sweep of tiny rotations
//    and a check sweep);
//  * the whole factorisation of a well-conditioned Brand rank-1 core (cap
//    1e-4): off-diagonals ~1e-7 relative reach the stop in two steps, with
//    no dependent chain of 32 rotation rounds.
// Returns 0 if G already meets the reference's stop (|M_pq| <= 1e-14
// sqrt(M_pp M_qq) for every pair: G unchanged); 1 after a step; 2 after a
// step with every |theta| <= 1e-8, which leaves O(1e-16) off-diagonals (past
// the stop without another Gram); -1 (G and ws unchanged) if some |theta|
// exceeds tcap (nearly equal columns).
__device__ __forceinline__ int j32_step(double (&x)[32], double* gs, double* ws, double* dg,
                                        int lane, double null2, double tcap) {
  auto T = [&](double* t, int i, int j) -> double& { return t[i * 32 + (j ^ ((i & 1) << 3))]; };
  const int g = lane >> 2, qd = lane & 3;
  double n4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    T(gs, i, lane) = x[i];
    n4[i & 3] = fma(x[i], x[i], n4[i & 3]);
  }
  dg[lane] = (n4[0] + n4[1]) + (n4[2] + n4[3]);
  __syncwarp();
  // M tile (mi, ni), mi <= ni: A = G^T rows 8mi.., B = G columns 8ni..; both
  // fragments are G(4kk + qd, 8t + g).  acc -> theta in place.
  double th[10][2];
#pragma unroll
  for (int t = 0; t < 10; ++t) th[t][0] = th[t][1] = 0.0;
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    double f[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) f[t] = T(gs, 4 * kk + qd, 8 * t + g);
    int idx = 0;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = mi; ni < 4; ++ni, ++idx) dmma_8x8x4(th[idx][0], th[idx][1], f[mi], f[ni]);
  }
  bool viol = false;
  double tmax = 0.0;
  {
    int idx = 0;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = mi; ni < 4; ++ni, ++idx)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = 8 * mi + g, c = 8 * ni + 2 * qd + e;
          const double dr = dg[r], dc = dg[c], mrc = th[idx][e];
          const bool live = r != c && dr > null2 && dc > null2;
          viol |= live && mrc * mrc > (kOrthoEps * kOrthoEps) * (dr * dc);
          const double t = live ? mrc * j32_rcp1(dc - dr) : 0.0;  // theta_rc
          tmax = fmax(tmax, (t - t == 0.0) ? fabs(t) : 1e300);  // inf / NaN: fail
          th[idx][e] = t;
        }
  }
  if (!__any_sync(0xffffffffu, viol)) return 0;
  const double tm = warp_max(tmax);
  if (tm > tcap) return -1;
  // |theta| <= 1e-8: the Theta^2 term is below rounding and the step
  // leaves O(theta^2) <= 1e-16 relative off-diagonals -- past the stop
  // without another Gram (returns 2)
  const bool second = tm > 1e-8;
  {
    int idx = 0;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = mi; ni < 4; ++ni, ++idx) {
        const int r = 8 * mi + g, c = 8 * ni + 2 * qd;
        *reinterpret_cast<double2*>(&T(ws, r, c)) = make_double2(th[idx][0], th[idx][1]);
        if (mi != ni) {  // theta is skew
          T(ws, c, r) = -th[idx][0];
          T(ws, c + 1, r) = -th[idx][1];
        }
      }
  }
  __syncwarp();
  double d[4][4][2];
  if (second) {
    // ws <- Theta + Theta^2 / 2 (tile-wise in the accumulator layout)
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) d[mi][ni][0] = d[mi][ni][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        a[t] = T(ws, 8 * t + g, 4 * kk + qd);
        b[t] = T(ws, 4 * kk + qd, 8 * t + g);
      }
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma_8x8x4(d[mi][ni][0], d[mi][ni][1], a[mi], b[ni]);
    }
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        const double2 t2 = *reinterpret_cast<const double2*>(&T(ws, 8 * mi + g, 8 * ni + 2 * qd));
        d[mi][ni][0] = fma(0.5, d[mi][ni][0], t2.x);
        d[mi][ni][1] = fma(0.5, d[mi][ni][1], t2.y);
      }
    __syncwarp();  // every lane has read Theta
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
        *reinterpret_cast<double2*>(&T(ws, 8 * mi + g, 8 * ni + 2 * qd)) =
            make_double2(d[mi][ni][0], d[mi][ni][1]);
    __syncwarp();
  }
  // G (J - I): A = G rows 8mi.. (G(8mi + g, 4kk + qd)), B = (J - I) rows 4kk..
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) d[mi][ni][0] = d[mi][ni][1] = 0.0;
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    double a[4], b[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      a[t] = T(gs, 8 * t + g, 4 * kk + qd);
      b[t] = T(ws, 4 * kk + qd, 8 * t + g);
    }
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) dmma_8x8x4(d[mi][ni][0], d[mi][ni][1], a[mi], b[ni]);
  }
  __syncwarp();  // every lane has read J - I
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
      *reinterpret_cast<double2*>(&T(ws, 8 * mi + g, 8 * ni + 2 * qd)) =
          make_double2(d[mi][ni][0], d[mi][ni][1]);
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = T(gs, i, lane) + T(ws, i, lane);
  __syncwarp();
  return second ? 1 : 2;
}

// Per-warp shared state: the (c, s) log of one sweep (32 rounds x 16 pairs)
// and V (32 x 33).  V is kept out of registers while the G rounds run (so
// the G phase needs ~half the registers and more cores fit per SM) and is
// rotated once per sweep by replaying the log.
struct J32Smem {
  double2 log[32 * 16];  // also the 32 x 32 (XOR-swizzled) staging tile of G for the U output
  double V[32][33];
  double nrm[32];
  double inv[32];
  int pos[32];
  int ipos[32];
};

// ---------------------------------------------------------------------------
// Column layout: lane l holds the column at position l (32 doubles in
// registers).  A round's two lanes of a pair exchange their columns with 32
// register shuffles and both compute a_pq = <g_p, g_q> with the same
// operands in the same order (bit-identical on both lanes), so no
// cross-lane reduction tree and no selects sit on the round's critical path
// (a row layout -- lane = row, pair Grams reduce-scattered across the warp --
// needed ~30% more instructions per core).
template <bool ODD>
__device__ __forceinline__ void j32c_round(double (&x)[32], int lane, double2* cs_log, double& nrm,
                                           bool& any, float& relmax, double null2) {
  // even rounds pair positions (2k, 2k+1); odd rounds (2k+1, 2k+2), 0 and 31 idle
  const int partner = ODD ? ((lane & 1) ? lane + 1 : lane - 1) : (lane ^ 1);
  const bool idle = ODD && (lane == 0 || lane == 31);
  const int src = idle ? lane : partner;
  const bool lower = lane < partner;
  double y[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) y[i] = __shfl_sync(0xffffffffu, x[i], src);
  const double pn = __shfl_sync(0xffffffffu, nrm, src);
  // fma(x, y, .) == fma(y, x, .): both lanes get the same a_pq bit for bit
  double d4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int i = 0; i < 32; ++i) d4[i & 3] = fma(x[i], y[i], d4[i & 3]);
  const double apq = (d4[0] + d4[1]) + (d4[2] + d4[3]);
  const double app = lower ? nrm : pn, aqq = lower ? pn : nrm;
  double c = 1.0, sn = 0.0, t = 0.0;
  const double apq2 = apq * apq, pq = app * aqq;
  const bool rot = !idle && apq2 > (kOrthoEps * kOrthoEps) * pq && fmin(app, aqq) > null2;
  if (rot) {
    relmax = fmaxf(relmax, __fdividef((float)apq2, (float)pq));
    const double d = aqq - app, h = 2.0 * apq;
    const double big = fmax(fabs(d), fabs(h));
    const double ad = fabs(d), ah = fabs(h);
    if (ah <= 1e-3 * ad && ad < 1e150 && ad > 1e-140) {
      // small rotation (the Brand rank-1 cores: |h / d| ~ 1e-5): the same
      // t, c, s as below from series in eps = (h/d)^2 <= 1e-6 -- one
      // reciprocal instead of two reciprocal square roots and a reciprocal
      // on the round's critical path; truncation < 1e-19 relative.
      //   u / |d| = 1 + sqrt(1 + eps) = 2 + del, del = eps/2 - eps^2/8
      //   tau = |h| / u = (|h|/|d|) / (2 + del),  c = (1 + tau^2)^(-1/2)
      const double hr = ah * j32_rcp(ad);
      const double eps = hr * hr;
      const double del = eps * fma(-0.125, eps, 0.5);
      const double tau = 0.5 * hr * fma(del, fma(0.25, del, -0.5), 1.0);
      const double tau2 = tau * tau;
      c = fma(tau2, fma(0.375, tau2, -0.5), 1.0);
      t = ((d < 0.0) != (h < 0.0)) ? -tau : tau;  // sign(d) h / u
      sn = t * c;
    } else if (big < 1e150 && big > 1e-140) {
      const double x2 = fma(d, d, h * h);
      const double u = fabs(d) + x2 * j32_rsqrt(x2);
      const double qq = j32_rsqrt(fma(u, u, h * h));
      const double sh = d < 0.0 ? -h : h;
      c = u * qq;
      sn = sh * qq;
      t = sh * j32_rcp(u);
    } else {
      const double zeta = d * j32_rcp(h);
      const double w = fma(zeta, zeta, 1.0);
      const double root = fabs(zeta) > 1e100 ? fabs(zeta) : w * j32_rsqrt(w);
      t = copysign(j32_rcp(fabs(zeta) + root), zeta);
      c = j32_rsqrt(fma(t, t, 1.0));
      sn = t * c;
    }
  }
  any |= rot;
  // rotate and swap places: position p <- s g_p + c g_q, p+1 <- c g_p - s g_q
  // (idle lanes: c = 1, s = 0, y = x, so x is kept exactly)
  const double al = lower ? sn : -sn;
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = fma(al, x[i], c * y[i]);
  if (!idle) {
    nrm = lower ? fma(t, apq, aqq) : fma(-t, apq, app);
    if (lower) cs_log[ODD ? (lane - 1) >> 1 : lane >> 1] = make_double2(c, sn);
  }
}

template <bool BUILD>
__device__ __forceinline__ void j32c_body(
    int b, int s, const double* __restrict__ core, int64_t core_stride, int ldcore,
    double* __restrict__ uk, double* __restrict__ vk, int64_t out_stride, int ldo,
    double* __restrict__ sv, int64_t sv_stride, const Rank1Core& rc, double* __restrict__ s_out,
    int64_t s_out_stride) {
  extern __shared__ __align__(16) unsigned char j32_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  J32Smem& W = reinterpret_cast<J32Smem*>(j32_raw)[warp];
  double* nrmv = W.nrm;
  int* pos = W.pos;
  double x[32];  // column `lane` of G
  double ka = 0.0, kb = 0.0, ks = 0.0, kdel = 0.0;  // K = diag(s) + delta a b^T (lane entries)
  if constexpr (BUILD) {
    // Fused K6 (_kernels.pyx:209-213): K = diag(s) + delta U[i,:]^T Vt[:,j]^T,
    // column q = s_q e_q + (delta b_q) a, with a = U[i, :] and b = V_eff[j, :]
    // gathered through the deferred bases (U = [Ub 0; 0 I] W, V_eff = [V | Z^T] G)
    const int64_t i = rc.ii[b], j = rc.jj[b];
    const double d = rc.delta[b];
    const LazyBasis& lz = rc.lz;
    double ap = 0.0;
    if (lane < s) {
      if (!lz.active) {
        ap = rc.U.p[b * rc.U.stride + i * rc.U.ld + lane];
      } else if (i >= lz.m_base) {
        ap = lz.W.p[b * lz.W.stride + (lz.r_base + (i - lz.m_base)) * lz.W.ld + lane];
      } else {
        // every load issued before the first FMA (the gather is otherwise a
        // chain of dependent L2 round trips)
        const double* ur = rc.U.p + b * rc.U.stride + i * rc.U.ld;
        const double* Wb = lz.W.p + b * lz.W.stride;
        double uv[32], wv[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const bool ok = c < lz.r_base;
          uv[c] = ok ? ur[c] : 0.0;
          wv[c] = ok ? Wb[c * lz.W.ld + lane] : 0.0;
        }
        double a4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int c = 0; c < 32; ++c) a4[c & 3] = fma(uv[c], wv[c], a4[c & 3]);
        ap = (a4[0] + a4[1]) + (a4[2] + a4[3]);
      }
    }
    const double* vr = rc.V.p + b * rc.V.stride + j * rc.V.ld;
    double vq = 0.0;
    if (lane < s) {
      const VDefer& vd = rc.vd;
      if (!vd.G) {
        vq = vr[lane];
      } else {
        // V_eff[j, :] = [V[j, :fw] | Z[:, j]^T] G
        const double* Gb = vd.G + b * vd.g_stride;
        const double* Zb = vd.Z + b * vd.z_stride + j;
        double a4[4] = {0.0, 0.0, 0.0, 0.0};
        {
          double vv[32], gv[32];
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            const bool ok = c < vd.fw;
            vv[c] = ok ? vr[c] : 0.0;
            gv[c] = ok ? Gb[c * vd.ldg + lane] : 0.0;
          }
#pragma unroll
          for (int c = 0; c < 32; ++c) a4[c & 3] = fma(vv[c], gv[c], a4[c & 3]);
        }
        {
          double zv[kVWin], gz[kVWin];
#pragma unroll
          for (int t = 0; t < kVWin; ++t) {
            const bool ok = t < vd.nz;
            zv[t] = ok ? Zb[(int64_t)t * vd.ldz] : 0.0;
            gz[t] = ok ? Gb[(vd.fw + t) * vd.ldg + lane] : 0.0;
          }
#pragma unroll
          for (int t = 0; t < kVWin; ++t) a4[t & 3] = fma(zv[t], gz[t], a4[t & 3]);
        }
        vq = (a4[0] + a4[1]) + (a4[2] + a4[3]);
      }
    }
    const double sp = lane < s ? rc.s[(int64_t)b * rc.lds + lane] : 0.0;
    ka = ap;
    kb = vq;
    ks = sp;
    kdel = d;
    // the same product as the row layout (delta a_p) b_q, computed by lane q
#pragma unroll
    for (int r2 = 0; r2 < 32; ++r2) {
      const double da = d * __shfl_sync(0xffffffffu, ap, r2);
      double v = 0.0;
      if (lane < s && r2 < s) {
        v = da * vq;
        if (r2 == lane) v += sp;
      }
      x[r2] = v;
      W.V[lane][r2] = (lane == r2 && lane < s) ? 1.0 : 0.0;
    }
    if (lane == 0 && rc.A) {
      double* e = rc.A + b * rc.a_stride + i * rc.lda + j;
      const double old = *e;
      *e = old + d;
      const double nn = rc.N[b] + (2.0 * d * old + d * d);
      rc.N[b] = nn;
      if (rc.ring) {
        rc.ring[b] = nn;
        rc.ring[rc.ring_stride + b] = rc.rho[b];
        rc.ring[2 * rc.ring_stride + b] = rc.xnorm[b];
      }
    }
  } else {
    const double* K = core + b * core_stride;
#pragma unroll
    for (int r2 = 0; r2 < 32; ++r2) {
      x[r2] = (lane < s && r2 < s) ? K[r2 * ldcore + lane] : 0.0;
      W.V[lane][r2] = (lane == r2 && lane < s) ? 1.0 : 0.0;
    }
  }
  auto col_norm = [&]() {
    double n4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int i = 0; i < 32; ++i) n4[i & 3] = fma(x[i], x[i], n4[i & 3]);
    return (n4[0] + n4[1]) + (n4[2] + n4[3]);
  };
  // V from the structure of a rank-1 core (G = K V = U Sigma, so v =
  // K^T g / sigma^2 with K^T g = s o g + delta b (a . g); error ~ eps
  // sigma_max / sigma_min per tick once G is orthogonal to working
  // precision).  `reversed`: one sweep reversed the column positions.
  auto formula_v = [&](bool reversed) {
    const double n2 = col_norm();
    const bool live_col = (reversed ? 31 - lane : lane) < s;
    double* kv = reinterpret_cast<double*>(W.log);  // [a | b | s] (the log is not needed)
    kv[lane] = ka;
    kv[32 + lane] = kb;
    kv[64 + lane] = ks;
    __syncwarp();
    double d4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int i = 0; i < 32; ++i) d4[i & 3] = fma(kv[i], x[i], d4[i & 3]);
    const double dot = kdel * ((d4[0] + d4[1]) + (d4[2] + d4[3]));
    const double in2 = live_col ? 1.0 / n2 : 0.0;
    __syncwarp();  // every lane's reads of the staged G are done before V's tile is written
#pragma unroll
    for (int k = 0; k < 32; ++k) W.V[k][lane] = fma(kv[64 + k], x[k], kv[32 + k] * dot) * in2;
  };
  int sweeps = 0;
  bool fast = false, formula = false;
  // delta == 0 (a rejected device payload is staged as (0, 0, 0.0)): K =
  // diag(s) and the factors must come out bit for bit unchanged, so Uk and
  // Vk are written as exact identities below instead of G / sigma and the
  // structure formula (whose x * (1 / x) need not round to 1)
  const bool trivial = BUILD && kdel == 0.0;
  if (trivial) fast = true;
  if (BUILD && !trivial) {
    // Fast path for a well-conditioned Brand rank-1 core (every s live and
    // within a factor of 100): simultaneous steps (j32_step,
    // DMMA) from K itself to the reference's stop -- no chain of 32
    // dependent rotation rounds -- and V from the structure.  Cores with
    // close or dead singular values (a step's theta above 1e-4, or no
    // convergence in 4 steps) restart from K on the sweep path below.
    const double smax = warp_max(lane < s ? ks : 0.0);
    const double smin = -warp_max(lane < s ? -ks : -1e300);
    if (smin >= 1e-2 * smax && smin > 0.0) {
      const double null2 = fmax(1e-30 * warp_max(col_norm()), 1e-290);
      int pol = 1, steps = 0;
      for (; steps < 4 && pol == 1; ++steps)
        pol = j32_step(x, &W.V[0][0], reinterpret_cast<double*>(W.log), W.nrm, lane, null2, 1e-4);
      if (lane == 0) atomicAdd(&g_debug_counters[2], (unsigned long long)steps);
      if (pol == 0 || pol == 2) {
        fast = formula = true;
        if (lane == 0) atomicAdd(&g_debug_counters[3], 1ull);
      } else {
        // back to K and V = I (bit-identical to the fused build above)
#pragma unroll
        for (int r2 = 0; r2 < 32; ++r2) {
          const double da = kdel * __shfl_sync(0xffffffffu, ka, r2);
          double v = 0.0;
          if (lane < s && r2 < s) {
            v = da * kb;
            if (r2 == lane) v += ks;
          }
          x[r2] = v;
          W.V[lane][r2] = (lane == r2 && lane < s) ? 1.0 : 0.0;
        }
        __syncwarp();
      }
    }
  }
  for (; !fast && sweeps < kMaxSweeps;) {
    bool any = false;
    float relmax = 0.0f;
    double nrm = col_norm();  // exact squared norm at the sweep start
    const double null2 = fmax(1e-30 * warp_max(nrm), 1e-290);
    for (int rr = 0; rr < 16; ++rr) {
      j32c_round<false>(x, lane, W.log + (2 * rr) * 16, nrm, any, relmax, null2);
      j32c_round<true>(x, lane, W.log + (2 * rr + 1) * 16, nrm, any, relmax, null2);
    }
    __syncwarp();
    const bool rotated = __any_sync(0xffffffffu, any);
    // generic cores -- and rank-1 cores off the fast path -- stop exactly as
    // the reference: after a sweep without a rotation (_kernels.pyx:38-59)
    bool done = !rotated;
    // One-sweep rank-1 cores of moderate condition (every rotation of the
    // first sweep below kConvRel, sigma_max / sigma_min <= 100): the
    // finishing step (j32_step) brings G to the reference's stop, and the
    // right vectors follow from the structure instead of replaying the
    // sweep's rotations on V: G = K V = U Sigma, so v = K^T g / sigma^2 with
    // K^T g = s o g + delta b (a . g) (O(s^2) per core; error ~ eps
    // sigma_max / sigma_min per tick with G orthogonal to working precision).
    if constexpr (BUILD) {
      if (rotated && sweeps == 0 && warp_max((double)relmax) <= kConvRel * kConvRel) {
        const double n2 = col_norm();
        const bool live_col = (31 - lane) < s;  // one sweep reverses the positions
        const double mx = warp_max(live_col ? n2 : 0.0);
        const double mn = -warp_max(live_col ? -n2 : -1e300);
        if (mn >= 1e-4 * mx && mx > 0.0) {
          // V's tile (identity so far) holds the staged G; the log is the scratch
          const int pol = j32_step(x, &W.V[0][0], reinterpret_cast<double*>(W.log), W.nrm,
                                   lane, null2, 1e-7);
          if (pol >= 0) {
            formula = true;
            done = true;
          } else {
            // nearly equal columns: V's tile back to the identity (the log is
            // intact), replay this sweep and keep sweeping
#pragma unroll
            for (int r2 = 0; r2 < 32; ++r2) W.V[lane][r2] = (lane == r2 && lane < s) ? 1.0 : 0.0;
            __syncwarp();
          }
        }
      }
    }
    if (!formula) {
      double v[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = W.V[lane][j];
      j32_apply_v(v, W.log);
#pragma unroll
      for (int j = 0; j < 32; ++j) W.V[lane][j] = v[j];
    }
    if (formula) formula_v(true);
    __syncwarp();
    ++sweeps;
    if (done) break;
  }
  if (fast && !trivial) formula_v(false);
  __syncwarp();
  if (lane == 0) atomicAdd(&g_debug_counters[0], (unsigned long long)sweeps);
  if (lane == 0) atomicAdd(&g_debug_counters[1], 1ull);
  // position l holds original column id(l): a sweep reverses the order
  const bool rev = sweeps & 1;
  auto id_of = [&](int p) { return rev ? 31 - p : p; };
  const double myn = sqrt(col_norm());
  nrmv[lane] = myn;
  __syncwarp();
  {
    const int myid = id_of(lane);
    int rank = 0;
    for (int p = 0; p < 32; ++p) {
      const double o = nrmv[p];
      const int oid = id_of(p);
      rank += (o > myn) || (o == myn && oid < myid);
    }
    pos[lane] = rank;
    W.ipos[rank] = lane;
  }
  const double s0 = warp_max(myn);
  double* U = uk + b * out_stride;
  double* Vo = (BUILD && rc.vk_out) ? rc.vk_out + b * rc.vk_stride : vk + b * out_stride;
  const int ldv = (BUILD && rc.vk_out) ? rc.ldvk : ldo;
  double* S = sv + b * sv_stride;
  const bool live = myn > 0.0 && !(myn < kZeroSvRtol * s0);
  const bool mine = id_of(lane) < s;
  if (mine) {
    S[pos[lane]] = live ? myn : 0.0;
    if (s_out) s_out[b * s_out_stride + pos[lane]] = live ? myn : 0.0;  // install s directly
  }
  const bool any_dead = __any_sync(0xffffffffu, mine && !live);
  __syncwarp();
  if (BUILD && rc.uw_mode) {
    // Fused epilogue: Uk (= G / sigma_raw) staged in smem (the free log area,
    // columns XOR-swizzled by row parity so the B-fragment reads are
    // conflict-free), the core's dead-column completion done there, then the
    // deferred bases rotated by this warp and the engine-level completion.
    double* Us = reinterpret_cast<double*>(W.log);
    auto us = [&](int k, int n) -> double& { return Us[k * 32 + (n ^ ((k & 1) << 3))]; };
    {
      const double iv = live ? 1.0 / myn : 0.0;
      const int oc = pos[lane];
#pragma unroll
      for (int k = 0; k < 32; ++k)
        us(k, oc) = (k < s && mine) ? (trivial ? (x[k] != 0.0 ? 1.0 : 0.0) : x[k] * iv) : 0.0;
    }
    __syncwarp();
    if (any_dead) {
      for (int t = 0; t < s; ++t) {
        if (S[t] > 0.0) continue;
        for (int axis = 0; axis < s; ++axis) {
          double val = 0.0;
          if (lane < s) {
            val = (lane == axis) ? 1.0 : 0.0;
            for (int c = 0; c < s; ++c)
              if (c != t) val -= us(lane, c) * us(axis, c);
          }
          const double nrm2 = warp_sum(val * val);
          if (sqrt(nrm2) > 0.5) {
            __syncwarp();
            if (lane < s) us(lane, t) = val / sqrt(nrm2);
            __syncwarp();
            break;
          }
        }
      }
    }
    double* uwb = rc.uw.p + b * rc.uw.stride;
    if (rc.uw_mode == 1) {
      for (int i = 0; i < s; ++i)
        for (int c = lane; c < rc.uw.ld; c += 32) uwb[(int64_t)i * rc.uw.ld + c] = c < s ? us(i, c) : 0.0;
    } else {
      warp_rotate(uwb, rc.uw.ld, rc.uw_rows, s, s, [&](int k, int n) { return us(k, n); }, false, 1.0);
    }
    const int* ipos = W.ipos;
    if (rc.gw_rows > 0) {
      warp_rotate(rc.gw.p + b * rc.gw.stride, rc.gw.ld, rc.gw_rows, s, s,
                  [&](int k, int n) { return W.V[k][ipos[n]]; }, false, 1.0);
    } else if (lane < s) {
      const int srcl = ipos[lane];
      for (int i = 0; i < s; ++i) Vo[i * ldv + lane] = W.V[i][srcl];
    }
    __syncwarp();
    VDefer zvd = rc.zvd;
    if (zvd.G) {
      zvd.G += b * zvd.g_stride;
      if (zvd.Z) zvd.Z += b * zvd.z_stride;
    }
    warp_complete_zero(s, s_out + b * s_out_stride, Mat{rc.zU.p + b * rc.zU.stride, 0, rc.zU.ld},
                       rc.zm, Mat{rc.zV.p + b * rc.zV.stride, 0, rc.zV.ld}, rc.zn, zvd, nrmv);
    return;
  }
  // U = G / sigma_raw (_kernels.pyx:104): row i is written by all lanes at
  // their sorted columns (one 256-byte row per instruction); V from smem
  {
    const double iv = live ? 1.0 / myn : 0.0;
    const int oc = pos[lane];
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i < s && mine) U[i * ldo + oc] = trivial ? (x[i] != 0.0 ? 1.0 : 0.0) : x[i] * iv;
    if (lane < s) {
      const int srcl = W.ipos[lane];
      for (int i = 0; i < s; ++i) Vo[i * ldv + lane] = W.V[i][srcl];
    }
  }
  __syncwarp();
  if (!any_dead) return;
  __threadfence_block();
  for (int t = 0; t < s; ++t) {
    if (S[t] > 0.0) continue;
    for (int axis = 0; axis < s; ++axis) {
      double val = 0.0;
      if (lane < s) {
        val = (lane == axis) ? 1.0 : 0.0;
        for (int c = 0; c < s; ++c)
          if (c != t) val -= U[lane * ldo + c] * U[axis * ldo + c];
      }
      const double nrm2 = warp_sum(val * val);
      if (sqrt(nrm2) > 0.5) {
        __syncwarp();
        if (lane < s) U[lane * ldo + t] = val / sqrt(nrm2);
        __syncwarp();
        break;
      }
    }
  }
}


// One warp per core.  List mode (rc.fb_list, BUILD): the cores that
// rank1_fast_kernel handed back, *fb_count of them; the last CTA to finish
// resets the list for the next tick.
template <bool BUILD>
__global__ void __launch_bounds__(kJ32Warps * 32, 3) jacobi32c_kernel(
    int s, const double* __restrict__ core, int64_t core_stride, int ldcore, double* __restrict__ uk,
    double* __restrict__ vk, int64_t out_stride, int ldo, double* __restrict__ sv,
    int64_t sv_stride, int batch, Rank1Core rc, double* __restrict__ s_out, int64_t s_out_stride) {
  const int warp = threadIdx.x >> 5;
  if constexpr (!BUILD) {
    const int b = blockIdx.x * kJ32Warps + warp;
    if (b >= batch) return;
    j32c_body<false>(b, s, core, core_stride, ldcore, uk, vk, out_stride, ldo, sv, sv_stride, rc,
                     s_out, s_out_stride);
    return;
  }
  const bool list = BUILD && rc.fb_list;
  const int cnt = list ? *reinterpret_cast<volatile int*>(rc.fb_count) : batch;
  const int step = list ? gridDim.x * kJ32Warps : cnt;
  // one call site (the body is inlined once)
  for (int idx = blockIdx.x * kJ32Warps + warp; idx < cnt; idx += step)
    j32c_body<BUILD>(list ? rc.fb_list[idx] : idx, s, core, core_stride, ldcore, uk, vk, out_stride,
                     ldo, sv, sv_stride, rc, s_out, s_out_stride);
  if (list) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(rc.fb_done, 1) == (int)gridDim.x - 1) {
        *rc.fb_count = 0;
        *rc.fb_done = 0;
        __threadfence();
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Rank-1 Brand core on one CTA (4 warps) from the structure of
// K = diag(s) + delta a b^T (_kernels.pyx:190-237: the core of the
// projection rule, engine.py:149-167).  For a well-conditioned core (every
// s live and within a factor of 100, the steady state of a rank-1 stream)
// two simultaneous Jacobi steps reach the reference's stop (|M_pq| <=
// 1e-14 sqrt(M_pp M_qq), _kernels.pyx:38-59), as j32_step does, but
//   * the first Gram M1 = K^T K = diag(s^2) + delta (s o a) b^T + delta
//     b (s o a)^T + delta^2 |a|^2 b b^T is formed from the structure
//     (O(s^2) scalar work, no DMMA),
//   * the first rotation G1 = K J1 = K + diag(s)(J1 - I) + delta a
//     (b^T (J1 - I)) also from the structure (J1 = I + Theta1 +
//     Theta1^2 / 2, Theta1^2 on DMMA, symmetric: upper tiles only),
//   * only the second step (Gram of G1, first-order rotation G2 = G1 (I +
//     Theta2)) runs on dense 32 x 32 products -- 80 + 128 DMMA.8x8x4
//     instead of 544 for two dense steps;
// the work of one core is split over four warps (tiles and row groups), so
// the per-core dependent chain is ~4x shorter than the one-warp kernel's.
// V follows from the structure (v = K^T g / sigma^2, as formula_v), and the
// epilogue rotates the deferred bases (W rows by warps 0-1, Gv rows by
// warps 2-3) straight from the shared-memory Uk / Vk.
// Cores outside the fast path (close or dead singular values, a third
// step, delta == 0) are appended to a list and finished by the one-warp
// kernel (jacobi32c_kernel, list mode) with the engine state untouched;
// the tracked entry / N / read-back ring are updated here for every core.
constexpr int kR1Threads = 128;
constexpr int kLdT = 36;  // row pitch: conflict-free A (row g) / B (row q) fragment reads and row stores

struct R1Smem {
  double T0[32 * kLdT];  // Theta1 -> J1 - I -> Theta2 -> Uk
  double T1[32 * kLdT];  // G1 -> G2 -> Vk
  double a[32], bv[32], sv[32], d[32], beta[32], inv[32], nrm2[32];
  double acc[4];         // A[i, j], N, rho, |x| of this stream
  double red[2][4][32];
  double wt[4];
  int wv[4];
  int pos[32], ipos[32];
  int status;
};

__device__ __forceinline__ void r1_tile(int idx, int& mi, int& ni) {
  // upper-triangular 4 x 4 tile enumeration (10 tiles)
  mi = idx < 4 ? 0 : (idx < 7 ? 1 : (idx < 9 ? 2 : 3));
  ni = idx < 4 ? idx : (idx < 7 ? idx - 3 : (idx < 9 ? idx - 5 : 3));
}

// X[0:rows, :] <- X[0:rows, 0:r] Q (Q: 32 x 32 in shared memory, pitch kLdT,
// zero beyond r rows / keep columns), row groups rg0, rg0 + step, ... of one
// warp; the next group's operands are loaded before this group's stores.
__device__ __forceinline__ void r1_rotate(double* X, int ld, int rows, int r, const double* Q,
                                          int rg0, int step) {
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  auto load_a = [&](double (&a)[8], int row0) {
    const int row = row0 + g;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const int k = kk * 4 + q;
      a[kk] = (row < rows && k < r) ? X[(int64_t)row * ld + k] : 0.0;
    }
  };
  double a[8];
  if (8 * rg0 < rows) load_a(a, 8 * rg0);
  for (int row0 = 8 * rg0; row0 < rows; row0 += 8 * step) {
    double an[8];
    if (row0 + 8 * step < rows) load_a(an, row0 + 8 * step);
    double d[4][2];
#pragma unroll
    for (int nn = 0; nn < 4; ++nn) d[nn][0] = d[nn][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk)
#pragma unroll
      for (int nn = 0; nn < 4; ++nn)
        dmma_8x8x4(d[nn][0], d[nn][1], a[kk], Q[(kk * 4 + q) * kLdT + nn * 8 + g]);
    const int row = row0 + g;
    if (row < rows) {
#pragma unroll
      for (int nn = 0; nn < 4; ++nn) {
        const int c0 = nn * 8 + 2 * q;
        if (c0 < ld) *reinterpret_cast<double2*>(X + (int64_t)row * ld + c0) = make_double2(d[nn][0], d[nn][1]);
      }
    }
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) a[kk] = an[kk];
  }
}

__device__ __forceinline__ void rank1_fast_body(
    int s, int batch, const Rank1Core& rc, double* __restrict__ uk, double* __restrict__ vk,
    int64_t out_stride, int ldo, double* __restrict__ sv_out, int64_t sv_stride,
    double* __restrict__ s_out, int64_t s_out_stride, int* __restrict__ fb_list,
    int* __restrict__ fb_count, int& done_old) {
  extern __shared__ __align__(16) unsigned char r1_raw[];
  R1Smem& S = *reinterpret_cast<R1Smem*>(r1_raw);
  const int b = blockIdx.x;
  if (b >= batch) return;
  R1_MARK(0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int c = lane;          // column handled in the scalar phases
  const int r0 = 8 * warp;     // and its rows r0 .. r0 + 7
  double* T0 = S.T0;
  double* T1 = S.T1;
  // the epilogue's operands (deferred window W, right basis Gv) start
  // moving into L2 while the core is factored
  if (tid == 0 && rc.uw_mode == 2 && rc.uw_rows > 0)
    bulk_prefetch_l2(rc.uw.p + b * rc.uw.stride, (uint32_t)(rc.uw_rows * rc.uw.ld * sizeof(double)));
  if (tid == 32 && rc.gw_rows > 0)
    bulk_prefetch_l2(rc.gw.p + b * rc.gw.stride, (uint32_t)(rc.gw_rows * rc.gw.ld * sizeof(double)));
  const int64_t ii = rc.ii[b], jj = rc.jj[b];
  const double del = rc.delta[b];
  // ---- gathers (K6, _kernels.pyx:209-213) through the deferred bases:
  // a = U[i, :] = [U_base 0; 0 I] W, b = V_eff[j, :] = [V | Z^T] G; thread
  // (c, warp) forms the partial over a quarter of the contraction
  {
    const LazyBasis& lz = rc.lz;
    double pa = 0.0, pb = 0.0;
    if (c < s) {
      if (!lz.active) {
        if (warp == 0) pa = rc.U.p[b * rc.U.stride + ii * rc.U.ld + c];
      } else if (ii >= lz.m_base) {
        if (warp == 0) pa = lz.W.p[b * lz.W.stride + (lz.r_base + (ii - lz.m_base)) * lz.W.ld + c];
      } else {
        const double* ur = rc.U.p + b * rc.U.stride + ii * rc.U.ld;
        const double* Wb = lz.W.p + b * lz.W.stride;
        double uv[8], wv[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const int k = r0 + t;
          const bool ok = k < lz.r_base;
          uv[t] = ok ? ur[k] : 0.0;
          wv[t] = ok ? Wb[k * lz.W.ld + c] : 0.0;
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) pa = fma(uv[t], wv[t], pa);
      }
      const VDefer& vd = rc.vd;
      const double* vr = rc.V.p + b * rc.V.stride + jj * rc.V.ld;
      if (!vd.G) {
        if (warp == 0) pb = vr[c];
      } else {
        const double* Gb = vd.G + b * vd.g_stride;
        const double* Zb = vd.Z ? vd.Z + b * vd.z_stride + jj : nullptr;
        double vv[10], gv[10];
#pragma unroll
        for (int t = 0; t < 10; ++t) {
          const int k = 10 * warp + t;
          double x = 0.0, y = 0.0;
          if (k < vd.fw) {
            x = vr[k];
            y = Gb[k * vd.ldg + c];
          } else if (k - vd.fw < vd.nz) {
            x = Zb[(int64_t)(k - vd.fw) * vd.ldz];
            y = Gb[k * vd.ldg + c];
          }
          vv[t] = x;
          gv[t] = y;
        }
#pragma unroll
        for (int t = 0; t < 10; ++t) pb = fma(vv[t], gv[t], pb);
      }
    }
    S.red[0][warp][c] = pa;
    S.red[1][warp][c] = pb;
    if (tid < 32) S.sv[c] = c < s ? rc.s[(int64_t)b * rc.lds + c] : 0.0;
    // tracked entry, N and read-back ring (engine.py:162-166): the loads
    // are issued with the gathers, the stores after the epilogue
    if (tid == 96 && rc.A) {
      S.acc[0] = rc.A[b * rc.a_stride + ii * rc.lda + jj];
      S.acc[1] = rc.N[b];
      if (rc.ring) {
        S.acc[2] = rc.rho[b];
        S.acc[3] = rc.xnorm[b];
      }
    }
  }
  __syncthreads();
  R1_MARK(1);
  // the stores of the tracked-entry update (every core, fast or handed back)
  auto finish_acc = [&]() {
    if (tid == 96 && rc.A) {
      const double aij = S.acc[0];
      rc.A[b * rc.a_stride + ii * rc.lda + jj] = aij + del;
      const double nn = S.acc[1] + (2.0 * del * aij + del * del);
      rc.N[b] = nn;
      if (rc.ring) {
        rc.ring[b] = nn;
        rc.ring[rc.ring_stride + b] = S.acc[2];
        rc.ring[2 * rc.ring_stride + b] = S.acc[3];
      }
    }
  };

  if (tid < 32) {
    S.a[c] = ((S.red[0][0][c] + S.red[0][1][c]) + S.red[0][2][c]) + S.red[0][3][c];
    S.bv[c] = ((S.red[1][0][c] + S.red[1][1][c]) + S.red[1][2][c]) + S.red[1][3][c];
  }
  __syncthreads();
  // ---- column norms of K (K_rc = (delta a_r) b_c + [r == c] s_c) and the gate
  const double bc = S.bv[c], sc = S.sv[c];
  {
    double p = 0.0;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int r = r0 + t;
      double k = (del * S.a[r]) * bc;
      if (r == c) k += sc;
      p = fma(k, k, p);
    }
    S.red[0][warp][c] = p;
  }
  __syncthreads();
  if (tid < 32) {
    const double dc = ((S.red[0][0][c] + S.red[0][1][c]) + S.red[0][2][c]) + S.red[0][3][c];
    S.d[c] = dc;
    const double smax = warp_max(c < s ? sc : 0.0);
    const double smin = -warp_max(c < s ? -sc : -1e300);
    const double a2 = warp_sum(S.a[c] * S.a[c]);
    const double dmax = warp_max(dc);
    if (c == 0) {
      S.beta[0] = a2;
      S.beta[1] = fmax(1e-30 * dmax, 1e-290);  // null2
      // delta == 0 (a rejected device payload is staged as (0, 0, 0.0)) must
      // leave the factors unchanged bit for bit: the one-warp kernel's exact
      // path.  Outside the structure gate (a dead or a >100x smaller s): sweeps.
      S.status = del == 0.0 ? -1 : ((smin > 0.0 && smin >= 1e-2 * smax) ? 1 : 2);
    }
  }
  __syncthreads();
  if (S.status < 0) {
    if (tid == 0) {
      fb_list[atomicAdd(fb_count, 1)] = b;
      done_old = fb_arrive(rc.fb_fast_done, true);
    }
    finish_acc();
    return;
  }
  const double a2 = S.beta[0], null2 = S.beta[1];
  R1_MARK(2);
  bool sweep = S.status == 2;
  int steps = 0, nsw = 0;
  // warp-level reduction of (violation, max |theta|) -> block verdict:
  // 0 converged, 1 second-order step, 2 first-order step, -1 over the cap
  auto verdict = [&](bool viol, double tmax) {
    const bool wv = __any_sync(0xffffffffu, viol);
    const double wt = warp_max(tmax);
    if (lane == 0) {
      S.wv[warp] = wv;
      S.wt[warp] = wt;
    }
    __syncthreads();
    const bool v = S.wv[0] | S.wv[1] | S.wv[2] | S.wv[3];
    const double tm = fmax(fmax(S.wt[0], S.wt[1]), fmax(S.wt[2], S.wt[3]));
    __syncthreads();  // S.wv / S.wt reusable
    return !v ? 0 : (tm > 1e-4 ? -1 : (tm > 1e-8 ? 1 : 2));
  };
  // T0 <- J - I = Theta + Theta^2 / 2 (Theta skew in T0; Theta^2 symmetric:
  // upper tiles on DMMA, mirrored)
  auto second_order = [&]() {
    double acc[3][2], th[3][2];
#pragma unroll
    for (int nt = 0; nt < 3; ++nt) {
      const int idx = warp + 4 * nt;
      if (idx >= 10) break;
      int mi, ni;
      r1_tile(idx, mi, ni);
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        dmma_8x8x4(d0, d1, T0[(8 * mi + g) * kLdT + 4 * kk + q], T0[(4 * kk + q) * kLdT + 8 * ni + g]);
      acc[nt][0] = d0;
      acc[nt][1] = d1;
      const double2 tv = *reinterpret_cast<const double2*>(&T0[(8 * mi + g) * kLdT + 8 * ni + 2 * q]);
      th[nt][0] = tv.x;
      th[nt][1] = tv.y;
    }
    __syncthreads();
#pragma unroll
    for (int nt = 0; nt < 3; ++nt) {
      const int idx = warp + 4 * nt;
      if (idx >= 10) break;
      int mi, ni;
      r1_tile(idx, mi, ni);
      const int r = 8 * mi + g, cc = 8 * ni + 2 * q;
      *reinterpret_cast<double2*>(&T0[r * kLdT + cc]) =
          make_double2(fma(0.5, acc[nt][0], th[nt][0]), fma(0.5, acc[nt][1], th[nt][1]));
      if (mi != ni) {
        T0[cc * kLdT + r] = fma(0.5, acc[nt][0], -th[nt][0]);
        T0[(cc + 1) * kLdT + r] = fma(0.5, acc[nt][1], -th[nt][1]);
      }
    }
    __syncthreads();
  };
  // K (K_rc = (delta a_r) b_c + [r == c] s_c) into T1
  auto build_k = [&]() {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int r = r0 + t;
      double k = (del * S.a[r]) * bc;
      if (r == c) k += sc;
      T1[r * kLdT + c] = k;
    }
  };
  // ---- simultaneous steps (as j32_step) on G in T1: Gram on DMMA (upper
  // tiles), rotation G <- G + G (J - I); true once G meets the reference's
  // stop (|theta| <= 1e-8 for the last step: O(1e-16) off-diagonals left)
  auto dense_steps = [&](int maxit) -> bool {
    bool done = false;
  for (int it = 0; it < maxit && !done; ++it) {
    double th[3][2];
    bool viol = false;
    double tmax = 0.0;
#pragma unroll
    for (int nt = 0; nt < 3; ++nt) {
      const int idx = warp + 4 * nt;
      if (idx >= 10) break;
      int mi, ni;
      r1_tile(idx, mi, ni);
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        dmma_8x8x4(d0, d1, T1[(4 * kk + q) * kLdT + 8 * mi + g], T1[(4 * kk + q) * kLdT + 8 * ni + g]);
      th[nt][0] = d0;
      th[nt][1] = d1;
      if (mi == ni) {
#pragma unroll
        for (int e = 0; e < 2; ++e)
          if (g == 2 * q + e) S.d[8 * mi + g] = e ? d1 : d0;
      }
    }
    __syncthreads();
#pragma unroll
    for (int nt = 0; nt < 3; ++nt) {
      const int idx = warp + 4 * nt;
      if (idx >= 10) break;
      int mi, ni;
      r1_tile(idx, mi, ni);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = 8 * mi + g, cc = 8 * ni + 2 * q + e;
        const double dr = S.d[r], dc = S.d[cc], m = th[nt][e];
        const bool live = r != cc && dr > null2 && dc > null2;
        viol |= live && m * m > (kOrthoEps * kOrthoEps) * (dr * dc);
        const double t = live ? m * j32_rcp1(dc - dr) : 0.0;
        tmax = fmax(tmax, (t - t == 0.0) ? fabs(t) : 1e300);
        th[nt][e] = t;
      }
    }
    const int stv = verdict(viol, tmax);
    if (stv == 0) {
      done = true;
      break;
    }
    if (stv < 0) break;
#pragma unroll
    for (int nt = 0; nt < 3; ++nt) {
      const int idx = warp + 4 * nt;
      if (idx >= 10) break;
      int mi, ni;
      r1_tile(idx, mi, ni);
      const int r = 8 * mi + g, cc = 8 * ni + 2 * q;
      *reinterpret_cast<double2*>(&T0[r * kLdT + cc]) = make_double2(th[nt][0], th[nt][1]);
      if (mi != ni) {
        T0[cc * kLdT + r] = -th[nt][0];
        T0[(cc + 1) * kLdT + r] = -th[nt][1];
      }
    }
    __syncthreads();
    if (stv == 1) second_order();
    // G <- G + G (J - I): warp w owns row tile w
    double d[4][2];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) d[ni][0] = d[ni][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const double av = T1[(8 * warp + g) * kLdT + 4 * kk + q];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
        dmma_8x8x4(d[ni][0], d[ni][1], av, T0[(4 * kk + q) * kLdT + 8 * ni + g]);
    }
    double2 gn[4];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const double2 gv = *reinterpret_cast<const double2*>(&T1[(8 * warp + g) * kLdT + 8 * ni + 2 * q]);
      gn[ni] = make_double2(gv.x + d[ni][0], gv.y + d[ni][1]);
    }
    __syncthreads();
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
      *reinterpret_cast<double2*>(&T1[(8 * warp + g) * kLdT + 8 * ni + 2 * q]) = gn[ni];
    __syncthreads();
    ++steps;
    if (stv == 2) done = true;  // |theta| <= 1e-8: O(1e-16) off-diagonals left
  }
    return done;
  };
  if (!sweep) {
    // ---- step 1: Theta1 from the structured Gram (theta_rc = M_rc / (d_c - d_r))
    int st1;
    {
      bool viol = false;
      double tmax = 0.0;
      const double dc = S.d[c];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int r = r0 + t;
        const double dr = S.d[r];
        const bool live = r != c && dr > null2 && dc > null2;
        double th = 0.0;
        if (live) {
          // symmetric in (r, c) bit for bit: operands in (min, max) order
          const int p = min(r, c), qx = max(r, c);
          const double m = del * fma(S.sv[p] * S.a[p], S.bv[qx], (S.sv[qx] * S.a[qx]) * S.bv[p]) +
                           ((del * del) * a2) * (S.bv[r] * bc);
          viol |= m * m > (kOrthoEps * kOrthoEps) * (dr * dc);
          th = m * j32_rcp1(dc - dr);
          tmax = fmax(tmax, (th - th == 0.0) ? fabs(th) : 1e300);
        }
        T0[r * kLdT + c] = th;
      }
      st1 = verdict(viol, tmax);
    }
  R1_MARK(3);
    if (st1 < 0) {
      sweep = true;
    } else {
      if (st1 == 1) second_order();
      if (st1 > 0) {
        ++steps;
        // beta = b^T (J1 - I)
        double p = 0.0;
#pragma unroll
        for (int t = 0; t < 8; ++t) p = fma(S.bv[r0 + t], T0[(r0 + t) * kLdT + c], p);
        S.red[0][warp][c] = p;
        __syncthreads();
        if (tid < 32) S.beta[c] = ((S.red[0][0][c] + S.red[0][1][c]) + S.red[0][2][c]) + S.red[0][3][c];
        __syncthreads();
      }
      // G1 = K + K (J1 - I) = K + diag(s) (J1 - I) + (delta a) beta^T   (G1 = K when st1 == 0)
      {
        const double betac = st1 > 0 ? S.beta[c] : 0.0;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const int r = r0 + t;
          const double da = del * S.a[r];
          double k = da * bc;
          if (r == c) k += sc;
          double gv = k;
          if (st1 > 0) gv = k + fma(S.sv[r], T0[r * kLdT + c], da * betac);
          T1[r * kLdT + c] = gv;
        }
      }
      __syncthreads();
      // ---- steps 2..4 (dense): G meets the stop, or the sweeps take over
  R1_MARK(4);
      if (st1 == 1 && !dense_steps(3)) sweep = true;
    }
  }
  R1_MARK(5);
  if (sweep) {
    // ---- close or graded singular values: one-sided Jacobi sweeps from K
    // with the reference's rotation and stop (_kernels.pyx:38-59), V
    // accumulated in T0.  Circle-method pairing, 16 pairs per round, 8
    // threads per pair (rows sub, sub + 8, ...); the pair's Gram entries
    // are reduced by an xor butterfly, so all 8 threads agree bit for bit.
    // Inside the structure gate, a first sweep whose rotations were all
    // below kConvRel leaves O(1e-12) off-diagonals (quadratic convergence):
    // the simultaneous steps finish G and V follows from the structure (as
    // the one-warp kernel's one-sweep exit).
    const bool gate_ok = S.status == 1;
    build_k();
#pragma unroll
    for (int t = 0; t < 8; ++t) T0[(r0 + t) * kLdT + c] = (r0 + t == c && c < s) ? 1.0 : 0.0;
    __syncthreads();
    const int pr = tid >> 3, sub = tid & 7;
    bool conv = false;
    for (int sw = 0; sw < kMaxSweeps && !conv; ++sw) {
      ++nsw;
      bool rot = false;
      float relmax = 0.0f;
      for (int rr = 0; rr < 31; ++rr) {
        const int x0 = tour_slot(pr, rr, 32), x1 = tour_slot(31 - pr, rr, 32);
        const int p = min(x0, x1), qq = max(x0, x1);
        double gp[4], gq[4], app = 0.0, aqq = 0.0, apq = 0.0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int i = sub + 8 * k;
          gp[k] = T1[i * kLdT + p];
          gq[k] = T1[i * kLdT + qq];
          app = fma(gp[k], gp[k], app);
          aqq = fma(gq[k], gq[k], aqq);
          apq = fma(gp[k], gq[k], apq);
        }
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
          app += __shfl_xor_sync(0xffffffffu, app, o);
          aqq += __shfl_xor_sync(0xffffffffu, aqq, o);
          apq += __shfl_xor_sync(0xffffffffu, apq, o);
        }
        const double pq = app * aqq;
        if (qq < s && apq * apq > (kOrthoEps * kOrthoEps) * pq) {
          relmax = fmaxf(relmax, __fdividef((float)(apq * apq), (float)pq));
          // zeta = (aqq - app) / (2 apq), t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)),
          // c = 1 / sqrt(1 + t^2), s = c t, in the overflow-safe form
          // u = |d| + sqrt(d^2 + h^2) (d = aqq - app, h = 2 apq): c = u / sqrt(u^2 + h^2)
          const double d = aqq - app, h = 2.0 * apq;
          const double big = fmax(fabs(d), fabs(h));
          double cs, sn;
          if (big < 1e150 && big > 1e-140) {
            const double x2 = fma(d, d, h * h);
            const double u = fabs(d) + x2 * j32_rsqrt(x2);
            const double qv = j32_rsqrt(fma(u, u, h * h));
            cs = u * qv;
            sn = (d < 0.0 ? -h : h) * qv;
          } else {
            const double zeta = d / h;
            const double t = zeta >= 0.0 ? 1.0 / (zeta + sqrt(1.0 + zeta * zeta))
                                         : -1.0 / (-zeta + sqrt(1.0 + zeta * zeta));
            cs = 1.0 / sqrt(1.0 + t * t);
            sn = t * cs;
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int i = sub + 8 * k;
            T1[i * kLdT + p] = cs * gp[k] - sn * gq[k];
            T1[i * kLdT + qq] = sn * gp[k] + cs * gq[k];
            const double vp = T0[i * kLdT + p], vq = T0[i * kLdT + qq];
            T0[i * kLdT + p] = cs * vp - sn * vq;
            T0[i * kLdT + qq] = sn * vp + cs * vq;
          }
          rot = true;
        }
        __syncthreads();
      }
      const bool wr = __any_sync(0xffffffffu, rot);
      const float wm = (float)warp_max((double)relmax);
      if (lane == 0) {
        S.wv[warp] = wr;
        S.wt[warp] = wm;
      }
      __syncthreads();
      const bool any = S.wv[0] | S.wv[1] | S.wv[2] | S.wv[3];
      const double rm = fmax(fmax(S.wt[0], S.wt[1]), fmax(S.wt[2], S.wt[3]));
      __syncthreads();
      conv = !any;
      if (!conv && sw == 0 && gate_ok && rm <= kConvRel * kConvRel) {
        if (dense_steps(3)) {
          sweep = false;  // V from the structure below
          conv = true;
        }
        break;
      }
    }
    if (!conv) {
      if (tid == 0) {
      fb_list[atomicAdd(fb_count, 1)] = b;
      done_old = fb_arrive(rc.fb_fast_done, true);
    }
    finish_acc();
      return;
    }
  }
  R1_MARK(6);
  // ---- sigma = column norms of G, stable descending order (_kernels.pyx:94-101)
  {
    double p = 0.0, pd = 0.0;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const double gv = T1[(r0 + t) * kLdT + c];
      p = fma(gv, gv, p);
      pd = fma(S.a[r0 + t], gv, pd);
    }
    S.red[0][warp][c] = p;
    S.red[1][warp][c] = pd;
  }
  __syncthreads();
  if (tid < 32) {
    const double n2 = ((S.red[0][0][c] + S.red[0][1][c]) + S.red[0][2][c]) + S.red[0][3][c];
    const double ad = ((S.red[1][0][c] + S.red[1][1][c]) + S.red[1][2][c]) + S.red[1][3][c];
    const double myn = sqrt(n2);
    S.nrm2[c] = myn;
    __syncwarp();
    int rank = 0;
    for (int p2 = 0; p2 < 32; ++p2) {
      const double o = S.nrm2[p2];
      rank += (o > myn) || (o == myn && p2 < c);
    }
    const double s0 = warp_max(myn);
    const bool live = myn > 0.0 && !(myn < kZeroSvRtol * s0);
    const bool dead = __any_sync(0xffffffffu, c < s && !live);
    __syncwarp();
    S.pos[c] = rank;
    S.ipos[rank] = c;
    S.inv[c] = (c < s && live) ? 1.0 / myn : 0.0;
    S.d[c] = (c < s && live) ? 1.0 / n2 : 0.0;
    S.beta[c] = del * ad;  // delta (a . g_c)
    if (c == 0) S.status = dead ? -1 : 0;
    if (!dead && c < s) {
      sv_out[b * sv_stride + rank] = myn;
      if (s_out) s_out[b * s_out_stride + rank] = myn;
    }
  }
  __syncthreads();
  if (S.status < 0) {
    if (tid == 0) {
      fb_list[atomicAdd(fb_count, 1)] = b;
      done_old = fb_arrive(rc.fb_fast_done, true);
    }
    finish_acc();
    return;
  }
  if (tid == 0) {
    done_old = fb_arrive(rc.fb_fast_done, false);  // this core stays here
    atomicAdd(&g_debug_counters[1], 1ull);
    if (sweep) {
      atomicAdd(&g_debug_counters[0], (unsigned long long)nsw);
    } else {
      atomicAdd(&g_debug_counters[2], (unsigned long long)steps);
      atomicAdd(&g_debug_counters[3], 1ull);
    }
  }
  R1_MARK(7);
  // ---- Uk = G / sigma (sorted columns) -> T0; Vk = K^T g / sigma^2 -> T1
  {
    const int pc = S.pos[c];
    const double iv = S.inv[c], in2 = S.d[c], dt = S.beta[c];
    double vv[8], uu[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int k = r0 + t;
      const double gv = T1[k * kLdT + c];
      uu[t] = gv * iv;  // 0 for columns >= s (iv = 0); rows >= s of G are 0
      // sweeps: the accumulated rotations; steps: the structure (v = K^T g / sigma^2)
      vv[t] = sweep ? (c < s ? T0[k * kLdT + c] : 0.0) : fma(S.sv[k], gv, S.bv[k] * dt) * in2;
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      T0[(r0 + t) * kLdT + pc] = uu[t];
      T1[(r0 + t) * kLdT + pc] = vv[t];
    }
  }
  __syncthreads();
  R1_MARK(8);
  // ---- outputs: deferred window W and deferred right basis Gv (their 8-row
  // groups dealt round-robin to the four warps); other modes: W / U by
  // warps 0-1, Gv / V by warps 2-3
  if (rc.uw_mode == 2 && rc.gw_rows > 0) {
    double* uwb = rc.uw.p + b * rc.uw.stride;
    double* gwb = rc.gw.p + b * rc.gw.stride;
    const int nwg = (rc.uw_rows + 7) / 8, ngg = (rc.gw_rows + 7) / 8;
    // the next item's operands are loaded before this item's stores
    auto load_item = [&](int item, double (&a)[8]) {
      const bool isw = item < nwg;
      const double* X = isw ? uwb : gwb;
      const int ld = isw ? rc.uw.ld : rc.gw.ld;
      const int rows = isw ? rc.uw_rows : rc.gw_rows;
      const int row = 8 * (isw ? item : item - nwg) + g;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const int k = kk * 4 + q;
        a[kk] = (row < rows && k < s) ? X[(int64_t)row * ld + k] : 0.0;
      }
    };
    double a[8];
    if (warp < nwg + ngg) load_item(warp, a);
    for (int item = warp; item < nwg + ngg; item += 4) {
      double an[8];
      if (item + 4 < nwg + ngg) load_item(item + 4, an);
      const bool isw = item < nwg;
      double* X = isw ? uwb : gwb;
      const int ld = isw ? rc.uw.ld : rc.gw.ld;
      const int rows = isw ? rc.uw_rows : rc.gw_rows;
      const int row = 8 * (isw ? item : item - nwg) + g;
      const double* Q = isw ? T0 : T1;
      double d[4][2];
#pragma unroll
      for (int nn = 0; nn < 4; ++nn) d[nn][0] = d[nn][1] = 0.0;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
#pragma unroll
        for (int nn = 0; nn < 4; ++nn)
          dmma_8x8x4(d[nn][0], d[nn][1], a[kk], Q[(kk * 4 + q) * kLdT + nn * 8 + g]);
      if (row < rows) {
#pragma unroll
        for (int nn = 0; nn < 4; ++nn) {
          const int c0 = nn * 8 + 2 * q;
          if (c0 < ld) *reinterpret_cast<double2*>(X + (int64_t)row * ld + c0) = make_double2(d[nn][0], d[nn][1]);
        }
      }
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) a[kk] = an[kk];
    }
  } else if (warp < 2) {
    if (rc.uw_mode == 2) {
      r1_rotate(rc.uw.p + b * rc.uw.stride, rc.uw.ld, rc.uw_rows, s, T0, warp, 2);
    } else if (rc.uw_mode == 1) {
      double* uwb = rc.uw.p + b * rc.uw.stride;
      for (int idx = tid; idx < s * rc.uw.ld; idx += 64) {
        const int i = idx / rc.uw.ld, cc = idx % rc.uw.ld;
        uwb[(int64_t)i * rc.uw.ld + cc] = cc < s ? T0[i * kLdT + cc] : 0.0;
      }
    } else {
      double* U = uk + b * out_stride;
      for (int idx = tid; idx < s * s; idx += 64) {
        const int i = idx / s, cc = idx % s;
        U[i * ldo + cc] = T0[i * kLdT + cc];
      }
    }
  } else {
    if (rc.gw_rows > 0) {
      r1_rotate(rc.gw.p + b * rc.gw.stride, rc.gw.ld, rc.gw_rows, s, T1, warp - 2, 2);
    } else {
      double* Vo = rc.vk_out ? rc.vk_out + b * rc.vk_stride : vk + b * out_stride;
      const int ldv = rc.vk_out ? rc.ldvk : ldo;
      for (int idx = tid - 64; idx < s * s; idx += 64) {
        const int i = idx / s, cc = idx % s;
        Vo[i * ldv + cc] = T1[i * kLdT + cc];
      }
    }
  }
  finish_acc();
#ifdef ISVD_R1_TRACE
  __syncthreads();
#endif
  R1_MARK(9);
}

// The CTA whose decision completes the count (fb_arrive) hands the cores on
// the fallback list (if any) to the one-warp kernel by a device-side tail
// launch (it starts when this grid has completed): no host launch per tick
// for the rare fallback.
__global__ void __launch_bounds__(kR1Threads, 8) rank1_fast_kernel(
    int s, int batch, Rank1Core rc, double* __restrict__ uk, double* __restrict__ vk,
    int64_t out_stride, int ldo, double* __restrict__ sv_out, int64_t sv_stride,
    double* __restrict__ s_out, int64_t s_out_stride) {
  int done_old = -1;
  rank1_fast_body(s, batch, rc, uk, vk, out_stride, ldo, sv_out, sv_stride, s_out, s_out_stride,
                  rc.fb_list, rc.fb_count, done_old);
  if (threadIdx.x == 0 && done_old == (int)gridDim.x - 1) {
    __threadfence();  // the other CTAs' list entries (each ordered before its count)
    *rc.fb_fast_done = 0;
    const int cnt = *reinterpret_cast<volatile int*>(rc.fb_count);
    if (cnt > 0) {
      Rank1Core fb = rc;
      fb.A = nullptr;  // tracked entry / N / ring already updated
      const int grid = min((cnt + kJ32Warps - 1) / kJ32Warps, 2 * 148);
      jacobi32c_kernel<true><<<grid, kJ32Warps * 32, sizeof(J32Smem) * kJ32Warps,
                               cudaStreamTailLaunch>>>(s, nullptr, 0, 0, uk, vk, out_stride, ldo,
                                                       sv_out, sv_stride, batch, fb, s_out,
                                                       s_out_stride);
    }
  }
}

}  // namespace

int read_r1_trace(int64_t* out, int n) {
  std::vector<long long> h((size_t)4096 * 10);
  ISVD_CUDA(cudaMemcpyFromSymbol(h.data(), g_r1_trace, sizeof(long long) * h.size()));
  for (int i = 0; i < n * 10; ++i) out[i] = h[i];
  return ISVD_OK;
}

int read_debug_counters(int64_t* out, int reset) {
  unsigned long long h[8];
  ISVD_CUDA(cudaMemcpyFromSymbol(h, g_debug_counters, sizeof(h)));
  for (int i = 0; i < 2; ++i) out[i] = (int64_t)h[i];
  out[6] = (int64_t)h[2];  // simultaneous-step (fast path) steps
  out[7] = (int64_t)h[3];  // rank-1 cores finished on the fast path
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    ISVD_CUDA(cudaMemcpyToSymbol(g_debug_counters, z, sizeof(z)));
  }
  return read_arrow_counters(out + 2, reset);
}

size_t core_svd_smem_bytes(int s, bool v_in_smem) {
  int ps = s | 1;
  return sizeof(double) * (size_t)s * ps * (v_in_smem ? 2 : 1);
}

int launch_rank1_core_svd32(int batch, int s, const Rank1Core& rc, double* uk, double* vk,
                            int64_t out_stride, int ldo, double* sv, int64_t sv_stride,
                            cudaStream_t st, double* s_out, int64_t s_out_stride) {
  if (s < 1 || s > 32) {
    set_error("fused rank-1 core: width out of range");
    return ISVD_EINVAL;
  }
  if (batch == 0) return ISVD_OK;
  static bool attr = false;
  const size_t smem = sizeof(J32Smem) * kJ32Warps;
  if (!attr) {
    ISVD_CUDA(cudaFuncSetAttribute(jacobi32c_kernel<true>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  // ISVD_RANK1_WARP=1 (A/B experiments): the one-warp kernel for every core
  static const bool warp_only = [] {
    const char* v = getenv("ISVD_RANK1_WARP");
    return v && v[0] == '1';
  }();
  if (!rc.fb_list || warp_only) {
    Rank1Core direct = rc;
    direct.fb_list = nullptr;
    jacobi32c_kernel<true><<<ceil_div(batch, kJ32Warps), kJ32Warps * 32, smem, st>>>(
        s, nullptr, 0, 0, uk, vk, out_stride, ldo, sv, sv_stride, batch, direct, s_out, s_out_stride);
    ISVD_LAUNCHED();
    return ISVD_OK;
  }
  // CTA-per-core structured fast path; the one-warp kernel on the cores it
  // hands back is tail-launched from the device (tracked entry / N / ring
  // already updated there)
  rank1_fast_kernel<<<batch, kR1Threads, sizeof(R1Smem), st>>>(
      s, batch, rc, uk, vk, out_stride, ldo, sv, sv_stride, s_out, s_out_stride);
  ISVD_LAUNCHED();
  return ISVD_OK;
}

int launch_core_svd(int batch, int s, const double* core, int64_t core_stride, int ldcore,
                    double* uk, double* vk, int64_t out_stride, int ldo, double* sv,
                    int64_t sv_stride, double* vscratch, const int* active, cudaStream_t st) {
  if (s < 1 || s > kCoreMaxS) {
    set_error("core size out of range (1.." + std::to_string(kCoreMaxS) + ")");
    return ISVD_EINVAL;
  }
  if (batch == 0) return ISVD_OK;
  if (s <= 32 && !active) {
    static bool j32_attr = false;
    const size_t smem = sizeof(J32Smem) * kJ32Warps;
    if (!j32_attr) {
      ISVD_CUDA(cudaFuncSetAttribute(jacobi32c_kernel<false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      j32_attr = true;
    }
    jacobi32c_kernel<false><<<ceil_div(batch, kJ32Warps), kJ32Warps * 32, smem, st>>>(
        s, core, core_stride, ldcore, uk, vk, out_stride, ldo, sv, sv_stride, batch, Rank1Core{},
        nullptr, 0);
    ISVD_LAUNCHED();
    return ISVD_OK;
  }
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
