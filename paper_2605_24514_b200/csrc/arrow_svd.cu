// K2a -- SVD of the Brand append core by the secular equation (O(s^2)).
//
// The append core of _kernels.pyx:149-157 / _kernels_py.py:36-42 is a
// "broken arrow":   K = [[diag(d), 0], [p^T, rho]]   (s = r + 1).
// Its squared singular values are the eigenvalues of K^T K =
// diag(d^2, 0) + z z^T with z = (p, rho), i.e. the roots of the secular
// equation  f(sigma) = 1 + sum_j z_j^2 / (delta_j^2 - sigma^2) = 0  with poles
// delta = (d, 0).  The reference obtains the same factorisation with a
// cyclic Jacobi sweep (O(s^3) per core, _kernels.pyx:22-59) or LAPACK gesdd;
// this kernel returns the same singular triplets (to rounding) with:
//   1. deflation: |z_j| <= tol -> sigma = delta_j with unit vectors; poles
//      closer than tol merged by a Givens rotation; all poles <= tol form one
//      zero pole (their z mass rotated into one slot);
//   2. one thread per root: bracketing by the interval midpoint, origin at the
//      nearer pole (sigma^2 = delta_o^2 + mu, differences formed without
//      cancellation), iteration on a two-pole rational model of f with
//      bisection safeguard;
//   3. Gu-Eisenstat: z is recomputed from the computed roots (Loewner
//      formula) so the singular vectors are orthogonal to working precision;
//   4. v_i ~ zhat_j / (delta_j^2 - sigma_i^2),  u_i ~ (delta_j zhat_j /
//      (delta_j^2 - sigma_i^2), -1 in the z row), normalised;
//   5. the reference's output conventions (_kernels.pyx:94-109): descending
//      sort, snap below 1e-12 sigma_0, dead left columns completed over
//      e_0, e_1, ... in order.
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <chrono>
#include <cooperative_groups.h>
#include "common.cuh"
#include "core_svd.cuh"
#include "warp_rot.cuh"
#include "../../include/isvd.h"

namespace isvd {

#ifdef ISVD_R1_TRACE
extern __device__ long long g_r1_trace[4096][10];  // core_svd.cu (relocatable device code)
#endif

namespace {

constexpr int kN = kCoreMaxS;  // max core size
constexpr int kArrowCluster = 8;      // CTAs per wide core when the batch is small
// A core of more than 128 roots on very few streams (config 5b: one 129 core
// per tick): 16 CTAs x 16 warps give every root / Loewner product / vector
// its own warp in ONE round -- with 8 CTAs the 129th item made one warp run a
// second round, which was half of each phase (tools/trace_5b.py).
constexpr int kArrowClusterWide = 16;  // non-portable cluster size
constexpr int kClusterWideMaxBatch = 4;
constexpr int kClusterMaxBatch = 32;  // up to 256 CTAs
__device__ unsigned long long g_arrow_counters[4];

// Shared state sized by a compile-time bound on the core size (one
// instantiation per bound keeps the per-CTA footprint small: ~4.6 KB at
// s <= 40, so ~40 cores can be resident per SM).
template <int kN>
struct ArrowSmem {
  double delta[kN];   // pole value per original column (zero group forced to 0)
  double z[kN];       // z per original column, updated by the deflation rotations
  double kd[kN];      // kept poles, ascending
  double kz[kN];      // their z
  double zhat[kN];    // Loewner-corrected z
  double mu[kN];      // root i: sigma_i^2 = kd[org[i]]^2 + mu[i]
  double sig[kN];     // all n singular values (kept roots then deflated)
  double rc[kN], rs[kN];
  int ra[kN], rb[kN], rboth[kN];  // rotation list
  int kcol[kN];       // kept slot -> original column
  int org[kN];        // root -> origin index into kd
  int dcol[kN];       // deflated -> original column
  int dzero[kN];      // deflated with a zero left direction (completion)
  int pos[kN];        // triple -> output column (sorted)
  int order[kN];      // ascending pole order of the original columns
  int nkept, ndefl, nrot;
  double scale;
};

// 1/x to ~1 ulp: MUFU.RCP64H seed + two Newton steps (no IEEE-division
// fix-up path); used for the secular-function terms and vector entries.
__device__ __forceinline__ double frcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// One step of the two-pole rational iteration for the secular equation
// g(x) = 1 + psi(x) + phi(x) (poles below / above the root, squared
// distances Di, Dn from the origin): the model psi ~ a1 + b1 / (Di - x'),
// phi ~ a2 + b2 / (Dn - x') matches value and slope at x (b1 = psi' (Di -
// x)^2, a1 = psi - psi' (Di - x): no division), its root comes from the
// stable quadratic formula with ~1 ulp reciprocals for the two quotients --
// the iterate only has to land inside the bracket (lo, hi), the stop tests
// are on g and on the bracket -- and falls back to bisection otherwise.
// `last`: the root beyond the largest pole (phi is a plain constant there).
__device__ __forceinline__ double secular_model_step(bool last, double x, double psi, double dpsi,
                                                     double phi, double dphi, double Di, double Dn,
                                                     double lo, double hi) {
  const double pi_ = Di - x;
  const double dp1 = dpsi * pi_;
  const double b1 = dp1 * pi_;
  const double a1 = psi - dp1;
  double xn = 0.5 * (lo + hi);
  if (!last) {
    const double qn = Dn - x;
    const double dp2 = dphi * qn;
    const double b2 = dp2 * qn;
    const double a2 = phi - dp2;
    const double A = 1.0 + a1 + a2;
    const double Dl = Dn - Di;
    // A p^2 + (A Dl + b1 + b2) p + b1 Dl = 0 with p = Di - x'
    const double B = A * Dl + b1 + b2, C = b1 * Dl;
    const double disc = B * B - 4.0 * A * C;
    if (disc >= 0.0) {
      const double qv = -0.5 * (B + copysign(sqrt(disc), B));
      const double p1 = (A != 0.0) ? qv * frcp(A) : -1e300;
      const double p2 = (qv != 0.0) ? C * frcp(qv) : -1e300;
      const double x1 = Di - p1, x2 = Di - p2;
      if (x1 > lo && x1 < hi) xn = x1;
      else if (x2 > lo && x2 < hi) xn = x2;
    }
  } else {
    const double A = 1.0 + a1 + phi;
    const double xc = (A > 0.0) ? Di + b1 * frcp(A) : xn;
    if (xc > lo && xc < hi) xn = xc;
  }
  return xn;
}

template <class SM>
__device__ __forceinline__ void apply_rots(double* col, int64_t stride, const SM& S,
                                           bool left) {
  // x_orig = G_1 G_2 ... G_k x : apply the last rotation first
  for (int k = S.nrot - 1; k >= 0; --k) {
    if (left && !S.rboth[k]) continue;
    const int a = S.ra[k], b = S.rb[k];
    const double c = S.rc[k], s = S.rs[k];
    double xa = col[a * stride], xb = col[b * stride];
    col[a * stride] = c * xa - s * xb;
    col[b * stride] = s * xa + c * xb;
  }
}

// WIDE (cores above 40, e.g. config 5b's 129): 512 threads, a parallel
// no-deflation check, and one warp per root / per Loewner product / per
// singular vector with the lanes over the poles (the one-thread-per-root
// form leaves one latency-bound warp per SM sub-partition at B = 1).
//
// CL > 1 (WIDE, few cores): a thread-block cluster of CL CTAs per core.
// Every CTA redoes the cheap O(n) set-up (load, sort, deflation --
// deterministic, so identical everywhere); roots, Loewner products and
// vectors are split over the CL * 16 warps, each result is stored into
// every CTA's shared memory over DSMEM, and cluster barriers separate the
// phases.  At B = 1 this spreads the 129-root core over CL SMs.
// phase marks of the wide (cluster) solver in trace builds: rank-0 CTA, thread 0
#ifdef ISVD_R1_TRACE
#define AB_MARK(k)                                                                     \
  do {                                                                                 \
    if (WIDE && crank == 0 && threadIdx.x == 0 && b < 4096) g_r1_trace[b][k] = clock64(); \
  } while (0)
#else
#define AB_MARK(k) \
  do {             \
  } while (0)
#endif
template <int kN, bool WIDE, int CL>
__device__ __forceinline__ void arrow_body(int b, int n, const double* __restrict__ core,
                                           int64_t core_stride, int ldcore,
                                           double* __restrict__ uk, double* __restrict__ vk,
                                           int64_t out_stride, int ldo, double* __restrict__ sv,
                                           int64_t sv_stride, double* __restrict__ s_out,
                                           int64_t s_out_stride, int nkeep, const ArrowFuse& af) {
  __shared__ ArrowSmem<kN> S;
  namespace cg = cooperative_groups;
  const int crank = CL > 1 ? (int)cg::this_cluster().block_rank() : 0;
  // cluster-wide barrier (release/acquire at cluster scope) or a CTA barrier
  auto csync = [&]() {
    if constexpr (CL > 1) cg::this_cluster().sync(); else __syncthreads();
  };
  // pointer to member `p` of S in CTA `rk` of the cluster (DSMEM)
  auto remote = [&](auto* p, int rk) {
    if constexpr (CL > 1) return cg::this_cluster().map_shared_rank(p, rk);
    else return p;
  };
  const int tid = threadIdx.x;
  const int r = n - 1;
  const double* K = core + b * core_stride;
  double* U = uk + b * out_stride;
  double* V = vk + b * out_stride;
  double* SV = sv + b * sv_stride;
  // the engine's s (first nkeep values) is written directly: no separate install copy
  double* SO = s_out ? s_out + b * s_out_stride : nullptr;
  auto put_sv = [&](int pc, double v) {
    SV[pc] = v;
    if (SO && pc < nkeep) SO[pc] = v;
  };
  const double eps = 2.220446049250313e-16;
  constexpr int kPL = (kN + 31) / 32;  // poles per lane when a warp shares one root / vector
  AB_MARK(0);

  // ---- load, scale (max over the block: warp maxima, then one smem pass)
  __shared__ double wmax[16];
  double mx = 0.0;
  for (int c = tid; c < n; c += blockDim.x) {
    const double dc = c < r ? fabs(K[c * ldcore + c]) : 0.0, zc = K[r * ldcore + c];
    S.delta[c] = dc;
    S.z[c] = zc;
    mx = fmax(mx, fmax(dc, fabs(zc)));
  }
  mx = warp_max(mx);
  if ((tid & 31) == 0) wmax[tid >> 5] = mx;
  __syncthreads();
  if (tid == 0) {
    double m2 = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m2 = fmax(m2, wmax[w]);
    S.scale = m2 > 0.0 ? m2 : 1.0;
  }
  __syncthreads();
  const double scale = S.scale;
  for (int c = tid; c < n; c += blockDim.x) {
    S.delta[c] /= scale;
    S.z[c] /= scale;
  }
  __syncthreads();
  // ascending order of poles; ties: higher column first (the rho column r
  // leads the zero group).  The poles are the installed singular values:
  // normally strictly descending and positive, so the order is r, r - 1,
  // ..., 0 (one parallel check instead of the O(n^2) rank pass).
  {
    bool unsorted = false;
    for (int c = tid; c < r; c += blockDim.x)
      unsorted |= !(S.delta[c] > (c + 1 < r ? S.delta[c + 1] : 0.0));
    if (!__syncthreads_or(unsorted)) {
      for (int p = tid; p < n; p += blockDim.x) S.order[p] = r - p;
    } else {
      for (int c = tid; c < n; c += blockDim.x) {
        double dc = S.delta[c];
        int rank = 0;
        for (int e = 0; e < n; ++e) {
          double de = S.delta[e];
          rank += (de < dc) || (de == dc && e > c);
        }
        S.order[rank] = c;
      }
    }
  }
  __syncthreads();

  // ---- deflation.  If no pole needs deflating (every |z| > tol, no pole
  // pair closer than tol, only the rho column at zero) every pole is kept in
  // sorted order -- filled in parallel; otherwise the sequential pass.
  bool serial = true;
  {
    const double tol = 8.0 * eps;
    bool need = false;
    for (int p = tid; p < n; p += blockDim.x) {
      const int c = S.order[p];
      const double dc = S.delta[c];
      need |= fabs(S.z[c]) <= tol;
      if (p > 0) {
        const double dp = S.delta[S.order[p - 1]];
        need |= dc <= tol || dc - dp <= tol;
      }
    }
    serial = __syncthreads_or(need);
    if (!serial) {
      for (int p = tid; p < n; p += blockDim.x) {
        const int c = S.order[p];
        const double dc = p == 0 ? 0.0 : S.delta[c];
        S.kcol[p] = c;
        S.kd[p] = dc;
        S.kz[p] = S.z[c];
        if (p == 0) S.delta[c] = 0.0;
      }
      if (tid == 0) {
        S.nkept = n;
        S.ndefl = 0;
        S.nrot = 0;
      }
    }
  }
#ifdef ISVD_ARROW_STATS
  if (tid == 0) {
    atomicAdd(&g_arrow_counters[2], 1ull);
    if (serial) atomicAdd(&g_arrow_counters[3], 1ull);
  }
#endif
  if (serial && tid == 0) {
    const double tol = 8.0 * eps;  // all values scaled to <= 1
    int nk = 0, nd = 0, nr = 0;
    // zero group: poles <= tol, combined into the first one (column r)
    int first = -1;
    int p = 0;
    for (; p < n; ++p) {
      const int c = S.order[p];
      if (S.delta[c] > tol) break;
      S.delta[c] = 0.0;
      if (first < 0) {
        first = c;
        continue;
      }
      const double z1 = S.z[first], z2 = S.z[c];
      const double t = hypot(z1, z2);
      if (t > 0.0) {
        S.ra[nr] = first; S.rb[nr] = c; S.rc[nr] = z1 / t; S.rs[nr] = z2 / t; S.rboth[nr] = 0;
        ++nr;
        S.z[first] = t;
        S.z[c] = 0.0;
      }
      S.dcol[nd] = c; S.dzero[nd] = 1; S.sig[nd] = 0.0;  // sig filled in later slots
      ++nd;
    }
    if (first >= 0) {
      if (fabs(S.z[first]) <= tol) {
        S.dcol[nd] = first; S.dzero[nd] = 1; ++nd;
      } else {
        S.kcol[nk] = first; S.kd[nk] = 0.0; S.kz[nk] = S.z[first]; ++nk;
      }
    }
    // regular poles, ascending
    for (; p < n; ++p) {
      const int c = S.order[p];
      if (fabs(S.z[c]) <= tol) {
        S.dcol[nd] = c; S.dzero[nd] = 0; ++nd;
        continue;
      }
      if (nk > 0 && S.kd[nk - 1] > 0.0 && S.delta[c] - S.kd[nk - 1] <= tol) {
        // merge the previous kept pole into c: zero its z, deflate it
        const int l = S.kcol[nk - 1];
        const double zl = S.kz[nk - 1], zc = S.z[c];
        const double t = hypot(zl, zc);
        S.ra[nr] = c; S.rb[nr] = l; S.rc[nr] = zc / t; S.rs[nr] = zl / t; S.rboth[nr] = 1;
        ++nr;
        S.z[c] = t;
        S.z[l] = 0.0;
        --nk;
        S.dcol[nd] = l; S.dzero[nd] = 0; ++nd;
      }
      S.kcol[nk] = c; S.kd[nk] = S.delta[c]; S.kz[nk] = S.z[c]; ++nk;
    }
    S.nkept = nk;
    S.ndefl = nd;
    S.nrot = nr;
  }
  AB_MARK(1);
  csync();  // CL > 1: also guarantees every CTA of the cluster is resident before DSMEM use
  AB_MARK(2);
  const int N = S.nkept, ND = S.ndefl;

  // ---- roots: thread (WIDE: warp) i solves for sigma_i in (kd[i], kd[i+1]).
  // warp_root: the 32 lanes of a warp solve one root together (lanes over the
  // poles); used for every root when WIDE and, otherwise, for the roots left
  // over once every thread has one (n = 33 with one warp per core).
  auto warp_root = [&](int i) {
    const int lane = tid & 31;
      // The first evaluation is at the interval midpoint (origin kd[i]); its
      // sign picks the origin (the nearer pole) and the half-interval, and
      // its terms already feed the first rational-model step (no separate
      // bracketing pass).  x lies strictly between poles i and i + 1, so the
      // terms of the poles below are negative and the others positive: the
      // sign of w sorts them into psi / phi, and sum |w| = phi - psi.
      const double di = S.kd[i];
      const double dn = i < N - 1 ? S.kd[i + 1] : 0.0;
      const double sm = 0.5 * (di + dn);
      const double mum = (sm - di) * (sm + di);
      int o = i;
      double dorg = di, lo, hi, x, Di = 0.0, Dn = 0.0;
      bool first = i < N - 1;
      if (first) {
        lo = 0.0;
        hi = mum;
        x = mum;
      } else {
        double zz = 0.0;
        for (int j = lane; j < N; j += 32) zz += S.kz[j] * S.kz[j];
        lo = 0.0;
        hi = warp_sum(zz);
        x = 0.5 * (lo + hi);
      }
      int iters = 0;
      for (int it = 0; it < 80; ++it) {
        ++iters;
        double psi = 0.0, dpsi = 0.0, phi = 0.0, dphi = 0.0;
        // a lane's poles fully unrolled (at most kPL): their reciprocal
        // chains are independent and a dependent FP64 instruction issues
        // only every ~40 cycles, so the rolled loop ran them back to back
#pragma unroll
        for (int ip = 0; ip < kPL; ++ip) {
          const int j = lane + 32 * ip;
          if (j < N) {
            const double dj = S.kd[j];
            const double t = frcp((dj - dorg) * (dj + dorg) - x);
            const double w = S.kz[j] * S.kz[j] * t;
            const bool below = __double2hiint(w) < 0;
            const double wl = below ? w : 0.0, wu = below ? 0.0 : w;
            psi += wl;
            dpsi = fma(wl, t, dpsi);
            phi += wu;
            dphi = fma(wu, t, dphi);
          }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          psi += __shfl_xor_sync(0xffffffffu, psi, off);
          dpsi += __shfl_xor_sync(0xffffffffu, dpsi, off);
          phi += __shfl_xor_sync(0xffffffffu, phi, off);
          dphi += __shfl_xor_sync(0xffffffffu, dphi, off);
        }
        // identical in every lane from here on (xor-reduced inputs)
        const double aps = phi - psi;
        const double g = 1.0 + psi + phi;
        if (first) {
          first = false;
          if (!(g > 0.0)) {  // root above the midpoint: origin at kd[i+1]
            o = i + 1;
            dorg = dn;
            lo = (sm - dn) * (sm + dn);
            hi = 0.0;
            x = lo;
          }
          Di = (di - dorg) * (di + dorg);
          Dn = (dn - dorg) * (dn + dorg);
        } else if (g < 0.0) {
          lo = x;
        } else {
          hi = x;
        }
        if (fabs(g) <= 4.0 * eps * (1.0 + aps) * N || !(g == g)) break;
        const double xn = secular_model_step(i == N - 1, x, psi, dpsi, phi, dphi, Di, Dn, lo, hi);
        if (fabs(xn - x) <= 2.0 * eps * fmax(fabs(xn), 1e-300) ||
            hi - lo <= 2.0 * eps * fmax(fabs(lo), fabs(hi))) {
          x = xn;
          break;
        }
        x = xn;
      }
      if (lane < CL) {
        auto* R = remote(&S, lane);
        R->org[i] = o;
        R->mu[i] = x;
        R->sig[ND + i] = sqrt(dorg * dorg + x);
      }
      if (lane == 0) {
#ifdef ISVD_ARROW_STATS
        atomicAdd(&g_arrow_counters[0], 1ull);
        atomicAdd(&g_arrow_counters[1], (unsigned long long)iters);
#endif
      }
      };
  if (WIDE) {
    const int nwarp = (blockDim.x >> 5) * CL;
    for (int i = crank * (blockDim.x >> 5) + (tid >> 5); i < N; i += nwarp) warp_root(i);
  } else {
    for (int i = (int)blockDim.x + (tid >> 5); i < N; i += (int)(blockDim.x >> 5)) warp_root(i);
  }
  if (!WIDE)
  for (int i = tid; i < N && i < (int)blockDim.x; i += blockDim.x) {
    int o;
    double lo, hi;
    const double di = S.kd[i];
    if (i < N - 1) {
      const double dn = S.kd[i + 1];
      const double sm = 0.5 * (di + dn);
      const double mum = (sm - di) * (sm + di);
      double f = 1.0;
      for (int j = 0; j < N; ++j) {
        const double dj = S.kd[j];
        f += S.kz[j] * S.kz[j] * frcp((dj - di) * (dj + di) - mum);
      }
      if (f > 0.0) {
        o = i; lo = 0.0; hi = mum;
      } else {
        o = i + 1; lo = (sm - dn) * (sm + dn); hi = 0.0;
      }
    } else {
      o = i;
      double zz = 0.0;
      for (int j = 0; j < N; ++j) zz += S.kz[j] * S.kz[j];
      lo = 0.0;
      hi = zz;
    }
    const double dorg = S.kd[o];
    const double Di = (di - dorg) * (di + dorg);
    const double Dn = (i < N - 1) ? (S.kd[i + 1] - dorg) * (S.kd[i + 1] + dorg) : 0.0;
    double x = 0.5 * (lo + hi);
    for (int it = 0; it < 80; ++it) {
      double psi = 0.0, dpsi = 0.0, phi = 0.0, dphi = 0.0, aps = 0.0;
      for (int j = 0; j < N; ++j) {
        const double dj = S.kd[j];
        const double t = frcp((dj - dorg) * (dj + dorg) - x);
        const double w = S.kz[j] * S.kz[j] * t;
        if (j <= i) {
          psi += w;
          dpsi += w * t;
        } else {
          phi += w;
          dphi += w * t;
        }
        aps += fabs(w);
      }
      const double g = 1.0 + psi + phi;
      if (g < 0.0) lo = x; else hi = x;
      if (fabs(g) <= 4.0 * eps * (1.0 + aps) * N || !(g == g)) break;
      // two-pole rational model through (psi, dpsi) and (phi, dphi)
      const double xn = secular_model_step(i == N - 1, x, psi, dpsi, phi, dphi, Di, Dn, lo, hi);
      if (fabs(xn - x) <= 2.0 * eps * fmax(fabs(xn), 1e-300) || hi - lo <= 2.0 * eps * fmax(fabs(lo), fabs(hi))) {
        x = xn;
        break;
      }
      x = xn;
    }
    S.org[i] = o;
    S.mu[i] = x;
    S.sig[ND + i] = sqrt(dorg * dorg + x);
  }
  // deflated singular values (unscaled positions 0..ND-1)
  for (int k = tid; k < ND; k += blockDim.x) S.sig[k] = S.dzero[k] ? 0.0 : S.delta[S.dcol[k]];
  AB_MARK(3);
  csync();
  AB_MARK(4);

  // ---- Loewner: zhat_j^2 = prod_k (sigma_k^2 - d_j^2) / prod_{k != j} (d_k^2 - d_j^2)
  if (WIDE) {
    const int lane = tid & 31, nwarp = (blockDim.x >> 5) * CL;
    for (int j = crank * (blockDim.x >> 5) + (tid >> 5); j < N; j += nwarp) {
      const double dj = S.kd[j];
      auto sdiff = [&](int k) {
        const double dk = S.kd[S.org[k]];
        return S.mu[k] - (dj - dk) * (dj + dk);
      };
      double acc = 1.0;
#pragma unroll
      for (int ip = 0; ip < kPL; ++ip) {  // independent quotients, then the lane's product
        const int k = lane + 32 * ip;
        if (k < N - 1) {
          const double dk = k < j ? S.kd[k] : S.kd[k + 1];
          acc *= sdiff(k) * frcp((dk - dj) * (dk + dj));
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc *= __shfl_xor_sync(0xffffffffu, acc, off);
      acc *= sdiff(N - 1);
      if (lane < CL) remote(&S, lane)->zhat[j] = copysign(sqrt(fmax(acc, 0.0)), S.kz[j]);
    }
  } else
  for (int j = tid; j < N; j += blockDim.x) {
    const double dj = S.kd[j];
    auto sdiff = [&](int k) {  // sigma_k^2 - d_j^2, accurate
      const double dk = S.kd[S.org[k]];
      return S.mu[k] - (dj - dk) * (dj + dk);
    };
    double acc = sdiff(N - 1);
    for (int k = 0; k < j; ++k) acc *= sdiff(k) * frcp((S.kd[k] - dj) * (S.kd[k] + dj));
    for (int k = j; k < N - 1; ++k) acc *= sdiff(k) * frcp((S.kd[k + 1] - dj) * (S.kd[k + 1] + dj));
    S.zhat[j] = copysign(sqrt(fmax(acc, 0.0)), S.kz[j]);
  }
  // ---- sorted output positions: descending sigma, ties by triple index.
  // Without deflation the interlacing kd_i < sigma_i < kd_{i+1} makes the
  // roots strictly ascending: position n - 1 - t unless rounding broke the
  // order (then, or with deflated values in front, the rank pass).
  {
    bool unsorted = false;
    for (int t = tid; t + 1 < n; t += blockDim.x) unsorted |= !(S.sig[t] < S.sig[t + 1]);
    if (!__syncthreads_or(unsorted)) {
      for (int t = tid; t < n; t += blockDim.x) S.pos[t] = n - 1 - t;
    } else {
      for (int t = tid; t < n; t += blockDim.x) {
        const double st = S.sig[t];
        int rank = 0;
        for (int e = 0; e < n; ++e) {
          const double se = S.sig[e];
          rank += (se > st) || (se == st && e < t);
        }
        S.pos[t] = rank;
      }
    }
  }
  // largest singular value: block max (the previous sync made sig visible)
  {
    double m1 = 0.0;
    for (int t = tid; t < n; t += blockDim.x) m1 = fmax(m1, S.sig[t]);
    m1 = warp_max(m1);
    if ((tid & 31) == 0) wmax[tid >> 5] = m1;
  }
  AB_MARK(5);
  csync();
  AB_MARK(6);
  double smax = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) smax = fmax(smax, wmax[w]);

  // ---- vectors, written straight into their sorted columns
  bool wide_done = false;
  if constexpr (WIDE) {
    if (ND == 0 && S.nrot == 0) {
      // One warp per vector.  A warp's column goes through shared memory so
      // that the CTA's (up to) 16 columns -- contiguous output columns when the
      // roots are in order -- leave as 128-byte row segments: written lane by
      // lane, every store instruction touched 32 different rows and the
      // uncoalesced stores were two thirds of this phase (4.5 K of 7 K cycles).
      wide_done = true;
      constexpr int kVW = 16;                 // warps per CTA (512 threads)
      __shared__ double vst[kN][kVW + 1];     // [row][warp]: V's columns, then U's
      __shared__ int vpc[kVW];                // output column per warp, -1: none
      const int lane = tid & 31, warp = tid >> 5, nwarp = kVW * CL;
      for (int base = crank * kVW; base < n; base += nwarp) {
        const int t = base + warp;
        const bool have = t < n;
        double vjs[kPL], djs[kPL];  // the lane's entries, kept for the write passes
        double iv = 0.0, iu = 0.0;
        bool dead = true;
        if (have) {
          const double dorg = S.kd[S.org[t]];
          const double mu = S.mu[t];
          double nv = 0.0, nu = 0.0;
#pragma unroll
          for (int ip = 0; ip < kPL; ++ip) {
            const int j = lane + 32 * ip;
            double vj = 0.0, dj = 0.0;
            if (j < N) {
              dj = S.kd[j];
              vj = S.zhat[j] * frcp((dj - dorg) * (dj + dorg) - mu);
            }
            vjs[ip] = vj;
            djs[ip] = dj;
            nv = fma(vj, vj, nv);
            nu = fma(dj * vj, dj * vj, nu);
          }
          nv = warp_sum(nv);
          nu = 1.0 + warp_sum(nu);  // the z-row entry of u is -1
          iv = rsqrt(nv);
          iu = rsqrt(nu);
          const double sg = S.sig[t];
          dead = !(sg > 0.0) || sg < kZeroSvRtol * smax;
          if (lane == 0) {
            vpc[warp] = S.pos[t];
            put_sv(S.pos[t], dead ? 0.0 : sg * scale);
          }
        } else if (lane == 0) {
          vpc[warp] = -1;
        }
        // (every row 0 .. n-1 is some pole's row: no deflation here)
        for (int pass = 0; pass < 2; ++pass) {
          if (have) {
#pragma unroll
            for (int ip = 0; ip < kPL; ++ip) {
              const int j = lane + 32 * ip;
              if (j < N) {
                const int row = S.kcol[j];
                if (pass == 0) vst[row][warp] = vjs[ip] * iv;
                else if (row != r) vst[row][warp] = dead ? 0.0 : djs[ip] * vjs[ip] * iu;
              }
            }
            if (pass == 1 && lane == 0) vst[r][warp] = dead ? 0.0 : -iu;
          }
          __syncthreads();
          double* X = pass == 0 ? V : U;
          for (int idx = tid; idx < n * kVW; idx += blockDim.x) {
            const int row = idx / kVW, w = idx % kVW;
            const int pc = vpc[w];
            if (pc >= 0) X[row * ldo + pc] = vst[row][w];
          }
          __syncthreads();
        }
      }
    }
  }
  if (wide_done) {
  } else if (ND == 0 && S.nrot == 0) {
    // common case (no deflation): every row of both columns is written once
    for (int t = tid; t < n; t += blockDim.x) {
      const int pc = S.pos[t];
      const int i = t;
      const double dorg = S.kd[S.org[i]];
      const double mu = S.mu[i];
      double nv = 0.0, nu = 1.0;  // the z-row entry of u is -1
      for (int j = 0; j < N; ++j) {
        const double dj = S.kd[j];
        const double vj = S.zhat[j] * frcp((dj - dorg) * (dj + dorg) - mu);
        nv = fma(vj, vj, nv);
        nu = fma(dj * vj, dj * vj, nu);
      }
      const double iv = rsqrt(nv), iu = rsqrt(nu);
      const double sg = S.sig[t];
      const bool dead = !(sg > 0.0) || sg < kZeroSvRtol * smax;
      for (int j = 0; j < N; ++j) {
        const double dj = S.kd[j];
        const double vj = S.zhat[j] * frcp((dj - dorg) * (dj + dorg) - mu);
        const int row = S.kcol[j];
        V[row * ldo + pc] = vj * iv;
        if (row != r) U[row * ldo + pc] = dead ? 0.0 : dj * vj * iu;
      }
      U[r * ldo + pc] = dead ? 0.0 : -iu;
      put_sv(pc, dead ? 0.0 : sg * scale);
    }
  } else
  for (int t = crank * blockDim.x + tid; t < n; t += blockDim.x * CL) {
    const int pc = S.pos[t];
    double* vcol = V + pc;
    double* ucol = U + pc;
    for (int l = 0; l < n; ++l) {
      vcol[l * ldo] = 0.0;
      ucol[l * ldo] = 0.0;
    }
    const double sg = S.sig[t];
    const bool dead = !(sg > 0.0) || sg < kZeroSvRtol * smax;
    if (t < ND) {
      const int c = S.dcol[t];
      vcol[c * ldo] = 1.0;
      apply_rots(vcol, ldo, S, false);
      if (!S.dzero[t] && !dead) {
        ucol[c * ldo] = 1.0;
        apply_rots(ucol, ldo, S, true);
      }
    } else {
      const int i = t - ND;
      const double dorg = S.kd[S.org[i]];
      double nv = 0.0, nu = 1.0;  // the z-row entry of u is -1
      for (int j = 0; j < N; ++j) {
        const double dj = S.kd[j];
        const double inv = 1.0 / ((dj - dorg) * (dj + dorg) - S.mu[i]);
        const double vj = S.zhat[j] * inv;
        const double uj = dj * vj;
        nv = fma(vj, vj, nv);
        nu = fma(uj, uj, nu);
        vcol[S.kcol[j] * ldo] = vj;
        if (dj > 0.0) ucol[S.kcol[j] * ldo] = uj;
      }
      const double iv = 1.0 / sqrt(nv), iu = 1.0 / sqrt(nu);
      for (int j = 0; j < N; ++j) {
        vcol[S.kcol[j] * ldo] *= iv;
        if (S.kd[j] > 0.0) ucol[S.kcol[j] * ldo] *= iu;
      }
      ucol[r * ldo] = -iu;
      apply_rots(vcol, ldo, S, false);
      apply_rots(ucol, ldo, S, true);
      if (dead)
        for (int l = 0; l < n; ++l) ucol[l * ldo] = 0.0;
    }
    put_sv(pc, dead ? 0.0 : sg * scale);
  }
  AB_MARK(7);
  csync();  // every column of U / V / SV written (global, cluster scope)
  AB_MARK(8);
  if (crank != 0) return;

  // ---- dead-column completion over e_0, e_1, ... (_kernels.pyx:62-79)
  bool mine_dead = false;
  for (int t = tid; t < n; t += blockDim.x) mine_dead |= !(SV[t] > 0.0);
  if (__syncthreads_or(mine_dead) && tid < 32) {
    const int lane = tid;
    for (int t = 0; t < n; ++t) {
      if (SV[t] > 0.0) continue;
      for (int axis = 0; axis < n; ++axis) {
        double nrm2 = 0.0;
        for (int i = lane; i < n; i += 32) {
          double v = (i == axis) ? 1.0 : 0.0;
          for (int c = 0; c < n; ++c)
            if (c != t) v -= U[i * ldo + c] * U[axis * ldo + c];
          nrm2 = fma(v, v, nrm2);
        }
        nrm2 = warp_sum(nrm2);
        const double nrm = sqrt(nrm2);
        if (nrm > 0.5) {
          double vals[(kN + 31) / 32];
          int cnt = 0;
          for (int i = lane; i < n; i += 32) {
            double v = (i == axis) ? 1.0 : 0.0;
            for (int c = 0; c < n; ++c)
              if (c != t) v -= U[i * ldo + c] * U[axis * ldo + c];
            vals[cnt++] = v / nrm;
          }
          __syncwarp();
          cnt = 0;
          for (int i = lane; i < n; i += 32) U[i * ldo + t] = vals[cnt++];
          __syncwarp();
          break;
        }
      }
    }
  }
  if constexpr (!WIDE && CL == 1) {
    if (af.uw_mode) {
      // fused epilogue (ArrowFuse): this warp's Uk / Vk are in global memory
      // (L2) -- read them back through L2 and rotate the deferred bases
      __syncthreads();
      const int keep = nkeep;
      double* uwb = af.uw.p + b * af.uw.stride;
      if (af.uw_mode == 1) {
        // lane = column; eight rows of loads in flight before their stores
        for (int i0 = 0; i0 < n; i0 += 8) {
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            v[u] = (i0 + u < n && tid < keep) ? __ldcg(U + (i0 + u) * ldo + tid) : 0.0;
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (i0 + u < n && tid < af.uw.ld) uwb[(int64_t)(i0 + u) * af.uw.ld + tid] = v[u];
        }
      } else {
        warp_rotate(uwb, af.uw.ld, af.uw_rows, r, keep,
                    [&](int k, int c) { return __ldcg(U + k * ldo + c); }, true, 1.0);
      }
      warp_rotate(af.gw.p + b * af.gw.stride, af.gw.ld, af.gw_rows, r, keep,
                  [&](int k, int c) { return __ldcg(V + k * ldo + c); }, true, af.inj[b]);
      __syncwarp();
      VDefer zvd = af.zvd;
      if (zvd.G) {
        zvd.G += b * zvd.g_stride;
        if (zvd.Z) zvd.Z += b * zvd.z_stride;
      }
      warp_complete_zero(keep, SO, Mat{af.zU.p + b * af.zU.stride, 0, af.zU.ld}, af.zm,
                         Mat{af.zV.p + b * af.zV.stride, 0, af.zV.ld}, af.zn, zvd, S.delta);  // S.delta: free scratch by now
    }
  }
}

// One CTA (CL > 1: one cluster) per core.  List mode (!WIDE, af.fb_list):
// the cores arrow_cta_kernel handed back, *af.fb_count of them; the last
// CTA to finish resets the list for the next tick.
template <int kN, bool WIDE, int CL>
__global__ void __launch_bounds__(WIDE ? 512 : 32, 1) arrow_svd_kernel(int n, const double* __restrict__ core,
                                                       int64_t core_stride, int ldcore,
                                                       double* __restrict__ uk,
                                                       double* __restrict__ vk, int64_t out_stride,
                                                       int ldo, double* __restrict__ sv,
                                                       int64_t sv_stride, double* __restrict__ s_out,
                                                       int64_t s_out_stride, int nkeep,
                                                       const int* __restrict__ gate,
                                                       ArrowFuse af) {
  griddep_launch_dependents();
  griddep_wait();
  if (gate && *gate) return;
  const bool list = !WIDE && CL == 1 && af.fb_list;
  const int cnt = list ? *reinterpret_cast<volatile int*>(af.fb_count) : (int)(gridDim.x / CL);
  const int step = list ? (int)gridDim.x : cnt;
  // one call site (the body is inlined once)
  for (int idx = blockIdx.x / CL; idx < cnt; idx += step)
    arrow_body<kN, WIDE, CL>(list ? af.fb_list[idx] : idx, n, core, core_stride, ldcore, uk, vk,
                             out_stride, ldo, sv, sv_stride, s_out, s_out_stride, nkeep, af);
  if (list) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(af.fb_done, 1) == (int)gridDim.x - 1) {
        *af.fb_count = 0;
        *af.fb_done = 0;
        __threadfence();
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Append core of a batched k <= 32 stream (s = r + 1 <= 33) on one CTA of
// five warps: the same secular-equation solution as arrow_body (roots by the
// two-pole rational iteration with bisection safeguard, Loewner zhat,
// vectors from zhat, the reference's sort and snap), with four threads per
// root / Loewner product / vector (the lanes of a quad split the poles and
// combine their partial sums with an xor butterfly, so the quad's branch
// decisions agree bit for bit) instead of one thread, Uk / Vk kept in shared
// memory, and the fused epilogue (W <- [W 0; 0 1] Uk, Gv <- [Gv 0; 0 1/rho]
// Vk on DMMA) spread over the five warps' row groups.  Cores that need
// deflation (a tiny z entry, coincident poles), or with a dead singular
// value, are handed to the one-warp kernel (list mode) untouched.
#ifdef ISVD_R1_TRACE
#define AC_MARK(k)                                                   \
  do {                                                               \
    if (threadIdx.x == 0 && b < 4096) g_r1_trace[b][k] = clock64();  \
  } while (0)
#else
#define AC_MARK(k) \
  do {             \
  } while (0)
#endif
constexpr int kACThreads = 160;
constexpr int kACN = 40;   // root capacity (one quad each)
constexpr int kACLd = 36;  // Uk / Vk tile pitch

struct ArrowCtaSmem {
  double Uk[33 * kACLd];
  double Vk[33 * kACLd];
  double d[kACN], kd[kACN], kz[kACN], kz2[kACN], mu[kACN], sig[kACN], zhat[kACN];
  int kcol[kACN], org[kACN], pos[kACN];
  double wmax[8];
};

__device__ __forceinline__ void arrow_cta_body(
    int n, const double* __restrict__ core, int64_t core_stride, int ldcore,
    double* __restrict__ uk, double* __restrict__ vk, int64_t out_stride, int ldo,
    double* __restrict__ sv, int64_t sv_stride, double* __restrict__ s_out, int64_t s_out_stride,
    int nkeep, const int* __restrict__ gate, const ArrowFuse& af, int& done_old) {
  if (gate && *gate) return;
  extern __shared__ __align__(16) unsigned char ac_raw[];
  ArrowCtaSmem& S = *reinterpret_cast<ArrowCtaSmem*>(ac_raw);
  const int b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int quad = tid >> 2, ql = tid & 3;
  const unsigned qmask = 0xFu << (lane & 28);
  const int r = n - 1;
  const double eps = 2.220446049250313e-16;
  const double* K = core + b * core_stride;
  auto qsum = [&](double v) {
    v += __shfl_xor_sync(qmask, v, 1);
    return v + __shfl_xor_sync(qmask, v, 2);
  };
  // the epilogue's operands (W, Gv) start moving into L2 while the core is solved
  if (tid == 0 && af.uw_mode == 2 && af.uw_rows > 0)
    bulk_prefetch_l2(af.uw.p + b * af.uw.stride, (uint32_t)(af.uw_rows * af.uw.ld * sizeof(double)));
  if (tid == 32 && af.gw_rows > 0)
    bulk_prefetch_l2(af.gw.p + b * af.gw.stride, (uint32_t)(af.gw_rows * af.gw.ld * sizeof(double)));
  AC_MARK(0);
  // ---- zero the tiles (rows / columns beyond the core feed the DMMA epilogue)
  for (int i = tid; i < 33 * kACLd; i += kACThreads) {
    S.Uk[i] = 0.0;
    S.Vk[i] = 0.0;
  }
  // ---- load and scale
  double mx = 0.0, dv = 0.0, zv = 0.0;
  if (tid < n) {
    dv = tid < r ? fabs(K[tid * ldcore + tid]) : 0.0;
    zv = K[r * ldcore + tid];
    mx = fmax(dv, fabs(zv));
  }
  mx = warp_max(mx);
  if (lane == 0) S.wmax[warp] = mx;
  __syncthreads();
  double scale = 0.0;
  for (int w = 0; w < kACThreads / 32; ++w) scale = fmax(scale, S.wmax[w]);
  scale = scale > 0.0 ? scale : 1.0;
  if (tid < n) {
    const double rs = 1.0 / scale;
    dv *= rs;
    zv *= rs;
    S.d[tid] = dv;
  }
  __syncthreads();
  AC_MARK(1);
  // ---- deflation check.  The poles are the installed singular values,
  // sorted descending, plus the rho column's zero: without deflation (every
  // |z| > tol, consecutive poles more than tol apart -- which also means
  // strictly sorted) the ascending order is column r, then r - 1, ..., 0.
  // Anything else (deflation, or unsorted poles) goes to the one-warp kernel.
  {
    const double tol = 8.0 * eps;
    bool need = false;
    if (tid < n) {
      need = fabs(zv) <= tol;
      if (tid < r) need |= !(dv - S.d[tid + 1] > tol);  // S.d[r] = 0
      const int pk = tid == r ? 0 : r - tid;
      S.kcol[pk] = tid;
      S.kd[pk] = dv;
      S.kz[pk] = zv;
      S.kz2[pk] = zv * zv;
    }
    if (__syncthreads_or(need)) {
      if (tid == 0) {
        af.fb_list[atomicAdd(af.fb_count, 1)] = b;
        done_old = fb_arrive(af.fb_fast_done, true);
      }
      return;
    }
  }
  AC_MARK(2);
  const int N = n;
  // ---- roots: quad i solves for sigma_i in (kd[i], kd[i+1]) (the last beyond kd[N-1]).
  // The first evaluation is at the interval midpoint (origin kd[i]); its sign
  // picks the origin (the nearer pole) and the half-interval, and its terms
  // already feed the first rational-model step (no separate bracketing pass).
  if (quad < N) {
    const int i = quad;
    const double di = S.kd[i];
    const double dn = i < N - 1 ? S.kd[i + 1] : 0.0;
    const double sm = 0.5 * (di + dn);
    const double mum = (sm - di) * (sm + di);
    int o = i;
    double dorg = di, lo, hi, x, Di = 0.0, Dn = 0.0;
    bool first = i < N - 1;
    if (first) {
      lo = 0.0;
      hi = mum;
      x = mum;
    } else {
      double zz = 0.0;
      for (int j = ql; j < N; j += 4) zz += S.kz2[j];
      lo = 0.0;
      hi = qsum(zz);
      x = 0.5 * (lo + hi);
    }
    int iters = 0;
    for (int it = 0; it < 80; ++it) {
      ++iters;
      // x lies strictly between poles i and i + 1, so the terms of the
      // poles below (j <= i) are negative and the others positive: the sign
      // of w sorts them into psi / phi (selects instead of predicated pairs
      // of FP64 instructions), and sum |w| = phi - psi
      double psi = 0.0, dpsi = 0.0, phi = 0.0, dphi = 0.0;
      for (int j = ql; j < N; j += 4) {
        const double dj = S.kd[j];
        const double t = frcp((dj - dorg) * (dj + dorg) - x);
        const double w = S.kz2[j] * t;
        const bool below = __double2hiint(w) < 0;
        const double wl = below ? w : 0.0, wu = below ? 0.0 : w;
        psi += wl;
        dpsi = fma(wl, t, dpsi);
        phi += wu;
        dphi = fma(wu, t, dphi);
      }
      psi = qsum(psi);
      dpsi = qsum(dpsi);
      phi = qsum(phi);
      dphi = qsum(dphi);
      const double aps = phi - psi;
      // identical in the four lanes from here on (xor-reduced inputs)
      const double g = 1.0 + psi + phi;
      if (first) {
        first = false;
        if (!(g > 0.0)) {  // root above the midpoint: origin at kd[i+1]
          o = i + 1;
          dorg = dn;
          lo = (sm - dn) * (sm + dn);
          hi = 0.0;
          x = lo;
        }
        Di = (di - dorg) * (di + dorg);
        Dn = (dn - dorg) * (dn + dorg);
      } else if (g < 0.0) {
        lo = x;
      } else {
        hi = x;
      }
      if (fabs(g) <= 4.0 * eps * (1.0 + aps) * N || !(g == g)) break;
      const double xn = secular_model_step(i == N - 1, x, psi, dpsi, phi, dphi, Di, Dn, lo, hi);
      if (fabs(xn - x) <= 2.0 * eps * fmax(fabs(xn), 1e-300) ||
          hi - lo <= 2.0 * eps * fmax(fabs(lo), fabs(hi))) {
        x = xn;
        break;
      }
      x = xn;
    }
#ifdef ISVD_ARROW_STATS
    if (ql == 0) {
      atomicAdd(&g_arrow_counters[0], 1ull);
      atomicAdd(&g_arrow_counters[1], (unsigned long long)iters);
    }
#endif
    if (ql == 0) {
      S.org[i] = o;
      S.mu[i] = x;
      S.sig[i] = sqrt(dorg * dorg + x);
    }
  }
  __syncthreads();
  AC_MARK(3);
  // ---- Loewner: zhat_j^2 = prod_k (sigma_k^2 - d_j^2) / prod_{k != j} (d_k^2 - d_j^2)
  if (quad < N) {
    const int j = quad;
    const double dj = S.kd[j];
    auto sdiff = [&](int k) {
      const double dk = S.kd[S.org[k]];
      return S.mu[k] - (dj - dk) * (dj + dk);
    };
    double acc = 1.0;
    for (int k = ql; k < N - 1; k += 4) {
      const double dk = k < j ? S.kd[k] : S.kd[k + 1];
      acc *= sdiff(k) * frcp((dk - dj) * (dk + dj));
    }
    acc *= __shfl_xor_sync(qmask, acc, 1);
    acc *= __shfl_xor_sync(qmask, acc, 2);
    acc *= sdiff(N - 1);
    if (ql == 0) S.zhat[j] = copysign(sqrt(fmax(acc, 0.0)), S.kz[j]);
  }
  // ---- sorted output positions: descending sigma, ties by index; sigma_max.
  // Strict interlacing (kd_i < sigma_i < kd_{i+1}) makes the roots ascending,
  // so position N - 1 - t unless rounding broke the order (then the ranks).
  bool unsorted = false;
  if (tid < n - 1) unsorted = !(S.sig[tid] < S.sig[tid + 1]);
  if (__syncthreads_or(unsorted)) {
    double m1 = 0.0;
    if (tid < n) {
      const double st = S.sig[tid];
      int rank = 0;
      for (int e = 0; e < n; ++e) {
        const double se = S.sig[e];
        rank += (se > st) || (se == st && e < tid);
      }
      S.pos[tid] = rank;
      m1 = st;
    }
    m1 = warp_max(m1);
    if (lane == 0) S.wmax[warp] = m1;
  } else if (tid < n) {
    S.pos[tid] = n - 1 - tid;
    if (tid == n - 1)
      for (int w = 0; w < kACThreads / 32; ++w) S.wmax[w] = S.sig[n - 1];
  }
  __syncthreads();
  double smax = 0.0;
  for (int w = 0; w < kACThreads / 32; ++w) smax = fmax(smax, S.wmax[w]);
  AC_MARK(4);
  // ---- vectors into the shared tiles (quad per root)
  bool dead = false;
  if (quad < N) {
    const int t = quad;
    const int pc = S.pos[t];
    const double dorg = S.kd[S.org[t]];
    const double mu = S.mu[t];
    double nv = 0.0, nu = 0.0;
    for (int j = ql; j < N; j += 4) {
      const double dj = S.kd[j];
      const double vj = S.zhat[j] * frcp((dj - dorg) * (dj + dorg) - mu);
      nv = fma(vj, vj, nv);
      nu = fma(dj * vj, dj * vj, nu);
    }
    nv = qsum(nv);
    nu = 1.0 + qsum(nu);  // the z-row entry of u is -1
    const double iv = rsqrt(nv), iu = rsqrt(nu);
    const double sg = S.sig[t];
    dead = !(sg > 0.0) || sg < kZeroSvRtol * smax;
    for (int j = ql; j < N; j += 4) {
      const double dj = S.kd[j];
      const double vj = S.zhat[j] * frcp((dj - dorg) * (dj + dorg) - mu);
      const int row = S.kcol[j];
      S.Vk[row * kACLd + pc] = vj * iv;
      if (row != r) S.Uk[row * kACLd + pc] = dj * vj * iu;
    }
    if (ql == 0) S.Uk[r * kACLd + pc] = -iu;
  }
  if (__syncthreads_or(dead)) {
    if (tid == 0) {
      af.fb_list[atomicAdd(af.fb_count, 1)] = b;
      done_old = fb_arrive(af.fb_fast_done, true);
    }
    return;
  }
  if (tid == 0) done_old = fb_arrive(af.fb_fast_done, false);  // this core stays here
  AC_MARK(5);
  // install sigma; columns >= keep of the tiles out of the rotation
  const int keep = nkeep;
  if (tid < n) {
    const int pc = S.pos[tid];
    const double v = S.sig[tid] * scale;
    sv[b * sv_stride + pc] = v;
    if (s_out && pc < keep) s_out[b * s_out_stride + pc] = v;
  }
  for (int idx = tid; idx < n * 32; idx += kACThreads) {
    const int i = idx >> 5, cc = idx & 31;
    if (cc >= keep) {
      S.Uk[i * kACLd + cc] = 0.0;
      S.Vk[i * kACLd + cc] = 0.0;
    }
  }
  __syncthreads();
  AC_MARK(6);
  if (!af.uw_mode) {
    // unfused (single streams): the core's U / V to uk / vk for the
    // rotation launch (every column; those >= keep are zero, as the
    // rotation never reads them)
    double* U = uk + b * out_stride;
    double* V = vk + b * out_stride;
    for (int idx = tid; idx < n * n; idx += kACThreads) {
      const int i = idx / n, cc = idx % n;
      U[i * ldo + cc] = S.Uk[i * kACLd + cc];
      V[i * ldo + cc] = S.Vk[i * kACLd + cc];
    }
    return;
  }
  // ---- fused epilogue: W <- [W 0; 0 1] Uk[:, :keep], Gv <- [Gv 0; 0 1/rho] Vk[:, :keep]
  double* uwb = af.uw.p + b * af.uw.stride;
  double* gwb = af.gw.p + b * af.gw.stride;
  const int nwg = af.uw_mode == 2 ? (af.uw_rows + 7) / 8 : 0;
  const int ngg = (af.gw_rows + 7) / 8;
  const int g = lane >> 2, q = lane & 3;
  // (the next row group's operand is loaded before the current group's DMMAs)
  auto load_item = [&](int item, double (&a)[8]) {
    const bool isw = item < nwg;
    const double* X = isw ? uwb : gwb;
    const int ld = isw ? af.uw.ld : af.gw.ld;
    const int rows = isw ? af.uw_rows : af.gw_rows;
    const int row = 8 * (isw ? item : item - nwg) + g;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const int k = kk * 4 + q;
      a[kk] = (row < rows && k < r) ? X[(int64_t)row * ld + k] : 0.0;
    }
  };
  double a[8];
  if (warp < nwg + ngg) load_item(warp, a);
  for (int item = warp; item < nwg + ngg; item += kACThreads / 32) {
    const bool isw = item < nwg;
    double* X = isw ? uwb : gwb;
    const int ld = isw ? af.uw.ld : af.gw.ld;
    const int rows = isw ? af.uw_rows : af.gw_rows;
    const double* Q = isw ? S.Uk : S.Vk;
    const int row = 8 * (isw ? item : item - nwg) + g;
    double an[8];
    const int nxt = item + kACThreads / 32;
    if (nxt < nwg + ngg) load_item(nxt, an);
    double d[4][2];
#pragma unroll
    for (int nn = 0; nn < 4; ++nn) d[nn][0] = d[nn][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk)
#pragma unroll
      for (int nn = 0; nn < 4; ++nn)
        dmma_8x8x4(d[nn][0], d[nn][1], a[kk], Q[(kk * 4 + q) * kACLd + nn * 8 + g]);
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
  // new rows: W[uw_rows] = Uk[r, :keep] (mode 2) or W = Uk[:, :keep] (mode 1);
  // Gv[gw_rows] = (1/rho) Vk[r, :keep]
  if (af.uw_mode == 1) {
    for (int idx = tid; idx < n * af.uw.ld; idx += kACThreads) {
      const int i = idx / af.uw.ld, cc = idx % af.uw.ld;
      uwb[(int64_t)i * af.uw.ld + cc] = cc < 32 ? S.Uk[i * kACLd + cc] : 0.0;
    }
  } else if (tid < af.uw.ld) {
    uwb[(int64_t)af.uw_rows * af.uw.ld + tid] = tid < 32 ? S.Uk[r * kACLd + tid] : 0.0;
  }
  if (tid >= 64 && tid - 64 < af.gw.ld) {
    const int cc = tid - 64;
    gwb[(int64_t)af.gw_rows * af.gw.ld + cc] = cc < 32 ? af.inj[b] * S.Vk[r * kACLd + cc] : 0.0;
  }
#ifdef ISVD_R1_TRACE
  __syncthreads();
#endif
  AC_MARK(7);
}

// The CTA whose decision completes the count (fb_arrive) hands the cores on
// the fallback list (if any) to the one-warp kernel by a device-side tail
// launch, which starts when this grid has completed (no host launch per tick).
__global__ void __launch_bounds__(kACThreads, 6) arrow_cta_kernel(
    int n, const double* __restrict__ core, int64_t core_stride, int ldcore,
    double* __restrict__ uk, double* __restrict__ vk, int64_t out_stride, int ldo,
    double* __restrict__ sv, int64_t sv_stride, double* __restrict__ s_out, int64_t s_out_stride,
    int nkeep, const int* __restrict__ gate, ArrowFuse af) {
  int done_old = -1;
  arrow_cta_body(n, core, core_stride, ldcore, uk, vk, out_stride, ldo, sv, sv_stride, s_out,
                 s_out_stride, nkeep, gate, af, done_old);
  if (threadIdx.x == 0 && done_old == (int)gridDim.x - 1) {
    __threadfence();  // the other CTAs' list entries (each ordered before its count)
    *af.fb_fast_done = 0;
    const int cnt = *reinterpret_cast<volatile int*>(af.fb_count);
    if (cnt > 0)
      arrow_svd_kernel<40, false, 1><<<min(cnt, 4 * 148), 32, 0, cudaStreamTailLaunch>>>(
          n, core, core_stride, ldcore, uk, vk, out_stride, ldo, sv, sv_stride, s_out,
          s_out_stride, nkeep, gate, af);
  }
}

}  // namespace

int read_arrow_counters(int64_t* out4, int reset) {
  unsigned long long h[4];
  ISVD_CUDA(cudaMemcpyFromSymbol(h, g_arrow_counters, sizeof(h)));
  for (int i = 0; i < 4; ++i) out4[i] = (int64_t)h[i];
  if (reset) {
    unsigned long long z[4] = {0, 0, 0, 0};
    ISVD_CUDA(cudaMemcpyToSymbol(g_arrow_counters, z, sizeof(z)));
  }
  return ISVD_OK;
}

int launch_arrow_svd(int batch, int s, const double* core, int64_t core_stride, int ldcore,
                     double* uk, double* vk, int64_t out_stride, int ldo, double* sv,
                     int64_t sv_stride, cudaStream_t st, double* s_out, int64_t s_out_stride,
                     int nkeep, const ArrowFuse* af) {
  if (s < 1 || s > kN) {
    set_error("arrow core size out of range");
    return ISVD_EINVAL;
  }
  if (batch == 0) return ISVD_OK;
  if (s <= 33 && af && af->fb_list) {
    // k <= 32 streams: CTA per core (fused epilogue for the batched steady
    // state, else Uk / Vk out for the rotation launch); the one-warp kernel
    // takes the cores it hands back (deflation, dead sigma)
    arrow_cta_kernel<<<batch, kACThreads, sizeof(ArrowCtaSmem), st>>>(
        s, core, core_stride, ldcore, uk, vk, out_stride, ldo, sv, sv_stride, s_out, s_out_stride,
        nkeep, g_gate, *af);
  } else if (s <= 40) {
    // one warp per core: roots 32..39 (s = 33 is the k = 32 append core) are
    // solved warp-cooperatively after the one-root-per-lane pass
    ArrowFuse a1 = af ? *af : ArrowFuse{};
    a1.fb_list = nullptr;
    arrow_svd_kernel<40, false, 1><<<batch, 32, 0, st>>>(s, core, core_stride, ldcore, uk, vk,
                                                         out_stride, ldo, sv, sv_stride, s_out, s_out_stride, nkeep, g_gate,
                                                         a1);
  } else if (batch <= kClusterMaxBatch) {
    // few wide cores (config 5b: one 129 core per tick): a cluster per core
    cudaLaunchConfig_t cfg = {};
    bool wide16 = s > 128 && batch <= kClusterWideMaxBatch;
    if (wide16) {
      // a 16-CTA cluster of 512-thread CTAs must fit one GPC: checked once,
      // the portable 8-CTA cluster otherwise
      static int wide_ok = -1;
      if (wide_ok < 0) {
        wide_ok = 0;
        cudaLaunchConfig_t qc = {};
        qc.gridDim = dim3(kArrowClusterWide);
        qc.blockDim = dim3(512);
        cudaLaunchAttribute qa[1];
        qa[0].id = cudaLaunchAttributeClusterDimension;
        qa[0].val.clusterDim.x = kArrowClusterWide;
        qa[0].val.clusterDim.y = 1;
        qa[0].val.clusterDim.z = 1;
        qc.attrs = qa;
        qc.numAttrs = 1;
        int nclusters = 0;
        if (cudaFuncSetAttribute(arrow_svd_kernel<136, true, kArrowClusterWide>,
                                 cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess &&
            cudaFuncSetAttribute(arrow_svd_kernel<kN, true, kArrowClusterWide>,
                                 cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess &&
            cudaOccupancyMaxActiveClusters(&nclusters, arrow_svd_kernel<kN, true, kArrowClusterWide>,
                                           &qc) == cudaSuccess &&
            nclusters >= 1)
          wide_ok = 1;
        cudaGetLastError();
      }
      wide16 = wide_ok == 1;
    }
    const int clsz = wide16 ? kArrowClusterWide : kArrowCluster;
    cfg.gridDim = dim3(batch * clsz);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = clsz;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    cudaError_t e;
    if (wide16) {
      if (s <= 136)
        e = cudaLaunchKernelEx(&cfg, arrow_svd_kernel<136, true, kArrowClusterWide>, s, core,
                               core_stride, ldcore, uk, vk, out_stride, ldo, sv, sv_stride, s_out, s_out_stride, nkeep, g_gate, ArrowFuse{});
      else
        e = cudaLaunchKernelEx(&cfg, arrow_svd_kernel<kN, true, kArrowClusterWide>, s, core,
                               core_stride, ldcore, uk, vk, out_stride, ldo, sv, sv_stride, s_out, s_out_stride, nkeep, g_gate, ArrowFuse{});
    } else
    if (s <= 72)
      e = cudaLaunchKernelEx(&cfg, arrow_svd_kernel<72, true, kArrowCluster>, s, core, core_stride,
                             ldcore, uk, vk, out_stride, ldo, sv, sv_stride, s_out, s_out_stride, nkeep, g_gate, ArrowFuse{});
    else if (s <= 136)
      e = cudaLaunchKernelEx(&cfg, arrow_svd_kernel<136, true, kArrowCluster>, s, core,
                             core_stride, ldcore, uk, vk, out_stride, ldo, sv, sv_stride, s_out, s_out_stride, nkeep, g_gate, ArrowFuse{});
    else
      e = cudaLaunchKernelEx(&cfg, arrow_svd_kernel<kN, true, kArrowCluster>, s, core, core_stride,
                             ldcore, uk, vk, out_stride, ldo, sv, sv_stride, s_out, s_out_stride, nkeep, g_gate, ArrowFuse{});
    ISVD_CUDA(e);
  } else if (s <= 72) {
    arrow_svd_kernel<72, true, 1><<<batch, 512, 0, st>>>(s, core, core_stride, ldcore, uk, vk,
                                                         out_stride, ldo, sv, sv_stride, s_out, s_out_stride, nkeep, g_gate, ArrowFuse{});
  } else if (s <= 136) {
    arrow_svd_kernel<136, true, 1><<<batch, 512, 0, st>>>(s, core, core_stride, ldcore, uk, vk,
                                                          out_stride, ldo, sv, sv_stride, s_out, s_out_stride, nkeep, g_gate, ArrowFuse{});
  } else {
    arrow_svd_kernel<kN, true, 1><<<batch, 512, 0, st>>>(s, core, core_stride, ldcore, uk, vk,
                                                         out_stride, ldo, sv, sv_stride, s_out, s_out_stride, nkeep, g_gate, ArrowFuse{});
  }
  ISVD_LAUNCHED();
  return ISVD_OK;
}

}  // namespace isvd
