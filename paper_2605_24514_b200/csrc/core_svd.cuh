#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace isvd {

constexpr int kCoreMaxS = 160;   // largest core: k_max + 1 (k <= 159)
constexpr int kSmemMaxS = 112;   // G and V both in shared memory up to here

size_t core_svd_smem_bytes(int s, bool v_in_smem);
int read_debug_counters(int64_t* out, int reset);
int read_r1_trace(int64_t* out, int n);
// [0] secular roots solved, [1] their iterations, [2] cores, [3] cores that
// took the sequential deflation pass (arrow_svd.cu)
int read_arrow_counters(int64_t* out4, int reset);

// Batched core SVD.  core[b] is s x s row-major at core + b*core_stride with
// row pitch ldcore.  Outputs uk[b], vk[b] (row-major s x s, pitch ldo, the
// columns are the singular vectors), sv[b] (s values).  `active` (optional)
// skips streams whose flag is 0.  vscratch: batch * s * (s|1) doubles, needed
// when s > kSmemMaxS.
int launch_core_svd(int batch, int s, const double* core, int64_t core_stride, int ldcore,
                    double* uk, double* vk, int64_t out_stride, int ldo, double* sv,
                    int64_t sv_stride, double* vscratch, const int* active, cudaStream_t st);

}  // namespace isvd

#include "tick.cuh"
namespace isvd {
// Rank-1 core description for the fused build + Jacobi (K6 + K2b) kernel.
struct Rank1Core {
  Mat U, V;
  const double* s = nullptr;
  int lds = 0;
  const int64_t* ii = nullptr;
  const int64_t* jj = nullptr;
  const double* delta = nullptr;
  double* A = nullptr;
  int64_t a_stride = 0;
  int lda = 0;
  double* N = nullptr;
  LazyBasis lz{};
  // Deferred right basis (tick.cuh VDefer): V_eff = [V | Z^T] G when vd.G
  VDefer vd{};
  // optional read-back ring row of this tick: (N, rho, xnorm) at b,
  // ring_stride + b, 2 ring_stride + b (rho / xnorm unchanged by the tick)
  double* ring = nullptr;
  int64_t ring_stride = 0;
  const double* rho = nullptr;
  const double* xnorm = nullptr;
  // Fused rotations (one warp per stream, warp_rot.cuh; the steady state of
  // a batched k <= 32 stream): uw_mode 1 = the core's U becomes the new
  // deferred window uw (s rows), 2 = uw[0:uw_rows] <- uw Uk; gw_rows > 0:
  // gw[0:gw_rows] <- gw Vk (the deferred right basis; else Vk goes to
  // vk_out).  Then the engine-level zero-sigma completion (engine.py:59-70)
  // on (zU, zm rows) and (zV, zn rows) with zvd the deferred right basis.
  // The core's U / V are not written to uk / vk.
  int uw_mode = 0;
  Mat uw{};
  int uw_rows = 0;
  Mat gw{};
  int gw_rows = 0;
  Mat zU{}, zV{};
  int zm = 0, zn = 0;
  VDefer zvd{};
  // Optional separate destination for the core's right vectors (row-major,
  // vk_stride per stream, leading dimension ldvk) instead of vk/ldo
  double* vk_out = nullptr;
  int64_t vk_stride = 0;
  int ldvk = 0;
  // Fallback list (batch ints) and its count / completion counters (one int
  // each, zero between ticks): with fb_list set, a CTA-per-core structured
  // kernel factors the well-conditioned cores and the one-warp Jacobi the rest
  int* fb_list = nullptr;
  int* fb_count = nullptr;
  int* fb_done = nullptr;
  int* fb_fast_done = nullptr;  // CTA completion count of the fast kernel
};
// K = diag(s) + delta U[i,:]^T Vt[:,j]^T built in registers and factored by
// the warp Jacobi (s <= 32); also applies A[i,j] += delta and the N update.
int launch_rank1_core_svd32(int batch, int s, const Rank1Core& rc, double* uk, double* vk,
                            int64_t out_stride, int ldo, double* sv, int64_t sv_stride,
                            cudaStream_t st, double* s_out = nullptr, int64_t s_out_stride = 0);

// Secular-equation SVD of the Brand append core [[diag d, 0], [p, rho]]
// (arrow_svd.cu).  Same outputs and conventions as launch_core_svd.
// s_out (optional): the first nkeep singular values are also written there
// (the engine's s), replacing the separate install copy.
// Fused row-append epilogue of the one-warp arrow kernel (s <= 40): the
// deferred bases are rotated by the core's warp (warp_rot.cuh) --
// uw_mode 1: the core's U[:, :keep] becomes the new window uw (s rows);
// 2: uw <- [uw 0; 0 1] Uk[:, :keep] (uw_rows old rows); gw <- [gw 0; 0
// inj] Vk[:, :keep] (gw_rows old rows, inj = 1/rho per stream); then the
// engine-level zero-sigma completion on (zU, zm) / (zV, zn, zvd).  All Mats
// and pointers per batch (stride applied per stream).
struct ArrowFuse {
  int uw_mode = 0;
  Mat uw{};
  int uw_rows = 0;
  Mat gw{};
  int gw_rows = 0;
  const double* inj = nullptr;
  Mat zU{}, zV{};
  int zm = 0, zn = 0;
  VDefer zvd{};
  // fallback list (as Rank1Core): with fb_list set and s <= 33, a CTA-per-core
  // secular kernel takes the cores without deflation, the one-warp kernel the rest
  int* fb_list = nullptr;
  int* fb_count = nullptr;
  int* fb_done = nullptr;
  int* fb_fast_done = nullptr;  // CTA completion count of the CTA kernel
};
int launch_arrow_svd(int batch, int s, const double* core, int64_t core_stride, int ldcore,
                     double* uk, double* vk, int64_t out_stride, int ldo, double* sv,
                     int64_t sv_stride, cudaStream_t st, double* s_out = nullptr,
                     int64_t s_out_stride = 0, int nkeep = 0, const ArrowFuse* af = nullptr);
}  // namespace isvd
