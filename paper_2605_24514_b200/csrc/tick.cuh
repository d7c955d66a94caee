#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace isvd {

struct Allreducer;  // shard.cuh

// Strided view of B per-stream matrices: X[b] = base + b*stride, row pitch ld.
struct Mat {
  double* p;
  int64_t stride;
  int ld;
};

// K1 (+ core build, K9 tracked-matrix write, N update) for appends.
// F[b] (rows x r, row-major pitch F.ld) is the factor whose row space the
// appended vector x[b] (length rows) is projected on: V for a row append,
// U for a column append (engine.py:137-139 transpose trick).
// Deferred right basis (engine.cu): V_eff = [F(:, :fw) | Z^T] G with G
// (gr = fw + nz rows, r columns, leading dimension ldg, g_stride per stream)
// and Z holding nz appended residuals (Z[t * ldz + c], z_stride per stream).
// nz = 0 and fw = r is the rank-1-only deferral V_eff = V G.
constexpr int kVWin = 8;             // residual columns per deferred window
// rows of G the k <= 32 kernels handle (a multiple of 8: the materialising
// rotation's K dimension is rounded up to 8)
constexpr int kGMaxRows = (32 + kVWin + 7) / 8 * 8;
struct VDefer {
  const double* G = nullptr;
  int64_t g_stride = 0;
  int ldg = 0;
  int fw = 0, nz = 0;
  const double* Z = nullptr;
  int64_t z_stride = 0;
  int ldz = 0;
};

// K1.  With vd.G set, the projection goes through the deferred basis and z
// (the unnormalised residual) is written to z (the next Z slot when nz is
// being appended).
int launch_project_append(int batch, int rows, int r, Mat F, const double* x, int64_t x_stride,
                          const double* s, int lds, double tol, double* core, int64_t core_stride,
                          int ldcore, double* z, int64_t z_stride, double* inj_scale,
                          double* rho_out, double* xnorm_out, double* A, int64_t a_stride,
                          int64_t a_off, int64_t a_step, double* N, cudaStream_t st,
                          const struct Allreducer* ar = nullptr, int arrow_only = 0,
                          const VDefer* vd = nullptr, double* ring = nullptr,
                          int64_t ring_stride = 0);
// Whether launch_project_append accepts a deferred right basis G (F_eff =
// F G) for this shape (the one-CTA-per-stream path does; the split and
// cluster paths for few long streams do not).
bool project_append_takes_g(int batch, int rows, int r);
bool project_append_gateable(int batch, int rows, int r);

// Deferred left basis: while active, the true U is
// [Ub 0; 0 I] . W where Ub = the first m_base rows of the U buffer (width
// r_base) and W has r_base + (rows appended since) rows.
struct LazyBasis {
  int active;
  int m_base, r_base;
  Mat W;
};

// Row-sharded rank-1 pieces (B = 1, see tick.cu): gather U[i,:] / A[i,j] on
// the owning shard into out (r + 1), then the replicated core from out.
int launch_rank1_gather(int r, Mat U, int64_t i, int64_t j, const double* A, int lda,
                        struct LazyBasis lz, double* out, cudaStream_t st);
int launch_rank1_vec_build(int r, const double* vec, Mat V, const double* s, int64_t j, double d,
                           double* core, int ldcore, double* N, double* Aij, cudaStream_t st);

// K6: rank-1 core K = diag(s) + delta U[i,:]^T V[j,:] plus the tracked entry
// update A[i,j] += delta and N += 2 delta a_old + delta^2 (engine.py:162-166).
int launch_rank1_build(int batch, int r, Mat U, Mat V, const double* s, int lds,
                       const int64_t* ii, const int64_t* jj, const double* delta, double* core,
                       int64_t core_stride, int ldcore, double* A, int64_t a_stride, int lda,
                       double* N, LazyBasis lz, cudaStream_t st);

// One rotation job: X[b][0:rows, 0:keep] = X[b][0:rows, 0:r] . Q[b][0:r, 0:keep]
//   (+ z[b][i] * inj_scale[b] * Q[b][r, c])      if z != nullptr
//   and X[b][rows, 0:keep] = Q[b][r, 0:keep]       if new_row
// in place (each output row depends only on the same input row).
struct RotJob {
  Mat X;
  int rows;
  const double* Q;
  int64_t q_stride;
  int ldq;
  const double* z;
  int64_t z_stride;
  const double* inj_scale;
  int new_row;
  // optional deferred right basis: Q[:r] is replaced by G[:r, :r] Q[:r]
  // (rotate_reg_kernel only: KP <= 32, keep <= 32)
  const double* G = nullptr;
  int64_t g_stride = 0;
  int ldg = 0;
  // new_row: the appended row is nr_scale[b] * Q[r, :] (1 when null)
  const double* nr_scale = nullptr;
  // optional second source of the left operand (rotate_reg_kernel): columns
  // k >= zfw of X are read from zs[(k - zfw) * ldzs + row] (the deferred
  // residuals Z of a VDefer, materialised by V <- [V | Z^T] G)
  const double* zs = nullptr;
  int64_t zs_stride = 0;
  int ldzs = 0;
  int zfw = 0;
};

// K3/K4: both factor rotations of a tick in one launch (FP64 DMMA).
// Zero-sigma completion (_install, engine.py:59-70) fused into the rotation:
// the last CTA of each stream to finish its rows completes U / V columns of
// zero singular values (complete_zero_kernel's work).  counter: B unsigned
// ints, zero between launches (the last CTA resets its stream's entry).
struct ZeroFix {
  const double* s = nullptr;
  int lds = 0, w = 0;
  Mat U{};
  int m = 0;
  Mat V{};
  int n = 0;
  unsigned* counter = nullptr;
  // V deferred (vd.G set): V is V_base; a stream that needs a completion
  // first materialises V_eff into V and resets its G to [I; 0]
  VDefer vd{};
};
// zf (optional): fuse the completion when the launch goes to
// rotate_reg_kernel; *fused tells the caller whether it did (else the caller
// launches complete_zero itself).
int launch_rotate(int batch, int r, int keep, const RotJob& j0, const RotJob* j1, cudaStream_t st,
                  const ZeroFix* zf = nullptr, bool* fused = nullptr);

// engine.py:59-70 -- repair factor columns paired with exact-zero singular
// values (no-op launch when none are zero).
int launch_complete_zero(int batch, int w, const double* s, int lds, Mat U, int m, Mat V, int n,
                         cudaStream_t st, const VDefer* vd = nullptr);

// linalg.py:63-75 -- sign canonicalisation of (U, V) per stream.
int launch_canonicalize(int batch, int w, Mat U, int m, Mat V, int n, cudaStream_t st);
// Row-sharded K5 (B = 1): post writes this shard's per-column candidates
// (max |u|, global row, sign) into slot `rank` of pk (world x w x 3, zeroed
// elsewhere); after a cross-shard sum, apply picks the winners and flips.
int launch_canon_shard_post(int w, Mat U, int m, int64_t row0, int rank, int world, double* pk,
                            cudaStream_t st);
int launch_canon_shard_apply(int w, Mat U, int m, Mat V, int n, int world, const double* pk,
                             cudaStream_t st);

// Copy helpers.
// out[0:B] = N, out[B:2B] = rho, out[2B:3B] = xnorm for streams [b0, b0+nb)
// (out: a device-mapped pinned host buffer)
int launch_scalars_out(int b0, int nb, int B, const double* N, const double* rho,
                       const double* xnorm, double* out, cudaStream_t st);
// X[:rows, :cols] <- I per stream
int launch_eye(int batch, Mat X, int rows, int cols, cudaStream_t st);
int launch_copy_rows(int batch, int rows, int cols, const double* src, int64_t src_stride,
                     int ld_src, double* dst, int64_t dst_stride, int ld_dst, cudaStream_t st);
int launch_zero(double* p, size_t n, cudaStream_t st);
int launch_transpose_square(int batch, int s, double* a, cudaStream_t st);
int launch_sumsq(int batch, int rows, int cols, const double* a, int64_t a_stride, int lda,
                 double* out, cudaStream_t st);
int launch_check_finite(size_t n, const double* p, int* flag, cudaStream_t st);
int launch_stage_rank1(int B, const int64_t* i, const int64_t* j, const double* d, int64_t* si,
                       int64_t* sj, double* sd, int64_t m, int64_t n, int* flag, cudaStream_t st);
int read_k1_trace(int64_t* out, int n);

}  // namespace isvd
