/*
 * isvd.h -- C ABI of libisvd, the B200-native incremental-SVD engine.
 *
 * This is the drop-in boundary for the reference `svdstream` per-tick update
 * path (arxiv/paper_2605_24514).  All citations are relative to
 * /root/reference/pkg/src/svdstream/.
 *
 * Two layers, mirroring the reference's two boundaries:
 *
 *  1. Functional kernel entry points -- the `svdstream.backend` contract
 *     (backend.py:54-63): core_svd, row_append, rank_one.  Inputs are read,
 *     outputs are written to caller buffers; nothing is retained.
 *
 *  2. An engine handle -- the `SvdEngine` state machine (engine.py:73-217),
 *     holding B independent streams of identical shape ("batch") whose
 *     factors, tracked matrix and squared norm live in HBM.  B = 1 is the
 *     reference's single engine; B > 1 is the batched-stream workload.
 *
 * Conventions
 *  - Every entry point returns 0 on success, nonzero on failure; the message
 *    is available from isvd_last_error() (thread-local).  Argument errors the
 *    reference raises as ValueError return ISVD_EINVAL *before* any state is
 *    touched, so a rejected event leaves the engine unchanged
 *    (tests/test_engine.py:88-95).
 *  - Matrices are row-major float64.  `on_device` flags say whether a
 *    pointer is a device pointer (1) or host memory (0).
 *  - `stream` arguments are cudaStream_t passed as void*; 0 = legacy stream.
 *  - No CPU fallback exists: without a CUDA device every compute call fails
 *    with ISVD_ENODEV.
 */
#ifndef ISVD_H_
#define ISVD_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ISVD_OK 0
#define ISVD_EINVAL 1   /* invalid argument (reference: ValueError)        */
#define ISVD_ENODEV 2   /* no CUDA device / CUDA runtime failure            */
#define ISVD_ENOMEM 3   /* device allocation failed                         */
#define ISVD_ESTATE 4   /* operation not valid in the current engine state  */

/* Library / error reporting ------------------------------------------------ */
const char* isvd_last_error(void);
int isvd_version(void);
/* Number of kernel launches issued by this process so far (evidence counter
 * reported by bench.py as `gpu_launches`). */
int64_t isvd_launch_count(void);
/* Device profiling counters (out8[0] = Jacobi sweeps summed over cores,
 * out8[1] = cores factored by the warp Jacobi kernel, out8[2..5] = arrow
 * solver counters, out8[6] = simultaneous steps on the rank-1 fast path,
 * out8[7] = rank-1 cores finished on it); reset if nonzero. */
int isvd_debug_counters(int64_t* out8, int reset);
/* Diagnostics: per-core phase timestamps (SM clock) of the last rank-1 core
 * launch, recorded only by a library built with -DISVD_R1_TRACE (else all
 * zero): out[b * 10 + k], k = 0..9, for b < n (n <= 4096).  A negative n
 * reads the marks of the last projection (K1) launch for -n streams. */
int isvd_debug_trace(int64_t* out, int n);

/* 1. Functional kernels (backend.py:54-63) ---------------------------------- */

/* core_svd: batched full SVD of `batch` square s x s cores (row-major,
 * contiguous, stride s*s).  One-sided Jacobi + stable descending sort + snap
 * below 1e-12*s[0] + dead-column completion, as _kernels.pyx:82-109.
 * Outputs u (s x s), sv (s), vt (s x s) per core.  Device pointers. */
int isvd_core_svd(int batch, int s, const double* core, double* u, double* sv,
                  double* vt, void* stream);

/* row_append (_kernels_py.py:22-49, _kernels.pyx:112-187): u (m x r),
 * s (r), vt (r x n), x (n) -> u_out ((m+1) x keep), s_out (keep),
 * vt_out (keep x n), *rho.  Host pointers; synchronous. */
int isvd_row_append(int m, int r, int n, const double* u, const double* s,
                    const double* vt, const double* x, double tol, int keep,
                    double* u_out, double* s_out, double* vt_out, double* rho);

/* rank_one (_kernels_py.py:52-58, _kernels.pyx:190-237): projection rule
 * K = diag(s) + delta U[i,:]^T Vt[:,j]^T.  Host pointers; synchronous. */
int isvd_rank_one(int m, int r, int n, const double* u, const double* s,
                  const double* vt, int64_t i, int64_t j, double delta, int keep,
                  double* u_out, double* s_out, double* vt_out);

/* 2. Engine handle (engine.py:73-217) --------------------------------------- */

typedef struct isvd_engine isvd_engine;

/* Create B streams of shape m x n with work rank k (engine.py:76-94).
 * Capacities (rows, cols, rank) are hints; the engine grows by doubling.
 * Returns ISVD_EINVAL for k < 1, tol <= 0, empty shape. */
int isvd_engine_create(isvd_engine** out, int batch, int m, int n, int k,
                       double tol, int reortho_guard, int m_cap, int n_cap,
                       int k_cap, void* stream);
int isvd_engine_destroy(isvd_engine* e);

/* Row sharding of one tall stream over ranks (BASELINE config 5b, SURVEY.md
 * 8(e); north star: "U is row-sharded, with an NCCL allreduce of the
 * k-length projections and k x k Gram blocks").  Call after create (B = 1,
 * m = this rank's rows) and before init.  This rank holds global rows
 * [row0, row0 + m) of U and of the tracked matrix; the rank with
 * owns_appends = 1 (the last shard) also stores every appended row.  s, V
 * and the deferred-window W are replicated and updated identically on every
 * rank, so a row append needs no communication; `fn` is called (in the same
 * order on every rank) to sum `count` doubles of a device buffer in place
 * across ranks, ordered after the work already issued on `stream` and before
 * the work issued after it returns:
 *   init / refresh   n x n Gram, two w x w CholeskyQR Grams, ||A||^2
 *   column append    the projection U^T y (+ ||y||^2), then ||z||^2
 *   rank-1 update    the (owner's) row U[i, :] and A[i, j]
 *   metrics / signs  U Grams (k x k), ||A - U S V^T||^2, column-max packets
 * Observation calls (factors, metrics, set_reference, flush) are therefore
 * collective in this mode.  Not available: eager U rotation (set_lazy(0)),
 * the device oracle on the tracked matrix. */
typedef int (*isvd_allreduce_fn)(void* ctx, double* buf, int64_t count, void* stream);
int isvd_engine_set_shard(isvd_engine* e, int rank, int world, int64_t row0, int m_global,
                          int owns_appends, isvd_allreduce_fn fn, void* ctx);
/* row0, local rows, global rows (m_local = m_global when not sharded). */
int isvd_engine_shard_info(const isvd_engine* e, int64_t* row0, int* m_local, int* m_global);

/* Initialise from a0 (B x m x n, row-major per stream): copies the tracked
 * matrix, N0 = sum a0^2, factors = truncated_svd(a0, k) on the device
 * (engine.py:87-89, linalg.py:84-109).  Non-finite entries -> ISVD_EINVAL. */
int isvd_engine_init(isvd_engine* e, const double* a0, int on_device);

/* Events.  x: B x n (row append, engine.py:117-129); y: B x m (column
 * append, engine.py:131-147); i, j, delta: B each (rank-1 update,
 * engine.py:149-167).  Host inputs are validated (finite, in bounds) before
 * any device work; device inputs are trusted. */
int isvd_engine_row_append(isvd_engine* e, const double* x, int on_device);
int isvd_engine_col_append(isvd_engine* e, const double* y, int on_device);
int isvd_engine_rank_one(isvd_engine* e, const int64_t* i, const int64_t* j,
                         const double* delta, int on_device);

/* Maintenance: refresh (engine.py:171-176), set_reference (:178-180),
 * set_rank (:182-198). */
int isvd_engine_refresh(isvd_engine* e, int store_reference);
int isvd_engine_set_reference(isvd_engine* e);
int isvd_engine_set_rank(isvd_engine* e, int k_new);

/* Shape / scalar state. */
int isvd_engine_shape(const isvd_engine* e, int* batch, int* m, int* n,
                      int* rank, int* work_rank, int64_t* step);
int isvd_engine_has_reference(const isvd_engine* e, int* has_ref, int* ref_m,
                              int* ref_r);

/* Host copies (synchronous).  Factors are returned in canonical sign form
 * (linalg.py:63-75).  b = stream index.  u: m x r, s: r, v: n x r (V, i.e.
 * the transpose of the reference's vt; the host shim exposes vt = v.T). */
int isvd_engine_get_factors(isvd_engine* e, int b, double* u, double* s, double* v);
int isvd_engine_get_tracked(isvd_engine* e, int b, double* a);
int isvd_engine_get_reference(isvd_engine* e, int b, double* ref);
/* sq_norm: B values; last_residual / last_input_norm: B values each. */
/* Pipelined read of the per-step result: enqueue the copy of (sq_norm,
 * last_residual, last_input_norm) -- 3 x B doubles: [sq_norm | residual |
 * input norm] -- into `host` (pinned memory) and return at once; ticket
 * `slot` (0..7) completes with isvd_engine_scalars_wait.  Lets a host loop
 * issue steps t+1.. before step t's result lands.  After a tick whose
 * kernels wrote the read-back ring (the batched K1 / fused rank-1 paths) the
 * copy runs on a separate read-back stream once every stream group has
 * finished that tick; otherwise it is issued per group. */
int isvd_engine_scalars_async(isvd_engine* e, double* host, int slot);
int isvd_engine_scalars_wait(isvd_engine* e, int slot);
int isvd_engine_get_scalars(isvd_engine* e, double* sq_norm, double* last_residual,
                            double* last_input_norm);
/* Overwrite the factors / reference of stream b from host memory (test and
 * checkpoint hook; the reference tests mutate factors in place). */
int isvd_engine_set_factors(isvd_engine* e, int b, int r, const double* u,
                            const double* s, const double* v);
int isvd_engine_put_reference(isvd_engine* e, int b, int ref_m, int ref_r,
                              const double* ref);

/* Device views (no copy).  Pointers stay valid until the next event that
 * grows a capacity.  Leading dimensions are in elements.  U_dev and V_dev
 * hold stream b at offset b*stride.  NOTE: signs are lazy -- call
 * isvd_engine_canonicalize() first when the canonical form is required. */
int isvd_engine_device_views(isvd_engine* e, double** u, int64_t* u_stride, int* ldu,
                             double** v, int64_t* v_stride, int* ldv, double** s,
                             int* lds, double** a, int64_t* a_stride, int* lda);
int isvd_engine_canonicalize(isvd_engine* e);
/* The engine stream (cudaStream_t as void*).  Batches of >= 512 streams
 * run their ticks on stream groups that may run ahead of it; every entry
 * point other than the three event calls (and this one) first makes the
 * engine stream wait for them, so work enqueued on the returned stream after
 * a call of this function is ordered after all engine work so far. */
void* isvd_engine_stream(isvd_engine* e);
/* Every CUDA stream that may read a device-resident event payload (the
 * engine stream first, then the stream groups created so far), without
 * joining them.  Writes min(count, cap) handles to out; returns the count.
 * A caller passing device buffers to the event calls keeps them alive until
 * all of these streams pass the call (torch: Tensor.record_stream on each). */
int isvd_engine_streams(isvd_engine* e, void** out, int cap);
/* Waits for the engine's work.  Device-resident rank-1 payloads are checked
 * on the device (index in bounds, finite delta); a rejected entry is applied
 * as a no-op to its stream and this call (and get_scalars / get_factors)
 * then returns ISVD_EINVAL once. */
int isvd_engine_synchronize(isvd_engine* e);
/* Per-phase device timing (CUDA events on the engine stream around each
 * phase of every event): phase 0 = projection / rank-1 gather (K1/K6),
 * 1 = core SVD (K2), 2 = factor rotation (K3/K4), 3 = install.  phase_times
 * returns the summed milliseconds of the ticks recorded since the last call
 * and resets the record. */
int isvd_engine_set_timing(isvd_engine* e, int on);
/* Verification hook: 1 = factor append cores with the generic one-sided
 * Jacobi kernel (the reference's compiled algorithm), 0 (default) = the
 * secular-equation kernel for the broken-arrow core.  Both are exact SVDs;
 * the parity tests run both. */
int isvd_engine_set_append_solver(isvd_engine* e, int jacobi);
/* Deferred left-basis rotation, on by default: row
 * appends and rank-1 updates rotate a small W (U = [U_base 0; 0 I] W) and U
 * is materialised every lazy-window rows (isvd_engine_set_lazy_window) and
 * before any read of U.
 * set_lazy(0) rotates U eagerly every event (the reference's order of
 * operations); flush() materialises U now. */
int isvd_engine_set_lazy(isvd_engine* e, int on);
/* Rows appended per deferred window before U is materialised (default
 * ~sqrt(2 m) clamped to [32, 4096]); flushes first.  isvd_engine_lazy_window
 * returns the current value (-1 for a null handle). */
int isvd_engine_set_lazy_window(isvd_engine* e, int rows);
int isvd_engine_lazy_window(isvd_engine* e);
/* Deferred right-basis rotation: rank-1 updates rotate a small r x r G
 * (V = V_base G) instead of V; the next row append projects through G and
 * folds it into its own V rotation; flush() and every read of V materialise
 * it.  mode 0 = off, 1 = on for batches >= 64 streams with r <= 32 (default),
 * 2 = whenever the kernels support it (r <= 32, not row-sharded).  Flushes
 * first. */
int isvd_engine_set_vdefer(isvd_engine* e, int mode);
/* Stream groups: a batch of B streams is split into up to `groups` slices
 * (each >= 256 streams) issued on separate CUDA streams so one slice's
 * latency-bound core SVDs overlap another's HBM-bound passes (default 4). */
int isvd_engine_set_groups(isvd_engine* e, int groups);
/* Defect threshold of the optional re-orthonormalisation guard
 * (REORTHO_THRESHOLD, engine.py:30; default 1e-6). */
int isvd_engine_set_reortho_threshold(isvd_engine* e, double threshold);
/* Device-side checkpoint of the full engine state (factors, tracked matrix,
 * squared norms, shape, step; a deferred rotation is flushed first) and its
 * restore.  Used by bench.py to rerun the same ticks without a new init. */
int isvd_engine_snapshot(isvd_engine* e);
int isvd_engine_restore(isvd_engine* e);
int isvd_engine_flush(isvd_engine* e);
int isvd_engine_phase_times(isvd_engine* e, double* ms4, int64_t* ticks);

/* 3. Metrics (metrics.py:56-145, linalg.py:126-153) ------------------------- */

/* Per-stream frob_error = ||A - U diag(s) Vt||_F without materialising the
 * product (metrics.py:74-76).  out: B doubles (host). */
int isvd_engine_frob_error(isvd_engine* e, double* out);
/* Orthonormality defects ||U^T U - I||_F and ||V^T V - I||_F (linalg.py:126-130). */
int isvd_engine_ortho_defect(isvd_engine* e, double* du, double* dv);
/* Largest principal angle arccos(sigma_min(U^T Q)) against the stored
 * reference (which = 0) or an explicit basis q (B x m x r, host or device;
 * which = 1), linalg.py:133-153.  Returns -1 in out[b] when undefined
 * (no reference / shape mismatch -> reference returns None).  Raises
 * ISVD_EINVAL when either basis has defect > 1e-6 (linalg.py:148-150). */
int isvd_engine_angle(isvd_engine* e, int which, const double* q, int q_cols,
                      int on_device, double* out);

/* Per-tick risk of BASELINE config 3 (finance.py:326-371), for every stream:
 * cov = V diag(s^2) V^T / (t - 1) symmetrised (low_rank_covariance),
 * D = max(0, diag(A^T A) / (t - 1) - diag(cov)) over the mean-centred tracked
 * returns (the diagonal term BASELINE adds), and for each of the P
 * portfolios w (host, P x n): out[b][p] = {sqrt(w'cov w) (portfolio_vol),
 * sqrt(w'(cov + D) w), 2.3263478740408408 * that (99% Gaussian VaR, zero
 * mean), w'cov w}.  cov_out (B x n x n) and diag_out (B x n) may be NULL.
 * t = rows the covariance is estimated from (>= 2, else ISVD_EINVAL); a
 * quadratic form below -1e-10 is the reference's not-PSD ValueError. */
int isvd_engine_risk(isvd_engine* e, int t, const double* w, int P, double* cov_out,
                     double* diag_out, double* out);
/* low_rank_covariance (finance.py:326-335) of host factors: cov (n x n) =
 * V diag(s^2) V^T / (t - 1), symmetrised, computed by the same device kernel
 * (v is n x r row-major, i.e. Vt^T).  t >= 2 else ISVD_EINVAL. */
int isvd_low_rank_cov(int n, int r, const double* v, const double* s, int t, double* cov);

/* Dense thin SVD of B matrices (m x n each) on the device, in canonical
 * form (linalg.py:84-92).  Outputs: s (B x min(m,n)); u (B x m x w) and
 * vt (B x w x n) for the leading w = min(w_keep, min(m,n)) triplets; u/vt
 * may be NULL.  All pointers host; synchronous.  Used by compute_oracle. */
int isvd_dense_svd(int batch, int m, int n, const double* a, int w_keep, double* s,
                   double* u, double* vt);
/* Same, from the engine's tracked matrices (no host copy of A). */
int isvd_engine_oracle(isvd_engine* e, int w_keep, double* s, double* u);
/* Host-basis metrics on the device (linalg.py:126-153), host pointers,
 * synchronous.  ortho_defect: out[b] = ||Q_b^T Q_b - I||_F for B bases
 * (rows x w each).  principal_angle: largest principal angle between the
 * spans of q1 and q2 (rows x w each, w <= 160); ISVD_EINVAL if either basis
 * is not orthonormal to 1e-6. */
int isvd_ortho_defect(int batch, int rows, int w, const double* q, double* out);
int isvd_principal_angle(int rows, int w, const double* q1, const double* q2, double* out);

/* The two dense contractions on the FP64 tensor path (DMMA), device
 * pointers, row-major, asynchronous on `stream` (NULL = legacy stream).
 * gram: out (wa x wb) = xa(rows x wa, pitch lda)^T xb(rows x wb, pitch ldb);
 * xa == xb with equal shapes computes the symmetric Gram's upper tiles only.
 * gemm: c (rows x wc, pitch ldc) = x (rows x n, pitch ldx) q (n x wc, ldq).
 * These back the Gram/QR of the guard and metrics and the tall-matrix SVD
 * (init/refresh/oracle of configs 4 and 5b). */
int isvd_gram(int rows, int wa, int wb, const double* xa, int lda, const double* xb, int ldb,
              double* out, void* stream);
int isvd_gemm_tall(int rows, int n, int wc, const double* x, int ldx, const double* q, int ldq,
                   double* c, int ldc, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ISVD_H_ */
