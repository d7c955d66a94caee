// libisvd C ABI: functional kernels + engine handle (include/isvd.h).
//
// The engine mirrors SvdEngine (engine.py:73-217).  Device state per stream
// b (B streams of identical shape):
//   U  [m_cap x ld]  row-major, columns 0..r-1 live (ld = padded rank cap)
//   V  [n_cap x ld]  row-major (V = Vt^T, so U and V rotate with one kernel
//                    and the column-append transpose trick is a pointer swap)
//   s  [ld], A [m_cap x n_cap] (tracked matrix, lda = n_cap), N (||A||^2)
// Per-tick sequence (row append, engine.py:117-129):
//   K1 project_append  -> p, z, rho, ||x||, core, A row write, N += x.x
//   K2 core_svd        -> Uk, s', Vk (Jacobi, sort, snap, complete)
//   K3/K4 rotate       -> U <- [U 0; 0 1] Uk[:, :keep], V <- V Vk[:r] + z^ Vk[r]
//   install            -> s <- s'[:keep]; zero-sigma completion (engine.py:59-70)
// Sign canonicalisation (engine.py:207) is deferred to observation: the
// update is exactly sign-equivariant (flipping a U column and V column pair
// flips the core by a +-1 diagonal similarity, the Jacobi rotations by the
// same similarity, and the rotated factors come out bit-identical), so the
// canonical form is produced whenever factors are read.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>
#include "common.cuh"
#include "core_svd.cuh"
#include "dense_svd.cuh"
#include "shard.cuh"
#include "tall.cuh"
#include "guard.cuh"
#include "metrics.cuh"
#include "tick.cuh"
#include "../../include/isvd.h"

namespace isvd {
// Host-side section timer for the per-event path (ISVD_HOST_PROF=1: totals
// printed to stderr at engine destruction; tools/b1_breakdown.py)
struct HostProf {
  bool on = false;
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long n[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  HostProf() {
    const char* v = std::getenv("ISVD_HOST_PROF");
    on = v && v[0] == '1';
  }
  static double now() {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
  }
  void add(int k, double t0) {
    if (!on) return;
    acc[k] += now() - t0;
    n[k] += 1;
  }
  void report() {
    if (!on) return;
    static const char* names[8] = {"append:pre", "append:staging", "append:issue", "append:post",
                                   "issue:K1", "issue:core", "issue:rotate", "rank1:total"};
    for (int k = 0; k < 8; ++k)
      if (n[k]) std::fprintf(stderr, "[isvd host] %-16s %8.2f us x %ld\n", names[k], acc[k] / n[k], n[k]);
  }
};
static HostProf g_hprof;
#define HP_T0(v) const double v = g_hprof.on ? HostProf::now() : 0.0


static thread_local std::string g_err;
thread_local const int* g_gate = nullptr;
static int64_t g_launches = 0;
void set_error(const std::string& msg) { g_err = msg; }
void count_launch(int n) { __atomic_add_fetch(&g_launches, n, __ATOMIC_RELAXED); }

template <typename T>
static int dalloc(T** p, size_t n) {
  *p = nullptr;
  if (n == 0) return ISVD_OK;
  cudaError_t e = cudaMalloc((void**)p, n * sizeof(T));
  if (e != cudaSuccess) {
    set_error(std::string("cudaMalloc(") + std::to_string(n * sizeof(T)) + "): " +
              cudaGetErrorString(e));
    cudaGetLastError();
    *p = nullptr;
    return e == cudaErrorMemoryAllocation ? ISVD_ENOMEM : ISVD_ENODEV;
  }
  return ISVD_OK;
}
template <typename T>
static void dfree(T*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}

static int check_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    set_error("no CUDA device available (libisvd has no CPU fallback)");
    return ISVD_ENODEV;
  }
  // Stream-ordered scratch (cudaMallocAsync) comes from the device's default
  // pool; with the default release threshold (0) every synchronize hands the
  // memory back to the driver and the next tick re-maps it (~0.1 ms per
  // allocation on a synchronous per-step loop).  Keep it.
  static bool pool_set = false;
  if (!pool_set) {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
    pool_set = true;
  }
  return ISVD_OK;
}

// Work streams (the engine stream and the stream groups) come from a
// process-wide pool per device and return to it when an engine is destroyed,
// instead of being destroyed: a caller that passed device payloads may still
// have its caching allocator record events on the streams that read them
// (isvd_engine_streams, Tensor.record_stream) after the engine is gone.
// An engine synchronises its streams before returning them.
static std::mutex g_pool_mu;
static std::map<int, std::vector<cudaStream_t>> g_pool;
static cudaError_t stream_get(cudaStream_t* s) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    auto& v = g_pool[dev];
    if (!v.empty()) {
      *s = v.back();
      v.pop_back();
      return cudaSuccess;
    }
  }
  return cudaStreamCreateWithFlags(s, cudaStreamNonBlocking);
}
static void stream_put(cudaStream_t s) {
  int dev = 0;
  if (!s || cudaGetDevice(&dev) != cudaSuccess) return;
  cudaStreamSynchronize(s);
  std::lock_guard<std::mutex> lk(g_pool_mu);
  g_pool[dev].push_back(s);
}

// Host-side finiteness check of event payloads (the reference's as_vector,
// linalg.py:31-40).  Branch-free exponent test so the loop vectorises.
static bool finite_chunk(const double* p, size_t n) {
  // x - x is 0 for finite x and NaN for +-inf / NaN; eight independent
  // accumulators let the compiler keep the loop in SIMD registers (the scan
  // is bound by host memory bandwidth, one pass)
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  size_t i = 0;
  for (; i + 8 <= n; i += 8)
    for (int k = 0; k < 8; ++k) acc[k] += p[i + k] - p[i + k];
  double tail = 0.0;
  for (; i < n; ++i) tail += p[i] - p[i];
  const double tot = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7])) + tail;
  return tot == 0.0;
}

// One pass on the calling thread (a 5a row tick carries 8 MB): helper
// threads were measured to slow the GPU work the host overlaps the scan with
// (tools/e2e_loop_probe.py), so it stays serial.
static bool all_finite(const double* p, size_t n) { return finite_chunk(p, n); }

}  // namespace isvd

using namespace isvd;

// Leading triplets and spectrum of the tracked matrix kept from the last
// oracle observation (device buffers, owned here): the refresh that the
// policies fire right after observing the same matrix (stream.py:291-333:
// observe, decide, refresh) installs them instead of factoring A a second
// time.  Valid until an event changes the tracked matrix.
struct OracleKeep {
  double *U = nullptr, *V = nullptr, *sw = nullptr, *sa = nullptr;
  int B = 0, m = 0, n = 0, w = 0, ldw = 0, nc = 0;
  bool valid = false;
  bool nozero = false;  // every kept sigma > 0 (no zero-sigma completion involved)
  void drop() {
    if (U) cudaFree(U);
    if (V) cudaFree(V);
    if (sw) cudaFree(sw);
    if (sa) cudaFree(sa);
    U = V = sw = sa = nullptr;
    valid = false;
  }
};

struct isvd_engine {
  int B = 0, m = 0, n = 0, r = 0, k = 0;
  // Row sharding (isvd_engine_set_shard): this rank holds global rows
  // [row0, row0 + m) of U and A; m_glob counts all rows; the owner (last
  // shard) also stores the appended rows.  Not sharded: m_glob == m.
  bool sharded = false, owner = true;
  int shard_rank = 0, shard_world = 1;
  int64_t row0 = 0;
  int m_glob = 0;
  Allreducer ar;
  const Allreducer* arp() const { return sharded ? &ar : nullptr; }
  int allreduce(double* p, int64_t cnt) { return sharded ? ar(p, cnt) : ISVD_OK; }
  int gm() const { return sharded ? m_glob : m; }
  int64_t sh_i = 0, sh_j = 0;  // the rank-1 event being issued (sharded)
  double sh_d = 0.0;
  double* shv = nullptr;  // [kCoreMaxS + 2] cross-shard vector scratch
  // Completion ticket of work that may still run on the group streams: one
  // event per pending group (or one on st).
  struct Ticket {
    std::vector<cudaEvent_t> ev;
    int n = 0;
  };
  Ticket sc_tk[8];  // isvd_engine_scalars_async tickets
  // host-payload staging: copy stream, two slots of ev, their events
  cudaStream_t cp_st = nullptr;
  // host-payload staging slots: a host loop may run this many ticks ahead
  // of the device before an upload waits for its slot
  static constexpr int kStageSlots = 4;
  Ticket stage_tk[kStageSlots];  // the ticks that last read each staging slot
  cudaEvent_t stage_ready = nullptr;
  int stage_slot = 0;
  volatile int* vflag_h = nullptr;  // pinned: the device finiteness verdict per slot
  // Device-resident rank-1 payloads are validated by the staging kernel;
  // a rejected entry sets dflag[kDevBad] (sticky) and is applied as a no-op.
  // The verdict is read at the next synchronisation point.
  static constexpr int kDevBad = 1 + kStageSlots;
  bool dev_inputs = false;
  int dev_input_verdict() {
    if (!dev_inputs) return ISVD_OK;
    dev_inputs = false;
    int bad = 0;
    ISVD_CUDA(cudaMemcpyAsync(&bad, dflag + kDevBad, sizeof(int), cudaMemcpyDeviceToHost, st));
    ISVD_CUDA(cudaStreamSynchronize(st));
    if (!bad) return ISVD_OK;
    ISVD_CUDA(cudaMemsetAsync(dflag + kDevBad, 0, sizeof(int), st));
    set_error("a device-resident rank-1 event had an index out of bounds or a non-finite delta; "
              "it was applied as a no-op to its stream");
    return ISVD_EINVAL;
  }
  int ensure_copy_stream() {
    if (cp_st) return ISVD_OK;
    ISVD_CUDA(cudaHostAlloc((void**)&vflag_h, kStageSlots * sizeof(int), cudaHostAllocDefault));
    for (int i = 0; i < kStageSlots; ++i) vflag_h[i] = 0;
    // highest priority: the payload check gates the tick kernels queued
    // behind it, so its CTAs go ahead of the running ticks'
    int lo = 0, hi = 0;
    ISVD_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    ISVD_CUDA(cudaStreamCreateWithPriority(&cp_st, cudaStreamNonBlocking, hi));
    ISVD_CUDA(cudaEventCreateWithFlags(&stage_ready, cudaEventDisableTiming));
    return ISVD_OK;
  }
  int64_t step = 0;
  double tol = 1e-10;
  bool guard = false;
  double reortho_threshold = 1e-6;  // engine.py:30
  // engine.py:205-206,210-217: after an event, refactor if the factors drifted
  int guard_step() {
    if (!guard || r < 1) return ISVD_OK;
    join();
    ISVD_TRY(flush());
    std::vector<double> du(B), dv(B);
    ISVD_TRY(reortho_defects(B, r, Um(), m, Vm(), n, du.data(), dv.data(), st, arp()));
    bool any = false;
    for (int b = 0; b < B; ++b) any |= std::max(du[b], dv[b]) > reortho_threshold;
    if (!any) return ISVD_OK;
    ISVD_TRY(reortho_apply(B, r, Um(), m, Vm(), n, s, ld, core, uk, vk, cstride(), S(), sv, vscr,
                           st, arp()));
    canonical = false;
    return ISVD_OK;
  }
  int m_cap = 0, n_cap = 0, ld = 0;
  cudaStream_t st = nullptr;
  bool own_stream = false;
  bool canonical = true;
  bool initialized = false;
  double *U = nullptr, *V = nullptr, *s = nullptr, *A = nullptr, *N = nullptr;
  double *core = nullptr, *uk = nullptr, *vk = nullptr, *sv = nullptr, *vscr = nullptr;
  double *z = nullptr, *inj = nullptr, *rho = nullptr, *xnorm = nullptr, *ev = nullptr;
  int64_t *ei = nullptr, *ej = nullptr;
  double* ed = nullptr;
  int* dflag = nullptr;
  unsigned* zf_cnt = nullptr;  // per-stream CTA arrival counts (fused zero-sigma completion)
  int64_t* pack_dev = nullptr;          // small host rank-1 payloads: (i, j, delta) per slot
  std::vector<int64_t> pack_host;
  int* fbbuf = nullptr;        // core fallback list [0, B), counts [B, 2B), done counts [2B, 3B) and [3B, 4B)
  double* ref = nullptr;
  int ref_m = 0, ref_r = 0, ref_cap = 0;
  bool has_ref = false;
  // dense-SVD / metrics workspace
  double *wx = nullptr, *wj = nullptr, *wpart = nullptr, *wout = nullptr;
  // Full spectrum of the tracked matrix from the last init / refresh, valid
  // until anything changes the state: the oracle observation that follows a
  // refresh of the same matrix (stream.py:291-333 observes right after the
  // refresh) is served from it and from the refreshed factors instead of a
  // second dense SVD of the same A (config 4: 13 of 37 dense SVDs).
  double* svdc_sall = nullptr;
  int64_t svdc_cap = 0;
  bool svdc_valid = false;
  int svdc_w = 0;
  OracleKeep okeep;
  int64_t wx_n = 0, wj_n = 0, wpart_n = 0, wout_n = 0;
  int* wflags = nullptr;
  std::vector<int> hflags;
  // optional per-phase timing (CUDA events on the engine stream):
  // phase 0 = K1/K6 project+build, 1 = K2 core SVD, 2 = K3/K4 rotation,
  // 3 = install (s copy + zero-sigma completion)
  bool timing = false;
  // verification hook: solve append cores with the generic Jacobi kernel
  // instead of the secular-equation kernel (both are exact SVDs)
  bool append_jacobi = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<cudaEvent_t> ev_marks;  // 5 per recorded tick
  int64_t timed_ticks = 0;
  std::vector<int> tick_kind;  // 0 = append, 1 = rank-1, per recorded tick
  // Deferred left-basis rotation.  Row appends and rank-1
  // updates multiply the small W (U = [Ub 0; 0 I] W) instead of the tall U;
  // U is materialised every lazy_rows appended rows and whenever it is read.
  // Window: a flush costs ~2 m r doubles, a tick inside the window ~2 (r + t) r,
  // so T ~ sqrt(2 m) balances them (48 rows at m = 1024; 2896 at m = 2^22).
  static constexpr int kLazyRows = 32;
  int lazy_rows = kLazyRows;
  static int lazy_window_for(int m) {
    int t = (int)std::lround(std::sqrt(2.0 * (double)std::max(m, 1)));
    t = (t + 7) / 8 * 8;
    return std::min(std::max(t, kLazyRows), 4096);
  }
  bool lazy_mode = true;
  bool lazy_active = false;
  int m_base = 0, r_base = 0, lazy_b = 0;
  double* W = nullptr;
  int r_base_next = 0, lazy_b_next = 0;  // window state after the event being issued
  // Deferred right-basis rotation: while vpend, the true V is V . Gv (Gv is
  // r x r per stream; ld + 1 rows so a row append can grow it in place).
  // Rank-1 ticks rotate the small Gv instead of the n x r V; the next row
  // append projects through Gv and folds it into its own V rotation, so a
  // rank-1 tick costs no pass over V.
  // Full-rank row appends defer V as well: V_eff = [V(:, :vfw) | Z^T] Gv
  // with Z the vnz unnormalised residuals appended since (kVWin at most);
  // the row tick then writes one residual and grows Gv by a row instead of
  // rotating V, and V is materialised every kVWin row appends.
  int vdefer_mode = 1;  // 0 off, 1 on for batches >= 64, 2 whenever the kernels allow
  bool vpend = false;
  double* Gv = nullptr;
  double* Zv = nullptr;
  int zv_ncap = 0;
  int vfw = 0, vnz = 0;
  int64_t gstride() const { return (int64_t)(ld + kVWin + 1) * ld; }
  Mat Gm() const { return Mat{Gv, gstride(), ld}; }
  int64_t zvstride() const { return (int64_t)kVWin * n_cap; }
  VDefer vdesc(int b0, int nz) const {
    VDefer d;
    d.G = Gv + b0 * gstride();
    d.g_stride = gstride();
    d.ldg = ld;
    d.fw = vfw;
    d.nz = nz;
    d.Z = Zv ? Zv + b0 * zvstride() : nullptr;
    d.z_stride = zvstride();
    d.ldz = n_cap;
    return d;
  }
  bool vdefer_ok() const {
    return vdefer_mode != 0 && !sharded && r >= 1 && k <= 32 && (vdefer_mode == 2 || B >= 64);
  }
  int ensure_gv() {
    if (!Gv) ISVD_TRY(dalloc(&Gv, (size_t)B * gstride()));
    if (Zv && zv_ncap != n_cap) dfree(Zv);
    if (!Zv) {
      ISVD_TRY(dalloc(&Zv, (size_t)B * zvstride()));
      zv_ncap = n_cap;
    }
    return ISVD_OK;
  }
  struct Snap {
    double *U = nullptr, *V = nullptr, *A = nullptr, *s = nullptr, *N = nullptr;
    double* ref = nullptr;  // the drift reference (set_reference / refresh(store_reference))
    size_t nu = 0, nv = 0, na = 0, ns = 0, nref = 0;
    int m = 0, n = 0, r = 0, k = 0, m_cap = 0, n_cap = 0, ld = 0, m_glob = 0;
    int ref_m = 0, ref_r = 0, ref_cap = 0;
    int64_t step = 0;
    bool canonical = true, valid = false, has_ref = false;
  } snap;
  // stream groups (pipelining across streams of the batch)
  static constexpr int kGroupMin = 256;
  int ngroups = 4, ngroups_active = 1;
  std::vector<cudaStream_t> gst;
  cudaEvent_t fork_ev = nullptr;
  std::vector<cudaEvent_t> join_ev;
  // Deferred join: a tick leaves its group streams running (each group's next
  // tick is ordered after its own previous one on the same group stream), so
  // successive ticks of different groups overlap -- one group's core SVDs run
  // beside another's HBM passes.  Every other use of the engine stream joins
  // first (join()), so st still orders all engine work for the caller.
  bool async_groups = true, pend = false;
  int pend_G = 0;
  void join() {
    ring_last = -1;  // conservatively: the next read-back takes the general path
    if (!pend) return;
    for (int g = 0; g < pend_G; ++g) cudaStreamWaitEvent(st, join_ev[g], 0);
    pend = false;
  }
  // Read-back ring: the tick kernels that update (N, rho, xnorm) also write
  // them to ring slot tick % kRing, so isvd_engine_scalars_async copies that
  // slot on its own stream after the groups' tick instead of putting a copy
  // between two ticks of every group stream.
  static constexpr int kRing = 8;
  double* sring = nullptr;
  int64_t ring_cnt = 0;
  int ring_slot = 0, ring_last = -1;
  cudaStream_t rd_st = nullptr;
  cudaEvent_t rd_done[kRing] = {};
  bool rd_used[kRing] = {};
  Ticket rd_tk;  // the groups' point a ring copy waits for
  double* ring_row(int slot, int b0) const { return sring + (int64_t)slot * 3 * B + b0; }
  // record: the point every group stream (or st) has reached now
  int ticket_record(Ticket& t) {
    const int n = pend ? pend_G : 1;
    while ((int)t.ev.size() < n) {
      cudaEvent_t ev;
      ISVD_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      t.ev.push_back(ev);
    }
    for (int g = 0; g < n; ++g) ISVD_CUDA(cudaEventRecord(t.ev[g], pend ? gst[g] : st));
    t.n = n;
    return ISVD_OK;
  }
  int ticket_record_on(Ticket& t, cudaStream_t s2) {
    if (t.ev.empty()) {
      cudaEvent_t ev;
      ISVD_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      t.ev.push_back(ev);
    }
    ISVD_CUDA(cudaEventRecord(t.ev[0], s2));
    t.n = 1;
    return ISVD_OK;
  }
  int ticket_wait(cudaStream_t s2, const Ticket& t) {
    for (int g = 0; g < t.n; ++g) ISVD_CUDA(cudaStreamWaitEvent(s2, t.ev[g], 0));
    return ISVD_OK;
  }
  int ticket_sync(const Ticket& t) {
    for (int g = 0; g < t.n; ++g) ISVD_CUDA(cudaEventSynchronize(t.ev[g]));
    return ISVD_OK;
  }
  int ensure_groups(int G) {
    if (!fork_ev) ISVD_CUDA(cudaEventCreateWithFlags(&fork_ev, cudaEventDisableTiming));
    while ((int)gst.size() < G) {
      cudaStream_t s2;
      cudaEvent_t ev;
      ISVD_CUDA(stream_get(&s2));
      ISVD_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      gst.push_back(s2);
      join_ev.push_back(ev);
    }
    return ISVD_OK;
  }
  int64_t wstride() const { return (int64_t)(ld + lazy_rows + 1) * ld; }
  Mat Wm() const { return Mat{W, wstride(), ld}; }
  LazyBasis lazy() const { return LazyBasis{lazy_active ? 1 : 0, m_base, r_base, Wm()}; }

  // flush timing (CUDA events around each flush) and its algorithmic bytes
  std::vector<cudaEvent_t> flush_marks;
  double flush_bytes = 0.0;

  // V <- [V(:, :vfw) | Z^T] Gv ; ends the deferred right basis.  in_tick:
  // per stream group on the group streams when they are pending.
  int flush_v(bool in_tick = false) {
    if (!vpend) return ISVD_OK;
    const bool grouped = in_tick && pend && !timing;
    if (!grouped) join();
    auto body = [&](int b0, int nb, cudaStream_t s2) -> int {
      RotJob jv{Mat{V + b0 * vstride(), vstride(), ld}, n, Gv + b0 * gstride(), gstride(), ld,
                nullptr, 0, nullptr, 0};
      if (vnz > 0) {
        jv.zs = Zv + b0 * zvstride();
        jv.zs_stride = zvstride();
        jv.ldzs = n_cap;
        jv.zfw = vfw;
      }
      return launch_rotate(nb, vfw + vnz, r, jv, nullptr, s2);
    };
    if (grouped) {
      for (int g = 0; g < pend_G; ++g) {
        const int b0 = (int)((int64_t)B * g / pend_G), b1 = (int)((int64_t)B * (g + 1) / pend_G);
        ISVD_TRY(body(b0, b1 - b0, gst[g]));
        ISVD_CUDA(cudaEventRecord(join_ev[g], gst[g]));
      }
    } else {
      ISVD_TRY(body(0, B, st));
    }
    vpend = false;
    vnz = 0;
    return ISVD_OK;
  }
  // materialise both deferred bases
  int flush() {
    ISVD_TRY(flush_u());
    return flush_v();
  }

  // U <- [Ub 0; 0 I] W ; ends the deferred window.  in_tick: issued per
  // stream group on the group streams (no join) when the groups are pending.
  int flush_u(bool in_tick = false) {
    if (!lazy_active) return ISVD_OK;
    const bool grouped = in_tick && pend && !timing;
    if (!grouped) join();
    if (timing) {
      cudaEvent_t ev;
      cudaEventCreate(&ev);
      cudaEventRecord(ev, st);
      flush_marks.push_back(ev);
      // U base rows read (r_base wide) + written (r wide); W rows read; new rows written
      flush_bytes += 8.0 * B * ((double)m_base * (r_base + r) + (double)(r_base + lazy_b) * r +
                                (double)lazy_b * r);
    }
    auto body = [&](int b0, int nb, cudaStream_t s2) -> int {
      RotJob ju{Mat{U + b0 * ustride(), ustride(), ld}, m_base, W + b0 * wstride(), wstride(), ld,
                nullptr, 0, nullptr, 0};
      ISVD_TRY(launch_rotate(nb, r_base, r, ju, nullptr, s2));
      if (timing) {
        cudaEvent_t ev;
        cudaEventCreate(&ev);
        cudaEventRecord(ev, s2);
        flush_marks.push_back(ev);
      }
      if (lazy_b > 0 && owner)  // appended rows live on the owner shard only
        ISVD_TRY(launch_copy_rows(nb, lazy_b, r, W + b0 * wstride() + (int64_t)r_base * ld,
                                  wstride(), ld, U + b0 * ustride() + (int64_t)m_base * ld,
                                  ustride(), ld, s2));
      return ISVD_OK;
    };
    if (grouped) {
      for (int g = 0; g < pend_G; ++g) {
        const int b0 = (int)((int64_t)B * g / pend_G), b1 = (int)((int64_t)B * (g + 1) / pend_G);
        ISVD_TRY(body(b0, b1 - b0, gst[g]));
        ISVD_CUDA(cudaEventRecord(join_ev[g], gst[g]));
      }
    } else {
      ISVD_TRY(body(0, B, st));
    }
    lazy_active = false;
    lazy_b = 0;
    return ISVD_OK;
  }

  void mark() {
    if (!timing) return;
    cudaEvent_t ev;
    if (ev_pool.empty()) {
      cudaEventCreate(&ev);
    } else {
      ev = ev_pool.back();
      ev_pool.pop_back();
    }
    cudaEventRecord(ev, st);
    ev_marks.push_back(ev);
  }

  // core pitch: ld + 1 rounded to even (16-byte rows for the TMA-staged rotation)
  int S() const { return ld + 2; }
  int64_t ustride() const { return (int64_t)m_cap * ld; }
  int64_t vstride() const { return (int64_t)n_cap * ld; }
  int64_t astride() const { return (int64_t)m_cap * n_cap; }
  int64_t cstride() const { return (int64_t)S() * S(); }
  int zlen() const { return std::max(m_cap, n_cap) + 8; }
  Mat Um() const { return Mat{U, ustride(), ld}; }
  Mat Vm() const { return Mat{V, vstride(), ld}; }

  int alloc_core_bufs() {
    dfree(core); dfree(uk); dfree(vk); dfree(sv); dfree(vscr);
    size_t cs = (size_t)B * cstride();
    ISVD_TRY(dalloc(&core, cs));
    ISVD_TRY(dalloc(&uk, cs));
    ISVD_TRY(dalloc(&vk, cs));
    ISVD_TRY(dalloc(&sv, (size_t)B * S()));
    if (S() > kSmemMaxS) ISVD_TRY(dalloc(&vscr, (size_t)B * S() * (S() | 1)));
    return ISVD_OK;
  }

  int alloc_vec_bufs() {
    dfree(z); dfree(ev);
    ISVD_TRY(dalloc(&z, (size_t)B * zlen()));
    ISVD_TRY(dalloc(&ev, (size_t)kStageSlots * B * zlen()));
    return ISVD_OK;
  }

  int ensure_work(int64_t x_n, int64_t j_n, int64_t part_n, int64_t out_n) {
    if (x_n > wx_n) { dfree(wx); ISVD_TRY(dalloc(&wx, x_n)); wx_n = x_n; }
    if (j_n > wj_n) { dfree(wj); ISVD_TRY(dalloc(&wj, j_n)); wj_n = j_n; }
    if (part_n > wpart_n) { dfree(wpart); ISVD_TRY(dalloc(&wpart, part_n)); wpart_n = part_n; }
    if (out_n > wout_n) { dfree(wout); ISVD_TRY(dalloc(&wout, out_n)); wout_n = out_n; }
    if (!wflags) ISVD_TRY(dalloc(&wflags, (size_t)B));
    hflags.resize(B);
    return ISVD_OK;
  }

  // grow U (rows) and A (rows) to hold at least rows_needed rows
  int grow_rows(int rows_needed) {
    if (rows_needed <= m_cap) return ISVD_OK;
    join();
    int nc = std::max(rows_needed, m_cap * 2);
    double *U2, *A2;
    ISVD_TRY(dalloc(&U2, (size_t)B * nc * ld));
    ISVD_CUDA(cudaMemsetAsync(U2, 0, sizeof(double) * B * nc * ld, st));
    ISVD_TRY(launch_copy_rows(B, m, ld, U, ustride(), ld, U2, (int64_t)nc * ld, ld, st));
    ISVD_TRY(dalloc(&A2, (size_t)B * nc * n_cap));
    ISVD_TRY(launch_copy_rows(B, m, n, A, astride(), n_cap, A2, (int64_t)nc * n_cap, n_cap, st));
    ISVD_CUDA(cudaStreamSynchronize(st));
    dfree(U); dfree(A);
    U = U2; A = A2;
    m_cap = nc;
    return alloc_vec_bufs();
  }

  int grow_cols(int cols_needed) {
    if (cols_needed <= n_cap) return ISVD_OK;
    ISVD_TRY(flush_v());  // Z and Gv describe the old V layout
    join();
    int nc = std::max(cols_needed, n_cap * 2);
    double *V2, *A2;
    ISVD_TRY(dalloc(&V2, (size_t)B * nc * ld));
    ISVD_CUDA(cudaMemsetAsync(V2, 0, sizeof(double) * B * nc * ld, st));
    ISVD_TRY(launch_copy_rows(B, n, ld, V, vstride(), ld, V2, (int64_t)nc * ld, ld, st));
    ISVD_TRY(dalloc(&A2, (size_t)B * m_cap * nc));
    ISVD_TRY(launch_copy_rows(B, m, n, A, astride(), n_cap, A2, (int64_t)m_cap * nc, nc, st));
    ISVD_CUDA(cudaStreamSynchronize(st));
    dfree(V); dfree(A);
    V = V2; A = A2;
    n_cap = nc;
    return alloc_vec_bufs();
  }

  int grow_rank(int k_needed) {
    int nld = round_up(std::max(k_needed, 1), 8);
    if (nld <= ld) return ISVD_OK;
    if (nld + 1 > kCoreMaxS) {
      set_error("work rank exceeds the supported maximum (" + std::to_string(kCoreMaxS - 1) + ")");
      return ISVD_EINVAL;
    }
    ISVD_TRY(flush());
    double *U2, *V2, *s2;
    ISVD_TRY(dalloc(&U2, (size_t)B * m_cap * nld));
    ISVD_TRY(dalloc(&V2, (size_t)B * n_cap * nld));
    ISVD_TRY(dalloc(&s2, (size_t)B * nld));
    ISVD_CUDA(cudaMemsetAsync(U2, 0, sizeof(double) * B * m_cap * nld, st));
    ISVD_CUDA(cudaMemsetAsync(V2, 0, sizeof(double) * B * n_cap * nld, st));
    ISVD_CUDA(cudaMemsetAsync(s2, 0, sizeof(double) * B * nld, st));
    if (U) {
      ISVD_TRY(launch_copy_rows(B, m, ld, U, ustride(), ld, U2, (int64_t)m_cap * nld, nld, st));
      ISVD_TRY(launch_copy_rows(B, n, ld, V, vstride(), ld, V2, (int64_t)n_cap * nld, nld, st));
      ISVD_TRY(launch_copy_rows(B, 1, ld, s, ld, ld, s2, nld, nld, st));
    }
    double* ref2 = nullptr;
    if (ref) {
      ISVD_TRY(dalloc(&ref2, (size_t)B * ref_cap * nld));
      ISVD_TRY(launch_copy_rows(B, ref_m, ld, ref, (int64_t)ref_cap * ld, ld, ref2,
                                (int64_t)ref_cap * nld, nld, st));
    }
    ISVD_CUDA(cudaStreamSynchronize(st));
    dfree(U); dfree(V); dfree(s);
    U = U2; V = V2; s = s2;
    if (ref) { dfree(ref); ref = ref2; }
    ld = nld;
    dfree(Gv);  // re-allocated with the new leading dimension when next used
    dfree(W);
    ISVD_TRY(dalloc(&W, (size_t)B * wstride()));
    ISVD_CUDA(cudaMemsetAsync(W, 0, sizeof(double) * B * wstride(), st));
    return alloc_core_bufs();
  }

  int canonicalize() {
    ISVD_TRY(flush());
    if (canonical) return ISVD_OK;
    if (sharded) {
      // global argmax |U[:, c]| (lowest global row on ties): every rank posts
      // its column maxima into its own slot, one sum-allreduce gathers them
      double* pk = nullptr;
      const int64_t cnt = (int64_t)shard_world * r * 3;
      ISVD_CUDA(cudaMallocAsync((void**)&pk, sizeof(double) * std::max<int64_t>(cnt, 1), st));
      int rc = launch_canon_shard_post(r, Um(), m, row0, shard_rank, shard_world, pk, st);
      if (rc == ISVD_OK) rc = ar(pk, cnt);
      if (rc == ISVD_OK) rc = launch_canon_shard_apply(r, Um(), m, Vm(), n, shard_world, pk, st);
      cudaFreeAsync(pk, st);
      ISVD_TRY(rc);
    } else {
      ISVD_TRY(launch_canonicalize(B, r, Um(), m, Vm(), n, st));
    }
    canonical = true;
    return ISVD_OK;
  }

  int install_from_core(int keep) {
    // s <- sv[:, :keep]
    if (keep > 0)
      ISVD_CUDA(cudaMemcpy2DAsync(s, sizeof(double) * ld, sv, sizeof(double) * S(),
                                  sizeof(double) * keep, B, cudaMemcpyDeviceToDevice, st));
    return ISVD_OK;
  }

  // dense thin SVD of the tracked matrix into U, V, s (engine init/refresh)
  int factor_tracked() {
    int w = std::min(k, std::min(gm(), n));
    int sweeps = 0;
    lazy_active = false;  // U is recomputed from A
    lazy_b = 0;
    vpend = false;
    vnz = 0;
    if (sharded) {
      ISVD_TRY(gram_svd_run(m, n, A, n_cap, w, Um(), Vm(), s, nullptr, st, arp()));
    } else {
      DenseSvdPlan P = dense_svd_plan(m, n, w);
      ISVD_TRY(ensure_work((int64_t)B * P.x_elems(), (int64_t)B * P.j_elems(), 0, 0));
      const int nc = std::min(m, n);
      svdc_valid = false;
      if ((int64_t)B * nc > svdc_cap) {
        dfree(svdc_sall);
        svdc_sall = nullptr;
        svdc_cap = 0;
        ISVD_TRY(dalloc(&svdc_sall, (size_t)B * nc));
        svdc_cap = (int64_t)B * nc;
      }
      if (okeep.valid && okeep.nozero && okeep.B == B && okeep.m == m && okeep.n == n &&
          okeep.nc == nc && w <= okeep.w) {
        // the matrix just observed: its leading w triplets and spectrum
        ISVD_TRY(launch_copy_rows(B, m, w, okeep.U, (int64_t)m * okeep.ldw, okeep.ldw, U, ustride(),
                                  ld, st));
        ISVD_TRY(launch_copy_rows(B, n, w, okeep.V, (int64_t)n * okeep.ldw, okeep.ldw, V, vstride(),
                                  ld, st));
        ISVD_TRY(launch_copy_rows(B, 1, w, okeep.sw, okeep.ldw, okeep.ldw, s, ld, ld, st));
        ISVD_CUDA(cudaMemcpyAsync(svdc_sall, okeep.sa, sizeof(double) * B * nc,
                                  cudaMemcpyDeviceToDevice, st));
      } else {
        ISVD_TRY(dense_svd_run(B, m, n, A, astride(), n_cap, w, Um(), Vm(), s, ld, svdc_sall, nc, wx,
                               wj, wflags, hflags.data(), st, &sweeps));
      }
      svdc_w = w;
    }
    r = w;
    // (sharded: U's zero-sigma columns would need a distributed completion;
    // only V -- replicated -- is completed here)
    ISVD_TRY(launch_complete_zero(B, r, s, ld, Um(), sharded ? 0 : m, Vm(), n, st));
    canonical = false;
    ISVD_TRY(canonicalize());
    svdc_valid = !sharded;
    return ISVD_OK;
  }

  ~isvd_engine() {
    dfree(svdc_sall);
    okeep.drop();
    dfree(U); dfree(V); dfree(s); dfree(A); dfree(N);
    dfree(core); dfree(uk); dfree(vk); dfree(sv); dfree(vscr);
    dfree(z); dfree(inj); dfree(rho); dfree(xnorm); dfree(ev);
    dfree(ei); dfree(ej); dfree(ed); dfree(dflag);
    if (zf_cnt) cudaFree(zf_cnt);
    if (fbbuf) cudaFree(fbbuf);
    dfree(pack_dev);
    dfree(ref); dfree(W); dfree(Gv); dfree(Zv);
    dfree(wx); dfree(wj); dfree(wpart); dfree(wout); dfree(wflags);
    dfree(snap.U); dfree(snap.V); dfree(snap.A); dfree(snap.s); dfree(snap.N); dfree(snap.ref);
    dfree(shv);
    for (auto g : gst) stream_put(g);
    for (auto ev : join_ev) cudaEventDestroy(ev);
    if (fork_ev) cudaEventDestroy(fork_ev);
    for (auto ev : ev_marks) cudaEventDestroy(ev);
    for (auto ev : ev_pool) cudaEventDestroy(ev);
    for (auto& t : sc_tk)
      for (auto ev : t.ev) cudaEventDestroy(ev);
    for (auto& t : stage_tk)
      for (auto ev : t.ev) cudaEventDestroy(ev);
    if (stage_ready) cudaEventDestroy(stage_ready);
    for (auto ev : rd_done)
      if (ev) cudaEventDestroy(ev);
    for (auto ev : rd_tk.ev) cudaEventDestroy(ev);
    if (rd_st) cudaStreamDestroy(rd_st);
    dfree(sring);
    if (cp_st) cudaStreamDestroy(cp_st);
    if (vflag_h) cudaFreeHost((void*)vflag_h);
    if (own_stream && st) stream_put(st);
  }
};

extern "C" {

const char* isvd_last_error(void) { return g_err.c_str(); }
int isvd_version(void) { return 1; }
int isvd_debug_counters(int64_t* out8, int reset) {
  if (!out8) { set_error("null argument"); return ISVD_EINVAL; }
  ISVD_TRY(check_device());
  return read_debug_counters(out8, reset);
}
int isvd_debug_trace(int64_t* out, int n) {
  if (!out || n < -4096 || n > 4096) { set_error("bad argument"); return ISVD_EINVAL; }
  ISVD_TRY(check_device());
  if (n < 0) return read_k1_trace(out, -n);  // the projection kernel's marks
  return read_r1_trace(out, n);
}
int64_t isvd_launch_count(void) { return __atomic_load_n(&g_launches, __ATOMIC_RELAXED); }

int isvd_engine_create(isvd_engine** out, int batch, int m, int n, int k, double tol,
                       int reortho_guard, int m_cap, int n_cap, int k_cap, void* stream) {
  if (!out) { set_error("out is null"); return ISVD_EINVAL; }
  *out = nullptr;
  if (batch < 1) { set_error("batch must be >= 1"); return ISVD_EINVAL; }
  if (m < 1 || n < 1) { set_error("initial matrix must be nonempty"); return ISVD_EINVAL; }
  if (k < 1) { set_error("work rank must be >= 1, got " + std::to_string(k)); return ISVD_EINVAL; }
  if (!(tol > 0.0)) { set_error("tol must be positive"); return ISVD_EINVAL; }
  ISVD_TRY(check_device());
  auto* e = new isvd_engine();
  e->B = batch; e->m = m; e->n = n; e->k = k; e->tol = tol; e->guard = reortho_guard != 0;
  e->m_glob = m;
  e->m_cap = std::max(m_cap, m + 1);
  e->n_cap = std::max(n_cap, n);
  int kc = std::max(std::max(k_cap, k), 1);
  e->ld = round_up(kc, 8);
  e->lazy_rows = isvd_engine::lazy_window_for(m);
  if (e->ld + 1 > kCoreMaxS) {
    delete e;
    set_error("work rank exceeds the supported maximum");
    return ISVD_EINVAL;
  }
  if (stream) {
    e->st = (cudaStream_t)stream;
  } else {
    if (stream_get(&e->st) != cudaSuccess) {
      delete e;
      set_error("cudaStreamCreate failed");
      return ISVD_ENODEV;
    }
    e->own_stream = true;
  }
  int rc = ISVD_OK;
  auto A = [&](int x) { if (rc == ISVD_OK) rc = x; };
  A(dalloc(&e->U, (size_t)batch * e->m_cap * e->ld));
  A(dalloc(&e->V, (size_t)batch * e->n_cap * e->ld));
  A(dalloc(&e->s, (size_t)batch * e->ld));
  A(dalloc(&e->A, (size_t)batch * e->m_cap * e->n_cap));
  A(dalloc(&e->N, (size_t)batch));
  A(dalloc(&e->inj, (size_t)batch));
  A(dalloc(&e->rho, (size_t)batch));
  A(dalloc(&e->xnorm, (size_t)batch));
  A(dalloc(&e->ei, (size_t)isvd_engine::kStageSlots * batch));  // staging slots
  A(dalloc(&e->ej, (size_t)isvd_engine::kStageSlots * batch));
  A(dalloc(&e->ed, (size_t)isvd_engine::kStageSlots * batch));
  A(dalloc(&e->dflag, 2 + isvd_engine::kStageSlots));
  if (rc == ISVD_OK && cudaMemset(e->dflag, 0, sizeof(int) * (2 + isvd_engine::kStageSlots)) != cudaSuccess) {
    set_error("cudaMemset failed");
    rc = ISVD_ENODEV;
  }
  A(dalloc(&e->W, (size_t)batch * e->wstride()));
  A(dalloc(&e->sring, (size_t)isvd_engine::kRing * 3 * batch));
  if (rc == ISVD_OK) {
    if (cudaMalloc((void**)&e->zf_cnt, sizeof(unsigned) * batch) != cudaSuccess ||
        cudaMemset(e->zf_cnt, 0, sizeof(unsigned) * batch) != cudaSuccess ||
        cudaMalloc((void**)&e->fbbuf, sizeof(int) * 4 * batch) != cudaSuccess ||
        cudaMemset(e->fbbuf, 0, sizeof(int) * 4 * batch) != cudaSuccess) {
      set_error("out of device memory");
      rc = ISVD_ENOMEM;
    }
  }
  if (rc == ISVD_OK) rc = e->alloc_core_bufs();
  if (rc == ISVD_OK) rc = e->alloc_vec_bufs();
  if (rc == ISVD_OK) {
    cudaMemsetAsync(e->U, 0, sizeof(double) * batch * e->m_cap * e->ld, e->st);
    cudaMemsetAsync(e->V, 0, sizeof(double) * batch * e->n_cap * e->ld, e->st);
    cudaMemsetAsync(e->s, 0, sizeof(double) * batch * e->ld, e->st);
    cudaMemsetAsync(e->W, 0, sizeof(double) * batch * e->wstride(), e->st);
    std::vector<double> nanv(batch, std::nan(""));
    cudaMemcpyAsync(e->rho, nanv.data(), sizeof(double) * batch, cudaMemcpyHostToDevice, e->st);
    cudaMemcpyAsync(e->xnorm, nanv.data(), sizeof(double) * batch, cudaMemcpyHostToDevice, e->st);
    if (cudaStreamSynchronize(e->st) != cudaSuccess) {
      set_error("initialisation failed");
      rc = ISVD_ENODEV;
    }
  }
  if (rc != ISVD_OK) {
    delete e;
    return rc;
  }
  *out = e;
  return ISVD_OK;
}

int isvd_engine_destroy(isvd_engine* e) {
  g_hprof.report();
  if (e) e->join();
  if (e) {
    if (e->st) cudaStreamSynchronize(e->st);
    delete e;
  }
  return ISVD_OK;
}

void* isvd_engine_stream(isvd_engine* e) {
  if (!e) return nullptr;
  e->join();
  return (void*)e->st;
}

int isvd_engine_set_shard(isvd_engine* e, int rank, int world, int64_t row0, int m_global,
                          int owns_appends, isvd_allreduce_fn fn, void* ctx) {
  if (e) e->join();
  if (!e) { set_error("null engine"); return ISVD_EINVAL; }
  if (e->initialized) { set_error("set_shard must precede init"); return ISVD_ESTATE; }
  if (e->B != 1) { set_error("row sharding needs a single stream (B = 1)"); return ISVD_EINVAL; }
  if (!fn || world < 1 || rank < 0 || rank >= world || row0 < 0 || m_global < e->m ||
      row0 + e->m > m_global) {
    set_error("set_shard: bad arguments");
    return ISVD_EINVAL;
  }
  e->sharded = true;
  e->shard_rank = rank;
  e->shard_world = world;
  e->row0 = row0;
  e->m_glob = m_global;
  e->owner = owns_appends != 0;
  e->ar = Allreducer{fn, ctx, e->st};
  if (!e->shv) ISVD_TRY(dalloc(&e->shv, (size_t)kCoreMaxS + 2));
  e->lazy_mode = true;
  e->lazy_rows = isvd_engine::lazy_window_for(m_global);
  dfree(e->W);
  ISVD_TRY(dalloc(&e->W, (size_t)e->B * e->wstride()));
  ISVD_CUDA(cudaMemsetAsync(e->W, 0, sizeof(double) * e->B * e->wstride(), e->st));
  return ISVD_OK;
}

int isvd_engine_shard_info(const isvd_engine* e, int64_t* row0, int* m_local, int* m_global) {
  if (!e) { set_error("null engine"); return ISVD_EINVAL; }
  if (row0) *row0 = e->row0;
  if (m_local) *m_local = e->m;
  if (m_global) *m_global = e->gm();
  return ISVD_OK;
}

int isvd_engine_init(isvd_engine* e, const double* a0, int on_device) {
  if (e) e->join();
  if (!e || !a0) { set_error("null argument"); return ISVD_EINVAL; }
  e->svdc_valid = false;
  e->okeep.valid = false;
  const size_t cnt = (size_t)e->B * e->m * e->n;
  if (!on_device) {
    if (!all_finite(a0, cnt)) { set_error("initial matrix contains non-finite entries"); return ISVD_EINVAL; }
    // stage per stream (row-major m x n) into the pitched tracked matrix
    for (int b = 0; b < e->B; ++b)
      ISVD_CUDA(cudaMemcpy2DAsync(e->A + b * e->astride(), sizeof(double) * e->n_cap,
                                  a0 + (size_t)b * e->m * e->n, sizeof(double) * e->n,
                                  sizeof(double) * e->n, e->m, cudaMemcpyHostToDevice, e->st));
  } else {
    ISVD_CUDA(cudaMemsetAsync(e->dflag, 0, sizeof(int), e->st));
    ISVD_TRY(launch_check_finite(cnt, a0, e->dflag, e->st));
    int hf = 0;
    ISVD_CUDA(cudaMemcpyAsync(&hf, e->dflag, sizeof(int), cudaMemcpyDeviceToHost, e->st));
    ISVD_CUDA(cudaStreamSynchronize(e->st));
    if (hf) { set_error("initial matrix contains non-finite entries"); return ISVD_EINVAL; }
    ISVD_TRY(launch_copy_rows(e->B, e->m, e->n, a0, (int64_t)e->m * e->n, e->n, e->A, e->astride(),
                              e->n_cap, e->st));
  }
  ISVD_TRY(launch_sumsq(e->B, e->m, e->n, e->A, e->astride(), e->n_cap, e->N, e->st));
  ISVD_TRY(e->allreduce(e->N, 1));
  ISVD_TRY(e->factor_tracked());
  e->step = 0;
  e->has_ref = false;
  e->initialized = true;
  std::vector<double> nanv(e->B, std::nan(""));
  ISVD_CUDA(cudaMemcpyAsync(e->rho, nanv.data(), sizeof(double) * e->B, cudaMemcpyHostToDevice, e->st));
  ISVD_CUDA(cudaMemcpyAsync(e->xnorm, nanv.data(), sizeof(double) * e->B, cudaMemcpyHostToDevice, e->st));
  ISVD_CUDA(cudaStreamSynchronize(e->st));
  return ISVD_OK;
}

// ---------------------------------------------------------------------------
// Per-tick launch sequences, issued for a slice of streams [b0, b0 + nb) on
// CUDA stream `st`.  With B large the batch is split into groups on separate
// CUDA streams so the latency/FP64-bound core-SVD kernels of one group run
// concurrently with the HBM-bound projection/rotation kernels of another.
struct Slice {
  int b0, nb;
  cudaStream_t st;
};

static Mat mat_at(const Mat& M, int b0) { return Mat{M.p + b0 * M.stride, M.stride, M.ld}; }

// lazy_state: 0 = eager rotation, 1 = open a deferred window, 2 = continue it
// vp: the right basis is deferred (V_eff = V Gv); this row append projects
// through Gv and folds it into the V rotation
// vrow: full-rank row append with the right basis deferred -- the residual
// goes to Z, Gv grows by a row, V is not touched (vstart: Gv <- I first)
static int issue_append(isvd_engine* e, const Slice& sl, const double* xd, int len, bool is_row,
                        int keep, int lazy_state, bool vp, bool vrow, bool vstart) {
  const int b0 = sl.b0, nb = sl.nb, r = e->r;
  cudaStream_t st = sl.st;
  const int S = e->S();
  const int64_t cs = e->cstride();
  Mat F = mat_at(is_row ? e->Vm() : e->Um(), b0);
  const int64_t a_off = is_row ? (int64_t)e->m * e->n_cap : (int64_t)e->n;
  const int64_t a_step = is_row ? 1 : e->n_cap;
  double* core = e->core + b0 * cs;
  double* uk = e->uk + b0 * cs;
  double* vk = e->vk + b0 * cs;
  double* sv = e->sv + (int64_t)b0 * S;
  double* z = e->z + (int64_t)b0 * e->zlen();
  double* inj = e->inj + b0;
  const bool one = e->ngroups_active == 1;
  if (one) e->mark();
  // sharded: only the owner stores an appended row; a column append projects
  // on the row-sharded U (sums across shards)
  double* Adst = (is_row && !e->owner) ? nullptr : e->A + b0 * e->astride();
  // the read-back ring slot this tick writes must have been copied out
  if (e->rd_used[e->ring_slot]) ISVD_CUDA(cudaStreamWaitEvent(st, e->rd_done[e->ring_slot], 0));
  if (vstart) ISVD_TRY(launch_eye(nb, mat_at(e->Gm(), b0), r, r, st));
  VDefer vd = e->vdesc(b0, vrow ? e->vnz : 0);
  double* zdst = z;
  int64_t zdst_stride = e->zlen();
  if (vrow) {  // the residual becomes column vfw + vnz of the deferred basis
    zdst = e->Zv + b0 * e->zvstride() + (int64_t)e->vnz * e->n_cap;
    zdst_stride = e->zvstride();
  }
  HP_T0(hk1);
  ISVD_TRY(launch_project_append(nb, len, r, F, xd + (int64_t)b0 * len, len,
                                 e->s + (int64_t)b0 * e->ld, e->ld, e->tol, core, cs, S, zdst,
                                 zdst_stride, inj, e->rho + b0, e->xnorm + b0, Adst, e->astride(),
                                 a_off, a_step, e->N + b0, st,
                                 (e->sharded && !is_row) ? &e->ar : nullptr,
                                 e->append_jacobi ? 0 : 1, (vp || vrow) ? &vd : nullptr,
                                 e->ring_row(e->ring_slot, b0), e->B));
  g_hprof.add(4, hk1);
  HP_T0(hk2);
  if (one) e->mark();
  // steady state of a batched k <= 32 stream: the arrow kernel's warp also
  // rotates the deferred bases (no rotation launch, no Uk / Vk re-read)
  const bool fuse_rot = !e->append_jacobi && !e->sharded && is_row && vrow && lazy_state != 0 &&
                        r + 1 <= 40;
  ArrowFuse af;
  if (fuse_rot) {
    af.uw_mode = lazy_state;
    af.uw = mat_at(e->Wm(), b0);
    af.uw_rows = lazy_state == 2 ? e->r_base + e->lazy_b : 0;
    af.gw = mat_at(e->Gm(), b0);
    af.gw_rows = e->vfw + e->vnz;
    af.inj = inj;
    af.zU = mat_at(e->Wm(), b0);
    af.zm = e->r_base_next + e->lazy_b_next;
    af.zV = mat_at(e->Vm(), b0);
    af.zn = e->n;
    af.zvd = e->vdesc(b0, e->vnz + 1);
  }
  // CTA-per-core append cores (k <= 32): fused epilogue above, or Uk / Vk
  // out for the rotation launch below; fallback list per slice
  af.fb_list = e->fbbuf + b0;
  af.fb_count = e->fbbuf + e->B + b0;
  af.fb_done = e->fbbuf + 2 * e->B + b0;
  af.fb_fast_done = e->fbbuf + 3 * e->B + b0;
  if (e->append_jacobi)
    ISVD_TRY(launch_core_svd(nb, r + 1, core, cs, S, uk, vk, cs, S, sv, S,
                             e->vscr ? e->vscr + (int64_t)b0 * S * (S | 1) : nullptr, nullptr, st));
  else
    ISVD_TRY(launch_arrow_svd(nb, r + 1, core, cs, S, uk, vk, cs, S, sv, S, st,
                              e->s + (int64_t)b0 * e->ld, e->ld, keep,
                              (fuse_rot || !e->sharded) ? &af : nullptr));
  g_hprof.add(5, hk2);
  if (fuse_rot) {
    if (one) { e->mark(); e->mark(); }
    return ISVD_OK;
  }
  HP_T0(hk3);
  if (one) e->mark();
  // row: U <- [U 0; 0 1] Uk, V <- V Vk[:r] + z^ Vk[r] ; col: the same with U<->V
  RotJob grow{mat_at(is_row ? e->Um() : e->Vm(), b0), is_row ? e->m : e->n, uk, cs, S, nullptr, 0,
              nullptr, 1};
  RotJob injj{mat_at(is_row ? e->Vm() : e->Um(), b0), is_row ? e->n : e->m, vk, cs, S, z,
              e->zlen(), inj, 0};
  RotJob uj = grow;  // the left side: U itself, or the deferred window W
  bool has_u = true;
  if (lazy_state == 1) {
    // open a deferred window: W = Uk[:, :keep] (rows: r base columns + the new row)
    ISVD_TRY(launch_copy_rows(nb, r + 1, keep, uk, cs, S, e->W + b0 * e->wstride(), e->wstride(),
                              e->ld, st));
    has_u = false;
  } else if (lazy_state == 2) {
    // W <- [W 0; 0 1] Uk[:, :keep]  (in place, new row appended)
    uj = RotJob{mat_at(e->Wm(), b0), e->r_base + e->lazy_b, uk, cs, S, nullptr, 0, nullptr, 1};
  }
  if (vp) {
    // fold the deferred right basis into this rotation: V <- V (Gv Vk[:r]) +
    // z^ Vk[r] (the kernel forms Gv Vk[:r] per CTA) -- one pass over V
    injj.G = e->Gv + b0 * e->gstride();
    injj.g_stride = e->gstride();
    injj.ldg = e->ld;
  }
  if (vrow) {
    // Gv <- [Gv 0; 0 1/rho] Vk[:, :keep]: the rows of the basis rotate, the
    // new residual's row is (1/rho) Vk[r, :] (0 when rho <= tol)
    injj = RotJob{mat_at(e->Gm(), b0), e->vfw + e->vnz, vk, cs, S, nullptr, 0, nullptr, 1};
    injj.nr_scale = inj;
  }
  // zero-sigma completion (_install) over the post-tick factors: fused into
  // the rotation when the secular kernel already installed s
  const int m_new = is_row ? e->m + 1 : e->m, n_new = is_row ? e->n : e->n + 1;
  ZeroFix zf;
  zf.s = e->s + (int64_t)b0 * e->ld;
  zf.lds = e->ld;
  zf.w = keep;
  zf.U = lazy_state != 0 ? mat_at(e->Wm(), b0) : mat_at(e->Um(), b0);
  zf.m = lazy_state != 0 ? e->r_base_next + e->lazy_b_next : (e->sharded ? 0 : m_new);
  zf.V = mat_at(e->Vm(), b0);
  zf.n = n_new;
  zf.counter = e->zf_cnt + b0;
  if (vrow) zf.vd = e->vdesc(b0, e->vnz + 1);
  const ZeroFix* zfp = e->append_jacobi ? nullptr : &zf;
  bool fused = false;
  if (has_u) {
    ISVD_TRY(launch_rotate(nb, r, keep, uj, &injj, st, zfp, &fused));
  } else {
    ISVD_TRY(launch_rotate(nb, r, keep, injj, nullptr, st, zfp, &fused));
  }
  if (one) e->mark();
  // install: s <- sv[:, :keep] (the secular kernel already wrote it), then the
  // zero-sigma completion check
  if (keep > 0 && e->append_jacobi)
    ISVD_CUDA(cudaMemcpy2DAsync(e->s + (int64_t)b0 * e->ld, sizeof(double) * e->ld, sv,
                                sizeof(double) * S, sizeof(double) * keep, nb,
                                cudaMemcpyDeviceToDevice, st));
  if (!fused)
    ISVD_TRY(launch_complete_zero(nb, keep, zf.s, zf.lds, zf.U, zf.m, zf.V, zf.n, st,
                                  vrow ? &zf.vd : nullptr));
  g_hprof.add(6, hk3);
  return ISVD_OK;
}

// defer: leave V in place and rotate the deferred basis Gv instead (vp: Gv
// is already pending; otherwise the core's right vectors open it)
static int issue_rank_one(isvd_engine* e, const Slice& sl, const int64_t* di, const int64_t* dj,
                          const double* dd, int lazy_state, bool defer, bool vp) {
  const int b0 = sl.b0, nb = sl.nb, r = e->r;
  cudaStream_t st = sl.st;
  const int S = e->S();
  const int64_t cs = e->cstride();
  double* core = e->core + b0 * cs;
  double* uk = e->uk + b0 * cs;
  double* vk = e->vk + b0 * cs;
  double* sv = e->sv + (int64_t)b0 * S;
  const bool one = e->ngroups_active == 1;
  LazyBasis lz = e->lazy();
  lz.W = mat_at(lz.W, b0);
  const bool fused = !e->sharded && r <= 32;
  const bool fuse_rot = fused && defer && lazy_state != 0;
  if (e->rd_used[e->ring_slot]) ISVD_CUDA(cudaStreamWaitEvent(st, e->rd_done[e->ring_slot], 0));
  if (one) e->mark();
  if (fused) {
    // K6 + K2b in one kernel: the core is built in registers (no HBM round trip)
    Rank1Core rc;
    rc.U = mat_at(e->Um(), b0);
    rc.V = mat_at(e->Vm(), b0);
    rc.s = e->s + (int64_t)b0 * e->ld;
    rc.lds = e->ld;
    rc.ii = di + b0;
    rc.jj = dj + b0;
    rc.delta = dd + b0;
    rc.A = e->A + b0 * e->astride();
    rc.a_stride = e->astride();
    rc.lda = e->n_cap;
    rc.N = e->N + b0;
    rc.lz = lz;
    rc.ring = e->ring_row(e->ring_slot, b0);
    rc.ring_stride = e->B;
    rc.rho = e->rho + b0;
    rc.xnorm = e->xnorm + b0;
    rc.fb_list = e->fbbuf + b0;
    rc.fb_count = e->fbbuf + e->B + b0;
    rc.fb_done = e->fbbuf + 2 * e->B + b0;
    rc.fb_fast_done = e->fbbuf + 3 * e->B + b0;
    if (vp) {
      rc.vd = e->vdesc(b0, e->vnz);
    } else if (defer) {
      rc.vk_out = e->Gv + b0 * e->gstride();
      rc.vk_stride = e->gstride();
      rc.ldvk = e->ld;
    }
    if (fuse_rot) {
      // the deferred bases are rotated by the core kernel's warps (no
      // rotation launch, no Uk / Vk round trip through HBM)
      rc.uw_mode = lazy_state;
      rc.uw = mat_at(e->Wm(), b0);
      rc.uw_rows = lazy_state == 2 ? e->r_base + e->lazy_b : r;
      if (vp) {
        rc.gw = mat_at(e->Gm(), b0);
        rc.gw_rows = e->vfw + e->vnz;
      }
      rc.zU = mat_at(e->Wm(), b0);
      rc.zm = e->r_base_next + e->lazy_b_next;
      rc.zV = mat_at(e->Vm(), b0);
      rc.zn = e->n;
      rc.zvd = e->vdesc(b0, e->vnz);
    }
    if (one) e->mark();
    ISVD_TRY(launch_rank1_core_svd32(nb, r, rc, uk, vk, cs, S, sv, S, st,
                                     e->s + (int64_t)b0 * e->ld, e->ld));
    if (fuse_rot) {
      if (one) { e->mark(); e->mark(); }
      return ISVD_OK;
    }
  } else if (e->sharded) {
    // U[i, :] and A[i, j] from the shard owning row i, summed across shards
    const int64_t il = e->sh_i - e->row0;
    const bool mine = 0 <= il && il < e->m;
    ISVD_CUDA(cudaMemsetAsync(e->shv, 0, sizeof(double) * (r + 1), st));
    if (mine)
      ISVD_TRY(launch_rank1_gather(r, e->Um(), il, e->sh_j, e->A, e->n_cap, lz, e->shv, st));
    ISVD_TRY(e->allreduce(e->shv, r + 1));
    ISVD_TRY(launch_rank1_vec_build(r, e->shv, e->Vm(), e->s, e->sh_j, e->sh_d, core, S, e->N,
                                    mine ? e->A + il * e->n_cap + e->sh_j : nullptr, st));
  } else {
    ISVD_TRY(launch_rank1_build(nb, r, mat_at(e->Um(), b0), mat_at(e->Vm(), b0),
                                e->s + (int64_t)b0 * e->ld, e->ld, di + b0, dj + b0, dd + b0, core,
                                cs, S, e->A + b0 * e->astride(), e->astride(), e->n_cap, e->N + b0,
                                lz, st));
  }
  if (!fused) {
    if (one) e->mark();
    ISVD_TRY(launch_core_svd(nb, r, core, cs, S, uk, vk, cs, S, sv, S,
                             e->vscr ? e->vscr + (int64_t)b0 * S * (S | 1) : nullptr, nullptr,
                             st));
  }
  if (one) e->mark();
  RotJob uj{mat_at(e->Um(), b0), e->m, uk, cs, S, nullptr, 0, nullptr, 0};
  bool has_u = true;
  if (lazy_state == 1) {
    ISVD_TRY(launch_copy_rows(nb, r, r, uk, cs, S, e->W + b0 * e->wstride(), e->wstride(), e->ld,
                              st));
    has_u = false;
  } else if (lazy_state == 2) {
    uj = RotJob{mat_at(e->Wm(), b0), e->r_base + e->lazy_b, uk, cs, S, nullptr, 0, nullptr, 0};
  }
  // the right side: V itself, or Gv <- Gv Vk while deferred (nothing when
  // the core kernel wrote Vk straight into a fresh Gv)
  RotJob vj{mat_at(e->Vm(), b0), e->n, vk, cs, S, nullptr, 0, nullptr, 0};
  bool has_v = true;
  if (defer) {
    if (vp)
      vj = RotJob{mat_at(e->Gm(), b0), e->vfw + e->vnz, vk, cs, S, nullptr, 0, nullptr, 0};
    else
      has_v = false;
  }
  ZeroFix zf;
  zf.s = e->s + (int64_t)b0 * e->ld;
  zf.lds = e->ld;
  zf.w = r;
  zf.U = lazy_state != 0 ? mat_at(e->Wm(), b0) : mat_at(e->Um(), b0);
  zf.m = lazy_state != 0 ? e->r_base_next + e->lazy_b_next : e->m;
  zf.V = mat_at(e->Vm(), b0);
  zf.n = e->n;
  zf.counter = e->zf_cnt + b0;
  if (defer) zf.vd = e->vdesc(b0, e->vnz);
  bool zfused = false;
  // the completion can ride on the rotation once s is installed (the fused
  // Jacobi writes it directly)
  if (has_u || has_v)
    ISVD_TRY(launch_rotate(nb, r, r, has_u ? uj : vj, (has_u && has_v) ? &vj : nullptr, st,
                           fused ? &zf : nullptr, &zfused));
  if (one) e->mark();
  if (!fused)  // the fused kernel installed s itself
    ISVD_CUDA(cudaMemcpy2DAsync(e->s + (int64_t)b0 * e->ld, sizeof(double) * e->ld, sv,
                                sizeof(double) * S, sizeof(double) * r, nb,
                                cudaMemcpyDeviceToDevice, st));
  if (!zfused)
    ISVD_TRY(launch_complete_zero(nb, r, zf.s, zf.lds, zf.U, zf.m, zf.V, zf.n, st,
                                  defer ? &zf.vd : nullptr));
  return ISVD_OK;
}

// Run `issue(slice)` over the batch: one slice on the engine stream, or
// ngroups slices forked onto the group streams and joined back.
}  // extern "C"
// stream groups a tick of this engine is split into (1: everything on e->st)
static int groups_for(const isvd_engine* e) {
  int G = e->timing ? 1 : e->ngroups;
  if (e->B < 2 * isvd_engine::kGroupMin) G = 1;
  G = std::min(G, e->B / isvd_engine::kGroupMin);
  return G < 1 ? 1 : G;
}

// Small host payloads of a single-group engine (single streams, configs
// 1-4): one H2D on the engine stream itself.  The staging slot cannot be
// overwritten early -- every reader is on the same stream -- so the copy
// stream, its events and the slot tickets (five API calls) are skipped
// (config-4 rows of 40 KB: 103 -> 94 us per synchronised event; config 1:
// enqueue 37 -> 28 us).
static bool small_host_path(const isvd_engine* e, size_t bytes) {
  return groups_for(e) == 1 && !e->pend && bytes <= (size_t(64) << 10);
}

template <class F>
static int run_groups(isvd_engine* e, F&& issue) {
  const int G = groups_for(e);
  e->ngroups_active = G;
  if (G == 1 || (e->pend && e->pend_G != G)) e->join();
  if (G == 1) return issue(Slice{0, e->B, e->st});
  ISVD_TRY(e->ensure_groups(G));
  ISVD_CUDA(cudaEventRecord(e->fork_ev, e->st));
  for (int g = 0; g < G; ++g) {
    const int b0 = (int)((int64_t)e->B * g / G), b1 = (int)((int64_t)e->B * (g + 1) / G);
    ISVD_CUDA(cudaStreamWaitEvent(e->gst[g], e->fork_ev, 0));
    ISVD_TRY(issue(Slice{b0, b1 - b0, e->gst[g]}));
    ISVD_CUDA(cudaEventRecord(e->join_ev[g], e->gst[g]));
    if (!e->async_groups) ISVD_CUDA(cudaStreamWaitEvent(e->st, e->join_ev[g], 0));
  }
  if (e->async_groups) {
    e->pend = true;
    e->pend_G = G;
  }
  return ISVD_OK;
}
extern "C" {

static int append_common(isvd_engine* e, const double* x, int on_device, bool is_row) {
  HP_T0(hp0);
  if (!e || !x) { set_error("null argument"); return ISVD_EINVAL; }
  if (!e->initialized) { set_error("engine not initialised"); return ISVD_ESTATE; }
  e->svdc_valid = false;
  e->okeep.valid = false;
  const int len = is_row ? e->n : e->m;
  // Finiteness of a host payload (the reference's as_vector, linalg.py:31-40)
  // is checked before anything changes the engine's logical state: small
  // payloads on the host, large ones (a 5a row tick carries 8 MB) on the
  // device right after the upload (below) -- the host then waits only for the
  // transfer instead of scanning 8 MB itself.
  const size_t nelem = (size_t)e->B * len;
  const bool device_check = !on_device && nelem >= (size_t(1) << 16);
  // every kernel this tick can launch honours the gate (g_gate) on these paths
  const bool gated = device_check && !e->append_jacobi && !e->sharded && !e->timing && !e->guard &&
                     project_append_gateable(e->B, len, e->r);
  const std::string bad_msg =
      std::string(is_row ? "appended row" : "appended column") + " contains non-finite entries";
  if (!on_device && !device_check && !all_finite(x, nelem)) {
    set_error(bad_msg);
    return ISVD_EINVAL;
  }

  // keep = min(r+1, k, m+1, n) (row) | min(r+1, k, m, n+1) (col): engine.py:122,136
  const int keep = is_row ? std::min(std::min(e->r + 1, e->k), std::min(e->gm() + 1, e->n))
                          : std::min(std::min(e->r + 1, e->k), std::min(e->gm(), e->n + 1));
  const int r_before = e->r;
  if (is_row) {
    if (e->owner) ISVD_TRY(e->grow_rows(e->m + 1));  // appended rows live on the owner
  } else {
    ISVD_TRY(e->grow_cols(e->n + 1));
  }
  if (!is_row) ISVD_TRY(e->flush());  // the column append projects on, and rotates, U
  // a pending right basis is folded by this row append when its projection
  // path can read through Gv, else materialised first
  // full-rank row appends of a deferral-capable batch keep V deferred (the
  // residual joins Z); other appends fold a pending rank-1-only Gv into
  // their V rotation when the projection path can, else materialise V first
  const bool vrow = is_row && e->vdefer_ok() && keep == e->r &&
                    project_append_takes_g(e->B, e->n, e->r);
  if (e->vpend && !vrow && (e->vnz > 0 || !project_append_takes_g(e->B, e->n, e->r)))
    ISVD_TRY(e->flush_v());
  const bool vp = is_row && e->vpend && !vrow;
  const bool vstart = vrow && !e->vpend;
  if (vrow) ISVD_TRY(e->ensure_gv());
  if (vstart) {
    e->vfw = e->r;
    e->vnz = 0;
  }
  const int lazy_state = !(is_row && e->lazy_mode) ? 0 : (e->lazy_active ? 2 : 1);
  // window bookkeeping after this event (used by the completion check)
  e->r_base_next = lazy_state == 1 ? e->r : e->r_base;
  e->lazy_b_next = lazy_state == 1 ? 1 : e->lazy_b + 1;
  // Host payload: one H2D on the copy stream into a double-buffered staging
  // slot, issued before this tick's kernels wait for the previous tick, so
  // the upload overlaps the previous tick's work; the slot is reused only
  // after the tick that last read it has finished.
  g_hprof.add(0, hp0);
  HP_T0(hp1);
  double* staged = nullptr;
  int slot = 0;
  const bool small = !on_device && !device_check && small_host_path(e, sizeof(double) * nelem);
  if (small) {
    slot = e->stage_slot;
    e->stage_slot = (e->stage_slot + 1) % isvd_engine::kStageSlots;
    staged = e->ev + (int64_t)slot * e->B * e->zlen();
    ISVD_CUDA(cudaMemcpyAsync(staged, x, sizeof(double) * nelem, cudaMemcpyHostToDevice, e->st));
  } else if (!on_device) {
    ISVD_TRY(e->ensure_copy_stream());
    slot = e->stage_slot;
    e->stage_slot = (e->stage_slot + 1) % isvd_engine::kStageSlots;
    staged = e->ev + (int64_t)slot * e->B * e->zlen();
    ISVD_TRY(e->ticket_wait(e->cp_st, e->stage_tk[slot]));
    ISVD_CUDA(cudaMemcpyAsync(staged, x, sizeof(double) * e->B * len, cudaMemcpyHostToDevice,
                              e->cp_st));
    if (device_check) {
      ISVD_CUDA(cudaMemsetAsync(e->dflag + 1 + slot, 0, sizeof(int), e->cp_st));
      ISVD_TRY(launch_check_finite(nelem, staged, e->dflag + 1 + slot, e->cp_st));
      ISVD_CUDA(cudaMemcpyAsync((void*)(e->vflag_h + slot), e->dflag + 1 + slot, sizeof(int),
                                cudaMemcpyDeviceToHost, e->cp_st));
    }
    ISVD_CUDA(cudaEventRecord(e->stage_ready, e->cp_st));
    if (device_check && !gated) {
      ISVD_CUDA(cudaEventSynchronize(e->stage_ready));
      if (e->vflag_h[slot]) {
        set_error(bad_msg);
        return ISVD_EINVAL;  // nothing consumed the staging slot; state unchanged
      }
    }
    ISVD_CUDA(cudaStreamWaitEvent(e->st, e->stage_ready, 0));
  }
  g_hprof.add(1, hp1);
  HP_T0(hp2);
  e->ring_slot = (int)(e->ring_cnt % isvd_engine::kRing);
  // Gated tick: the kernels are queued before the verdict is known and skip
  // themselves on the device if the payload was rejected, so the host's wait
  // for the upload overlaps their launch instead of preceding it.
  g_gate = gated ? e->dflag + 1 + slot : nullptr;
  const int rc_issue = run_groups(e, [&](const Slice& sl) {
    const double* xd = x;
    if (!on_device) xd = staged;
    return issue_append(e, sl, xd, len, is_row, keep, lazy_state, vp, vrow, vstart);
  });
  g_gate = nullptr;
  ISVD_TRY(rc_issue);
  g_hprof.add(2, hp2);
  HP_T0(hp3);
  // the staging slot is free again once every group has run this tick (also
  // after a small-path tick: a later large payload reuses the slot from the
  // copy stream)
  if (!on_device) ISVD_TRY(e->ticket_record(e->stage_tk[slot]));
  if (gated) {
    ISVD_CUDA(cudaEventSynchronize(e->stage_ready));
    if (e->vflag_h[slot]) {
      set_error(bad_msg);
      return ISVD_EINVAL;  // every queued kernel of this tick exits at once; state unchanged
    }
  }
  if (vp) e->vpend = false;
  if (vrow) {
    e->vpend = true;
    e->vnz += 1;
  }
  if (lazy_state == 1) {
    e->lazy_active = true;
    e->m_base = e->m;
    e->r_base = e->r;
    e->lazy_b = 1;
  } else if (lazy_state == 2) {
    e->lazy_b += 1;
  }
  if (is_row) {
    if (e->owner) e->m += 1;
    e->m_glob += 1;
  } else {
    e->n += 1;
  }
  e->r = keep;
  if (e->lazy_active && e->lazy_b >= e->lazy_rows) ISVD_TRY(e->flush_u(true));
  if (e->vpend && e->vnz >= kVWin) ISVD_TRY(e->flush_v(true));
  ISVD_TRY(e->guard_step());
  if (e->ngroups_active == 1) e->mark();
  if (e->timing) { e->timed_ticks += 1; e->tick_kind.push_back(0); }
  // K1's main path wrote this tick's (N, rho, xnorm) into the ring slot
  e->rd_used[e->ring_slot] = false;
  e->ring_last = (!e->sharded && project_append_gateable(e->B, len, r_before)) ? e->ring_slot : -1;
  e->ring_cnt += 1;
  e->canonical = false;
  e->step += 1;
  g_hprof.add(3, hp3);
  return ISVD_OK;
}

int isvd_engine_row_append(isvd_engine* e, const double* x, int on_device) {
  return append_common(e, x, on_device, true);
}

int isvd_engine_col_append(isvd_engine* e, const double* y, int on_device) {
  return append_common(e, y, on_device, false);
}

int isvd_engine_rank_one(isvd_engine* e, const int64_t* i, const int64_t* j, const double* delta,
                         int on_device) {
  HP_T0(hr0);
  struct HpEnd {
    double t0;
    ~HpEnd() { g_hprof.add(7, t0); }
  } hp_end{hr0};
  if (!e || !i || !j || !delta) { set_error("null argument"); return ISVD_EINVAL; }
  if (!e->initialized) { set_error("engine not initialised"); return ISVD_ESTATE; }
  e->svdc_valid = false;
  e->okeep.valid = false;
  const int64_t *di = i, *dj = j;
  const double* dd = delta;
  int rslot = 0;
  if (e->sharded) {
    e->join();
    // the owner of row i is decided on the host
    if (on_device) {
      ISVD_CUDA(cudaMemcpyAsync(&e->sh_i, i, sizeof(int64_t), cudaMemcpyDeviceToHost, e->st));
      ISVD_CUDA(cudaMemcpyAsync(&e->sh_j, j, sizeof(int64_t), cudaMemcpyDeviceToHost, e->st));
      ISVD_CUDA(cudaMemcpyAsync(&e->sh_d, delta, sizeof(double), cudaMemcpyDeviceToHost, e->st));
      ISVD_CUDA(cudaStreamSynchronize(e->st));
    } else {
      e->sh_i = i[0];
      e->sh_j = j[0];
      e->sh_d = delta[0];
    }
  }
  if (!on_device) {
    for (int b = 0; b < e->B; ++b) {
      if (!(0 <= i[b] && i[b] < e->gm() && 0 <= j[b] && j[b] < e->n)) {
        set_error("index (" + std::to_string(i[b]) + ", " + std::to_string(j[b]) +
                  ") out of bounds for shape (" + std::to_string(e->gm()) + ", " +
                  std::to_string(e->n) + ")");
        return ISVD_EINVAL;
      }
      if (!std::isfinite(delta[b])) { set_error("delta must be finite"); return ISVD_EINVAL; }
    }
    if (small_host_path(e, 24 * (size_t)e->B)) {
      // (i, j, delta) packed into one H2D on the engine stream
      rslot = e->stage_slot;
      e->stage_slot = (e->stage_slot + 1) % isvd_engine::kStageSlots;
      if (!e->pack_dev) ISVD_TRY(dalloc(&e->pack_dev, (size_t)isvd_engine::kStageSlots * 3 * e->B));
      e->pack_host.resize((size_t)3 * e->B);
      int64_t* hp = e->pack_host.data();
      std::memcpy(hp, i, sizeof(int64_t) * e->B);
      std::memcpy(hp + e->B, j, sizeof(int64_t) * e->B);
      std::memcpy(hp + 2 * e->B, delta, sizeof(double) * e->B);
      int64_t* dp = e->pack_dev + (int64_t)rslot * 3 * e->B;
      ISVD_CUDA(cudaMemcpyAsync(dp, hp, sizeof(int64_t) * 3 * e->B, cudaMemcpyHostToDevice, e->st));
      di = dp;
      dj = dp + e->B;
      dd = reinterpret_cast<const double*>(dp + 2 * e->B);
      rslot = -1;  // no copy-stream ticket
    } else {
    // double-buffered staging on the copy stream, as for appended rows
    ISVD_TRY(e->ensure_copy_stream());
    rslot = e->stage_slot;
    e->stage_slot = (e->stage_slot + 1) % isvd_engine::kStageSlots;
    int64_t* si = e->ei + (int64_t)rslot * e->B;
    int64_t* sj = e->ej + (int64_t)rslot * e->B;
    double* sd = e->ed + (int64_t)rslot * e->B;
    ISVD_TRY(e->ticket_wait(e->cp_st, e->stage_tk[rslot]));
    ISVD_CUDA(cudaMemcpyAsync(si, i, sizeof(int64_t) * e->B, cudaMemcpyHostToDevice, e->cp_st));
    ISVD_CUDA(cudaMemcpyAsync(sj, j, sizeof(int64_t) * e->B, cudaMemcpyHostToDevice, e->cp_st));
    ISVD_CUDA(cudaMemcpyAsync(sd, delta, sizeof(double) * e->B, cudaMemcpyHostToDevice, e->cp_st));
    ISVD_CUDA(cudaEventRecord(e->stage_ready, e->cp_st));
    ISVD_CUDA(cudaStreamWaitEvent(e->st, e->stage_ready, 0));
    di = si; dj = sj; dd = sd;
    }
  } else if (!e->sharded) {
    // device payload: copied into a staging slot on the engine stream and
    // bounds/finiteness-checked there (the caller's buffer is then free
    // once the engine stream passes this point)
    rslot = e->stage_slot;
    e->stage_slot = (e->stage_slot + 1) % isvd_engine::kStageSlots;
    int64_t* si = e->ei + (int64_t)rslot * e->B;
    int64_t* sj = e->ej + (int64_t)rslot * e->B;
    double* sd = e->ed + (int64_t)rslot * e->B;
    ISVD_TRY(e->ticket_wait(e->st, e->stage_tk[rslot]));
    ISVD_TRY(launch_stage_rank1(e->B, i, j, delta, si, sj, sd, e->gm(), e->n,
                                e->dflag + isvd_engine::kDevBad, e->st));
    e->dev_inputs = true;
    di = si; dj = sj; dd = sd;
  }
  const int lazy_state = !e->lazy_mode ? 0 : (e->lazy_active ? 2 : 1);
  e->r_base_next = lazy_state == 1 ? e->r : e->r_base;
  e->lazy_b_next = lazy_state == 1 ? 0 : e->lazy_b;
  if (e->vpend && !e->vdefer_ok()) ISVD_TRY(e->flush_v());
  const bool defer = e->vdefer_ok(), vp = e->vpend;
  if (defer) ISVD_TRY(e->ensure_gv());
  if (defer && !vp) {  // the core writes Vk straight into a fresh Gv
    e->vfw = e->r;
    e->vnz = 0;
  }
  e->ring_slot = (int)(e->ring_cnt % isvd_engine::kRing);
  ISVD_TRY(run_groups(e, [&](const Slice& sl) {
    return issue_rank_one(e, sl, di, dj, dd, lazy_state, defer, vp);
  }));
  if (defer) e->vpend = true;
  if (rslot >= 0 && (!on_device || !e->sharded)) ISVD_TRY(e->ticket_record(e->stage_tk[rslot]));
  if (lazy_state == 1) {
    e->lazy_active = true;
    e->m_base = e->m;
    e->r_base = e->r;
    e->lazy_b = 0;
  }
  ISVD_TRY(e->guard_step());
  if (e->ngroups_active == 1) e->mark();
  if (e->timing) { e->timed_ticks += 1; e->tick_kind.push_back(1); }
  // the fused rank-1 kernel wrote this tick's (N, rho, xnorm) into the ring
  e->rd_used[e->ring_slot] = false;
  e->ring_last = (!e->sharded && e->r <= 32) ? e->ring_slot : -1;
  e->ring_cnt += 1;
  e->canonical = false;
  e->step += 1;
  return ISVD_OK;
}

static int copy_reference(isvd_engine* e) {
  ISVD_TRY(e->canonicalize());
  if (!e->ref || e->ref_cap < e->m) {
    dfree(e->ref);
    e->ref_cap = e->m_cap;
    ISVD_TRY(dalloc(&e->ref, (size_t)e->B * e->ref_cap * e->ld));
  }
  ISVD_TRY(launch_copy_rows(e->B, e->m, e->r, e->U, e->ustride(), e->ld, e->ref,
                            (int64_t)e->ref_cap * e->ld, e->ld, e->st));
  e->ref_m = e->m;
  e->ref_r = e->r;
  e->has_ref = true;
  return ISVD_OK;
}

int isvd_engine_refresh(isvd_engine* e, int store_reference) {
  if (e) e->join();
  if (!e || !e->initialized) { set_error("engine not initialised"); return ISVD_ESTATE; }
  ISVD_TRY(e->grow_rank(e->k));
  ISVD_TRY(e->factor_tracked());
  ISVD_TRY(launch_sumsq(e->B, e->m, e->n, e->A, e->astride(), e->n_cap, e->N, e->st));
  ISVD_TRY(e->allreduce(e->N, 1));
  if (store_reference) ISVD_TRY(copy_reference(e));
  ISVD_CUDA(cudaStreamSynchronize(e->st));
  return ISVD_OK;
}

int isvd_engine_set_reference(isvd_engine* e) {
  if (e) e->join();
  if (!e || !e->initialized) { set_error("engine not initialised"); return ISVD_ESTATE; }
  ISVD_TRY(copy_reference(e));
  return ISVD_OK;
}

int isvd_engine_set_rank(isvd_engine* e, int k_new) {
  if (e) e->join();
  if (!e) { set_error("null engine"); return ISVD_EINVAL; }
  if (k_new < 1) { set_error("work rank must be >= 1, got " + std::to_string(k_new)); return ISVD_EINVAL; }
  e->svdc_valid = false;
  ISVD_TRY(e->flush());
  ISVD_TRY(e->grow_rank(k_new));
  e->k = k_new;
  if (e->r > k_new) e->r = k_new;
  return ISVD_OK;
}

int isvd_engine_shape(const isvd_engine* e, int* batch, int* m, int* n, int* rank, int* work_rank,
                      int64_t* step) {
  if (!e) { set_error("null engine"); return ISVD_EINVAL; }
  if (batch) *batch = e->B;
  if (m) *m = e->gm();
  if (n) *n = e->n;
  if (rank) *rank = e->r;
  if (work_rank) *work_rank = e->k;
  if (step) *step = e->step;
  return ISVD_OK;
}

int isvd_engine_has_reference(const isvd_engine* e, int* has_ref, int* ref_m, int* ref_r) {
  if (!e) { set_error("null engine"); return ISVD_EINVAL; }
  *has_ref = e->has_ref;
  *ref_m = e->ref_m;
  *ref_r = e->ref_r;
  return ISVD_OK;
}

int isvd_engine_get_factors(isvd_engine* e, int b, double* u, double* sv, double* v) {
  if (e) e->join();
  if (!e || b < 0 || b >= e->B) { set_error("bad stream index"); return ISVD_EINVAL; }
  // the singular values alone need neither the deferred bases materialised
  // nor the sign convention applied (metrics read them every tick)
  if (u || v) ISVD_TRY(e->canonicalize());
  const int r = e->r;
  if (r > 0) {
    if (u)
      ISVD_CUDA(cudaMemcpy2DAsync(u, sizeof(double) * r, e->U + b * e->ustride(), sizeof(double) * e->ld,
                                  sizeof(double) * r, e->m, cudaMemcpyDeviceToHost, e->st));
    if (v)
      ISVD_CUDA(cudaMemcpy2DAsync(v, sizeof(double) * r, e->V + b * e->vstride(), sizeof(double) * e->ld,
                                  sizeof(double) * r, e->n, cudaMemcpyDeviceToHost, e->st));
    if (sv)
      ISVD_CUDA(cudaMemcpyAsync(sv, e->s + (int64_t)b * e->ld, sizeof(double) * r,
                                cudaMemcpyDeviceToHost, e->st));
  }
  ISVD_CUDA(cudaStreamSynchronize(e->st));
  return e->dev_input_verdict();
}

int isvd_engine_get_tracked(isvd_engine* e, int b, double* a) {
  if (e) e->join();
  if (!e || b < 0 || b >= e->B || !a) { set_error("bad argument"); return ISVD_EINVAL; }
  ISVD_CUDA(cudaMemcpy2DAsync(a, sizeof(double) * e->n, e->A + b * e->astride(),
                              sizeof(double) * e->n_cap, sizeof(double) * e->n, e->m,
                              cudaMemcpyDeviceToHost, e->st));
  ISVD_CUDA(cudaStreamSynchronize(e->st));
  return ISVD_OK;
}

int isvd_engine_get_reference(isvd_engine* e, int b, double* out) {
  if (e) e->join();
  if (!e || b < 0 || b >= e->B || !out) { set_error("bad argument"); return ISVD_EINVAL; }
  if (!e->has_ref) { set_error("no reference stored"); return ISVD_ESTATE; }
  ISVD_CUDA(cudaMemcpy2DAsync(out, sizeof(double) * e->ref_r, e->ref + (int64_t)b * e->ref_cap * e->ld,
                              sizeof(double) * e->ld, sizeof(double) * e->ref_r, e->ref_m,
                              cudaMemcpyDeviceToHost, e->st));
  ISVD_CUDA(cudaStreamSynchronize(e->st));
  return ISVD_OK;
}

int isvd_engine_get_scalars(isvd_engine* e, double* sq_norm, double* last_residual,
                            double* last_input_norm) {
  if (e) e->join();
  if (!e) { set_error("null engine"); return ISVD_EINVAL; }
  if (sq_norm) ISVD_CUDA(cudaMemcpyAsync(sq_norm, e->N, sizeof(double) * e->B, cudaMemcpyDeviceToHost, e->st));
  if (last_residual) ISVD_CUDA(cudaMemcpyAsync(last_residual, e->rho, sizeof(double) * e->B, cudaMemcpyDeviceToHost, e->st));
  if (last_input_norm) ISVD_CUDA(cudaMemcpyAsync(last_input_norm, e->xnorm, sizeof(double) * e->B, cudaMemcpyDeviceToHost, e->st));
  ISVD_CUDA(cudaStreamSynchronize(e->st));
  return e->dev_input_verdict();
}

int isvd_engine_scalars_async(isvd_engine* e, double* host, int slot) {
  if (!e || !host || slot < 0 || slot >= 8) { set_error("bad argument"); return ISVD_EINVAL; }
  if (e->ring_last >= 0) {
    // the last tick's kernels left (N, rho, xnorm) in a ring slot: copy it on
    // the read-back stream once every group has finished that tick
    if (!e->rd_st) {
      ISVD_CUDA(cudaStreamCreateWithFlags(&e->rd_st, cudaStreamNonBlocking));
      for (auto& ev : e->rd_done) ISVD_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    }
    ISVD_TRY(e->ticket_record(e->rd_tk));
    ISVD_TRY(e->ticket_wait(e->rd_st, e->rd_tk));
    ISVD_CUDA(cudaMemcpyAsync(host, e->ring_row(e->ring_last, 0), sizeof(double) * 3 * e->B,
                              cudaMemcpyDeviceToHost, e->rd_st));
    ISVD_CUDA(cudaEventRecord(e->rd_done[e->ring_last], e->rd_st));
    e->rd_used[e->ring_last] = true;
    return e->ticket_record_on(e->sc_tk[slot], e->rd_st);
  }
  // Pinned (device-mapped) destinations are written by one small kernel per
  // group straight over PCIe: three DMA copies per group would each hold the
  // group stream for their latency between two ticks.  Others: DMA copies.
  double* mapped = nullptr;
  {
    cudaPointerAttributes pa;
    if (cudaPointerGetAttributes(&pa, host) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
        pa.devicePointer)
      mapped = static_cast<double*>(pa.devicePointer);
    cudaGetLastError();
  }
  // per group on the group streams while they run ahead (no join), else on st
  const int G = e->pend ? e->pend_G : 1;
  for (int g = 0; g < G; ++g) {
    const int b0 = (int)((int64_t)e->B * g / G), b1 = (int)((int64_t)e->B * (g + 1) / G);
    cudaStream_t s2 = e->pend ? e->gst[g] : e->st;
    if (mapped) {
      ISVD_TRY(launch_scalars_out(b0, b1 - b0, e->B, e->N, e->rho, e->xnorm, mapped, s2));
      continue;
    }
    const size_t nb = sizeof(double) * (b1 - b0);
    ISVD_CUDA(cudaMemcpyAsync(host + b0, e->N + b0, nb, cudaMemcpyDeviceToHost, s2));
    ISVD_CUDA(cudaMemcpyAsync(host + e->B + b0, e->rho + b0, nb, cudaMemcpyDeviceToHost, s2));
    ISVD_CUDA(cudaMemcpyAsync(host + 2 * e->B + b0, e->xnorm + b0, nb, cudaMemcpyDeviceToHost, s2));
  }
  return e->ticket_record(e->sc_tk[slot]);
}

int isvd_engine_scalars_wait(isvd_engine* e, int slot) {
  if (!e || slot < 0 || slot >= 8 || e->sc_tk[slot].n == 0) { set_error("bad ticket"); return ISVD_EINVAL; }
  return e->ticket_sync(e->sc_tk[slot]);
}

int isvd_engine_set_factors(isvd_engine* e, int b, int r, const double* u, const double* sv,
                            const double* v) {
  if (e) e->join();
  if (!e || b < 0 || b >= e->B) { set_error("bad stream index"); return ISVD_EINVAL; }
  if (r != e->r) { set_error("set_factors: rank must match the current factor width"); return ISVD_EINVAL; }
  e->svdc_valid = false;
  ISVD_TRY(e->canonicalize());
  ISVD_CUDA(cudaMemcpy2DAsync(e->U + b * e->ustride(), sizeof(double) * e->ld, u, sizeof(double) * r,
                              sizeof(double) * r, e->m, cudaMemcpyHostToDevice, e->st));
  ISVD_CUDA(cudaMemcpy2DAsync(e->V + b * e->vstride(), sizeof(double) * e->ld, v, sizeof(double) * r,
                              sizeof(double) * r, e->n, cudaMemcpyHostToDevice, e->st));
  ISVD_CUDA(cudaMemcpyAsync(e->s + (int64_t)b * e->ld, sv, sizeof(double) * r, cudaMemcpyHostToDevice, e->st));
  ISVD_CUDA(cudaStreamSynchronize(e->st));
  e->canonical = true;  // the caller's factors are taken verbatim
  return ISVD_OK;
}

int isvd_engine_put_reference(isvd_engine* e, int b, int ref_m, int ref_r, const double* refh) {
  if (e) e->join();
  if (!e || b < 0 || b >= e->B || ref_r < 0 || ref_m < 0) { set_error("bad argument"); return ISVD_EINVAL; }
  if (!refh) { e->has_ref = false; return ISVD_OK; }
  if (ref_r > e->ld) { set_error("reference wider than the rank capacity"); return ISVD_EINVAL; }
  if (!e->ref || e->ref_cap < ref_m) {
    dfree(e->ref);
    e->ref_cap = std::max(ref_m, e->m_cap);
    ISVD_TRY(dalloc(&e->ref, (size_t)e->B * e->ref_cap * e->ld));
  }
  ISVD_CUDA(cudaMemcpy2DAsync(e->ref + (int64_t)b * e->ref_cap * e->ld, sizeof(double) * e->ld, refh,
                              sizeof(double) * ref_r, sizeof(double) * ref_r, ref_m,
                              cudaMemcpyHostToDevice, e->st));
  ISVD_CUDA(cudaStreamSynchronize(e->st));
  e->ref_m = ref_m;
  e->ref_r = ref_r;
  e->has_ref = true;
  return ISVD_OK;
}

int isvd_engine_device_views(isvd_engine* e, double** u, int64_t* u_stride, int* ldu, double** v,
                             int64_t* v_stride, int* ldv, double** s, int* lds, double** a,
                             int64_t* a_stride, int* lda) {
  if (e) e->join();
  if (!e) { set_error("null engine"); return ISVD_EINVAL; }
  ISVD_TRY(e->flush());
  e->svdc_valid = false;  // the caller may write through the views
  e->okeep.valid = false;
  if (u) *u = e->U;
  if (u_stride) *u_stride = e->ustride();
  if (ldu) *ldu = e->ld;
  if (v) *v = e->V;
  if (v_stride) *v_stride = e->vstride();
  if (ldv) *ldv = e->ld;
  if (s) *s = e->s;
  if (lds) *lds = e->ld;
  if (a) *a = e->A;
  if (a_stride) *a_stride = e->astride();
  if (lda) *lda = e->n_cap;
  return ISVD_OK;
}

int isvd_engine_flush(isvd_engine* e) {
  if (e) e->join();
  if (!e) { set_error("null engine"); return ISVD_EINVAL; }
  return e->flush();
}

// ---- snapshot / restore (device-side checkpoint of the whole engine state)
int isvd_engine_snapshot(isvd_engine* e) {
  if (e) e->join();
  if (!e || !e->initialized) { set_error("engine not initialised"); return ISVD_ESTATE; }
  ISVD_TRY(e->flush());
  auto& S = e->snap;
  const size_t nu = (size_t)e->B * e->ustride(), nv = (size_t)e->B * e->vstride();
  const size_t na = (size_t)e->B * e->astride(), ns = (size_t)e->B * e->ld;
  if (S.nu != nu) { dfree(S.U); ISVD_TRY(dalloc(&S.U, nu)); S.nu = nu; }
  if (S.nv != nv) { dfree(S.V); ISVD_TRY(dalloc(&S.V, nv)); S.nv = nv; }
  if (S.na != na) { dfree(S.A); ISVD_TRY(dalloc(&S.A, na)); S.na = na; }
  if (S.ns != ns) { dfree(S.s); ISVD_TRY(dalloc(&S.s, ns)); S.ns = ns; }
  if (!S.N) ISVD_TRY(dalloc(&S.N, (size_t)e->B * 3));
  ISVD_CUDA(cudaMemcpyAsync(S.U, e->U, nu * 8, cudaMemcpyDeviceToDevice, e->st));
  ISVD_CUDA(cudaMemcpyAsync(S.V, e->V, nv * 8, cudaMemcpyDeviceToDevice, e->st));
  ISVD_CUDA(cudaMemcpyAsync(S.A, e->A, na * 8, cudaMemcpyDeviceToDevice, e->st));
  ISVD_CUDA(cudaMemcpyAsync(S.s, e->s, ns * 8, cudaMemcpyDeviceToDevice, e->st));
  ISVD_CUDA(cudaMemcpyAsync(S.N, e->N, e->B * 8, cudaMemcpyDeviceToDevice, e->st));
  ISVD_CUDA(cudaMemcpyAsync(S.N + e->B, e->rho, e->B * 8, cudaMemcpyDeviceToDevice, e->st));
  ISVD_CUDA(cudaMemcpyAsync(S.N + 2 * e->B, e->xnorm, e->B * 8, cudaMemcpyDeviceToDevice, e->st));
  S.m = e->m; S.n = e->n; S.r = e->r; S.k = e->k; S.step = e->step; S.m_glob = e->m_glob;
  S.m_cap = e->m_cap; S.n_cap = e->n_cap; S.ld = e->ld; S.canonical = e->canonical;
  S.has_ref = e->has_ref && e->ref;
  if (S.has_ref) {
    const size_t nref = (size_t)e->B * e->ref_cap * e->ld;
    if (S.nref != nref) { dfree(S.ref); ISVD_TRY(dalloc(&S.ref, nref)); S.nref = nref; }
    ISVD_CUDA(cudaMemcpyAsync(S.ref, e->ref, nref * 8, cudaMemcpyDeviceToDevice, e->st));
    S.ref_m = e->ref_m; S.ref_r = e->ref_r; S.ref_cap = e->ref_cap;
  }
  S.valid = true;
  ISVD_CUDA(cudaStreamSynchronize(e->st));
  return ISVD_OK;
}

int isvd_engine_restore(isvd_engine* e) {
  if (e) e->join();
  if (!e || !e->snap.valid) { set_error("no snapshot to restore"); return ISVD_ESTATE; }
  e->svdc_valid = false;
  e->okeep.valid = false;
  auto& S = e->snap;
  if (S.m_cap != e->m_cap || S.n_cap != e->n_cap || S.ld != e->ld) {
    set_error("capacities changed since the snapshot");
    return ISVD_ESTATE;
  }
  e->lazy_active = false;
  e->lazy_b = 0;
  e->vpend = false;
  e->vnz = 0;
  ISVD_CUDA(cudaMemcpyAsync(e->U, S.U, S.nu * 8, cudaMemcpyDeviceToDevice, e->st));
  ISVD_CUDA(cudaMemcpyAsync(e->V, S.V, S.nv * 8, cudaMemcpyDeviceToDevice, e->st));
  ISVD_CUDA(cudaMemcpyAsync(e->A, S.A, S.na * 8, cudaMemcpyDeviceToDevice, e->st));
  ISVD_CUDA(cudaMemcpyAsync(e->s, S.s, S.ns * 8, cudaMemcpyDeviceToDevice, e->st));
  ISVD_CUDA(cudaMemcpyAsync(e->N, S.N, e->B * 8, cudaMemcpyDeviceToDevice, e->st));
  ISVD_CUDA(cudaMemcpyAsync(e->rho, S.N + e->B, e->B * 8, cudaMemcpyDeviceToDevice, e->st));
  ISVD_CUDA(cudaMemcpyAsync(e->xnorm, S.N + 2 * e->B, e->B * 8, cudaMemcpyDeviceToDevice, e->st));
  e->m = S.m; e->n = S.n; e->r = S.r; e->k = S.k; e->step = S.step; e->canonical = S.canonical;
  e->m_glob = S.m_glob;
  // the drift reference belongs to the checkpointed timeline too
  e->has_ref = S.has_ref;
  if (S.has_ref) {
    if (!e->ref || e->ref_cap != S.ref_cap) {
      dfree(e->ref);
      ISVD_TRY(dalloc(&e->ref, S.nref));
      e->ref_cap = S.ref_cap;
    }
    ISVD_CUDA(cudaMemcpyAsync(e->ref, S.ref, S.nref * 8, cudaMemcpyDeviceToDevice, e->st));
    e->ref_m = S.ref_m;
    e->ref_r = S.ref_r;
  }
  ISVD_CUDA(cudaStreamSynchronize(e->st));
  return ISVD_OK;
}

int isvd_engine_set_reortho_threshold(isvd_engine* e, double threshold) {
  if (e) e->join();
  if (!e) { set_error("null engine"); return ISVD_EINVAL; }
  e->reortho_threshold = threshold;
  return ISVD_OK;
}

int isvd_engine_set_lazy(isvd_engine* e, int on) {
  if (e) e->join();
  if (!e) { set_error("null engine"); return ISVD_EINVAL; }
  if (e->sharded && !on) { set_error("eager U rotation is not available in shard mode"); return ISVD_EINVAL; }
  ISVD_TRY(e->flush());
  e->lazy_mode = on != 0;
  return ISVD_OK;
}

int isvd_engine_set_lazy_window(isvd_engine* e, int rows) {
  if (e) e->join();
  if (!e) { set_error("null engine"); return ISVD_EINVAL; }
  if (rows < 1 || rows > 1 << 16) { set_error("lazy window out of range"); return ISVD_EINVAL; }
  ISVD_TRY(e->flush());
  ISVD_CUDA(cudaStreamSynchronize(e->st));
  e->lazy_rows = rows;
  dfree(e->W);
  ISVD_TRY(dalloc(&e->W, (size_t)e->B * e->wstride()));
  ISVD_CUDA(cudaMemsetAsync(e->W, 0, sizeof(double) * e->B * e->wstride(), e->st));
  return ISVD_OK;
}

int isvd_engine_lazy_window(isvd_engine* e) { return e ? e->lazy_rows : -1; }

int isvd_engine_set_vdefer(isvd_engine* e, int mode) {
  if (e) e->join();
  if (!e) { set_error("null engine"); return ISVD_EINVAL; }
  if (mode < 0 || mode > 2) { set_error("vdefer mode must be 0, 1 or 2"); return ISVD_EINVAL; }
  ISVD_TRY(e->flush_v());
  e->vdefer_mode = mode;
  return ISVD_OK;
}

int isvd_engine_set_groups(isvd_engine* e, int groups) {
  if (!e) { set_error("null engine"); return ISVD_EINVAL; }
  if (groups < 1 || groups > 64) { set_error("groups must be in 1..64"); return ISVD_EINVAL; }
  e->ngroups = groups;
  return ISVD_OK;
}

int isvd_engine_set_append_solver(isvd_engine* e, int jacobi) {
  if (e) e->join();
  if (!e) { set_error("null engine"); return ISVD_EINVAL; }
  e->append_jacobi = jacobi != 0;
  return ISVD_OK;
}

int isvd_engine_set_timing(isvd_engine* e, int on) {
  if (e) e->join();
  if (!e) { set_error("null engine"); return ISVD_EINVAL; }
  e->timing = on != 0;
  return ISVD_OK;
}

int isvd_engine_phase_times(isvd_engine* e, double* ms, int64_t* ticks) {
  if (e) e->join();
  if (!e || !ms) { set_error("bad argument"); return ISVD_EINVAL; }
  ISVD_CUDA(cudaStreamSynchronize(e->st));
  for (int p = 0; p < 10; ++p) ms[p] = 0.0;
  int64_t cnt[2] = {0, 0};
  const size_t nt = e->ev_marks.size() / 5;
  for (size_t t = 0; t < nt; ++t) {
    const int kind = t < e->tick_kind.size() ? e->tick_kind[t] : 0;
    cnt[kind] += 1;
    for (int p = 0; p < 4; ++p) {
      float f = 0.f;
      ISVD_CUDA(cudaEventElapsedTime(&f, e->ev_marks[t * 5 + p], e->ev_marks[t * 5 + p + 1]));
      ms[kind * 4 + p] += f;
    }
  }
  if (ticks) { ticks[0] = cnt[0]; ticks[1] = cnt[1]; }
  // [8] = summed flush-rotation ms, [9] = their algorithmic bytes; ticks[2] = flushes
  ms[8] = 0.0;
  for (size_t f = 0; f + 1 < e->flush_marks.size(); f += 2) {
    float v = 0.f;
    ISVD_CUDA(cudaEventElapsedTime(&v, e->flush_marks[f], e->flush_marks[f + 1]));
    ms[8] += v;
  }
  ms[9] = e->flush_bytes;
  if (ticks) ticks[2] = (int64_t)(e->flush_marks.size() / 2);
  for (auto ev : e->flush_marks) cudaEventDestroy(ev);
  e->flush_marks.clear();
  e->flush_bytes = 0.0;
  for (auto ev : e->ev_marks) e->ev_pool.push_back(ev);
  e->ev_marks.clear();
  e->tick_kind.clear();
  e->timed_ticks = 0;
  return ISVD_OK;
}

int isvd_engine_canonicalize(isvd_engine* e) {
  if (e) e->join();
  if (!e) { set_error("null engine"); return ISVD_EINVAL; }
  return e->canonicalize();
}

int isvd_engine_synchronize(isvd_engine* e) {
  if (e) e->join();
  if (!e) { set_error("null engine"); return ISVD_EINVAL; }
  ISVD_CUDA(cudaStreamSynchronize(e->st));
  return e->dev_input_verdict();
}

int isvd_engine_streams(isvd_engine* e, void** out, int cap) {
  if (!e) { set_error("null engine"); return ISVD_EINVAL; }
  int cnt = 0;
  if (out && cap > 0) out[cnt] = (void*)e->st;
  cnt += 1;
  for (auto g : e->gst) {
    if (out && cnt < cap) out[cnt] = (void*)g;
    cnt += 1;
  }
  return cnt;
}

// ------------------------------------------------------------------ metrics

int isvd_engine_frob_error(isvd_engine* e, double* out) {
  if (e) e->join();
  if (!e || !e->initialized) { set_error("engine not initialised"); return ISVD_ESTATE; }
  ISVD_TRY(e->flush());
  ISVD_TRY(e->ensure_work(0, 0, (int64_t)e->B * frob_nblk(e->m, e->n), e->B));
  ISVD_TRY(launch_frob_error_sq(e->B, e->m, e->n, e->r, e->A, e->astride(), e->n_cap, e->Um(), e->s,
                                e->ld, e->Vm(), e->wpart, e->wout, e->st));
  ISVD_TRY(e->allreduce(e->wout, e->B));  // row shards: sum of the per-shard squares
  ISVD_CUDA(cudaMemcpyAsync(out, e->wout, sizeof(double) * e->B, cudaMemcpyDeviceToHost, e->st));
  ISVD_CUDA(cudaStreamSynchronize(e->st));
  for (int b = 0; b < e->B; ++b) out[b] = std::sqrt(out[b]);
  return ISVD_OK;
}

int isvd_engine_risk(isvd_engine* e, int t, const double* w, int P, double* cov_out,
                     double* diag_out, double* out) {
  if (e) e->join();
  if (!e || !e->initialized) { set_error("engine not initialised"); return ISVD_ESTATE; }
  if (!w || !out || P < 1) { set_error("risk: bad argument"); return ISVD_EINVAL; }
  if (t < 2) { set_error("need at least 2 rows for a covariance, got t=" + std::to_string(t)); return ISVD_EINVAL; }
  if (e->sharded) { set_error("risk needs the whole tracked matrix (not in shard mode)"); return ISVD_EINVAL; }
  ISVD_TRY(e->flush_v());
  const int B = e->B, n = e->n;
  double *wd = nullptr, *cd = nullptr, *dd = nullptr, *od = nullptr;
  int rc = ISVD_OK;
  auto T = [&](int v) { if (rc == ISVD_OK) rc = v; };
  T(dalloc(&wd, (size_t)P * n));
  T(dalloc(&od, (size_t)B * P * 4));
  if (cov_out) T(dalloc(&cd, (size_t)B * n * n));
  if (diag_out) T(dalloc(&dd, (size_t)B * n));
  if (rc == ISVD_OK)
    T(cudaMemcpyAsync(wd, w, sizeof(double) * P * n, cudaMemcpyHostToDevice, e->st) == cudaSuccess
          ? ISVD_OK : ISVD_ENODEV);
  if (rc == ISVD_OK)
    T(launch_risk(B, n, e->r, e->Vm(), e->s, e->ld, e->A, e->astride(), e->n_cap, e->m,
                  1.0 / (t - 1.0), wd, P, cd, dd, od, e->st));
  if (rc == ISVD_OK) {
    cudaMemcpyAsync(out, od, sizeof(double) * B * P * 4, cudaMemcpyDeviceToHost, e->st);
    if (cov_out) cudaMemcpyAsync(cov_out, cd, sizeof(double) * B * n * n, cudaMemcpyDeviceToHost, e->st);
    if (diag_out) cudaMemcpyAsync(diag_out, dd, sizeof(double) * B * n, cudaMemcpyDeviceToHost, e->st);
    if (cudaStreamSynchronize(e->st) != cudaSuccess) { set_error("risk: device failure"); rc = ISVD_ENODEV; }
  }
  if (rc == ISVD_OK)
    for (int i = 0; i < B * P; ++i)
      if (out[(size_t)i * 4 + 3] < -1e-10) {
        set_error("covariance is not PSD: w'Cw = " + std::to_string(out[(size_t)i * 4 + 3]));
        rc = ISVD_EINVAL;
        break;
      }
  cudaStreamSynchronize(e->st);
  dfree(wd); dfree(cd); dfree(dd); dfree(od);
  return rc;
}

int isvd_low_rank_cov(int n, int r, const double* v, const double* s, int t, double* cov) {
  if (n < 1 || r < 0 || !cov || (r > 0 && (!v || !s))) { set_error("bad argument"); return ISVD_EINVAL; }
  if (t < 2) { set_error("need at least 2 rows for a covariance, got t=" + std::to_string(t)); return ISVD_EINVAL; }
  ISVD_TRY(check_device());
  double *vd = nullptr, *sd = nullptr, *cd = nullptr;
  int rc = ISVD_OK;
  auto T = [&](int x) { if (rc == ISVD_OK) rc = x; };
  const int rr = std::max(r, 1);
  T(dalloc(&vd, (size_t)n * rr));
  T(dalloc(&sd, (size_t)rr));
  T(dalloc(&cd, (size_t)n * n));
  cudaStream_t st = 0;
  if (rc == ISVD_OK && r > 0) {
    T(cudaMemcpy(vd, v, sizeof(double) * n * r, cudaMemcpyHostToDevice) == cudaSuccess ? ISVD_OK : ISVD_ENODEV);
    T(cudaMemcpy(sd, s, sizeof(double) * r, cudaMemcpyHostToDevice) == cudaSuccess ? ISVD_OK : ISVD_ENODEV);
  }
  if (rc == ISVD_OK)
    T(launch_risk(1, n, r, Mat{vd, 0, rr}, sd, rr, nullptr, 0, 0, 0, 1.0 / (t - 1.0), nullptr, 0,
                  cd, nullptr, nullptr, st));
  if (rc == ISVD_OK)
    T(cudaMemcpy(cov, cd, sizeof(double) * n * n, cudaMemcpyDeviceToHost) == cudaSuccess ? ISVD_OK : ISVD_ENODEV);
  dfree(vd); dfree(sd); dfree(cd);
  return rc;
}

static int gram_defect(isvd_engine* e, Mat X, int rows, int w, double* host_out,
                       bool row_sharded = false) {
  ISVD_TRY(e->ensure_work(0, 0, gram_part_elems(e->B, rows, w, w), (int64_t)e->B * w * w + e->B));
  ISVD_TRY(launch_gram(e->B, rows, w, w, X, X, e->wpart, e->wout, e->st));
  if (row_sharded) ISVD_TRY(e->allreduce(e->wout, (int64_t)e->B * w * w));
  ISVD_TRY(launch_defect(e->B, w, e->wout, e->wout + (int64_t)e->B * w * w, e->st));
  ISVD_CUDA(cudaMemcpyAsync(host_out, e->wout + (int64_t)e->B * w * w, sizeof(double) * e->B,
                            cudaMemcpyDeviceToHost, e->st));
  ISVD_CUDA(cudaStreamSynchronize(e->st));
  return ISVD_OK;
}

int isvd_engine_ortho_defect(isvd_engine* e, double* du, double* dv) {
  if (e) e->join();
  if (!e || !e->initialized) { set_error("engine not initialised"); return ISVD_ESTATE; }
  ISVD_TRY(e->flush());
  if (du) ISVD_TRY(gram_defect(e, e->Um(), e->m, e->r, du, e->sharded));
  if (dv) ISVD_TRY(gram_defect(e, e->Vm(), e->n, e->r, dv));
  return ISVD_OK;
}

int isvd_engine_angle(isvd_engine* e, int which, const double* q, int q_cols, int on_device,
                      double* out) {
  if (e) e->join();
  if (!e || !e->initialized || !out) { set_error("engine not initialised"); return ISVD_ESTATE; }
  ISVD_TRY(e->flush());
  const int B = e->B, m = e->m, r = e->r;
  Mat Qm;
  double* qbuf = nullptr;
  if (which == 0) {
    if (!e->has_ref || e->ref_m != m || e->ref_r != r) {
      for (int b = 0; b < B; ++b) out[b] = -1.0;
      return ISVD_OK;
    }
    Qm = Mat{e->ref, (int64_t)e->ref_cap * e->ld, e->ld};
  } else {
    if (!q) { set_error("basis is null"); return ISVD_EINVAL; }
    if (q_cols != r) {
      set_error("column counts differ: " + std::to_string(r) + " vs " + std::to_string(q_cols));
      return ISVD_EINVAL;
    }
    if (r == 0) { set_error("subspaces must have at least one column"); return ISVD_EINVAL; }
    if (on_device) {
      Qm = Mat{const_cast<double*>(q), (int64_t)m * q_cols, q_cols};
    } else {
      ISVD_TRY(dalloc(&qbuf, (size_t)B * m * q_cols));
      cudaMemcpyAsync(qbuf, q, sizeof(double) * B * m * q_cols, cudaMemcpyHostToDevice, e->st);
      Qm = Mat{qbuf, (int64_t)m * q_cols, q_cols};
    }
  }
  int rc = ISVD_OK;
  std::vector<double> d1(B), d2(B);
  rc = gram_defect(e, e->Um(), m, r, d1.data(), e->sharded);
  if (rc == ISVD_OK) rc = gram_defect(e, Qm, m, r, d2.data(), e->sharded);
  if (rc == ISVD_OK) {
    for (int b = 0; b < B; ++b)
      if (d1[b] > 1e-6 || d2[b] > 1e-6) {
        set_error(std::string(d1[b] > 1e-6 ? "q1" : "q2") + " is not orthonormal (defect > 1e-6)");
        rc = ISVD_EINVAL;
        break;
      }
  }
  if (rc == ISVD_OK) {
    // C = U^T Q (r x r) -> sigma_min via the core SVD kernel
    int S = e->S();
    rc = e->ensure_work(0, 0, gram_part_elems(B, m, r, r), (int64_t)B * r * r + B);
    if (rc == ISVD_OK) rc = launch_gram(B, m, r, r, e->Um(), Qm, e->wpart, e->wout, e->st);
    if (rc == ISVD_OK) rc = e->allreduce(e->wout, (int64_t)B * r * r);  // U^T Q over shards
    if (rc == ISVD_OK)
      rc = launch_core_svd(B, r, e->wout, (int64_t)r * r, r, e->uk, e->vk, e->cstride(), S, e->sv,
                           S, e->vscr, nullptr, e->st);
    if (rc == ISVD_OK) {
      std::vector<double> svh((size_t)B * S);
      cudaMemcpyAsync(svh.data(), e->sv, sizeof(double) * B * S, cudaMemcpyDeviceToHost, e->st);
      if (cudaStreamSynchronize(e->st) != cudaSuccess) {
        set_error("angle: device failure");
        rc = ISVD_ENODEV;
      } else {
        for (int b = 0; b < B; ++b) {
          double cmin = svh[(size_t)b * S + r - 1];
          out[b] = std::acos(std::min(1.0, std::max(0.0, cmin)));
        }
      }
    }
  }
  if (qbuf) {
    cudaStreamSynchronize(e->st);
    cudaFree(qbuf);
  }
  return rc;
}

static int oracle_common(int B, int m, int n, const double* a_dev, int64_t a_stride, int lda,
                         int w_keep, double* s_host, double* u_host, double* vt_host,
                         cudaStream_t st, OracleKeep* keep = nullptr) {
  const int w = std::max(0, std::min(w_keep, std::min(m, n)));
  DenseSvdPlan P = dense_svd_plan(m, n, w);
  const int nc = P.nc;
  const int ldw = round_up(std::max(w, 1), 8);
  double *x = nullptr, *jac = nullptr, *U = nullptr, *V = nullptr, *sa = nullptr, *sw = nullptr;
  int* fl = nullptr;
  std::vector<int> hf(B);
  int rc = ISVD_OK;
  auto T = [&](int v) { if (rc == ISVD_OK) rc = v; };
  T(dalloc(&x, (size_t)B * P.x_elems()));
  T(dalloc(&jac, (size_t)B * P.j_elems()));
  T(dalloc(&U, (size_t)B * m * ldw));
  T(dalloc(&V, (size_t)B * n * ldw));
  T(dalloc(&sa, (size_t)B * nc));
  T(dalloc(&sw, (size_t)B * ldw));
  T(dalloc(&fl, (size_t)B));
  if (rc == ISVD_OK) {
    Mat Um{U, (int64_t)m * ldw, ldw}, Vm{V, (int64_t)n * ldw, ldw};
    T(dense_svd_run(B, m, n, a_dev, a_stride, lda, w, Um, Vm, sw, ldw, sa, nc, x, jac, fl, hf.data(),
                    st, nullptr));
    if (w > 0) {
      T(launch_complete_zero(B, w, sw, ldw, Um, m, Vm, n, st));
      T(launch_canonicalize(B, w, Um, m, Vm, n, st));
    }
    if (rc == ISVD_OK && s_host)
      T(cudaMemcpyAsync(s_host, sa, sizeof(double) * B * nc, cudaMemcpyDeviceToHost, st) == cudaSuccess
            ? ISVD_OK : ISVD_ENODEV);
    if (rc == ISVD_OK && u_host && w > 0)
      for (int b = 0; b < B && rc == ISVD_OK; ++b)
        T(cudaMemcpy2DAsync(u_host + (size_t)b * m * w, sizeof(double) * w, U + (size_t)b * m * ldw,
                            sizeof(double) * ldw, sizeof(double) * w, m, cudaMemcpyDeviceToHost,
                            st) == cudaSuccess ? ISVD_OK : ISVD_ENODEV);
    if (rc == ISVD_OK && vt_host && w > 0) {
      // V (n x w) -> vt (w x n) on the host after download
      std::vector<double> vh((size_t)n * w);
      for (int b = 0; b < B && rc == ISVD_OK; ++b) {
        T(cudaMemcpy2DAsync(vh.data(), sizeof(double) * w, V + (size_t)b * n * ldw, sizeof(double) * ldw,
                            sizeof(double) * w, n, cudaMemcpyDeviceToHost, st) == cudaSuccess
              ? ISVD_OK : ISVD_ENODEV);
        if (cudaStreamSynchronize(st) != cudaSuccess) T(ISVD_ENODEV);
        for (int t = 0; t < w; ++t)
          for (int i = 0; i < n; ++i) vt_host[(size_t)b * w * n + (size_t)t * n + i] = vh[(size_t)i * w + t];
      }
    }
    if (cudaStreamSynchronize(st) != cudaSuccess) T(ISVD_ENODEV);
  }
  cudaError_t last = cudaStreamSynchronize(st);
  if (keep) {
    keep->drop();
    if (rc == ISVD_OK && w > 0) {
      keep->U = U; keep->V = V; keep->sw = sw; keep->sa = sa;
      keep->B = B; keep->m = m; keep->n = n; keep->w = w; keep->ldw = ldw; keep->nc = nc;
      keep->valid = true;
      U = V = sw = sa = nullptr;
    }
  }
  dfree(x); dfree(jac); dfree(U); dfree(V); dfree(sa); dfree(sw); dfree(fl);
  if (rc == ISVD_ENODEV && g_err.empty())
    set_error(std::string("oracle: device failure: ") + cudaGetErrorString(last));
  return rc;
}

int isvd_dense_svd(int batch, int m, int n, const double* a, int w_keep, double* s, double* u,
                   double* vt) {
  if (batch < 1 || m < 1 || n < 1 || !a) { set_error("bad argument"); return ISVD_EINVAL; }
  if (!all_finite(a, (size_t)batch * m * n)) { set_error("matrix contains non-finite entries"); return ISVD_EINVAL; }
  ISVD_TRY(check_device());
  double* ad = nullptr;
  ISVD_TRY(dalloc(&ad, (size_t)batch * m * n));
  cudaStream_t st = 0;
  int rc = cudaMemcpy(ad, a, sizeof(double) * batch * m * n, cudaMemcpyHostToDevice) == cudaSuccess
               ? ISVD_OK : ISVD_ENODEV;
  if (rc == ISVD_OK) rc = oracle_common(batch, m, n, ad, (int64_t)m * n, n, w_keep, s, u, vt, st);
  cudaDeviceSynchronize();
  dfree(ad);
  return rc;
}

int isvd_engine_oracle(isvd_engine* e, int w_keep, double* s, double* u) {
  if (e) e->join();
  if (!e || !e->initialized) { set_error("engine not initialised"); return ISVD_ESTATE; }
  if (e->sharded) { set_error("the device oracle needs the whole tracked matrix (not in shard mode)"); return ISVD_EINVAL; }
  const int nc = std::min(e->m, e->n);
  if (e->svdc_valid && std::max(0, std::min(w_keep, nc)) == e->svdc_w && e->r == e->svdc_w) {
    // the tracked matrix and the factors are exactly those of the last init /
    // refresh: the same dense SVD, already computed (same kernels on the
    // same input, so the bits match a recomputation)
    const int w = e->svdc_w;
    ISVD_TRY(e->canonicalize());
    if (s) ISVD_CUDA(cudaMemcpyAsync(s, e->svdc_sall, sizeof(double) * e->B * nc, cudaMemcpyDeviceToHost, e->st));
    if (u && w > 0)
      for (int b = 0; b < e->B; ++b)
        ISVD_CUDA(cudaMemcpy2DAsync(u + (size_t)b * e->m * w, sizeof(double) * w, e->U + b * e->ustride(),
                                    sizeof(double) * e->ld, sizeof(double) * w, e->m,
                                    cudaMemcpyDeviceToHost, e->st));
    ISVD_CUDA(cudaStreamSynchronize(e->st));
    return ISVD_OK;
  }
  std::vector<double> s_tmp;
  double* s_out = s;
  if (!s_out) {
    s_tmp.resize((size_t)e->B * nc);
    s_out = s_tmp.data();
  }
  ISVD_TRY(oracle_common(e->B, e->m, e->n, e->A, e->astride(), e->n_cap, w_keep, s_out, u, nullptr,
                         e->st, &e->okeep));
  if (e->okeep.valid) {
    bool nz = true;
    for (int b = 0; b < e->B; ++b) nz = nz && s_out[(size_t)b * nc + e->okeep.w - 1] > 0.0;
    e->okeep.nozero = nz;
  }
  return ISVD_OK;
}

// ------------------------------------------- functional metrics (host bases)

// ||Q^T Q - I||_F of host bases Q (B x rows x w), Gram on the FP64 tensor path
// (linalg.py:126-130).  Host pointers; synchronous.
int isvd_ortho_defect(int batch, int rows, int w, const double* q, double* out) {
  if (batch < 1 || rows < 1 || w < 1 || !q || !out) { set_error("bad argument"); return ISVD_EINVAL; }
  ISVD_TRY(check_device());
  double *qd = nullptr, *part = nullptr, *g = nullptr;
  int rc = dalloc(&qd, (size_t)batch * rows * w);
  if (rc == ISVD_OK) rc = dalloc(&part, (size_t)std::max<int64_t>(1, gram_part_elems(batch, rows, w, w)));
  if (rc == ISVD_OK) rc = dalloc(&g, (size_t)batch * w * w);
  if (rc == ISVD_OK && cudaMemcpy(qd, q, sizeof(double) * batch * rows * w, cudaMemcpyHostToDevice) != cudaSuccess)
    rc = ISVD_ENODEV;
  Mat Q{qd, (int64_t)rows * w, w};
  if (rc == ISVD_OK) rc = launch_gram(batch, rows, w, w, Q, Q, part, g, 0);
  std::vector<double> gh((size_t)batch * w * w);
  if (rc == ISVD_OK && cudaMemcpy(gh.data(), g, sizeof(double) * gh.size(), cudaMemcpyDeviceToHost) != cudaSuccess)
    rc = ISVD_ENODEV;
  if (rc == ISVD_OK)
    for (int b = 0; b < batch; ++b) {
      double acc = 0.0;
      for (int i = 0; i < w; ++i)
        for (int j = 0; j < w; ++j) {
          const double d = gh[((size_t)b * w + i) * w + j] - (i == j ? 1.0 : 0.0);
          acc += d * d;
        }
      out[b] = std::sqrt(acc);
    }
  dfree(qd); dfree(part); dfree(g);
  return rc;
}

// Largest principal angle between host bases q1, q2 (rows x w each):
// arccos of the smallest singular value of q1^T q2, clamped into [0, 1]
// (linalg.py:133-153); the Gram on DMMA, the w x w SVD by the core kernel.
// Each basis must be orthonormal to 1e-6 (else ISVD_EINVAL, as the reference).
int isvd_principal_angle(int rows, int w, const double* q1, const double* q2, double* out) {
  if (rows < 1 || w < 1 || !q1 || !q2 || !out) {
    set_error(w < 1 ? "subspaces must have at least one column" : "bad argument");
    return ISVD_EINVAL;
  }
  if (w > kCoreMaxS) { set_error("principal angle: too many columns for the core kernel"); return ISVD_EINVAL; }
  double d1 = 0.0, d2 = 0.0;
  ISVD_TRY(isvd_ortho_defect(1, rows, w, q1, &d1));
  if (d1 > 1e-6) { set_error("q1 is not orthonormal (defect > 1e-6)"); return ISVD_EINVAL; }
  ISVD_TRY(isvd_ortho_defect(1, rows, w, q2, &d2));
  if (d2 > 1e-6) { set_error("q2 is not orthonormal (defect > 1e-6)"); return ISVD_EINVAL; }
  double *a = nullptr, *b = nullptr, *part = nullptr, *c = nullptr, *uk = nullptr, *vk = nullptr,
         *sv = nullptr, *vscr = nullptr;
  int rc = dalloc(&a, (size_t)rows * w);
  if (rc == ISVD_OK) rc = dalloc(&b, (size_t)rows * w);
  if (rc == ISVD_OK) rc = dalloc(&part, (size_t)std::max<int64_t>(1, gram_part_elems(1, rows, w, w)));
  if (rc == ISVD_OK) rc = dalloc(&c, (size_t)w * w);
  if (rc == ISVD_OK) rc = dalloc(&uk, (size_t)w * w);
  if (rc == ISVD_OK) rc = dalloc(&vk, (size_t)w * w);
  if (rc == ISVD_OK) rc = dalloc(&sv, (size_t)w);
  if (rc == ISVD_OK && w > kSmemMaxS) rc = dalloc(&vscr, (size_t)w * (w | 1));
  if (rc == ISVD_OK && (cudaMemcpy(a, q1, sizeof(double) * rows * w, cudaMemcpyHostToDevice) != cudaSuccess ||
                        cudaMemcpy(b, q2, sizeof(double) * rows * w, cudaMemcpyHostToDevice) != cudaSuccess))
    rc = ISVD_ENODEV;
  if (rc == ISVD_OK) rc = launch_gram(1, rows, w, w, Mat{a, 0, w}, Mat{b, 0, w}, part, c, 0);
  if (rc == ISVD_OK)
    rc = launch_core_svd(1, w, c, (int64_t)w * w, w, uk, vk, (int64_t)w * w, w, sv, w, vscr, nullptr, 0);
  double smin = 0.0;
  if (rc == ISVD_OK && cudaMemcpy(&smin, sv + (w - 1), sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
    rc = ISVD_ENODEV;
  if (rc == ISVD_OK) *out = std::acos(std::min(1.0, std::max(0.0, smin)));
  dfree(a); dfree(b); dfree(part); dfree(c); dfree(uk); dfree(vk); dfree(sv); dfree(vscr);
  return rc;
}

// --------------------------------------------------------- functional kernels

int isvd_gram(int rows, int wa, int wb, const double* xa, int lda, const double* xb, int ldb,
              double* out, void* stream) {
  if (rows < 0 || wa < 0 || wb < 0 || !xa || !xb || !out || lda < wa || ldb < wb) {
    set_error("gram: bad argument");
    return ISVD_EINVAL;
  }
  ISVD_TRY(check_device());
  cudaStream_t st = (cudaStream_t)stream;
  double* part = nullptr;
  ISVD_CUDA(cudaMallocAsync((void**)&part, sizeof(double) * std::max<int64_t>(1, gram_part_elems(1, rows, wa, wb)), st));
  Mat Xa{const_cast<double*>(xa), 0, lda}, Xb{const_cast<double*>(xb), 0, ldb};
  const int sym = (xa == xb && wa == wb && lda == ldb) ? 1 : 0;
  int rc = launch_gram_tiles(1, rows, wa, wb, Xa, Xb, sym, part, out, st);
  cudaFreeAsync(part, st);
  return rc;
}

int isvd_gemm_tall(int rows, int n, int wc, const double* x, int ldx, const double* q, int ldq,
                   double* c, int ldc, void* stream) {
  if (rows < 0 || n < 0 || wc < 0 || !x || !q || !c || ldx < n || ldq < wc || ldc < wc) {
    set_error("gemm_tall: bad argument");
    return ISVD_EINVAL;
  }
  ISVD_TRY(check_device());
  Mat X{const_cast<double*>(x), 0, ldx}, Q{const_cast<double*>(q), 0, ldq}, C{c, 0, ldc};
  return launch_gemm_tall(1, rows, n, wc, X, Q, C, (cudaStream_t)stream);
}

int isvd_core_svd(int batch, int s, const double* core, double* u, double* sv, double* vt,
                  void* stream) {
  if (batch < 0 || s < 1 || !core || !u || !sv || !vt) { set_error("bad argument"); return ISVD_EINVAL; }
  if (s > kCoreMaxS) { set_error("core too large"); return ISVD_EINVAL; }
  ISVD_TRY(check_device());
  cudaStream_t st = (cudaStream_t)stream;
  double* vscr = nullptr;
  if (s > kSmemMaxS) ISVD_TRY(dalloc(&vscr, (size_t)batch * s * (s | 1)));
  // V is produced in vt's storage, then transposed in place on the device
  int rc = launch_core_svd(batch, s, core, (int64_t)s * s, s, u, vt, (int64_t)s * s, s, sv, s, vscr,
                           nullptr, st);
  if (rc == ISVD_OK) rc = launch_transpose_square(batch, s, vt, st);
  if (vscr) {
    cudaStreamSynchronize(st);
    dfree(vscr);
  }
  return rc;
}

// Functional row_append / rank_one: the reference's kernel contract
// (_kernels_py.py:22-58): raw factors in, raw factors out (no _install).
static int functional_common(bool is_row, int m, int r, int n, const double* u, const double* s,
                             const double* vt, const double* x, double tol, int64_t i, int64_t j,
                             double delta, int keep, double* u_out, double* s_out, double* vt_out,
                             double* rho) {
  if (m < 1 || n < 1 || r < 1 || keep < 1 || keep > (is_row ? r + 1 : r) || !u || !s || !vt ||
      !u_out || !s_out || !vt_out) {
    set_error("bad argument");
    return ISVD_EINVAL;
  }
  if (!is_row && !(0 <= i && i < m && 0 <= j && j < n)) { set_error("index out of bounds"); return ISVD_EINVAL; }
  ISVD_TRY(check_device());
  const int ld = round_up(std::max(r + 1, keep), 8);
  const int S = ld + 1;
  if (S > kCoreMaxS) { set_error("rank too large"); return ISVD_EINVAL; }
  const int mo = is_row ? m + 1 : m;
  std::vector<double> Uh((size_t)(mo) * ld, 0.0), Vh((size_t)n * ld, 0.0), sh(ld, 0.0);
  for (int a = 0; a < m; ++a)
    for (int c = 0; c < r; ++c) Uh[(size_t)a * ld + c] = u[(size_t)a * r + c];
  for (int c = 0; c < r; ++c)
    for (int a = 0; a < n; ++a) Vh[(size_t)a * ld + c] = vt[(size_t)c * n + a];
  for (int c = 0; c < r; ++c) sh[c] = s[c];
  double *U = nullptr, *V = nullptr, *sd = nullptr, *core = nullptr, *uk = nullptr, *vk = nullptr,
         *sv = nullptr, *z = nullptr, *inj = nullptr, *rd = nullptr, *xn = nullptr, *xd = nullptr,
         *N = nullptr, *vscr = nullptr, *dd = nullptr;
  int64_t *di = nullptr, *dj = nullptr;
  int rc = ISVD_OK;
  auto T = [&](int v) { if (rc == ISVD_OK) rc = v; };
  T(dalloc(&U, Uh.size())); T(dalloc(&V, Vh.size())); T(dalloc(&sd, ld));
  T(dalloc(&core, (size_t)S * S)); T(dalloc(&uk, (size_t)S * S)); T(dalloc(&vk, (size_t)S * S));
  T(dalloc(&sv, S)); T(dalloc(&z, n + 8)); T(dalloc(&inj, 1)); T(dalloc(&rd, 1)); T(dalloc(&xn, 1));
  T(dalloc(&xd, n + 8)); T(dalloc(&N, 1)); T(dalloc(&dd, 1)); T(dalloc(&di, 1)); T(dalloc(&dj, 1));
  if (S > kSmemMaxS) T(dalloc(&vscr, (size_t)S * (S | 1)));
  cudaStream_t st = 0;
  if (rc == ISVD_OK) {
    cudaMemcpy(U, Uh.data(), sizeof(double) * Uh.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(V, Vh.data(), sizeof(double) * Vh.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(sd, sh.data(), sizeof(double) * ld, cudaMemcpyHostToDevice);
    cudaMemset(N, 0, sizeof(double));
    Mat Um{U, 0, ld}, Vm{V, 0, ld};
    if (is_row) {
      cudaMemcpy(xd, x, sizeof(double) * n, cudaMemcpyHostToDevice);
      T(launch_project_append(1, n, r, Vm, xd, n, sd, ld, tol, core, 0, S, z, 0, inj, rd, xn,
                              nullptr, 0, 0, 0, N, st));
      T(launch_arrow_svd(1, r + 1, core, 0, S, uk, vk, 0, S, sv, 0, st));
      RotJob grow{Um, m, uk, 0, S, nullptr, 0, nullptr, 1};
      RotJob injj{Vm, n, vk, 0, S, z, 0, inj, 0};
      T(launch_rotate(1, r, keep, grow, &injj, st));
    } else {
      cudaMemcpy(di, &i, sizeof(int64_t), cudaMemcpyHostToDevice);
      cudaMemcpy(dj, &j, sizeof(int64_t), cudaMemcpyHostToDevice);
      cudaMemcpy(dd, &delta, sizeof(double), cudaMemcpyHostToDevice);
      T(launch_rank1_build(1, r, Um, Vm, sd, ld, di, dj, dd, core, 0, S, nullptr, 0, 0, N, LazyBasis{0, 0, 0, Mat{nullptr, 0, 0}}, st));
      T(launch_core_svd(1, r, core, 0, S, uk, vk, 0, S, sv, 0, vscr, nullptr, st));
      RotJob ju{Um, m, uk, 0, S, nullptr, 0, nullptr, 0};
      RotJob jv{Vm, n, vk, 0, S, nullptr, 0, nullptr, 0};
      T(launch_rotate(1, r, keep, ju, &jv, st));
    }
    if (cudaDeviceSynchronize() != cudaSuccess) {
      set_error(std::string("functional kernel: ") + cudaGetErrorString(cudaGetLastError()));
      T(ISVD_ENODEV);
    }
  }
  if (rc == ISVD_OK) {
    cudaMemcpy(Uh.data(), U, sizeof(double) * (size_t)mo * ld, cudaMemcpyDeviceToHost);
    cudaMemcpy(Vh.data(), V, sizeof(double) * Vh.size(), cudaMemcpyDeviceToHost);
    std::vector<double> svh(S);
    cudaMemcpy(svh.data(), sv, sizeof(double) * S, cudaMemcpyDeviceToHost);
    for (int a = 0; a < mo; ++a)
      for (int c = 0; c < keep; ++c) u_out[(size_t)a * keep + c] = Uh[(size_t)a * ld + c];
    for (int c = 0; c < keep; ++c)
      for (int a = 0; a < n; ++a) vt_out[(size_t)c * n + a] = Vh[(size_t)a * ld + c];
    for (int c = 0; c < keep; ++c) s_out[c] = svh[c];
    if (is_row && rho) cudaMemcpy(rho, rd, sizeof(double), cudaMemcpyDeviceToHost);
  }
  dfree(U); dfree(V); dfree(sd); dfree(core); dfree(uk); dfree(vk); dfree(sv); dfree(z); dfree(inj);
  dfree(rd); dfree(xn); dfree(xd); dfree(N); dfree(dd); dfree(di); dfree(dj); dfree(vscr);
  return rc;
}

int isvd_row_append(int m, int r, int n, const double* u, const double* s, const double* vt,
                    const double* x, double tol, int keep, double* u_out, double* s_out,
                    double* vt_out, double* rho) {
  if (!x) { set_error("x is null"); return ISVD_EINVAL; }
  return functional_common(true, m, r, n, u, s, vt, x, tol, 0, 0, 0.0, keep, u_out, s_out, vt_out, rho);
}

int isvd_rank_one(int m, int r, int n, const double* u, const double* s, const double* vt, int64_t i,
                  int64_t j, double delta, int keep, double* u_out, double* s_out, double* vt_out) {
  return functional_common(false, m, r, n, u, s, vt, nullptr, 0.0, i, j, delta, keep, u_out, s_out,
                           vt_out, nullptr);
}

}  // extern "C"
