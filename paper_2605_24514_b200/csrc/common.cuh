// Shared device helpers for libisvd (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <utility>

namespace isvd {

// Relative snap cutoff (linalg.py:18, _kernels.pyx:15).
constexpr double kZeroSvRtol = 1e-12;
// Jacobi orthogonality target and sweep cap (_kernels.pyx:17-19).
constexpr double kOrthoEps = 1e-14;
constexpr int kMaxSweeps = 64;

void set_error(const std::string& msg);
// Tick gate (engine.cu): while set, the launchers of the append path pass it
// to their kernels, which exit at once when *gate != 0 (a rejected payload
// leaves the engine state untouched though its kernels were already queued).
extern thread_local const int* g_gate;
void count_launch(int n = 1);

#define ISVD_CUDA(call)                                                        \
  do {                                                                         \
    cudaError_t _e = (call);                                                   \
    if (_e != cudaSuccess) {                                                   \
      ::isvd::set_error(std::string(#call) + ": " + cudaGetErrorString(_e));   \
      return ISVD_ENODEV;                                                      \
    }                                                                          \
  } while (0)

#define ISVD_LAUNCHED()                                                        \
  do {                                                                         \
    ::isvd::count_launch();                                                    \
    cudaError_t _e = cudaGetLastError();                                       \
    if (_e != cudaSuccess) {                                                   \
      ::isvd::set_error(std::string("kernel launch: ") + cudaGetErrorString(_e)); \
      return ISVD_ENODEV;                                                      \
    }                                                                          \
  } while (0)

#define ISVD_TRY(x)                 \
  do {                              \
    int _rc = (x);                  \
    if (_rc != 0) return _rc;       \
  } while (0)

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Eight warp sums at once (transposing butterfly: 9 shuffle pairs, depth 5,
// instead of 40): returns sum over the warp of v[t] with
// t = 4 * bit4(lane) + 2 * bit3(lane) + bit2(lane) (see warp_sum8_slot).
__device__ __forceinline__ double warp_sum8(const double (&v)[8]) {
  const int lane = threadIdx.x & 31;
  double w4[4], w2[2];
  {
    const bool hi = lane & 16;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double keep = hi ? v[k + 4] : v[k], send = hi ? v[k] : v[k + 4];
      w4[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
  }
  {
    const bool hi = lane & 8;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const double keep = hi ? w4[k + 2] : w4[k], send = hi ? w4[k] : w4[k + 2];
      w2[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
  }
  const bool hi = lane & 4;
  const double keep = hi ? w2[1] : w2[0], send = hi ? w2[0] : w2[1];
  double r = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  r += __shfl_xor_sync(0xffffffffu, r, 2);
  r += __shfl_xor_sync(0xffffffffu, r, 1);
  return r;
}
__device__ __forceinline__ int warp_sum8_slot(int lane) {
  return ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
}

// Block-wide sum; `red` must hold >= 32 doubles of shared memory.  Result is
// returned to every thread.
__device__ __forceinline__ double block_sum(double v, double* red) {
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = (threadIdx.x < nw) ? red[threadIdx.x] : 0.0;
  if (warp == 0) t = warp_sum(t);
  if (threadIdx.x == 0) red[0] = t;
  __syncthreads();
  double r = red[0];
  __syncthreads();
  return r;
}

// CTA-per-core kernels with a device-launched fallback: every CTA counts
// itself once it has decided whether it keeps its core (`handed`: it appended
// the core to the fallback list, which is ordered before the count); the CTA
// whose arrival completes the count tail-launches the fallback kernel when it
// finishes.  Counting at the decision instead of at the end keeps the fence
// and the atomic's round trip (20-35 % of a CTA's lifetime in ncu's stall
// samples) off the end of every CTA: the count is in flight during the
// epilogue.  Returns the previous count (thread 0 only).
__device__ __forceinline__ int fb_arrive(int* done, bool handed) {
  if (handed) __threadfence();
  return atomicAdd(done, 1);
}

// D(8x8) += A(8x4, row) * B(4x8, col), FP64 tensor path (DMMA.8x8x4).
// Fragment layout (verified on B200, profiles/r01_fp64_peaks.txt):
//   a = A[lane>>2][lane&3], b = B[lane&3][lane>>2],
//   d0,d1 = D[lane>>2][2*(lane&3) + {0,1}].
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// Launch with optional programmatic stream serialization (PDL) and an
// optional thread-block cluster; used for the latency-bound few-stream ticks.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_ex(bool pdl, int cluster, void (*kernel)(KArgs...), dim3 grid, dim3 block,
                             size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (cluster > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = cluster;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
inline int round_up(int a, int b) { return (a + b - 1) / b * b; }

// ---- Programmatic dependent launch (sm_90+): a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start while its
// stream predecessor runs; griddep_wait() blocks until the predecessor has
// completed and its writes are visible (a no-op for ordinary launches);
// griddep_launch_dependents() lets the next such kernel start launching.
__device__ __forceinline__ void griddep_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" :::);
}

}  // namespace isvd

// ---- TMA bulk copies (cp.async.bulk) with mbarrier completion, sm_90+/sm_100a
namespace isvd {
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// global -> shared bulk copy; bytes multiple of 16, both addresses 16-byte aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// bulk L2 prefetch of [src, src + bytes) (fire and forget); src 16-byte
// aligned, bytes a multiple of 16
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
}  // namespace isvd
