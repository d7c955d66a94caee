// FP64 throughput probes for the B200 design decisions in DESIGN.md:
//   * DFMA (FP64 FMA pipe) peak
//   * DMMA (mma.sync m8n8k4 f64, FP64 tensor path) peak
//   * both at once (are they separate hardware?)
//   * m8n8k4 fragment layout check against a CPU product
//   * double-precision streaming copy bandwidth (LDG.128/STG.128)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peaks tools/fp64_peaks.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
               : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void dmma_kernel(double* out, int iters, double a, double b) {
  double c0[CHAINS], c1[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) { c0[c] = threadIdx.x * 1e-3 + c; c1[c] = c0[c] + 0.5; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) dmma(c0[c], c1[c], a, b, c0[c], c1[c]);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += c0[c] + c1[c];
  if (s == 12345.678) out[0] = s;
}

// half of the warps run DFMA, the other half DMMA
template <int CHAINS>
__global__ void mixed_kernel(double* out, int iters_fma, int iters_mma, double a, double b) {
  int warp = threadIdx.x >> 5;
  double s = 0;
  if (warp & 1) {
    double c0[CHAINS], c1[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) { c0[c] = threadIdx.x * 1e-3 + c; c1[c] = c0[c] + 0.5; }
    for (int i = 0; i < iters_mma; ++i) {
#pragma unroll
      for (int c = 0; c < CHAINS; ++c) dmma(c0[c], c1[c], a, b, c0[c], c1[c]);
    }
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += c0[c] + c1[c];
  } else {
    double acc[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-3 + c;
    for (int i = 0; i < iters_fma; ++i) {
#pragma unroll
      for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
    }
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += acc[c];
  }
  if (s == 12345.678) out[0] = s;
}

__global__ void layout_kernel(const double* A, const double* B, double* D) {
  int lane = threadIdx.x;
  double a = A[(lane >> 2) * 4 + (lane & 3)];   // A 8x4 row-major: row = lane>>2, col = lane&3
  double b = B[(lane & 3) * 8 + (lane >> 2)];   // B 4x8 row-major: row = lane&3, col = lane>>2
  double d0, d1;
  dmma(d0, d1, a, b, 0.0, 0.0);
  D[(lane >> 2) * 8 + (lane & 3) * 2 + 0] = d0;
  D[(lane >> 2) * 8 + (lane & 3) * 2 + 1] = d1;
}

__global__ void copy_kernel(const double2* __restrict__ src, double2* __restrict__ dst, size_t n2) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n2; i += stride) dst[i] = src[i];
}

int main() {
  int dev = 0;
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  int sms = prop.multiProcessorCount;
  double* out;
  CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float ms;

  // ---- layout check
  {
    double hA[32], hB[32], hD[64], ref[64];
    for (int i = 0; i < 32; ++i) { hA[i] = 1.0 + i; hB[i] = 0.5 * i - 3.0; }
    for (int r = 0; r < 8; ++r)
      for (int c = 0; c < 8; ++c) {
        double s = 0;
        for (int k = 0; k < 4; ++k) s += hA[r * 4 + k] * hB[k * 8 + c];
        ref[r * 8 + c] = s;
      }
    double *dA, *dB, *dD;
    CK(cudaMalloc(&dA, 256)); CK(cudaMalloc(&dB, 256)); CK(cudaMalloc(&dD, 512));
    CK(cudaMemcpy(dA, hA, 256, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice));
    layout_kernel<<<1, 32>>>(dA, dB, dD);
    CK(cudaMemcpy(hD, dD, 512, cudaMemcpyDeviceToHost));
    double err = 0;
    for (int i = 0; i < 64; ++i) err = fmax(err, fabs(hD[i] - ref[i]));
    printf("{\"probe\": \"dmma_layout\", \"max_abs_err\": %g}\n", err);
  }

  const int iters = 4096;
  // ---- DFMA
  for (int blocks_per_sm : {4, 8}) {
    int threads = 256;
    int grid = sms * blocks_per_sm;
    dfma_kernel<8><<<grid, threads>>>(out, 16, 1.0000001, 1e-9);
    CK(cudaEventRecord(e0));
    dfma_kernel<8><<<grid, threads>>>(out, iters, 1.0000001, 1e-9);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    double flops = 2.0 * 8 * iters * (double)grid * threads;
    printf("{\"probe\": \"dfma\", \"blocks_per_sm\": %d, \"tflops\": %.2f, \"ms\": %.3f}\n",
           blocks_per_sm, flops / ms / 1e9, ms);
  }
  // ---- DMMA
  for (int blocks_per_sm : {4, 8}) {
    int threads = 256;
    int grid = sms * blocks_per_sm;
    dmma_kernel<4><<<grid, threads>>>(out, 16, 1.0000001, 1e-9);
    CK(cudaEventRecord(e0));
    dmma_kernel<4><<<grid, threads>>>(out, iters, 1.0000001, 1e-9);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    double flops = 2.0 * 256 * 4 * iters * (double)grid * (threads / 32);
    printf("{\"probe\": \"dmma\", \"blocks_per_sm\": %d, \"tflops\": %.2f, \"ms\": %.3f}\n",
           blocks_per_sm, flops / ms / 1e9, ms);
  }
  // ---- mixed: time with equal per-warp flop counts
  {
    int threads = 256, grid = sms * 8;
    int it_fma = iters * 8;  // DFMA warp: 8 chains * 32 lanes * it_fma FMAs
    int it_mma = iters;      // DMMA warp: 4 chains * 256 FMAs * it_mma
    mixed_kernel<4><<<grid, threads>>>(out, 16, 16, 1.0000001, 1e-9);
    CK(cudaEventRecord(e0));
    mixed_kernel<4><<<grid, threads>>>(out, it_fma, it_mma, 1.0000001, 1e-9);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    double warps = (double)grid * threads / 32;
    double flops = warps / 2 * (2.0 * 4 * 32 * it_fma) + warps / 2 * (2.0 * 256 * 4 * it_mma);
    printf("{\"probe\": \"mixed_dfma_dmma\", \"tflops_total\": %.2f, \"ms\": %.3f}\n", flops / ms / 1e9, ms);
  }
  // ---- copy bandwidth (fp64, 2 GiB each way)
  {
    size_t bytes = (size_t)2 << 30;
    double2 *a, *b;
    CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes));
    CK(cudaMemset(a, 0, bytes));
    size_t n2 = bytes / 16;
    int grid = sms * 8;
    copy_kernel<<<grid, 512>>>(a, b, n2);
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(e0));
      copy_kernel<<<grid, 512>>>(a, b, n2);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
      best = fminf(best, ms);
    }
    printf("{\"probe\": \"copy_f64x2\", \"gbs\": %.1f}\n", 2.0 * bytes / best / 1e6);
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
