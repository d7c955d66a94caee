// Dependent-chain latencies on the B200 (cycles): DFMA, DMUL, DADD, SHFL.64,
// MUFU rcp64h, rsqrt64h, LDS.64, plus DFMA throughput per warp.
#include <cstdio>
__global__ void k(double* out, long long* cyc, int n, double x0) {
  double x = x0 + threadIdx.x * 1e-9, y = 1.0000001;
  long long t0, t1;
  __shared__ double sm[64];
  sm[threadIdx.x] = x;
  __syncwarp();
#define TIME(idx, body) t0 = clock64(); for (int i = 0; i < n; ++i) { body; } t1 = clock64(); if (threadIdx.x == 0) cyc[idx] = (t1 - t0);
  TIME(0, x = fma(x, y, 1e-30); x = fma(x, y, 1e-30); x = fma(x, y, 1e-30); x = fma(x, y, 1e-30))
  TIME(1, x = x * y; x = x * y; x = x * y; x = x * y)
  TIME(2, x = x + 1e-20; x = x + 1e-20; x = x + 1e-20; x = x + 1e-20)
  TIME(3, x = __shfl_xor_sync(0xffffffffu, x, 1); x = __shfl_xor_sync(0xffffffffu, x, 2); x = __shfl_xor_sync(0xffffffffu, x, 4); x = __shfl_xor_sync(0xffffffffu, x, 8))
  TIME(4, double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r;)
  TIME(5, double r; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r+1.0; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r+1.0;)
  int idx = threadIdx.x;
  TIME(6, idx = (int)sm[idx & 31] & 31; idx = (int)sm[idx] & 31; idx = (int)sm[idx] & 31; idx = (int)sm[idx] & 31)
  double a0 = x, a1 = x + 1, a2 = x + 2, a3 = x + 3, a4 = x + 4, a5 = x + 5, a6 = x + 6, a7 = x + 7;
  TIME(7, a0 = fma(a0, y, 1e-30); a1 = fma(a1, y, 1e-30); a2 = fma(a2, y, 1e-30); a3 = fma(a3, y, 1e-30); a4 = fma(a4, y, 1e-30); a5 = fma(a5, y, 1e-30); a6 = fma(a6, y, 1e-30); a7 = fma(a7, y, 1e-30))
  out[threadIdx.x] = x + idx + a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 256 * 8); cudaMalloc(&cyc, 64 * 8);
  const int n = 4096;
  k<<<1, 32>>>(out, cyc, n, 1.0); cudaDeviceSynchronize();
  k<<<1, 32>>>(out, cyc, n, 1.0); cudaDeviceSynchronize();
  long long h[8]; cudaMemcpy(h, cyc, 64, cudaMemcpyDeviceToHost);
  const char* nm[8] = {"dfma", "dmul", "dadd", "shfl64", "rcp64", "rsqrt64+dadd", "lds+cvt", "dfma x8 indep (per instr)"};
  int per[8] = {4, 4, 4, 4, 4, 2, 4, 8};
  for (int i = 0; i < 8; ++i) printf("%-28s %.1f cyc\n", nm[i], (double)h[i] / n / per[i]);
  return 0;
}
