#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "tick.cuh"
#include "shard.cuh"

namespace isvd {
// ||U^T U - I||_F and ||V^T V - I||_F per stream, copied to host (synchronous)
// ar (row-sharded U): the U Gram is summed across ranks before use
int reortho_defects(int batch, int w, Mat U, int m, Mat V, int n, double* host_du, double* host_dv,
                    cudaStream_t st, const Allreducer* ar = nullptr);
// engine.py:214-217 re-factorisation of (U, s, V) for every stream
int reortho_apply(int batch, int w, Mat U, int m, Mat V, int n, double* s, int lds, double* core,
                  double* uk, double* vk, int64_t cstride, int S, double* sv, double* vscr,
                  cudaStream_t st, const Allreducer* ar = nullptr);
}  // namespace isvd
