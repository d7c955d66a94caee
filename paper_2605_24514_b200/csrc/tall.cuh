#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "tick.cuh"

namespace isvd {

// Row splits of a Gram (deterministic in the shape only).
int gram_splits(int batch, int rows, int wa, int wb);
// Partial-buffer size (doubles) launch_gram_tiles needs.
int64_t gram_part_elems(int batch, int rows, int wa, int wb);
// out[b] (wa x wb, dense row-major) = Xa[b][0:rows, 0:wa]^T Xb[b][0:rows, 0:wb]
// on DMMA; sym = 1 computes only the upper tiles of Xa^T Xa and mirrors.
int launch_gram_tiles(int batch, int rows, int wa, int wb, Mat Xa, Mat Xb, int sym, double* part,
                      double* out, cudaStream_t st);
// C[b] (rows x wc) = X[b] (rows x n) . Q[b] (n x wc) on DMMA.
int launch_gemm_tall(int batch, int rows, int n, int wc, Mat X, Mat Q, Mat C, cudaStream_t st);

}  // namespace isvd
