#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "tick.cuh"
#include "shard.cuh"

namespace isvd {

// Workspace sizes (doubles per stream) for a dense SVD of an m x n matrix.
struct DenseSvdPlan {
  int m, n, nc, len, ncp, ldx, nb;
  int64_t x_elems() const { return (int64_t)ncp * ldx; }
  int64_t j_elems() const { return (int64_t)ncp * ncp; }
};
// w = number of leading triplets wanted (selects the Gram path, see below).
DenseSvdPlan dense_svd_plan(int m, int n, int w);

// Thin SVD of `batch` row-major m x n matrices A[b] = a + b*a_stride (pitch
// lda), in the reference's canonical form (linalg.py:84-92): singular
// values nonincreasing, snapped below 1e-12 s0, zero-sigma columns of the
// orthonormal side completed, signs canonical.  Writes the leading w
// triplets: U (m x w) into u, V (n x w) into v (both row-major), and all
// nc = min(m, n) singular values into s_all (stride s_stride) when non-null.
// Workspace x: batch * plan.x_elems(), jac: batch * plan.j_elems(),
// flags: batch ints.
int dense_svd_run(int batch, int m, int n, const double* a, int64_t a_stride, int lda, int w,
                  Mat u, Mat v, double* s_w, int64_t s_w_stride, double* s_all,
                  int64_t s_all_stride, double* x, double* jac, int* flags, int* flags_host,
                  cudaStream_t st, int* sweeps_out);

// Very tall matrices (m >= 4n, m*n >= kGramMinElems) with w <= kGramMaxW
// leading triplets wanted take the Gram path of gram_svd.cu inside
// dense_svd_run; the plan then needs no x/jac workspace.
constexpr int64_t kGramMinElems = int64_t(1) << 24;
constexpr int kGramMaxW = 160;  // Rayleigh-Ritz core = one core SVD (kCoreMaxS)
bool use_gram_path(int m, int n, int w);
// ar: row-sharded A (each rank holds m of the rows): the Grams are summed
// across ranks, everything else is replicated or row-local.
int gram_svd_run(int m, int n, const double* a, int lda, int w, Mat u, Mat v, double* s_w,
                 double* s_all, cudaStream_t st, const Allreducer* ar = nullptr);

}  // namespace isvd
