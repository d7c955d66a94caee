#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "tick.cuh"
#include "tall.cuh"

namespace isvd {

int frob_nblk(int m, int n);
// out[b] = ||A[b] - U[b] diag(s[b]) V[b]^T||_F^2 ; partial: batch * frob_nblk(m, n)
int launch_frob_error_sq(int batch, int m, int n, int w, const double* A, int64_t a_stride, int lda,
                         Mat U, const double* s, int lds, Mat V, double* partial, double* out,
                         cudaStream_t st);
// out[b] (wa x wb) = Xa[b][0:rows,0:wa]^T Xb[b][0:rows,0:wb] (DMMA, tall.cu);
// partial: gram_part_elems(batch, rows, wa, wb) doubles
int launch_gram(int batch, int rows, int wa, int wb, Mat Xa, Mat Xb, double* partial, double* out,
                cudaStream_t st);
int launch_defect(int batch, int w, const double* G, double* out, cudaStream_t st);
// a13 per-tick risk (see metrics.cu): out[b][p] = {vol_lr, vol_lr+diag, VaR99, w'cov w}
int launch_risk(int batch, int n, int r, Mat V, const double* s, int lds, const double* A,
                int64_t a_stride, int lda, int m, double inv_t1, const double* w, int P,
                double* cov, double* diag, double* out, cudaStream_t st);

}  // namespace isvd
