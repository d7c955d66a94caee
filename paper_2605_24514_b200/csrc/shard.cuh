#pragma once
// Cross-rank sum used by the row-sharded mode (isvd_engine_set_shard).
#include <cuda_runtime.h>
#include <stdint.h>
#include "common.cuh"
#include "../../include/isvd.h"

namespace isvd {

struct Allreducer {
  isvd_allreduce_fn fn = nullptr;
  void* ctx = nullptr;
  cudaStream_t st = nullptr;
  bool active() const { return fn != nullptr; }
  // In-place sum of n doubles of a device buffer across ranks (stream-ordered).
  int operator()(double* p, int64_t n) const {
    if (!fn || n <= 0) return ISVD_OK;
    if (fn(ctx, p, n, (void*)st) != 0) {
      set_error("allreduce callback failed");
      return ISVD_ENODEV;
    }
    return ISVD_OK;
  }
};

}  // namespace isvd
