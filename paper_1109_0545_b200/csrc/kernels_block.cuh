// Warp-per-monomial-block kernels (placeholder: enabled in a later step).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "arith.cuh"

namespace phc {

struct BlockTables {
  uint32_t* fac = nullptr;
  double* coeff = nullptr;
  int32_t* blk = nullptr;
};

struct HostBlockPlan {
  bool usable = false;
  int64_t cm_per_point = 0;
  int64_t ca_per_point = 0;
  int launches = 0;
};

template <class S>
void plan_blocks(const S&, HostBlockPlan* plan) {
  plan->usable = false;
}

inline int upload_block_tables(const HostBlockPlan&, BlockTables*) { return 0; }

template <int L>
int run_block(const HostBlockPlan&, const BlockTables&, int, int, int64_t, const double*, double*, double*,
              cudaStream_t) {
  return -1;
}

}  // namespace phc
