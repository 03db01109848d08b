// ccd.cuh -- complementary cumulative distribution of one orbit column (the paper's VOC
// distributions: "for x, we plot the fraction of vertices whose orbit count is
// at least x").  Column gather -> radix sort -> run-length encode -> suffix sums, all on the
// device; the host gets the distinct values (ascending) and, for each, the number of
// vertices whose count is >= it.
#pragma once
#include <cub/cub.cuh>
#include "common.cuh"

__global__ void k_ccd_gather(const u64* __restrict__ dim, int64_t n, int orbit, u64* __restrict__ col) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    col[v] = dim[v * EVOKE_NUM_ORBITS_DEV + orbit];
}

// counts[i] <- sum_{j >= i} counts[j] (one block per tile would be overkill: n distinct
// values at most; a reverse inclusive scan via reversed iterators)
__global__ void k_ccd_reverse(const u64* __restrict__ in, int64_t k, u64* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[k - 1 - i];
}
