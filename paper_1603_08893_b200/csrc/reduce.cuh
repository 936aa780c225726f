// Deterministic block reduction (fixed order: warp shuffle tree, then warp
// sums added in warp order by thread 0).  blockDim must be a multiple of 32.
#pragma once

namespace fm {

__device__ __forceinline__ double block_sum_any(double v) {
  __shared__ double wsum_[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) wsum_[wid] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < int(blockDim.x >> 5); ++w) s += wsum_[w];
  return s;  // valid in thread 0
}

}  // namespace fm
