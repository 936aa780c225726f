// Deterministic block reduction (fixed order: warp shuffle tree, then warp
// sums added in warp order by thread 0).  Any blockDim: a partial last warp
// only adds lanes that exist (full warps reduce exactly as before).
#pragma once

namespace fm {

__device__ __forceinline__ double block_sum_any(double v) {
  __shared__ double wsum_[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int wsize = min(32, int(blockDim.x) - wid * 32);
  const unsigned mask = wsize == 32 ? 0xffffffffu : ((1u << wsize) - 1u);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double t = __shfl_down_sync(mask, v, o);
    if (lane + o < wsize) v += t;
  }
  __syncthreads();
  if (lane == 0) wsum_[wid] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < int((blockDim.x + 31) >> 5); ++w) s += wsum_[w];
  return s;  // valid in thread 0
}

}  // namespace fm
