// Lane-pair radix-2 steps that join two H-point half-line transforms into an
// N = 2H-point one (decimation in time forward, decimation in frequency
// inverse), shared by the long-line x passes (projection_fast.cu,
// projection_xw.cu).  See the comment above k_x_direct for the slot order.
#pragma once

#include "fft_reg.cuh"

namespace fm {

__device__ __forceinline__ double2 shfl_xor2(double2 v, int mask) {
  return make_double2(__shfl_xor_sync(0xffffffffu, v.x, mask), __shfl_xor_sync(0xffffffffu, v.y, mask));
}
template <int TH, int H>
__device__ __forceinline__ int kslot(int t, int h, int s) {  // frequency held in slot s (E = 16)
  return t + TH * ((s & 7) + 8 * h) + H * ((s >> 3) ^ h);
}
// Forward radix-2 DIT combine of the lane pair (E = 16): lane h = 0 holds
// E[t + TH m], h = 1 holds O[t + TH m]; h = 0 keeps slots m < 8 (gives
// E[m + 8]), h = 1 keeps m >= 8 (gives O[m]); the kept slot ends as X[k],
// the other as X[k + H] (kslot).  tw: the W_N table, N = 2H, read at stride TS
// (TS = 2: the table of a line twice as long).
template <int TH, int TW, int TS = 1>
__device__ __forceinline__ void pair_dit(double2 (&v)[16], int t, int h, const double2* __restrict__ tw) {
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const double2 got = shfl_xor2(h == 0 ? v[m + 8] : v[m], TW);
    const double2 e = h == 0 ? v[m] : got, o = h == 0 ? got : v[m + 8];
    const int k = t + TH * (m + 8 * h);
    const double2 wo = reg::tw_mul(o, __ldg(&tw[k * TS]), -1);
    const double2 lo = make_double2(e.x + wo.x, e.y + wo.y), hi = make_double2(e.x - wo.x, e.y - wo.y);
    v[m] = h == 0 ? lo : hi;
    v[m + 8] = h == 0 ? hi : lo;
  }
}
// Inverse radix-2 DIF split (the mirror image): from the kslot order, the
// sums X[k] + X[k + H] go to lane h = 0 (even output rows), the differences
// (X[k] - X[k + H]) W_N^-k to h = 1, each as slot m of k = t + TH m.
template <int TH, int TW, int TS = 1>
__device__ __forceinline__ void pair_dif(double2 (&v)[16], int t, int h, const double2* __restrict__ tw) {
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const double2 xa = h == 0 ? v[m] : v[m + 8], xb = h == 0 ? v[m + 8] : v[m];  // X[k], X[k + H]
    const int k = t + TH * (m + 8 * h);
    const double2 sum = make_double2(xa.x + xb.x, xa.y + xb.y);
    const double2 dif = reg::tw_mul(make_double2(xa.x - xb.x, xa.y - xb.y), __ldg(&tw[k * TS]), +1);
    const double2 got = shfl_xor2(h == 0 ? dif : sum, TW);
    v[m] = h == 0 ? sum : got;
    v[m + 8] = h == 0 ? got : dif;
  }
}

}  // namespace fm
