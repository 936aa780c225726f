// Shared-memory Stockham FFT engine for fp64 complex lines (any length).
//
// Generic path of the projection passes: a CTA holds `nl` lines of length
// N in shared memory (element e of line l at a[l*ls + e*es]) and runs the
// mixed-radix Stockham autosort recursion in place between two buffers.
// Each work item produces ONE output of a radix-R stage:
//   out[o] = sum_r in[j + r N/R] * W_N^{ r (j mod Ns + k Ns) N/(Ns R) }
// with o = (j/Ns) Ns R + j mod Ns + k Ns, which covers any radix (including
// a prime such as 31) with one table lookup per term.  Specialised
// register-resident kernels for power-of-two N are layered on top of this
// (fft_reg.cuh); this engine is the correctness baseline for every size.
#pragma once

#include "fm_internal.cuh"

namespace fm {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // a * conj(b)
  return make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}
__device__ __forceinline__ double2 csub(double2 a, double2 b) {
  return make_double2(a.x - b.x, a.y - b.y);
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }

// Runs all stages of plan P over nl lines; returns the buffer holding the
// result (a or b).  sign = -1 forward, +1 backward (unnormalised).
// lfast: thread index maps to the line first (use when lines are
// interleaved element-wise, ls == 1) so smem accesses are consecutive.
// tws: shared-memory space for the N-entry twiddle table (staged here once;
// latency-bound small grids otherwise wait on one L2 round trip per term).
__device__ __forceinline__ double2* fft_smem(double2* a, double2* b, int nl, int ls, int es,
                                             const AxisPlan& P, int sign, bool lfast, double2* tws) {
  const int N = P.N;
  for (int i = threadIdx.x; i < N; i += blockDim.x) tws[i] = __ldg(&P.tw[i]);
  __syncthreads();
  int Ns = 1;
  for (int s = 0; s < P.nst; ++s) {
    const int R = P.radix[s];
    const int NR = N / R;
    const int tstep = N / (Ns * R);
    const int total = nl * N;
    for (int w = threadIdx.x; w < total; w += blockDim.x) {
      int l, o;
      if (lfast) {
        l = w % nl;
        o = w / nl;
      } else {
        l = w / N;
        o = w - l * N;
      }
      const int k = (o / Ns) % R;
      const int jm = o % Ns;
      const int j = (o / (Ns * R)) * Ns + jm;
      const int e0 = (jm + k * Ns) * tstep;  // < N
      const double2* src = a + l * ls + j * es;
      double2 acc = src[0];
      int ex = 0;
      // unrolled: the loads of 4 terms are issued together (small grids are
      // load-latency bound here); the accumulation order is unchanged
#pragma unroll 4
      for (int r = 1; r < R; ++r) {
        ex += e0;
        if (ex >= N) ex -= N;
        const double2 v = src[r * NR * es];
        const double2 t = tws[ex];
        acc = cadd(acc, sign < 0 ? cmul(v, t) : cmulc(v, t));
      }
      b[l * ls + o * es] = acc;
    }
    __syncthreads();
    double2* t = a;
    a = b;
    b = t;
    Ns *= R;
  }
  return a;
}

}  // namespace fm
