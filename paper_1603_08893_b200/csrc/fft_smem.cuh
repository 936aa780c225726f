// Shared-memory Stockham FFT engine for fp64 complex lines (any length).
//
// Generic path of the projection passes: a CTA holds `nl` lines of length
// N in shared memory (element e of line l at a[l*ls + e*es]) and runs the
// mixed-radix Stockham autosort recursion in place between two buffers.
// A radix-R stage computes
//   out[o] = sum_r in[j + r N/R] * W_N^{ r (j mod Ns + k Ns) N/(Ns R) }
// with o = (j/Ns) Ns R + j mod Ns + k Ns, which covers any radix (including
// a prime such as 31) with one table lookup per term; each work item forms up
// to four outputs k of one input set j.  Specialised
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
// tw_pre: the table already staged in shared memory (persistent kernels stage
// each axis's table once), else it is staged into tws here.
__device__ __forceinline__ double2* fft_smem(double2* a, double2* b, int nl, int ls, int es,
                                             const AxisPlan& P, int sign, bool lfast, double2* tws,
                                             const double2* tw_pre = nullptr) {
  const int N = P.N;
  if (tw_pre) {
    tws = const_cast<double2*>(tw_pre);
  } else {
    for (int i = threadIdx.x; i < N; i += blockDim.x) tws[i] = __ldg(&P.tw[i]);
    __syncthreads();
  }
  int Ns = 1;
  for (int s = 0; s < P.nst; ++s) {
    const int R = P.radix[s];
    const int NR = N / R;
    const int tstep = N / (Ns * R);
    // outputs (j, k) with the same j read the same R inputs: each work item
    // computes up to KB of them (k = kg + KG q) from one pass over the inputs,
    // cutting the shared-memory input traffic by KB (same accumulation order
    // per output as one output per item, so results are bit-identical)
    constexpr int KB = 4;
    const int KG = (R + KB - 1) / KB;
    const int total = nl * NR * KG;
    for (int w = threadIdx.x; w < total; w += blockDim.x) {
      int l, rest;
      if (lfast) {
        l = w % nl;
        rest = w / nl;
      } else {
        l = w / (NR * KG);
        rest = w - l * (NR * KG);
      }
      const int kg = rest % KG;
      const int j = rest / KG;
      const int jm = j % Ns;
      const double2* src = a + l * ls + j * es;
      const double2 x0 = src[0];
      double2 acc[KB];
      int e0[KB], ex[KB];
#pragma unroll
      for (int q = 0; q < KB; ++q) {
        const int k = kg + KG * q;
        e0[q] = (jm + k * Ns) * tstep % N;  // < N (k < R); k >= R is computed and discarded
        ex[q] = 0;
        acc[q] = x0;
      }
#pragma unroll 2
      for (int r = 1; r < R; ++r) {
        const double2 v = src[r * NR * es];
#pragma unroll
        for (int q = 0; q < KB; ++q) {
          ex[q] += e0[q];
          if (ex[q] >= N) ex[q] -= N;
          const double2 t = tws[ex[q]];
          acc[q] = cadd(acc[q], sign < 0 ? cmul(v, t) : cmulc(v, t));
        }
      }
      const int ob = (j / Ns) * Ns * R + jm;
#pragma unroll
      for (int q = 0; q < KB; ++q) {
        const int k = kg + KG * q;
        if (k < R) b[l * ls + (ob + k * Ns) * es] = acc[q];
      }
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
