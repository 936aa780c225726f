// Register-resident Stockham FFT engine for power-of-two lines (fp64).
//
// A line of N complex values is spread over T = N/E threads, thread t holding
// elements {t + T m : m < E} in registers.  Every Stockham stage of radix R
// (R | E) reads exactly that element set back (j = t + T b, inputs
// j + r N/R = t + T (b + r E/R)), so the first stage loads straight from HBM,
// the last stage leaves its outputs in the same pattern for a straight store,
// and only the inter-stage permutations go through shared memory.  Lines are
// interleaved in shared memory (element p of line l at sm[p*LS + l]) so that
// the lanes of a warp, lines fastest, hit consecutive 16-byte words: a full
// 128-byte wavefront per 8 lanes, conflict-free for every permutation.
#pragma once

#include "fft_smem.cuh"

namespace fm {
namespace reg {

// W_16^k = exp(-2 pi i k / 16), folded to immediates after unrolling.
__host__ __device__ constexpr double c16(int k) {
  return k == 0 ? 1.0 : k == 1 ? 0.92387953251128674 : k == 2 ? 0.70710678118654757
       : k == 3 ? 0.38268343236508978 : k == 4 ? 0.0 : k == 5 ? -0.38268343236508978
       : k == 6 ? -0.70710678118654757 : k == 7 ? -0.92387953251128674 : k == 8 ? -1.0
       : k == 9 ? -0.92387953251128674 : k == 10 ? -0.70710678118654757
       : k == 11 ? -0.38268343236508978 : k == 12 ? 0.0 : k == 13 ? 0.38268343236508978
       : k == 14 ? 0.70710678118654757 : 0.92387953251128674;
}
__host__ __device__ constexpr double s16(int k) { return -c16((k + 12) & 15); }  // sin(-2 pi k/16)

// x * W_R^k for compile-time R, k (SIGN = -1 forward, +1 inverse).
template <int R, int K, int SIGN>
__device__ __forceinline__ double2 twc(double2 x) {
  constexpr int k16 = (K * (16 / R)) & 15;
  if constexpr (k16 == 0) {
    return x;
  } else if constexpr (k16 == 8) {
    return make_double2(-x.x, -x.y);
  } else if constexpr (k16 == 4) {  // forward: -i ; inverse: +i
    return SIGN < 0 ? make_double2(x.y, -x.x) : make_double2(-x.y, x.x);
  } else if constexpr (k16 == 12) {
    return SIGN < 0 ? make_double2(-x.y, x.x) : make_double2(x.y, -x.x);
  } else {
    constexpr double c = c16(k16);
    constexpr double s = SIGN < 0 ? s16(k16) : -s16(k16);
    return make_double2(x.x * c - x.y * s, x.x * s + x.y * c);
  }
}

// In-register DFT of R points (decimation in time, radix-2 recursion).
template <int R, int SIGN>
struct Dft {
  template <int I>
  __device__ __forceinline__ static void combine(double2* a, const double2* e, const double2* o) {
    if constexpr (I < R / 2) {
      const double2 t = twc<R, I, SIGN>(o[I]);
      a[I] = make_double2(e[I].x + t.x, e[I].y + t.y);
      a[I + R / 2] = make_double2(e[I].x - t.x, e[I].y - t.y);
      combine<I + 1>(a, e, o);
    }
  }
  __device__ __forceinline__ static void run(double2* a) {
    double2 e[R / 2], o[R / 2];
#pragma unroll
    for (int i = 0; i < R / 2; ++i) {
      e[i] = a[2 * i];
      o[i] = a[2 * i + 1];
    }
    Dft<R / 2, SIGN>::run(e);
    Dft<R / 2, SIGN>::run(o);
    combine<0>(a, e, o);
  }
};
template <int SIGN>
struct Dft<1, SIGN> {
  __device__ __forceinline__ static void run(double2*) {}
};
template <int SIGN>
struct Dft<2, SIGN> {
  __device__ __forceinline__ static void run(double2* a) {
    const double2 x = a[0], y = a[1];
    a[0] = make_double2(x.x + y.x, x.y + y.y);
    a[1] = make_double2(x.x - y.x, x.y - y.y);
  }
};

__device__ __forceinline__ double2 tw_mul(double2 x, double2 w, int sign) {
  return sign < 0 ? make_double2(x.x * w.x - x.y * w.y, x.x * w.y + x.y * w.x)
                  : make_double2(x.x * w.x + x.y * w.y, x.y * w.x - x.x * w.y);
}

// Exchange-buffer address of element p.  SW = 0: lines interleaved,
// sm[p*LS + l] (the lanes of a warp are lines).  SW = log2(E) > 0: one line
// per contiguous region with an XOR swizzle p ^ ((p >> SW) & 7), for lanes
// that are the T threads of a line: every group of 8 lanes that a 16-byte
// access serves in one phase then hits 8 distinct bank groups, both for the
// strided Stockham writes (p = E j + k) and the unit-stride reads.
template <int SW>
__device__ __forceinline__ int xaddr(int p, int LS) {
  if constexpr (SW == 0) return p * LS;
  else return p ^ ((p >> SW) & 7);
}

// One Stockham stage of radix R (Ns = product of earlier radices).
// tw: table W_N^e, e < N (global or shared), or, with TS > 1, a table of
// W_{N TS} read at stride TS.  sml = sm + line offset.
template <int N, int E, int R, int Ns, int SIGN, int SW = 0, int TS = 1>
__device__ __forceinline__ void stage(double2 (&v)[E], double2* sml, int LS, int t,
                                      const double2* __restrict__ tw) {
  constexpr int T = N / E;
  constexpr int B = E / R;
  constexpr bool last = (Ns * R == N);
  // Butterfly b reads v[b + r B] and (last stage) writes v[b + k B]: the
  // same residue class mod B, so the update is in place.
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const int j = t + T * b;
    const int jm = j & (Ns - 1);
    double2 a[R];
#pragma unroll
    for (int r = 0; r < R; ++r) a[r] = v[b + r * B];
    if constexpr (Ns > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) a[r] = tw_mul(a[r], __ldg(&tw[jm * r * (N / (Ns * R)) * TS]), SIGN);
    }
    Dft<R, SIGN>::run(a);
    if constexpr (last) {
#pragma unroll
      for (int k = 0; k < R; ++k) v[b + k * B] = a[k];
    } else {
      const int base = (j / Ns) * Ns * R + jm;
#pragma unroll
      for (int k = 0; k < R; ++k) sml[xaddr<SW>(base + k * Ns, LS)] = a[k];
    }
  }
  if constexpr (!last) {
    // SW > 0: a line's T threads are lanes of one warp and own its region
    if constexpr (SW > 0) __syncwarp(); else __syncthreads();
#pragma unroll
    for (int m = 0; m < E; ++m) v[m] = sml[xaddr<SW>(t + T * m, LS)];
    if constexpr (SW > 0) __syncwarp(); else __syncthreads();
  }
}

template <int N, int E, int Ns, int SIGN, int SW, int TS = 1>
struct Stages {
  static constexpr int R = (N / Ns >= E) ? E : N / Ns;
  __device__ __forceinline__ static void run(double2 (&v)[E], double2* sml, int LS, int t,
                                             const double2* __restrict__ tw) {
    stage<N, E, R, Ns, SIGN, SW, TS>(v, sml, LS, t, tw);
    Stages<N, E, Ns * R, SIGN, SW, TS>::run(v, sml, LS, t, tw);
  }
};
template <int N, int E, int SIGN, int SW, int TS>
struct Stages<N, E, N, SIGN, SW, TS> {
  __device__ __forceinline__ static void run(double2 (&)[E], double2*, int, int, const double2*) {}
};

// Full N-point transform of the register-resident line (unnormalised).
// TS > 1: tw is the W_{N TS} table (a longer line's), read at stride TS.
template <int N, int E, int SIGN, int TS = 1>
__device__ __forceinline__ void fft(double2 (&v)[E], double2* sml, int LS, int t,
                                    const double2* __restrict__ tw) {
  static_assert(N % E == 0, "E must divide N");
  Stages<N, E, 1, SIGN, 0, TS>::run(v, sml, LS, t, tw);
}

constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x / 2); }

// Same transform for lanes that are the T threads of one line (T | 32, so a
// line never straddles a warp and warp-level syncs suffice), exchanging
// through the line's own swizzled region of N elements (sml = sm + line * N).
// Every lane of the warp must call it.
template <int N, int E, int SIGN>
__device__ __forceinline__ void fft_swz(double2 (&v)[E], double2* sml, int t, const double2* __restrict__ tw) {
  static_assert(N % E == 0 && E >= 8, "E must divide N; the swizzle needs E >= 8");
  Stages<N, E, 1, SIGN, ilog2(E)>::run(v, sml, 1, t, tw);
}

// Elements per thread used by each pass for a line length N.
__host__ __device__ constexpr int e_line(int N) { return N >= 128 ? 16 : (N >= 8 ? 8 : N); }
__host__ __device__ constexpr int e_z(int M) { return M >= 8 ? 8 : M; }
__host__ __device__ constexpr int e_x(int N) { return N >= 8 ? 8 : N; }

}  // namespace reg
}  // namespace fm
