// Register-resident projection passes for power-of-two line lengths
// (fft_reg.cuh).  Same five-pass structure, spectral layout and arithmetic
// contract as the generic passes in projection.cu (reference
// projection.cpp:123-194); these are the kernels the 128^3..1024^3 configs run.
//
// Per pass and voxel the HBM traffic is one 9-component read and one write
// (pass 1 additionally reads K4); everything else stays on chip:
//   z passes : G z-lines x 9 components staged in shared memory (prologue /
//              epilogue one thread per voxel, coalesced), M = Nz/2-point
//              complex FFT with lines interleaved, r2c/c2r untangling in smem.
//   y pass   : TW = 8 consecutive kz columns per CTA, loads straight into
//              registers (8 lanes x 16 B = one 128-byte segment).
//   x pass   : one thread holds all 3 components of its row, so the
//              projection Bhat_i. = (Ahat_i . xi) xi / |xi|^2 is applied in
//              registers between the forward and inverse x transforms.
#include <cuda.h>  // CUtensorMap (the encoder is fetched with cudaGetDriverEntryPoint)

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <type_traits>
#include <vector>

#include "bulk.cuh"
#include "fft_pair.cuh"
#include "proj_common.cuh"

namespace fm {

using reg::e_line;
using reg::e_x;

// ------------------------------------------------------------------ y pass
// In place on one device.  P > 1: SIGN -1 stores each element into the x-pass
// input of the rank that owns its y (the fused forward slab transpose,
// store_yf); SIGN +1 runs in place on the spectrum of the x-slab.
// (Register budget of 128 for every instantiation: the routed forward pass
// otherwise takes 146 registers at 512 points and loses its second CTA per SM
// -- 6.5 instead of 3.2 ms at 512^3 with 8 ranks.)
template <int N, int TW>
constexpr int y_minb() {
  return std::max(1, 512 / (TW * (N / e_line(N))));
}
template <int N, int TW, int SIGN, bool RT = false>
__global__ void __launch_bounds__(TW*(N / e_line(N)), y_minb<N, TW>()) k_y_fast(Geo g, const double2* __restrict__ tw,
                                                               const double2* in, double2* out) {
  constexpr int E = e_line(N), T = N / E;
  extern __shared__ double2 sm[];
  const int l = threadIdx.x % TW, t = threadIdx.x / TW;
  const int kz = blockIdx.x * TW + l;
  const int x = blockIdx.y, c = blockIdx.z;
  double2 v[E];
#pragma unroll
  for (int m = 0; m < E; ++m) v[m] = in[spec_std(g, c, x, t + T * m, kz)];
  reg::fft<N, E, SIGN>(v, sm + l, TW, t, tw);
  if constexpr (!RT) {
#pragma unroll
    for (int m = 0; m < E; ++m) out[spec_std(g, c, x, t + T * m, kz)] = v[m];
  } else {
    // route_yf (proj_common.cuh) with the per-line part hoisted: element y goes
    // to rank d = y / Yl at base + yl nzh, base = ((c Nxg + rank Xl + x) Yl) nzh + kz.
    // Yl is a power of two here (N is, and P divides it), so d and yl are a
    // shift and a mask instead of a division per element.
    const int64_t base = ((int64_t(c) * g.Nxg + int64_t(g.rank) * g.Nx + x) * g.Yl) * g.nzh + kz;
    const int sh = 31 - __clz(g.Yl);
#pragma unroll
    for (int m = 0; m < E; ++m) {
      const int y = t + T * m;
      g.dst[y >> sh][base + int64_t(y & (g.Yl - 1)) * g.nzh] = v[m];
    }
  }
}

// ------------------------------------------------------------------ x pass
// All x passes: in place on one device; P > 1 they read the y-slab input B
// (disjoint from every destination, so __restrict__ holds in both cases)
// and store each element into the spectrum of the rank that owns its x (the
// fused backward slab transpose, store_xb).
template <int N, int TW, int TD, bool RT = false>
__global__ void __launch_bounds__(TW*(N / e_x(N)), 2) k_x_fast(Geo g, const double2* __restrict__ tw,
                                                            double2* __restrict__ spec) {
  constexpr int E = e_x(N), T = N / E;
  extern __shared__ double2 sm[];
  const int l = threadIdx.x % TW, t = threadIdx.x / TW;
  const int kz = blockIdx.x * TW + l;
  const int y = blockIdx.y, i = blockIdx.z;
  const int64_t xstride = int64_t(g.Ny) * g.nzh;
  double2* base = spec + int64_t(i * TD) * N * xstride + int64_t(y) * g.nzh + kz;
  double2 v[TD][E];
#pragma unroll
  for (int j = 0; j < TD; ++j)
#pragma unroll
    for (int m = 0; m < E; ++m) v[j][m] = base[(int64_t(j) * N + t + T * m) * xstride];
#pragma unroll
  for (int j = 0; j < TD; ++j) reg::fft<N, E, -1>(v[j], sm + l, TW, t, tw);
  // Bhat_ij = sum_l Ahat_il ghat_lj  (projection.cpp:87-104, 139-152)
  const int yg = g.y0 + y;  // global y (slab decomposition: y-slab of this rank)
  const int qy = freq_of(yg, g.Nyg), qz = freq_of(kz, g.Nz);
  const bool nyq_yz = ((g.Nyg % 2 == 0) && (yg == g.Nyg / 2)) || ((g.Nz % 2 == 0) && (kz == g.Nz / 2));
  const double xiy = qy * g.invL[1], xiz = (g.dim == 3) ? qz * g.invL[2] : 0.0;
#pragma unroll
  for (int m = 0; m < E; ++m) {
    const int kx = t + T * m;
    const double xix = freq_of(kx, N) * g.invL[0];
    const double xi[3] = {xix, xiy, xiz};
    const double norm2 = xix * xix + xiy * xiy + xiz * xiz;
    const bool nyq = nyq_yz || (kx == N / 2);
    if (norm2 == 0.0 || (nyq && g.mode == FM_NYQUIST_ZERO_COMPATIBLE)) {
#pragma unroll
      for (int j = 0; j < TD; ++j) v[j][m] = make_double2(0.0, 0.0);
    } else if (!nyq) {
      double sx = 0.0, sy = 0.0;
#pragma unroll
      for (int q = 0; q < TD; ++q)
        if (q < g.dim) {
          sx += v[q][m].x * xi[q];
          sy += v[q][m].y * xi[q];
        }
      const double inv = 1.0 / norm2;
#pragma unroll
      for (int j = 0; j < TD; ++j) {
        const double f = j < g.dim ? xi[j] * inv : 0.0;
        v[j][m] = make_double2(sx * f, sy * f);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < TD; ++j) reg::fft<N, E, +1>(v[j], sm + l, TW, t, tw);
  if constexpr (!RT) {
#pragma unroll
    for (int j = 0; j < TD; ++j)
#pragma unroll
      for (int m = 0; m < E; ++m) base[(int64_t(j) * N + t + T * m) * xstride] = v[j][m];
  } else {
#pragma unroll
    for (int j = 0; j < TD; ++j)
#pragma unroll
      for (int m = 0; m < E; ++m) store_xb(g, nullptr, i * TD + j, t + T * m, y, kz, v[j][m]);
  }
}

// x pass, prefetching variant: the whole tile (3 components x N x TW) is
// requested from HBM at once with cp.async (16 B per request, 8 lanes per
// 128-byte row) so all of it is in flight together; the components are then
// transformed one at a time out of shared memory, projected on the
// thread-owned positions, transformed back and stored.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n" ::);
  asm volatile("cp.async.wait_group 0;\n" ::);
}

template <int N, int TW, int E, bool RT = false>
__global__ void __launch_bounds__(TW*(N / E)) k_x_fast3(Geo g, const double2* __restrict__ tw,
                                                       double2* __restrict__ spec) {
  constexpr int T = N / E;
  extern __shared__ double2 sm[];
  const int l = threadIdx.x % TW, t = threadIdx.x / TW;
  const int kz = blockIdx.x * TW + l;
  const int y = blockIdx.y, i = blockIdx.z;
  const int64_t xstride = int64_t(g.Ny) * g.nzh;
  double2* tile = spec + int64_t(i * 3) * N * xstride + int64_t(y) * g.nzh + blockIdx.x * TW;
  for (int w = threadIdx.x; w < 3 * N * TW; w += blockDim.x) {
    const int row = w / TW, ll = w - row * TW;  // row = j * N + e
    cp_async16(sm + w, tile + int64_t(row) * xstride + ll);
  }
  cp_async_wait_all();
  __syncthreads();
  double2* base = tile + l;
#pragma unroll 1
  for (int j = 0; j < 3; ++j) {
    double2* S = sm + j * N * TW + l;
    double2 v[E];
#pragma unroll
    for (int m = 0; m < E; ++m) v[m] = S[(t + T * m) * TW];
    __syncthreads();
    reg::fft<N, E, -1>(v, S, TW, t, tw);
#pragma unroll
    for (int m = 0; m < E; ++m) S[(t + T * m) * TW] = v[m];
  }
  const int yg = g.y0 + y;
  const int qy = freq_of(yg, g.Nyg), qz = freq_of(kz, g.Nz);
  const bool nyq_yz = ((g.Nyg % 2 == 0) && (yg == g.Nyg / 2)) || ((g.Nz % 2 == 0) && (kz == g.Nz / 2));
  const double xiy = qy * g.invL[1], xiz = (g.dim == 3) ? qz * g.invL[2] : 0.0;
#pragma unroll 2
  for (int m = 0; m < E; ++m) {  // own positions only: no barrier needed
    const int kx = t + T * m;
    double2* s0 = sm + kx * TW + l;
    const double xix = freq_of(kx, N) * g.invL[0];
    const double norm2 = xix * xix + xiy * xiy + xiz * xiz;
    const bool nyq = nyq_yz || (kx == N / 2);
    double2 a0 = s0[0], a1 = s0[N * TW], a2 = s0[2 * N * TW];
    if (norm2 == 0.0 || (nyq && g.mode == FM_NYQUIST_ZERO_COMPATIBLE)) {
      a0 = a1 = a2 = make_double2(0.0, 0.0);
    } else if (!nyq) {
      const double sx = a0.x * xix + a1.x * xiy + a2.x * xiz;
      const double sy = a0.y * xix + a1.y * xiy + a2.y * xiz;
      const double inv = 1.0 / norm2;
      const double f0 = xix * inv, f1 = xiy * inv, f2 = xiz * inv;
      a0 = make_double2(sx * f0, sy * f0);
      a1 = make_double2(sx * f1, sy * f1);
      a2 = make_double2(sx * f2, sy * f2);
    }
    s0[0] = a0;
    s0[N * TW] = a1;
    s0[2 * N * TW] = a2;
  }
#pragma unroll 1
  for (int j = 0; j < 3; ++j) {
    double2 v[E];
    double2* S = sm + j * N * TW + l;
#pragma unroll
    for (int m = 0; m < E; ++m) v[m] = S[(t + T * m) * TW];
    __syncthreads();
    reg::fft<N, E, +1>(v, S, TW, t, tw);
    if constexpr (!RT) {
#pragma unroll
      for (int m = 0; m < E; ++m) base[(int64_t(j) * N + t + T * m) * xstride] = v[m];
    } else {
#pragma unroll
      for (int m = 0; m < E; ++m) store_xb(g, nullptr, i * 3 + j, t + T * m, y, kz, v[m]);
    }
  }
}

// x pass, scalar-accumulating variant (ZeroCompatible mode only).  The
// projection of row i is Bhat_ij = s xi_j / |xi|^2 with s = sum_q Ahat_iq xi_q,
// so the forward transforms only have to accumulate s in registers: per
// thread E values of s plus E working values, instead of all 3 x E.  Since
// xi_y and xi_z are constant along an x-line, linearity folds the row into
// two forward and two inverse transforms instead of three and three.
// Component tiles (N x TW) are double-buffered in shared memory with cp.async
// (component q+2 streams in while q is transformed) and each buffer doubles
// as the transform's exchange scratch; the inverse transforms store straight
// from registers.  64 KB per CTA at N = 256, TW = 8.
template <int N, int TW, int E>
constexpr int x4_minb() {  // CTAs/SM the register budget targets: capped by the two tile buffers
  return std::max(1, std::min(E >= 16 ? 3 : 2, int((227 * 1024) / (2 * size_t(N) * TW * 16 + 1024))));
}
// FM_X4_DBG (builds with -DFM_X4_DEBUG only; timing experiments): bit 0 skips
// the transforms, bit 1 the stores, bit 2 the tile loads.
#ifdef FM_X4_DEBUG
__device__ int x4_dbg_bits;
#define X4_DBG(bit) (x4_dbg_bits & (bit))
#else
#define X4_DBG(bit) 0
#endif
template <int N, int TW, int E, bool RT = false>
__global__ void __launch_bounds__(TW*(N / E), x4_minb<N, TW, E>()) k_x_fast4(Geo g, const double2* __restrict__ tw,
                                                       double2* __restrict__ spec) {
  constexpr int T = N / E;
  extern __shared__ double2 sm[];
  const int l = threadIdx.x % TW, t = threadIdx.x / TW;
  const int kz = blockIdx.x * TW + l;
  const int y = blockIdx.y, i = blockIdx.z;
  const int64_t xstride = int64_t(g.Ny) * g.nzh;
  double2* tile = spec + int64_t(i * 3) * N * xstride + int64_t(y) * g.nzh + blockIdx.x * TW;
  auto fetch = [&](int q, double2* buf) {
    const double2* src = tile + int64_t(q) * N * xstride;
    if (X4_DBG(4)) return;
    for (int w = threadIdx.x; w < N * TW; w += blockDim.x) {
      const int row = w / TW, ll = w - row * TW;
      cp_async16(buf + w, src + int64_t(row) * xstride + ll);
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  double2* buf0 = sm;
  double2* buf1 = sm + N * TW;
  fetch(0, buf0);
  fetch(1, buf1);
  const int yg = g.y0 + y;
  const int qy = freq_of(yg, g.Nyg), qz = freq_of(kz, g.Nz);
  const bool nyq_yz = ((g.Nyg % 2 == 0) && (yg == g.Nyg / 2)) || ((g.Nz % 2 == 0) && (kz == g.Nz / 2));
  const double xiy = qy * g.invL[1], xiz = qz * g.invL[2];
  double2 s[E], v[E];
  // s = FFT(A_i0) xi_x + FFT(A_i1) xi_y + FFT(A_i2) xi_z.  xi_y and xi_z are
  // constant along the x-line, so by linearity the last two terms are ONE
  // transform, FFT(xi_y A_i1 + xi_z A_i2): two forward FFTs instead of three.
  // (Rolled loops keep one copy of each transform: the register budget.)
#pragma unroll 1
  for (int q = 0; q < 2; ++q) {
    if (q == 0) asm volatile("cp.async.wait_group 1;\n" ::);  // tile 0 (tile 1 may still be in flight)
    else asm volatile("cp.async.wait_group 0;\n" ::);          // tiles 1 and 2
    __syncthreads();
    if (q == 0) {
#pragma unroll
      for (int m = 0; m < E; ++m) v[m] = buf0[(t + T * m) * TW + l];
    } else {
#pragma unroll
      for (int m = 0; m < E; ++m) {
        const double2 a1 = buf1[(t + T * m) * TW + l], a2 = buf0[(t + T * m) * TW + l];
        v[m] = make_double2(fma(a1.x, xiy, a2.x * xiz), fma(a1.y, xiy, a2.y * xiz));
      }
    }
    __syncthreads();
    double2* X = q == 0 ? buf0 : buf1;
    if (!X4_DBG(1)) reg::fft<N, E, -1>(v, X + l, TW, t, tw);  // ends past a barrier: X is free again
    else __syncthreads();
    if (q == 0) {
      fetch(2, buf0);
#pragma unroll
      for (int m = 0; m < E; ++m) {
        const double xq = freq_of(t + T * m, N) * g.invL[0];
        s[m] = make_double2(v[m].x * xq, v[m].y * xq);
      }
    } else {
#pragma unroll
      for (int m = 0; m < E; ++m) s[m] = make_double2(s[m].x + v[m].x, s[m].y + v[m].y);
    }
  }
  // s <- s / |xi|^2, zero at xi = 0 and on Nyquist planes (ZeroCompatible)
#pragma unroll
  for (int m = 0; m < E; ++m) {
    const int kx = t + T * m;
    const double xix = freq_of(kx, N) * g.invL[0];
    const double norm2 = xix * xix + xiy * xiy + xiz * xiz;
    const bool zero = norm2 == 0.0 || nyq_yz || kx == N / 2;
    const double inv = zero ? 0.0 : 1.0 / norm2;
    s[m] = make_double2(s[m].x * inv, s[m].y * inv);
  }
  // Bhat_i0 = IFFT(s xi_x); Bhat_i1 = xi_y IFFT(s), Bhat_i2 = xi_z IFFT(s): two
  // inverse FFTs instead of three, by the same linearity
  double2* base = tile + l;
#pragma unroll 1
  for (int q = 0; q < 2; ++q) {
#pragma unroll
    for (int m = 0; m < E; ++m) {
      const double f = q == 0 ? freq_of(t + T * m, N) * g.invL[0] : 1.0;
      v[m] = make_double2(s[m].x * f, s[m].y * f);
    }
    if (!X4_DBG(1)) reg::fft<N, E, +1>(v, (q == 0 ? buf0 : buf1) + l, TW, t, tw);
#pragma unroll 1
    for (int j = q; j < (q == 0 ? 1 : 3); ++j) {
      const double f = j == 0 ? 1.0 : (j == 1 ? xiy : xiz);
      if (X4_DBG(2)) continue;
      if constexpr (!RT) {
#pragma unroll
        for (int m = 0; m < E; ++m)
          base[(int64_t(j) * N + t + T * m) * xstride] = make_double2(v[m].x * f, v[m].y * f);
      } else {
        const int sh = 31 - __clz(g.Xl);
        const int64_t rb = xb_base(g, i * 3 + j, y, kz);
#pragma unroll
        for (int m = 0; m < E; ++m)
          store_xb_pow2(g, sh, rb, t + T * m, make_double2(v[m].x * f, v[m].y * f));
      }
    }
  }
}

// x pass for N = 2H (512 = 2 x 256), scalar-accumulating like k_x_fast4, with
// the outermost radix-2 step done across a lane pair instead of through
// shared memory.  Decimation in time: X[k] = E[k] + W_N^k O[k] and
// X[k + H] = E[k] - W_N^k O[k], E and O the H-point transforms of the even and
// odd rows.  The T = N/E threads of a line are two groups of TH = H/E: group
// h = 0 transforms the even rows, h = 1 the odd ones (each an H-point
// register FFT with ONE shared-memory exchange at H = 256, where the N-point
// transform needs two), then the lane pair (lanes TW apart) swaps half its
// values with one shuffle per element and each lane forms both outputs of its
// half of the butterflies.  Spectrum slot s of lane (t, h) then holds
// frequency kslot(t, h, s) below; every frequency-domain step of this pass is
// pointwise, so the permuted order is used as is, and the inverse transforms
// run the mirror image (decimation in frequency: the radix-2 split by
// shuffle, then two H-point inverse FFTs whose outputs are rows 2n and
// 2n + 1).
// The same 512-point x pass without tile staging, shaped like the y pass:
// 8-column tiles (one 128-byte segment per row and component, where the
// staged pass's 64 KB double buffer only allows 4 columns = 64-byte
// segments), every lane loading its rows straight from HBM into registers and
// storing its results straight from registers; shared memory is only the
// one H-point exchange buffer (64 KB), 2 CTAs x 256 threads per SM.  The
// forward transform of B = xi_y A_1 + xi_z A_2 runs first, so the
// accumulator is not live while A_1 and A_2 are loaded.
template <int N, int TW, bool RT = false>
__global__ void __launch_bounds__(TW * 32, 2) k_x_direct(Geo g, const double2* __restrict__ tw,
                                                         double2* __restrict__ spec) {
  constexpr int E = 16, H = N / 2, TH = H / E;
  static_assert(TH == 16 && TW * 2 <= 32, "lane pairs inside a warp");
  extern __shared__ double2 sm[];
  const int l = threadIdx.x % TW, u = threadIdx.x / TW;
  const int h = u & 1, t = u >> 1;
  const int kz = blockIdx.x * TW + l;
  const int y = blockIdx.y, i = blockIdx.z;
  const int64_t xstride = int64_t(g.Ny) * g.nzh;
  // rows 2 (t + TH m) + h of this lane: one base pointer, 32-bit element offsets
  // (the launcher checks 3 N xstride < 2^31)
  const int rs = 2 * TH * int(xstride);
  double2* const row0 = spec + int64_t(i * 3) * N * xstride + (2 * t + h) * xstride + int64_t(y) * g.nzh + kz;
  const int cs = N * int(xstride);  // component stride
  const int yg = g.y0 + y;
  const int qy = freq_of(yg, g.Nyg), qz = freq_of(kz, g.Nz);
  const bool nyq_yz = ((g.Nyg % 2 == 0) && (yg == g.Nyg / 2)) || ((g.Nz % 2 == 0) && (kz == g.Nz / 2));
  const double xiy = qy * g.invL[1], xiz = qz * g.invL[2];
  double2* const X = sm + l + TW * h;  // sub-line of the H-point exchange (2 TW per CTA, interleaved)
  auto ld = [&](int off) { return row0[off]; };
  double2 s[E], v[E];
#pragma unroll
  for (int m = 0; m < E; ++m) v[m] = ld(cs + m * rs);
#pragma unroll
  for (int m = 0; m < E; ++m) {
    const double2 a2 = ld(2 * cs + m * rs);
    v[m] = make_double2(fma(v[m].x, xiy, a2.x * xiz), fma(v[m].y, xiy, a2.y * xiz));
  }
  reg::fft<H, E, -1, 2>(v, X, 2 * TW, t, tw);
  pair_dit<TH, TW>(v, t, h, tw);
#pragma unroll
  for (int m = 0; m < E; ++m) s[m] = v[m];
#pragma unroll
  for (int m = 0; m < E; ++m) v[m] = ld(m * rs);
  reg::fft<H, E, -1, 2>(v, X, 2 * TW, t, tw);
  pair_dit<TH, TW>(v, t, h, tw);
  // s = (xi_x FFT(A_0) + FFT(B)) / |xi|^2, zero at xi = 0 and on Nyquist planes
#pragma unroll
  for (int m = 0; m < E; ++m) {
    const int kx = kslot<TH, H>(t, h, m);
    const double xix = freq_of(kx, N) * g.invL[0];
    const double norm2 = xix * xix + xiy * xiy + xiz * xiz;
    const bool zero = norm2 == 0.0 || nyq_yz || kx == N / 2;
    const double inv = zero ? 0.0 : 1.0 / norm2;
    s[m] = make_double2((v[m].x * xix + s[m].x) * inv, (v[m].y * xix + s[m].y) * inv);
  }
  // Bhat_i0 = IFFT(s xi_x); Bhat_i1 = xi_y IFFT(s), Bhat_i2 = xi_z IFFT(s)
#pragma unroll 1
  for (int q = 0; q < 2; ++q) {
#pragma unroll
    for (int m = 0; m < E; ++m) {
      const double f = q == 0 ? freq_of(kslot<TH, H>(t, h, m), N) * g.invL[0] : 1.0;
      v[m] = make_double2(s[m].x * f, s[m].y * f);
    }
    pair_dif<TH, TW>(v, t, h, tw);
    reg::fft<H, E, +1, 2>(v, X, 2 * TW, t, tw);
#pragma unroll 1
    for (int j = q; j < (q == 0 ? 1 : 3); ++j) {
      const double f = j == 0 ? 1.0 : (j == 1 ? xiy : xiz);
      if constexpr (!RT) {
#pragma unroll
        for (int m = 0; m < E; ++m)
          row0[j * cs + m * rs] = make_double2(v[m].x * f, v[m].y * f);
      } else {
#pragma unroll
        for (int m = 0; m < E; ++m)
          store_xb(g, nullptr, i * 3 + j, 2 * (t + TH * m) + h, y, kz, make_double2(v[m].x * f, v[m].y * f));
      }
    }
  }
}

// The x pass for long lines (N = 512, 1024), streamed: the component tiles
// of a row (N x TW each) arrive in shared memory by bulk async copies
// (cp.async.bulk, one 16*TW-byte row segment per copy, mbarrier completion)
// instead of register loads, so no HBM latency is exposed to the transforms
// and nothing caps the registers: persistent CTAs (one per SM, TW * N/16
// threads) walk the (kz block, y, row) tiles.  Buffers C1 / C2 (components
// 1, 2) are refilled with the NEXT tile's as soon as the forward transform of
// B = xi_y A_1 + xi_z A_2 has consumed them, C0 once the inverse transforms
// (which exchange through it) are done; every buffer doubles as the exchange
// scratch of the transform that consumed it.  The transforms are the plain
// N-point register FFT of k_x_fast4 (E = 16 elements per thread: 16 x 16 x 2
// at 512), whose 168-register footprint fits where k_x_direct's lane-pair
// variant spilled at 128.
// Thread shape of k_x_stream: E elements per thread; PAIR: the lane-pair
// split of k_x_direct (two H = N/2-point half-line transforms joined by a
// shuffle radix-2 step: one shared-memory exchange per transform at 512
// instead of two).
template <int N, int E, bool PAIR>
struct XsShape {
  static constexpr int T = N / E;  // threads per line
  static constexpr int H = N / 2, TH = H / E;
};
template <int N, int TW, int E, bool PAIR, bool RT = false>
__global__ void __launch_bounds__(TW * (N / E), 1) k_x_stream(Geo g, const double2* __restrict__ tw,
                                                             double2* spec, int tiles,
                                                             const __grid_constant__ CUtensorMap tmap, int dbg) {
  using S = XsShape<N, E, PAIR>;
  constexpr int T = S::T, TH = S::TH, H = S::H;
  static_assert(!PAIR || (E == 16 && TH == 16 && TW * 2 <= 32), "lane pairs inside a warp");
  constexpr int TILE = N * TW;  // complex elements of one component tile
  extern __shared__ __align__(128) double2 sm[];
  __shared__ uint64_t bar[3];
  const int l = threadIdx.x % TW, u = threadIdx.x / TW;
  const int h = PAIR ? (u & 1) : 0, t = PAIR ? (u >> 1) : u;
  const int64_t xstride = int64_t(g.Ny) * g.nzh;
  const int kzb = g.nzh / TW;
  auto buf = [&](int q) { return sm + q * TILE; };
  // The twiddles only depend on t, so the compiler would hoist all of them out
  // of the persistent loop and keep them live (~90 registers, spills): each
  // transform gets the table through an opaque copy of the pointer instead.
  auto twp = [&]() {
    const double2* p;
    asm volatile("mov.b64 %0, %1;\n" : "=l"(p) : "l"(tw));
    return p;
  };
  // row of slot m; frequency held in slot m after the forward transform
  auto row_of = [&](int m) { return PAIR ? 2 * (t + TH * m) + h : t + T * m; };
  auto kx_of = [&](int m) { return PAIR ? kslot<TH, H>(t, h, m) : t + T * m; };
  // dbg (FM_X_DBG, timing experiments only): bit 0 skips the transforms,
  // bit 1 the stores
  auto fwd = [&](double2(&v)[E], double2* X) {
    if (dbg & 1) return;
    if constexpr (PAIR) {
      reg::fft<H, E, -1, 2>(v, X + l + TW * h, 2 * TW, t, twp());
      pair_dit<TH, TW>(*reinterpret_cast<double2(*)[16]>(&v), t, h, twp());
    } else {
      reg::fft<N, E, -1>(v, X + l, TW, t, twp());
    }
  };
  auto inv = [&](double2(&v)[E], double2* X) {
    if (dbg & 1) return;
    if constexpr (PAIR) {
      pair_dif<TH, TW>(*reinterpret_cast<double2(*)[16]>(&v), t, h, twp());
      reg::fft<H, E, +1, 2>(v, X + l + TW * h, 2 * TW, t, twp());
    } else {
      reg::fft<N, E, +1>(v, X + l, TW, t, twp());
    }
  };
  // tile -> (kz block fastest, y, row i): neighbouring CTAs read neighbouring
  // 16 TW-byte segments of the same rows
  auto tile_base = [&](int T_, int& kz0, int& y, int& i) {
    kz0 = (T_ % kzb) * TW;
    const int r = T_ / kzb;
    y = r % g.Ny;
    i = r / g.Ny;
    return spec + int64_t(i * 3) * N * xstride + int64_t(y) * g.nzh + kz0;
  };
  // thread 0 fills buffer q with component q of tile T_: N / 256 tensor-map
  // boxes of 256 rows x TW columns (the map views the spectrum as
  // [comp * N + x][y][2 kz] doubles)
  auto issue = [&](int T_, int q) {
    if (threadIdx.x != 0 || (dbg & 4)) return;
    int kz0, y, i;
    tile_base(T_, kz0, y, i);
    bulk::mbar_expect_tx(&bar[q], TILE * 16);
#pragma unroll
    for (int r0 = 0; r0 < N; r0 += 256)
      bulk::tma3d(buf(q) + r0 * TW, &tmap, 2 * kz0, y, (i * 3 + q) * N + r0, &bar[q]);
  };
  if (threadIdx.x < 3) bulk::mbar_init(&bar[threadIdx.x], 1);
  __syncthreads();
  int T_ = blockIdx.x;
  if (T_ < tiles)
    for (int q = 0; q < 3; ++q) issue(T_, q);
  unsigned par = 0;
  for (; T_ < tiles; T_ += gridDim.x, par ^= 1) {
    int kz0, y, i;
    double2* const base = tile_base(T_, kz0, y, i);
    const int kz = kz0 + l;
    const int yg = g.y0 + y;
    const int qy = freq_of(yg, g.Nyg), qz = freq_of(kz, g.Nz);
    const bool nyq_yz = ((g.Nyg % 2 == 0) && (yg == g.Nyg / 2)) || ((g.Nz % 2 == 0) && (kz == g.Nz / 2));
    const double xiy = qy * g.invL[1], xiz = qz * g.invL[2];
    const int Tn = T_ + gridDim.x;  // next tile of this CTA
    double2 s[E], v[E];
    // forward transform of B = xi_y A_1 + xi_z A_2
    if (!(dbg & 4)) {
      bulk::mbar_wait(&bar[1], par);
      bulk::mbar_wait(&bar[2], par);
    }
#pragma unroll
    for (int m = 0; m < E; ++m) {
      const double2 a1 = buf(1)[row_of(m) * TW + l], a2 = buf(2)[row_of(m) * TW + l];
      v[m] = make_double2(fma(a1.x, xiy, a2.x * xiz), fma(a1.y, xiy, a2.y * xiz));
    }
    __syncthreads();  // C1, C2 consumed
    if (Tn < tiles) issue(Tn, 2);
    fwd(v, buf(1));
    // C1 held the exchange: order those generic writes before the async refill
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (Tn < tiles) issue(Tn, 1);
#pragma unroll
    for (int m = 0; m < E; ++m) s[m] = v[m];
    // forward transform of A_0
    if (!(dbg & 4)) bulk::mbar_wait(&bar[0], par);
#pragma unroll
    for (int m = 0; m < E; ++m) v[m] = buf(0)[row_of(m) * TW + l];
    __syncthreads();
    fwd(v, buf(0));
    // s = (xi_x FFT(A_0) + FFT(B)) / |xi|^2, zero at xi = 0 and on Nyquist planes
#pragma unroll
    for (int m = 0; m < E; ++m) {
      const int kx = kx_of(m);
      const double xix = freq_of(kx, N) * g.invL[0];
      const double norm2 = xix * xix + xiy * xiy + xiz * xiz;
      const bool zero = norm2 == 0.0 || nyq_yz || kx == N / 2;
      const double iv = zero ? 0.0 : 1.0 / norm2;
      s[m] = make_double2((v[m].x * xix + s[m].x) * iv, (v[m].y * xix + s[m].y) * iv);
    }
    // Bhat_i0 = IFFT(s xi_x); Bhat_i1 = xi_y IFFT(s), Bhat_i2 = xi_z IFFT(s)
    // (dbg bit 3: every tile stores over tile 0's rows -- L2-resident writes)
    double2* const rowp = ((dbg & 8) ? spec : base) + l;
#pragma unroll 1
    for (int q = 0; q < 2; ++q) {
#pragma unroll
      for (int m = 0; m < E; ++m) {
        const double f = q == 0 ? freq_of(kx_of(m), N) * g.invL[0] : 1.0;
        v[m] = make_double2(s[m].x * f, s[m].y * f);
      }
      inv(v, buf(0));
      if (q == 1) {
        // C0 (the inverse transforms' exchange) is free: refill it before the
        // last two components are stored, so that neither the fence nor the
        // next tile's load waits behind those stores
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncthreads();
        if (Tn < tiles) issue(Tn, 0);
        // every store reads its own registers (component 1 scaled into s, dead
        // by now; component 2 in place): a shared temporary would chain each
        // store behind the previous one's operand read
#pragma unroll
        for (int m = 0; m < E; ++m) {
          s[m] = make_double2(v[m].x * xiy, v[m].y * xiy);
          v[m] = make_double2(v[m].x * xiz, v[m].y * xiz);
        }
      }
      if (dbg & 2) continue;
      if constexpr (!RT) {
        double2* const o = rowp + (int64_t(q) * N + row_of(0)) * xstride;
        const int64_t ms = int64_t(row_of(1) - row_of(0)) * xstride;
        if (q == 0) {
#pragma unroll
          for (int m = 0; m < E; ++m) o[m * ms] = v[m];
        } else {
#pragma unroll
          for (int m = 0; m < E; ++m) o[m * ms] = s[m];
#pragma unroll
          for (int m = 0; m < E; ++m) o[int64_t(N) * xstride + m * ms] = v[m];
        }
      } else {
        if (q == 0) {
#pragma unroll
          for (int m = 0; m < E; ++m) store_xb(g, nullptr, i * 3, row_of(m), y, kz, v[m]);
        } else {
#pragma unroll
          for (int m = 0; m < E; ++m) store_xb(g, nullptr, i * 3 + 1, row_of(m), y, kz, s[m]);
#pragma unroll
          for (int m = 0; m < E; ++m) store_xb(g, nullptr, i * 3 + 2, row_of(m), y, kz, v[m]);
        }
      }
    }
  }
}

// r2c / c2r untangling pairs element k of a z-line with M - k.  With the
// line's elements spread as k = t + T m over its T lanes (T | 32), the partner
// of (t, m) sits in lane (T - t) mod T of the same warp:
// Value the mirror partner of this lane wants in round m (see above): lane t
// of a line hands out element (M - k') of its receiver's k' = (T - t) + T m.
template <int E>
__device__ __forceinline__ double2 mirror_give(const double2 (&v)[E], int t, int m) {
  return t == 0 ? v[(E - m) & (E - 1)] : v[E - 1 - m];
}
template <int T>
__device__ __forceinline__ double2 mirror_take(double2 give, int t) {
  const int lane = threadIdx.x & 31;
  const int src = lane - t + ((T - t) & (T - 1));
  return make_double2(__shfl_sync(0xffffffffu, give.x, src), __shfl_sync(0xffffffffu, give.y, src));
}

// --------------------------------------------------------------- z passes
// HEAVY: K4 / SVK prologue (720 B read per voxel): larger E, ~144 threads and
// ~40 KB per CTA so 4 CTAs per SM overlap their load and FFT phases.
template <int M, int E_, int G_, int MINB_ = 4>
struct ZS {
  static constexpr int MINB = MINB_;  // CTAs per SM the register budget targets
  static constexpr int E = E_;
  static constexpr int T = M / E;
  static constexpr int G = G_;                     // z-lines per CTA
  static constexpr int LSL = 9 * G;                // smem lines (9 components x G)
  static constexpr int LSP = LSL | 1;              // odd pitch: conflict-free strided access
  static constexpr int THREADS = LSL * T;
  static constexpr size_t SMEM = size_t(M) * LSP * 16;
};
template <int M, bool HEAVY = false>
struct ZShapeSel {
  // (a line's T = M / E lanes must fit one warp: E = 16 from M = 512 up)
  static constexpr int E = HEAVY ? e_line(M) : (M / reg::e_z(M) > 32 ? 16 : reg::e_z(M));
  static constexpr int T = M / E;
  static constexpr int TT = HEAVY ? 16 : 32;
  using type = ZS<M, E, (T >= TT ? 1 : TT / T)>;
};
template <int M, bool HEAVY = false>
using ZShape = typename ZShapeSel<M, HEAVY>::type;

// Register budget (CTAs/SM) of pass 1 with a staged prologue: 4 for the
// materialised K4 (96 registers, more loads in flight: 256^3 pass 1 2.36 ->
// 1.96 ms), 3 for the compact J2 and SVK prologues.  (Persistent CTAs that
// prefetch the next line group into L2 measured slower at every budget.)
// (Capped so that no budget falls below 96 registers: the 288-thread shape of
// 1024-point lines keeps 2.)
#ifndef FM_ZF_J2C_MINB
#define FM_ZF_J2C_MINB 3
#endif
#ifndef FM_ZF_SVK_MINB
#define FM_ZF_SVK_MINB 3  // (4: 96 registers, measured with FM_ZPIPE=0 at 256^3: see profiles/r2_svk_pass1_dbg.md)
#endif
template <int PRO, int M>
constexpr int zf_minb() {
  return std::min(PRO == PRO_K4 ? 4 : (PRO == PRO_COPY ? 1 : (PRO == PRO_J2C ? FM_ZF_J2C_MINB : FM_ZF_SVK_MINB)),
                  std::max(1, 65536 / (ZShape<M, PRO != PRO_COPY>::THREADS * 96)));
}
template <int M, int PRO, bool DIR, bool PAP = false>
__global__ void __launch_bounds__(ZShape<M, PRO != PRO_COPY>::THREADS, zf_minb<PRO, M>()) k_zf_fast(Geo g, const double2* __restrict__ twM,
                                                                const double2* __restrict__ twN,
                                                                ProArgs pa, double2* __restrict__ spec) {
  using S = ZShape<M, PRO != PRO_COPY>;
  constexpr int N = 2 * M, G = S::G, T = S::T, E = S::E;
  // line l = c G + gi owns the swizzled region sm + l M (reg::fft_swz)
  constexpr int SW = reg::ilog2(E);
  static_assert(32 % T == 0, "a line must not straddle a warp");
  extern __shared__ double2 sm[];
  const int nxy = g.Nx * g.Ny;
  const int L0 = blockIdx.x * G;
  const int Gb = min(G, nxy - L0);
  // phase 1: prologue, one thread per voxel; z -> packed complex m = z/2
  // voxel pairs (z, z+1) per thread: both voxels' loads in flight together,
  // one 16-byte shared store per component (the packed complex z_m)
  // light prologues (copy, SVK action): voxel pairs (z, z+1) per thread, both
  // voxels' loads in flight together and one 16-byte shared store per
  // component; heavy ones (K4, compact J2) one voxel per thread (registers)
  constexpr bool PAIRS = (PRO == PRO_COPY || PRO == PRO_SVK);
  double pap = 0.0;  // fused CG: <p, dP> over this CTA's voxels
  if constexpr (PAIRS) {
    constexpr int N2 = N / 2;
    for (int w = threadIdx.x; w < Gb * N2; w += blockDim.x) {
      const int gi = w / N2, m = w - gi * N2;
      const int64_t node = g.roff + int64_t(L0 + gi) * N + 2 * m;
      double v0[9], v1[9];
      prologue_voxel<3, PRO, DIR, PAP>(pa, g.n, node, v0, &pap);
      prologue_voxel<3, PRO, DIR, PAP>(pa, g.n, node + 1, v1, &pap);
#pragma unroll
      for (int c = 0; c < 9; ++c) sm[(c * G + gi) * M + reg::xaddr<SW>(m, 0)] = make_double2(v0[c], v1[c]);
    }
  } else {
    double* smd = reinterpret_cast<double*>(sm);
    for (int w = threadIdx.x; w < Gb * N; w += blockDim.x) {
      const int gi = w / N, z = w - gi * N;
      const int64_t node = g.roff + int64_t(L0 + gi) * N + z;
      double v[9];
      prologue_voxel<3, PRO, DIR, PAP>(pa, g.n, node, v, &pap);
#pragma unroll
      for (int c = 0; c < 9; ++c) smd[((c * G + gi) * M + reg::xaddr<SW>(z >> 1, 0)) * 2 + (z & 1)] = v[c];
    }
  }
  __syncthreads();
  // phase 2: each line transformed by its T lanes (swizzled exchange, warp
  // syncs), r2c untangling X[k] = E[k] + W_N^k O[k] with the partner M - k by
  // shuffle, k < M stored from registers (kz = M dropped)
  {
    const int l = threadIdx.x / T, t = threadIdx.x % T;
    const int c = l / G, gi = l - c * G;
    double2* line = sm + l * M;
    double2 v[E];
#pragma unroll
    for (int m = 0; m < E; ++m) v[m] = line[reg::xaddr<SW>(t + T * m, 0)];
    __syncwarp();
    reg::fft_swz<M, E, -1>(v, line, t, twM);
    double2* dst = spec + (int64_t(c) * nxy + L0 + gi) * M;
#pragma unroll
    for (int m = 0; m < E; ++m) {
      const int k = t + T * m;
      const double2 a = v[m];
      const double2 b = cconj(mirror_take<T>(mirror_give<E>(v, t, m), t));
      const double2 Ev = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y + b.y));
      const double2 D = csub(a, b);
      const double2 O = make_double2(0.5 * D.y, -0.5 * D.x);
      if (gi < Gb) dst[k] = cadd(Ev, cmul(O, __ldg(&twN[k])));
    }
  }
  if constexpr (PAP) {
    pap = block_sum_any(pap);
    if (threadIdx.x == 0) pa.pap_partial[blockIdx.x] = pap;
  }
}

// Pipelined z-forward pass for the light prologues (projection input copy,
// matrix-free SVK action, optionally fused with the CG direction update):
// a persistent CTA walks z-lines; one thread streams the next line's inputs
// (contiguous N-voxel chunks of every input component: 9 / 20 / 29 of them)
// into a shared staging area with TMA bulk copies while the CTA transforms
// the current line, so HBM reads stay in flight through the FFT phases.
#ifndef FM_PIPE_COPY_MINB
#define FM_PIPE_COPY_MINB 5
#endif
constexpr int kPipeCopyMinB = FM_PIPE_COPY_MINB;
#ifndef FM_PIPE_LAB_MINB
#define FM_PIPE_LAB_MINB 3
#endif
// SVK with phase labels: 4 CTAs/SM would fit the shared memory, but the
// 96-register budget spills (256^3 pass 1: 0.83 ms at 4, 0.69 ms at 3 CTAs/SM)
constexpr int kPipeLabMinB = FM_PIPE_LAB_MINB;

// FM_ZP_DBG (timing experiments: parts of the pipelined pass switched off) only
// exists in builds with -DFM_ZP_DEBUG: the run-time tests cost the SVK pass 7 %.
#ifdef FM_ZP_DEBUG
#define ZP_DBG(pa, bit) ((pa).dbg & (bit))
#else
#define ZP_DBG(pa, bit) 0
#endif

// FM_ZPIPE_EF: elements per lane of the pipelined pass's transforms at M = 128
// (8: 16 lanes per component line, all 144 threads transform, 128 = 8 x 8 x 2
// with two exchanges; 16: 8 lanes per line, 128 = 16 x 8 with one exchange, the
// 72 lanes of lines 0..8 in three warps).
#ifndef FM_ZPIPE_EF
#define FM_ZPIPE_EF 8
#endif
template <int M>
struct ZPipe {
  static constexpr int EF = (M == 128) ? FM_ZPIPE_EF : reg::e_z(M);  // transform shape
  static constexpr int TF = M / EF;
  static constexpr int E = reg::e_z(M), T = M / E;
  static constexpr int LSP = 9;  // one line per CTA: 9 component lines (line-major, swizzled)
  static constexpr int THREADS = 9 * T;
  static constexpr size_t FFT_SM = size_t(M) * LSP * 16;
};
// fp64 input chunks per line; LAB: the lambda and mu chunks replaced by one
// N-byte phase-label chunk (ProArgs::lab)
template <int PRO, bool DIR, bool XUPD = false, bool LAB = false>
constexpr int pipe_chunks() {
  return (PRO == PRO_COPY ? 9 : (DIR ? (XUPD ? 38 : 29) : 20)) - (LAB ? 2 : 0);
}
// LB2: two line buffers, so the next line's prologue may start while slow
// warps still transform the current one (one block barrier per line)
template <int M, int PRO, bool DIR, bool XUPD = false, bool LAB = false, bool LB2 = false>
constexpr size_t pipe_smem() {
  return (LB2 ? 2 : 1) * ZPipe<M>::FFT_SM + size_t(pipe_chunks<PRO, DIR, XUPD, LAB>()) * 2 * M * 8 +
         (LAB ? size_t(2 * M) : 0);
}

template <int M, int PRO, bool DIR, int MINB, bool PAP = false, bool XUPD = false, bool LAB = false,
          bool LB2 = false>
__global__ void __launch_bounds__(ZPipe<M>::THREADS, MINB) k_zf_pipe(Geo g, const double2* __restrict__ twM,
                                                               const double2* __restrict__ twN, ProArgs pa,
                                                               double2* __restrict__ spec) {
  using S = ZPipe<M>;
  constexpr int N = 2 * M, T = S::T, E = S::E, NCH = pipe_chunks<PRO, DIR, XUPD, LAB>();
  static_assert(!LAB || PRO == PRO_SVK, "phase labels replace the SVK lambda / mu chunks");
  constexpr int EF = S::EF, TF = S::TF;
  constexpr int SW = reg::ilog2(EF);  // line-major swizzled line buffer (reg::fft_swz)
  static_assert(32 % T == 0 && 32 % TF == 0, "a component line must not straddle a warp");
  static_assert(!XUPD || (DIR && PRO == PRO_SVK), "x update rides on the SVK direction prologue");
  extern __shared__ __align__(16) double2 sm[];
  double* stage = reinterpret_cast<double*>(sm + (LB2 ? 2 : 1) * M * S::LSP);  // NCH chunks of N doubles
  __shared__ uint64_t bar;
  const int nxy = g.Nx * g.Ny;
  const int64_t n = g.n;
  auto issue = [&](int L) {
    if (ZP_DBG(pa, 8)) return;
    const int64_t node0 = g.roff + int64_t(L) * N;
    bulk::mbar_expect_tx(&bar, NCH * N * 8 + (LAB ? N : 0));
    int q = 0;
    auto cp = [&](const double* base) { bulk::g2s(stage + (q++) * N, base + node0, N * 8, &bar); };
    if constexpr (PRO == PRO_COPY) {
      for (int c = 0; c < 9; ++c) cp(pa.A + c * n);
    } else {
      if constexpr (DIR) {
        for (int c = 0; c < 9; ++c) cp(pa.r + c * n);
        for (int c = 0; c < 9; ++c) cp(pa.p + c * n);
        if constexpr (XUPD)
          for (int c = 0; c < 9; ++c) cp(pa.x + c * n);
      } else {
        for (int c = 0; c < 9; ++c) cp(pa.A + c * n);
      }
      for (int c = 0; c < 9; ++c) cp(pa.F + c * n);
      if constexpr (LAB) {
        bulk::g2s(stage + NCH * N, pa.lab + node0, N, &bar);
      } else {
        cp(pa.lam);
        cp(pa.mu);
      }
    }
  };
  if (threadIdx.x == 0) bulk::mbar_init(&bar, 1);
  __syncthreads();
  double pap = 0.0;  // fused CG: <p, dP> over this CTA's voxels
  int L = blockIdx.x;
  if (threadIdx.x == 0 && L < nxy) issue(L);
  unsigned phase = 0;
  for (; L < nxy; L += gridDim.x) {
    if (!ZP_DBG(pa, 8)) bulk::mbar_wait(&bar, phase);
    double2* const lsm = sm + (LB2 && phase ? M * S::LSP : 0);  // this line's buffer
    phase ^= 1;
    // prologue on voxel pairs (z, z+1) out of the staging area
    for (int m = threadIdx.x; m < N / 2; m += blockDim.x) {
      double v0[9], v1[9];
      if constexpr (PRO == PRO_COPY) {
#pragma unroll
        for (int c = 0; c < 9; ++c) {
          const double2 a = *reinterpret_cast<const double2*>(stage + c * N + 2 * m);
          v0[c] = a.x;
          v1[c] = a.y;
        }
      } else {
        double d0[9], d1[9], f0[9], f1[9];
        if constexpr (DIR) {
          const double beta = *pa.beta;
          double alpha = 0.0;
          if constexpr (XUPD) alpha = *pa.alpha;
#pragma unroll
          for (int c = 0; c < 9; ++c) {
            const double2 r = *reinterpret_cast<const double2*>(stage + c * N + 2 * m);
            const double2 p = *reinterpret_cast<const double2*>(stage + (9 + c) * N + 2 * m);
            d0[c] = __dadd_rn(__dmul_rn(p.x, beta), r.x);
            d1[c] = __dadd_rn(__dmul_rn(p.y, beta), r.y);
            if constexpr (XUPD) {  // x += alpha p_old (solver.cpp:46, k_cg_update rounding)
              double2 xv = *reinterpret_cast<const double2*>(stage + (18 + c) * N + 2 * m);
              xv.x = __dadd_rn(xv.x, __dmul_rn(alpha, p.x));
              xv.y = __dadd_rn(xv.y, __dmul_rn(alpha, p.y));
              *reinterpret_cast<double2*>(pa.x + c * n + g.roff + int64_t(L) * N + 2 * m) = xv;
            }
          }
        } else {
#pragma unroll
          for (int c = 0; c < 9; ++c) {
            const double2 a = *reinterpret_cast<const double2*>(stage + c * N + 2 * m);
            d0[c] = a.x;
            d1[c] = a.y;
          }
        }
        constexpr int FB = DIR ? (XUPD ? 27 : 18) : 9;
#pragma unroll
        for (int c = 0; c < 9; ++c) {
          const double2 a = *reinterpret_cast<const double2*>(stage + (FB + c) * N + 2 * m);
          f0[c] = a.x;
          f1[c] = a.y;
        }
        double2 lm, mu;
        if constexpr (LAB) {
          const uchar2 ph = *reinterpret_cast<const uchar2*>(reinterpret_cast<const uint8_t*>(stage + NCH * N) + 2 * m);
          lm = make_double2(__ldg(pa.ptab + ph.x), __ldg(pa.ptab + ph.y));
          mu = make_double2(__ldg(pa.ptab + 256 + ph.x), __ldg(pa.ptab + 256 + ph.y));
        } else {
          lm = *reinterpret_cast<const double2*>(stage + (FB + 9) * N + 2 * m);
          mu = *reinterpret_cast<const double2*>(stage + (FB + 10) * N + 2 * m);
        }
        if (ZP_DBG(pa, 1)) {
#pragma unroll
          for (int c = 0; c < 9; ++c) v0[c] = d0[c] + f0[c] * lm.x, v1[c] = d1[c] + f1[c] * mu.y;
        } else {
          svk_action<3>(f0, d0, lm.x, mu.x, v0);
          svk_action<3>(f1, d1, lm.y, mu.y, v1);
        }
        if constexpr (PAP) {
#pragma unroll
          for (int c = 0; c < 9; ++c) pap += d0[c] * v0[c];
#pragma unroll
          for (int c = 0; c < 9; ++c) pap += d1[c] * v1[c];
        }
        if constexpr (DIR) {
          const int64_t node = g.roff + int64_t(L) * N + 2 * m;
#pragma unroll
          for (int c = 0; c < 9; ++c)
            *reinterpret_cast<double2*>(pa.p + c * n + node) = make_double2(d0[c], d1[c]);
        }
      }
#pragma unroll
      for (int c = 0; c < 9; ++c) lsm[c * M + reg::xaddr<SW>(m, 0)] = make_double2(v0[c], v1[c]);
    }
    __syncthreads();  // staging consumed, packed line in lsm
    if (threadIdx.x == 0 && L + int(gridDim.x) < nxy) issue(L + gridDim.x);
    // component c's line in the TF lanes of one warp: swizzled exchange with
    // warp syncs, untangling by shuffle, spectrum stored from registers.  With
    // TF < T only the first 9 TF lanes hold lines; the rest of their last warp
    // redoes line 8 (same values to the same addresses) so that the warp-level
    // syncs stay full, and stores nothing.
    constexpr int FT = ((9 * TF + 31) / 32) * 32;  // transform threads: whole warps
    if (int(threadIdx.x) < FT) {
      const int cs = threadIdx.x / TF, c = cs < 9 ? cs : 8, t = threadIdx.x % TF;
      double2* line = lsm + c * M;
      double2 v[EF];
#pragma unroll
      for (int m = 0; m < EF; ++m) v[m] = line[reg::xaddr<SW>(t + TF * m, 0)];
      __syncwarp();
      if (!ZP_DBG(pa, 2)) reg::fft_swz<M, EF, -1>(v, line, t, twM);
      double2* dst = spec + (int64_t(c) * nxy + L) * M;
#pragma unroll
      for (int m = 0; m < EF; ++m) {
        const int k = t + TF * m;
        const double2 a = v[m];
        double2 res = a;
        if (!ZP_DBG(pa, 2)) {
          const double2 b = cconj(mirror_take<TF>(mirror_give<EF>(v, t, m), t));
          const double2 Ev = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y + b.y));
          const double2 D = csub(a, b);
          const double2 O = make_double2(0.5 * D.y, -0.5 * D.x);
          res = cadd(Ev, cmul(O, __ldg(&twN[k])));
        }
        if (!ZP_DBG(pa, 4) && cs < 9) dst[k] = res;
      }
    }
    // one buffer: wait until every warp is done with it; two: the next
    // prologue writes the other one, and the barrier after it orders this
    // buffer's reads before its reuse two lines on
    if constexpr (!LB2) __syncthreads();
  }
  if constexpr (PAP) {
    pap = block_sum_any(pap);
    if (threadIdx.x == 0) pa.pap_partial[blockIdx.x] = pap;
  }
}

template <int M, typename S = ZShape<M>>
__global__ void __launch_bounds__(S::THREADS, 2048 / S::THREADS >= S::MINB ? S::MINB : 1)
    k_zi_fast(Geo g, const double2* __restrict__ twM, const double2* __restrict__ twN,
              const double2* __restrict__ spec, double* __restrict__ out, double scale, EpiArgs epi) {
  constexpr int N = 2 * M, G = S::G, LSP = S::LSP, T = S::T, E = S::E;
  extern __shared__ double2 sm[];
  const int nxy = g.Nx * g.Ny;
  const int L0 = blockIdx.x * G;
  const int Gb = min(G, nxy - L0);
  for (int w = threadIdx.x; w < 9 * Gb * M; w += blockDim.x) {  // all loads in flight at once
    const int c = w / (Gb * M), rem = w - c * (Gb * M);
    const int gi = rem / M, k = rem - gi * M;
    cp_async16(sm + k * LSP + c * G + gi, spec + (int64_t(c) * nxy + L0 + gi) * M + k);
  }
  // fused CG: the residual lines the epilogue updates, staged next to the spectrum
  double2* rs = sm + M * LSP;  // [gi][c][N/2] voxel pairs
  if (epi.r) {
    for (int w = threadIdx.x; w < 9 * Gb * (N / 2); w += blockDim.x) {
      const int gc = w / (N / 2), m = w - gc * (N / 2);
      const int gi = gc / 9, c = gc - gi * 9;
      cp_async16(rs + w, epi.r + c * g.n + g.roff + int64_t(L0 + gi) * N + 2 * m);
    }
  }
  cp_async_wait_all();
  __syncthreads();
  // Z[k] = (X[k] + X*[M-k]) + i W_N^-k (X[k] - X*[M-k]), X[M] = 0 (ZeroCompatible),
  // formed straight into the registers of the thread that transforms Z[k]
  {
    const int l = threadIdx.x % S::LSL, t = threadIdx.x / S::LSL;
    double2 v[E];
#pragma unroll
    for (int m = 0; m < E; ++m) {
      const int k = t + T * m;
      double2 xk = sm[k * LSP + l];
      double2 b = make_double2(0.0, 0.0);
      if (k == 0) xk.y = 0.0;  // Re(ifft): drop the round-off imaginary part of kz = 0
      else b = cconj(sm[(M - k) * LSP + l]);
      const double2 tt = cmulc(csub(xk, b), __ldg(&twN[k]));
      v[m] = make_double2(xk.x + b.x - tt.y, xk.y + b.y + tt.x);
    }
    __syncthreads();
    reg::fft<M, E, +1>(v, sm + l, LSP, t, twM);
#pragma unroll
    for (int m = 0; m < E; ++m) sm[(t + T * m) * LSP + l] = v[m];
  }
  __syncthreads();
  // epilogue on z pairs: one 16-byte shared read and one 16-byte store per
  // component (node is even: N, the slab offset and the slab stride are even)
  double dot = 0.0;
  constexpr int N2 = N / 2;
  if (epi.r) {
    // fused CG update, solver.cpp:46-48 with the rounding of k_cg_update:
    // Ap stays on chip; r -= alpha Ap, x += alpha p, partial <r, r>
    if (epi.scal[S_FLAG] == 0.0) {
      const double alpha = epi.scal[S_ALPHA];
      for (int w = threadIdx.x; w < Gb * N2; w += blockDim.x) {
        const int gi = w / N2, m = w - gi * N2;
        const int64_t node = g.roff + int64_t(L0 + gi) * N + 2 * m;
#pragma unroll
        for (int c = 0; c < 9; ++c) {
          const double2 zz = sm[m * LSP + c * G + gi];
          const double2 av = make_double2(zz.x * scale, zz.y * scale);
          double2 rv = rs[(gi * 9 + c) * N2 + m];
          if (epi.x) {  // else the next pass 1 applies x += alpha p (ProArgs::x)
            double2* xp = reinterpret_cast<double2*>(epi.x + c * g.n + node);
            const double2 pv = __ldg(reinterpret_cast<const double2*>(epi.p + c * g.n + node));
            double2 xv = *xp;
            xv.x = __dadd_rn(xv.x, __dmul_rn(alpha, pv.x));
            xv.y = __dadd_rn(xv.y, __dmul_rn(alpha, pv.y));
            *xp = xv;
          }
          rv.x = __dadd_rn(rv.x, __dmul_rn(-alpha, av.x));
          rv.y = __dadd_rn(rv.y, __dmul_rn(-alpha, av.y));
          *reinterpret_cast<double2*>(epi.r + c * g.n + node) = rv;
          dot += rv.x * rv.x;
          dot += rv.y * rv.y;
        }
      }
    }
    dot = block_sum_any(dot);
    if (threadIdx.x == 0) epi.partial[blockIdx.x] = dot;
    return;
  }
  for (int w = threadIdx.x; w < Gb * N2; w += blockDim.x) {
    const int gi = w / N2, m = w - gi * N2;
    const int64_t node = g.roff + int64_t(L0 + gi) * N + 2 * m;
#pragma unroll
    for (int c = 0; c < 9; ++c) {
      const double2 zz = sm[m * LSP + c * G + gi];
      const double2 val = make_double2(zz.x * scale, zz.y * scale);
      *reinterpret_cast<double2*>(out + c * g.n + node) = val;
      if (epi.partial) {
        const double2 pp = __ldg(reinterpret_cast<const double2*>(epi.pdot + c * g.n + node));
        dot += pp.x * val.x;
        dot += pp.y * val.y;
      }
    }
  }
  if (epi.partial) {  // fused <p, Ap> partial (solver.cpp:37)
    dot = block_sum_any(dot);
    if (threadIdx.x == 0) epi.partial[blockIdx.x] = dot;
  }
}

// ----------------------------------------------- z passes, lines in registers
// One component z-line per T = M/E lanes (T | 32), LPC lines per CTA.  The
// line goes from HBM straight into registers and back (16-byte accesses, T
// lanes per contiguous run), the r2c / c2r untangling pairs k with M - k by
// warp shuffle (the partner element sits in lane (T - t) mod T), and the FFT
// exchanges through the line's own swizzled shared-memory region with
// warp-level syncs only -- two shared-memory accesses per element and
// exchange instead of the staged passes' six to eight.  Components are
// independent here, so this is the shape of the z-inverse (every operator)
// and of the z-forward of G (no per-voxel prologue coupling the components).

// PF: the epilogue reads operands (fused CG r / x / p, or the <p, Ap> pdot):
// prefetch them into L2 at entry.  The plain store variant carries no such code.
template <int M, int E, int LPC, int MINB, bool PF = false>
__global__ void __launch_bounds__(LPC*(M / E), MINB)
    k_zi_reg(Geo g, const double2* __restrict__ twM, const double2* __restrict__ twN,
             const double2* __restrict__ spec, double* __restrict__ out, double scale, EpiArgs epi) {
  constexpr int T = M / E, N = 2 * M;
  static_assert(32 % T == 0, "a line must not straddle a warp");
  extern __shared__ double2 sm[];
  const int t = threadIdx.x % T, w = threadIdx.x / T;
  const int nxy = g.Nx * g.Ny;
  const int64_t nl = int64_t(9) * nxy;
  int64_t gl = int64_t(blockIdx.x) * LPC + w;
  const bool live = gl < nl;
  if (!live) gl = nl - 1;  // tail lanes transform a valid line (warp-synchronous) and store nothing
  const int c = int(gl / nxy);
  const int L = int(gl - int64_t(c) * nxy);
  const double2* X = spec + gl * M;
  const int64_t base = int64_t(c) * g.n + g.roff + int64_t(L) * N;
  if (PF && t == 0 && live) {  // epilogue operands stream into L2 while the line is transformed
    if (epi.r) bulk::prefetch_l2(epi.r + base, N * 8);
    if (epi.x) {
      bulk::prefetch_l2(epi.x + base, N * 8);
      bulk::prefetch_l2(epi.p + base, N * 8);
    }
    if (epi.pdot) bulk::prefetch_l2(epi.pdot + base, N * 8);
  }
  double2 xk[E];
#pragma unroll
  for (int m = 0; m < E; ++m) xk[m] = X[t + T * m];
  // Z[k] = (X[k] + X*[M-k]) + i W_N^-k (X[k] - X*[M-k]), X[M] = 0 (ZeroCompatible)
  double2 v[E];
#pragma unroll
  for (int m = 0; m < E; ++m) {
    const double2 xm = mirror_take<T>(mirror_give<E>(xk, t, m), t);
    const int k = t + T * m;
    double2 a = xk[m];
    double2 b = make_double2(0.0, 0.0);
    if (k == 0) a.y = 0.0;  // Re(ifft): drop the round-off imaginary part of kz = 0
    else b = cconj(xm);
    const double2 tt = cmulc(csub(a, b), __ldg(&twN[k]));
    v[m] = make_double2(a.x + b.x - tt.y, a.y + b.y + tt.x);
  }
  reg::fft_swz<M, E, +1>(v, sm + w * M, t, twM);
  // v[m] = z[n], n = t + T m: the real voxel pair (2n, 2n + 1)
  double dot = 0.0;
  if (epi.r) {
    // fused CG update, solver.cpp:46-48 with the rounding of k_cg_update:
    // Ap stays on chip; r -= alpha Ap, x += alpha p, partial <r, r>
    if (live && epi.scal[S_FLAG] == 0.0) {
      const double alpha = epi.scal[S_ALPHA];
      double2* rp = reinterpret_cast<double2*>(epi.r + base) + t;
      // r is read and written through one pointer: load a batch of KB lines'
      // worth before any store so the loads are not serialised behind them
      constexpr int KB = 8;
#pragma unroll
      for (int m0 = 0; m0 < E; m0 += KB) {
        double2 rv[KB];
#pragma unroll
        for (int q = 0; q < KB; ++q) rv[q] = __ldcg(rp + T * (m0 + q));
#pragma unroll
        for (int q = 0; q < KB; ++q) {
          const int m = m0 + q;
          const double2 av = make_double2(v[m].x * scale, v[m].y * scale);
          rv[q].x = __dadd_rn(rv[q].x, __dmul_rn(-alpha, av.x));
          rv[q].y = __dadd_rn(rv[q].y, __dmul_rn(-alpha, av.y));
          rp[T * m] = rv[q];
          dot += rv[q].x * rv[q].x;
          dot += rv[q].y * rv[q].y;
        }
      }
      if (epi.x) {  // K4 / compact J2: x += alpha p here (SVK: the next pass 1 applies it, ProArgs::x)
        double2* xp = reinterpret_cast<double2*>(epi.x + base) + t;
        const double2* pp = reinterpret_cast<const double2*>(epi.p + base) + t;
#pragma unroll
        for (int m0 = 0; m0 < E; m0 += KB) {
          double2 xv[KB];
#pragma unroll
          for (int q = 0; q < KB; ++q) xv[q] = __ldcg(xp + T * (m0 + q));
#pragma unroll
          for (int q = 0; q < KB; ++q) {
            const double2 pv = __ldg(pp + T * (m0 + q));
            xv[q].x = __dadd_rn(xv[q].x, __dmul_rn(alpha, pv.x));
            xv[q].y = __dadd_rn(xv[q].y, __dmul_rn(alpha, pv.y));
            xp[T * (m0 + q)] = xv[q];
          }
        }
      }
    }
  } else if (live) {
#pragma unroll
    for (int m = 0; m < E; ++m) {
      const int64_t o = base + 2 * (t + T * m);
      const double2 val = make_double2(v[m].x * scale, v[m].y * scale);
      *reinterpret_cast<double2*>(out + o) = val;
      if (epi.partial) {
        const double2 pp = __ldg(reinterpret_cast<const double2*>(epi.pdot + o));
        dot += pp.x * val.x;
        dot += pp.y * val.y;
      }
    }
  }
  if (epi.partial) {  // fused <p, Ap> or <r, r> partial (solver.cpp:37, 48)
    dot = block_sum_any(dot);
    if (threadIdx.x == 0) epi.partial[blockIdx.x] = dot;
  }
}

// z-forward of G (PRO_COPY): real pairs straight into registers, M-point FFT,
// r2c untangling with the mirror partner by shuffle, spectrum stored from
// registers.  Same arithmetic as the staged z-forward passes.
template <int M, int E, int LPC, int MINB>
__global__ void __launch_bounds__(LPC*(M / E), MINB)
    k_zf_reg(Geo g, const double2* __restrict__ twM, const double2* __restrict__ twN, const double* __restrict__ A,
             double2* __restrict__ spec) {
  constexpr int T = M / E, N = 2 * M;
  static_assert(32 % T == 0, "a line must not straddle a warp");
  extern __shared__ double2 sm[];
  const int t = threadIdx.x % T, w = threadIdx.x / T;
  const int nxy = g.Nx * g.Ny;
  const int64_t nl = int64_t(9) * nxy;
  int64_t gl = int64_t(blockIdx.x) * LPC + w;
  const bool live = gl < nl;
  if (!live) gl = nl - 1;
  const int c = int(gl / nxy);
  const int L = int(gl - int64_t(c) * nxy);
  const double* src = A + int64_t(c) * g.n + g.roff + int64_t(L) * N;
  double2 v[E];
#pragma unroll
  for (int m = 0; m < E; ++m) v[m] = __ldg(reinterpret_cast<const double2*>(src + 2 * (t + T * m)));
  reg::fft_swz<M, E, -1>(v, sm + w * M, t, twM);
  double2* dst = spec + gl * M;
#pragma unroll
  for (int m = 0; m < E; ++m) {
    const int k = t + T * m;
    const double2 a = v[m];
    const double2 b = cconj(mirror_take<T>(mirror_give<E>(v, t, m), t));
    const double2 Ev = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y + b.y));
    const double2 D = csub(a, b);
    const double2 O = make_double2(0.5 * D.y, -0.5 * D.x);
    if (live) dst[k] = cadd(Ev, cmul(O, __ldg(&twN[k])));
  }
}

// ------------------------------------------------------------------- host
namespace {

template <typename K>
void allow(K kernel, size_t bytes) {  // per device, memoised (set_smem_limit)
  if (bytes > 48 * 1024) set_smem_limit(reinterpret_cast<const void*>(kernel), int(bytes));
}

int tw_of(int N) { return N >= 1024 ? 4 : 8; }
constexpr int tw_x(int N) { return N >= 1024 ? 2 : (N >= 512 ? 4 : 8); }

int launched(fm_ctx* ctx, const char* what) {
  ctx->cnt.launches++;
  ctx->cnt.note(what);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? FM_OK : check_cuda(ctx, e, what);
}

template <int N, int TW>
bool y_launch_tw(fm_ctx* ctx, const Geo& g, int sign, const double2* in, double2* out, int* st) {
  constexpr int T = N / e_line(N);
  const size_t smem = size_t(N) * TW * 16;
  const dim3 grid(ctx->nzh / TW, g.Nx, ctx->ncomp);
  if (sign < 0 && g.P > 1) {  // forward pass with the fused slab transpose
    allow(k_y_fast<N, TW, -1, true>, smem);
    k_y_fast<N, TW, -1, true><<<grid, TW * T, smem, ctx->stream>>>(g, ctx->py.tw, in, out);
  } else if (sign < 0) {
    allow(k_y_fast<N, TW, -1>, smem);
    k_y_fast<N, TW, -1><<<grid, TW * T, smem, ctx->stream>>>(g, ctx->py.tw, in, out);
  } else {
    allow(k_y_fast<N, TW, +1>, smem);
    k_y_fast<N, TW, +1><<<grid, TW * T, smem, ctx->stream>>>(g, ctx->py.tw, in, out);
  }
  *st = launched(ctx, "k_y_fast");
  return true;
}
template <int N>
bool y_launch(fm_ctx* ctx, const Geo& g, int sign, const double2* in, double2* out, int* st) {
  // 8 kz columns = one 128-byte segment per row (4-column tiles measured slower
  // at 256^3 and 512^3).  At 1024 points 8 columns are a 128 KB exchange buffer
  // and one 512-thread CTA per SM; FM_Y1024_TW=4 selects 4 columns (two CTAs of
  // 256 threads, 64-byte segments) for the A/B.
  if constexpr (N >= 1024) {
    static const int tw = [] {
      const char* e = getenv("FM_Y1024_TW");
      return e ? atoi(e) : 4;
    }();
    // the cluster form (k_y_warp, projection_xw.cu), in place on one device: 31.3 / 32.0 ms against 34.9 / 35.0 ms
    // at 1024^3; FM_YW1024=0 restores k_y_fast (which the routed P > 1 passes use)
    static const bool yw = [] {
      const char* e = getenv("FM_YW1024");
      return !e || atoi(e) != 0;
    }();
    if (yw && N == 1024 && g.P == 1 && in == out) {
      if (yw_launch(ctx, g, sign, out)) {
        *st = launched(ctx, "k_y_warp");
        return true;
      }
      cudaGetLastError();
    }
    if (tw == 8 && ctx->nzh % 8 == 0) return y_launch_tw<N, 8>(ctx, g, sign, in, out, st);
    return y_launch_tw<N, 4>(ctx, g, sign, in, out, st);
  } else {
    return y_launch_tw<N, 8>(ctx, g, sign, in, out, st);
  }
}

// RT: the slab-transpose-fused instantiation (P > 1); P = 1 runs the plain one
template <int N, int TW, int E, bool RT>
void x3_rt(fm_ctx* ctx, const Geo& g, double2* spec) {
  constexpr int T = N / E;
  const size_t smem = size_t(3) * N * TW * 16;
  allow(k_x_fast3<N, TW, E, RT>, smem);
  const dim3 grid(ctx->nzh / TW, g.Ny, 3);
  k_x_fast3<N, TW, E, RT><<<grid, TW * T, smem, ctx->stream>>>(g, ctx->px.tw, spec);
}
template <int N, int TW, int E>
void x3_go(fm_ctx* ctx, const Geo& g, double2* spec) {
  g.P > 1 ? x3_rt<N, TW, E, true>(ctx, g, spec) : x3_rt<N, TW, E, false>(ctx, g, spec);
}

template <int N, int TW, int E, bool RT>
void x4_rt(fm_ctx* ctx, const Geo& g, double2* spec) {
  constexpr int T = N / E;
  const size_t smem = size_t(2) * N * TW * 16;
  allow(k_x_fast4<N, TW, E, RT>, smem);
#ifdef FM_X4_DEBUG
  {
    const char* e = getenv("FM_X4_DBG");
    const int bits = e ? atoi(e) : 0;
    cudaMemcpyToSymbolAsync(x4_dbg_bits, &bits, sizeof(bits), 0, cudaMemcpyHostToDevice, ctx->stream);
  }
#endif
  const dim3 grid(ctx->nzh / TW, g.Ny, 3);
  k_x_fast4<N, TW, E, RT><<<grid, TW * T, smem, ctx->stream>>>(g, ctx->px.tw, spec);
}
template <int N, int TW, int E>
void x4_go(fm_ctx* ctx, const Geo& g, double2* spec) {
  g.P > 1 ? x4_rt<N, TW, E, true>(ctx, g, spec) : x4_rt<N, TW, E, false>(ctx, g, spec);
}

template <int N, int TW, bool RT>
void xd_rt(fm_ctx* ctx, const Geo& g, double2* spec) {
  const size_t smem = size_t(N) * TW * 16;
  allow(k_x_direct<N, TW, RT>, smem);
  const dim3 grid(ctx->nzh / TW, g.Ny, 3);
  k_x_direct<N, TW, RT><<<grid, TW * 32, smem, ctx->stream>>>(g, ctx->px.tw, spec);
}

// Tensor map of a spectral buffer viewed as [9 N][Ny][2 nzh] doubles with a
// (2 TW, 1, 256) box -- the x pass's component-tile rows.  Encoded on the
// host (cuTensorMapEncodeTiled through the runtime's driver entry point, no
// libcuda link) and cached: the map is a pure function of its arguments.
// swz128: rows laid out in shared memory with the 128-byte swizzle (16-byte
// chunk c of row r at chunk c ^ (r & 7); needs 2 TW doubles = 128 bytes).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
}  // namespace
bool x_tensor_map(const void* base, int rows, int Ny, int nzh, int TW, bool swz128, int box_rows, void* out_map,
                  bool split2) {
  CUtensorMap* out = static_cast<CUtensorMap*>(out_map);
  struct Entry {
    const void* base;
    int rows, Ny, nzh, TW;
    bool swz;
    int box_rows;
    bool split2;
    CUtensorMap map;
  };
  static std::mutex mx;
  static std::vector<Entry> cache;
  static EncodeTiledFn enc = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    cudaGetLastError();
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  if (!enc) return false;
  std::lock_guard<std::mutex> lk(mx);
  for (const Entry& e : cache)
    if (e.base == base && e.rows == rows && e.Ny == Ny && e.nzh == nzh && e.TW == TW && e.swz == swz128 && e.box_rows == box_rows && e.split2 == split2) {
      *out = e.map;
      return true;
    }
  Entry e{base, rows, Ny, nzh, TW, swz128, box_rows, split2, {}};
  const cuuint64_t dims[3] = {cuuint64_t(2 * nzh), cuuint64_t(Ny), cuuint64_t(rows)};
  const cuuint64_t strides[2] = {cuuint64_t(nzh) * 16, cuuint64_t(Ny) * nzh * 16};
  const cuuint32_t box[3] = {cuuint32_t(2 * TW), 1, cuuint32_t(box_rows)};
  const cuuint32_t estr[3] = {1, 1, 1};
  // L2 promotion (A/B: FM_TMA_PROMO 0 none, 1 64 B, 2 128 B, 3 256 B); a
  // promotion wider than the 16 TW-byte row segment would fetch neighbours
  static const int promo = [] {
    const char* p = getenv("FM_TMA_PROMO");
    return p ? atoi(p) : -1;
  }();
  const int pm = promo >= 0 ? promo : (TW >= 8 ? 2 : 1);
  const CUtensorMapL2promotion pr = pm == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                    : pm == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                    : pm == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                              : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  CUresult rc;
  if (!split2) {
    rc = enc(&e.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, swz128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, pr,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    // rows split by parity: [rows / 2][2][Ny][2 nzh] -- even and odd x-rows of every component are separate boxes
    const cuuint64_t d4[4] = {cuuint64_t(2 * nzh), cuuint64_t(Ny), 2, cuuint64_t(rows / 2)};
    const cuuint64_t s4[3] = {cuuint64_t(nzh) * 16, cuuint64_t(Ny) * nzh * 16, cuuint64_t(2) * Ny * nzh * 16};
    const cuuint32_t b4[4] = {cuuint32_t(2 * TW), 1, 1, cuuint32_t(box_rows)};
    const cuuint32_t e4[4] = {1, 1, 1, 1};
    rc = enc(&e.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<void*>(base), d4, s4, b4, e4,
             CU_TENSOR_MAP_INTERLEAVE_NONE, swz128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, pr,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (rc != CUDA_SUCCESS) return false;
  if (cache.size() > 256) cache.clear();
  cache.push_back(e);
  *out = e.map;
  return true;
}
// Uncached encode of a tiled fp64 tensor map of any rank (dims innermost first,
// strides in bytes for dims 1.., box in elements), 128-byte swizzle optional.
bool tensor_map_encode(const void* base, int rank, const uint64_t* dims, const uint64_t* strides, const uint32_t* box,
                       bool swz128, void* out_map) {
  static EncodeTiledFn enc = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    cudaGetLastError();
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  if (!enc || rank < 1 || rank > 5) return false;
  cuuint64_t d[5], st[4];
  cuuint32_t b[5], e[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    e[i] = 1;
    if (i > 0) st[i - 1] = strides[i - 1];
  }
  return enc(static_cast<CUtensorMap*>(out_map), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, cuuint32_t(rank),
             const_cast<void*>(base), d, st, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
             swz128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
namespace {

template <int N, int TW, int E, bool PAIR, bool RT>
bool xs_rt(fm_ctx* ctx, const Geo& g, double2* spec) {
  CUtensorMap map;
  if (!x_tensor_map(spec, 9 * N, g.Ny, g.nzh, TW, false, 256, &map)) return false;
  const size_t smem = size_t(3) * N * TW * 16;
  constexpr int THREADS = TW * (N / E);
  allow(k_x_stream<N, TW, E, PAIR, RT>, smem);
  static const int per_sm = [] {  // (occupancy: the same on every B200 of the node)
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_x_stream<N, TW, E, PAIR, RT>, THREADS, smem);
    cudaGetLastError();
    return b > 0 ? b : 1;
  }();
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int tiles = (ctx->nzh / TW) * g.Ny * 3;
  const int grid = std::min(tiles, std::max(sms, 1) * per_sm);
  static const int dbg = [] {
    const char* e = getenv("FM_X_DBG");
    return e ? atoi(e) : 0;
  }();
  k_x_stream<N, TW, E, PAIR, RT><<<grid, THREADS, smem, ctx->stream>>>(g, ctx->px.tw, spec, tiles, map, dbg);
  return true;
}
template <int N, int TW, int E, bool PAIR>
bool xs_go(fm_ctx* ctx, const Geo& g, double2* spec) {
  return g.P > 1 ? xs_rt<N, TW, E, PAIR, true>(ctx, g, spec) : xs_rt<N, TW, E, PAIR, false>(ctx, g, spec);
}

// FM_XDIRECT=0: the 512-point x pass falls back to the staged k_x_fast4;
// FM_XDIRECT=1: k_x_direct (register loads); 2: k_x_stream, TW 8; 3: TW 4
// (two CTAs per SM); 4: lane-pair k_x_stream, TW 8 (the routed P > 1 pass);
// 5: E = 8; 6: lane pair, TW 4; 7 (default): k_x_warp (projection_xw.cu).
// Measured at 512^3 (profiles/r2_x512_ab.md): 5.81 / 5.31 / 5.11 / 7.27 / 4.91 /
// 4.98 / 7.47 / 3.75 ms.
int xdirect_mode() {
  static int v = [] {
    const char* e = getenv("FM_XDIRECT");
    return e ? atoi(e) : 7;
  }();
  return v;
}

template <int N>
bool x_launch(fm_ctx* ctx, const Geo& g, double2* spec, int* st) {
  constexpr int TW = tw_x(N);
  constexpr int T = N / e_x(N);
  const size_t smem = size_t(N) * TW * 16;
  // Measured (scripts/xvar.py, pass_times.py): ZeroCompatible -> scalar-accumulating
  // k_x_fast4 (8-column tiles up to 256, 4-column tiles at 512 and 1024); other modes
  // -> whole-tile prefetch k_x_fast3; registers-only k_x_fast as the fallback.
  // (512: 8-column tiles, 1 CTA/SM, measured no faster; 1024: 72.7 ms at 1024^3
  // against 120 ms for the registers-only pass)
  const bool zc = ctx->mode == FM_NYQUIST_ZERO_COMPATIBLE;
  constexpr int X4TW = N >= 512 ? 4 : 8;
  bool done = false;
  const char* name = "k_x_fast";
  if constexpr (N == 512) {  // 5.3 vs 6.0 ms at 512^3 (k_x_fast4, 4-column tiles)
    const bool fits = 3 * int64_t(N) * g.Ny * ctx->nzh < (int64_t(1) << 31);
    // (two thread groups transforming A_0 and B side by side without spills,
    // k_x_split, measured 6.0 ms at 4 columns / 2 CTAs per SM, 6.8 ms at 8 / 1)
    const int xm = xdirect_mode();
    static const int xdbg = [] {
      const char* e = getenv("FM_X_DBG");
      return e ? atoi(e) : 0;
    }();
    if (zc && xm == 7 && xw_launch(ctx, g, spec, xdbg)) {
      done = true;
      name = "k_x_warp";
    } else if (zc && ctx->nzh % 8 == 0 && xm >= 2 &&
        (xm == 3   ? xs_go<N, 4, 16, false>(ctx, g, spec)
         : (xm == 4 || xm == 7) ? xs_go<N, 8, 16, true>(ctx, g, spec)
         : xm == 5 ? xs_go<N, 8, 8, false>(ctx, g, spec)
         : xm == 6 ? xs_go<N, 4, 16, true>(ctx, g, spec)
                   : xs_go<N, 8, 16, false>(ctx, g, spec))) {
      done = true;
      name = "k_x_stream";
    } else if (zc && ctx->nzh % 8 == 0 && xm == 1 && fits) {
      // (streaming evict-first loads / stores, to keep the spills in L2: 5.8 vs 5.2 ms)
      g.P > 1 ? xd_rt<N, 8, true>(ctx, g, spec) : xd_rt<N, 8, false>(ctx, g, spec);
      done = true;
      name = "k_x_direct";
    }
  }
  if constexpr (N == 1024) {
    // the cluster form of k_x_warp (projection_xw.cu): 40.4 vs 58.6 ms at 1024^3; FM_XW1024=0: k_x_fast4 on
    // 4-column tiles (also the routed P > 1 pass)
    static const bool xw1024 = [] {
      const char* e = getenv("FM_XW1024");
      return !e || atoi(e) != 0;
    }();
    if (zc && xw1024) {  // (P > 1: routed TMA stores, where xw_launch allows them)
      static const int xdbg1024 = [] {
        const char* e = getenv("FM_X_DBG");
        return e ? atoi(e) : 0;
      }();
      if (xw_launch(ctx, g, spec, xdbg1024)) {
        done = true;
        name = "k_x_warp";
      } else {
        cudaGetLastError();
      }
    }
  }
  if (done) {
  } else if (N == 128 && zc && ctx->nzh % 16 == 0) {
    // 128-point lines: 16-column tiles (256-byte row segments, 128 threads and three CTAs per SM) instead
    // of 8 (64 threads at 255 registers): 0.0761 -> 0.0722 ms at 128^3, 0.256 -> 0.231 ms on 128 x 256 x 256
    x4_go<N, 16, e_line(N)>(ctx, g, spec);
    name = "k_x_fast4";
  } else if (zc && N >= 64 && ctx->nzh % X4TW == 0) {  // (8 elements/thread at 512: 6.5 vs 5.9 ms)
    // (16-column tiles = 256-byte row segments at 256 points, one CTA per SM: 0.656 vs 0.479 ms in the debug build)
#ifndef FM_X4_E128
#define FM_X4_E128 16  // elements per thread of the 128-point x pass (A/B: 8)
#endif
    x4_go<N, X4TW, (N == 128 ? FM_X4_E128 : e_line(N))>(ctx, g, spec);
    name = "k_x_fast4";
  } else if (N <= 512 && ctx->nzh % 8 == 0 && !(zc && N < 64)) {
    x3_go<N, 8, e_line(N)>(ctx, g, spec);
    name = "k_x_fast3";
  } else {
    const dim3 grid(ctx->nzh / TW, g.Ny, 3);
    if (g.P > 1) {
      allow(k_x_fast<N, TW, 3, true>, smem);
      k_x_fast<N, TW, 3, true><<<grid, TW * T, smem, ctx->stream>>>(g, ctx->px.tw, spec);
    } else {
      allow(k_x_fast<N, TW, 3>, smem);
      k_x_fast<N, TW, 3><<<grid, TW * T, smem, ctx->stream>>>(g, ctx->px.tw, spec);
    }
  }
  *st = launched(ctx, name);
  return true;
}

template <int M, int PRO, bool DIR, bool PAP>
void zf_go(fm_ctx* ctx, const Geo& g, const ProArgs& pa, double2* spec) {
  using S = ZShape<M, PRO != PRO_COPY>;
  allow(k_zf_fast<M, PRO, DIR, PAP>, S::SMEM);
  const int nxy = g.Nx * g.Ny;
  const dim3 grid((nxy + S::G - 1) / S::G);
  k_zf_fast<M, PRO, DIR, PAP><<<grid, S::THREADS, S::SMEM, ctx->stream>>>(g, ctx->pzh.tw, ctx->pz.tw, pa, spec);
  ctx->zf_partials = int(grid.x);
}

int zpipe_mode() {  // FM_ZPIPE=0 disables the pipelined z-forward pass
  static int v = [] {
    const char* e = getenv("FM_ZPIPE");
    return e ? atoi(e) : 1;
  }();
  return v;
}

// 3 CTAs/SM register budget (measured best of 1..4 and single-voxel variants)
template <int PRO, int M, bool LAB = false, bool DIR = false>
constexpr int pipe_minb() {  // copy: fewer registers suffice up to M = 128 (512^3: 5 CTAs/SM is slower)
  return (PRO == PRO_COPY && M <= 128) ? kPipeCopyMinB : (LAB && !DIR && M <= 128 ? kPipeLabMinB : 3);
}

// FM_ZPIPE_LB2=0: one line buffer (two block barriers per line; A/B)
int zpipe_lb2_mode() {
  static int v = [] {
    const char* e = getenv("FM_ZPIPE_LB2");
    return e ? atoi(e) : 1;
  }();
  return v;
}

template <int M, int PRO, bool DIR, bool PAP, bool XUPD, bool LAB, bool LB2>
bool zpipe_go2(fm_ctx* ctx, const Geo& g, const ProArgs& pa, double2* spec);

// CTAs per SM a pipelined pass gets: shared memory (227 KB / SM, 1 KB reserved per CTA) or the register budget
template <int M, int PRO, bool DIR, bool XUPD, bool LAB, bool LB2>
constexpr int pipe_per_sm() {
  return std::min(int((227 * 1024) / (pipe_smem<M, PRO, DIR, XUPD, LAB, LB2>() + 1024)), pipe_minb<PRO, M, LAB, DIR>());
}
// the second line buffer is used where it costs no CTA per SM
template <int M, int PRO, bool DIR, bool XUPD, bool LAB>
constexpr bool lb2_free() {
  return pipe_per_sm<M, PRO, DIR, XUPD, LAB, true>() == pipe_per_sm<M, PRO, DIR, XUPD, LAB, false>();
}

template <int M, int PRO, bool DIR, bool PAP, bool XUPD = false, bool LAB = false>
bool zpipe_go(fm_ctx* ctx, const Geo& g, const ProArgs& pa, double2* spec) {
  if constexpr (lb2_free<M, PRO, DIR, XUPD, LAB>()) {
    if (zpipe_lb2_mode()) return zpipe_go2<M, PRO, DIR, PAP, XUPD, LAB, true>(ctx, g, pa, spec);
  }
  return zpipe_go2<M, PRO, DIR, PAP, XUPD, LAB, false>(ctx, g, pa, spec);
}

template <int M, int PRO, bool DIR, bool PAP, bool XUPD, bool LAB, bool LB2>
bool zpipe_go2(fm_ctx* ctx, const Geo& g, const ProArgs& pa, double2* spec) {
  constexpr int MB = pipe_minb<PRO, M, LAB, DIR>();
  constexpr size_t smem = pipe_smem<M, PRO, DIR, XUPD, LAB, LB2>();
  // one CTA per SM does not pay (512^3: 2x slower); single-buffered passes above 100 KB lose to k_zf_fast
  if constexpr ((!LB2 && smem > 100 * 1024) || pipe_per_sm<M, PRO, DIR, XUPD, LAB, LB2>() < 2 || M < 16) {
    return false;
  } else {
    allow(k_zf_pipe<M, PRO, DIR, MB, PAP, XUPD, LAB, LB2>, smem);
    static const int per_sm = [] {  // (occupancy: the same on every B200 of the node)
      int b = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_zf_pipe<M, PRO, DIR, MB, PAP, XUPD, LAB, LB2>,
                                                    ZPipe<M>::THREADS, smem);
      cudaGetLastError();
      return b > 0 ? b : 1;
    }();
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int nxy = g.Nx * g.Ny;
    const int grid = std::min(nxy, std::max(sms, 1) * per_sm);
    static const int zdbg = [] {
      const char* e = getenv("FM_ZP_DBG");
      return e ? atoi(e) : 0;
    }();
    ProArgs pad = pa;
    pad.dbg = zdbg;
    k_zf_pipe<M, PRO, DIR, MB, PAP, XUPD, LAB, LB2>
        <<<grid, ZPipe<M>::THREADS, smem, ctx->stream>>>(g, ctx->pzh.tw, ctx->pz.tw, pad, spec);
    ctx->zf_partials = grid;
    return true;
  }
}

template <int M, int PRO, bool PAP>
void zf_kind(fm_ctx* ctx, const Geo& g, const ProArgs& pa, double2* spec, bool dir, int* st) {
  if constexpr (PRO == PRO_SVK) {
    const bool lab = pa.lab != nullptr;
    if (pa.x) {  // fused CG x update: only the pipelined kernel carries it (cg_xupd_supported)
      if (dir && PAP && (lab ? zpipe_go<M, PRO, true, PAP, true, true>(ctx, g, pa, spec)
                             : zpipe_go<M, PRO, true, PAP, true>(ctx, g, pa, spec))) {
        *st = launched(ctx, "k_zf_pipe");
      } else {
        *st = set_error(ctx, FM_E_UNSUPPORTED, "fused x update without the pipelined z-forward pass");
      }
      return;
    }
    bool ok = false;
    if (zpipe_mode()) {
      if (lab && dir) ok = zpipe_go<M, PRO, true, PAP, false, true>(ctx, g, pa, spec);
      else if (lab) ok = zpipe_go<M, PRO, false, PAP, false, true>(ctx, g, pa, spec);
      else ok = dir ? zpipe_go<M, PRO, true, PAP>(ctx, g, pa, spec) : zpipe_go<M, PRO, false, PAP>(ctx, g, pa, spec);
    }
    if (ok) {
      *st = launched(ctx, "k_zf_pipe");
      return;
    }
  }
  if (dir) zf_go<M, PRO, true, PAP>(ctx, g, pa, spec);
  else zf_go<M, PRO, false, PAP>(ctx, g, pa, spec);
  *st = launched(ctx, "k_zf_fast");
}

// Register-resident z passes (k_zi_reg / k_zf_reg): E elements per lane,
// 128 threads per CTA, MINB CTAs/SM for the register budget.  FM_ZREG=0
// selects the staged passes instead (A/B measurements).
int zreg_mode() {
  static int v = [] {
    const char* e = getenv("FM_ZREG");
    return e ? atoi(e) : 1;
  }();
  return v;
}
template <int M>
struct ZReg {
  static constexpr int E = M >= 128 ? 16 : 8;
  static constexpr int T = M / E;
  static constexpr int LPC = 128 / T;
  static constexpr int THREADS = LPC * T;
#ifndef FM_ZREG_MINB256
#define FM_ZREG_MINB256 4  // CTAs/SM of the 256-point (Nz = 512) z passes; 3 (no spills, 168 registers): 3.22 vs 3.09 ms forward, 3.37 vs 3.35 ms inverse at 512^3
#endif
  static constexpr int MINB = M == 256 ? FM_ZREG_MINB256 : 4;
  static constexpr size_t SMEM = size_t(LPC) * M * 16;
  static constexpr bool OK = M >= 16 && 32 % T == 0;
};

template <int M>
bool zf_reg_go(fm_ctx* ctx, const Geo& g, const ProArgs& pa, double2* spec) {
  using S = ZReg<M>;
  if constexpr (!S::OK) {
    return false;
  } else {
    allow(k_zf_reg<M, S::E, S::LPC, S::MINB>, S::SMEM);
    const int64_t nl = int64_t(9) * g.Nx * g.Ny;
    const dim3 grid(unsigned((nl + S::LPC - 1) / S::LPC));
    k_zf_reg<M, S::E, S::LPC, S::MINB>
        <<<grid, S::THREADS, S::SMEM, ctx->stream>>>(g, ctx->pzh.tw, ctx->pz.tw, pa.A, spec);
    ctx->zf_partials = 0;
    return true;
  }
}

template <int M>
bool zi_reg_go(fm_ctx* ctx, const Geo& g, const double2* spec, double* out, double scale, const EpiArgs& epi) {
  using S = ZReg<M>;
  if constexpr (!S::OK) {
    return false;
  } else {
    const int64_t nl = int64_t(9) * g.Nx * g.Ny;
    const dim3 grid(unsigned((nl + S::LPC - 1) / S::LPC));
    if (epi.r || epi.partial) {
      allow(k_zi_reg<M, S::E, S::LPC, S::MINB, true>, S::SMEM);
      k_zi_reg<M, S::E, S::LPC, S::MINB, true>
          <<<grid, S::THREADS, S::SMEM, ctx->stream>>>(g, ctx->pzh.tw, ctx->pz.tw, spec, out, scale, epi);
    } else {
      allow(k_zi_reg<M, S::E, S::LPC, S::MINB>, S::SMEM);
      k_zi_reg<M, S::E, S::LPC, S::MINB>
          <<<grid, S::THREADS, S::SMEM, ctx->stream>>>(g, ctx->pzh.tw, ctx->pz.tw, spec, out, scale, epi);
    }
    ctx->zi_partials = int(grid.x);
    return true;
  }
}

template <int M>
bool zf_launch(fm_ctx* ctx, const Geo& g, const ProArgs& pa, double2* spec, int* st) {
  const bool dir = pa.r != nullptr;
  const bool pap = pa.pap_partial != nullptr;
  if (pa.kind == PRO_COPY && zreg_mode() && zf_reg_go<M>(ctx, g, pa, spec)) {
    *st = launched(ctx, "k_zf_reg");
    return true;
  }
  if (pa.kind == PRO_COPY) {
    if (zpipe_mode() && zpipe_go<M, PRO_COPY, false, false>(ctx, g, pa, spec)) {
      *st = launched(ctx, "k_zf_pipe");
      return true;
    }
    zf_go<M, PRO_COPY, false, false>(ctx, g, pa, spec);
    *st = launched(ctx, "k_zf_fast");
  } else if (pa.kind == PRO_K4) {
    pap ? zf_kind<M, PRO_K4, true>(ctx, g, pa, spec, dir, st) : zf_kind<M, PRO_K4, false>(ctx, g, pa, spec, dir, st);
  } else if (pa.kind == PRO_J2C) {
    pap ? zf_kind<M, PRO_J2C, true>(ctx, g, pa, spec, dir, st) : zf_kind<M, PRO_J2C, false>(ctx, g, pa, spec, dir, st);
  } else {
    pap ? zf_kind<M, PRO_SVK, true>(ctx, g, pa, spec, dir, st) : zf_kind<M, PRO_SVK, false>(ctx, g, pa, spec, dir, st);
  }
  return true;
}

template <int M, typename S>
void zi_go(fm_ctx* ctx, const Geo& g, const double2* spec, double* out, double scale, const EpiArgs& epi) {
  constexpr size_t kR = size_t(9) * S::G * 2 * M * 8;  // fused CG: staged residual lines
  allow(k_zi_fast<M, S>, S::SMEM + kR);
  const int nxy = g.Nx * g.Ny;
  const dim3 grid((nxy + S::G - 1) / S::G);
  const size_t smem = S::SMEM + (epi.r ? kR : 0);
  k_zi_fast<M, S><<<grid, S::THREADS, smem, ctx->stream>>>(g, ctx->pzh.tw, ctx->pz.tw, spec, out, scale, epi);
}

// z-inverse shape: 16 elements per thread, one z-line per CTA from M = 128 up,
// registers budgeted for 6 CTAs/SM (measured at 256^3: E8/G2 643 us, E16/G1
// 4 CTAs 636 us, 6 CTAs 580 us; 512^3: E8/G1 4.95 ms, E16/G1 4 CTAs 4.67 ms,
// 6 CTAs spills)
template <int M>
using ZiShape = std::conditional_t<(M >= 128), ZS<M, 16, 1, (M == 128 ? 6 : 4)>, ZShape<M>>;

template <int M>
bool zi_launch(fm_ctx* ctx, const Geo& g, const double2* spec, double* out, double scale, const EpiArgs& epi,
               int* st) {
  if (zreg_mode() && zi_reg_go<M>(ctx, g, spec, out, scale, epi)) {
    *st = launched(ctx, "k_zi_reg");
    return true;
  }
  zi_go<M, ZiShape<M>>(ctx, g, spec, out, scale, epi);
  ctx->zi_partials = (g.Nx * g.Ny + ZiShape<M>::G - 1) / ZiShape<M>::G;
  *st = launched(ctx, "k_zi_fast");
  return true;
}

bool fast_z_ok(const fm_ctx* ctx) {
  return ctx->tdim == 3 && ctx->mode == FM_NYQUIST_ZERO_COMPATIBLE && ctx->Nz % 2 == 0 &&
         ctx->nzh == ctx->Nz / 2;
}
bool fast_xy_ok(const fm_ctx* ctx, int N) {
  return ctx->tdim == 3 && ctx->nzh % tw_of(N) == 0 && ctx->nzh % tw_x(N) == 0;
}

}  // namespace

#define FM_POW2_CASES(X, N_, ...)              \
  switch (N_) {                                \
    case 32: return X<32>(__VA_ARGS__);        \
    case 64: return X<64>(__VA_ARGS__);        \
    case 128: return X<128>(__VA_ARGS__);      \
    case 256: return X<256>(__VA_ARGS__);      \
    case 512: return X<512>(__VA_ARGS__);      \
    case 1024: return X<1024>(__VA_ARGS__);    \
    default: return false;                     \
  }

#define FM_HALF_CASES(X, M_, ...)              \
  switch (M_) {                                \
    case 16: return X<16>(__VA_ARGS__);        \
    case 32: return X<32>(__VA_ARGS__);        \
    case 64: return X<64>(__VA_ARGS__);        \
    case 128: return X<128>(__VA_ARGS__);      \
    case 256: return X<256>(__VA_ARGS__);      \
    case 512: return X<512>(__VA_ARGS__);      \
    default: return false;                     \
  }

bool y_fast(fm_ctx* ctx, const Geo& g, int sign, const double2* in, double2* out, int* st) {
  if (!fast_xy_ok(ctx, g.Ny)) return false;
  FM_POW2_CASES(y_launch, g.Ny, ctx, g, sign, in, out, st)
}

bool x_fast(fm_ctx* ctx, const Geo& g, double2* spec, int* st) {
  if (!fast_xy_ok(ctx, g.Nx)) return false;
  FM_POW2_CASES(x_launch, g.Nx, ctx, g, spec, st)
}

bool zf_fast(fm_ctx* ctx, const Geo& g, const ProArgs& pa, double2* spec, int* st) {
  if (!fast_z_ok(ctx)) return false;
  FM_HALF_CASES(zf_launch, ctx->Nz / 2, ctx, g, pa, spec, st)
}

bool zi_fast(fm_ctx* ctx, const Geo& g, const double2* spec, double* out, double scale, const EpiArgs& epi,
             int* st) {
  if (!fast_z_ok(ctx)) return false;
  FM_HALF_CASES(zi_launch, ctx->Nz / 2, ctx, g, spec, out, scale, epi, st)
}

bool cg_xupd_supported(const fm_ctx* ctx, int kind) {
  const int M = ctx->Nz / 2;
  return kind == PRO_SVK && zpipe_mode() && cg_fused_supported(ctx) &&
         pipe_smem<128, PRO_SVK, true, true>() <= 100 * 1024 && M <= 128;
}

bool cg_fused_supported(const fm_ctx* ctx) {
  const int M = ctx->Nz / 2;
  const bool pow2 = M >= 16 && M <= 512 && (M & (M - 1)) == 0;
  // slab ranks: each rank's pass-1 partials are summed across ranks in rank
  // order (combine_ranks) before alpha is formed
  const int64_t lines = int64_t(ctx->Nx / ctx->P) * ctx->Ny * ctx->P;
  return fast_z_ok(ctx) && pow2 && lines <= ctx->epi_cap;
}

}  // namespace fm
