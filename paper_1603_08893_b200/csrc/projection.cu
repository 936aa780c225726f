#include <cstdio>
#include <cstdlib>
// Compatibility projection G and the projected tangent G(K : dF^T) on sm_100a.
//
// Restates apply_projection / apply_projected_tangent
// (reference proj/core/src/projection.cpp:123-194) as five HBM passes over
// the r2c half spectrum, with the reference's stored ĝ table
// (projection.cpp:87-104, 72 B/voxel) replaced by an analytic evaluation
// from the wave vector inside the x pass:
//   pass 1  z  : prologue (copy | K:dF^T | SVK action) + real-to-complex FFT
//   pass 2  y  : forward complex FFT (writes the all-to-all packed layout)
//   pass 3  x  : forward FFT, Bhat_i. = (Ahat_i . xi) xi / |xi|^2, inverse FFT
//   pass 4  y  : inverse complex FFT (reads the packed layout)
//   pass 5  z  : complex-to-real inverse FFT, scale 1/n
// ghat(-q) = ghat(q) and the Nyquist set is symmetric, so the half spectrum
// is exact; the imaginary residue the reference checks
// (projection.cpp:157-169) is dropped exactly as its Re() does.
//
// Slab decomposition over P ranks: passes 1-2 and 4-5 run
// on x-slabs, pass 3 on y-slabs, with the all-to-all between them (dist.cu).
// This file holds the generic kernels (any line length, tdim 2 or 3) and the
// pass dispatcher; projection_fast.cu the register-resident ones.
#include <algorithm>
#include <cmath>

#include <cooperative_groups.h>

#include "proj_common.cuh"

namespace fm {

// ------------------------------------------------------------------ pass 1
// Work item `bx` (G z-lines) of pass 1.  PAP: per-item partial of <dF, dP>
// (fused CG curvature) into pa.pap_partial[bx].
template <int TD, int PRO, bool DIR, bool PAP = false>
__device__ __forceinline__ void zfwd_body(const Geo& g, const AxisPlan& plan, const double2* __restrict__ twN,
                                          const ProArgs& pa, double2* __restrict__ spec, int G, int ls, int bx,
                                          double2* sm, const double2* tw_pre = nullptr) {
  constexpr int NC = TD * TD;
  const int nxy = g.Nx * g.Ny;
  const int L0 = bx * G;
  const int Gb = min(G, nxy - L0);
  double2* A = sm;
  double2* B = sm + NC * G * ls;
  const bool even = (g.Nz % 2 == 0);
  double pap = 0.0;
  for (int w = threadIdx.x; w < Gb * g.Nz; w += blockDim.x) {
    const int gi = w / g.Nz, z = w - gi * g.Nz;
    const int64_t node = g.roff + int64_t(L0 + gi) * g.Nz + z;
    double v[NC];
    prologue_voxel<TD, PRO, DIR, PAP>(pa, g.n, node, v, &pap);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      double2* line = A + (c * G + gi) * ls;
      if (even)
        reinterpret_cast<double*>(line)[z] = v[c];
      else
        line[z] = make_double2(v[c], 0.0);
    }
  }
  __syncthreads();
  double2* R = fft_smem(A, B, NC * G, ls, 1, plan, -1, false, sm + 2 * NC * G * ls, tw_pre);
  const int M = g.Lz;
  for (int w = threadIdx.x; w < NC * Gb * g.nzh; w += blockDim.x) {
    const int line = w / g.nzh, k = w - line * g.nzh;
    const int c = line / Gb, gi = line - c * Gb;
    const double2* Z = R + (c * G + gi) * ls;
    double2 X;
    if (even) {
      // X[k] = E[k] + W_N^k O[k], E = (Z[k] + Z*[M-k])/2, O = -i (Z[k] - Z*[M-k])/2
      const double2 a = Z[k % M];
      const double2 b = cconj(Z[(M - k) % M]);
      const double2 E = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y + b.y));
      const double2 D = csub(a, b);
      const double2 O = make_double2(0.5 * D.y, -0.5 * D.x);
      X = cadd(E, cmul(O, __ldg(&twN[k])));
    } else {
      X = Z[k];
    }
    spec[(int64_t(c) * nxy + L0 + gi) * g.nzh + k] = X;
  }
  if constexpr (PAP) {
    pap = block_sum_any(pap);
    if (threadIdx.x == 0) pa.pap_partial[bx] = pap;
  }
  __syncthreads();  // smem reusable by the next work item
}

template <int TD, int PRO, bool DIR>
__global__ void __launch_bounds__(256) k_zfwd(Geo g, AxisPlan plan, const double2* __restrict__ twN,
                                              ProArgs pa, double2* __restrict__ spec, int G, int ls) {
  extern __shared__ double2 sm[];
  zfwd_body<TD, PRO, DIR>(g, plan, twN, pa, spec, G, ls, blockIdx.x, sm);
}

// -------------------------------------------------------------- pass 2 / 4
// In place on one device; P > 1 the forward pass (sign -1) stores into the
// x-pass inputs of the y-slab owners (store_yf, the fused slab transpose).
__device__ __forceinline__ void ypass_body(const Geo& g, const AxisPlan& plan, const double2* in, double2* out,
                                           int TW, int sign, int bx, int by, int bz, double2* sm,
                                           const double2* tw_pre = nullptr) {
  const int kz0 = bx * TW;
  const int x = by, c = bz;
  const int Ny = g.Ny;
  double2* A = sm;
  double2* B = sm + Ny * TW;
  for (int w = threadIdx.x; w < Ny * TW; w += blockDim.x) {
    const int e = w / TW, t = w - e * TW;
    const int kz = kz0 + t;
    if (kz < g.nzh)
      A[w] = in[spec_std(g, c, x, e, kz)];
    else
      A[w] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  double2* R = fft_smem(A, B, TW, 1, TW, plan, sign, true, sm + 2 * Ny * TW, tw_pre);
  for (int w = threadIdx.x; w < Ny * TW; w += blockDim.x) {
    const int e = w / TW, t = w - e * TW;
    const int kz = kz0 + t;
    if (kz >= g.nzh) continue;
    if (sign < 0) store_yf(g, out, c, x, e, kz, R[w]);
    else out[spec_std(g, c, x, e, kz)] = R[w];
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) k_ypass(Geo g, AxisPlan plan, const double2* in,
                                               double2* out, int TW, int sign) {  // in == out when P = 1
  extern __shared__ double2 sm[];
  ypass_body(g, plan, in, out, TW, sign, blockIdx.x, blockIdx.y, blockIdx.z, sm);
}

// ------------------------------------------------------------------ pass 3
template <int TD>
__device__ __forceinline__ void xpass_body(const Geo& g, const AxisPlan& plan, double2* spec, int TW,
                                           int bx, int by, int bz, double2* sm, const double2* tw_pre = nullptr) {
  const int kz0 = bx * TW;
  const int y = by, i = bz;
  const int Nx = g.Nx;
  const int nl = TD * TW;
  double2* A = sm;
  double2* B = sm + Nx * nl;
  const int64_t xstride = int64_t(g.Ny) * g.nzh;
  for (int w = threadIdx.x; w < Nx * nl; w += blockDim.x) {
    const int t = w % TW, j = (w / TW) % TD, e = w / nl;
    const int kz = kz0 + t;
    A[w] = kz < g.nzh
               ? spec[(int64_t(i * TD + j) * Nx + e) * xstride + int64_t(y) * g.nzh + kz]
               : make_double2(0.0, 0.0);
  }
  __syncthreads();
  double2* R = fft_smem(A, B, nl, 1, nl, plan, -1, true, sm + 2 * Nx * nl, tw_pre);
  double2* S = (R == A) ? B : A;
  // Bhat_ij = sum_l Ahat_il ghat_lj, ghat = xi (x) xi / |xi|^2 (projection.cpp:87-104,139-152)
  const int yg = g.y0 + y;
  const int qy = freq_of(yg, g.Nyg);
  const bool ny_y = (g.Nyg % 2 == 0) && (yg == g.Nyg / 2);
  for (int w = threadIdx.x; w < Nx * TW; w += blockDim.x) {
    const int e = w / TW, t = w - e * TW;
    const int kz = kz0 + t;
    if (kz >= g.nzh) continue;
    const int qx = freq_of(e, Nx), qz = freq_of(kz, g.Nz);
    const bool nyq = ny_y || ((Nx % 2 == 0) && (e == Nx / 2)) || ((g.Nz % 2 == 0) && (kz == g.Nz / 2));
    double xi[3] = {qx * g.invL[0], qy * g.invL[1], g.dim == 3 ? qz * g.invL[2] : 0.0};
    const double norm2 = xi[0] * xi[0] + xi[1] * xi[1] + xi[2] * xi[2];
    double2* v = R + e * nl + t;
    if (norm2 == 0.0 || (nyq && g.mode == FM_NYQUIST_ZERO_COMPATIBLE)) {
#pragma unroll
      for (int j = 0; j < TD; ++j) v[j * TW] = make_double2(0.0, 0.0);
    } else if (!nyq) {
      double2 s = make_double2(0.0, 0.0);
#pragma unroll
      for (int l = 0; l < TD; ++l) {
        if (l < g.dim) {
          const double2 a = v[l * TW];
          s.x += a.x * xi[l];
          s.y += a.y * xi[l];
        }
      }
      const double inv = 1.0 / norm2;
#pragma unroll
      for (int j = 0; j < TD; ++j) {
        const double f = j < g.dim ? xi[j] * inv : 0.0;
        v[j * TW] = make_double2(s.x * f, s.y * f);
      }
    }  // Nyquist in IdentityEquilibrium mode: ghat = I, keep v
  }
  __syncthreads();
  R = fft_smem(R, S, nl, 1, nl, plan, +1, true, sm + 2 * Nx * nl, tw_pre);
  for (int w = threadIdx.x; w < Nx * nl; w += blockDim.x) {
    const int t = w % TW, j = (w / TW) % TD, e = w / nl;
    const int kz = kz0 + t;
    if (kz < g.nzh)
      store_xb(g, spec + (int64_t(i * TD + j) * Nx + e) * xstride + int64_t(y) * g.nzh + kz, i * TD + j, e, y, kz,
               R[w]);
  }
  __syncthreads();
}

template <int TD>
__global__ void __launch_bounds__(256) k_xpass(Geo g, AxisPlan plan, double2* spec,
                                               int TW) {
  extern __shared__ double2 sm[];
  xpass_body<TD>(g, plan, spec, TW, blockIdx.x, blockIdx.y, blockIdx.z, sm);
}

// ------------------------------------------------------------------ pass 5
// Work item `bx` (G z-lines) of pass 5.  Epilogue: store out (and the <pdot,
// out> partial), or -- fused CG, epi.r set -- r -= alpha Ap (x += alpha p when
// epi.x) with the partial of <r, r>; partials go to epi.partial[bx].
template <int TD>
__device__ __forceinline__ void zinv_body(const Geo& g, const AxisPlan& plan, const double2* __restrict__ twN,
                                          const double2* __restrict__ spec, double* __restrict__ out, int G,
                                          int ls, double scale, const EpiArgs& epi, int bx, double2* sm,
                                          const double2* tw_pre = nullptr) {
  constexpr int NC = TD * TD;
  const int nxy = g.Nx * g.Ny;
  const int L0 = bx * G;
  const int Gb = min(G, nxy - L0);
  double2* A = sm;
  double2* B = sm + NC * G * ls;
  const bool even = (g.Nz % 2 == 0);
  for (int w = threadIdx.x; w < NC * Gb * g.nzh; w += blockDim.x) {
    const int line = w / g.nzh, k = w - line * g.nzh;
    const int c = line / Gb, gi = line - c * Gb;
    A[(c * G + gi) * ls + k] = spec[(int64_t(c) * nxy + L0 + gi) * g.nzh + k];
  }
  __syncthreads();
  const int M = g.Lz;
  for (int w = threadIdx.x; w < NC * Gb * M; w += blockDim.x) {
    const int line = w / M, k = w - line * M;
    const int c = line / Gb, gi = line - c * Gb;
    const double2* X = A + (c * G + gi) * ls;
    double2 Z;
    if (even) {
      // Z[k] = (X[k] + X*[M-k]) + i W_N^{-k} (X[k] - X*[M-k]); X[M] = 0 when not stored.
      // Re(ifft) as the reference takes it (projection.cpp:157-162): the kz = 0
      // and kz = M columns of a real field are real, so their (round-off)
      // imaginary parts are dropped, not folded into the output.
      double2 a = X[k];
      if (k == 0) a.y = 0.0;
      double2 b = (M - k < g.nzh) ? cconj(X[M - k]) : make_double2(0.0, 0.0);
      if (k == 0) b.y = 0.0;
      const double2 t = cmulc(csub(a, b), __ldg(&twN[k]));
      Z = make_double2(a.x + b.x - t.y, a.y + b.y + t.x);
    } else {
      Z = k < g.nzh ? X[k] : cconj(X[g.Nz - k]);
    }
    B[(c * G + gi) * ls + k] = Z;
  }
  __syncthreads();
  double2* R = fft_smem(B, A, NC * G, ls, 1, plan, +1, false, sm + 2 * NC * G * ls, tw_pre);
  double dot = 0.0;
  for (int w = threadIdx.x; w < NC * Gb * g.Nz; w += blockDim.x) {
    const int line = w / g.Nz, z = w - line * g.Nz;
    const int c = line / Gb, gi = line - c * Gb;
    const double2* Zl = R + (c * G + gi) * ls;
    double v;
    if (even) {
      const double2 zz = Zl[z >> 1];
      v = (z & 1) ? zz.y : zz.x;
    } else {
      v = Zl[z].x;
    }
    const int64_t idx = int64_t(c) * g.n + g.roff + int64_t(L0 + gi) * g.Nz + z;
    if (epi.r) {  // fused CG update, solver.cpp:46-48 with k_cg_update's rounding
      if (epi.scal[S_FLAG] == 0.0) {
        const double alpha = epi.scal[S_ALPHA];
        const double rv = __dadd_rn(epi.r[idx], __dmul_rn(-alpha, v * scale));
        epi.r[idx] = rv;
        if (epi.x) epi.x[idx] = __dadd_rn(epi.x[idx], __dmul_rn(alpha, epi.p[idx]));
        dot += rv * rv;
      }
      continue;
    }
    out[idx] = v * scale;
    if (epi.partial) dot += __ldg(epi.pdot + idx) * (v * scale);
  }
  if (epi.partial) {
    dot = block_sum_any(dot);
    if (threadIdx.x == 0) epi.partial[bx] = dot;
  }
  __syncthreads();
}

template <int TD>
__global__ void __launch_bounds__(256) k_zinv(Geo g, AxisPlan plan, const double2* __restrict__ twN,
                                              const double2* __restrict__ spec,
                                              double* __restrict__ out, int G, int ls,
                                              double scale, EpiArgs epi) {
  extern __shared__ double2 sm[];
  zinv_body<TD>(g, plan, twN, spec, out, G, ls, scale, epi, blockIdx.x, sm);
}

// ------------------------------------------------- persistent small-grid CG
// The whole CG loop (solver.cpp:19-58) of a latency-bound grid as ONE
// cooperative launch: the five passes are phases over work items separated
// by grid-wide barriers, the curvature / residual reductions are summed by
// every block in the same fixed order (so every block takes the same branch),
// and the iteration loop runs on the device.  Fused iteration as on the
// register-resident path: <p, K:p> from pass 1, r -= alpha Ap and
// x += alpha p in pass 5, Ap never stored.
struct CgSmallArgs {
  Geo gz, gx;
  AxisPlan pz, py, px;
  const double2* twN;
  ProArgs op;
  double2* spec;
  double *x, *r, *p;
  double* pap_part;
  double* rr_part;
  double* scal;
  int G, ls, tw_y, tw_x, nz_items, ny_items, nx_items, ny_gx, nx_gx;
  int tw_off;  // dynamic-smem offset (double2) of the staged twiddle tables
  double rr0, thr, scale;
  int64_t cap;
  unsigned long long* tdbg;  // optional: block-0 phase timestamps of the first 8 iterations (FM_CG_SMALL_TIMING)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// sum of n per-item partials, identical in every block (fixed thread -> index map)
__device__ __forceinline__ double items_sum(const double* part, int n, double* bcast) {
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
  s = block_sum_any(s);
  if (threadIdx.x == 0) *bcast = s;
  __syncthreads();
  s = *bcast;
  __syncthreads();
  return s;
}

template <int PRO>
__global__ void __launch_bounds__(256) k_cg_small(CgSmallArgs a) {
  namespace cgp = cooperative_groups;
  extern __shared__ double2 sm[];
  __shared__ double ssc[16];
  cgp::grid_group grid = cgp::this_grid();
  double rr = a.rr0, rr_new = 0.0, pap = 0.0, beta = 0.0;
  int64_t it = 0;
  int exit_kind = 3;  // 1: !(pAp > 0), 2: converged, 3: cap
  // the three axes' twiddle tables, staged once for the whole CG loop
  double2* twz = sm + a.tw_off;
  double2* twy = twz + a.pz.N;
  double2* twx = twy + a.py.N;
  for (int i = threadIdx.x; i < a.pz.N; i += blockDim.x) twz[i] = __ldg(&a.pz.tw[i]);
  for (int i = threadIdx.x; i < a.py.N; i += blockDim.x) twy[i] = __ldg(&a.py.tw[i]);
  for (int i = threadIdx.x; i < a.px.N; i += blockDim.x) twx[i] = __ldg(&a.px.tw[i]);
  __syncthreads();
  auto mark = [&](int k) {
    if (a.tdbg && blockIdx.x == 0 && threadIdx.x == 0 && it <= 8) a.tdbg[(it - 1) * 8 + k] = gtimer();
  };
  while (it < a.cap) {
    ++it;
    mark(0);
    if (threadIdx.x == 0) ssc[S_BETA] = beta;  // 0 in the first iteration: p = r = b
    __syncthreads();
    ProArgs pa = a.op;
    pa.A = a.p;
    pa.r = a.r;
    pa.p = a.p;
    pa.beta = &ssc[S_BETA];
    pa.pap_partial = a.pap_part;
    for (int w = blockIdx.x; w < a.nz_items; w += gridDim.x)
      zfwd_body<3, PRO, true, true>(a.gz, a.pz, a.twN, pa, a.spec, a.G, a.ls, w, sm, twz);
    mark(1);
    grid.sync();
    mark(2);
    pap = items_sum(a.pap_part, a.nz_items, &ssc[8]);
    if (!(pap > 0.0)) {  // :38-44, x not updated
      exit_kind = 1;
      break;
    }
    if (threadIdx.x == 0) {
      ssc[S_ALPHA] = rr / pap;
      ssc[S_FLAG] = 0.0;
    }
    __syncthreads();
    for (int w = blockIdx.x; w < a.ny_items; w += gridDim.x) {
      const int bx = w % a.ny_gx, rest = w / a.ny_gx;
      ypass_body(a.gz, a.py, a.spec, a.spec, a.tw_y, -1, bx, rest % a.gz.Nx, rest / a.gz.Nx, sm, twy);
    }
    grid.sync();
    mark(3);
    for (int w = blockIdx.x; w < a.nx_items; w += gridDim.x) {
      const int bx = w % a.nx_gx, rest = w / a.nx_gx;
      xpass_body<3>(a.gx, a.px, a.spec, a.tw_x, bx, rest % a.gx.Ny, rest / a.gx.Ny, sm, twx);
    }
    grid.sync();
    mark(4);
    for (int w = blockIdx.x; w < a.ny_items; w += gridDim.x) {
      const int bx = w % a.ny_gx, rest = w / a.ny_gx;
      ypass_body(a.gz, a.py, a.spec, a.spec, a.tw_y, +1, bx, rest % a.gz.Nx, rest / a.gz.Nx, sm, twy);
    }
    grid.sync();
    mark(5);
    EpiArgs e;
    e.r = a.r;
    e.x = a.x;
    e.p = a.p;
    e.scal = ssc;
    e.partial = a.rr_part;
    for (int w = blockIdx.x; w < a.nz_items; w += gridDim.x)
      zinv_body<3>(a.gz, a.pz, a.twN, a.spec, nullptr, a.G, a.ls, a.scale, e, w, sm, twz);
    mark(6);
    grid.sync();
    rr_new = items_sum(a.rr_part, a.nz_items, &ssc[8]);
    mark(7);
    if (sqrt(rr_new) <= a.thr) {  // :49-50
      exit_kind = 2;
      break;
    }
    beta = rr_new / rr;  // :51-55
    rr = rr_new;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.scal[S_IT] = double(it);
    a.scal[S_RR] = rr;
    a.scal[S_RRNEW] = rr_new;
    a.scal[S_PAP] = pap;
    a.scal[S_FLAG] = exit_kind == 1 ? 1.0 : 0.0;
    a.scal[S_OUT] = double(exit_kind);
  }
}

// ------------------------------------------------------------------- host
namespace {
constexpr int kMaxSmem = 227 * 1024;

template <typename K>
void allow_smem(K kernel) {
  // dynamic limit = 227 KB minus the kernel's static shared memory
  cudaFuncAttributes attr{};
  cudaFuncGetAttributes(&attr, kernel);
  cudaGetLastError();
  set_smem_limit(reinterpret_cast<const void*>(kernel), kMaxSmem - int(attr.sharedSizeBytes));
}

int tile_width(int nzh, int N, int lines_per_col, int& TW, int64_t other_blocks) {
  TW = std::min(8, nzh);
  while (TW > 1 && size_t(2 * TW * lines_per_col + 1) * N * 16 > size_t(kMaxSmem)) TW /= 2;
  // small grids: prefer more CTAs (>= 2 per SM) over wider tiles
  while (TW > 2 && int64_t((nzh + TW - 1) / TW) * other_blocks < 2 * 148) TW /= 2;
  return size_t(2 * TW * lines_per_col + 1) * N * 16 <= size_t(kMaxSmem) ? 0 : -1;
}

// Launch shape of the generic z passes for a (slab) geometry.
struct ZLaunch {
  int G, ls, threads;
  size_t smem;
  dim3 grid;
};

ZLaunch z_launch(const fm_ctx* ctx, const Geo& g) {
  const int NC = ctx->ncomp;
  const int nxy = g.Nx * g.Ny;
  ZLaunch L;
  L.ls = std::max(ctx->Lz, ctx->nzh);
  if (L.ls % 2 == 0) L.ls += 1;  // odd pitch: fewer bank conflicts
  int G = int(std::max<size_t>(1, std::min<size_t>(16, size_t(96 * 1024) / (size_t(2) * NC * L.ls * 16))));
  G = std::min(G, std::max(1, nxy / (2 * 148)));  // small grids: >= 2 CTAs per SM
  // latency-bound small grids (the 31^3 configs): one line group per CTA and
  // 128 threads -- config 1 2.54 -> 2.29 s (more threads per line measured no gain)
  if (nxy <= 148 * 16) G = 1;
  L.G = std::min(G, nxy);
  L.threads = (L.G * NC * ctx->Nz >= 2048 || L.G * ctx->Nz >= 256) ? 256 : 128;
  L.smem = size_t(2) * NC * L.G * L.ls * 16 + size_t((ctx->Nz % 2 == 0) ? ctx->pzh.N : ctx->pz.N) * 16;
  L.grid = dim3((nxy + L.G - 1) / L.G);
  return L;
}

void prof_mark(fm_ctx* ctx) {
  if (!ctx->prof.on || ctx->capturing) return;
  cudaEvent_t e;
  if (!ctx->prof.pool.empty()) {
    e = ctx->prof.pool.back();
    ctx->prof.pool.pop_back();
  } else {
    cudaEventCreate(&e);
  }
  cudaEventRecord(e, ctx->stream);
  ctx->prof.pending.push_back(e);
}

template <int TD>
void init_generic() {  // once per device (function attributes are per device)
  static bool init[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || init[dev]) return;
  allow_smem(k_zfwd<TD, PRO_COPY, false>);
  allow_smem(k_zfwd<TD, PRO_K4, false>);
  allow_smem(k_zfwd<TD, PRO_SVK, false>);
  allow_smem(k_zfwd<TD, PRO_K4, true>);
  allow_smem(k_zfwd<TD, PRO_SVK, true>);
  allow_smem(k_zfwd<TD, PRO_J2C, false>);
  allow_smem(k_zfwd<TD, PRO_J2C, true>);
  allow_smem(k_ypass);
  allow_smem(k_xpass<TD>);
  allow_smem(k_zinv<TD>);
  init[dev] = true;
}

template <int TD>
int pass_zf(fm_ctx* ctx, const Geo& g, const ProArgs& pa, double2* A) {
  int st = FM_OK;
  if (TD == 3 && zf_fast(ctx, g, pa, A, &st)) return st;
  const ZLaunch L = z_launch(ctx, g);
  if (L.smem + 1024 > size_t(kMaxSmem)) return set_error(ctx, FM_E_UNSUPPORTED, "z line too long for the shared-memory FFT");
  const bool even = ctx->Nz % 2 == 0;
  const AxisPlan& pzp = even ? ctx->pzh : ctx->pz;
  const bool dir = pa.r != nullptr;
  cudaStream_t s = ctx->stream;
  if (pa.kind == PRO_COPY)
    k_zfwd<TD, PRO_COPY, false><<<L.grid, L.threads, L.smem, s>>>(g, pzp, ctx->pz.tw, pa, A, L.G, L.ls);
  else if (pa.kind == PRO_K4 && !dir)
    k_zfwd<TD, PRO_K4, false><<<L.grid, L.threads, L.smem, s>>>(g, pzp, ctx->pz.tw, pa, A, L.G, L.ls);
  else if (pa.kind == PRO_K4)
    k_zfwd<TD, PRO_K4, true><<<L.grid, L.threads, L.smem, s>>>(g, pzp, ctx->pz.tw, pa, A, L.G, L.ls);
  else if (pa.kind == PRO_J2C && !dir)
    k_zfwd<TD, PRO_J2C, false><<<L.grid, L.threads, L.smem, s>>>(g, pzp, ctx->pz.tw, pa, A, L.G, L.ls);
  else if (pa.kind == PRO_J2C)
    k_zfwd<TD, PRO_J2C, true><<<L.grid, L.threads, L.smem, s>>>(g, pzp, ctx->pz.tw, pa, A, L.G, L.ls);
  else if (!dir)
    k_zfwd<TD, PRO_SVK, false><<<L.grid, L.threads, L.smem, s>>>(g, pzp, ctx->pz.tw, pa, A, L.G, L.ls);
  else
    k_zfwd<TD, PRO_SVK, true><<<L.grid, L.threads, L.smem, s>>>(g, pzp, ctx->pz.tw, pa, A, L.G, L.ls);
  FM_LAUNCHED_K(ctx, "k_zfwd");
  return FM_OK;
}

template <int TD>
int pass_y(fm_ctx* ctx, const Geo& g, int sign, const double2* in, double2* out) {
  if (g.Ny <= 1 && g.P == 1) return FM_OK;  // length-1 transform, identical layouts
  int st = FM_OK;
  if (TD == 3 && y_fast(ctx, g, sign, in, out, &st)) return st;
  int TW;
  if (tile_width(ctx->nzh, g.Ny, 1, TW, int64_t(g.Nx) * ctx->ncomp))
    return set_error(ctx, FM_E_UNSUPPORTED, "y line too long for the shared-memory FFT");
  const dim3 grid((ctx->nzh + TW - 1) / TW, g.Nx, ctx->ncomp);
  k_ypass<<<grid, 256, size_t(2 * TW + 1) * g.Ny * 16, ctx->stream>>>(g, ctx->py, in, out, TW, sign);
  FM_LAUNCHED_K(ctx, "k_ypass");
  return FM_OK;
}

template <int TD>
int pass_x(fm_ctx* ctx, const Geo& g, double2* T) {
  int st = FM_OK;
  if (TD == 3 && x_fast(ctx, g, T, &st)) return st;
  int TW;
  if (tile_width(ctx->nzh, g.Nx, TD, TW, int64_t(g.Ny) * TD))
    return set_error(ctx, FM_E_UNSUPPORTED, "x line too long for the shared-memory FFT");
  const dim3 grid((ctx->nzh + TW - 1) / TW, g.Ny, TD);
  k_xpass<TD><<<grid, 256, size_t(2 * TD * TW + 1) * g.Nx * 16, ctx->stream>>>(g, ctx->px, T, TW);
  FM_LAUNCHED_K(ctx, "k_xpass");
  return FM_OK;
}

template <int TD>
int pass_zi(fm_ctx* ctx, const Geo& g, const double2* A, double* out, double scale, const EpiArgs& epi,
            int* nparts) {
  int st = FM_OK;
  if (TD == 3 && zi_fast(ctx, g, A, out, scale, epi, &st)) {
    if (nparts) *nparts = ctx->zi_partials;  // partial sums the fast z-inverse wrote
    return st;
  }
  const ZLaunch L = z_launch(ctx, g);
  const AxisPlan& pzp = (ctx->Nz % 2 == 0) ? ctx->pzh : ctx->pz;
  k_zinv<TD><<<L.grid, L.threads, L.smem, ctx->stream>>>(g, pzp, ctx->pz.tw, A, out, L.G, L.ls, scale, epi);
  FM_LAUNCHED_K(ctx, "k_zinv");
  if (nparts) *nparts = int(L.grid.x);
  return FM_OK;
}

// Debug mode: the imaginary residue of the reference's c2c inverse transform
// (projection.cpp:157-169).  With a half spectrum the other half is DEFINED by
// Hermitian symmetry, so the only imaginary output a c2c transform of the same
// data could produce comes from the self-conjugate kz planes (kz = 0, and
// kz = Nz/2 when stored): after the inverse x and y transforms their lines must
// be real, and what pass 5 discards there is Im b(x, y), the same at every z.
// residue^2 = Nz * sum_{c,x,y} Im b^2 / n^2.
__global__ void k_im_residue(const double2* __restrict__ spec, int64_t lines, int nzh, int nyq, double inject,
                             double* __restrict__ sum) {
  double s = 0.0;
  for (int64_t l = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; l < lines; l += int64_t(gridDim.x) * blockDim.x) {
    double im = spec[l * nzh].y;
    if (l == 0) im += inject;  // test hook (FM_DEBUG_RESIDUE_INJECT): a Hermitian violation on purpose
    s += im * im;
    if (nyq > 0) {
      const double in = spec[l * nzh + nyq].y;
      s += in * in;
    }
  }
  s = block_sum_any(s);
  if (threadIdx.x == 0 && s != 0.0) atomicAdd(sum, s);
}

int residue_accumulate(fm_ctx* ctx, int r0, int r1) {
  double* slot = ctx->d_scal + 61;
  FM_CUDA(ctx, cudaMemsetAsync(slot, 0, sizeof(double), ctx->stream));
  const int nyq = (ctx->Nz % 2 == 0 && ctx->nzh == ctx->Nz / 2 + 1) ? ctx->Nz / 2 : 0;
  for (int r = r0; r < r1; ++r) {
    const int64_t lines = int64_t(ctx->ncomp) * (ctx->Nx / ctx->P) * ctx->Ny;
    k_im_residue<<<int(std::min<int64_t>((lines + 255) / 256, 148 * 8)), 256, 0, ctx->stream>>>(
        spec_a(ctx, r), lines, ctx->nzh, nyq, (r == 0 && ctx->rank == 0) ? ctx->debug_inject : 0.0, slot);
    FM_LAUNCHED_K(ctx, "k_im_residue");
  }
  return combine_ranks(ctx, slot, 1);
}

// tolerance 1e-10 ||A|| as the reference for apply_projection; the fused
// operator forms never materialise their A = K : dF, so they use ||G(A)|| <= ||A||.
int residue_check(fm_ctx* ctx, const ProArgs& pa, const double* out, double scale) {
  double s = 0.0, ref = 0.0;
  FM_CUDA(ctx, cudaMemcpyAsync(&s, ctx->d_scal + 61, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  const int64_t count = int64_t(ctx->ncomp) * ctx->n;
  if (int st = norm_sync(ctx, pa.kind == PRO_COPY && pa.A ? pa.A : out, count, &ref)) return st;
  const double residue = std::sqrt(double(ctx->Nz) * s) * std::abs(scale) / double(ctx->n_global);
  const double tol = 1e-10 * std::max(ref, 1e-300);
  if (residue > tol) {
    const int st = set_error(ctx, FM_E_COMPLEX_RESIDUE, "complex residue " + std::to_string(residue) +
                                                            " exceeds tolerance " + std::to_string(tol));
    ctx->last_info = fm_error_info{FM_E_COMPLEX_RESIDUE, 0, -1, residue};
    return st;
  }
  ctx->last_info = fm_error_info{FM_OK, 0, -1, residue};  // the residue of the last checked projection
  return FM_OK;
}

template <int TD>
int run_td(fm_ctx* ctx, const ProArgs& pa, double* out, double scale, const EpiArgs& epi, int* nparts) {
  init_generic<TD>();
  const int r0 = ctx->virt ? 0 : ctx->rank;
  const int r1 = ctx->virt ? ctx->P : ctx->rank + 1;
  const double sc = scale / double(ctx->n_global);
  prof_mark(ctx);
  int pap_total = 0;
  for (int r = r0; r < r1; ++r) {
    ProArgs par = pa;
    if (par.pap_partial) {  // virtual ranks: partials side by side
      const Geo gr = geo_zy(ctx, r);
      const int64_t most = std::max<int64_t>(int64_t(gr.Nx) * gr.Ny, 148 * 32);  // line groups / resident CTAs
      if (pap_total + most > ctx->epi2_cap) return set_error(ctx, FM_E_UNSUPPORTED, "fused CG: too many pass-1 partials");
      par.pap_partial += pap_total;
    }
    if (int st = pass_zf<TD>(ctx, geo_zy(ctx, r), par, spec_a(ctx, r))) return st;
    if (par.pap_partial) pap_total += ctx->zf_partials;
  }
  if (pa.pap_partial)  // fused CG: alpha from <p, K:p> (summed over ranks) before the remaining passes
    if (int st = cg_pap_finalize_from(ctx, pa.pap_partial, pap_total)) return st;
  prof_mark(ctx);
  // P > 1: the forward y pass stores into the ranks' x-pass inputs B, the x
  // pass into the ranks' spectra A (the fused slab transposes, dist.cu)
  // (transpose == 1, the A/B arm: both passes run locally in place and staged
  // all-to-all transposes sit between them, dist_transpose_staged)
  const bool staged = ctx->P > 1 && ctx->transpose == 1;
  auto local = [&](Geo g) {  // the pass's own extents, stores in place
    if (staged) g.P = 1;
    return g;
  };
  for (int r = r0; r < r1; ++r)
    if (int st = pass_y<TD>(ctx, local(geo_zy(ctx, r)), -1, spec_a(ctx, r), spec_a(ctx, r))) return st;
  if (int st = staged ? dist_transpose_staged(ctx, +1) : rank_barrier(ctx)) return st;
  prof_mark(ctx);
  for (int r = r0; r < r1; ++r)
    if (int st = pass_x<TD>(ctx, local(geo_x(ctx, r)), spec_b(ctx, r))) return st;
  if (int st = staged ? dist_transpose_staged(ctx, -1) : rank_barrier(ctx)) return st;
  prof_mark(ctx);
  for (int r = r0; r < r1; ++r)
    if (int st = pass_y<TD>(ctx, geo_zy(ctx, r), +1, spec_a(ctx, r), spec_a(ctx, r))) return st;
  prof_mark(ctx);
  const bool residue = ctx->debug_residue && !ctx->capturing;
  if (residue)
    if (int st = residue_accumulate(ctx, r0, r1)) return st;
  int total = 0;
  for (int r = r0; r < r1; ++r) {
    EpiArgs e = epi;
    if (e.partial) e.partial += total;
    int np = 0;
    if (int st = pass_zi<TD>(ctx, geo_zy(ctx, r), spec_a(ctx, r), out, sc, e, &np)) return st;
    total += np;
  }
  if (nparts) *nparts = total;
  prof_mark(ctx);
  if (ctx->prof.on) ctx->prof.calls++;
  if (residue) return residue_check(ctx, pa, out, scale);
  return FM_OK;
}
}  // namespace

int profile_collect(fm_ctx* ctx) {
  auto& pr = ctx->prof;
  FM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  for (size_t g0 = 0; g0 + kPasses < pr.pending.size(); g0 += kPasses + 1) {
    for (int s = 0; s < kPasses; ++s) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, pr.pending[g0 + s], pr.pending[g0 + s + 1]);
      pr.ms[s] += ms;
    }
  }
  for (cudaEvent_t e : pr.pending) pr.pool.push_back(e);
  pr.pending.clear();
  return FM_OK;
}

bool cg_small_supported(const fm_ctx* ctx) {
  static const int env = [] {
    const char* e = getenv("FM_CG_SMALL");
    return e ? atoi(e) : 1;
  }();
  if (!env || ctx->tdim != 3 || ctx->P != 1 || ctx->virt || ctx->n_global > (int64_t(1) << 20)) return false;
  if (cg_fused_supported(ctx)) return false;  // power-of-two grids run the register-resident passes
  int dev = 0, coop = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  return coop != 0;
}

template <int PRO>
static int cg_small_blocks(size_t smem);

template <int PRO>
static int cg_small_go(fm_ctx* ctx, CgSmallArgs& a, size_t smem, int items_max) {
  const int co = cg_small_blocks<PRO>(smem);  // co-residency bound of the cooperative launch
  if (co < 1) return FM_E_UNSUPPORTED;
  const int grid = std::max(1, std::min(co, items_max));
  void* args[] = {&a};
  const cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_cg_small<PRO>), dim3(grid), dim3(256),
                                                    args, smem, ctx->stream);
  ctx->cnt.launches++;
  ctx->cnt.note("k_cg_small");
  return e == cudaSuccess ? FM_OK : check_cuda(ctx, e, "k_cg_small");
}

template <int PRO>
static int cg_small_blocks(size_t smem) {
  set_smem_limit(reinterpret_cast<const void*>(k_cg_small<PRO>), 200 * 1024);
  int per_sm = 0, dev = 0, sms = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cg_small<PRO>, 256, smem);
  cudaGetLastError();
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return per_sm * sms;
}

int cg_small_run(fm_ctx* ctx, const ProArgs& op, double* x, double* r, double* p, int64_t cap, double thr,
                 double rr0) {
  init_generic<3>();
  const Geo gz = geo_zy(ctx, 0), gx = geo_x(ctx, 0);
  // every phase in ONE round of work items: the co-resident block count
  // (estimated at 64 KB of shared memory) sets the z-line group and the
  // y / x tile widths
  const int blocks0 = op.kind == PRO_K4 ? cg_small_blocks<PRO_K4>(64 * 1024)
                      : op.kind == PRO_J2C ? cg_small_blocks<PRO_J2C>(64 * 1024)
                                           : cg_small_blocks<PRO_SVK>(64 * 1024);
  if (blocks0 < 1) return FM_E_UNSUPPORTED;
  const int nxy = gz.Nx * gz.Ny;
  ZLaunch L = z_launch(ctx, gz);
  L.G = std::max(1, (nxy + blocks0 - 1) / blocks0);
  L.smem = size_t(2) * 9 * L.G * L.ls * 16 + size_t((ctx->Nz % 2 == 0) ? ctx->pzh.N : ctx->pz.N) * 16;
  L.grid = dim3((nxy + L.G - 1) / L.G);
  int twy = 1, twx = 1;
  while (twy < ctx->nzh && int64_t((ctx->nzh + twy - 1) / twy) * gz.Nx * 9 > blocks0) twy *= 2;
  while (twx < ctx->nzh && int64_t((ctx->nzh + twx - 1) / twx) * gx.Ny * 3 > blocks0) twx *= 2;
  CgSmallArgs a;
  a.gz = gz;
  a.gx = gx;
  a.pz = (ctx->Nz % 2 == 0) ? ctx->pzh : ctx->pz;
  a.py = ctx->py;
  a.px = ctx->px;
  a.twN = ctx->pz.tw;
  a.op = op;
  a.spec = spec_a(ctx, 0);
  a.x = x;
  a.r = r;
  a.p = p;
  a.pap_part = ctx->d_epi2;
  a.rr_part = ctx->d_epi;
  a.scal = ctx->d_scal;
  a.G = L.G;
  a.ls = L.ls;
  a.tw_y = twy;
  a.tw_x = twx;
  a.nz_items = int(L.grid.x);
  a.ny_gx = (ctx->nzh + twy - 1) / twy;
  a.ny_items = a.ny_gx * gz.Nx * ctx->ncomp;
  a.nx_gx = (ctx->nzh + twx - 1) / twx;
  a.nx_items = a.nx_gx * gx.Ny * 3;
  a.rr0 = rr0;
  a.thr = thr;
  a.scale = 1.0 / double(ctx->n_global);
  a.cap = cap;
  a.tdbg = nullptr;
  static const bool timing = getenv("FM_CG_SMALL_TIMING") != nullptr;
  static unsigned long long* tdbg = nullptr;
  if (timing) {
    if (!tdbg) cudaMalloc(&tdbg, 64 * sizeof(unsigned long long));
    cudaMemsetAsync(tdbg, 0, 64 * sizeof(unsigned long long), ctx->stream);
    a.tdbg = tdbg;
  }
  const size_t body = std::max({L.smem, size_t(2 * twy + 1) * gz.Ny * 16, size_t(2 * 3 * twx + 1) * gx.Nx * 16});
  a.tw_off = int((body + 15) / 16);
  const size_t smem = size_t(a.tw_off + a.pz.N + a.py.N + a.px.N) * 16;
  const int items = std::max({a.nz_items, a.ny_items, a.nx_items});
  if (smem > size_t(64 * 1024) || a.nz_items > ctx->epi_cap) return FM_E_UNSUPPORTED;
  int st = FM_E_UNSUPPORTED;
  switch (op.kind) {
    case PRO_K4: st = cg_small_go<PRO_K4>(ctx, a, smem, items); break;
    case PRO_J2C: st = cg_small_go<PRO_J2C>(ctx, a, smem, items); break;
    case PRO_SVK: st = cg_small_go<PRO_SVK>(ctx, a, smem, items); break;
    default: break;
  }
  if (timing && st == FM_OK) {
    unsigned long long h[64];
    cudaMemcpyAsync(h, tdbg, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream);
    cudaStreamSynchronize(ctx->stream);
    fprintf(stderr, "cg_small G=%d twy=%d twx=%d items z/y/x=%d/%d/%d:", a.G, a.tw_y, a.tw_x, a.nz_items, a.ny_items,
            a.nx_items);
    for (int i = 1; i < 4; ++i) {
      fprintf(stderr, " [it%d", i + 1);
      for (int k = 1; k < 8; ++k) fprintf(stderr, " %.1f", (h[i * 8 + k] - h[i * 8 + k - 1]) * 1e-3);
      fprintf(stderr, "]");
    }
    fprintf(stderr, "\n");
  }
  return st;
}

int projection_run(fm_ctx* ctx, const ProArgs& pa, double* out, double scale, const EpiArgs& epi,
                   int* n_partials) {
  if (n_partials) *n_partials = 0;
  if (ctx->tdim == 3) return run_td<3>(ctx, pa, out, scale, epi, n_partials);
  return run_td<2>(ctx, pa, out, scale, epi, n_partials);
}

}  // namespace fm
