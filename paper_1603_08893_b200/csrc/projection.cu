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

#include "proj_common.cuh"

namespace fm {

// ------------------------------------------------------------------ pass 1
template <int TD, int PRO, bool DIR>
__global__ void __launch_bounds__(256) k_zfwd(Geo g, AxisPlan plan, const double2* __restrict__ twN,
                                              ProArgs pa, double2* __restrict__ spec, int G, int ls) {
  extern __shared__ double2 sm[];
  constexpr int NC = TD * TD;
  const int nxy = g.Nx * g.Ny;
  const int L0 = blockIdx.x * G;
  const int Gb = min(G, nxy - L0);
  double2* A = sm;
  double2* B = sm + NC * G * ls;
  const bool even = (g.Nz % 2 == 0);
  for (int w = threadIdx.x; w < Gb * g.Nz; w += blockDim.x) {
    const int gi = w / g.Nz, z = w - gi * g.Nz;
    const int64_t node = g.roff + int64_t(L0 + gi) * g.Nz + z;
    double v[NC];
    prologue_voxel<TD, PRO, DIR>(pa, g.n, node, v);
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
  double2* R = fft_smem(A, B, NC * G, ls, 1, plan, -1, false, sm + 2 * NC * G * ls);
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
}

// -------------------------------------------------------------- pass 2 / 4
// sign -1: std in -> packed out (forward); +1: packed in -> std out.
__global__ void __launch_bounds__(256) k_ypass(Geo g, AxisPlan plan, const double2* in,
                                               double2* out, int TW, int sign) {  // in == out when P = 1
  extern __shared__ double2 sm[];
  const int kz0 = blockIdx.x * TW;
  const int x = blockIdx.y, c = blockIdx.z, NC = gridDim.z;
  const int Ny = g.Ny;
  double2* A = sm;
  double2* B = sm + Ny * TW;
  for (int w = threadIdx.x; w < Ny * TW; w += blockDim.x) {
    const int e = w / TW, t = w - e * TW;
    const int kz = kz0 + t;
    if (kz < g.nzh)
      A[w] = in[sign < 0 ? spec_std(g, c, x, e, kz) : spec_packed(g, NC, c, x, e, kz)];
    else
      A[w] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  double2* R = fft_smem(A, B, TW, 1, TW, plan, sign, true, sm + 2 * Ny * TW);
  for (int w = threadIdx.x; w < Ny * TW; w += blockDim.x) {
    const int e = w / TW, t = w - e * TW;
    const int kz = kz0 + t;
    if (kz < g.nzh) out[sign < 0 ? spec_packed(g, NC, c, x, e, kz) : spec_std(g, c, x, e, kz)] = R[w];
  }
}

// ------------------------------------------------------------------ pass 3
template <int TD>
__global__ void __launch_bounds__(256) k_xpass(Geo g, AxisPlan plan, double2* __restrict__ spec,
                                               int TW) {
  extern __shared__ double2 sm[];
  const int kz0 = blockIdx.x * TW;
  const int y = blockIdx.y, i = blockIdx.z;
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
  double2* R = fft_smem(A, B, nl, 1, nl, plan, -1, true, sm + 2 * Nx * nl);
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
  R = fft_smem(R, S, nl, 1, nl, plan, +1, true, sm + 2 * Nx * nl);
  for (int w = threadIdx.x; w < Nx * nl; w += blockDim.x) {
    const int t = w % TW, j = (w / TW) % TD, e = w / nl;
    const int kz = kz0 + t;
    if (kz < g.nzh)
      spec[(int64_t(i * TD + j) * Nx + e) * xstride + int64_t(y) * g.nzh + kz] = R[w];
  }
}

// ------------------------------------------------------------------ pass 5
template <int TD>
__global__ void __launch_bounds__(256) k_zinv(Geo g, AxisPlan plan, const double2* __restrict__ twN,
                                              const double2* __restrict__ spec,
                                              double* __restrict__ out, int G, int ls,
                                              double scale, EpiArgs epi) {
  extern __shared__ double2 sm[];
  constexpr int NC = TD * TD;
  const int nxy = g.Nx * g.Ny;
  const int L0 = blockIdx.x * G;
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
  double2* R = fft_smem(B, A, NC * G, ls, 1, plan, +1, false, sm + 2 * NC * G * ls);
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
    out[idx] = v * scale;
    if (epi.partial) dot += __ldg(epi.pdot + idx) * (v * scale);
  }
  if (epi.partial) {
    dot = block_sum_any(dot);
    if (threadIdx.x == 0) epi.partial[blockIdx.x] = dot;
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
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       kMaxSmem - int(attr.sharedSizeBytes));
  cudaGetLastError();  // attribute calls must not leave a sticky launch error behind
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
void init_generic() {
  static bool init = false;
  if (init) return;
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
  init = true;
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
  FM_LAUNCHED(ctx);
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
  FM_LAUNCHED(ctx);
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
  FM_LAUNCHED(ctx);
  return FM_OK;
}

template <int TD>
int pass_zi(fm_ctx* ctx, const Geo& g, const double2* A, double* out, double scale, const EpiArgs& epi,
            int* nparts) {
  int st = FM_OK;
  if (TD == 3 && zi_fast(ctx, g, A, out, scale, epi, &st)) {
    if (nparts) *nparts = zi_fast_blocks(ctx, g);
    return st;
  }
  const ZLaunch L = z_launch(ctx, g);
  const AxisPlan& pzp = (ctx->Nz % 2 == 0) ? ctx->pzh : ctx->pz;
  k_zinv<TD><<<L.grid, L.threads, L.smem, ctx->stream>>>(g, pzp, ctx->pz.tw, A, out, L.G, L.ls, scale, epi);
  FM_LAUNCHED(ctx);
  if (nparts) *nparts = int(L.grid.x);
  return FM_OK;
}

template <int TD>
int run_td(fm_ctx* ctx, const ProArgs& pa, double* out, double scale, const EpiArgs& epi, int* nparts) {
  init_generic<TD>();
  const int r0 = ctx->virt ? 0 : ctx->rank;
  const int r1 = ctx->virt ? ctx->P : ctx->rank + 1;
  const double sc = scale / double(ctx->n_global);
  prof_mark(ctx);
  for (int r = r0; r < r1; ++r)
    if (int st = pass_zf<TD>(ctx, geo_zy(ctx, r), pa, spec_a(ctx, r))) return st;
  if (pa.pap_partial)  // fused CG: alpha from <p, K:p> before the remaining passes
    if (int st = cg_pap_finalize_from(ctx, pa.pap_partial, ctx->zf_partials)) return st;
  prof_mark(ctx);
  for (int r = r0; r < r1; ++r)
    if (int st = pass_y<TD>(ctx, geo_zy(ctx, r), -1, spec_a(ctx, r), spec_b(ctx, r))) return st;
  prof_mark(ctx);
  if (ctx->P > 1)
    if (int st = transpose(ctx, +1)) return st;
  for (int r = r0; r < r1; ++r)
    if (int st = pass_x<TD>(ctx, geo_x(ctx, r), spec_a(ctx, r))) return st;
  if (ctx->P > 1)
    if (int st = transpose(ctx, -1)) return st;
  prof_mark(ctx);
  for (int r = r0; r < r1; ++r)
    if (int st = pass_y<TD>(ctx, geo_zy(ctx, r), +1, spec_b(ctx, r), spec_a(ctx, r))) return st;
  prof_mark(ctx);
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

int projection_run(fm_ctx* ctx, const ProArgs& pa, double* out, double scale, const EpiArgs& epi,
                   int* n_partials) {
  if (n_partials) *n_partials = 0;
  if (ctx->tdim == 3) return run_td<3>(ctx, pa, out, scale, epi, n_partials);
  return run_td<2>(ctx, pa, out, scale, epi, n_partials);
}

}  // namespace fm
