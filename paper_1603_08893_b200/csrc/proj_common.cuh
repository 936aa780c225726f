// Shared pieces of the projection passes (generic and register-resident).
#pragma once

#include "fft_reg.cuh"
#include "reduce.cuh"

namespace fm {

// Geometry one pass sees.  Single device: the whole grid.  Slab rank r of P
// (SURVEY.md §8(e)): z / y passes see the x-slab (Nx = Nx_global / P, all y,
// all z); the x pass sees all x for its y-slab (Ny = Ny_global / P, y0 = r Ny).
struct Geo {
  int Nx, Ny, Nz, nzh, Lz, dim, mode;
  int64_t n;     // component stride of real fields
  int64_t roff;  // node offset of this slab inside the real fields
  double invL[3];
  int P, Yl;     // ranks, y per rank
  int y0, Nyg;   // x pass: global y of local y = 0, global Ny (frequencies)
  int rank, Xl, Nxg;  // slab rank of this pass, x per rank, global Nx
  // P > 1: the slab transpose is fused into the forward y pass and the x pass,
  // which store each element straight into the buffer of the rank that owns
  // it next (device array of P pointers: peer memory over NVLink when the
  // ranks are devices, the side-by-side rank buffers in the virtual mode)
  double2* const* dst;
};

// Spectral layout of every pass: std [c][x][y][kz] on the pass's own extents.
__device__ __forceinline__ int64_t spec_std(const Geo& g, int c, int x, int y, int kz) {
  return ((int64_t(c) * g.Nx + x) * g.Ny + y) * g.nzh + kz;
}

// Routes of the fused slab transpose (shared by the kernels and fm_dist_route).
// Forward, epilogue of the y pass on the x-slab of rank s: element
// (c, xl, y, kz) goes to rank d = y / Yl, into its x-pass input B_d =
// [c][x = s Xl + xl][yl][kz] (all x, the y-slab of d).
__host__ __device__ __forceinline__ int64_t route_yf(int Nxg, int Xl, int Yl, int nzh, int s, int c, int xl, int y,
                                                     int kz, int& d) {
  d = y / Yl;
  const int yl = y - d * Yl;
  return ((int64_t(c) * Nxg + int64_t(s) * Xl + xl) * Yl + yl) * nzh + kz;
}
// Backward, epilogue of the x pass on the y-slab of rank d: element
// (c, x, yl, kz) goes to rank s = x / Xl, into its spectrum A_s =
// [c][xl][y = d Yl + yl][kz] (the x-slab of s, all y), where the inverse y
// pass continues in place.
__host__ __device__ __forceinline__ int64_t route_xb(int Nyg, int Xl, int Yl, int nzh, int d, int c, int x, int yl,
                                                     int kz, int& s) {
  s = x / Xl;
  const int xl = x - s * Xl;
  return ((int64_t(c) * Xl + xl) * Nyg + int64_t(d) * Yl + yl) * nzh + kz;
}
// Store of the forward y pass: in place on one device, routed when P > 1.
__device__ __forceinline__ void store_yf(const Geo& g, double2* out, int c, int x, int y, int kz, double2 v) {
  if (g.P == 1) {
    out[spec_std(g, c, x, y, kz)] = v;
  } else {
    int d;
    const int64_t o = route_yf(g.Nxg, g.Nx, g.Yl, g.nzh, g.rank, c, x, y, kz, d);
    g.dst[d][o] = v;
  }
}
// Store of the x pass: in place on one device (`local` = the element's
// address), routed to the owning x-slab when P > 1.
__device__ __forceinline__ void store_xb(const Geo& g, double2* local, int c, int x, int y, int kz, double2 v) {
  if (g.P == 1) {
    *local = v;
  } else {
    int s;
    const int64_t o = route_xb(g.Nyg, g.Xl, g.Ny, g.nzh, g.rank, c, x, y, kz, s);
    g.dst[s][o] = v;
  }
}

// The same store for the register-resident passes, whose extents are powers of
// two (Xl = 2^sh): the owner and the local x are a shift and a mask, and the
// per-line part of route_xb, base = ((c Xl) Nyg + rank Yl + yl) nzh + kz, is
// computed once per line instead of per element.
__device__ __forceinline__ int64_t xb_base(const Geo& g, int c, int yl, int kz) {
  return ((int64_t(c) * g.Xl) * g.Nyg + int64_t(g.rank) * g.Ny + yl) * g.nzh + kz;
}
__device__ __forceinline__ void store_xb_pow2(const Geo& g, int sh, int64_t base, int x, double2 v) {
  g.dst[x >> sh][base + int64_t(x & (g.Xl - 1)) * g.Nyg * g.nzh] = v;
}

__device__ __forceinline__ int freq_of(int i, int n) { return (i < (n + 1) / 2) ? i : i - n; }

// ------------------------------------------------------------------ pass 1
// dF of one voxel: either read, or (fused CG direction) p = beta p + r.
// The new p is only formed here; store_dir() writes it back after every load
// of the voxel has been issued (a store before the K4 loads would, through
// possible aliasing, serialise them).
template <int NC, bool DIR>
__device__ __forceinline__ void load_dF(const ProArgs& pa, int64_t n, int64_t node, double* d) {
  if constexpr (DIR) {
    const double beta = *pa.beta;
#pragma unroll
    for (int c = 0; c < NC; ++c)
      d[c] = __dadd_rn(__dmul_rn(__ldg(pa.p + c * n + node), beta), __ldg(pa.r + c * n + node));
  } else {
#pragma unroll
    for (int c = 0; c < NC; ++c) d[c] = __ldg(pa.A + c * n + node);
  }
}
template <int NC, bool DIR>
__device__ __forceinline__ void store_dir(const ProArgs& pa, int64_t n, int64_t node, const double* d) {
  if constexpr (DIR) {
#pragma unroll
    for (int c = 0; c < NC; ++c) pa.p[c * n + node] = d[c];
  }
}

// SVK tangent action of one voxel (hyperelastic.cpp:55-63 contracted
// analytically): dP = lam tr(F^T dF) F + mu F dF^T F + mu F F^T dF + dF S,
// S = lam tr(E) I + 2 mu E, E = (F^T F - I) / 2.  With A = F^T dF the two mu
// terms are mu F (A + A^T) and tr(F^T dF) = tr A, which halves the fp64 work
// (~140 operations per voxel).  Shared by every kernel that forms the action
// so that all of them round identically.
template <int TD>
__device__ __forceinline__ void svk_action(const double* f, const double* d, double lam, double mu, double* v) {
  double A[TD * TD], C[TD * TD];
#pragma unroll
  for (int i = 0; i < TD; ++i)
#pragma unroll
    for (int j = 0; j < TD; ++j) {
      double a = 0.0;
#pragma unroll
      for (int k = 0; k < TD; ++k) a = fma(f[k * TD + i], d[k * TD + j], a);  // (F^T dF)_ij
      A[i * TD + j] = a;
    }
#pragma unroll
  for (int i = 0; i < TD; ++i)
#pragma unroll
    for (int j = i; j < TD; ++j) {
      double c = 0.0;
#pragma unroll
      for (int k = 0; k < TD; ++k) c = fma(f[k * TD + i], f[k * TD + j], c);  // (F^T F)_ij
      C[i * TD + j] = c;
      C[j * TD + i] = c;
    }
  double trA = 0.0, trE = 0.0;
#pragma unroll
  for (int i = 0; i < TD; ++i) {
    trA += A[i * TD + i];
    trE += 0.5 * (C[i * TD + i] - 1.0);
  }
  // B = mu (A + A^T), S = 2 mu E + lam tr(E) I (both symmetric)
  double B[TD * TD], S[TD * TD];
#pragma unroll
  for (int i = 0; i < TD; ++i)
#pragma unroll
    for (int j = i; j < TD; ++j) {
      const double bij = mu * (A[i * TD + j] + A[j * TD + i]);
      const double sij = (i == j) ? fma(mu, C[i * TD + i] - 1.0, lam * trE) : mu * C[i * TD + j];
      B[i * TD + j] = B[j * TD + i] = bij;
      S[i * TD + j] = S[j * TD + i] = sij;
    }
  const double lt = lam * trA;
#pragma unroll
  for (int i = 0; i < TD; ++i)
#pragma unroll
    for (int j = 0; j < TD; ++j) {
      double a = lt * f[i * TD + j];
#pragma unroll
      for (int k = 0; k < TD; ++k) {
        a = fma(f[i * TD + k], B[k * TD + j], a);  // mu F (A + A^T)
        a = fma(d[i * TD + k], S[k * TD + j], a);  // dF S
      }
      v[i * TD + j] = a;
    }
}

// PAP: also accumulate <dF, dP> of the voxel into *pap (fused CG curvature).
template <int TD, int PRO, bool DIR = false, bool PAP = false>
__device__ __forceinline__ void prologue_voxel(const ProArgs& pa, int64_t n, int64_t node,
                                               double v[TD * TD], double* pap = nullptr) {
  constexpr int NC = TD * TD;
  if (PRO == PRO_COPY) {
#pragma unroll
    for (int c = 0; c < NC; ++c) v[c] = __ldg(pa.A + c * n + node);
  } else if (PRO == PRO_K4) {
    // dP_ij = K_jikl dF_kl (projection.cpp:184)
    double df[NC];
    load_dF<NC, DIR>(pa, n, node, df);
#pragma unroll
    for (int i = 0; i < TD; ++i)
#pragma unroll
      for (int j = 0; j < TD; ++j) {
        double s = 0.0;
#pragma unroll
        for (int kl = 0; kl < NC; ++kl) s += __ldg(pa.K + ((j * TD + i) * NC + kl) * n + node) * df[kl];
        v[i * TD + j] = s;
      }
    if constexpr (PAP) {
#pragma unroll
      for (int c = 0; c < NC; ++c) *pap += df[c] * v[c];
    }
    store_dir<NC, DIR>(pa, n, node, df);
  } else if (PRO == PRO_J2C) {
    // Compact J2 tangent action (constitutive.cu, simo.cpp:131-194 in the
    // eigenbasis): D = V^T dF U, W_qp = b_pq D_pq + c_pq D_qp + d_pq sum_r a_pr D_rr,
    // dP = V W U^T  (== K_jikl dF_kl of the assembled K4).
    if constexpr (TD == 3) {
      double d[9];
      load_dF<9, DIR>(pa, n, node, d);
      double V[9], U[9], D[9], T[9];
#pragma unroll
      for (int e = 0; e < 9; ++e) {
        V[e] = __ldg(pa.K + (0 + e) * n + node);
        U[e] = __ldg(pa.K + (9 + e) * n + node);
      }
#pragma unroll
      for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int b = 0; b < 3; ++b)
          T[k * 3 + b] = d[k * 3 + 0] * U[0 * 3 + b] + d[k * 3 + 1] * U[1 * 3 + b] + d[k * 3 + 2] * U[2 * 3 + b];
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
          D[a * 3 + b] = V[0 * 3 + a] * T[0 * 3 + b] + V[1 * 3 + a] * T[1 * 3 + b] + V[2 * 3 + a] * T[2 * 3 + b];
      double W[9];
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        double ap = 0.0;
#pragma unroll
        for (int r = 0; r < 3; ++r) ap += __ldg(pa.K + (18 + p * 3 + r) * n + node) * D[r * 3 + r];
#pragma unroll
        for (int qq = 0; qq < 3; ++qq)
          W[qq * 3 + p] = __ldg(pa.K + (27 + p * 3 + qq) * n + node) * D[p * 3 + qq] +
                          __ldg(pa.K + (36 + p * 3 + qq) * n + node) * D[qq * 3 + p] + (p == qq ? ap : 0.0);
      }
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int p = 0; p < 3; ++p)
          T[i * 3 + p] = V[i * 3 + 0] * W[0 * 3 + p] + V[i * 3 + 1] * W[1 * 3 + p] + V[i * 3 + 2] * W[2 * 3 + p];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
          v[i * 3 + j] = T[i * 3 + 0] * U[j * 3 + 0] + T[i * 3 + 1] * U[j * 3 + 1] + T[i * 3 + 2] * U[j * 3 + 2];
      if constexpr (PAP) {
#pragma unroll
        for (int c = 0; c < 9; ++c) *pap += d[c] * v[c];
      }
      store_dir<9, DIR>(pa, n, node, d);
    }
  } else {
    // SVK tangent action (hyperelastic.cpp:55-63 contracted analytically)
    double f[NC], d[NC];
    load_dF<NC, DIR>(pa, n, node, d);
#pragma unroll
    for (int c = 0; c < NC; ++c) f[c] = __ldg(pa.F + c * n + node);
    svk_action<TD>(f, d, __ldg(pa.lam + node), __ldg(pa.mu + node), v);
    if constexpr (PAP) {
#pragma unroll
      for (int c = 0; c < NC; ++c) *pap += d[c] * v[c];
    }
    store_dir<NC, DIR>(pa, n, node, d);
  }
}

inline Geo make_geo(const fm_ctx* ctx) {
  Geo g;
  g.Nx = ctx->Nx;
  g.Ny = ctx->Ny;
  g.Nz = ctx->Nz;
  g.nzh = ctx->nzh;
  g.Lz = ctx->Lz;
  g.dim = ctx->dim;
  g.mode = ctx->mode;
  g.n = ctx->n;
  g.roff = 0;
  for (int a = 0; a < 3; ++a) g.invL[a] = 1.0 / ctx->len[a];
  g.P = 1;
  g.Yl = ctx->Ny;
  g.y0 = 0;
  g.Nyg = ctx->Ny;
  g.rank = 0;
  g.Xl = ctx->Nx;
  g.Nxg = ctx->Nx;
  g.dst = nullptr;
  return g;
}
// z and y passes of slab rank r: local x-slab, all y and z.  The forward y
// pass stores into the x-pass inputs B of the destination ranks.
inline Geo geo_zy(const fm_ctx* ctx, int r) {
  Geo g = make_geo(ctx);
  g.P = ctx->P;
  g.Nx = ctx->Nx / ctx->P;
  g.Xl = g.Nx;
  g.Yl = ctx->Ny / ctx->P;
  g.rank = r;
  g.roff = ctx->virt ? int64_t(r) * g.Nx * ctx->Ny * ctx->Nz : 0;
  g.n = ctx->n_local_stride;
  g.dst = ctx->d_dst_b;
  return g;
}
// Spectral buffers of slab rank r: A (z / y side, std layout on the x-slab)
// and B (the x-pass input, std layout on the y-slab), one rank per device
// when distributed, all P ranks side by side in the virtual mode.  P = 1:
// B == A (every pass runs in place).
inline double2* spec_a(fm_ctx* ctx, int r) {
  return ctx->spec + (ctx->virt ? int64_t(r) * ctx->spec_rank_elems : 0);
}
inline double2* spec_b(fm_ctx* ctx, int r) {
  if (ctx->P == 1) return ctx->spec;
  return ctx->spec2 + (ctx->virt ? int64_t(r) * ctx->spec_rank_elems : 0);
}
// x pass of slab rank r: all x, local y-slab; stores into the spectra A of
// the x-slab owners.
inline Geo geo_x(const fm_ctx* ctx, int r) {
  Geo g = make_geo(ctx);
  g.P = ctx->P;
  g.Ny = ctx->Ny / ctx->P;
  g.Yl = g.Ny;
  g.Xl = ctx->Nx / ctx->P;
  g.y0 = r * g.Ny;
  g.rank = r;
  g.dst = ctx->d_dst_a;
  return g;
}


// Pass launchers of the register-resident path (projection_fast.cu); each
// returns true when it launched (false: no fast kernel for this shape).
bool zf_fast(fm_ctx* ctx, const Geo& g, const ProArgs& pa, double2* spec, int* st);
bool y_fast(fm_ctx* ctx, const Geo& g, int sign, const double2* in, double2* out, int* st);
bool x_fast(fm_ctx* ctx, const Geo& g, double2* spec, int* st);
bool zi_fast(fm_ctx* ctx, const Geo& g, const double2* spec, double* out, double scale, const EpiArgs& epi,
             int* st);
// Cached CUtensorMap (written to out_map) of a spectral buffer viewed as
// [rows][Ny][2 nzh] doubles with a (2 TW, 1, box_rows) box (projection_fast.cu).
// split2: rows viewed as [rows / 2][2]: the even and the odd rows are separate boxes (4-D map).
bool x_tensor_map(const void* base, int rows, int Ny, int nzh, int TW, bool swz128, int box_rows, void* out_map,
                  bool split2 = false);
bool tensor_map_encode(const void* base, int rank, const uint64_t* dims, const uint64_t* strides, const uint32_t* box,
                       bool swz128, void* out_map);
// 1024-point y pass in place, the line split over a 2-CTA cluster (projection_xw.cu).
bool yw_launch(fm_ctx* ctx, const Geo& g, int sign, double2* spec);
// 512-point x pass, one warp per line, TMA in and out (projection_xw.cu).
bool xw_launch(fm_ctx* ctx, const Geo& g, double2* spec, int dbg);

}  // namespace fm
