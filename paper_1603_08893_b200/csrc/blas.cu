// BLAS-1 and reductions over component-major fields (fields.cpp:14-67,
// tensor_ops.cpp:276-294).  Reductions are deterministic: a fixed number of
// blocks (fixed per context) accumulate grid-strided chunks in a fixed order,
// reduce with warp shuffles, and one block sums the partials in a fixed
// order -- byte-identical reruns, as the reference requires
// (test_config_io.cpp:203-229).
#include "fm_internal.cuh"

namespace fm {

constexpr int kRedThreads = 256;

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double wsum[kRedThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) wsum[wid] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int w = 0; w < kRedThreads / 32; ++w) s += wsum[w];
  }
  return s;  // valid in thread 0
}

// Scalar slots in ctx->d_scal used by the CG driver (solver.cu).

__global__ void __launch_bounds__(kRedThreads) k_dot_partial(const double* __restrict__ a,
                                                             const double* __restrict__ b,
                                                             int64_t count, double* partial) {
  double s = 0.0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const int64_t c2 = count / 2;
  const double2* a2 = reinterpret_cast<const double2*>(a);
  const double2* b2 = reinterpret_cast<const double2*>(b);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < c2; i += stride) {
    const double2 x = __ldg(a2 + i), y = __ldg(b2 + i);
    s += x.x * y.x;
    s += x.y * y.y;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (count & 1)) s += a[count - 1] * b[count - 1];
  s = block_sum(s);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// per-component sums: grid (blocks, ncomp)
__global__ void __launch_bounds__(kRedThreads) k_sum_comp_partial(const double* __restrict__ a,
                                                                  int64_t n, double* partial) {
  const double* slab = a + int64_t(blockIdx.y) * n;
  double s = 0.0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += stride)
    s += __ldg(slab + i);
  s = block_sum(s);
  if (threadIdx.x == 0) partial[blockIdx.y * gridDim.x + blockIdx.x] = s;
}

// CG scalar logic on the (globally summed) value s.
__device__ __forceinline__ void cg_scalar_op(double* scal, int op, double s) {
  if (op == 1) {  // solver.cpp:37-45
    scal[S_PAP] = s;
    const bool bad = !(s > 0.0);
    scal[S_FLAG] = bad ? 1.0 : 0.0;
    scal[S_ALPHA] = bad ? 0.0 : scal[S_RR] / s;
  } else if (op == 2) {  // solver.cpp:48-53
    if (scal[S_FLAG] != 0.0) return;
    scal[S_RRNEW] = s;
    scal[S_BETA] = s / scal[S_RR];
    scal[S_RR] = s;
  }
}

// op: 0 -> out[slot + comp] = sum;  1 -> CG pAp step;  2 -> CG rr_new step
__global__ void __launch_bounds__(kRedThreads) k_finalize(const double* __restrict__ partial,
                                                          int nb, double* scal, int op, int slot) {
  const double* p = partial + blockIdx.x * nb;
  double s = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) s += p[i];
  s = block_sum(s);
  if (threadIdx.x != 0) return;
  if (op == 0)
    scal[slot + blockIdx.x] = s;
  else
    cg_scalar_op(scal, op, s);
}

// First level of a two-level finalisation: block b sums partials
// [b*kFold, (b+1)*kFold) in a fixed order (deterministic).
constexpr int kFold = 1024;
__global__ void __launch_bounds__(kRedThreads) k_fold(const double* __restrict__ partial, int nb,
                                                      double* __restrict__ out) {
  const int lo = blockIdx.x * kFold, hi = min(nb, lo + kFold);
  double s = 0.0;
  for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) s += partial[i];
  s = block_sum(s);
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}

// distributed: the CG op applied after the cross-rank combination of scal[slot]
__global__ void k_scalar_op(double* scal, int op, int slot) { cg_scalar_op(scal, op, scal[slot]); }

// x += alpha p; r -= alpha Ap; partial <r,r>   (solver.cpp:46-48)
__global__ void __launch_bounds__(kRedThreads) k_cg_update(double* __restrict__ x,
                                                           double* __restrict__ r,
                                                           const double* __restrict__ p,
                                                           const double* __restrict__ Ap,
                                                           int64_t count, const double* scal,
                                                           double* partial) {
  if (scal[S_FLAG] != 0.0) return;
  const double alpha = scal[S_ALPHA];
  double s = 0.0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const int64_t c2 = count / 2;
  double2* x2 = reinterpret_cast<double2*>(x);
  double2* r2 = reinterpret_cast<double2*>(r);
  const double2* p2 = reinterpret_cast<const double2*>(p);
  const double2* a2 = reinterpret_cast<const double2*>(Ap);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < c2; i += stride) {
    const double2 pv = __ldg(p2 + i), av = __ldg(a2 + i);
    double2 xv = x2[i], rv = r2[i];
    xv.x = __dadd_rn(xv.x, __dmul_rn(alpha, pv.x));
    xv.y = __dadd_rn(xv.y, __dmul_rn(alpha, pv.y));
    rv.x = __dadd_rn(rv.x, __dmul_rn(-alpha, av.x));
    rv.y = __dadd_rn(rv.y, __dmul_rn(-alpha, av.y));
    x2[i] = xv;
    r2[i] = rv;
    s += rv.x * rv.x;
    s += rv.y * rv.y;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (count & 1)) {
    const int64_t i = count - 1;
    x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
    const double ri = __dadd_rn(r[i], __dmul_rn(-alpha, Ap[i]));
    r[i] = ri;
    s += ri * ri;
  }
  s = block_sum(s);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// x += alpha p with the device alpha (the fused CG loop's last update)
__global__ void k_cg_xfinal(double* __restrict__ x, const double* __restrict__ p, int64_t count,
                            const double* scal) {
  const double alpha = scal[S_ALPHA];
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count; i += stride)
    x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
}

// p = beta p + r   (solver.cpp:51-55, p *= beta; p += r)
__global__ void k_cg_direction(double* __restrict__ p, const double* __restrict__ r,
                               int64_t count, const double* scal) {
  const double beta = scal[S_BETA];
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count; i += stride)
    p[i] = __dadd_rn(__dmul_rn(p[i], beta), r[i]);
}

__global__ void k_axpy(double a, const double* __restrict__ x, double* __restrict__ y, int64_t count) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count; i += stride)
    y[i] = __dadd_rn(y[i], __dmul_rn(a, x[i]));
}

__global__ void k_scale(double* x, double s, int64_t count) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count; i += stride)
    x[i] *= s;
}

__global__ void k_add(double* __restrict__ y, const double* __restrict__ x, double sign, int64_t count) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count; i += stride)
    y[i] = sign > 0 ? y[i] + x[i] : y[i] - x[i];
}

struct Uni {
  double t[9];
};

__global__ void k_uniform(double* f, Uni u, int ncomp, int64_t n, int add) {
  const int64_t count = n * ncomp;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count; i += stride) {
    const double v = u.t[i / n];
    f[i] = add ? f[i] + v : 0.0 + v;
  }
}

// ---------------------------------------------------------------- host side
static int ew_blocks(int64_t count) {
  const int64_t b = (count + 255) / 256;
  return int(b < 148 * 16 ? (b < 1 ? 1 : b) : 148 * 16);
}

// Finalise a reduction whose block partials are in `partial`: op 0 stores the
// sum in scal[slot]; op 1/2 run the CG scalar step on it.  Distributed: the
// local sum is combined across ranks (ordered) before the op is applied.
static int finalize(fm_ctx* ctx, const double* partial, int nb, double* scal, int op, int slot) {
  if (nb > 2 * kFold) {  // one block over 65536 partials costs ~60 us: fold first
    const int nf = (nb + kFold - 1) / kFold;
    k_fold<<<nf, kRedThreads, 0, ctx->stream>>>(partial, nb, ctx->d_fold);
    FM_LAUNCHED_K(ctx, "k_fold");
    partial = ctx->d_fold;
    nb = nf;
  }
  if (!distributed(ctx) || op == 0) {
    k_finalize<<<1, kRedThreads, 0, ctx->stream>>>(partial, nb, scal, op, slot);
    FM_LAUNCHED_K(ctx, "k_finalize");
    return op == 0 ? combine_ranks(ctx, scal + slot, 1) : FM_OK;
  }
  constexpr int kLocal = 40;  // scratch slot for the local value
  k_finalize<<<1, kRedThreads, 0, ctx->stream>>>(partial, nb, scal, 0, kLocal);
  FM_LAUNCHED_K(ctx, "k_finalize");
  if (int st = combine_ranks(ctx, scal + kLocal, 1)) return st;
  k_scalar_op<<<1, 1, 0, ctx->stream>>>(scal, op, kLocal);
  FM_LAUNCHED_K(ctx, "k_scalar_op");
  return FM_OK;
}

int dot_async(fm_ctx* ctx, const double* a, const double* b, int64_t count, double* d_out) {
  k_dot_partial<<<ctx->red_blocks, kRedThreads, 0, ctx->stream>>>(a, b, count, ctx->d_partial);
  FM_LAUNCHED_K(ctx, "k_dot_partial");
  return finalize(ctx, ctx->d_partial, ctx->red_blocks, d_out, 0, 0);
}

int sum_comp_async(fm_ctx* ctx, const double* a, int ncomp, int64_t n, double* d_out) {
  const int nb = ctx->red_blocks / 16 > 0 ? ctx->red_blocks / 16 : 1;
  k_sum_comp_partial<<<dim3(nb, ncomp), kRedThreads, 0, ctx->stream>>>(a, n, ctx->d_partial);
  FM_LAUNCHED_K(ctx, "k_sum_comp_partial");
  k_finalize<<<ncomp, kRedThreads, 0, ctx->stream>>>(ctx->d_partial, nb, d_out, 0, 0);
  FM_LAUNCHED_K(ctx, "k_finalize");
  return combine_ranks(ctx, d_out, ncomp);
}

int axpy_async(fm_ctx* ctx, double a, const double* x, double* y, int64_t count) {
  k_axpy<<<ew_blocks(count), 256, 0, ctx->stream>>>(a, x, y, count);
  FM_LAUNCHED_K(ctx, "k_axpy");
  return FM_OK;
}

int scale_async(fm_ctx* ctx, double* x, double s, int64_t count) {
  k_scale<<<ew_blocks(count), 256, 0, ctx->stream>>>(x, s, count);
  FM_LAUNCHED_K(ctx, "k_scale");
  return FM_OK;
}

int add_async(fm_ctx* ctx, double* y, const double* x, double sign, int64_t count) {
  k_add<<<ew_blocks(count), 256, 0, ctx->stream>>>(y, x, sign, count);
  FM_LAUNCHED_K(ctx, "k_add");
  return FM_OK;
}

static int uniform_async(fm_ctx* ctx, double* f, const double* t, int ncomp, int64_t n, int add) {
  Uni u{};
  for (int c = 0; c < ncomp && c < 9; ++c) u.t[c] = t[c];
  k_uniform<<<ew_blocks(n * ncomp), 256, 0, ctx->stream>>>(f, u, ncomp, n, add);
  FM_LAUNCHED_K(ctx, "k_uniform");
  return FM_OK;
}
int add_uniform_async(fm_ctx* ctx, double* f, const double* t, int ncomp, int64_t n) {
  return uniform_async(ctx, f, t, ncomp, n, 1);
}
int fill_uniform_async(fm_ctx* ctx, double* f, const double* t, int ncomp, int64_t n) {
  return uniform_async(ctx, f, t, ncomp, n, 0);
}

int fetch_scalars(fm_ctx* ctx, int count) {
  FM_CUDA(ctx, cudaMemcpyAsync(ctx->h_scal, ctx->d_scal, sizeof(double) * count,
                               cudaMemcpyDeviceToHost, ctx->stream));
  FM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return FM_OK;
}

int cg_update_async(fm_ctx* ctx, double* x, double* r, const double* p, const double* Ap,
                    int64_t count) {
  k_cg_update<<<ctx->red_blocks, kRedThreads, 0, ctx->stream>>>(x, r, p, Ap, count, ctx->d_scal,
                                                                ctx->d_partial);
  FM_LAUNCHED_K(ctx, "k_cg_update");
  return finalize(ctx, ctx->d_partial, ctx->red_blocks, ctx->d_scal, 2, 0);
}

int cg_final_x_async(fm_ctx* ctx, double* x, const double* p, int64_t count) {
  k_cg_xfinal<<<ew_blocks(count), 256, 0, ctx->stream>>>(x, p, count, ctx->d_scal);
  FM_LAUNCHED_K(ctx, "k_cg_xfinal");
  return FM_OK;
}

int cg_direction_async(fm_ctx* ctx, double* p, const double* r, int64_t count) {
  k_cg_direction<<<ew_blocks(count), 256, 0, ctx->stream>>>(p, r, count, ctx->d_scal);
  FM_LAUNCHED_K(ctx, "k_cg_direction");
  return FM_OK;
}

// alpha / curvature flag from arbitrary per-block partials of <p, Ap>
int cg_pap_finalize_from(fm_ctx* ctx, const double* partials, int n) {
  return finalize(ctx, partials, n, ctx->d_scal, 1, 0);
}
// beta / rr from per-block partials of <r, r> (fused z-inverse update)
int cg_rr_finalize_from(fm_ctx* ctx, const double* partials, int n) {
  return finalize(ctx, partials, n, ctx->d_scal, 2, 0);
}

// <p,Ap> from the partials the fused z-inverse epilogue wrote (solver.cpp:37-45)
int cg_pap_finalize_async(fm_ctx* ctx, int n_partials) {
  return finalize(ctx, ctx->d_epi, n_partials, ctx->d_scal, 1, 0);
}

// pAp finalisation used by the CG driver
int cg_pap_async(fm_ctx* ctx, const double* p, const double* Ap, int64_t count) {
  k_dot_partial<<<ctx->red_blocks, kRedThreads, 0, ctx->stream>>>(p, Ap, count, ctx->d_partial);
  FM_LAUNCHED_K(ctx, "k_dot_partial");
  return finalize(ctx, ctx->d_partial, ctx->red_blocks, ctx->d_scal, 1, 0);
}

}  // namespace fm
