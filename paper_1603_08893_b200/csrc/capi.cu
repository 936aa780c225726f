// extern "C" boundary of libfftmech_b200.so (include/fftmech_b200.h).
// Every entry point validates its arguments the way the reference does
// (std::invalid_argument -> FM_E_INVALID) and returns an fm_status; there
// is no CPU fallback anywhere behind it.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include "fm_internal.cuh"

namespace fm {

int set_error(fm_ctx* ctx, int status, const std::string& msg) {
  if (ctx) {
    ctx->last_error = msg;
    ctx->last_info = fm_error_info{status, 0, -1, 0.0};
  }
  return status;
}

int check_cuda(fm_ctx* ctx, cudaError_t e, const char* what) {
  const int st = e == cudaErrorMemoryAllocation ? FM_E_OOM : FM_E_CUDA;
  return set_error(ctx, st, std::string(what) + ": " + cudaGetErrorString(e));
}

int ensure_field(fm_ctx* ctx, fm_field& f, int ncomp) {
  if (f.d && f.ncomp == ncomp) return FM_OK;
  if (f.d) cudaFree(f.d);
  f.d = nullptr;
  f.ncomp = ncomp;
  f.n = ctx->n;
  FM_CUDA(ctx, cudaMalloc(&f.d, sizeof(double) * size_t(ncomp) * size_t(ctx->n)));
  return FM_OK;
}

void set_smem_limit(const void* kernel, int bytes) {
  static std::mutex mx;
  static std::vector<std::pair<std::pair<int, const void*>, int>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mx);
  for (auto& d : done)
    if (d.first.first == dev && d.first.second == kernel) {
      if (d.second >= bytes) return;
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
      cudaGetLastError();
      d.second = bytes;
      return;
    }
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaGetLastError();  // attribute calls must not leave a sticky launch error behind
  done.push_back({{dev, kernel}, bytes});
}

void release_field(fm_field& f) {
  if (f.d) cudaFree(f.d);
  f = fm_field{};
}

// Radix plan: 4s, then 2, then odd primes ascending (any leftover prime is
// one direct stage) -- the generic Stockham engine takes any radix.
static void make_plan(AxisPlan& p, int N) {
  p.N = N;
  p.nst = 0;
  int m = N;
  while (m % 4 == 0 && p.nst < kMaxStages) { p.radix[p.nst++] = 4; m /= 4; }
  while (m % 2 == 0 && p.nst < kMaxStages) { p.radix[p.nst++] = 2; m /= 2; }
  for (int f = 3; f * f <= m; f += 2)
    while (m % f == 0 && p.nst < kMaxStages) { p.radix[p.nst++] = f; m /= f; }
  if (m > 1) p.radix[p.nst++] = m;
}

// exp(-2 pi i k / N), exact at the octant points: the angle is reduced to
// [0, pi/4] and mapped back with exact sign/swap rules, so W^{N/4} = -i,
// W^{N/2} = -1 and W^{N/8} = (s, -s) with s = sqrt(1/2) exactly once rounded.
static double2 unit_root(long long k, long long N) {
  k %= N;
  if (k < 0) k += N;
  const long long k8 = 8 * k;
  const int oct = int(k8 / N);            // octant 0..7 of the angle 2 pi k / N
  long long r = k8 - (long long)oct * N;  // remainder within the octant, in units of 1/(8N)
  const bool odd = oct & 1;
  if (odd) r = N - r;                     // reflect so the reduced angle is in [0, pi/4]
  const long double tau = 6.283185307179586476925286766559005768L;
  const long double a = tau * (long double)r / (8.0L * (long double)N);
  double c = (double)cosl(a), s = (double)sinl(a);
  if (r == 0) { c = 1.0; s = 0.0; }
  // angle theta = oct*pi/4 +/- a ; (cos theta, sin theta) by octant
  double ct, st;
  switch (oct) {
    case 0: ct = c; st = s; break;
    case 1: ct = s; st = c; break;
    case 2: ct = -s; st = c; break;
    case 3: ct = -c; st = s; break;
    case 4: ct = -c; st = -s; break;
    case 5: ct = -s; st = -c; break;
    case 6: ct = s; st = -c; break;
    default: ct = c; st = -s; break;
  }
  return make_double2(ct, -st);  // exp(-i theta)
}

static void twiddles(std::vector<double2>& all, int N, size_t& off) {
  off = all.size();
  for (int k = 0; k < N; ++k) all.push_back(unit_root(k, N));
}

}  // namespace fm

using namespace fm;

extern "C" {

namespace {
struct RestoreDevice {  // fm_ctx_create selects `device`; the caller's current device is restored
  int prev = -1;
  RestoreDevice() { cudaGetDevice(&prev); }
  ~RestoreDevice() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};
}  // namespace

int fm_ctx_create(int dim, const int32_t* points, const double* lengths, int tdim,
                  int nyquist_mode, int device, fm_ctx** out) {
  RestoreDevice restore_;
  if (!out || !points || !lengths) return FM_E_INVALID;
  *out = nullptr;
  if (dim != 2 && dim != 3) return FM_E_INVALID;
  for (int a = 0; a < dim; ++a)
    if (points[a] < 1 || !(lengths[a] > 0.0)) return FM_E_INVALID;
  if (tdim < dim || tdim > 3) return FM_E_INVALID;
  if (nyquist_mode != 0 && nyquist_mode != 1) return FM_E_INVALID;
  fm_ctx* ctx = new (std::nothrow) fm_ctx;
  if (!ctx) return FM_E_OOM;
  ctx->dim = dim;
  for (int a = 0; a < 3; ++a) {
    ctx->pts[a] = a < dim ? points[a] : 1;
    ctx->len[a] = a < dim ? lengths[a] : 1.0;
  }
  ctx->tdim = tdim;
  ctx->ncomp = tdim * tdim;
  ctx->mode = nyquist_mode;
  ctx->Nx = ctx->pts[0];
  ctx->Ny = ctx->pts[1];
  ctx->Nz = ctx->pts[2];
  ctx->n = int64_t(ctx->Nx) * ctx->Ny * ctx->Nz;
  ctx->n_global = ctx->n;
  ctx->n_local_stride = ctx->n;
  const bool even = ctx->Nz % 2 == 0;
  ctx->nzh = (even && nyquist_mode == FM_NYQUIST_ZERO_COMPATIBLE) ? ctx->Nz / 2 : ctx->Nz / 2 + 1;
  ctx->Lz = even ? ctx->Nz / 2 : ctx->Nz;
  ctx->device = device;
  auto fail = [&](int st) {
    fm_ctx_destroy(ctx);
    return st;
  };
  if (cudaSetDevice(device) != cudaSuccess) return fail(FM_E_CUDA);
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) return fail(FM_E_CUDA);
  make_plan(ctx->px, ctx->Nx);
  make_plan(ctx->py, ctx->Ny);
  make_plan(ctx->pz, ctx->Nz);
  make_plan(ctx->pzh, even ? ctx->Nz / 2 : 1);
  std::vector<double2> tw;
  size_t ox, oy, oz, ozh;
  twiddles(tw, ctx->Nx, ox);
  twiddles(tw, ctx->Ny, oy);
  twiddles(tw, ctx->Nz, oz);
  twiddles(tw, even ? ctx->Nz / 2 : 1, ozh);
  if (cudaMalloc(&ctx->d_tw, tw.size() * sizeof(double2)) != cudaSuccess) return fail(FM_E_OOM);
  if (cudaMemcpy(ctx->d_tw, tw.data(), tw.size() * sizeof(double2), cudaMemcpyHostToDevice) != cudaSuccess)
    return fail(FM_E_CUDA);
  ctx->px.tw = ctx->d_tw + ox;
  ctx->py.tw = ctx->d_tw + oy;
  ctx->pz.tw = ctx->d_tw + oz;
  ctx->pzh.tw = ctx->d_tw + ozh;
  const size_t spec_elems = size_t(ctx->ncomp) * ctx->Nx * ctx->Ny * ctx->nzh;
  if (cudaMalloc(&ctx->spec, spec_elems * sizeof(double2)) != cudaSuccess) return fail(FM_E_OOM);
  ctx->spec_rank_elems = int64_t(spec_elems);
  const int64_t half = (ctx->n * ctx->ncomp) / 2;
  int64_t rb = (half + 255) / 256;
  ctx->red_blocks = int(rb < 1 ? 1 : (rb > 148 * 4 ? 148 * 4 : rb));
  if (cudaMalloc(&ctx->d_partial, sizeof(double) * (ctx->red_blocks + 16) * 16) != cudaSuccess)
    return fail(FM_E_OOM);
  // pass-5 partials: one per z-line group (9 components x Nx Ny lines at most)
  ctx->epi_cap = int64_t(9) * ctx->Nx * ctx->Ny + 64;
  if (cudaMalloc(&ctx->d_epi, sizeof(double) * ctx->epi_cap) != cudaSuccess) return fail(FM_E_OOM);
  // pass-1 partials: one per z-line group, or one per resident CTA of the
  // persistent pass 1 (<= 148 SMs x 32) for each of up to 16 virtual ranks
  ctx->epi2_cap = ctx->epi_cap + int64_t(148) * 32 * 16;
  if (cudaMalloc(&ctx->d_epi2, sizeof(double) * ctx->epi2_cap) != cudaSuccess) return fail(FM_E_OOM);
  if (cudaMalloc(&ctx->d_fold, sizeof(double) * (ctx->epi2_cap / 1024 + 64)) != cudaSuccess) return fail(FM_E_OOM);
  if (cudaMalloc(&ctx->d_scal, sizeof(double) * 64) != cudaSuccess) return fail(FM_E_OOM);
  if (cudaMemset(ctx->d_scal, 0, sizeof(double) * 64) != cudaSuccess) return fail(FM_E_CUDA);
  if (cudaMallocHost(&ctx->h_scal, sizeof(double) * 64) != cudaSuccess) return fail(FM_E_OOM);
  if (cudaMalloc(&ctx->d_bad, sizeof(unsigned long long)) != cudaSuccess) return fail(FM_E_OOM);
  if (cudaMalloc(&ctx->d_badval, 2 * sizeof(double)) != cudaSuccess) return fail(FM_E_OOM);  // value + its key
  if (const char* dbg = getenv("FM_DEBUG_RESIDUE")) fm_ctx_set_debug(ctx, atoi(dbg));
  *out = ctx;
  return FM_OK;
}

int fm_ctx_destroy(fm_ctx* ctx) {
  FM_DEVICE_SCOPE(ctx);
  if (!ctx) return FM_OK;
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->cg_exec) cudaGraphExecDestroy(ctx->cg_exec);
  release_field(ctx->r);
  release_field(ctx->p);
  release_field(ctx->Ap);
  release_field(ctx->tmp);
  release_field(ctx->rhs);
  release_field(ctx->dF);
  release_field(ctx->Pw);
  if (ctx->d_tw) cudaFree(ctx->d_tw);
  if (ctx->spec) cudaFree(ctx->spec);
  if (ctx->d_partial) cudaFree(ctx->d_partial);
  if (ctx->d_epi) cudaFree(ctx->d_epi);
  if (ctx->d_epi2) cudaFree(ctx->d_epi2);
  if (ctx->d_fold) cudaFree(ctx->d_fold);
  if (ctx->spec2) cudaFree(ctx->spec2);
  if (ctx->spec3) cudaFree(ctx->spec3);
  if (ctx->d_gather) cudaFree(ctx->d_gather);
  dist_destroy(ctx);
  if (ctx->d_scal) cudaFree(ctx->d_scal);
  if (ctx->h_scal) cudaFreeHost(ctx->h_scal);
  if (ctx->d_bad) cudaFree(ctx->d_bad);
  if (ctx->d_badval) cudaFree(ctx->d_badval);
  for (cudaEvent_t e : ctx->prof.pending) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->prof.pool) cudaEventDestroy(e);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return FM_OK;
}

// ---- slab decomposition ----------------------------------------------------
static int setup_slabs(fm_ctx* ctx, int P) {
  if (P < 1 || ctx->Nx % P || ctx->Ny % P)
    return set_error(ctx, FM_E_UNSUPPORTED, "slab decomposition needs Nx and Ny divisible by the rank count");
  if (P > kMaxRanks) return set_error(ctx, FM_E_UNSUPPORTED, "more slab ranks than kMaxRanks (16)");
  ctx->P = P;
  ctx->spec_rank_elems = int64_t(ctx->ncomp) * (ctx->Nx / P) * ctx->Ny * ctx->nzh;
  if (P > 1 && !ctx->spec2) {
    const size_t bytes = size_t(ctx->spec_rank_elems) * (ctx->virt ? P : 1) * sizeof(double2);
    FM_CUDA(ctx, cudaMalloc(&ctx->spec2, bytes));
  }
  if (P > 1 && ctx->transpose == 1 && !ctx->spec3) {
    const size_t bytes = size_t(ctx->spec_rank_elems) * (ctx->virt ? P : 1) * sizeof(double2);
    FM_CUDA(ctx, cudaMalloc(&ctx->spec3, bytes));
  }
  if (!ctx->d_gather) FM_CUDA(ctx, cudaMalloc(&ctx->d_gather, sizeof(double) * 64 * size_t(P)));
  return dist_setup_routes(ctx);
}

// FM_TRANSPOSE=nccl (or "staged"): new contexts start with the staged
// all-to-all transposes instead of the fused peer stores.
static int transpose_from_env() {
  const char* e = getenv("FM_TRANSPOSE");
  return e && (!strcmp(e, "nccl") || !strcmp(e, "staged") || !strcmp(e, "1")) ? 1 : 0;
}

int fm_ctx_set_debug(fm_ctx* ctx, int residue_check) {
  if (!ctx) return FM_E_INVALID;
  ctx->debug_residue = residue_check != 0;
  const char* inj = getenv("FM_DEBUG_RESIDUE_INJECT");
  ctx->debug_inject = inj ? atof(inj) : 0.0;
  return FM_OK;
}

int fm_ctx_set_transpose(fm_ctx* ctx, int mode) {
  FM_DEVICE_SCOPE(ctx);
  if (!ctx || (mode != 0 && mode != 1)) return FM_E_INVALID;
  if (ctx->transpose == mode) return FM_OK;
  if (distributed(ctx))  // the peer mappings are made (or not) when the context is created
    return set_error(ctx, FM_E_INVALID, "the transpose mode of a distributed context is fixed at creation (FM_TRANSPOSE)");
  ctx->transpose = mode;
  if (ctx->P > 1) {  // virtual ranks already set up: add the staging buffer
    FM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return setup_slabs(ctx, ctx->P);
  }
  return FM_OK;
}

int fm_ctx_set_virtual_ranks(fm_ctx* ctx, int P) {
  FM_DEVICE_SCOPE(ctx);
  if (!ctx || P < 1) return FM_E_INVALID;
  if (ctx->nccl) return set_error(ctx, FM_E_INVALID, "context is distributed over devices");
  ctx->virt = P > 1;
  if (P == 1) {
    ctx->P = 1;
    ctx->spec_rank_elems = int64_t(ctx->ncomp) * ctx->Nx * ctx->Ny * ctx->nzh;
    return FM_OK;
  }
  return setup_slabs(ctx, P);
}

int fm_ctx_create_dist(int dim, const int32_t* points, const double* lengths, int tdim, int nyquist_mode,
                       int device, int nranks, int rank, const void* nccl_unique_id, fm_ctx** out) {
  if (!out || !nccl_unique_id || nranks < 1 || rank < 0 || rank >= nranks || !points) return FM_E_INVALID;
  if (nranks == 1) return fm_ctx_create(dim, points, lengths, tdim, nyquist_mode, device, out);
  if (dim != 3 || points[0] % nranks || points[1] % nranks) return FM_E_UNSUPPORTED;
  // the context is created for the whole grid (plans, workspace sized per slab below)
  int st = fm_ctx_create(dim, points, lengths, tdim, nyquist_mode, device, out);
  if (st) return st;
  fm_ctx* ctx = *out;
  FM_DEVICE_SCOPE(ctx);
  ctx->rank = rank;
  ctx->n_global = ctx->n;
  ctx->n = ctx->n_global / nranks;  // local x-slab: fields hold n_local nodes
  ctx->n_local_stride = ctx->n;
  ctx->node_offset = int64_t(rank) * ctx->n;
  // re-size the per-rank workspace: A and B hold one slab's spectrum each
  cudaFree(ctx->spec);
  ctx->spec = nullptr;
  const size_t rank_elems = size_t(ctx->ncomp) * (ctx->Nx / nranks) * ctx->Ny * ctx->nzh;
  if (cudaMalloc(&ctx->spec, rank_elems * sizeof(double2)) != cudaSuccess) st = FM_E_OOM;
  ctx->transpose = transpose_from_env();
  if (!st) st = dist_init_nccl(ctx, nccl_unique_id, nranks, rank);
  if (!st) st = setup_slabs(ctx, nranks);
  if (st) {
    fm_ctx_destroy(ctx);
    *out = nullptr;
  }
  return st;
}

int fm_ctx_ranks(const fm_ctx* ctx, int* nranks, int* rank, int* virtual_mode) {
  if (!ctx) return FM_E_INVALID;
  if (nranks) *nranks = ctx->P;
  if (rank) *rank = ctx->rank;
  if (virtual_mode) *virtual_mode = ctx->virt ? 1 : 0;
  return FM_OK;
}

const char* fm_last_error(const fm_ctx* ctx) { return ctx ? ctx->last_error.c_str() : "null context"; }

int fm_last_error_info(const fm_ctx* ctx, fm_error_info* out) {
  if (!ctx || !out) return FM_E_INVALID;
  *out = ctx->last_info;
  return FM_OK;
}

int64_t fm_ctx_nodes(const fm_ctx* ctx) { return ctx ? ctx->n : 0; }
int fm_ctx_tdim(const fm_ctx* ctx) { return ctx ? ctx->tdim : 0; }
void* fm_ctx_stream(fm_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }
int64_t fm_ctx_launch_count(const fm_ctx* ctx) { return ctx ? ctx->cnt.launches : 0; }

int fm_ctx_kernel_names(const fm_ctx* ctx, char* buf, int cap) {
  if (!ctx) return -1;
  std::string s;
  for (const char* k : ctx->cnt.kernels) {
    if (!s.empty()) s += ',';
    s += k;
  }
  if (buf && cap > 0) {
    const size_t m = std::min(s.size(), size_t(cap - 1));
    std::memcpy(buf, s.data(), m);
    buf[m] = '\0';
  }
  return int(s.size());
}

int fm_ctx_profile(fm_ctx* ctx, int enable) {
  FM_DEVICE_SCOPE(ctx);
  if (!ctx) return FM_E_INVALID;
  if (int st = profile_collect(ctx)) return st;
  ctx->prof.on = enable != 0;
  for (double& v : ctx->prof.ms) v = 0.0;
  ctx->prof.calls = 0;
  return FM_OK;
}

int fm_ctx_profile_read(fm_ctx* ctx, double* ms, int64_t* calls) {
  FM_DEVICE_SCOPE(ctx);
  if (!ctx || !ms || !calls) return FM_E_INVALID;
  if (int st = profile_collect(ctx)) return st;
  for (int s = 0; s < kPasses; ++s) ms[s] = ctx->prof.ms[s];
  *calls = ctx->prof.calls;
  return FM_OK;
}

int fm_ctx_synchronize(fm_ctx* ctx) {
  FM_DEVICE_SCOPE(ctx);
  if (!ctx) return FM_E_INVALID;
  FM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return FM_OK;
}

// ------------------------------------------------------------------ fields
int fm_field_alloc(fm_ctx* ctx, int ncomp, fm_field** out) {
  FM_DEVICE_SCOPE(ctx);
  if (!ctx || !out || ncomp < 1 || ncomp > 81) return FM_E_INVALID;
  fm_field* f = new (std::nothrow) fm_field;
  if (!f) return FM_E_OOM;
  if (int st = ensure_field(ctx, *f, ncomp)) {
    delete f;
    return st;
  }
  FM_CUDA(ctx, cudaMemsetAsync(f->d, 0, sizeof(double) * ncomp * size_t(ctx->n), ctx->stream));
  *out = f;
  return FM_OK;
}

int fm_field_free(fm_ctx* ctx, fm_field* f) {
  FM_DEVICE_SCOPE(ctx);
  if (!f) return FM_OK;
  if (ctx) cudaStreamSynchronize(ctx->stream);
  release_field(*f);
  delete f;
  return FM_OK;
}

double* fm_field_device_ptr(fm_field* f) { return f ? f->d : nullptr; }

int fm_field_upload(fm_ctx* ctx, fm_field* f, const double* host, int64_t count) {
  FM_DEVICE_SCOPE(ctx);
  if (!ctx || !f || !host || count != f->n * f->ncomp)
    return set_error(ctx, FM_E_INVALID, "fm_field_upload: size mismatch");
  FM_CUDA(ctx, cudaMemcpyAsync(f->d, host, sizeof(double) * count, cudaMemcpyHostToDevice, ctx->stream));
  FM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return FM_OK;
}

int fm_field_download(fm_ctx* ctx, const fm_field* f, double* host, int64_t count) {
  FM_DEVICE_SCOPE(ctx);
  if (!ctx || !f || !host || count != f->n * f->ncomp)
    return set_error(ctx, FM_E_INVALID, "fm_field_download: size mismatch");
  FM_CUDA(ctx, cudaMemcpyAsync(host, f->d, sizeof(double) * count, cudaMemcpyDeviceToHost, ctx->stream));
  FM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return FM_OK;
}

int fm_field_fill(fm_ctx* ctx, fm_field* f, double value) {
  FM_DEVICE_SCOPE(ctx);
  if (!ctx || !f) return FM_E_INVALID;
  if (value == 0.0) {
    FM_CUDA(ctx, cudaMemsetAsync(f->d, 0, sizeof(double) * f->ncomp * size_t(f->n), ctx->stream));
    return FM_OK;
  }
  std::vector<double> t(size_t(f->ncomp), value);
  if (f->ncomp > 9) return set_error(ctx, FM_E_INVALID, "fill: ncomp > 9 supports value 0 only");
  return fill_uniform_async(ctx, f->d, t.data(), f->ncomp, f->n);
}

int fm_field_copy(fm_ctx* ctx, const fm_field* src, fm_field* dst) {
  FM_DEVICE_SCOPE(ctx);
  if (!ctx || !src || !dst || src->ncomp != dst->ncomp) return set_error(ctx, FM_E_INVALID, "copy: shape mismatch");
  FM_CUDA(ctx, cudaMemcpyAsync(dst->d, src->d, sizeof(double) * src->ncomp * size_t(src->n),
                               cudaMemcpyDeviceToDevice, ctx->stream));
  return FM_OK;
}

// -------------------------------------------------------------- projection
int fm_projection_apply(fm_ctx* ctx, const fm_field* A, fm_field* out) {
  FM_DEVICE_SCOPE(ctx);
  if (!ctx || !A || !out || A->ncomp != ctx->ncomp || out->ncomp != ctx->ncomp)
    return set_error(ctx, FM_E_INVALID, "apply_projection: field does not match operator");
  ProArgs pa;
  pa.kind = PRO_COPY;
  pa.A = A->d;
  return projection_run(ctx, pa, out->d, 1.0);
}

int fm_projected_tangent_apply(fm_ctx* ctx, const fm_field* K, const fm_field* dF, fm_field* out) {
  FM_DEVICE_SCOPE(ctx);
  if (!ctx || !K || !dF || !out || K->ncomp != ctx->ncomp * ctx->ncomp || dF->ncomp != ctx->ncomp ||
      out->ncomp != ctx->ncomp)
    return set_error(ctx, FM_E_INVALID, "apply_projected_tangent: shape mismatch");
  ProArgs pa;
  pa.kind = PRO_K4;
  pa.A = dF->d;
  pa.K = K->d;
  return projection_run(ctx, pa, out->d, 1.0);
}

// ------------------------------------------------------------ constitutive
int fm_hyper_evaluate(fm_ctx* ctx, const fm_field* F, const fm_field* lambda, const fm_field* mu,
                      fm_field* P, fm_field* K) {
  FM_DEVICE_SCOPE(ctx);
  if (!ctx || !F || !lambda || !mu || !P || F->ncomp != ctx->ncomp || P->ncomp != ctx->ncomp ||
      lambda->ncomp != 1 || mu->ncomp != 1 || (K && K->ncomp != ctx->ncomp * ctx->ncomp))
    return set_error(ctx, FM_E_INVALID, "hyperelastic_evaluate: parameter field size mismatch");
  if (int st = hyper_eval_async(ctx, F->d, lambda->d, mu->d, P->d, K ? K->d : nullptr)) return st;
  return check_bad(ctx);
}

int fm_simo_evaluate(fm_ctx* ctx, const fm_field* F, const fm_field* F_old,
                     const fm_field* be_committed, const fm_field* epsp_committed,
                     const fm_field* lambda, const fm_field* mu, const fm_field* tau_y0,
                     const fm_field* hardening, fm_field* P, fm_field* K, fm_field* be_trial,
                     fm_field* epsp_trial) {
  FM_DEVICE_SCOPE(ctx);
  if (!ctx || ctx->tdim != 3) return set_error(ctx, FM_E_INVALID, "simo_evaluate: tensors must be 3x3");
  if (!F || !F_old || !be_committed || !epsp_committed || !lambda || !mu || !tau_y0 || !hardening ||
      !P || !be_trial || !epsp_trial || F->ncomp != 9 || F_old->ncomp != 9 || be_committed->ncomp != 9 ||
      epsp_committed->ncomp != 1 || P->ncomp != 9 || be_trial->ncomp != 9 || epsp_trial->ncomp != 1 ||
      (K && K->ncomp != 81))
    return set_error(ctx, FM_E_INVALID, "simo_evaluate: state size mismatch");
  if (int st = simo_eval_async(ctx, F->d, F_old->d, be_committed->d, epsp_committed->d, lambda->d,
                               mu->d, tau_y0->d, hardening->d, P->d, K ? K->d : nullptr,
                               be_trial->d, epsp_trial->d))
    return st;
  return check_bad(ctx);
}

int fm_equivalent_stress(fm_ctx* ctx, const fm_field* F, const fm_field* P, int kind, fm_field* out) {
  FM_DEVICE_SCOPE(ctx);
  if (!ctx || !P || !out || P->ncomp != ctx->ncomp || out->ncomp != 1 ||
      (kind != FM_EQ_TENSOR && (!F || F->ncomp != ctx->ncomp)) || kind < FM_EQ_TENSOR || kind > FM_EQ_KIRCHHOFF)
    return set_error(ctx, FM_E_INVALID, "equivalent_stress: field size mismatch");
  if (int st = eq_stress_async(ctx, kind, F ? F->d : nullptr, P->d, out->d)) return st;
  return check_bad(ctx);
}

// ------------------------------------------------------------------- BLAS
static bool same(const fm_field* a, const fm_field* b) { return a && b && a->ncomp == b->ncomp && a->n == b->n; }

int fm_dot(fm_ctx* ctx, const fm_field* a, const fm_field* b, double* out) {
  FM_DEVICE_SCOPE(ctx);
  if (!ctx || !same(a, b) || !out) return set_error(ctx, FM_E_INVALID, "tensor field shape/dimension mismatch");
  if (int st = dot_async(ctx, a->d, b->d, a->n * a->ncomp, ctx->d_scal + 8)) return st;
  if (int st = fetch_scalars(ctx, 9)) return st;
  *out = ctx->h_scal[8];
  return FM_OK;
}

int fm_norm(fm_ctx* ctx, const fm_field* a, double* out) {
  FM_DEVICE_SCOPE(ctx);
  double s;
  if (int st = fm_dot(ctx, a, a, &s)) return st;
  *out = std::sqrt(s);
  return FM_OK;
}

int fm_mean(fm_ctx* ctx, const fm_field* a, double* out) {
  FM_DEVICE_SCOPE(ctx);
  if (!ctx || !a || !out || a->ncomp > 9) return set_error(ctx, FM_E_INVALID, "mean: bad field");
  if (int st = sum_comp_async(ctx, a->d, a->ncomp, a->n, ctx->d_scal + 16)) return st;
  if (int st = fetch_scalars(ctx, 16 + a->ncomp)) return st;
  for (int c = 0; c < a->ncomp; ++c) out[c] = ctx->h_scal[16 + c] / double(ctx->n_global);
  return FM_OK;
}

int fm_axpy(fm_ctx* ctx, double a, const fm_field* x, fm_field* y) {
  FM_DEVICE_SCOPE(ctx);
  if (!ctx || !same(x, y)) return set_error(ctx, FM_E_INVALID, "tensor field shape/dimension mismatch");
  return axpy_async(ctx, a, x->d, y->d, x->n * x->ncomp);
}

int fm_scale(fm_ctx* ctx, fm_field* x, double s) {
  FM_DEVICE_SCOPE(ctx);
  if (!ctx || !x) return FM_E_INVALID;
  return scale_async(ctx, x->d, s, x->n * x->ncomp);
}

int fm_add(fm_ctx* ctx, fm_field* y, const fm_field* x, double sign) {
  FM_DEVICE_SCOPE(ctx);
  if (!ctx || !same(x, y)) return set_error(ctx, FM_E_INVALID, "tensor field shape/dimension mismatch");
  return add_async(ctx, y->d, x->d, sign, x->n * x->ncomp);
}

int fm_add_uniform(fm_ctx* ctx, fm_field* f, const double* t) {
  FM_DEVICE_SCOPE(ctx);
  if (!ctx || !f || !t || f->ncomp > 9) return set_error(ctx, FM_E_INVALID, "add_uniform: tensor dimension mismatch");
  return add_uniform_async(ctx, f->d, t, f->ncomp, f->n);
}

// ------------------------------------------------------------------ solver
int fm_cg_solve(fm_ctx* ctx, const fm_field* K, const fm_field* rhs, double eta_cg, int64_t max_cg,
                fm_field* x, int32_t* iterations, double* rel_residual) {
  FM_DEVICE_SCOPE(ctx);
  if (!ctx || !K || !rhs || !x || !iterations || !rel_residual || K->ncomp != ctx->ncomp * ctx->ncomp ||
      rhs->ncomp != ctx->ncomp || x->ncomp != ctx->ncomp)
    return set_error(ctx, FM_E_INVALID, "cg_solve: shape mismatch");
  if (!(eta_cg > 0.0 && eta_cg < 1.0)) return set_error(ctx, FM_E_INVALID, "eta_cg must be in (0,1)");
  if (max_cg < 0) return set_error(ctx, FM_E_INVALID, "max_cg must be >= 0");
  return cg_run_k4(ctx, K->d, rhs->d, eta_cg, max_cg, x->d, iterations, rel_residual);
}

// Matrix-free SVK: when the per-voxel (lambda, mu) pairs take at most 256
// distinct values (a phase microstructure, bind_parameters,
// microstructure.cpp:176-203), keep a 1-byte label per voxel and the pair
// table for the pipelined pass 1 (ProArgs::lab).  Pairs are compared bit for
// bit, so the table holds exactly the doubles the fields hold.
// FM_PHASE_LABELS=0 keeps the two per-voxel fields in pass 1.
static int build_phase_labels(fm_ctx* ctx, fm_model* m, const double* lambda, const double* mu) {
  static const int env = [] {
    const char* e = getenv("FM_PHASE_LABELS");
    return e ? atoi(e) : 1;
  }();
  if (!env) return FM_OK;
  std::vector<uint8_t> lab(size_t(ctx->n));
  std::vector<uint64_t> tl, tm;
  int last = -1;
  for (int64_t i = 0; i < ctx->n; ++i) {
    uint64_t a, b;
    std::memcpy(&a, lambda + i, 8);
    std::memcpy(&b, mu + i, 8);
    if (last < 0 || tl[last] != a || tm[last] != b) {
      last = -1;
      for (size_t k = 0; k < tl.size(); ++k)
        if (tl[k] == a && tm[k] == b) {
          last = int(k);
          break;
        }
      if (last < 0) {
        if (tl.size() == 256) return FM_OK;  // too many phases: per-voxel fields
        tl.push_back(a);
        tm.push_back(b);
        last = int(tl.size()) - 1;
      }
    }
    lab[size_t(i)] = uint8_t(last);
  }
  std::vector<uint64_t> tab(512, 0);
  std::copy(tl.begin(), tl.end(), tab.begin());
  std::copy(tm.begin(), tm.end(), tab.begin() + 256);
  FM_CUDA(ctx, cudaMalloc(&m->lab, size_t(ctx->n) + 16));
  FM_CUDA(ctx, cudaMalloc(&m->ptab, 512 * sizeof(double)));
  FM_CUDA(ctx, cudaMemcpy(m->lab, lab.data(), size_t(ctx->n), cudaMemcpyHostToDevice));
  FM_CUDA(ctx, cudaMemcpy(m->ptab, tab.data(), 512 * sizeof(double), cudaMemcpyHostToDevice));
  return FM_OK;
}

int fm_model_create_hyper(fm_ctx* ctx, const double* lambda, const double* mu, int matrix_free,
                          fm_model** out) {
  FM_DEVICE_SCOPE(ctx);
  if (!ctx || !lambda || !mu || !out) return FM_E_INVALID;
  fm_model* m = new (std::nothrow) fm_model;
  if (!m) return FM_E_OOM;
  m->kind = 0;
  m->matrix_free = matrix_free ? 1 : 0;
  int st = ensure_field(ctx, m->lambda, 1);
  if (!st) st = ensure_field(ctx, m->mu, 1);
  if (!st) st = m->matrix_free ? ensure_field(ctx, m->F_eval, ctx->ncomp)
                               : ensure_field(ctx, m->K, ctx->ncomp * ctx->ncomp);
  if (!st) st = fm_field_upload(ctx, &m->lambda, lambda, ctx->n);
  if (!st) st = fm_field_upload(ctx, &m->mu, mu, ctx->n);
  if (!st && m->matrix_free) st = build_phase_labels(ctx, m, lambda, mu);
  if (st) {
    fm_model_destroy(ctx, m);
    return st;
  }
  *out = m;
  return FM_OK;
}

int fm_model_create_simo(fm_ctx* ctx, const double* lambda, const double* mu, const double* tau_y0,
                         const double* hardening, fm_model** out) {
  FM_DEVICE_SCOPE(ctx);
  if (!ctx || !lambda || !mu || !tau_y0 || !hardening || !out) return FM_E_INVALID;
  if (ctx->tdim != 3) return set_error(ctx, FM_E_INVALID, "Simo model needs tdim 3");
  fm_model* m = new (std::nothrow) fm_model;
  if (!m) return FM_E_OOM;
  m->kind = 1;
  int st = FM_OK;
  fm_field* one[] = {&m->lambda, &m->mu, &m->tau_y0, &m->hard, &m->epsp_c, &m->epsp_t};
  for (fm_field* f : one)
    if (!st) st = ensure_field(ctx, *f, 1);
  fm_field* nine[] = {&m->be_c, &m->be_t, &m->f_old};
  for (fm_field* f : nine)
    if (!st) st = ensure_field(ctx, *f, 9);
  if (!st) st = ensure_field(ctx, m->K, 81);
  if (!st) st = fm_field_upload(ctx, &m->lambda, lambda, ctx->n);
  if (!st) st = fm_field_upload(ctx, &m->mu, mu, ctx->n);
  if (!st) st = fm_field_upload(ctx, &m->tau_y0, tau_y0, ctx->n);
  if (!st) st = fm_field_upload(ctx, &m->hard, hardening, ctx->n);
  // HistoryState init: be = I, eps_p = 0 (material.cpp:11-12); f_old = I (simo.cpp:208)
  const double I9[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  if (!st) st = fill_uniform_async(ctx, m->be_c.d, I9, 9, ctx->n);
  if (!st) st = fill_uniform_async(ctx, m->be_t.d, I9, 9, ctx->n);
  if (!st) st = fill_uniform_async(ctx, m->f_old.d, I9, 9, ctx->n);
  if (!st) {
    cudaMemsetAsync(m->epsp_c.d, 0, sizeof(double) * ctx->n, ctx->stream);
    cudaMemsetAsync(m->epsp_t.d, 0, sizeof(double) * ctx->n, ctx->stream);
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) st = FM_E_CUDA;
  }
  if (st) {
    fm_model_destroy(ctx, m);
    return st;
  }
  *out = m;
  return FM_OK;
}

int fm_model_destroy(fm_ctx* ctx, fm_model* m) {
  FM_DEVICE_SCOPE(ctx);
  if (!m) return FM_OK;
  if (ctx) cudaStreamSynchronize(ctx->stream);
  for (fm_field* f : {&m->lambda, &m->mu, &m->tau_y0, &m->hard, &m->K, &m->Kc, &m->F_eval, &m->be_c,
                      &m->epsp_c, &m->be_t, &m->epsp_t, &m->f_old})
    release_field(*f);
  if (m->lab) cudaFree(m->lab);
  if (m->ptab) cudaFree(m->ptab);
  delete m;
  return FM_OK;
}

int fm_model_evaluate(fm_ctx* ctx, fm_model* m, const fm_field* F, fm_field* P) {
  FM_DEVICE_SCOPE(ctx);
  if (!ctx || !m || !F || !P || F->ncomp != ctx->ncomp || P->ncomp != ctx->ncomp)
    return set_error(ctx, FM_E_INVALID, "evaluate: shape mismatch");
  return model_evaluate(ctx, m, F->d, P->d);
}

int fm_model_commit(fm_ctx* ctx, fm_model* m, const fm_field* F) {
  FM_DEVICE_SCOPE(ctx);
  if (!ctx || !m || !F || F->ncomp != ctx->ncomp) return set_error(ctx, FM_E_INVALID, "commit: shape mismatch");
  return model_commit(ctx, m, F->d);
}

fm_field* fm_model_tangent(fm_model* m) { return (m && m->K.d) ? &m->K : nullptr; }

int fm_model_set_tangent_form(fm_ctx* ctx, fm_model* m, int form) {
  FM_DEVICE_SCOPE(ctx);
  if (!ctx || !m || form < 0 || form > 1) return FM_E_INVALID;
  if (m->kind != 1) return form == 0 ? FM_OK : set_error(ctx, FM_E_INVALID, "compact tangent: Simo model only");
  if (form == m->compact) return FM_OK;
  cudaStreamSynchronize(ctx->stream);
  if (form == 1) {
    release_field(m->K);
    if (int st = ensure_field(ctx, m->Kc, 45)) return st;
  } else {
    release_field(m->Kc);
    if (int st = ensure_field(ctx, m->K, 81)) return st;
  }
  m->compact = form;
  return FM_OK;
}

int fm_model_get_history(fm_ctx* ctx, fm_model* m, int which, double* be, double* epsp) {
  FM_DEVICE_SCOPE(ctx);
  if (!ctx || !m || m->kind != 1) return set_error(ctx, FM_E_INVALID, "history: not a Simo model");
  const fm_field& b = which ? m->be_t : m->be_c;
  const fm_field& e = which ? m->epsp_t : m->epsp_c;
  if (be)
    if (int st = fm_field_download(ctx, &b, be, 9 * ctx->n)) return st;
  if (epsp)
    if (int st = fm_field_download(ctx, &e, epsp, ctx->n)) return st;
  return FM_OK;
}

int fm_model_set_history(fm_ctx* ctx, fm_model* m, const double* be, const double* epsp,
                         const double* f_old) {
  FM_DEVICE_SCOPE(ctx);
  if (!ctx || !m || m->kind != 1) return set_error(ctx, FM_E_INVALID, "history: not a Simo model");
  if (be)
    if (int st = fm_field_upload(ctx, &m->be_c, be, 9 * ctx->n)) return st;
  if (epsp)
    if (int st = fm_field_upload(ctx, &m->epsp_c, epsp, ctx->n)) return st;
  if (f_old)
    if (int st = fm_field_upload(ctx, &m->f_old, f_old, 9 * ctx->n)) return st;
  return FM_OK;
}

int fm_model_apply(fm_ctx* ctx, fm_model* m, const fm_field* dF, fm_field* out) {
  FM_DEVICE_SCOPE(ctx);
  if (!ctx || !m || !dF || !out || dF->ncomp != ctx->ncomp || out->ncomp != ctx->ncomp)
    return set_error(ctx, FM_E_INVALID, "apply: shape mismatch");
  return model_apply(ctx, m, dF->d, out->d);
}

int fm_solve_increment(fm_ctx* ctx, fm_model* m, fm_field* F, const double* fbar,
                       const fm_solver_params* params, fm_report* report, fm_field* P_out) {
  FM_DEVICE_SCOPE(ctx);
  if (!ctx || !m || !F || !fbar || !params || !report) return FM_E_INVALID;
  if (P_out && P_out->ncomp != ctx->ncomp) return set_error(ctx, FM_E_INVALID, "P_out shape mismatch");
  return solve_increment(ctx, m, F, fbar, *params, report, P_out);
}

}  // extern "C"
