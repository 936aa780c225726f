// Internal declarations of the sm_100a fftmech hot path.
// Layout in HBM:
//   real fields   : component-major [c][x][y][z] fp64 (the reference layout),
//   spectral work : [c][x][y][kz] complex fp64, kz in [0, nzh) -- the r2c half
//                   spectrum along z; for even Nz in ZeroCompatible mode the
//                   Nyquist column kz = Nz/2 is never stored (ghat = 0 there,
//                   projection.cpp:94-98), so nzh = Nz/2 and one spectral
//                   field is exactly as large as one real field.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/fftmech_b200.h"

namespace fm {

constexpr int kMaxStages = 24;
constexpr int kMaxRanks = 16;  // slab ranks (devices of one node, or virtual ranks)

// One axis of the 3-D transform: length N, radix plan, twiddle table
// tw[k] = exp(-2 pi i k / N) (long-double accurate, device resident).
struct AxisPlan {
  int N = 1;
  int nst = 0;
  int radix[kMaxStages] = {};
  const double2* tw = nullptr;
};

// Kinds of the fused first-pass prologue.
enum Prologue : int {
  PRO_COPY = 0,  // G(A): read A
  PRO_K4 = 1,    // G(K : dF^T): dP_ij = K_jikl dF_kl (projection.cpp:182-192)
  PRO_SVK = 2,   // matrix-free SVK tangent action from F, lambda, mu
  PRO_J2C = 3,   // compact J2 tangent (V, U, a, b, c): dP = V W U^T, W from D = V^T dF U
};

struct Counters {
  int64_t launches = 0;
  std::vector<const char*> kernels;  // distinct kernel names launched (string literals)
  void note(const char* k) {
    for (const char* s : kernels)
      if (s == k || std::string(s) == k) return;
    kernels.push_back(k);
  }
};

// Optional per-pass CUDA-event timing of the projection (bench roofline).
constexpr int kPasses = 5;
struct PassProfile {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  std::vector<cudaEvent_t> pending;  // groups of kPasses + 1 events
  double ms[kPasses] = {};
  int64_t calls = 0;
};

}  // namespace fm

struct fm_field {
  int ncomp = 0;
  int64_t n = 0;
  double* d = nullptr;
};

struct fm_model {
  int kind = 0;  // 0 hyperelastic, 1 Simo
  int matrix_free = 0;
  fm_field lambda, mu, tau_y0, hard;
  fm_field K;                   // tangent (81n or 16n); empty when matrix-free / compact
  int compact = 0;              // Simo: keep the 45-slab compact tangent instead of K4
  fm_field Kc;                  // compact J2 tangent (45n)
  fm_field F_eval;              // F at the last evaluate (matrix-free SVK action)
  uint8_t* lab = nullptr;       // matrix-free SVK: phase labels + (lambda, mu) table (ProArgs::lab)
  double* ptab = nullptr;
  fm_field be_c, epsp_c, be_t, epsp_t, f_old;  // Simo history
};

struct fm_ctx {
  int dim = 3;
  int pts[3] = {1, 1, 1};
  double len[3] = {1, 1, 1};
  int tdim = 3, ncomp = 9;
  int64_t n = 0;         // nodes held by this context (the local slab when distributed)
  int64_t n_global = 0;  // nodes of the whole grid (1/n of the transform, means, CG cap)
  int64_t node_offset = 0;  // global index of local node 0 (error reports)
  int mode = 0;
  int Nx = 1, Ny = 1, Nz = 1;
  int nzh = 1;  // stored kz columns
  int Lz = 1;   // complex FFT length along z (Nz/2 for even Nz, Nz otherwise)
  int device = 0;
  cudaStream_t stream = nullptr;
  fm::AxisPlan px, py, pz, pzh;  // pzh: half-length plan for even-Nz r2c
  double2* d_tw = nullptr;        // all twiddle tables
  double2* spec = nullptr;        // ncomp * Nx * Ny * nzh  (A: z/y side; also the x-pass buffer)
  double2* spec2 = nullptr;       // x-pass input B (y-slab), only when P > 1
  double2* spec3 = nullptr;       // pack / unpack staging of the staged all-to-all transposes (transpose == 1)
  int transpose = 0;              // P > 1: 0 = transposes fused into passes 2, 3 as peer stores, 1 = staged all-to-all
  // debug mode (FM_DEBUG_RESIDUE=1 / fm_ctx_set_debug): every projection checks the imaginary residue the
  // reference checks after its c2c inverse transform (projection.cpp:157-169); inject: test hook
  bool debug_residue = false;
  double debug_inject = 0.0;
  // slab decomposition over P ranks; P = 1: single device
  int P = 1, rank = 0;
  bool virt = false;              // all P ranks emulated on this one device
  int64_t n_local_stride = 0;     // component stride of real fields (n, or n_local when distributed)
  int64_t spec_rank_elems = 0;    // complex elements of one rank's spectral buffer
  void* nccl = nullptr;           // ncclComm_t when distributed over devices
  // destinations of the fused slab transpose (device arrays of P pointers):
  // A (spectrum, x-slab) and B (x-pass input, y-slab) of every rank -- peer
  // memory mapped through CUDA IPC when the ranks are devices
  double2** d_dst_a = nullptr;
  double2** d_dst_b = nullptr;
  std::vector<double2*> h_dst_a;  // host copy of d_dst_a (tensor maps of the routed TMA stores)
  std::vector<void*> ipc_open;    // peer buffers opened with cudaIpcOpenMemHandle
  double* d_gather = nullptr;     // all-gather staging of per-rank scalars
  // CG loop as one CUDA graph (a while-conditional node around the fused
  // iteration): cached for the last (operator, vectors) it was built for
  bool capturing = false;
  cudaGraphExec_t cg_exec = nullptr;
  int64_t cg_iter_launches = 0;   // kernels per graph iteration
  std::vector<const void*> cg_key;
  // reductions
  int red_blocks = 0;
  double* d_partial = nullptr;  // red_blocks * 16
  double* d_epi = nullptr;      // per-block partials of the fused <p,Ap>
  double* d_epi2 = nullptr;     // pass-1 partials of the fused-CG <p, K:p> (epi2_cap)
  int64_t epi2_cap = 0;
  double* d_fold = nullptr;     // first-level sums of a two-level finalisation (epi2_cap / 1024 + 64)
  int zf_partials = 0;          // partials the last pass 1 wrote
  int zi_partials = 0;          // partials the last fast pass 5 wrote
  int64_t epi_cap = 0;
  double* d_scal = nullptr;     // device scalars (64)
  double* h_scal = nullptr;     // pinned mirror (64)
  unsigned long long* d_bad = nullptr;  // lowest offending node (atomicMin)
  double* d_badval = nullptr;
  // CG workspace (allocated lazily, tdim^2 components each)
  fm_field r, p, Ap, tmp, rhs, dF, Pw;  // Pw: the stress workspace
  fm::Counters cnt;
  fm::PassProfile prof;
  std::string last_error;
  fm_error_info last_info{};
};

namespace fm {

// Device scalar slots of the CG driver (ctx->d_scal).
enum Slot { S_RR = 0, S_PAP = 1, S_RRNEW = 2, S_ALPHA = 3, S_BETA = 4, S_FLAG = 5, S_IT = 6, S_THR = 7, S_OUT = 8 };

// Launch/error helpers ------------------------------------------------------
int set_error(fm_ctx* ctx, int status, const std::string& msg);
int check_cuda(fm_ctx* ctx, cudaError_t e, const char* what);
#define FM_CUDA(ctx, call)                                      \
  do {                                                          \
    cudaError_t e_ = (call);                                    \
    if (e_ != cudaSuccess) return ::fm::check_cuda(ctx, e_, #call); \
  } while (0)
#define FM_LAUNCHED_K(ctx, name)                                                 \
  do {                                                                           \
    (ctx)->cnt.launches++;                                                       \
    (ctx)->cnt.note(name);                                                       \
    cudaError_t e_ = cudaGetLastError();                                         \
    if (e_ != cudaSuccess) return ::fm::check_cuda(ctx, e_, name);               \
  } while (0)

int ensure_field(fm_ctx* ctx, fm_field& f, int ncomp);
int norm_sync(fm_ctx* ctx, const double* a, int64_t count, double* out);  // solver.cu

// Function attributes are per device: raise a kernel's dynamic shared-memory
// limit on the CURRENT device once (memoised per (device, kernel)).
void set_smem_limit(const void* kernel, int bytes);

// Every entry point runs on its context's device and restores the caller's
// current device on return (a context may be driven from any thread, and two
// contexts of one process may live on different devices).
struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(const fm_ctx* c) {
    if (!c) return;
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != c->device && cudaSetDevice(c->device) == cudaSuccess) prev = cur;
  }
  ~DeviceScope() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceScope(const DeviceScope&) = delete;
  DeviceScope& operator=(const DeviceScope&) = delete;
};
#define FM_DEVICE_SCOPE(ctx) ::fm::DeviceScope fm_device_scope_(ctx)
void release_field(fm_field& f);

// projection.cu -------------------------------------------------------------
struct ProArgs {
  int kind = PRO_COPY;
  const double* A = nullptr;   // PRO_COPY input / PRO_K4, PRO_SVK: dF
  const double* K = nullptr;   // PRO_K4
  const double* F = nullptr;   // PRO_SVK
  const double* lam = nullptr; // PRO_SVK
  const double* mu = nullptr;  // PRO_SVK
  // PRO_SVK with at most 256 distinct (lambda, mu) pairs: a 1-byte phase label
  // per voxel and the pair table (lambda at [k], mu at [256 + k]) replace the
  // two per-voxel fields in the pipelined pass 1 (16 -> 1 B/voxel)
  const uint8_t* lab = nullptr;
  const double* ptab = nullptr;
  // CG direction update fused into the prologue (solver.cpp:51-55):
  // p = beta p + r is formed per voxel, written back to p and used as dF.
  const double* r = nullptr;
  double* p = nullptr;
  const double* beta = nullptr;  // device scalar
  // fused CG curvature: per-CTA partials of <p, dP> (= <p, G dP> = <p, Ap>
  // since p lies in range(G) and G is self-adjoint), written by pass 1
  double* pap_partial = nullptr;
  // fused CG: x += alpha p_old with the previous iteration's alpha, applied
  // where p_old is loaded anyway (pipelined SVK pass 1 only)
  double* x = nullptr;
  const double* alpha = nullptr;
  // timing experiments only (FM_ZP_DBG, pipelined pass 1): bit 0 skips the SVK
  // action, bit 1 the transforms, bit 2 the stores, bit 3 the TMA loads
  int dbg = 0;
};
// Epilogue of the last pass: per-block partial sums of <pdot, out>
// (the CG curvature <p, Ap>, solver.cpp:37) written to `partial`.
struct EpiArgs {
  const double* pdot = nullptr;
  double* partial = nullptr;
  // fused CG update (solver.cpp:46-48) instead of storing Ap: with alpha and
  // the curvature flag from `scal`, r -= alpha Ap, x += alpha p, and
  // per-block partials of <r, r> into `partial`
  double* r = nullptr;
  double* x = nullptr;
  const double* p = nullptr;
  const double* scal = nullptr;
};
// out = scale * n * G(prologue(args)); scale = 1 gives the reference G.
// Returns the number of partial sums written through epi (0 if none).
int projection_run(fm_ctx* ctx, const ProArgs& args, double* out, double scale,
                   const EpiArgs& epi = EpiArgs{}, int* n_partials = nullptr);
int profile_collect(fm_ctx* ctx);
int cg_pap_finalize_from(fm_ctx* ctx, const double* partials, int n);
int cg_rr_finalize_from(fm_ctx* ctx, const double* partials, int n);
int cg_final_x_async(fm_ctx* ctx, double* x, const double* p, int64_t count);
// True when passes 1 and 5 run the register-resident kernels that carry the
// fused CG iteration (single device, pow2 z, ZeroCompatible, tdim 3).
bool cg_fused_supported(const fm_ctx* ctx);
// True when pass 1 of operator `kind` runs the pipelined kernel that can also
// carry the CG x update (ProArgs::x).
bool cg_xupd_supported(const fm_ctx* ctx, int kind);
// Persistent cooperative CG for latency-bound generic grids (projection.cu).
bool cg_small_supported(const fm_ctx* ctx);
// Runs the CG iterations with x = 0, r = p = b already set; leaves S_IT,
// S_RR, S_RRNEW, S_FLAG and S_OUT (1 curvature exit, 2 converged, 3 cap) in
// d_scal.  FM_E_UNSUPPORTED: not applicable, nothing launched.
int cg_small_run(fm_ctx* ctx, const ProArgs& op, double* x, double* r, double* p, int64_t cap, double thr,
                 double rr0);
// dist.cu: cross-device barrier between the transpose-fused passes (the
// peer stores of one pass complete on every rank before the next reads them);
// no-op on one device and in the virtual mode (stream order suffices)
int rank_barrier(fm_ctx* ctx);
// route tables of the fused transpose: virtual ranks, or IPC-mapped peers
int dist_setup_routes(fm_ctx* ctx);
// staged slab transposes (FM_TRANSPOSE=nccl / fm_ctx_set_transpose(ctx, 1)):
// x-slabs A -> y-slabs B after a local forward y pass (dir +1), and back
// before the inverse y pass (dir -1)
int dist_transpose_staged(fm_ctx* ctx, int dir);
// Ordered cross-rank sum of `count` device scalars (no-op unless distributed).
int combine_ranks(fm_ctx* ctx, double* d_vals, int count);
int combine_min_u64(fm_ctx* ctx, unsigned long long* d_key);
int dist_init_nccl(fm_ctx* ctx, const void* unique_id, int nranks, int rank);
void dist_destroy(fm_ctx* ctx);
inline bool distributed(const fm_ctx* ctx) { return ctx->nccl != nullptr && ctx->P > 1; }

// blas.cu -------------------------------------------------------------------
int dot_async(fm_ctx* ctx, const double* a, const double* b, int64_t count, double* d_out);
int sum_comp_async(fm_ctx* ctx, const double* a, int ncomp, int64_t n, double* d_out);
int axpy_async(fm_ctx* ctx, double a, const double* x, double* y, int64_t count);
int scale_async(fm_ctx* ctx, double* x, double s, int64_t count);
int add_async(fm_ctx* ctx, double* y, const double* x, double sign, int64_t count);
int add_uniform_async(fm_ctx* ctx, double* f, const double* t, int ncomp, int64_t n);
int fill_uniform_async(fm_ctx* ctx, double* f, const double* t, int ncomp, int64_t n);
int fetch_scalars(fm_ctx* ctx, int count);  // d_scal[0:count] -> h_scal, synchronises
// CG helpers operating on device scalars (see solver.cu)
int cg_update_async(fm_ctx* ctx, double* x, double* r, const double* p, const double* Ap,
                    int64_t count);
int cg_direction_async(fm_ctx* ctx, double* p, const double* r, int64_t count);
int cg_pap_async(fm_ctx* ctx, const double* p, const double* Ap, int64_t count);
int cg_pap_finalize_async(fm_ctx* ctx, int n_partials);

// constitutive.cu -----------------------------------------------------------
int hyper_eval_async(fm_ctx* ctx, const double* F, const double* lam, const double* mu, double* P,
                     double* K);
int eq_stress_async(fm_ctx* ctx, int kind, const double* F, const double* P, double* out);
int simo_eval_async(fm_ctx* ctx, const double* F, const double* Fold, const double* be_c,
                    const double* epsp_c, const double* lam, const double* mu,
                    const double* ty0, const double* hard, double* P, double* K, double* be_t,
                    double* epsp_t, double* Kc = nullptr);
int reset_bad(fm_ctx* ctx);

// solver.cu -----------------------------------------------------------------
int cg_run_k4(fm_ctx* ctx, const double* K, const double* b, double eta_cg, int64_t max_cg,
              double* x, int32_t* iters, double* rel);
int model_evaluate(fm_ctx* ctx, fm_model* m, const double* F, double* P);
int model_commit(fm_ctx* ctx, fm_model* m, const double* F);
int model_apply(fm_ctx* ctx, fm_model* m, const double* dF, double* out);
int solve_increment(fm_ctx* ctx, fm_model* m, fm_field* F, const double* fbar,
                    const fm_solver_params& prm, fm_report* rep, fm_field* P_out);
// Reads the lowest offending node/status; returns FM_OK or the error status.
int check_bad(fm_ctx* ctx);

}  // namespace fm
