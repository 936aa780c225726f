// Device-resident CG and Newton drivers (host C++ control flow over the
// sm_100a kernels).  Control flow restates solver.cpp:19-160 statement by
// statement; all vectors stay in HBM, and only the 2-3 scalars the
// reference branches on cross to the host (one pinned read per CG step).
#include <chrono>
#include <cmath>
#include <cstdlib>

#include "fm_internal.cuh"

namespace fm {


// ---- CG loop as a CUDA graph --------------------------------------------
// Body of the while-conditional node: one fused CG iteration, then this
// control kernel decides -- with the reference's tests in the reference's
// order (solver.cpp:38, :49, loop cap :35) -- whether to run another.
__global__ void k_cg_control(cudaGraphConditionalHandle h, double* scal, double cap) {
  const double it = scal[S_IT] + 1.0;
  scal[S_IT] = it;
  bool stop = scal[S_FLAG] != 0.0;            // !(pAp > 0)
  if (!stop) stop = sqrt(scal[S_RRNEW]) <= scal[S_THR];  // sqrt(rr) <= eta |b|
  if (!stop) stop = it >= cap;
  cudaGraphSetConditional(h, stop ? 0u : 1u);
}

// beta = 0 makes the fused p = beta p + r of the first iteration p = r = b.
__global__ void k_cg_init(double* scal, double thr) {
  scal[S_BETA] = 0.0;
  scal[S_ALPHA] = 0.0;  // fused x update of the first iteration adds 0 p
  scal[S_IT] = 0.0;
  scal[S_THR] = thr;
  scal[S_FLAG] = 0.0;
}

static bool cg_graph_enabled(const fm_ctx* ctx) {
  static const int env = [] {
    const char* e = getenv("FM_CG_GRAPH");
    return e ? atoi(e) : 1;
  }();
  // graphs pay off where launch latency dominates (small grids); at 256^3 the
  // eager loop measured ~10% faster for the K4 operator
  if (env == 2) return !distributed(ctx);
  return env != 0 && !distributed(ctx) && ctx->n_global <= (int64_t(1) << 21);
}

struct Op {
  int kind = PRO_K4;
  const double* K = nullptr;
  const double* F = nullptr;
  const double* lam = nullptr;
  const double* mu = nullptr;
  const uint8_t* lab = nullptr;
  const double* ptab = nullptr;
};

int op_apply(fm_ctx* ctx, const Op& op, const double* x, double* out, double scale) {
  ProArgs pa;
  pa.kind = op.kind;
  pa.A = x;
  pa.K = op.K;
  pa.F = op.F;
  pa.lam = op.lam;
  pa.mu = op.mu;
  pa.lab = op.lab;
  pa.ptab = op.ptab;
  return projection_run(ctx, pa, out, scale);
}

// One CG matvec with the CG vector work fused into its first and last pass:
//   prologue: p = beta p + r (unless first), dF = p;  epilogue: <p, Ap> partials.
int op_apply_cg(fm_ctx* ctx, const Op& op, double* p, const double* r, bool first, double* Ap,
                int* n_partials) {
  ProArgs pa;
  pa.kind = op.kind;
  pa.A = p;
  pa.K = op.K;
  pa.F = op.F;
  pa.lam = op.lam;
  pa.mu = op.mu;
  pa.lab = op.lab;
  pa.ptab = op.ptab;
  if (!first) {
    pa.r = r;
    pa.p = p;
    pa.beta = ctx->d_scal + S_BETA;
  }
  EpiArgs epi;
  epi.pdot = p;
  epi.partial = ctx->d_epi;
  return projection_run(ctx, pa, Ap, 1.0, epi, n_partials);
}

// Fused CG iteration (single device, register-resident passes): pass 1 forms
// p = beta p + r, dP = K:p and the curvature <p, dP> = <p, G dP> = <p, Ap>
// (p stays in range(G), G is a self-adjoint projector); alpha is finalised
// before pass 2; pass 5 applies r -= alpha Ap, x += alpha p and writes the
// <r, r> partials without ever storing Ap (1456 -> 1240 B/voxel per iteration).
static bool cg_fused(const fm_ctx* ctx) {
  static const int env = [] {
    const char* e = getenv("FM_CG_FUSED");
    return e ? atoi(e) : 1;
  }();
  return env != 0 && cg_fused_supported(ctx);
}

int op_apply_cg_fused(fm_ctx* ctx, const Op& op, double* p, double* r, bool first, double* x, int* n_partials) {
  // SVK through the pipelined pass 1: x += alpha_prev p_old rides on pass 1
  // (p_old is staged there anyway) and the final update follows the loop
  const bool xupd = cg_xupd_supported(ctx, op.kind);
  ProArgs pa;
  pa.kind = op.kind;
  pa.A = p;
  pa.K = op.K;
  pa.F = op.F;
  pa.lam = op.lam;
  pa.mu = op.mu;
  pa.lab = op.lab;
  pa.ptab = op.ptab;
  pa.pap_partial = ctx->d_epi2;
  if (!first) {
    pa.r = r;
    pa.p = p;
    pa.beta = ctx->d_scal + S_BETA;
    if (xupd) {
      pa.x = x;
      pa.alpha = ctx->d_scal + S_ALPHA;
    }
  }
  EpiArgs epi;
  epi.r = r;
  epi.x = xupd ? nullptr : x;
  epi.p = p;
  epi.scal = ctx->d_scal;
  epi.partial = ctx->d_epi;
  return projection_run(ctx, pa, nullptr, 1.0, epi, n_partials);
}

// one CG iteration in either form; leaves S_FLAG / S_RRNEW / S_BETA / S_RR set
static int cg_iteration(fm_ctx* ctx, const Op& op, double* x, int64_t count, bool first) {
  int nparts = 0;
  if (cg_fused(ctx)) {
    if (int st = op_apply_cg_fused(ctx, op, ctx->p.d, ctx->r.d, first, x, &nparts)) return st;
    return cg_rr_finalize_from(ctx, ctx->d_epi, nparts);
  }
  if (int st = op_apply_cg(ctx, op, ctx->p.d, ctx->r.d, first, ctx->Ap.d, &nparts)) return st;
  if (int st = cg_pap_finalize_async(ctx, nparts)) return st;
  return cg_update_async(ctx, x, ctx->r.d, ctx->p.d, ctx->Ap.d, count);  // :46-48
}

// Converged: the last iteration's x += alpha p that pass 1 would have applied.
static int cg_finish_x(fm_ctx* ctx, const Op& op, double* x, int64_t count) {
  if (!cg_fused(ctx) || !cg_xupd_supported(ctx, op.kind)) return FM_OK;
  return cg_final_x_async(ctx, x, ctx->p.d, count);
}

Op model_op(fm_model* m) {
  Op op;
  if (m->kind == 0 && m->matrix_free) {
    op.kind = PRO_SVK;
    op.F = m->F_eval.d;
    op.lam = m->lambda.d;
    op.mu = m->mu.d;
    op.lab = m->lab;
    op.ptab = m->ptab;
  } else if (m->kind == 1 && m->compact) {
    op.kind = PRO_J2C;
    op.K = m->Kc.d;
  } else {
    op.kind = PRO_K4;
    op.K = m->K.d;
  }
  return op;
}

int norm_sync(fm_ctx* ctx, const double* a, int64_t count, double* out) {
  if (int st = dot_async(ctx, a, a, count, ctx->d_scal + S_OUT)) return st;
  if (int st = fetch_scalars(ctx, S_OUT + 1)) return st;
  *out = std::sqrt(ctx->h_scal[S_OUT]);
  return FM_OK;
}

int mean_sync(fm_ctx* ctx, const double* a, double* mean) {
  if (int st = sum_comp_async(ctx, a, ctx->ncomp, ctx->n, ctx->d_scal + 16)) return st;
  if (int st = fetch_scalars(ctx, 16 + ctx->ncomp)) return st;
  for (int c = 0; c < ctx->ncomp; ++c) mean[c] = ctx->h_scal[16 + c] / double(ctx->n_global);
  return FM_OK;
}

int op_apply_cg(fm_ctx* ctx, const Op& op, double* p, const double* r, bool first, double* Ap,
                int* n_partials);

// The CG iterations of cg_run as one graph launch: no host round trip per
// iteration (the 31^3 configurations are launch/latency bound).
int cg_loop_graph(fm_ctx* ctx, const Op& op, double* x, int64_t count, int64_t cap, double thr, double bnorm,
                  int32_t* iters, double* rel) {
  const std::vector<const void*> key = {reinterpret_cast<const void*>(intptr_t(op.kind)), op.K, op.F, op.lam, op.mu,
                                        op.lab, x, ctx->r.d, ctx->p.d, ctx->Ap.d, reinterpret_cast<const void*>(cap),
                                        reinterpret_cast<const void*>(intptr_t(ctx->P * 2 + (ctx->virt ? 1 : 0)))};
  k_cg_init<<<1, 1, 0, ctx->stream>>>(ctx->d_scal, thr);
  FM_LAUNCHED_K(ctx, "k_cg_init");
  bool built = false;
  if (!ctx->cg_exec || ctx->cg_key != key) {
    built = true;
    if (ctx->cg_exec) cudaGraphExecDestroy(ctx->cg_exec);
    ctx->cg_exec = nullptr;
    cudaGraph_t g;
    FM_CUDA(ctx, cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h;
    FM_CUDA(ctx, cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp{};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    FM_CUDA(ctx, cudaGraphAddNode(&node, g, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    FM_CUDA(ctx, cudaStreamBeginCaptureToGraph(ctx->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    ctx->capturing = true;
    const int64_t l0 = ctx->cnt.launches;
    int st = cg_iteration(ctx, op, x, count, false);
    if (!st) {
      k_cg_control<<<1, 1, 0, ctx->stream>>>(h, ctx->d_scal, double(cap));
      st = cudaGetLastError() == cudaSuccess ? FM_OK : set_error(ctx, FM_E_CUDA, "k_cg_control launch");
      ctx->cnt.launches++;
    }
    ctx->capturing = false;
    ctx->cg_iter_launches = ctx->cnt.launches - l0;
    cudaGraph_t captured = body;
    const cudaError_t ec = cudaStreamEndCapture(ctx->stream, &captured);
    if (st) {
      cudaGraphDestroy(g);
      return st;
    }
    if (ec != cudaSuccess) {
      cudaGraphDestroy(g);
      return check_cuda(ctx, ec, "cudaStreamEndCapture");
    }
    const cudaError_t ei = cudaGraphInstantiate(&ctx->cg_exec, g, 0);
    cudaGraphDestroy(g);
    if (ei != cudaSuccess) return check_cuda(ctx, ei, "cudaGraphInstantiate");
    ctx->cg_key = key;
  }
  FM_CUDA(ctx, cudaGraphLaunch(ctx->cg_exec, ctx->stream));
  if (int st = fetch_scalars(ctx, S_THR + 1)) return st;
  const double* hs = ctx->h_scal;
  const int64_t it = int64_t(hs[S_IT]);
  ctx->cnt.launches += (built ? it - 1 : it) * ctx->cg_iter_launches;  // kernels the graph ran
  *iters = int32_t(it);
  if (hs[S_FLAG] != 0.0) {  // !(pAp > 0): x not updated in that iteration (:38-44)
    *rel = std::sqrt(hs[S_RR]) / bnorm;
    return FM_OK;
  }
  if (std::sqrt(hs[S_RRNEW]) <= thr) {  // :49-50
    *rel = std::sqrt(hs[S_RRNEW]) / bnorm;
    return cg_finish_x(ctx, op, x, count);
  }
  *rel = std::sqrt(hs[S_RR]) / bnorm;
  const int st = set_error(ctx, FM_E_CG_STALLED, "conjugate gradient stalled after " + std::to_string(cap) + " iterations");
  ctx->last_info = fm_error_info{FM_E_CG_STALLED, int32_t(cap), -1, *rel};
  return st;
}

// cg_solve, solver.cpp:19-58.
int cg_run(fm_ctx* ctx, const Op& op, const double* b, double eta_cg, int64_t max_cg, double* x,
           int32_t* iters, double* rel) {
  const int64_t count = ctx->n * ctx->ncomp;
  if (int st = ensure_field(ctx, ctx->r, ctx->ncomp)) return st;
  if (int st = ensure_field(ctx, ctx->p, ctx->ncomp)) return st;
  if (!cg_fused(ctx))  // the fused iteration never stores Ap
    if (int st = ensure_field(ctx, ctx->Ap, ctx->ncomp)) return st;
  FM_CUDA(ctx, cudaMemsetAsync(x, 0, sizeof(double) * count, ctx->stream));  // :22
  // bnorm = |b|; rr = <r,r> with r = b  (:24, :31-33)
  if (int st = dot_async(ctx, b, b, count, ctx->d_scal + S_RR)) return st;
  if (int st = fetch_scalars(ctx, S_RR + 1)) return st;
  const double bnorm = std::sqrt(ctx->h_scal[S_RR]);
  if (bnorm == 0.0) {  // :25
    *iters = 0;
    *rel = 0.0;
    return FM_OK;
  }
  const int64_t cap = max_cg > 0 ? max_cg : ctx->n_global * ctx->ncomp;  // :27-29 (int64: no overflow past 620^3)
  if (b != ctx->r.d)  // the Newton driver builds its rhs in r directly (saves a field at 512^3)
    FM_CUDA(ctx, cudaMemcpyAsync(ctx->r.d, b, sizeof(double) * count, cudaMemcpyDeviceToDevice, ctx->stream));
  FM_CUDA(ctx, cudaMemcpyAsync(ctx->p.d, b, sizeof(double) * count, cudaMemcpyDeviceToDevice, ctx->stream));
  double rr = ctx->h_scal[S_RR];
  if (cg_small_supported(ctx)) {  // latency-bound generic grid: the whole loop in one cooperative launch
    ProArgs pa;
    pa.kind = op.kind;
    pa.K = op.K;
    pa.F = op.F;
    pa.lam = op.lam;
    pa.mu = op.mu;
    pa.lab = op.lab;
    pa.ptab = op.ptab;
    const int st = cg_small_run(ctx, pa, x, ctx->r.d, ctx->p.d, cap, eta_cg * bnorm, rr);
    if (st != FM_E_UNSUPPORTED) {
      if (st) return st;
      if (int s2 = fetch_scalars(ctx, S_OUT + 1)) return s2;
      const double* hs = ctx->h_scal;
      const int how = int(hs[S_OUT]);
      *iters = int32_t(hs[S_IT]);
      if (how == 1) {  // !(pAp > 0): x not updated in that iteration (:38-44)
        *rel = std::sqrt(hs[S_RR]) / bnorm;
        return FM_OK;
      }
      if (how == 2) {  // :49-50
        *rel = std::sqrt(hs[S_RRNEW]) / bnorm;
        return FM_OK;
      }
      *rel = std::sqrt(hs[S_RR]) / bnorm;
      const int se = set_error(ctx, FM_E_CG_STALLED,
                               "conjugate gradient stalled after " + std::to_string(cap) + " iterations");
      ctx->last_info = fm_error_info{FM_E_CG_STALLED, int32_t(cap), -1, *rel};
      return se;
    }
  }
  if (cg_graph_enabled(ctx)) return cg_loop_graph(ctx, op, x, count, cap, eta_cg * bnorm, bnorm, iters, rel);
  for (int64_t it = 1; it <= cap; ++it) {
    // :36-37 with :51-55 of the previous iteration folded in (p = beta p + r)
    if (int st = cg_iteration(ctx, op, x, count, it == 1)) return st;
    if (int st = fetch_scalars(ctx, S_FLAG + 1)) return st;
    if (ctx->h_scal[S_FLAG] != 0.0) {  // !(pAp > 0): return without updating x (:38-44)
      *iters = int32_t(it);
      *rel = std::sqrt(rr) / bnorm;
      return FM_OK;
    }
    const double rr_new = ctx->h_scal[S_RRNEW];
    if (std::sqrt(rr_new) <= eta_cg * bnorm) {  // :49-50
      *iters = int32_t(it);
      *rel = std::sqrt(rr_new) / bnorm;
      return cg_finish_x(ctx, op, x, count);
    }
    rr = rr_new;  // p *= beta; p += r happens in the next matvec's prologue
  }
  *iters = int32_t(cap);
  *rel = std::sqrt(rr) / bnorm;
  const int st = set_error(ctx, FM_E_CG_STALLED,
                           "conjugate gradient stalled after " + std::to_string(cap) + " iterations");
  ctx->last_info = fm_error_info{FM_E_CG_STALLED, int32_t(cap), -1, *rel};
  return st;
}

int model_evaluate(fm_ctx* ctx, fm_model* m, const double* F, double* P) {
  int st;
  if (m->kind == 0) {
    st = hyper_eval_async(ctx, F, m->lambda.d, m->mu.d, P, m->matrix_free ? nullptr : m->K.d);
    if (!st && m->matrix_free)
      FM_CUDA(ctx, cudaMemcpyAsync(m->F_eval.d, F, sizeof(double) * ctx->n * ctx->ncomp,
                                   cudaMemcpyDeviceToDevice, ctx->stream));
  } else {
    st = simo_eval_async(ctx, F, m->f_old.d, m->be_c.d, m->epsp_c.d, m->lambda.d, m->mu.d,
                         m->tau_y0.d, m->hard.d, P, m->compact ? nullptr : m->K.d, m->be_t.d, m->epsp_t.d,
                         m->compact ? m->Kc.d : nullptr);
  }
  if (st) return st;
  return check_bad(ctx);
}

int model_apply(fm_ctx* ctx, fm_model* m, const double* dF, double* out) {
  return op_apply(ctx, model_op(m), dF, out, 1.0);
}

int cg_run_k4(fm_ctx* ctx, const double* K, const double* b, double eta_cg, int64_t max_cg,
              double* x, int32_t* iters, double* rel) {
  Op op;
  op.kind = PRO_K4;
  op.K = K;
  return cg_run(ctx, op, b, eta_cg, max_cg, x, iters, rel);
}

int model_commit(fm_ctx* ctx, fm_model* m, const double* F) {
  if (m->kind != 1) return FM_OK;
  const size_t n = size_t(ctx->n);
  FM_CUDA(ctx, cudaMemcpyAsync(m->be_c.d, m->be_t.d, 9 * n * 8, cudaMemcpyDeviceToDevice, ctx->stream));
  FM_CUDA(ctx, cudaMemcpyAsync(m->epsp_c.d, m->epsp_t.d, n * 8, cudaMemcpyDeviceToDevice, ctx->stream));
  FM_CUDA(ctx, cudaMemcpyAsync(m->f_old.d, F, 9 * n * 8, cudaMemcpyDeviceToDevice, ctx->stream));
  return FM_OK;
}

static double det_host(const double* a, int d) {
  if (d == 2) return a[0] * a[3] - a[1] * a[2];
  return a[0] * (a[4] * a[8] - a[5] * a[7]) - a[1] * (a[3] * a[8] - a[5] * a[6]) +
         a[2] * (a[3] * a[7] - a[4] * a[6]);
}

// solve_increment, solver.cpp:73-160.
int solve_increment(fm_ctx* ctx, fm_model* m, fm_field* Ff, const double* fbar,
                    const fm_solver_params& prm, fm_report* rep, fm_field* P_out) {
  if (!(prm.eta_newton > 0.0 && prm.eta_newton < 1.0))
    return set_error(ctx, FM_E_INVALID, "eta_newton must be in (0,1)");
  if (!(prm.eta_cg > 0.0 && prm.eta_cg < 1.0)) return set_error(ctx, FM_E_INVALID, "eta_cg must be in (0,1)");
  // (any max_newton >= 1, as SolverParams::validate, solver.hpp: the report
  // keeps the per-pass record of the first FM_MAX_PASSES passes and the true
  // pass count)
  if (prm.max_newton < 1) return set_error(ctx, FM_E_INVALID, "max_newton must be >= 1");
  if (prm.max_cg < 0) return set_error(ctx, FM_E_INVALID, "max_cg must be >= 0");
  const int d = ctx->tdim, nc = ctx->ncomp;
  if (Ff->ncomp != nc) return set_error(ctx, FM_E_INVALID, "increment dimension does not match the state field");
  if (!(det_host(fbar, d) > 0.0)) return set_error(ctx, FM_E_INVALID, "det(Fbar) must be positive");
  *rep = fm_report{};
  const auto t0 = std::chrono::steady_clock::now();
  const int64_t count = ctx->n * nc;
  double* F = Ff->d;
  if (int st = ensure_field(ctx, ctx->Pw, nc)) return st;
  if (int st = ensure_field(ctx, ctx->dF, nc)) return st;
  // rhs lives in the CG residual r and the scratch field in Ap: both are CG
  // workspace that is free whenever the driver needs them.
  for (fm_field* f : {&ctx->r, &ctx->p, &ctx->Ap})
    if (int st = ensure_field(ctx, *f, nc)) return st;
  double* rhs = ctx->r.d;
  double* tmp = ctx->Ap.d;
  double* P = ctx->Pw.d;
  const auto finish = [&](bool conv) {
    rep->converged = conv ? 1 : 0;
    rep->wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  };
  double norm_ref;
  if (int st = norm_sync(ctx, F, count, &norm_ref)) return st;  // :88
  const Op op = model_op(m);
  const auto drift = [&](double* out) -> int {
    double mean[9];
    if (int st = mean_sync(ctx, F, mean)) return st;
    double dr = 0.0;
    for (int c = 0; c < nc; ++c) dr = std::max(dr, std::abs(mean[c] - fbar[c]));
    *out = dr;
    return FM_OK;
  };
  // ---- boundary-condition pass (:101-122)
  {
    if (int st = model_evaluate(ctx, m, F, P)) return st;
    double mean[9], dfbar[9];
    if (int st = mean_sync(ctx, F, mean)) return st;
    for (int c = 0; c < nc; ++c) dfbar[c] = fbar[c] - mean[c];
    if (int st = fill_uniform_async(ctx, tmp, dfbar, nc, ctx->n)) return st;
    if (int st = op_apply(ctx, op, tmp, rhs, -1.0)) return st;  // rhs = -G(K:dFbar^T)
    rep->matvecs++;
    int32_t it = 0;
    double rel = 0.0;
    if (int st = cg_run(ctx, op, rhs, prm.eta_cg, prm.max_cg, ctx->dF.d, &it, &rel)) {
      finish(false);
      return st;
    }
    rep->matvecs += it;
    if (int st = add_uniform_async(ctx, F, dfbar, nc, ctx->n)) return st;
    if (int st = add_async(ctx, F, ctx->dF.d, +1.0, count)) return st;
    double ndf;
    if (int st = norm_sync(ctx, ctx->dF.d, count, &ndf)) return st;
    rep->cg_iterations[0] = it;
    rep->cg_rel_residual[0] = rel;
    rep->rel_update[0] = ndf / norm_ref;
    rep->n_passes = 1;
    double dr;
    if (int st = drift(&dr)) return st;
    rep->max_mean_drift = std::max(rep->max_mean_drift, dr);
  }
  // ---- Newton equilibrium passes (:125-147)
  while (true) {
    if (rep->n_passes >= prm.max_newton) {
      finish(false);
      return set_error(ctx, FM_E_NEWTON_DIVERGED,
                       "Newton did not converge within " + std::to_string(rep->n_passes) + " passes");
    }
    if (int st = model_evaluate(ctx, m, F, P)) return st;
    if (int st = op_apply(ctx, Op{PRO_COPY}, P, rhs, -1.0)) return st;  // rhs = -G(P)
    int32_t it = 0;
    double rel = 0.0;
    if (int st = cg_run(ctx, op, rhs, prm.eta_cg, prm.max_cg, ctx->dF.d, &it, &rel)) {
      finish(false);
      return st;
    }
    rep->matvecs += it;
    if (int st = add_async(ctx, F, ctx->dF.d, +1.0, count)) return st;
    double ndf;
    if (int st = norm_sync(ctx, ctx->dF.d, count, &ndf)) return st;
    const double ru = ndf / norm_ref;
    const int k = rep->n_passes++;
    if (k < FM_MAX_PASSES) {
      rep->cg_iterations[k] = it;
      rep->cg_rel_residual[k] = rel;
      rep->rel_update[k] = ru;
    }
    double dr;
    if (int st = drift(&dr)) return st;
    rep->max_mean_drift = std::max(rep->max_mean_drift, dr);
    if (ru < prm.eta_newton) break;
  }
  // ---- refresh at the converged state, residual, commit (:151-155)
  if (int st = model_evaluate(ctx, m, F, P)) return st;
  double pnorm;
  if (int st = norm_sync(ctx, P, count, &pnorm)) return st;
  if (pnorm > 0.0) {
    if (int st = op_apply(ctx, Op{PRO_COPY}, P, tmp, 1.0)) return st;
    double gn;
    if (int st = norm_sync(ctx, tmp, count, &gn)) return st;
    rep->equilibrium_rel_residual = gn / pnorm;
  }
  if (int st = model_commit(ctx, m, F)) return st;
  if (P_out)
    FM_CUDA(ctx, cudaMemcpyAsync(P_out->d, P, sizeof(double) * count, cudaMemcpyDeviceToDevice, ctx->stream));
  FM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  finish(true);
  return FM_OK;
}

}  // namespace fm
