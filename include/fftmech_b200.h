/*
 * fftmech_b200.h -- C ABI of the B200-native (sm_100a) hot path of the
 * Galerkin-FFT finite-strain homogenisation solver (arXiv 1603.08893).
 *
 * The reference `fftmech` core exposes a C++ surface; this
 * ABI is what that surface (re-created in paper_1603_08893_b200/host/) and any
 * other FFI binds.  Plain pointers and sizes only; every call returns an
 * fm_status.  All fields live in device memory in the reference layout:
 * component-major slabs of n = node_count doubles, slab (i,j) at (i*tdim+j)*n,
 * fourth-order slab ((i*d+j)*d+k)*d+l (fields.hpp:41-139), nodes row-major
 * with the last axis fastest (grid.hpp:26-39).
 *
 * Threading: one host thread drives one context; calls are stream-ordered on
 * the context's stream, and calls returning host scalars synchronise.
 */
#ifndef FFTMECH_B200_H
#define FFTMECH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; the host C++ layer maps them onto the reference exception
 * hierarchy (errors.hpp:11-111, solver.hpp:60-78). */
typedef enum fm_status {
  FM_OK = 0,
  FM_E_INVALID = 1,         /* std::invalid_argument (shape/argument mismatch) */
  FM_E_CUDA = 2,            /* fftmech::Error (device failure) */
  FM_E_OOM = 3,             /* fftmech::Error (device allocation) */
  FM_E_INVERTED = 4,        /* InvertedElement(node)            errors.hpp:57-62 */
  FM_E_NOT_SPD = 5,         /* NotPositiveDefinite(node, value) errors.hpp:32-41 */
  FM_E_SINGULAR = 6,        /* SingularTensor(node)             errors.hpp:17-22 */
  FM_E_CG_STALLED = 7,      /* CgStalled(iterations, residual)  solver.hpp:69-78 */
  FM_E_COMPLEX_RESIDUE = 8, /* ComplexResidue                   errors.hpp:45-54 */
  FM_E_NEWTON_DIVERGED = 9, /* NewtonDiverged(report)           solver.hpp:60-67 */
  FM_E_NCCL = 10,           /* fftmech::Error (collective failure) */
  FM_E_UNSUPPORTED = 11     /* configuration outside what the kernels implement */
} fm_status;

/* NyquistMode, projection.hpp:12-15 */
enum { FM_NYQUIST_ZERO_COMPATIBLE = 0, FM_NYQUIST_IDENTITY_EQUILIBRIUM = 1 };

typedef struct fm_ctx fm_ctx;
typedef struct fm_field fm_field;
typedef struct fm_model fm_model;

/* Error detail of the last failing call (node-indexed errors report the
 * lowest offending node, i.e. the reference's first throw in node order). */
typedef struct fm_error_info {
  int32_t status;
  int32_t cg_iterations; /* FM_E_CG_STALLED */
  int64_t node;          /* FM_E_INVERTED / FM_E_NOT_SPD / FM_E_SINGULAR */
  double value;          /* eigenvalue (NOT_SPD) or relative residual (CG) */
} fm_error_info;

/* SolverParams, solver.hpp:15-22 */
typedef struct fm_solver_params {
  double eta_newton;  /* default 1e-5 */
  double eta_cg;      /* default 1e-8 */
  int32_t max_newton; /* default 30; any value >= 1 */
  int32_t max_cg;     /* 0 = n * tdim^2 */
} fm_solver_params;

#define FM_MAX_PASSES 64

/* SolveReport + NewtonPass, solver.hpp:34-58 */
typedef struct fm_report {
  int32_t n_passes; /* true pass count; the arrays record the first FM_MAX_PASSES passes */
  int32_t converged;
  int32_t cg_iterations[FM_MAX_PASSES];
  double cg_rel_residual[FM_MAX_PASSES];
  double rel_update[FM_MAX_PASSES];
  double equilibrium_rel_residual;
  double max_mean_drift;
  double wall_seconds;
  int64_t matvecs; /* matvecs issued (CG iterations + BC rhs), for throughput */
} fm_report;

/* ---- context ------------------------------------------------------------
 * Replaces build_projection (projection.hpp:65-66, projection.cpp:72-121):
 * the context owns the grid, the per-axis FFT plans and twiddles, the
 * spectral workspace and one CUDA stream on `device`.  The ĝ kernel is never
 * stored; it is evaluated from the wave vector inside the x pass.
 * dim in {2,3}; points/lengths have `dim` entries; tdim in [dim, 3]. */
int fm_ctx_create(int dim, const int32_t* points, const double* lengths, int tdim,
                  int nyquist_mode, int device, fm_ctx** out);
int fm_ctx_destroy(fm_ctx* ctx);
const char* fm_last_error(const fm_ctx* ctx);
int fm_last_error_info(const fm_ctx* ctx, fm_error_info* out);
int64_t fm_ctx_nodes(const fm_ctx* ctx);
int fm_ctx_tdim(const fm_ctx* ctx);
int fm_ctx_synchronize(fm_ctx* ctx);
/* cudaStream_t of the context, for callers that time with events. */
void* fm_ctx_stream(fm_ctx* ctx);
/* Per-pass CUDA-event timing of the projection passes (z fwd, y fwd,
 * x+ghat, y inv, z inv): enable/disable (resets the totals), then read the
 * accumulated milliseconds per pass and the number of timed applications. */
int fm_ctx_profile(fm_ctx* ctx, int enable);
int fm_ctx_profile_read(fm_ctx* ctx, double* ms /* 5 */, int64_t* calls);
/* Number of this library's kernels launched on the context so far. */
int64_t fm_ctx_launch_count(const fm_ctx* ctx);
/* Distinct names of the kernels launched on the context so far, comma
 * separated into buf (NUL-terminated, truncated to cap); returns the full
 * length.  Evidence of which kernel variants a call actually ran. */
int fm_ctx_kernel_names(const fm_ctx* ctx, char* buf, int cap);

/* ---- slab decomposition ---------------------------------
 * Rank r of P owns x-planes [r Nx/P, (r+1) Nx/P) of every field; the
 * projection runs its z/y passes on the x-slab and its x pass on the y-slab.
 * The two slab transposes are fused into the passes that produce the data:
 * the forward y pass and the x pass store every element straight into the
 * buffer of the rank that owns it next (peer memory over NVLink / NVSwitch,
 * mapped with CUDA IPC at context creation), with one cross-rank barrier
 * after each.  Nx and Ny must be divisible by P (P <= 16); CG scalars are
 * combined across ranks in rank order (deterministic). */
/* One rank per device.  `points` is the GLOBAL grid; fields created on this
 * context hold the local slab (Nx/P * Ny * Nz nodes per component).
 * nccl_unique_id: the 128-byte id from fm_nccl_unique_id on rank 0 (NCCL
 * carries the IPC handle exchange, the barriers and the CG scalars). */
int fm_ctx_create_dist(int dim, const int32_t* points, const double* lengths, int tdim, int nyquist_mode,
                       int device, int nranks, int rank, const void* nccl_unique_id, fm_ctx** out);
int fm_nccl_unique_id(void* out, int bytes);
/* Virtual ranks: run all P slab ranks on this one device (their buffers side
 * by side, the same transpose-fused kernels storing across them) -- validates
 * the decomposition against P = 1 bit for bit. */
/* Debug mode (also FM_DEBUG_RESIDUE=1 at creation): every projection checks
 * the imaginary residue that apply_projection checks after its c2c inverse
 * transform (projection.cpp:157-169) and fails with FM_E_COMPLEX_RESIDUE above
 * 1e-10 ||A||.  With the half spectrum kept here the residue can only come from
 * the self-conjugate kz planes, whose lines must be real before the c2r pass;
 * fm_last_error_info().value then holds the residue of the last projection. */
int fm_ctx_set_debug(fm_ctx* ctx, int residue_check);
int fm_ctx_set_virtual_ranks(fm_ctx* ctx, int P);
/* How the two slab transposes of a P > 1 projection are done (replaces the
 * single-process FFTW plans of projection.cpp:106-119 across ranks):
 * 0 (default) fused into the forward y pass and the x pass as stores into the
 * peers' buffers (NVLink, CUDA IPC); 1 the textbook form -- local passes,
 * pack, grouped ncclSend/ncclRecv all-to-all, unpack (SURVEY.md §8(e) steps 2
 * and 4) -- kept as the arm to measure the fused form against and for ranks
 * without peer access.  Distributed contexts take their mode from the
 * environment (FM_TRANSPOSE=nccl) at creation; virtual-rank contexts can
 * switch at any time. */
int fm_ctx_set_transpose(fm_ctx* ctx, int mode);
int fm_ctx_ranks(const fm_ctx* ctx, int* nranks, int* rank, int* virtual_mode);
/* Route of the fused transpose (host only, no device needed), the same
 * function the kernels evaluate.  dir +1 (forward y pass of x-slab `src`):
 * element (comp, xl = i0, y = i1, kz) -> rank *dst_rank, complex-element
 * index *dst_index in its x-pass input [c][x][yl][kz].  dir -1 (x pass of
 * y-slab `src`): element (comp, x = i0, yl = i1, kz) -> rank *dst_rank, index
 * in its spectrum [c][xl][y][kz]. */
int fm_dist_route(int P, int Nx, int Ny, int nzh, int ncomp, int dir, int src, int comp, int i0, int i1, int kz,
                  int32_t* dst_rank, int64_t* dst_index);

/* ---- fields -------------------------------------------------------------- */
int fm_field_alloc(fm_ctx* ctx, int ncomp, fm_field** out);
int fm_field_free(fm_ctx* ctx, fm_field* f);
double* fm_field_device_ptr(fm_field* f);
int fm_field_upload(fm_ctx* ctx, fm_field* f, const double* host, int64_t count);
int fm_field_download(fm_ctx* ctx, const fm_field* f, double* host, int64_t count);
int fm_field_fill(fm_ctx* ctx, fm_field* f, double value);
int fm_field_copy(fm_ctx* ctx, const fm_field* src, fm_field* dst);

/* ---- projection (hot path) ----------------------------------------------
 * apply_projection, projection.hpp:72 / projection.cpp:123-171:
 * out = Re F^-1{ Ahat_il ghat_lj } / n. */
int fm_projection_apply(fm_ctx* ctx, const fm_field* A, fm_field* out);
/* apply_projected_tangent, projection.hpp:76-77 / projection.cpp:173-194:
 * out = G(dP), dP_ij = K_jikl dF_kl, fused into the first FFT pass. */
int fm_projected_tangent_apply(fm_ctx* ctx, const fm_field* K, const fm_field* dF, fm_field* out);

/* ---- constitutive updates -------------------------------------------------
 * hyperelastic_evaluate, hyperelastic.hpp:13-14 / hyperelastic.cpp:10-65.
 * lambda, mu: 1-component fields.  K may be NULL (stress only). */
int fm_hyper_evaluate(fm_ctx* ctx, const fm_field* F, const fm_field* lambda, const fm_field* mu,
                      fm_field* P, fm_field* K);
/* simo_evaluate, simo.hpp:17-21 / simo.cpp:26-196 (tdim must be 3). */
int fm_simo_evaluate(fm_ctx* ctx, const fm_field* F, const fm_field* F_old,
                     const fm_field* be_committed, const fm_field* epsp_committed,
                     const fm_field* lambda, const fm_field* mu, const fm_field* tau_y0,
                     const fm_field* hardening, fm_field* P, fm_field* K, fm_field* be_trial,
                     fm_field* epsp_trial);

/* ---- output measures -----------------------------------
 * equivalent_stress, material.cpp:14-31, of
 *   FM_EQ_TENSOR    : T = P itself (F unused, may be NULL);
 *   FM_EQ_PK2       : S = F^-1 P   HyperelasticModel::equivalent_stress_field,
 *                     hyperelastic.cpp:89-92 (FM_E_SINGULAR at the first node
 *                     with |det F| < 1e-30, tensor_ops.cpp:257-266);
 *   FM_EQ_KIRCHHOFF : tau = P F^T  SimoPlasticityModel::equivalent_stress_field,
 *                     simo.cpp:225-228.
 * out: 1-component field. */
enum { FM_EQ_TENSOR = 0, FM_EQ_PK2 = 1, FM_EQ_KIRCHHOFF = 2 };
int fm_equivalent_stress(fm_ctx* ctx, const fm_field* F, const fm_field* P, int kind, fm_field* out);

/* ---- BLAS-1 / reductions (fields.cpp:14-67, tensor_ops.cpp:276-294) ------
 * Deterministic: fixed-order block partials then a fixed-order final sum. */
int fm_dot(fm_ctx* ctx, const fm_field* a, const fm_field* b, double* out);
int fm_norm(fm_ctx* ctx, const fm_field* a, double* out);
int fm_mean(fm_ctx* ctx, const fm_field* a, double* out /* ncomp */);
int fm_axpy(fm_ctx* ctx, double a, const fm_field* x, fm_field* y);
int fm_scale(fm_ctx* ctx, fm_field* x, double s);
int fm_add(fm_ctx* ctx, fm_field* y, const fm_field* x, double sign /* +1 or -1 */);
int fm_add_uniform(fm_ctx* ctx, fm_field* f, const double* t /* ncomp */);

/* ---- solver -------------------------------------------------------------
 * cg_solve, solver.hpp:111-112 / solver.cpp:19-58, with the projected
 * tangent operator of K. Returns FM_E_CG_STALLED at the cap. */
int fm_cg_solve(fm_ctx* ctx, const fm_field* K, const fm_field* rhs, double eta_cg,
                int64_t max_cg, fm_field* x, int32_t* iterations, double* rel_residual);

/* MaterialModel (material.hpp:45-65) on the device.  Parameters are per-node
 * host arrays of n doubles (bind_parameters, microstructure.cpp:176-203).
 * matrix_free = 1 keeps no K4: the SVK tangent action
 *   dP = lam tr(F^T dF) F + mu F dF^T F + mu F F^T dF + dF S
 * is recomputed from F inside the first FFT pass. */
int fm_model_create_hyper(fm_ctx* ctx, const double* lambda, const double* mu, int matrix_free,
                          fm_model** out);
int fm_model_create_simo(fm_ctx* ctx, const double* lambda, const double* mu,
                         const double* tau_y0, const double* hardening, fm_model** out);
int fm_model_destroy(fm_ctx* ctx, fm_model* m);
/* MaterialModel::evaluate -> P and (unless matrix-free) the model-owned K. */
int fm_model_evaluate(fm_ctx* ctx, fm_model* m, const fm_field* F, fm_field* P);
/* MaterialModel::commit (simo.cpp:220-223); no-op for hyperelastic. */
int fm_model_commit(fm_ctx* ctx, fm_model* m, const fm_field* F);
/* Tangent storage of a Simo model: 0 = K4 (81 slabs, the reference form,
 * default), 1 = compact eigenbasis form (45 slabs: V, U = F^-1 V and three
 * 3x3 coefficient sets; the matvec forms dP = V W U^T) -- what lets the
 * 512^3 J2 configuration fit on one B200.  K4 is then not materialised. */
int fm_model_set_tangent_form(fm_ctx* ctx, fm_model* m, int form);
/* Model-owned tangent field (NULL when matrix-free or compact). */
fm_field* fm_model_tangent(fm_model* m);
/* History access (Simo): which = 0 committed, 1 trial; be has 9n, epsp n. */
int fm_model_get_history(fm_ctx* ctx, fm_model* m, int which, double* be, double* epsp);
int fm_model_set_history(fm_ctx* ctx, fm_model* m, const double* be, const double* epsp,
                         const double* f_old);
/* Matvec of the model's current tangent: out = G(K : dF^T). */
int fm_model_apply(fm_ctx* ctx, fm_model* m, const fm_field* dF, fm_field* out);

/* solve_increment, solver.hpp:120-122 / solver.cpp:73-160, fully
 * device-resident: F (in/out) is a device field; fbar has tdim*tdim entries;
 * P_out (nullable) receives the converged P. */
int fm_solve_increment(fm_ctx* ctx, fm_model* m, fm_field* F, const double* fbar,
                       const fm_solver_params* params, fm_report* report, fm_field* P_out);

#ifdef __cplusplus
}
#endif
#endif /* FFTMECH_B200_H */
