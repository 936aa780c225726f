// Drop-in Newton / CG drivers.  The device-resident path (fm_solve_increment,
// fm_cg_solve) carries the reference control flow of solver.cpp:19-160; this
// file maps host fields and reports onto it, plus a path for user-defined
// host MaterialModel / LinearOperator subclasses whose vectors still live on
// the device.
#include "fftmech/solver.hpp"

#include <chrono>
#include <cmath>
#include <stdexcept>

#include "device.hpp"
#include "fftmech/tensor_ops.hpp"

namespace fftmech {

void SolverParams::validate() const {
  if (!(eta_newton > 0.0 && eta_newton < 1.0)) throw std::invalid_argument("eta_newton must be in (0,1)");
  if (!(eta_cg > 0.0 && eta_cg < 1.0)) throw std::invalid_argument("eta_cg must be in (0,1)");
  if (max_newton < 1) throw std::invalid_argument("max_newton must be >= 1");
  if (max_cg < 0) throw std::invalid_argument("max_cg must be >= 0");
}

namespace {

fm_solver_params to_abi(const SolverParams& p) { return fm_solver_params{p.eta_newton, p.eta_cg, p.max_newton, p.max_cg}; }

SolveReport to_report(const fm_report& r, const Increment& inc) {
  SolveReport out;
  out.label = inc.label;
  out.fbar = inc.fbar;
  // the ABI records the first FM_MAX_PASSES passes in detail; later ones count as passes without a record
  for (int k = 0; k < r.n_passes; ++k)
    out.passes.push_back(k < FM_MAX_PASSES ? NewtonPass{r.cg_iterations[k], r.cg_rel_residual[k], r.rel_update[k]}
                                           : NewtonPass{0, 0.0, 0.0});
  out.equilibrium_rel_residual = r.equilibrium_rel_residual;
  out.max_mean_drift = r.max_mean_drift;
  out.wall_seconds = r.wall_seconds;
  out.converged = r.converged != 0;
  return out;
}

// CG on the device for an arbitrary host LinearOperator: vectors and
// reductions stay in HBM; only p / Ap cross the bus for op.apply.
CgResult cg_generic(const LinearOperator& op, const Tensor2Field& rhs, const SolverParams& params, Tensor2Field& x) {
  const int d = rhs.tdim(), nc = d * d;
  auto dev = detail::device_for(rhs.shape(), d, 0);
  fm_ctx* h = dev->h;
  detail::DevField b(dev, nc), xd(dev, nc), r(dev, nc), p(dev, nc), ap(dev, nc);
  b.upload(rhs.data());
  x = Tensor2Field(rhs.shape(), d);
  double bnorm = 0.0;
  detail::check(h, fm_norm(h, b.get(), &bnorm), "cg");
  if (bnorm == 0.0) return {0, 0.0};
  const long cap = params.max_cg > 0 ? params.max_cg : static_cast<long>(rhs.nodes()) * nc;
  detail::check(h, fm_field_copy(h, b.get(), r.get()), "cg");
  detail::check(h, fm_field_copy(h, b.get(), p.get()), "cg");
  double rr = 0.0;
  detail::check(h, fm_dot(h, r.get(), r.get(), &rr), "cg");
  Tensor2Field ph(rhs.shape(), d);
  for (long it = 1; it <= cap; ++it) {
    p.download(ph.data());
    ap.upload(op.apply(ph).data());
    double pAp = 0.0;
    detail::check(h, fm_dot(h, p.get(), ap.get(), &pAp), "cg");
    if (!(pAp > 0.0)) {
      xd.download(x.data());
      return {static_cast<int>(it), std::sqrt(rr) / bnorm};
    }
    const double alpha = rr / pAp;
    detail::check(h, fm_axpy(h, alpha, p.get(), xd.get()), "cg");
    detail::check(h, fm_axpy(h, -alpha, ap.get(), r.get()), "cg");
    double rr_new = 0.0;
    detail::check(h, fm_dot(h, r.get(), r.get(), &rr_new), "cg");
    if (std::sqrt(rr_new) <= params.eta_cg * bnorm) {
      xd.download(x.data());
      return {static_cast<int>(it), std::sqrt(rr_new) / bnorm};
    }
    const double beta = rr_new / rr;
    rr = rr_new;
    detail::check(h, fm_scale(h, p.get(), beta), "cg");
    detail::check(h, fm_add(h, p.get(), r.get(), 1.0), "cg");
  }
  throw CgStalled(static_cast<int>(cap), std::sqrt(rr) / bnorm);
}

// Newton increment for a user-defined host MaterialModel: the constitutive
// update runs on the host (user code), projection and CG on the device.
SolveReport solve_host_model(Tensor2Field& F, MaterialModel& model, const ProjectionOperator& G, const Increment& inc,
                             const SolverParams& params, Tensor2Field* P_out) {
  const auto t0 = std::chrono::steady_clock::now();
  SolveReport rep;
  rep.label = inc.label;
  rep.fbar = inc.fbar;
  const auto stamp = [&](bool ok) {
    rep.converged = ok;
    rep.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  };
  const auto drift = [&]() {
    const Tensor2 m = field_mean(F);
    double dmax = 0.0;
    for (int c = 0; c < inc.fbar.dim * inc.fbar.dim; ++c) dmax = std::max(dmax, std::abs(m.v[c] - inc.fbar.v[c]));
    return dmax;
  };
  const double ref = field_norm(F);
  Tensor2Field P(F.shape(), F.tdim()), dF;
  Tensor4Field K(F.shape(), F.tdim());
  for (int pass = 0;; ++pass) {
    if (pass > 0 && rep.newton_iterations() >= params.max_newton) {
      stamp(false);
      throw NewtonDiverged(rep);
    }
    model.evaluate(F, P, K);
    Tensor2Field rhs;
    Tensor2 jump(F.tdim());
    if (pass == 0) {  // boundary-condition pass distributes Fbar - <F>
      jump = inc.fbar - field_mean(F);
      Tensor2Field u(F.shape(), F.tdim());
      u.add_uniform(jump);
      rhs = apply_projected_tangent(G, K, u);
    } else {
      rhs = apply_projection(G, P);
    }
    rhs *= -1.0;
    CgResult cg;
    try {
      cg = cg_solve(ProjectedTangentOperator(G, K), rhs, params, dF);
    } catch (...) {
      stamp(false);
      throw;
    }
    if (pass == 0) F.add_uniform(jump);
    F += dF;
    const double rel = field_norm(dF) / ref;
    rep.passes.push_back({cg.iterations, cg.rel_residual, rel});
    rep.max_mean_drift = std::max(rep.max_mean_drift, drift());
    if (pass > 0 && rel < params.eta_newton) break;
  }
  model.evaluate(F, P, K);
  const double pn = field_norm(P);
  rep.equilibrium_rel_residual = pn > 0.0 ? field_norm(apply_projection(G, P)) / pn : 0.0;
  model.commit(F);
  if (P_out) *P_out = P;
  stamp(true);
  return rep;
}

}  // namespace

CgResult cg_solve(const LinearOperator& op, const Tensor2Field& rhs, const SolverParams& params, Tensor2Field& x) {
  params.validate();
  const auto* pto = dynamic_cast<const ProjectedTangentOperator*>(&op);
  if (!pto) return cg_generic(op, rhs, params, x);
  const auto& dev = pto->projection().device();
  const int d = rhs.tdim(), nc = d * d;
  if (!(rhs.shape() == pto->projection().shape()) || d != pto->projection().tdim())
    throw std::invalid_argument("cg_solve: rhs does not match the operator");
  detail::DevField k(dev, nc * nc), b(dev, nc), xd(dev, nc);
  k.upload(pto->tangent().data());
  b.upload(rhs.data());
  int32_t it = 0;
  double rel = 0.0;
  const int st = fm_cg_solve(dev->h, k.get(), b.get(), params.eta_cg, params.max_cg, xd.get(), &it, &rel);
  if (st == FM_E_CG_STALLED) throw CgStalled(it, rel);
  detail::check(dev->h, st, "cg_solve");
  x = Tensor2Field(rhs.shape(), d);
  xd.download(x.data());
  return {it, rel};
}

SolveReport solve_increment(Tensor2Field& F, MaterialModel& model, const ProjectionOperator& G, const Increment& inc,
                            const SolverParams& params, Tensor2Field* P_converged) {
  params.validate();
  if (inc.fbar.dim != F.tdim()) throw std::invalid_argument("increment dimension does not match the state field");
  if (!(inc.fbar.det() > 0.0)) throw std::invalid_argument("det(Fbar) must be positive");
  const auto& dev = G.device();
  fm_model* dm = model.device_model(dev);
  if (!dm) return solve_host_model(F, model, G, inc, params, P_converged);
  const int d = F.tdim(), nc = d * d;
  detail::DevField f(dev, nc), p(dev, nc);
  f.upload(F.data());
  const fm_solver_params prm = to_abi(params);
  fm_report rep{};
  const int st = fm_solve_increment(dev->h, dm, f.get(), inc.fbar.v.data(), &prm, &rep, p.get());
  f.download(F.data());  // like the reference, F holds the last state even on failure
  if (st == FM_E_NEWTON_DIVERGED) throw NewtonDiverged(to_report(rep, inc));
  detail::check(dev->h, st, "solve_increment");
  model.device_committed(F);
  if (P_converged) {
    *P_converged = Tensor2Field(F.shape(), d);
    p.download(P_converged->data());
  }
  return to_report(rep, inc);
}

void run_program(Tensor2Field& F, MaterialModel& model, const ProjectionOperator& G, const LoadProgram& program,
                 const SolverParams& params, ProgramSink& sink) {
  for (std::size_t idx = 0; idx < program.size(); ++idx) {
    Tensor2Field P;
    const SolveReport report = solve_increment(F, model, G, program[idx], params, &P);
    sink.on_increment(idx, program[idx], report, F, P, model);
  }
}

}  // namespace fftmech
