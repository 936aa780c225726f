// Drop-in constitutive models backed by the sm_100a kernels (reference:
// hyperelastic.cpp:10-92, simo.cpp:26-228, material.cpp:11-31).
#include <algorithm>
#include <cmath>
#include <memory>
#include <stdexcept>

#include "device.hpp"
#include "fftmech/hyperelastic.hpp"
#include "fftmech/simo.hpp"
#include "fftmech/tensor_ops.hpp"

namespace fftmech {

HistoryState::HistoryState(const GridShape& shape, int tdim) : be(identity2(shape, tdim)), eps_p(shape, 0.0) {}

namespace {
// Output measures on the device (fm_equivalent_stress): compat-mode upload of
// the host fields, one kernel sweep, download of the scalar field.
ScalarField device_equivalent_stress(const Tensor2Field* F, const Tensor2Field& P, int kind, const char* where) {
  const int d = P.tdim();
  auto dev = detail::device_for(P.shape(), d, 0);
  detail::DevField p(dev, d * d), out(dev, 1);
  p.upload(P.data());
  std::unique_ptr<detail::DevField> f;
  if (F) {
    if (F->nodes() != P.nodes() || F->tdim() != d) throw std::invalid_argument(std::string(where) + ": size mismatch");
    f = std::make_unique<detail::DevField>(dev, d * d);
    f->upload(F->data());
  }
  detail::check(dev->h, fm_equivalent_stress(dev->h, f ? f->get() : nullptr, p.get(), kind, out.get()), where);
  ScalarField eq(P.shape());
  out.download(eq.data());
  return eq;
}
}  // namespace

ScalarField equivalent_stress(const Tensor2Field& T) {
  return device_equivalent_stress(nullptr, T, FM_EQ_TENSOR, "equivalent_stress");
}

double macroscopic_equivalent_strain(const Tensor2& fbar) {
  double f[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int i = 0; i < fbar.dim; ++i)
    for (int j = 0; j < fbar.dim; ++j) f[i][j] = fbar(i, j);
  double c[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) c[i][j] = f[0][i] * f[0][j] + f[1][i] * f[1][j] + f[2][i] * f[2][j];
  // cyclic Jacobi on the symmetric 3x3 (eigenvalues only)
  for (int sweep = 0; sweep < 64; ++sweep) {
    const double off = c[0][1] * c[0][1] + c[0][2] * c[0][2] + c[1][2] * c[1][2];
    const double dg = c[0][0] * c[0][0] + c[1][1] * c[1][1] + c[2][2] * c[2][2];
    if (off == 0.0 || off < 1e-36 * dg) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        if (c[p][q] == 0.0) continue;
        const double th = (c[q][q] - c[p][p]) / (2.0 * c[p][q]);
        const double t = (th >= 0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(th * th + 1.0));
        const double cs = 1.0 / std::sqrt(t * t + 1.0), sn = t * cs;
        for (int k = 0; k < 3; ++k) {
          const double a = c[k][p], b = c[k][q];
          c[k][p] = cs * a - sn * b;
          c[k][q] = sn * a + cs * b;
        }
        for (int k = 0; k < 3; ++k) {
          const double a = c[p][k], b = c[q][k];
          c[p][k] = cs * a - sn * b;
          c[q][k] = sn * a + cs * b;
        }
      }
  }
  double lam[3] = {c[0][0], c[1][1], c[2][2]};
  std::sort(lam, lam + 3);
  double le[3];
  for (int i = 0; i < 3; ++i) le[i] = 0.5 * std::log(lam[i]);
  const double tr = (le[0] + le[1] + le[2]) / 3.0;
  double s = 0.0;
  for (int i = 0; i < 3; ++i) s += (le[i] - tr) * (le[i] - tr);
  return std::sqrt(2.0 / 3.0 * s);
}

// ------------------------------------------------------------ hyperelastic
void hyperelastic_evaluate(const Tensor2Field& F, const ScalarField& lambda, const ScalarField& mu, Tensor2Field& P,
                           Tensor4Field& K) {
  if (lambda.nodes() != F.nodes() || mu.nodes() != F.nodes())
    throw std::invalid_argument("hyperelastic_evaluate: parameter field size mismatch");
  const int d = F.tdim();
  auto dev = detail::device_for(F.shape(), d, 0);
  detail::DevField f(dev, d * d), l(dev, 1), m(dev, 1), p(dev, d * d), k(dev, d * d * d * d);
  f.upload(F.data());
  l.upload(lambda.data());
  m.upload(mu.data());
  detail::check(dev->h, fm_hyper_evaluate(dev->h, f.get(), l.get(), m.get(), p.get(), k.get()), "hyperelastic_evaluate");
  P = Tensor2Field(F.shape(), d);
  K = Tensor4Field(F.shape(), d);
  p.download(P.data());
  k.download(K.data());
}

void hyperelastic_evaluate(const Tensor2Field& F, const ElasticParams& params, Tensor2Field& P, Tensor4Field& K) {
  hyperelastic_evaluate(F, ScalarField(F.shape(), params.lame_lambda()), ScalarField(F.shape(), params.lame_mu()), P, K);
}

HyperelasticModel::HyperelasticModel(const GridShape& shape, int tdim, ScalarField lambda, ScalarField mu)
    : shape_(shape), tdim_(tdim), lambda_(std::move(lambda)), mu_(std::move(mu)) {}

HyperelasticModel::HyperelasticModel(const GridShape& shape, int tdim, const ElasticParams& params)
    : HyperelasticModel(shape, tdim, ScalarField(shape, params.lame_lambda()), ScalarField(shape, params.lame_mu())) {}

HyperelasticModel::~HyperelasticModel() {
  if (dm_) fm_model_destroy(dev_->h, dm_);
}

void HyperelasticModel::set_matrix_free(bool on) {
  if (on == matrix_free_) return;
  matrix_free_ = on;
  if (dm_) fm_model_destroy(dev_->h, dm_);
  dm_ = nullptr;
}

fm_model* HyperelasticModel::device_model(const std::shared_ptr<detail::Device>& dev) {
  if (dm_ && dev_ == dev) return dm_;
  if (dm_) fm_model_destroy(dev_->h, dm_);
  dm_ = nullptr;
  dev_ = dev;
  detail::check(dev->h, fm_model_create_hyper(dev->h, lambda_.data().data(), mu_.data().data(), matrix_free_ ? 1 : 0, &dm_),
                "HyperelasticModel");
  return dm_;
}

void HyperelasticModel::evaluate(const Tensor2Field& F, Tensor2Field& P, Tensor4Field& K) {
  if (F.tdim() != tdim_ || !(F.shape() == shape_)) throw std::invalid_argument("evaluate: field does not match model");
  if (matrix_free_) {  // the host API always returns K: evaluate it explicitly
    hyperelastic_evaluate(F, lambda_, mu_, P, K);
    return;
  }
  auto dev = dev_ ? dev_ : detail::device_for(shape_, tdim_, 0);
  fm_model* dm = device_model(dev);
  detail::DevField f(dev, tdim_ * tdim_), p(dev, tdim_ * tdim_);
  f.upload(F.data());
  detail::check(dev->h, fm_model_evaluate(dev->h, dm, f.get(), p.get()), "HyperelasticModel::evaluate");
  P = Tensor2Field(F.shape(), tdim_);
  K = Tensor4Field(F.shape(), tdim_);
  p.download(P.data());
  detail::check(dev->h, fm_field_download(dev->h, fm_model_tangent(dm), K.data().data(), int64_t(K.size())), "tangent");
}

ScalarField HyperelasticModel::equivalent_stress_field(const Tensor2Field& F, const Tensor2Field& P) const {
  return device_equivalent_stress(&F, P, FM_EQ_PK2, "equivalent_stress_field");  // S = F^-1 P
}

// -------------------------------------------------------------------- Simo
void simo_evaluate(const Tensor2Field& F, const Tensor2Field& F_old, const HistoryState& committed,
                   const ScalarField& lambda, const ScalarField& mu, const ScalarField& tau_y0,
                   const ScalarField& hardening, Tensor2Field& P, Tensor4Field& K, HistoryState& trial) {
  if (F.tdim() != 3) throw std::invalid_argument("simo_evaluate: tensors must be 3x3");
  const std::size_t n = F.nodes();
  if (F_old.nodes() != n || committed.be.nodes() != n || committed.eps_p.nodes() != n)
    throw std::invalid_argument("simo_evaluate: state size mismatch");
  auto dev = detail::device_for(F.shape(), 3, 0);
  detail::DevField f(dev, 9), fo(dev, 9), bc(dev, 9), ec(dev, 1), l(dev, 1), m(dev, 1), ty(dev, 1), h(dev, 1);
  detail::DevField p(dev, 9), k(dev, 81), bt(dev, 9), et(dev, 1);
  f.upload(F.data());
  fo.upload(F_old.data());
  bc.upload(committed.be.data());
  ec.upload(committed.eps_p.data());
  l.upload(lambda.data());
  m.upload(mu.data());
  ty.upload(tau_y0.data());
  h.upload(hardening.data());
  detail::check(dev->h,
                fm_simo_evaluate(dev->h, f.get(), fo.get(), bc.get(), ec.get(), l.get(), m.get(), ty.get(), h.get(),
                                 p.get(), k.get(), bt.get(), et.get()),
                "simo_evaluate");
  P = Tensor2Field(F.shape(), 3);
  K = Tensor4Field(F.shape(), 3);
  trial = HistoryState(F.shape(), 3);
  p.download(P.data());
  k.download(K.data());
  bt.download(trial.be.data());
  et.download(trial.eps_p.data());
}

SimoPlasticityModel::SimoPlasticityModel(const GridShape& shape, ScalarField lambda, ScalarField mu, ScalarField tau_y0,
                                         ScalarField hardening)
    : shape_(shape),
      lambda_(std::move(lambda)),
      mu_(std::move(mu)),
      tau_y0_(std::move(tau_y0)),
      hardening_(std::move(hardening)),
      committed_(shape, 3),
      trial_(shape, 3),
      f_old_(identity2(shape, 3)) {}

SimoPlasticityModel::SimoPlasticityModel(const GridShape& shape, const PlasticParams& p)
    : SimoPlasticityModel(shape, ScalarField(shape, p.elastic.lame_lambda()), ScalarField(shape, p.elastic.lame_mu()),
                          ScalarField(shape, p.tau_y0), ScalarField(shape, p.hardening)) {}

SimoPlasticityModel::~SimoPlasticityModel() {
  if (dm_) fm_model_destroy(dev_->h, dm_);
}

fm_model* SimoPlasticityModel::device_model(const std::shared_ptr<detail::Device>& dev) {
  if (dm_ && dev_ == dev) return dm_;
  if (dm_) {  // migrate the committed history to the new context
    pull();
    fm_model_destroy(dev_->h, dm_);
    dm_ = nullptr;
  }
  dev_ = dev;
  detail::check(dev->h,
                fm_model_create_simo(dev->h, lambda_.data().data(), mu_.data().data(), tau_y0_.data().data(),
                                     hardening_.data().data(), &dm_),
                "SimoPlasticityModel");
  detail::check(dev->h,
                fm_model_set_history(dev->h, dm_, committed_.be.data().data(), committed_.eps_p.data().data(),
                                     f_old_.data().data()),
                "set_history");
  return dm_;
}

void SimoPlasticityModel::pull() const {
  if (!stale_ || !dm_) return;
  detail::check(dev_->h, fm_model_get_history(dev_->h, dm_, 0, committed_.be.data().data(), committed_.eps_p.data().data()),
                "history");
  detail::check(dev_->h, fm_model_get_history(dev_->h, dm_, 1, trial_.be.data().data(), trial_.eps_p.data().data()),
                "history");
  stale_ = false;
}

void SimoPlasticityModel::evaluate(const Tensor2Field& F, Tensor2Field& P, Tensor4Field& K) {
  if (F.tdim() != 3 || !(F.shape() == shape_)) throw std::invalid_argument("evaluate: field does not match model");
  auto dev = dev_ ? dev_ : detail::device_for(shape_, 3, 0);
  fm_model* dm = device_model(dev);
  detail::DevField f(dev, 9), p(dev, 9);
  f.upload(F.data());
  detail::check(dev->h, fm_model_evaluate(dev->h, dm, f.get(), p.get()), "SimoPlasticityModel::evaluate");
  P = Tensor2Field(F.shape(), 3);
  K = Tensor4Field(F.shape(), 3);
  p.download(P.data());
  detail::check(dev->h, fm_field_download(dev->h, fm_model_tangent(dm), K.data().data(), int64_t(K.size())), "tangent");
  stale_ = true;
}

void SimoPlasticityModel::commit(const Tensor2Field& F) {
  auto dev = dev_ ? dev_ : detail::device_for(shape_, 3, 0);
  fm_model* dm = device_model(dev);
  detail::DevField f(dev, 9);
  f.upload(F.data());
  detail::check(dev->h, fm_model_commit(dev->h, dm, f.get()), "commit");
  device_committed(F);
}

void SimoPlasticityModel::device_committed(const Tensor2Field& F) {
  f_old_ = F;
  stale_ = true;
}

const HistoryState& SimoPlasticityModel::committed() const {
  pull();
  return committed_;
}
const HistoryState& SimoPlasticityModel::trial() const {
  pull();
  return trial_;
}
const Tensor2Field& SimoPlasticityModel::reference_deformation() const { return f_old_; }

ScalarField SimoPlasticityModel::equivalent_stress_field(const Tensor2Field& F, const Tensor2Field& P) const {
  return device_equivalent_stress(&F, P, FM_EQ_KIRCHHOFF, "equivalent_stress_field");  // tau = P F^T
}

}  // namespace fftmech
