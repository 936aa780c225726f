// Drop-in material contract (reference API: proj/core/include/fftmech/material.hpp).
#pragma once

#include <memory>

#include "fftmech/fields.hpp"
#include "fftmech/tensor2.hpp"

struct fm_model;

namespace fftmech {

struct ElasticParams {
  double youngs = 1.0;
  double poisson = 0.3;
  double lame_lambda() const { return youngs * poisson / ((1.0 + poisson) * (1.0 - 2.0 * poisson)); }
  double lame_mu() const { return 0.5 * youngs / (1.0 + poisson); }
};

struct PlasticParams {
  ElasticParams elastic;
  double tau_y0 = 1.0;
  double hardening = 0.0;
};

struct HistoryState {
  Tensor2Field be;
  ScalarField eps_p;
  HistoryState() = default;
  HistoryState(const GridShape& shape, int tdim);
};

namespace detail {
struct Device;
}

class MaterialModel {
 public:
  virtual ~MaterialModel() = default;
  virtual int tensor_dim() const = 0;
  virtual void evaluate(const Tensor2Field& F, Tensor2Field& P, Tensor4Field& K) = 0;
  virtual void commit(const Tensor2Field& F_converged) = 0;
  virtual ScalarField equivalent_stress_field(const Tensor2Field& F, const Tensor2Field& P) const = 0;
  virtual const ScalarField* committed_eps_p() const { return nullptr; }

  // B200 extension: the device-resident twin of this model on `dev`
  // (nullptr for user-defined host models, which solve_increment then
  // evaluates on the host while the projection/CG stay on the device).
  virtual fm_model* device_model(const std::shared_ptr<detail::Device>&) { return nullptr; }
  // Called after a device-resident solve committed the history at F.
  virtual void device_committed(const Tensor2Field&) {}
};

ScalarField equivalent_stress(const Tensor2Field& T);

// sqrt(2/3 dev(ln U):dev(ln U)) of the macroscopic stretch, U^2 = Fbar^T Fbar
// (material.cpp:33-49; 2x2 inputs embedded as plane strain).  The eps_bar
// column of report.csv.
double macroscopic_equivalent_strain(const Tensor2& fbar);

}  // namespace fftmech
