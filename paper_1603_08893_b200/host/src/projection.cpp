// Drop-in projection over the sm_100a kernels (reference:
// projection.cpp:72-194).  apply_* are the reference's host-field ("compat")
// entry points: one upload, the fused five-pass device transform, one download.
#include "fftmech/projection.hpp"

#include <cmath>
#include <stdexcept>

#include "device.hpp"

namespace fftmech {

FrequencyGrid build_frequency_grid(const GridShape& shape) {
  shape.validate();
  const int d = shape.dim;
  const std::size_t n = shape.node_count();
  FrequencyGrid fg;
  fg.shape = shape;
  fg.q.resize(n * static_cast<std::size_t>(d));
  fg.xi.resize(n * static_cast<std::size_t>(d));
  fg.nyquist.assign(n, false);
  for (std::size_t k = 0; k < n; ++k) {
    const auto idx = shape.node_coords(k);
    for (int a = 0; a < d; ++a) {
      const int na = shape.points[a];
      const int q = 2 * idx[a] < na ? idx[a] : idx[a] - na;  // natural transform ordering
      fg.q[k * d + a] = q;
      fg.xi[k * d + a] = static_cast<double>(q) / shape.lengths[a];
      if (na % 2 == 0 && 2 * idx[a] == na) fg.nyquist[k] = true;
    }
  }
  return fg;
}

struct ProjectionOperator::Impl {
  GridShape shape;
  int tdim = 3;
  NyquistMode mode = NyquistMode::ZeroCompatible;
  std::shared_ptr<detail::Device> dev;
  mutable std::unique_ptr<Tensor2Field> ghat;  // host copy, built on first request
};

ProjectionOperator::ProjectionOperator() : impl_(new Impl) {}
ProjectionOperator::ProjectionOperator(ProjectionOperator&&) noexcept = default;
ProjectionOperator& ProjectionOperator::operator=(ProjectionOperator&&) noexcept = default;
ProjectionOperator::~ProjectionOperator() = default;

const GridShape& ProjectionOperator::shape() const { return impl_->shape; }
int ProjectionOperator::tdim() const { return impl_->tdim; }
NyquistMode ProjectionOperator::nyquist_mode() const { return impl_->mode; }
const std::shared_ptr<detail::Device>& ProjectionOperator::device() const { return impl_->dev; }

const Tensor2Field& ProjectionOperator::ghat() const {
  // Inspection only: the device never stores ghat (it is evaluated from the
  // wave vector in the x pass).  Same closed form as projection.cpp:87-104.
  if (!impl_->ghat) {
    const auto& s = impl_->shape;
    const int td = impl_->tdim, d = s.dim;
    auto g = std::make_unique<Tensor2Field>(s, td);
    const FrequencyGrid fg = build_frequency_grid(s);
    for (std::size_t k = 0; k < s.node_count(); ++k) {
      const double* xi = fg.xi_at(k);
      double n2 = 0.0;
      for (int a = 0; a < d; ++a) n2 += xi[a] * xi[a];
      if (n2 == 0.0) continue;
      if (fg.nyquist[k]) {
        if (impl_->mode == NyquistMode::IdentityEquilibrium)
          for (int i = 0; i < td; ++i) g->at(k, i, i) = 1.0;
        continue;
      }
      for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j) g->at(k, i, j) = xi[i] * xi[j] / n2;
    }
    impl_->ghat = std::move(g);
  }
  return *impl_->ghat;
}

ProjectionOperator build_projection(const GridShape& shape, int tdim, NyquistMode mode) {
  shape.validate();
  if (tdim < shape.dim || tdim > 3) throw std::invalid_argument("tensor dim must be in [grid dim, 3]");
  ProjectionOperator op;
  op.impl_->shape = shape;
  op.impl_->tdim = tdim;
  op.impl_->mode = mode;
  op.impl_->dev = detail::device_for(shape, tdim, mode == NyquistMode::ZeroCompatible ? 0 : 1);
  return op;
}

Tensor2Field apply_projection(const ProjectionOperator& G, const Tensor2Field& A) {
  if (!(A.shape() == G.shape()) || A.tdim() != G.tdim())
    throw std::invalid_argument("apply_projection: field does not match operator");
  const auto& dev = G.device();
  const int nc = G.tdim() * G.tdim();
  detail::DevField a(dev, nc), out(dev, nc);
  a.upload(A.data());
  detail::check(dev->h, fm_projection_apply(dev->h, a.get(), out.get()), "apply_projection");
  Tensor2Field result(A.shape(), A.tdim());
  out.download(result.data());
  return result;
}

Tensor2Field apply_projected_tangent(const ProjectionOperator& G, const Tensor4Field& K, const Tensor2Field& dF) {
  if (!(K.shape() == dF.shape()) || K.tdim() != dF.tdim() || !(dF.shape() == G.shape()) || dF.tdim() != G.tdim())
    throw std::invalid_argument("apply_projected_tangent: shape mismatch");
  const auto& dev = G.device();
  const int nc = G.tdim() * G.tdim();
  detail::DevField k(dev, nc * nc), d(dev, nc), out(dev, nc);
  k.upload(K.data());
  d.upload(dF.data());
  detail::check(dev->h, fm_projected_tangent_apply(dev->h, k.get(), d.get(), out.get()), "apply_projected_tangent");
  Tensor2Field result(dF.shape(), dF.tdim());
  out.download(result.data());
  return result;
}

}  // namespace fftmech
