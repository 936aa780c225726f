// Drop-in host fields (reference API: proj/core/include/fftmech/fields.hpp).
// Value types in host memory with the reference's component-major layout,
// so uploads to the device kernels are single memcpys: slab c of a
// tdim^k-component field starts at c * node_count.
#pragma once

#include <cstddef>
#include <span>
#include <vector>

#include "fftmech/grid.hpp"
#include "fftmech/tensor2.hpp"

namespace fftmech {

namespace detail {
// ncomp slabs of n doubles; the common storage of all field types.
class Slabs {
 public:
  Slabs() = default;
  Slabs(const GridShape& shape, int tdim, int order, double fill = 0.0);
  const GridShape& shape() const { return shape_; }
  int tdim() const { return tdim_; }
  std::size_t nodes() const { return n_; }
  std::size_t size() const { return data_.size(); }
  std::span<double> data() { return data_; }
  std::span<const double> data() const { return data_; }
  double* slab(std::size_t c) { return data_.data() + c * n_; }
  const double* slab(std::size_t c) const { return data_.data() + c * n_; }
  void fill(double value) { data_.assign(data_.size(), value); }

 protected:
  GridShape shape_;
  int tdim_ = 3;
  std::size_t n_ = 0;
  std::vector<double> data_;
};
}  // namespace detail

class ScalarField : public detail::Slabs {
 public:
  ScalarField() = default;
  explicit ScalarField(const GridShape& shape, double fill = 0.0) : Slabs(shape, 1, 0, fill) {}
  double& operator[](std::size_t k) { return data_[k]; }
  double operator[](std::size_t k) const { return data_[k]; }
};

class Tensor2Field : public detail::Slabs {
 public:
  Tensor2Field() = default;
  Tensor2Field(const GridShape& shape, int tdim) : Slabs(shape, tdim, 2) {}
  double* comp(int i, int j) { return slab(static_cast<std::size_t>(i * tdim_ + j)); }
  const double* comp(int i, int j) const { return slab(static_cast<std::size_t>(i * tdim_ + j)); }
  double& at(std::size_t node, int i, int j) { return comp(i, j)[node]; }
  double at(std::size_t node, int i, int j) const { return comp(i, j)[node]; }
  Tensor2 tensor(std::size_t node) const;
  void set_tensor(std::size_t node, const Tensor2& t);
  Tensor2Field& operator+=(const Tensor2Field& o);
  Tensor2Field& operator-=(const Tensor2Field& o);
  Tensor2Field& operator*=(double s);
  void add_uniform(const Tensor2& t);
};

class Tensor4Field : public detail::Slabs {
 public:
  Tensor4Field() = default;
  Tensor4Field(const GridShape& shape, int tdim) : Slabs(shape, tdim, 4) {}
  std::size_t comp_index(int i, int j, int k, int l) const {
    return static_cast<std::size_t>(((i * tdim_ + j) * tdim_ + k) * tdim_ + l);
  }
  double* comp(int i, int j, int k, int l) { return slab(comp_index(i, j, k, l)); }
  const double* comp(int i, int j, int k, int l) const { return slab(comp_index(i, j, k, l)); }
  double& at(std::size_t node, int i, int j, int k, int l) { return comp(i, j, k, l)[node]; }
  double at(std::size_t node, int i, int j, int k, int l) const { return comp(i, j, k, l)[node]; }
  Tensor4Field& operator+=(const Tensor4Field& o);
  Tensor4Field& operator*=(double s);
};

void axpy(double a, const Tensor2Field& x, Tensor2Field& y);
double field_dot(const Tensor2Field& a, const Tensor2Field& b);

}  // namespace fftmech
