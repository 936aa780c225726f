// Drop-in Tensor2 (reference API: proj/core/include/fftmech/tensor2.hpp): a
// 2x2 or 3x3 row-major tensor for macroscopic quantities.  det/inverse go
// through cofactors so one code path serves both dimensions.
#pragma once

#include <array>
#include <cmath>
#include <cstddef>
#include <stdexcept>

namespace fftmech {

struct Tensor2 {
  int dim = 3;
  std::array<double, 9> v{};

  Tensor2() = default;
  explicit Tensor2(int d) : dim(d) {
    if (d < 2 || d > 3) throw std::invalid_argument("Tensor2 dim must be 2 or 3");
  }
  static Tensor2 identity(int d) {
    Tensor2 t(d);
    for (int i = 0; i < d * d; i += d + 1) t.v[static_cast<std::size_t>(i)] = 1.0;
    return t;
  }
  static Tensor2 zero(int d) { return Tensor2(d); }

  double& operator()(int i, int j) { return v[static_cast<std::size_t>(i * dim + j)]; }
  double operator()(int i, int j) const { return v[static_cast<std::size_t>(i * dim + j)]; }

  template <class Op>
  Tensor2& zip(const Tensor2& o, Op op) {
    for (int i = 0; i < dim * dim; ++i) v[static_cast<std::size_t>(i)] = op(v[static_cast<std::size_t>(i)], o.v[static_cast<std::size_t>(i)]);
    return *this;
  }
  Tensor2& operator+=(const Tensor2& o) { return zip(o, [](double a, double b) { return a + b; }); }
  Tensor2& operator-=(const Tensor2& o) { return zip(o, [](double a, double b) { return a - b; }); }
  Tensor2& operator*=(double s) {
    for (double& x : v) x *= s;
    return *this;
  }
  friend Tensor2 operator+(Tensor2 a, const Tensor2& b) { return a += b; }
  friend Tensor2 operator-(Tensor2 a, const Tensor2& b) { return a -= b; }
  friend Tensor2 operator*(double s, Tensor2 a) { return a *= s; }

  Tensor2 transposed() const {
    Tensor2 t(dim);
    for (int k = 0; k < dim * dim; ++k) t(k % dim, k / dim) = v[static_cast<std::size_t>(k)];
    return t;
  }
  double trace() const {
    double s = 0.0;
    for (int i = 0; i < dim; ++i) s += (*this)(i, i);
    return s;
  }
  // cofactor C_ij = (-1)^{i+j} minor_ij
  double cofactor(int i, int j) const {
    if (dim == 2) return ((i + j) % 2 ? -1.0 : 1.0) * (*this)(1 - i, 1 - j);
    const int r0 = (i + 1) % 3, r1 = (i + 2) % 3, c0 = (j + 1) % 3, c1 = (j + 2) % 3;
    return (*this)(r0, c0) * (*this)(r1, c1) - (*this)(r0, c1) * (*this)(r1, c0);
  }
  double det() const {
    double s = 0.0;
    for (int j = 0; j < dim; ++j) s += (*this)(0, j) * cofactor(0, j);
    return s;
  }
  Tensor2 inverse() const {
    const double d = det();
    if (d == 0.0) throw std::domain_error("Tensor2::inverse: singular");
    Tensor2 inv(dim);
    for (int i = 0; i < dim; ++i)
      for (int j = 0; j < dim; ++j) inv(i, j) = cofactor(j, i) / d;
    return inv;
  }
  double norm() const {
    double s = 0.0;
    for (int i = 0; i < dim * dim; ++i) s += v[static_cast<std::size_t>(i)] * v[static_cast<std::size_t>(i)];
    return std::sqrt(s);
  }
  friend Tensor2 dot(const Tensor2& a, const Tensor2& b) {
    Tensor2 c(a.dim);
    for (int i = 0; i < a.dim; ++i)
      for (int j = 0; j < a.dim; ++j)
        for (int k = 0; k < a.dim; ++k) c(i, k) += a(i, j) * b(j, k);
    return c;
  }
};

}  // namespace fftmech
