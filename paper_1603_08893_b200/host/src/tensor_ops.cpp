// Host tensor helpers (reference semantics: tensor_ops.cpp; conventions in
// tensor_ops.hpp).  Setup / test / post-processing only.
#include "fftmech/tensor_ops.hpp"

#include <cmath>
#include <stdexcept>

namespace fftmech {

namespace {
template <class F>
Tensor4Field fill4(const GridShape& shape, int d, F value) {
  Tensor4Field out(shape, d);
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j)
      for (int k = 0; k < d; ++k)
        for (int l = 0; l < d; ++l) {
          const double v = value(i, j, k, l);
          if (v == 0.0) continue;
          double* s = out.comp(i, j, k, l);
          for (std::size_t q = 0; q < out.nodes(); ++q) s[q] = v;
        }
  return out;
}
}  // namespace

Tensor2Field identity2(const GridShape& shape, int tdim) {
  Tensor2Field I(shape, tdim);
  I.add_uniform(Tensor2::identity(tdim));
  return I;
}

Tensor4Field identity4(const GridShape& shape, int d) {
  return fill4(shape, d, [](int i, int j, int k, int l) { return double(i == l && j == k); });
}
Tensor4Field identity4rt(const GridShape& shape, int d) {
  return fill4(shape, d, [](int i, int j, int k, int l) { return double(i == k && j == l); });
}
Tensor4Field identity4sym(const GridShape& shape, int d) {
  return fill4(shape, d, [](int i, int j, int k, int l) { return 0.5 * (double(i == l && j == k) + double(i == k && j == l)); });
}

Tensor4Field dyad22(const Tensor2Field& A, const Tensor2Field& B) {
  const int d = A.tdim();
  Tensor4Field C(A.shape(), d);
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j)
      for (int k = 0; k < d; ++k)
        for (int l = 0; l < d; ++l) {
          double* c = C.comp(i, j, k, l);
          const double* a = A.comp(i, j);
          const double* b = B.comp(k, l);
          for (std::size_t q = 0; q < A.nodes(); ++q) c[q] = a[q] * b[q];
        }
  return C;
}

Tensor2Field ddot42(const Tensor4Field& A, const Tensor2Field& B) {  // C_ij = A_ijkl B_lk
  const int d = B.tdim();
  Tensor2Field C(B.shape(), d);
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) {
      double* c = C.comp(i, j);
      for (int k = 0; k < d; ++k)
        for (int l = 0; l < d; ++l) {
          const double* a = A.comp(i, j, k, l);
          const double* b = B.comp(l, k);
          for (std::size_t q = 0; q < B.nodes(); ++q) c[q] += a[q] * b[q];
        }
    }
  return C;
}

Tensor2Field dot22(const Tensor2Field& A, const Tensor2Field& B) {
  const int d = A.tdim();
  Tensor2Field C(A.shape(), d);
  for (std::size_t q = 0; q < A.nodes(); ++q) C.set_tensor(q, dot(A.tensor(q), B.tensor(q)));
  return C;
}

Tensor2Field trans2(const Tensor2Field& A) {
  Tensor2Field C(A.shape(), A.tdim());
  for (std::size_t q = 0; q < A.nodes(); ++q) C.set_tensor(q, A.tensor(q).transposed());
  return C;
}

Tensor2Field inv2(const Tensor2Field& A) {
  Tensor2Field C(A.shape(), A.tdim());
  for (std::size_t q = 0; q < A.nodes(); ++q) {
    const Tensor2 t = A.tensor(q);
    if (std::abs(t.det()) < detail::kSingularDetTol) throw std::domain_error("inv2: singular tensor");
    C.set_tensor(q, t.inverse());
  }
  return C;
}

ScalarField det2(const Tensor2Field& A) {
  ScalarField out(A.shape());
  for (std::size_t q = 0; q < A.nodes(); ++q) out[q] = A.tensor(q).det();
  return out;
}

double field_norm(const Tensor2Field& A) {
  double s = 0.0;
  for (double v : A.data()) s += v * v;
  return std::sqrt(s);
}

Tensor2 field_mean(const Tensor2Field& A) {
  const int d = A.tdim();
  Tensor2 m(d);
  for (int c = 0; c < d * d; ++c) {
    const double* s = A.slab(static_cast<std::size_t>(c));
    double acc = 0.0;
    for (std::size_t q = 0; q < A.nodes(); ++q) acc += s[q];
    m.v[static_cast<std::size_t>(c)] = acc / static_cast<double>(A.nodes());
  }
  return m;
}

}  // namespace fftmech
