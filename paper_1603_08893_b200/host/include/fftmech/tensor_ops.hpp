// Node-local tensor algebra used around the solver (reference API:
// proj/core/include/fftmech/tensor_ops.hpp).  Conventions (tensor_ops.hpp:7-19):
//   ddot42: C_ij = A_ijkl B_lk,  dot22: C_ik = A_ij B_jk,  dyad22: C_ijkl = A_ij B_kl,
//   II_ijkl = d_il d_jk,  IRT_ijkl = d_ik d_jl,  Is = (II + IRT)/2.
// These are host-side helpers for setup, tests and post-processing; the hot
// path never calls them.
#pragma once

#include "fftmech/fields.hpp"

namespace fftmech {

Tensor2Field identity2(const GridShape& shape, int tdim);
Tensor4Field identity4(const GridShape& shape, int tdim);
Tensor4Field identity4rt(const GridShape& shape, int tdim);
Tensor4Field identity4sym(const GridShape& shape, int tdim);
Tensor4Field dyad22(const Tensor2Field& A, const Tensor2Field& B);
Tensor2Field ddot42(const Tensor4Field& A, const Tensor2Field& B);
Tensor2Field dot22(const Tensor2Field& A, const Tensor2Field& B);
Tensor2Field trans2(const Tensor2Field& A);
Tensor2Field inv2(const Tensor2Field& A);
ScalarField det2(const Tensor2Field& A);

double field_norm(const Tensor2Field& A);
Tensor2 field_mean(const Tensor2Field& A);

namespace detail {
inline constexpr double kSingularDetTol = 1e-30;
inline constexpr double kMinLogEigenvalue = 1e-30;
}  // namespace detail

}  // namespace fftmech
