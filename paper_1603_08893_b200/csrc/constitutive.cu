// Per-voxel constitutive updates on sm_100a: St. Venant-Kirchhoff and the
// finite-strain J2 (Simo) model.  One thread per voxel, component-major
// coalesced loads/stores.  Errors report the LOWEST offending node via a
// 64-bit atomicMin on (node << 4 | status), reproducing the reference's
// first-throw-in-node-order semantics (hyperelastic.cpp:29, simo.cpp:49,77).
#include <cstdlib>

#include "fm_internal.cuh"

namespace fm {

// badval: two words, [0] the value reported with the error (the offending
// eigenvalue of NotPositiveDefinite) and [1] the key it belongs to.  The pair
// is updated under a one-word lock (key word = 0 while held) and only towards
// smaller keys, so after the launch it holds the value of the LOWEST node even
// when several nodes fail at once (a plain store after the atomicMin could be
// overtaken by a loser's).
__device__ __forceinline__ void report_bad(unsigned long long* bad, double* badval, int64_t node,
                                           int status, double value) {
  const unsigned long long key = (static_cast<unsigned long long>(node) << 4) | unsigned(status);
  const unsigned long long old = atomicMin(bad, key);
  if (!badval || key >= old) return;
  unsigned long long* vkey = reinterpret_cast<unsigned long long*>(badval + 1);
  unsigned long long cur = *reinterpret_cast<volatile unsigned long long*>(vkey);
  while (cur == 0ull || key < cur) {
    if (cur != 0ull && atomicCAS(vkey, cur, 0ull) == cur) {
      badval[0] = value;
      __threadfence();
      atomicExch(vkey, key);
      return;
    }
    cur = *reinterpret_cast<volatile unsigned long long*>(vkey);
  }
}

template <int TD>
__device__ __forceinline__ double det_t(const double* a) {
  if (TD == 2) return a[0] * a[3] - a[1] * a[2];
  return a[0] * (a[4] * a[8] - a[5] * a[7]) - a[1] * (a[3] * a[8] - a[5] * a[6]) +
         a[2] * (a[3] * a[7] - a[4] * a[6]);
}

// Tensor2::inverse, tensor2.hpp:91-113 (3x3 branch).
__device__ __forceinline__ bool inv3(const double* a, double* inv) {
  const double d = det_t<3>(a);
  if (d == 0.0) return false;
  inv[0] = (a[4] * a[8] - a[5] * a[7]) / d;
  inv[1] = (a[2] * a[7] - a[1] * a[8]) / d;
  inv[2] = (a[1] * a[5] - a[2] * a[4]) / d;
  inv[3] = (a[5] * a[6] - a[3] * a[8]) / d;
  inv[4] = (a[0] * a[8] - a[2] * a[6]) / d;
  inv[5] = (a[2] * a[3] - a[0] * a[5]) / d;
  inv[6] = (a[3] * a[7] - a[4] * a[6]) / d;
  inv[7] = (a[1] * a[6] - a[0] * a[7]) / d;
  inv[8] = (a[0] * a[4] - a[1] * a[3]) / d;
  return true;
}

// --------------------------------------------------------------------- SVK
// hyperelastic_evaluate, hyperelastic.cpp:10-65.
// MINB: CTAs per SM the register budget targets (A/B via FM_HYPER_MINB).
template <int TD, int MINB = 1>
__global__ void __launch_bounds__(128, MINB) k_hyper(int64_t n, const double* __restrict__ F,
                                               const double* __restrict__ lam_f,
                                               const double* __restrict__ mu_f,
                                               double* __restrict__ P, double* __restrict__ K,
                                               unsigned long long* bad, int64_t noff) {
  constexpr int NC = TD * TD;
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < n;
       q += int64_t(gridDim.x) * blockDim.x) {
    double f[NC], b[NC], e[NC], s[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) f[c] = __ldg(F + c * n + q);
    const double lam = __ldg(lam_f + q), g = __ldg(mu_f + q);
    if (det_t<TD>(f) <= 0.0) {
      report_bad(bad, nullptr, noff + q, FM_E_INVERTED, 0.0);
      continue;
    }
    double trE = 0.0;
#pragma unroll
    for (int i = 0; i < TD; ++i)
#pragma unroll
      for (int j = 0; j < TD; ++j) {
        double bij = 0.0, cij = 0.0;
#pragma unroll
        for (int k = 0; k < TD; ++k) {
          bij += f[i * TD + k] * f[j * TD + k];
          cij += f[k * TD + i] * f[k * TD + j];
        }
        b[i * TD + j] = bij;
        e[i * TD + j] = 0.5 * (cij - (i == j ? 1.0 : 0.0));
      }
#pragma unroll
    for (int i = 0; i < TD; ++i) trE += e[i * TD + i];
#pragma unroll
    for (int i = 0; i < TD; ++i)
#pragma unroll
      for (int j = 0; j < TD; ++j) s[i * TD + j] = lam * trE * (i == j ? 1.0 : 0.0) + 2.0 * g * e[i * TD + j];
#pragma unroll
    for (int i = 0; i < TD; ++i)
#pragma unroll
      for (int j = 0; j < TD; ++j) {
        double v = 0.0;
#pragma unroll
        for (int k = 0; k < TD; ++k) v += f[i * TD + k] * s[k * TD + j];
        P[(i * TD + j) * n + q] = v;
      }
    if (K) {
#pragma unroll
      for (int i = 0; i < TD; ++i)
#pragma unroll
        for (int j = 0; j < TD; ++j)
#pragma unroll
          for (int k = 0; k < TD; ++k)
#pragma unroll
            for (int l = 0; l < TD; ++l) {
              double v = lam * f[j * TD + i] * f[k * TD + l] + g * f[j * TD + l] * f[k * TD + i];
              if (i == l) v += g * b[j * TD + k];
              if (j == k) v += s[i * TD + l];
              K[(((i * TD + j) * TD + k) * TD + l) * n + q] = v;
            }
    }
  }
}

// The same update on voxel pairs (3-D, even n): 16-byte loads and stores,
// half the memory instructions of k_hyper for the 720 B/voxel of P and K4
// it writes.  The per-voxel arithmetic is k_hyper's, expression for
// expression, so both round identically.
template <int MINB>
__global__ void __launch_bounds__(128, MINB) k_hyper_v2(int64_t n, const double* __restrict__ F,
                                                        const double* __restrict__ lam_f,
                                                        const double* __restrict__ mu_f,
                                                        double* __restrict__ P, double* __restrict__ K,
                                                        unsigned long long* bad, int64_t noff) {
  constexpr int TD = 3, NC = 9;
  const int64_t np = n / 2;
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < np; p += int64_t(gridDim.x) * blockDim.x) {
    const int64_t q = 2 * p;
    double f[2][NC], b[2][NC], s[2][NC], lam[2], g[2];
    bool ok[2];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const double2 v = __ldg(reinterpret_cast<const double2*>(F + c * n + q));
      f[0][c] = v.x;
      f[1][c] = v.y;
    }
    {
      const double2 l2 = __ldg(reinterpret_cast<const double2*>(lam_f + q));
      const double2 m2 = __ldg(reinterpret_cast<const double2*>(mu_f + q));
      lam[0] = l2.x, lam[1] = l2.y, g[0] = m2.x, g[1] = m2.y;
    }
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      ok[v] = det_t<TD>(f[v]) > 0.0;
      if (!ok[v]) report_bad(bad, nullptr, noff + q + v, FM_E_INVERTED, 0.0);
      double e[NC];
      double trE = 0.0;
#pragma unroll
      for (int i = 0; i < TD; ++i)
#pragma unroll
        for (int j = 0; j < TD; ++j) {
          double bij = 0.0, cij = 0.0;
#pragma unroll
          for (int k = 0; k < TD; ++k) {
            bij += f[v][i * TD + k] * f[v][j * TD + k];
            cij += f[v][k * TD + i] * f[v][k * TD + j];
          }
          b[v][i * TD + j] = bij;
          e[i * TD + j] = 0.5 * (cij - (i == j ? 1.0 : 0.0));
        }
#pragma unroll
      for (int i = 0; i < TD; ++i) trE += e[i * TD + i];
#pragma unroll
      for (int i = 0; i < TD; ++i)
#pragma unroll
        for (int j = 0; j < TD; ++j)
          s[v][i * TD + j] = lam[v] * trE * (i == j ? 1.0 : 0.0) + 2.0 * g[v] * e[i * TD + j];
    }
    if (!ok[0] || !ok[1]) continue;  // (the scalar kernel skips only the bad voxel; the solve stops anyway)
#pragma unroll
    for (int i = 0; i < TD; ++i)
#pragma unroll
      for (int j = 0; j < TD; ++j) {
        double o[2];
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          double a = 0.0;
#pragma unroll
          for (int k = 0; k < TD; ++k) a += f[v][i * TD + k] * s[v][k * TD + j];
          o[v] = a;
        }
        *reinterpret_cast<double2*>(P + (i * TD + j) * n + q) = make_double2(o[0], o[1]);
      }
    if (K) {
#pragma unroll
      for (int i = 0; i < TD; ++i)
#pragma unroll
        for (int j = 0; j < TD; ++j)
#pragma unroll
          for (int k = 0; k < TD; ++k)
#pragma unroll
            for (int l = 0; l < TD; ++l) {
              double o[2];
#pragma unroll
              for (int v = 0; v < 2; ++v) {
                double a = lam[v] * f[v][j * TD + i] * f[v][k * TD + l] + g[v] * f[v][j * TD + l] * f[v][k * TD + i];
                if (i == l) a += g[v] * b[v][j * TD + k];
                if (j == k) a += s[v][i * TD + l];
                o[v] = a;
              }
              *reinterpret_cast<double2*>(K + (((i * TD + j) * TD + k) * TD + l) * n + q) = make_double2(o[0], o[1]);
            }
    }
  }
}

// -------------------------------------------------------------------- Simo
// Symmetric 3x3 eigen-decomposition restating Eigen's
// SelfAdjointEigenSolver<Matrix3d> (simo.cpp:74): cyclic Jacobi to
// convergence, ascending eigenvalues, eigenvectors in the columns of V.
__device__ void sym_eig3(const double Ain[9], double lam[3], double V[9]) {
  double a00 = Ain[0], a01 = Ain[1], a02 = Ain[2], a11 = Ain[4], a12 = Ain[5], a22 = Ain[8];
  double v[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  for (int sweep = 0; sweep < 64; ++sweep) {
    const double off = a01 * a01 + a02 * a02 + a12 * a12;
    const double dg = a00 * a00 + a11 * a11 + a22 * a22;
    if (off == 0.0 || off < 1e-36 * dg) break;
#pragma unroll
    for (int pq = 0; pq < 3; ++pq) {
      // (p,q) = (0,1), (0,2), (1,2)
      const int p = pq == 2 ? 1 : 0, q = pq == 0 ? 1 : 2;
      double App = p == 0 ? a00 : a11, Aqq = q == 1 ? a11 : a22;
      double Apq = pq == 0 ? a01 : (pq == 1 ? a02 : a12);
      if (Apq == 0.0) continue;
      const double theta = (Aqq - App) / (2.0 * Apq);
      const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
      const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
      // full symmetric matrix update A <- J^T A J for the rotation in (p,q)
      double A[3][3] = {{a00, a01, a02}, {a01, a11, a12}, {a02, a12, a22}};
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double akp = A[k][p], akq = A[k][q];
        A[k][p] = c * akp - s * akq;
        A[k][q] = s * akp + c * akq;
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double apk = A[p][k], aqk = A[q][k];
        A[p][k] = c * apk - s * aqk;
        A[q][k] = s * apk + c * aqk;
      }
      a00 = A[0][0];
      a11 = A[1][1];
      a22 = A[2][2];
      a01 = A[0][1];
      a02 = A[0][2];
      a12 = A[1][2];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double vkp = v[k * 3 + p], vkq = v[k * 3 + q];
        v[k * 3 + p] = c * vkp - s * vkq;
        v[k * 3 + q] = s * vkp + c * vkq;
      }
    }
  }
  double d[3] = {a00, a11, a22};
  int o0 = 0, o1 = 1, o2 = 2, tmp;
  if (d[o1] < d[o0]) { tmp = o0; o0 = o1; o1 = tmp; }
  if (d[o2] < d[o1]) { tmp = o1; o1 = o2; o2 = tmp; }
  if (d[o1] < d[o0]) { tmp = o0; o0 = o1; o1 = tmp; }
  const int ord[3] = {o0, o1, o2};
#pragma unroll
  for (int m = 0; m < 3; ++m) {
    lam[m] = d[ord[m]];
#pragma unroll
    for (int i = 0; i < 3; ++i) V[i * 3 + m] = v[i * 3 + ord[m]];
  }
}

// log_divided_difference, simo.cpp:18-22.
__device__ __forceinline__ double log_dd(double a, double b) {
  const double scale = fmax(a, b);
  if (fabs(b - a) < 1e-7 * scale) return 2.0 / (a + b);
  return (log(b) - log(a)) / (b - a);
}

// simo_evaluate, simo.cpp:26-196.  The algorithmic tangent is assembled in
// the eigenbasis of be_tr, where dln(be_tr) is diagonal (w_mp) and the
// isotropic-plus-N(x)N moduli D stay block sparse, so the reference's four
// 81-entry temporaries (simo.cpp:41) reduce to three 3x3 coefficient sets:
//   K_ijkl = sum_pq  a_pq U_ip V_jp V_kq U_lq + b_pq U_ip V_jq V_kp U_lq
//                  + c_pq U_ip V_jq V_kq U_lp,          U = F^-1 V,
// with a_pq = (lam - c1/3 + c2 N_p N_q) w_qq l_q,  b_pq = (mu + c1/2) w_pq l_q - tau_q,
//      c_pq = (mu + c1/2) w_qp l_p,  c1 = -6 mu^2 dg/taueq,
//      c2 = -4 mu^2 (1/(3mu+H) - dg/taueq)   (c1 = c2 = 0 on the elastic branch).
template <int MINB = 1>
__global__ void __launch_bounds__(128, MINB) k_simo(int64_t n, const double* __restrict__ F,
                                              const double* __restrict__ Fold,
                                              const double* __restrict__ be_c,
                                              const double* __restrict__ epsp_c,
                                              const double* __restrict__ lam_f,
                                              const double* __restrict__ mu_f,
                                              const double* __restrict__ ty0_f,
                                              const double* __restrict__ h_f,
                                              double* __restrict__ P, double* __restrict__ K,
                                              double* __restrict__ be_t,
                                              double* __restrict__ epsp_t,
                                              unsigned long long* bad, double* badval, int64_t noff,
                                              double* __restrict__ Kc) {
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < n;
       q += int64_t(gridDim.x) * blockDim.x) {
    const double lam = __ldg(lam_f + q), g = __ldg(mu_f + q), ty0 = __ldg(ty0_f + q),
                 h = __ldg(h_f + q);
    double Fm[9], Finv[9], f[9];
    {
      double Fo[9], Foinv[9];
#pragma unroll
      for (int c = 0; c < 9; ++c) {
        Fm[c] = __ldg(F + c * n + q);
        Fo[c] = __ldg(Fold + c * n + q);
      }
      if (det_t<3>(Fm) <= 0.0) {
        report_bad(bad, badval, noff + q, FM_E_INVERTED, 0.0);
        continue;
      }
      if (!inv3(Fm, Finv) || !inv3(Fo, Foinv)) {
        report_bad(bad, badval, noff + q, FM_E_SINGULAR, 0.0);
        continue;
      }
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
          f[i * 3 + j] = Fm[i * 3 + 0] * Foinv[0 * 3 + j] + Fm[i * 3 + 1] * Foinv[1 * 3 + j] +
                         Fm[i * 3 + 2] * Foinv[2 * 3 + j];
    }
    double bsym[9];
    {
      double be[9], tmp[9], bt[9];
#pragma unroll
      for (int c = 0; c < 9; ++c) be[c] = __ldg(be_c + c * n + q);
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
          tmp[i * 3 + j] = f[i * 3 + 0] * be[0 * 3 + j] + f[i * 3 + 1] * be[1 * 3 + j] +
                           f[i * 3 + 2] * be[2 * 3 + j];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
          bt[i * 3 + j] = tmp[i * 3 + 0] * f[j * 3 + 0] + tmp[i * 3 + 1] * f[j * 3 + 1] +
                          tmp[i * 3 + 2] * f[j * 3 + 2];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) bsym[i * 3 + j] = 0.5 * (bt[i * 3 + j] + bt[j * 3 + i]);
    }
    double lb[3], V[9];
    sym_eig3(bsym, lb, V);
    if (lb[0] < 1e-30 || lb[1] < 1e-30 || lb[2] < 1e-30) {  // kMinLogEigenvalue
      report_bad(bad, badval, noff + q, FM_E_NOT_SPD, lb[0] < 1e-30 ? lb[0] : (lb[1] < 1e-30 ? lb[1] : lb[2]));
      continue;
    }
    double eps[3], tau_d[3], dev[3];
#pragma unroll
    for (int m = 0; m < 3; ++m) eps[m] = 0.5 * log(lb[m]);
    const double tr_eps = eps[0] + eps[1] + eps[2];
#pragma unroll
    for (int m = 0; m < 3; ++m) tau_d[m] = lam * tr_eps + 2.0 * g * eps[m];
    const double tau_m = (tau_d[0] + tau_d[1] + tau_d[2]) / 3.0;
#pragma unroll
    for (int m = 0; m < 3; ++m) dev[m] = tau_d[m] - tau_m;
    const double taueq_tr = sqrt(1.5 * (dev[0] * dev[0] + dev[1] * dev[1] + dev[2] * dev[2]));
    const double ep0 = __ldg(epsp_c + q);
    const double tauy = ty0 + h * ep0;
    const double phi = taueq_tr - tauy;
    const bool plastic = phi >= -1e-12 * tauy;  // simo.cpp:96
    double dgamma = 0.0, N2[3] = {0.0, 0.0, 0.0}, eps_e[3] = {eps[0], eps[1], eps[2]};
    if (plastic) {
      dgamma = fmax(phi, 0.0) / (3.0 * g + h);
#pragma unroll
      for (int m = 0; m < 3; ++m) N2[m] = 1.5 * dev[m] / taueq_tr;
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        tau_d[m] -= 2.0 * g * dgamma * N2[m];
        eps_e[m] = eps[m] - dgamma * N2[m];
      }
    }
    // trial history (simo.cpp:110-120)
    {
      double ex[3];
#pragma unroll
      for (int m = 0; m < 3; ++m) ex[m] = exp(2.0 * eps_e[m]);
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
          be_t[(i * 3 + j) * n + q] = ex[0] * V[i * 3 + 0] * V[j * 3 + 0] +
                                      ex[1] * V[i * 3 + 1] * V[j * 3 + 1] +
                                      ex[2] * V[i * 3 + 2] * V[j * 3 + 2];
      epsp_t[q] = ep0 + dgamma;
    }
    // P = tau F^-T, tau = V diag(tau_d) V^T  (simo.cpp:122-128)
    {
      double tau[9];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
          tau[i * 3 + j] = tau_d[0] * V[i * 3 + 0] * V[j * 3 + 0] +
                           tau_d[1] * V[i * 3 + 1] * V[j * 3 + 1] +
                           tau_d[2] * V[i * 3 + 2] * V[j * 3 + 2];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
          P[(i * 3 + j) * n + q] = tau[i * 3 + 0] * Finv[j * 3 + 0] +
                                   tau[i * 3 + 1] * Finv[j * 3 + 1] +
                                   tau[i * 3 + 2] * Finv[j * 3 + 2];
    }
    if (!K && !Kc) continue;
    // eigenbasis coefficients of the algorithmic tangent (simo.cpp:131-194)
    const double a0 = plastic ? dgamma / taueq_tr : 0.0;
    const double c1 = plastic ? -6.0 * g * g * a0 : 0.0;
    const double c2 = plastic ? -4.0 * g * g * (1.0 / (3.0 * g + h) - a0) : 0.0;
    double w[9];
#pragma unroll
    for (int m = 0; m < 3; ++m)
#pragma unroll
      for (int p = 0; p < 3; ++p) w[m * 3 + p] = log_dd(lb[m], lb[p]);
    double ca[9], cb[9], cc[9];
    const double lamp = lam - c1 / 3.0, mup = g + 0.5 * c1;
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
      for (int qq = 0; qq < 3; ++qq) {
        ca[p * 3 + qq] = (lamp + c2 * N2[p] * N2[qq]) * w[qq * 3 + qq] * lb[qq];
        cb[p * 3 + qq] = mup * w[p * 3 + qq] * lb[qq] - tau_d[qq];
        cc[p * 3 + qq] = mup * w[qq * 3 + p] * lb[p];
      }
    double U[9];  // U = F^-1 V
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int p = 0; p < 3; ++p)
        U[i * 3 + p] = Finv[i * 3 + 0] * V[0 * 3 + p] + Finv[i * 3 + 1] * V[1 * 3 + p] +
                       Finv[i * 3 + 2] * V[2 * 3 + p];
    if (Kc) {  // compact J2 tangent: V, U, a, b, c (45 slabs, 360 B/voxel)
#pragma unroll
      for (int e = 0; e < 9; ++e) {
        Kc[(0 + e) * n + q] = V[e];
        Kc[(9 + e) * n + q] = U[e];
        Kc[(18 + e) * n + q] = ca[e];
        Kc[(27 + e) * n + q] = cb[e];
        Kc[(36 + e) * n + q] = cc[e];
      }
    }
    if (!K) continue;
#pragma unroll 1
    for (int ij = 0; ij < 9; ++ij) {
      const int i = ij / 3, j = ij % 3;
#pragma unroll
      for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int l = 0; l < 3; ++l) {
          double s = 0.0;
#pragma unroll
          for (int p = 0; p < 3; ++p) {
            const double Uip = U[i * 3 + p];
#pragma unroll
            for (int qq = 0; qq < 3; ++qq) {
              s += Uip * (ca[p * 3 + qq] * V[j * 3 + p] * V[k * 3 + qq] * U[l * 3 + qq] +
                          cb[p * 3 + qq] * V[j * 3 + qq] * V[k * 3 + p] * U[l * 3 + qq] +
                          cc[p * 3 + qq] * V[j * 3 + qq] * V[k * 3 + qq] * U[l * 3 + p]);
            }
          }
          K[((ij * 3 + k) * 3 + l) * n + q] = s;
        }
    }
  }
}

// ---------------------------------------------------------- output measures
// von Mises equivalent of a tensor field, equivalent_stress (material.cpp:
// 14-31): sqrt(3/2 dev(T):dev(T)), dev taken with tr(T)/tdim.  T is
//   FM_EQ_TENSOR    : the field itself;
//   FM_EQ_PK2       : S = F^-1 P (HyperelasticModel, hyperelastic.cpp:89-92;
//                     inv2 throws SingularTensor if |det F| < 1e-30,
//                     tensor_ops.cpp:257-266);
//   FM_EQ_KIRCHHOFF : tau = P F^T (SimoPlasticityModel, simo.cpp:225-228).
// Products accumulate over the inner index in order (dot22, tensor_ops.cpp:
// 138-153).  Reads 72 or 144 B and writes 8 B per voxel: one HBM sweep.
template <int TD, int KIND>
__global__ void __launch_bounds__(256) k_eq_stress(int64_t n, const double* __restrict__ F,
                                                   const double* __restrict__ P, double* __restrict__ out,
                                                   unsigned long long* bad, int64_t noff) {
  constexpr int NC = TD * TD;
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < n;
       q += int64_t(gridDim.x) * blockDim.x) {
    double p[NC], t[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) p[c] = __ldg(P + c * n + q);
    if constexpr (KIND == FM_EQ_TENSOR) {
#pragma unroll
      for (int c = 0; c < NC; ++c) t[c] = p[c];
    } else {
      double f[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) f[c] = __ldg(F + c * n + q);
      if constexpr (KIND == FM_EQ_PK2) {
        const double d = det_t<TD>(f);
        if (fabs(d) < 1e-30) {  // detail::kSingularDetTol
          report_bad(bad, nullptr, noff + q, FM_E_SINGULAR, 0.0);
          out[q] = 0.0;
          continue;
        }
        double fi[NC];
        if constexpr (TD == 2) {
          fi[0] = f[3] / d;
          fi[1] = -f[1] / d;
          fi[2] = -f[2] / d;
          fi[3] = f[0] / d;
        } else {
          inv3(f, fi);
        }
#pragma unroll
        for (int i = 0; i < TD; ++i)
#pragma unroll
          for (int k = 0; k < TD; ++k) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < TD; ++j) s += fi[i * TD + j] * p[j * TD + k];
            t[i * TD + k] = s;
          }
      } else {  // tau = P F^T
#pragma unroll
        for (int i = 0; i < TD; ++i)
#pragma unroll
          for (int k = 0; k < TD; ++k) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < TD; ++j) s += p[i * TD + j] * f[k * TD + j];
            t[i * TD + k] = s;
          }
      }
    }
    double tr = 0.0;
#pragma unroll
    for (int i = 0; i < TD; ++i) tr += t[i * TD + i];
    tr /= double(TD);
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < TD; ++i)
#pragma unroll
      for (int j = 0; j < TD; ++j) {
        const double dv = t[i * TD + j] - (i == j ? tr : 0.0);
        s += dv * dv;
      }
    out[q] = sqrt(1.5 * s);
  }
}

// -------------------------------------------------------------------- host
int reset_bad(fm_ctx* ctx) {
  FM_CUDA(ctx, cudaMemsetAsync(ctx->d_bad, 0xFF, sizeof(unsigned long long), ctx->stream));
  FM_CUDA(ctx, cudaMemsetAsync(ctx->d_badval + 1, 0xFF, sizeof(unsigned long long), ctx->stream));  // no value yet
  return FM_OK;
}

int check_bad(fm_ctx* ctx) {
  if (int st = combine_min_u64(ctx, ctx->d_bad)) return st;  // lowest offending node over all ranks
  unsigned long long key = 0;
  struct {
    double val;
    unsigned long long key;
  } rec{0.0, ~0ull};
  FM_CUDA(ctx, cudaMemcpyAsync(&key, ctx->d_bad, sizeof(key), cudaMemcpyDeviceToHost, ctx->stream));
  FM_CUDA(ctx, cudaMemcpyAsync(&rec, ctx->d_badval, sizeof(rec), cudaMemcpyDeviceToHost, ctx->stream));
  FM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if (key == ~0ull) return FM_OK;
  const int status = int(key & 15ull);
  const int64_t node = int64_t(key >> 4);
  // the value travels with its key: only the rank that owns the lowest node holds it
  double val = rec.key == key ? rec.val : 0.0;
  if (distributed(ctx)) {
    double* slot = ctx->d_scal + 62;
    FM_CUDA(ctx, cudaMemcpyAsync(slot, &val, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    if (int st = combine_ranks(ctx, slot, 1)) return st;  // ordered sum: one rank contributes, the others 0
    FM_CUDA(ctx, cudaMemcpyAsync(&val, slot, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    FM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  }
  const char* what = status == FM_E_INVERTED   ? "non-positive det(F) at node "
                     : status == FM_E_NOT_SPD ? "tensor log requires a positive-definite argument (node "
                                              : "singular tensor at node ";
  const int st = set_error(ctx, status, std::string(what) + std::to_string(node));
  ctx->last_info = fm_error_info{status, 0, node, val};
  return st;
}

static int grid_for(int64_t n, int threads) {
  const int64_t b = (n + threads - 1) / threads;
  return int(b < 148 * 64 ? (b < 1 ? 1 : b) : 148 * 64);
}

int hyper_eval_async(fm_ctx* ctx, const double* F, const double* lam, const double* mu, double* P,
                     double* K) {
  if (int st = reset_bad(ctx)) return st;
  const int blocks = grid_for(ctx->n, 128);
  // register budget / voxels per thread (A/B via FM_HYPER_MINB: 1, 4, 6, 8
  // one voxel per thread; 22 / 23 voxel pairs at 2 / 3 CTAs per SM)
  static const int minb = [] {
    const char* e = getenv("FM_HYPER_MINB");
    return e ? atoi(e) : 4;
  }();
  if (ctx->tdim == 3 && minb >= 20 && ctx->n % 2 == 0) {
    const int b2 = grid_for(ctx->n / 2, 128);
    if (minb == 23)
      k_hyper_v2<3><<<b2, 128, 0, ctx->stream>>>(ctx->n, F, lam, mu, P, K, ctx->d_bad, ctx->node_offset);
    else
      k_hyper_v2<2><<<b2, 128, 0, ctx->stream>>>(ctx->n, F, lam, mu, P, K, ctx->d_bad, ctx->node_offset);
  } else if (ctx->tdim == 3) {
    if (minb >= 8)
      k_hyper<3, 8><<<blocks, 128, 0, ctx->stream>>>(ctx->n, F, lam, mu, P, K, ctx->d_bad, ctx->node_offset);
    else if (minb >= 6)
      k_hyper<3, 6><<<blocks, 128, 0, ctx->stream>>>(ctx->n, F, lam, mu, P, K, ctx->d_bad, ctx->node_offset);
    else if (minb >= 4)
      k_hyper<3, 4><<<blocks, 128, 0, ctx->stream>>>(ctx->n, F, lam, mu, P, K, ctx->d_bad, ctx->node_offset);
    else
      k_hyper<3><<<blocks, 128, 0, ctx->stream>>>(ctx->n, F, lam, mu, P, K, ctx->d_bad, ctx->node_offset);
  } else {
    k_hyper<2><<<blocks, 128, 0, ctx->stream>>>(ctx->n, F, lam, mu, P, K, ctx->d_bad, ctx->node_offset);
  }
  FM_LAUNCHED_K(ctx, "k_hyper");
  return FM_OK;
}

template <int TD>
static void eq_launch(fm_ctx* ctx, int kind, const double* F, const double* P, double* out, int blocks) {
  if (kind == FM_EQ_TENSOR)
    k_eq_stress<TD, FM_EQ_TENSOR><<<blocks, 256, 0, ctx->stream>>>(ctx->n, F, P, out, ctx->d_bad, ctx->node_offset);
  else if (kind == FM_EQ_PK2)
    k_eq_stress<TD, FM_EQ_PK2><<<blocks, 256, 0, ctx->stream>>>(ctx->n, F, P, out, ctx->d_bad, ctx->node_offset);
  else
    k_eq_stress<TD, FM_EQ_KIRCHHOFF><<<blocks, 256, 0, ctx->stream>>>(ctx->n, F, P, out, ctx->d_bad,
                                                                      ctx->node_offset);
}

int eq_stress_async(fm_ctx* ctx, int kind, const double* F, const double* P, double* out) {
  if (int st = reset_bad(ctx)) return st;
  const int blocks = grid_for(ctx->n, 256);
  if (ctx->tdim == 3) eq_launch<3>(ctx, kind, F, P, out, blocks);
  else eq_launch<2>(ctx, kind, F, P, out, blocks);
  FM_LAUNCHED_K(ctx, "k_eq_stress");
  return FM_OK;
}

int simo_eval_async(fm_ctx* ctx, const double* F, const double* Fold, const double* be_c,
                    const double* epsp_c, const double* lam, const double* mu, const double* ty0,
                    const double* hard, double* P, double* K, double* be_t, double* epsp_t, double* Kc) {
  if (ctx->tdim != 3) return set_error(ctx, FM_E_INVALID, "simo_evaluate: tensors must be 3x3");
  if (int st = reset_bad(ctx)) return st;
  const int blocks = grid_for(ctx->n, 128);
  // register budget (A/B: FM_SIMO_MINB).  Measured at 256^3 (profiles/
  // r2_constitutive_256_v2.md): compact tangent 6.75 -> 5.55 ms at 3 CTAs/SM,
  // K4 11.1 -> 13.6 ms (its 81 stores want the registers): 3 / 1 by form.
  static const int env = [] {
    const char* e = getenv("FM_SIMO_MINB");
    return e ? atoi(e) : 0;
  }();
  const int minb = env ? env : (Kc ? 3 : 1);
  if (minb >= 3)
    k_simo<3><<<blocks, 128, 0, ctx->stream>>>(ctx->n, F, Fold, be_c, epsp_c, lam, mu, ty0, hard, P, K, be_t, epsp_t,
                                               ctx->d_bad, ctx->d_badval, ctx->node_offset, Kc);
  else if (minb == 2)
    k_simo<2><<<blocks, 128, 0, ctx->stream>>>(ctx->n, F, Fold, be_c, epsp_c, lam, mu, ty0, hard, P, K, be_t, epsp_t,
                                               ctx->d_bad, ctx->d_badval, ctx->node_offset, Kc);
  else
    k_simo<1><<<blocks, 128, 0, ctx->stream>>>(ctx->n, F, Fold, be_c, epsp_c, lam, mu, ty0, hard, P, K, be_t, epsp_t,
                                               ctx->d_bad, ctx->d_badval, ctx->node_offset, Kc);
  FM_LAUNCHED_K(ctx, "k_simo");
  return FM_OK;
}

}  // namespace fm
