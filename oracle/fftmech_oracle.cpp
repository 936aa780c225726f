// ============================================================================
// fftmech CPU ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A C++ restatement of the reference `fftmech` hot path
// (arXiv 1603.08893, Galerkin-FFT finite-strain homogenisation), used as the
// parity checker for the sm_100a product in paper_1603_08893_b200/.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference leg may load this library; the product never does.
//
// Why a restatement: the reference (/root/reference/proj/core) needs FFTW3
// and Eigen3, neither of which exists in this image or on the GPU box
// (SURVEY.md §8(c)), so oracle/_ref cannot be built.  The two third-party
// pieces are restated from their published algorithms:
//   * FFTW3 (unpinned; `FindFFTW3.cmake:2-3`) c2c DFT, sign -1 forward, +1
//     backward, unnormalised (`projection.cpp:115-118`) -> mixed-radix
//     Stockham FFT below with long-double twiddles.
//   * Eigen3 >= 3.3 `SelfAdjointEigenSolver<Matrix3d>` (`simo.cpp:74`) ->
//     cyclic Jacobi iteration to convergence below.
// Parity of this restatement is PINNED by tests/test_oracle_*.py against the
// reference's own golden run records (proj/unit_det_out1/report.csv: Newton
// 3/3/3, CG 5/6/6, rel_update to 17 digits; unit_run_out, unit_vtk_out) and
// against every property assertion of proj/tests/unit/test_projection.cpp,
// test_solver.cpp, test_hyperelastic.cpp and test_simo.cpp.
//
// Layout contract (grid.hpp:26-39, fields.hpp:41-139): nodes row-major with
// the last axis fastest; tensor fields component-major, slab (i,j) at offset
// (i*tdim+j)*n, 4th-order slab ((i*d+j)*d+k)*d+l.
// ============================================================================
#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>
#include <mutex>
#include <thread>

namespace oracle {

// ------------------------------------------------------------ threading
// par_for(count, body): body(begin, end) over contiguous chunks of [0, count)
// on g_threads std::threads (default 1, or $OR_THREADS).  Only independent
// work (FFT lines, nodes, vector entries) is split; every reduction stays the
// reference's sequential sum, so results never depend on the thread count.
static int g_threads = [] {
  const char* e = std::getenv("OR_THREADS");
  return e ? std::max(1, std::atoi(e)) : 1;
}();

template <class Body>
void par_for(int64_t count, Body body) {
  const int T = int(std::min<int64_t>(g_threads, std::max<int64_t>(1, count / 2048)));
  if (T <= 1) {
    body(int64_t(0), count);
    return;
  }
  std::vector<std::thread> pool;
  pool.reserve(size_t(T));
  for (int t = 0; t < T; ++t)
    pool.emplace_back([&, t] { body(count * t / T, count * (t + 1) / T); });
  for (auto& th : pool) th.join();
}

using cplx = std::complex<double>;

// ----------------------------------------------------------------- errors
// Status codes mirror include/fftmech_b200.h (and errors.hpp:11-111).
enum Status : int {
  OK = 0,
  E_INVALID = 1,
  E_INVERTED = 4,      // InvertedElement, errors.hpp:57-62
  E_NOT_SPD = 5,       // NotPositiveDefinite, errors.hpp:32-41
  E_SINGULAR = 6,      // SingularTensor / domain_error from Tensor2::inverse
  E_CG_STALLED = 7,    // CgStalled, solver.hpp:69-78
  E_COMPLEX_RES = 8,   // ComplexResidue, errors.hpp:45-54
  E_NEWTON_DIV = 9,    // NewtonDiverged, solver.hpp:60-67
};

struct OracleError {
  int code;
  int64_t node;
  double value;
};

// ------------------------------------------------------------------- grid
// GridShape, grid.hpp:15-58.
struct Grid {
  int dim = 3;
  int pts[3] = {1, 1, 1};
  double len[3] = {1, 1, 1};
  size_t n() const {
    size_t s = 1;
    for (int a = 0; a < dim; ++a) s *= size_t(pts[a]);
    return s;
  }
  void coords(size_t node, int idx[3]) const {  // node_coords, grid.hpp:32-39
    idx[0] = idx[1] = idx[2] = 0;
    for (int a = dim - 1; a >= 0; --a) {
      idx[a] = int(node % size_t(pts[a]));
      node /= size_t(pts[a]);
    }
  }
};

// ------------------------------------------------------------- 1-D FFT
// Twiddles as FFTW's trig generator produces them: octant-reduced, so the
// quarter / half / eighth points are exact.
static cplx unit_root(long long k, long long N) {
  k %= N;
  if (k < 0) k += N;
  const long long k8 = 8 * k;
  const int oct = int(k8 / N);            // octant 0..7 of the angle 2 pi k / N
  long long r = k8 - (long long)oct * N;  // remainder within the octant, in units of 1/(8N)
  const bool odd = oct & 1;
  if (odd) r = N - r;                     // reflect so the reduced angle is in [0, pi/4]
  const long double tau = 6.283185307179586476925286766559005768L;
  const long double a = tau * (long double)r / (8.0L * (long double)N);
  double c = (double)cosl(a), s = (double)sinl(a);
  if (r == 0) { c = 1.0; s = 0.0; }
  // angle theta = oct*pi/4 +/- a ; (cos theta, sin theta) by octant
  double ct, st;
  switch (oct) {
    case 0: ct = c; st = s; break;
    case 1: ct = s; st = c; break;
    case 2: ct = -s; st = c; break;
    case 3: ct = -c; st = s; break;
    case 4: ct = -c; st = -s; break;
    case 5: ct = -s; st = -c; break;
    case 6: ct = s; st = -c; break;
    default: ct = c; st = -s; break;
  }
  return cplx(ct, -st);  // exp(-i theta)
}


// Mixed-radix Stockham autosort FFT restating FFTW's unnormalised c2c DFT:
// X[k] = sum_n x[n] exp(sign * 2 pi i n k / N).  Radices 4,2,3,5 and any
// remaining prime by a direct O(p^2) butterfly.
struct Plan1D {
  int N = 1;
  std::vector<int> radix;
  std::vector<cplx> w;                    // w[k] = exp(-2 pi i k / N), long-double accurate
  std::vector<std::vector<cplx>> stw;     // per stage: twiddle (jm, r) -> W^(jm r tstep)
  std::vector<std::vector<cplx>> dft;     // per stage (generic radix): W_R^(r k)
  explicit Plan1D(int n) : N(n) {
    int m = n;
    while (m % 4 == 0) { radix.push_back(4); m /= 4; }
    while (m % 2 == 0) { radix.push_back(2); m /= 2; }
    for (int p = 3; p * p <= m; p += 2)
      while (m % p == 0) { radix.push_back(p); m /= p; }
    if (m > 1) radix.push_back(m);
    w.resize(size_t(n));
    for (int k = 0; k < n; ++k) w[size_t(k)] = unit_root(k, n);
    int Ns = 1;
    for (int R : radix) {
      const int tstep = N / (Ns * R);
      std::vector<cplx> t(size_t(Ns) * size_t(R));
      for (int jm = 0; jm < Ns; ++jm)
        for (int r = 0; r < R; ++r) t[size_t(jm) * R + r] = w[size_t((long long)jm * r * tstep % N)];
      stw.push_back(std::move(t));
      std::vector<cplx> d;
      if (R != 2 && R != 4) {
        d.resize(size_t(R) * size_t(R));
        for (int r = 0; r < R; ++r)
          for (int k = 0; k < R; ++k) d[size_t(r) * R + k] = w[size_t((long long)r * k % R) * (N / R)];
      }
      dft.push_back(std::move(d));
      Ns *= R;
    }
  }
  // In-place transform of x (contiguous, length N); scratch y of length N.
  void run(cplx* x, cplx* y, int sign) const {
    if (N == 1) return;
    cplx* src = x;
    cplx* dst = y;
    int Ns = 1;
    std::vector<cplx> vbig;
    for (size_t s = 0; s < radix.size(); ++s) {
      const int R = radix[s];
      const int stride = N / R;  // input element stride of a butterfly
      const cplx* T = stw[s].data();
      const cplx* Dm = dft[s].data();
      cplx v[64];
      cplx* vv = v;
      if (R > 64) { vbig.resize(size_t(R)); vv = vbig.data(); }
      for (int j = 0; j < N / R; ++j) {
        const int jm = j % Ns;
        for (int r = 0; r < R; ++r) {
          const cplx t = sign > 0 ? std::conj(T[size_t(jm) * R + r]) : T[size_t(jm) * R + r];
          vv[r] = src[j + r * stride] * t;
        }
        const int base = (j / Ns) * Ns * R + jm;
        if (R == 2) {
          dst[base] = vv[0] + vv[1];
          dst[base + Ns] = vv[0] - vv[1];
        } else if (R == 4) {
          const cplx a0 = vv[0] + vv[2], a1 = vv[0] - vv[2];
          const cplx b0 = vv[1] + vv[3], b1 = vv[1] - vv[3];
          // multiply b1 by -i (forward) or +i (backward)
          const cplx b1r = sign < 0 ? cplx(b1.imag(), -b1.real()) : cplx(-b1.imag(), b1.real());
          dst[base] = a0 + b0;
          dst[base + Ns] = a1 + b1r;
          dst[base + 2 * Ns] = a0 - b0;
          dst[base + 3 * Ns] = a1 - b1r;
        } else {
          for (int k = 0; k < R; ++k) {
            cplx s2 = 0.0;
            for (int r = 0; r < R; ++r) {
              const cplx t = sign > 0 ? std::conj(Dm[size_t(r) * R + k]) : Dm[size_t(r) * R + k];
              s2 += vv[r] * t;
            }
            dst[base + k * Ns] = s2;
          }
        }
      }
      std::swap(src, dst);
      Ns *= R;
    }
    if (src != x) std::memcpy(x, src, sizeof(cplx) * size_t(N));
  }
};

// Batched d-dimensional c2c over `howmany` slabs of n complex values
// (fftw_plan_many_dft with istride 1, idist n; projection.cpp:115-118).
struct PlanND {
  Grid g;
  std::vector<std::unique_ptr<Plan1D>> ax;
  explicit PlanND(const Grid& gr) : g(gr) {
    for (int a = 0; a < g.dim; ++a) ax.emplace_back(new Plan1D(g.pts[a]));
  }
  // Lines are independent, so they are transformed in parallel (OpenMP) and,
  // on strided axes, gathered kLB adjacent lines at a time (one contiguous
  // kLB*16-byte row per element) -- both change only the memory order of the
  // work, never the arithmetic of a line, so the output is bit-identical to
  // one line at a time on one thread.
  static constexpr size_t kLB = 16;
  void run(cplx* data, int howmany, int sign) const {
    const size_t n = g.n();
    int maxN = 1;
    for (int a = 0; a < g.dim; ++a) maxN = std::max(maxN, g.pts[a]);
    for (int a = 0; a < g.dim; ++a) {
      const int N = g.pts[a];
      if (N == 1) continue;
      size_t inner = 1;
      for (int b = a + 1; b < g.dim; ++b) inner *= size_t(g.pts[b]);
      const size_t outer = n / (inner * size_t(N));
      const size_t nblk = (inner + kLB - 1) / kLB;
      const int64_t jobs = int64_t(howmany) * int64_t(outer) * int64_t(nblk);
      par_for(jobs * int64_t(N) * int64_t(std::min(inner, kLB)), [&](int64_t w0, int64_t w1) {
        const int64_t per = int64_t(N) * int64_t(std::min(inner, kLB));
        std::vector<cplx> buf(size_t(maxN) * kLB), scratch(static_cast<size_t>(maxN));
        for (int64_t job = w0 / per; job < w1 / per; ++job) {
          const size_t ib = size_t(job) % nblk;
          const size_t o = (size_t(job) / nblk) % outer;
          const size_t h = size_t(job) / (nblk * outer);
          cplx* base = data + h * n + o * inner * size_t(N);
          if (inner == 1) {  // contiguous line: in place
            ax[size_t(a)]->run(base, scratch.data(), sign);
            continue;
          }
          const size_t i0 = ib * kLB, nb = std::min(kLB, inner - i0);
          for (int e = 0; e < N; ++e)
            for (size_t b = 0; b < nb; ++b) buf[b * size_t(N) + size_t(e)] = base[size_t(e) * inner + i0 + b];
          for (size_t b = 0; b < nb; ++b) ax[size_t(a)]->run(buf.data() + b * size_t(N), scratch.data(), sign);
          for (int e = 0; e < N; ++e)
            for (size_t b = 0; b < nb; ++b) base[size_t(e) * inner + i0 + b] = buf[b * size_t(N) + size_t(e)];
        }
      });
    }
  }
};

// ---------------------------------------------------------- projection
// index_to_frequency, projection.cpp:18.
inline int index_to_frequency(int i, int n) { return (i < (n + 1) / 2) ? i : i - n; }

struct Projection {
  Grid g;
  int tdim = 3;
  int mode = 0;  // 0 ZeroCompatible, 1 IdentityEquilibrium (projection.hpp:12-15)
  std::vector<double> ghat;  // Tensor2Field, component-major
  std::unique_ptr<PlanND> plan;

  // build_projection, projection.cpp:72-121 (via build_frequency_grid :24-46)
  Projection(const Grid& gr, int td, int md) : g(gr), tdim(td), mode(md) {
    const size_t n = g.n();
    const int d = g.dim;
    ghat.assign(n * size_t(td * td), 0.0);
    for (size_t k = 0; k < n; ++k) {
      int idx[3];
      g.coords(k, idx);
      double xi[3] = {0, 0, 0};
      bool ny = false;
      for (int a = 0; a < d; ++a) {
        const int na = g.pts[a];
        const int qa = index_to_frequency(idx[a], na);
        xi[a] = double(qa) / g.len[a];
        if (na % 2 == 0 && idx[a] == na / 2) ny = true;
      }
      double norm2 = 0.0;
      for (int a = 0; a < d; ++a) norm2 += xi[a] * xi[a];
      if (norm2 == 0.0) continue;  // :92
      if (ny) {                   // :94-98
        if (mode == 0) continue;
        for (int i = 0; i < td; ++i) ghat[size_t(i * td + i) * n + k] = 1.0;
        continue;
      }
      for (int i = 0; i < d; ++i)  // :100-103
        for (int j = 0; j < d; ++j) ghat[size_t(i * td + j) * n + k] = xi[i] * xi[j] / norm2;
    }
    plan.reset(new PlanND(g));
  }
};

double field_norm(const double* a, size_t cnt) {  // tensor_ops.cpp:276-280
  double s = 0.0;
  for (size_t i = 0; i < cnt; ++i) s += a[i] * a[i];
  return std::sqrt(s);
}
double field_dot(const double* a, const double* b, size_t cnt) {  // fields.cpp:60-67
  double s = 0.0;
  for (size_t i = 0; i < cnt; ++i) s += a[i] * b[i];
  return s;
}
void field_mean(const double* a, size_t n, int d, double* mean) {  // tensor_ops.cpp:282-294
  for (int c = 0; c < d * d; ++c) {
    const double* slab = a + size_t(c) * n;
    double s = 0.0;
    for (size_t k = 0; k < n; ++k) s += slab[k];
    mean[c] = s / double(n);
  }
}

// apply_projection, projection.cpp:123-171.  Returns E_COMPLEX_RES when the
// discarded imaginary part exceeds 1e-10 * |A| (:167-169).
int apply_projection(const Projection& G, const double* A, double* out, double* residue_out) {
  const int d = G.tdim;
  const size_t n = G.g.n();
  const size_t total = n * size_t(d * d);
  std::vector<cplx> buf(total);
  par_for(int64_t(total), [&](int64_t a, int64_t b) {
    for (int64_t i = a; i < b; ++i) buf[size_t(i)] = A[i];
  });
  G.plan->run(buf.data(), d * d, -1);
  std::vector<cplx> o(total, cplx(0, 0));
  for (int i = 0; i < d; ++i)  // :139-152, Bhat_ij = Ahat_il ghat_lj
    for (int j = 0; j < d; ++j) {
      cplx* dst = o.data() + size_t(i * d + j) * n;
      for (int l = 0; l < d; ++l) {
        const cplx* src = buf.data() + size_t(i * d + l) * n;
        const double* gg = G.ghat.data() + size_t(l * d + j) * n;
        par_for(int64_t(n), [&](int64_t a, int64_t b) {
          for (int64_t k = a; k < b; ++k) dst[k] += src[k] * gg[k];
        });
      }
    }
  G.plan->run(o.data(), d * d, +1);
  const double scale = 1.0 / double(n);  // :157-165
  double imag2 = 0.0;
  par_for(int64_t(total), [&](int64_t a, int64_t b) {
    for (int64_t i = a; i < b; ++i) out[i] = o[size_t(i)].real() * scale;
  });
  for (size_t i = 0; i < total; ++i) {  // sequential sum, as the reference's
    const double im = o[i].imag() * scale;
    imag2 += im * im;
  }
  const double tol = 1e-10 * std::max(field_norm(A, total), 1e-300);
  const double res = std::sqrt(imag2);
  if (residue_out) *residue_out = res;
  return res > tol ? E_COMPLEX_RES : OK;
}

// apply_projected_tangent, projection.cpp:173-194: dP_ij = K_jikl dF_kl.
int apply_projected_tangent(const Projection& G, const double* K, const double* dF, double* out) {
  const int d = G.tdim;
  const size_t n = G.g.n();
  std::vector<double> dP(n * size_t(d * d), 0.0);
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) {
      double* o = dP.data() + size_t(i * d + j) * n;
      for (int k = 0; k < d; ++k)
        for (int l = 0; l < d; ++l) {
          const double* a = K + size_t(((j * d + i) * d + k) * d + l) * n;
          const double* b = dF + size_t(k * d + l) * n;
          par_for(int64_t(n), [&](int64_t m0, int64_t m1) {
            for (int64_t m = m0; m < m1; ++m) o[m] += a[m] * b[m];
          });
        }
    }
  return apply_projection(G, dP.data(), out, nullptr);
}

// ---------------------------------------------------------- small tensors
// Tensor2::det / inverse, tensor2.hpp:63-113 (3x3 and 2x2 row-major).
double det_t(const double* a, int d) {
  if (d == 2) return a[0] * a[3] - a[1] * a[2];
  return a[0] * (a[4] * a[8] - a[5] * a[7]) - a[1] * (a[3] * a[8] - a[5] * a[6]) +
         a[2] * (a[3] * a[7] - a[4] * a[6]);
}
bool inv3(const double* a, double* inv) {
  const double d = det_t(a, 3);
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

// --------------------------------------------------------- hyperelastic
// hyperelastic_evaluate, hyperelastic.cpp:10-65.
// Nodes are independent: evaluated in parallel; the error reported is the
// one of the LOWEST failing node, i.e. the reference's first throw in node
// order (see for_each_node below).
struct NodeErr {
  int status;
  double value;
};

template <class Body>
int for_each_node(size_t n, Body body, int64_t* bad, double* bad_value) {
  // each chunk stops at its own first failure; the lowest one over all chunks
  // is the lowest failing node
  std::mutex mx;
  int64_t fq = INT64_MAX;
  NodeErr fe{OK, 0.0};
  par_for(int64_t(n), [&](int64_t q0, int64_t q1) {
    for (int64_t q = q0; q < q1; ++q) {
      const NodeErr e = body(size_t(q));
      if (e.status != OK) {
        std::lock_guard<std::mutex> lk(mx);
        if (q < fq) {
          fq = q;
          fe = e;
        }
        break;
      }
    }
  });
  const int fst = fe.status;
  const double fval = fe.value;
  if (fst != OK) {
    if (bad) *bad = fq;
    if (bad_value) *bad_value = fval;
  }
  return fst;
}

int hyper_evaluate(size_t n, int d, const double* F, const double* lambda, const double* mu,
                   double* P, double* K, int64_t* bad) {
  return for_each_node(n, [&](size_t q) -> NodeErr {
    double f[9], b[9], e[9], s[9];
    const double lam = lambda[q], g = mu[q];
    for (int c = 0; c < d * d; ++c) f[c] = F[size_t(c) * n + q];
    if (det_t(f, d) <= 0.0) return {E_INVERTED, 0.0};  // :29
    double trE = 0.0;
    for (int i = 0; i < d; ++i)
      for (int j = 0; j < d; ++j) {
        double bij = 0.0, cij = 0.0;
        for (int k = 0; k < d; ++k) {
          bij += f[i * d + k] * f[j * d + k];
          cij += f[k * d + i] * f[k * d + j];
        }
        b[i * d + j] = bij;
        e[i * d + j] = 0.5 * (cij - (i == j ? 1.0 : 0.0));
      }
    for (int i = 0; i < d; ++i) trE += e[i * d + i];
    for (int i = 0; i < d; ++i)
      for (int j = 0; j < d; ++j) s[i * d + j] = lam * trE * (i == j ? 1.0 : 0.0) + 2.0 * g * e[i * d + j];
    for (int i = 0; i < d; ++i)
      for (int j = 0; j < d; ++j) {
        double v = 0.0;
        for (int k = 0; k < d; ++k) v += f[i * d + k] * s[k * d + j];
        P[size_t(i * d + j) * n + q] = v;
      }
    if (K)
      for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j)
          for (int k = 0; k < d; ++k)
            for (int l = 0; l < d; ++l) {
              double v = lam * f[j * d + i] * f[k * d + l] + g * f[j * d + l] * f[k * d + i];
              if (i == l) v += g * b[j * d + k];
              if (j == k) v += s[i * d + l];
              K[size_t(((i * d + j) * d + k) * d + l) * n + q] = v;
            }
    return {OK, 0.0};
  }, bad, nullptr);
}

// ------------------------------------------------------------- eigen 3x3
// Restates Eigen::SelfAdjointEigenSolver<Matrix3d> (simo.cpp:74): ascending
// eigenvalues, orthonormal eigenvectors as columns of V.  Cyclic Jacobi
// rotations until the off-diagonal mass is below round-off.
void sym_eig3(const double Ain[9], double lam[3], double V[9]) {
  double A[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) A[i][j] = Ain[i * 3 + j];
  double v[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int sweep = 0; sweep < 64; ++sweep) {
    const double off = A[0][1] * A[0][1] + A[0][2] * A[0][2] + A[1][2] * A[1][2];
    const double dg = A[0][0] * A[0][0] + A[1][1] * A[1][1] + A[2][2] * A[2][2];
    if (off == 0.0 || off < 1e-36 * dg) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        const double apq = A[p][q];
        if (apq == 0.0) continue;
        const double theta = (A[q][q] - A[p][p]) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < 3; ++k) {  // A <- J^T A J
          const double akp = A[k][p], akq = A[k][q];
          A[k][p] = c * akp - s * akq;
          A[k][q] = s * akp + c * akq;
        }
        for (int k = 0; k < 3; ++k) {
          const double apk = A[p][k], aqk = A[q][k];
          A[p][k] = c * apk - s * aqk;
          A[q][k] = s * apk + c * aqk;
        }
        for (int k = 0; k < 3; ++k) {
          const double vkp = v[k][p], vkq = v[k][q];
          v[k][p] = c * vkp - s * vkq;
          v[k][q] = s * vkp + c * vkq;
        }
      }
  }
  int ord[3] = {0, 1, 2};
  std::sort(ord, ord + 3, [&](int a, int b) { return A[a][a] < A[b][b]; });
  for (int m = 0; m < 3; ++m) {
    lam[m] = A[ord[m]][ord[m]];
    for (int i = 0; i < 3; ++i) V[i * 3 + m] = v[i][ord[m]];
  }
}

// log_divided_difference, simo.cpp:18-22.
inline double log_divided_difference(double a, double b) {
  const double scale = std::max(a, b);
  if (std::abs(b - a) < 1e-7 * scale) return 2.0 / (a + b);
  return (std::log(b) - std::log(a)) / (b - a);
}

// ------------------------------------------------------------------ Simo
// simo_evaluate, simo.cpp:26-196; always 3x3 (plane strain on 2-d grids).
int simo_evaluate(size_t n, const double* F, const double* Fold, const double* be_c,
                  const double* epsp_c, const double* lambda, const double* mu,
                  const double* tau_y0, const double* hard, double* P, double* K, double* be_t,
                  double* epsp_t, int64_t* bad, double* bad_value) {
  return for_each_node(n, [&](size_t q) -> NodeErr {
    double D[3][3][3][3], L[3][3][3][3], DL[3][3][3][3], A4[3][3][3][3];
    const double lam = lambda[q], g = mu[q], ty0 = tau_y0[q], h = hard[q];
    double Fm[9], Fo[9], Finv[9], Foinv[9], f[9], be[9];
    for (int c = 0; c < 9; ++c) {
      Fm[c] = F[size_t(c) * n + q];
      Fo[c] = Fold[size_t(c) * n + q];
      be[c] = be_c[size_t(c) * n + q];
    }
    if (det_t(Fm, 3) <= 0.0) return {E_INVERTED, 0.0};  // :49
    if (!inv3(Fm, Finv) || !inv3(Fo, Foinv)) return {E_SINGULAR, 0.0};
    for (int i = 0; i < 3; ++i)  // f = F F_old^-1, :60-66
      for (int j = 0; j < 3; ++j) {
        double s = 0.0;
        for (int k = 0; k < 3; ++k) s += Fm[i * 3 + k] * Foinv[k * 3 + j];
        f[i * 3 + j] = s;
      }
    double tmp[9], betr[9], bsym[9];
    for (int i = 0; i < 3; ++i)  // be_tr = f be f^T, :70-72
      for (int j = 0; j < 3; ++j) {
        double s = 0.0;
        for (int k = 0; k < 3; ++k) s += f[i * 3 + k] * be[k * 3 + j];
        tmp[i * 3 + j] = s;
      }
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double s = 0.0;
        for (int k = 0; k < 3; ++k) s += tmp[i * 3 + k] * f[j * 3 + k];
        betr[i * 3 + j] = s;
      }
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) bsym[i * 3 + j] = 0.5 * (betr[i * 3 + j] + betr[j * 3 + i]);
    double lb[3], V[9];
    sym_eig3(bsym, lb, V);  // :74-78
    for (int m = 0; m < 3; ++m)
      if (lb[m] < 1e-30) return {E_NOT_SPD, lb[m]};  // kMinLogEigenvalue, tensor_ops.hpp:56
    double eps[3], tau_d[3], dev[3];
    for (int m = 0; m < 3; ++m) eps[m] = 0.5 * std::log(lb[m]);  // :81
    const double tr_eps = eps[0] + eps[1] + eps[2];
    for (int m = 0; m < 3; ++m) tau_d[m] = lam * tr_eps + 2.0 * g * eps[m];
    const double tau_m = (tau_d[0] + tau_d[1] + tau_d[2]) / 3.0;
    for (int m = 0; m < 3; ++m) dev[m] = tau_d[m] - tau_m;
    const double taueq_tr = std::sqrt(1.5 * (dev[0] * dev[0] + dev[1] * dev[1] + dev[2] * dev[2]));
    const double tauy = ty0 + h * epsp_c[q];
    const double phi = taueq_tr - tauy;
    const bool plastic = phi >= -1e-12 * tauy;  // :96
    double dgamma = 0.0, N2[3] = {0, 0, 0}, eps_e[3] = {eps[0], eps[1], eps[2]};
    if (plastic) {
      dgamma = std::max(phi, 0.0) / (3.0 * g + h);  // :101
      for (int m = 0; m < 3; ++m) N2[m] = 1.5 * dev[m] / taueq_tr;
      for (int m = 0; m < 3; ++m) {
        tau_d[m] -= 2.0 * g * dgamma * N2[m];
        eps_e[m] = eps[m] - dgamma * N2[m];
      }
    }
    double tau[9] = {0}, benew[9] = {0}, N2m[9] = {0};  // :110-120
    for (int m = 0; m < 3; ++m) {
      const double ex = std::exp(2.0 * eps_e[m]);
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
          const double pr = V[i * 3 + m] * V[j * 3 + m];
          tau[i * 3 + j] += tau_d[m] * pr;
          benew[i * 3 + j] += ex * pr;
          if (plastic) N2m[i * 3 + j] += N2[m] * pr;
        }
    }
    for (int c = 0; c < 9; ++c) be_t[size_t(c) * n + q] = benew[c];
    epsp_t[q] = epsp_c[q] + dgamma;
    for (int i = 0; i < 3; ++i)  // P = tau F^-T, :122-128
      for (int j = 0; j < 3; ++j) {
        double s = 0.0;
        for (int k = 0; k < 3; ++k) s += tau[i * 3 + k] * Finv[j * 3 + k];
        P[size_t(i * 3 + j) * n + q] = s;
      }
    if (!K) return {OK, 0.0};
    for (int i = 0; i < 3; ++i)  // D, :131-147
      for (int j = 0; j < 3; ++j)
        for (int k = 0; k < 3; ++k)
          for (int l = 0; l < 3; ++l) {
            const double did = i == j ? 1.0 : 0.0, dkl = k == l ? 1.0 : 0.0;
            const double is = 0.5 * (((i == k && j == l) ? 1.0 : 0.0) + ((i == l && j == k) ? 1.0 : 0.0));
            double v = lam * did * dkl + 2.0 * g * is;
            if (plastic) {
              const double isdev = is - did * dkl / 3.0;
              const double a0 = dgamma / taueq_tr;
              v += -6.0 * g * g * a0 * isdev -
                   4.0 * g * g * (1.0 / (3.0 * g + h) - a0) * N2m[i * 3 + j] * N2m[k * 3 + l];
            }
            D[i][j][k][l] = v;
          }
    std::memset(L, 0, sizeof(L));  // dln, :150-162
    for (int m = 0; m < 3; ++m)
      for (int p = 0; p < 3; ++p) {
        const double w = log_divided_difference(lb[m], lb[p]);
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j)
            for (int k = 0; k < 3; ++k)
              for (int l = 0; l < 3; ++l)
                L[i][j][k][l] += w * V[i * 3 + m] * V[j * 3 + p] * V[k * 3 + m] * V[l * 3 + p];
      }
    for (int i = 0; i < 3; ++i)  // :165-182
      for (int j = 0; j < 3; ++j)
        for (int m = 0; m < 3; ++m)
          for (int p = 0; p < 3; ++p) {
            double s = 0.0;
            for (int k = 0; k < 3; ++k)
              for (int l = 0; l < 3; ++l) s += D[i][j][k][l] * L[k][l][m][p];
            DL[i][j][m][p] = s;
          }
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        for (int k = 0; k < 3; ++k)
          for (int l = 0; l < 3; ++l) {
            double s = 0.0;
            for (int a = 0; a < 3; ++a) s += DL[i][j][k][a] * betr[a * 3 + l];
            if (i == k) s -= tau[j * 3 + l];
            A4[i][j][k][l] = s;
          }
    for (int i = 0; i < 3; ++i)  // K = F^-1 Kx F^-T, :183-194
      for (int j = 0; j < 3; ++j)
        for (int k = 0; k < 3; ++k)
          for (int l = 0; l < 3; ++l) {
            double s = 0.0;
            for (int a = 0; a < 3; ++a) {
              double t = 0.0;
              for (int b = 0; b < 3; ++b) t += A4[a][j][k][b] * Finv[l * 3 + b];
              s += Finv[i * 3 + a] * t;
            }
            K[size_t(((i * 3 + j) * 3 + k) * 3 + l) * n + q] = s;
          }
    return {OK, 0.0};
  }, bad, bad_value);
}

// ---------------------------------------------------------------- models
// MaterialModel contract, material.hpp:45-65.
struct Model {
  int kind = 0;  // 0 hyperelastic (tdim = grid dim or given), 1 Simo (tdim 3)
  int tdim = 3;
  size_t n = 0;
  std::vector<double> lambda, mu, ty0, hard;
  std::vector<double> be_c, epsp_c, be_t, epsp_t, f_old;  // Simo history, simo.cpp:198-223
  void init_history() {
    if (kind != 1) return;
    be_c.assign(9 * n, 0.0);
    f_old.assign(9 * n, 0.0);
    for (int i = 0; i < 3; ++i)
      for (size_t q = 0; q < n; ++q) {
        be_c[size_t(i * 4) * n + q] = 1.0;  // HistoryState init I, material.cpp:11-12
        f_old[size_t(i * 4) * n + q] = 1.0; // f_old_ = I, simo.cpp:208
      }
    epsp_c.assign(n, 0.0);
    be_t = be_c;
    epsp_t = epsp_c;
  }
  int evaluate(const double* F, double* P, double* K, OracleError* err) {
    int64_t bad = -1;
    double bv = 0.0;
    int st;
    if (kind == 0)
      st = hyper_evaluate(n, tdim, F, lambda.data(), mu.data(), P, K, &bad);
    else
      st = simo_evaluate(n, F, f_old.data(), be_c.data(), epsp_c.data(), lambda.data(), mu.data(),
                         ty0.data(), hard.data(), P, K, be_t.data(), epsp_t.data(), &bad, &bv);
    if (st != OK && err) *err = {st, bad, bv};
    return st;
  }
  void commit(const double* F) {  // simo.cpp:220-223
    if (kind != 1) return;
    be_c = be_t;
    epsp_c = epsp_t;
    std::memcpy(f_old.data(), F, sizeof(double) * 9 * n);
  }
};

// ---------------------------------------------------------------- solver
struct SolverParams {
  double eta_newton = 1e-5, eta_cg = 1e-8;
  int max_newton = 30, max_cg = 0;
};

struct CgResult {
  int iterations;
  double rel;
};

// cg_solve, solver.cpp:19-58.
int cg_solve(const Projection& G, const double* K, const double* b, const SolverParams& prm,
             double* x, CgResult* res) {
  const int d = G.tdim;
  const size_t cnt = G.g.n() * size_t(d * d);
  std::fill(x, x + cnt, 0.0);
  const double bnorm = field_norm(b, cnt);
  if (bnorm == 0.0) {
    *res = {0, 0.0};
    return OK;
  }
  const int cap = prm.max_cg > 0 ? prm.max_cg : int(G.g.n()) * d * d;
  std::vector<double> r(b, b + cnt), p(r), Ap(cnt);
  double rr = field_dot(r.data(), r.data(), cnt);
  for (int it = 1; it <= cap; ++it) {
    int st = apply_projected_tangent(G, K, p.data(), Ap.data());
    if (st != OK) return st;
    const double pAp = field_dot(p.data(), Ap.data(), cnt);
    if (!(pAp > 0.0)) {
      *res = {it, std::sqrt(rr) / bnorm};
      return OK;
    }
    const double alpha = rr / pAp;
    par_for(int64_t(cnt), [&](int64_t a, int64_t b) {
      for (int64_t i = a; i < b; ++i) {
        x[i] += alpha * p[size_t(i)];
        r[size_t(i)] += -alpha * Ap[size_t(i)];
      }
    });
    const double rr_new = field_dot(r.data(), r.data(), cnt);
    if (std::sqrt(rr_new) <= prm.eta_cg * bnorm) {
      *res = {it, std::sqrt(rr_new) / bnorm};
      return OK;
    }
    const double beta = rr_new / rr;
    rr = rr_new;
    par_for(int64_t(cnt), [&](int64_t a, int64_t b) {
      for (int64_t i = a; i < b; ++i) {
        p[size_t(i)] *= beta;
        p[size_t(i)] += r[size_t(i)];
      }
    });
  }
  *res = {cap, std::sqrt(rr) / bnorm};
  return E_CG_STALLED;
}

struct PassRec {
  int cg_it;
  double cg_rel, rel_update;
};

struct Report {
  std::vector<PassRec> passes;
  double eq_rel = 0.0, drift = 0.0, wall = 0.0;
  bool converged = false;
};

double mean_drift(const double* F, size_t n, int d, const double* fbar) {  // solver.cpp:62-69
  double mean[9];
  field_mean(F, n, d, mean);
  double drift = 0.0;
  for (int c = 0; c < d * d; ++c) drift = std::max(drift, std::abs(mean[c] - fbar[c]));
  return drift;
}

// solve_increment, solver.cpp:73-160.
int solve_increment(const Projection& G, Model& model, double* F, const double* fbar,
                    const SolverParams& prm, Report* rep, double* P_out, OracleError* err) {
  const int d = G.tdim;
  const size_t n = G.g.n();
  const size_t cnt = n * size_t(d * d);
  if (!(det_t(fbar, d) > 0.0)) return E_INVALID;  // :77-79
  const auto t0 = std::chrono::steady_clock::now();
  const double norm_ref = field_norm(F, cnt);  // :88
  std::vector<double> P(cnt), K(cnt * size_t(d * d)), dF(cnt), rhs(cnt), tmp(cnt);
  auto finish = [&](bool conv) {
    rep->converged = conv;
    rep->wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  };
  int st;
  {  // BC pass, :101-122
    if ((st = model.evaluate(F, P.data(), K.data(), err)) != OK) return st;
    double mean[9], dfbar[9];
    field_mean(F, n, d, mean);
    for (int c = 0; c < d * d; ++c) dfbar[c] = fbar[c] - mean[c];
    for (int c = 0; c < d * d; ++c)
      for (size_t q = 0; q < n; ++q) tmp[size_t(c) * n + q] = 0.0 + dfbar[c];
    if ((st = apply_projected_tangent(G, K.data(), tmp.data(), rhs.data())) != OK) return st;
    for (auto& v : rhs) v *= -1.0;
    CgResult cg;
    if ((st = cg_solve(G, K.data(), rhs.data(), prm, dF.data(), &cg)) != OK) {
      finish(false);
      if (err) *err = {st, cg.iterations, cg.rel};
      return st;
    }
    for (int c = 0; c < d * d; ++c)
      for (size_t q = 0; q < n; ++q) F[size_t(c) * n + q] += dfbar[c];
    for (size_t i = 0; i < cnt; ++i) F[i] += dF[i];
    rep->passes.push_back({cg.iterations, cg.rel, field_norm(dF.data(), cnt) / norm_ref});
    rep->drift = std::max(rep->drift, mean_drift(F, n, d, fbar));
  }
  while (true) {  // :125-147
    if (int(rep->passes.size()) >= prm.max_newton) {
      finish(false);
      return E_NEWTON_DIV;
    }
    if ((st = model.evaluate(F, P.data(), K.data(), err)) != OK) return st;
    if ((st = apply_projection(G, P.data(), rhs.data(), nullptr)) != OK) return st;
    for (auto& v : rhs) v *= -1.0;
    CgResult cg;
    if ((st = cg_solve(G, K.data(), rhs.data(), prm, dF.data(), &cg)) != OK) {
      finish(false);
      if (err) *err = {st, cg.iterations, cg.rel};
      return st;
    }
    for (size_t i = 0; i < cnt; ++i) F[i] += dF[i];
    const double rel = field_norm(dF.data(), cnt) / norm_ref;
    rep->passes.push_back({cg.iterations, cg.rel, rel});
    rep->drift = std::max(rep->drift, mean_drift(F, n, d, fbar));
    if (rel < prm.eta_newton) break;
  }
  if ((st = model.evaluate(F, P.data(), K.data(), err)) != OK) return st;  // :151-155
  const double pnorm = field_norm(P.data(), cnt);
  if (pnorm > 0.0) {
    if ((st = apply_projection(G, P.data(), tmp.data(), nullptr)) != OK) return st;
    rep->eq_rel = field_norm(tmp.data(), cnt) / pnorm;
  } else {
    rep->eq_rel = 0.0;
  }
  model.commit(F);
  if (P_out) std::memcpy(P_out, P.data(), sizeof(double) * cnt);
  finish(true);
  return OK;
}

}  // namespace oracle

// ============================================================ C ABI (ctypes)
using namespace oracle;

namespace {
Grid make_grid(int dim, const int* pts, const double* len) {
  Grid g;
  g.dim = dim;
  for (int a = 0; a < 3; ++a) {
    g.pts[a] = a < dim ? pts[a] : 1;
    g.len[a] = a < dim ? len[a] : 1.0;
  }
  return g;
}
}  // namespace

extern "C" {

// Worker threads of the parallel loops (default 1, or $OR_THREADS: the
// reference itself is single-threaded).  Results do not depend on it: only
// independent lines / nodes / vector entries are split across threads, every
// reduction is the reference's sequential sum (see PlanND::run).
int or_set_threads(int nthreads) {
  g_threads = nthreads < 1 ? 1 : nthreads;
  return g_threads;
}

struct or_report {
  int32_t n_passes;
  int32_t converged;
  int32_t status;
  int32_t pad_;
  int64_t err_node;
  double err_value;
  double eq_rel, drift, wall;
  int32_t cg_it[64];
  double cg_rel[64];
  double rel_update[64];
};

int or_apply_projection(int dim, const int* pts, const double* len, int tdim, int mode,
                        const double* A, double* out, double* residue) {
  Projection G(make_grid(dim, pts, len), tdim, mode);
  return apply_projection(G, A, out, residue);
}

int or_ghat(int dim, const int* pts, const double* len, int tdim, int mode, double* out) {
  Projection G(make_grid(dim, pts, len), tdim, mode);
  std::memcpy(out, G.ghat.data(), sizeof(double) * G.ghat.size());
  return OK;
}

int or_apply_projected_tangent(int dim, const int* pts, const double* len, int tdim, int mode,
                               const double* K, const double* dF, double* out) {
  Projection G(make_grid(dim, pts, len), tdim, mode);
  return apply_projected_tangent(G, K, dF, out);
}

// Unnormalised c2c DFT along every axis of `howmany` slabs (the restated
// FFTW transform itself), for pinning against a naive O(n^2) DFT.
int or_fft(int dim, const int* pts, int howmany, int sign, double* data_interleaved) {
  const double one[3] = {1, 1, 1};
  PlanND p(make_grid(dim, pts, one));
  p.run(reinterpret_cast<cplx*>(data_interleaved), howmany, sign);
  return OK;
}

int or_hyper_evaluate(int64_t n, int tdim, const double* F, const double* lambda,
                      const double* mu, double* P, double* K, int64_t* bad) {
  return hyper_evaluate(size_t(n), tdim, F, lambda, mu, P, K, bad);
}

int or_simo_evaluate(int64_t n, const double* F, const double* Fold, const double* be_c,
                     const double* epsp_c, const double* lambda, const double* mu,
                     const double* ty0, const double* hard, double* P, double* K, double* be_t,
                     double* epsp_t, int64_t* bad, double* bad_value) {
  return simo_evaluate(size_t(n), F, Fold, be_c, epsp_c, lambda, mu, ty0, hard, P, K, be_t, epsp_t,
                       bad, bad_value);
}

// equivalent_stress (material.cpp:14-31) of P, of inv2(F).P (hyperelastic.cpp:
// 89-92; inv2 = Tensor2::inverse with the kSingularDetTol check, tensor_ops.cpp:
// 257-266, tensor2.hpp:63-113) or of P.F^T (simo.cpp:225-228; dot22 sums the
// inner index in order, tensor_ops.cpp:138-153).  kind 0 / 1 / 2.
int or_equivalent_stress(int64_t n, int tdim, int kind, const double* F, const double* P, double* out,
                         int64_t* bad) {
  const int d = tdim;
  for (int64_t q = 0; q < n; ++q) {
    double p[9], f[9], t[9];
    for (int c = 0; c < d * d; ++c) p[c] = P[c * n + q];
    if (kind == 0) {
      for (int c = 0; c < d * d; ++c) t[c] = p[c];
    } else {
      for (int c = 0; c < d * d; ++c) f[c] = F[c * n + q];
      if (kind == 1) {
        double det, inv[9];
        if (d == 2) {
          det = f[0] * f[3] - f[1] * f[2];
        } else {
          det = f[0] * (f[4] * f[8] - f[5] * f[7]) - f[1] * (f[3] * f[8] - f[5] * f[6]) +
                f[2] * (f[3] * f[7] - f[4] * f[6]);
        }
        if (std::fabs(det) < 1e-30) {
          if (bad) *bad = q;
          return E_SINGULAR;
        }
        if (d == 2) {
          inv[0] = f[3] / det;
          inv[1] = -f[1] / det;
          inv[2] = -f[2] / det;
          inv[3] = f[0] / det;
        } else {
          inv[0] = (f[4] * f[8] - f[5] * f[7]) / det;
          inv[1] = (f[2] * f[7] - f[1] * f[8]) / det;
          inv[2] = (f[1] * f[5] - f[2] * f[4]) / det;
          inv[3] = (f[5] * f[6] - f[3] * f[8]) / det;
          inv[4] = (f[0] * f[8] - f[2] * f[6]) / det;
          inv[5] = (f[2] * f[3] - f[0] * f[5]) / det;
          inv[6] = (f[3] * f[7] - f[4] * f[6]) / det;
          inv[7] = (f[1] * f[6] - f[0] * f[7]) / det;
          inv[8] = (f[0] * f[4] - f[1] * f[3]) / det;
        }
        for (int i = 0; i < d; ++i)
          for (int k = 0; k < d; ++k) {
            double s = 0.0;
            for (int j = 0; j < d; ++j) s += inv[i * d + j] * p[j * d + k];
            t[i * d + k] = s;
          }
      } else {
        for (int i = 0; i < d; ++i)
          for (int k = 0; k < d; ++k) {
            double s = 0.0;
            for (int j = 0; j < d; ++j) s += p[i * d + j] * f[k * d + j];
            t[i * d + k] = s;
          }
      }
    }
    double tr = 0.0;
    for (int i = 0; i < d; ++i) tr += t[i * d + i];
    tr /= double(d);
    double s = 0.0;
    for (int i = 0; i < d; ++i)
      for (int j = 0; j < d; ++j) {
        const double dv = t[i * d + j] - (i == j ? tr : 0.0);
        s += dv * dv;
      }
    out[q] = std::sqrt(1.5 * s);
  }
  return OK;
}

int or_sym_eig3(const double* A, double* lam, double* V) {
  sym_eig3(A, lam, V);
  return OK;
}

int or_cg_solve(int dim, const int* pts, const double* len, int tdim, int mode, const double* K,
                const double* rhs, double eta_cg, int max_cg, double* x, int* iters,
                double* rel) {
  Projection G(make_grid(dim, pts, len), tdim, mode);
  SolverParams prm;
  prm.eta_cg = eta_cg;
  prm.max_cg = max_cg;
  CgResult r{0, 0.0};
  const int st = cg_solve(G, K, rhs, prm, x, &r);
  *iters = r.iterations;
  *rel = r.rel;
  return st;
}

// Runs a load program (run_program, solver.cpp:162-169) of n_inc increments
// with per-node parameters.  kind 0 = HyperelasticModel, 1 = SimoPlasticityModel.
// F (in/out) holds the state; P_out receives the last converged P; reports
// has n_inc entries; epsp_out (Simo only, may be null) the committed eps_p.
int or_run_program(int dim, const int* pts, const double* len, int tdim, int mode, int kind,
                   const double* lambda, const double* mu, const double* ty0, const double* hard,
                   int n_inc, const double* fbars, double eta_newton, double eta_cg,
                   int max_newton, int max_cg, double* F, double* P_out, double* epsp_out,
                   or_report* reports) {
  const Grid g = make_grid(dim, pts, len);
  Projection G(g, tdim, mode);
  Model m;
  m.kind = kind;
  m.tdim = tdim;
  m.n = g.n();
  m.lambda.assign(lambda, lambda + m.n);
  m.mu.assign(mu, mu + m.n);
  if (kind == 1) {
    m.ty0.assign(ty0, ty0 + m.n);
    m.hard.assign(hard, hard + m.n);
  }
  m.init_history();
  SolverParams prm{eta_newton, eta_cg, max_newton, max_cg};
  for (int t = 0; t < n_inc; ++t) {
    Report rep;
    OracleError err{0, -1, 0.0};
    const int st = solve_increment(G, m, F, fbars + size_t(t) * size_t(tdim * tdim), prm, &rep,
                                   P_out, &err);
    or_report& R = reports[t];
    std::memset(&R, 0, sizeof(R));
    R.n_passes = int(rep.passes.size());
    R.converged = rep.converged ? 1 : 0;
    R.status = st;
    R.err_node = err.node;
    R.err_value = err.value;
    R.eq_rel = rep.eq_rel;
    R.drift = rep.drift;
    R.wall = rep.wall;
    for (size_t i = 0; i < rep.passes.size() && i < 64; ++i) {
      R.cg_it[i] = rep.passes[i].cg_it;
      R.cg_rel[i] = rep.passes[i].cg_rel;
      R.rel_update[i] = rep.passes[i].rel_update;
    }
    if (st != OK) return st;
  }
  if (epsp_out && kind == 1) std::memcpy(epsp_out, m.epsp_c.data(), sizeof(double) * m.n);
  return OK;
}

// Times `reps` applications of apply_projected_tangent (the
// BM_apply_projected_tangent_3d pattern, bench_projection.cpp:31-44) on the
// given buffers; returns seconds per application.
double or_time_projected_tangent(int dim, const int* pts, const double* len, int tdim,
                                 const double* K, const double* dF, double* out, int reps) {
  Projection G(make_grid(dim, pts, len), tdim, 0);
  apply_projected_tangent(G, K, dF, out);  // warm-up (page-in)
  const auto t0 = std::chrono::steady_clock::now();
  for (int r = 0; r < reps; ++r) apply_projected_tangent(G, K, dF, out);
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / reps;
}

}  // extern "C"
