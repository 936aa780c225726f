// C++ drop-in check: reference-style client code written against the
// `namespace fftmech` API (the reference's headers' names and semantics),
// linked against libfftmech_host.so -> libfftmech_b200.so, running on the
// B200.  The assertions restate the reference's unit tests
// (proj/tests/unit/test_projection.cpp, test_solver.cpp,
// test_hyperelastic.cpp, test_simo.cpp) and its golden run record
// proj/unit_det_out1/report.csv.  Prints one line per case; exit code 0 iff
// every CHECK held.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <sstream>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "fftmech/hyperelastic.hpp"
#include "fftmech/microstructure.hpp"
#include "fftmech/projection.hpp"
#include "fftmech/run_config.hpp"
#include "fftmech/simo.hpp"
#include "fftmech/snapshot.hpp"
#include "fftmech/solver.hpp"
#include "fftmech/tensor_ops.hpp"

using namespace fftmech;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                           \
  do {                                                                        \
    ++g_checks;                                                               \
    if (!(cond)) {                                                            \
      ++g_fail;                                                               \
      std::printf("    CHECK FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                         \
  } while (0)

static void run(const char* name, const std::function<void()>& body) {
  const int before = g_fail;
  try {
    body();
  } catch (const std::exception& e) {
    ++g_fail;
    std::printf("    unexpected exception: %s\n", e.what());
  }
  std::printf("[%s] %s\n", g_fail == before ? "PASS" : "FAIL", name);
}

static Tensor2Field random_field(const GridShape& s, int tdim, std::mt19937& rng, double amp = 1.0) {
  std::uniform_real_distribution<double> u(-amp, amp);
  Tensor2Field f(s, tdim);
  for (double& v : f.data()) v = u(rng);
  return f;
}

static Tensor4Field stiffness(const GridShape& s, int d, double lam, double mu) {
  Tensor4Field C = dyad22(identity2(s, d), identity2(s, d));
  C *= lam;
  Tensor4Field Is = identity4sym(s, d);
  Is *= 2.0 * mu;
  C += Is;
  return C;
}

// A user-defined host material (not device-backed): exercises the path where
// the constitutive update is client code and projection/CG run on the GPU.
class HostSvk final : public MaterialModel {
 public:
  HostSvk(const GridShape& s, int d, ElasticParams p) : s_(s), d_(d), p_(p) {}
  int tensor_dim() const override { return d_; }
  void evaluate(const Tensor2Field& F, Tensor2Field& P, Tensor4Field& K) override {
    const double lam = p_.lame_lambda(), mu = p_.lame_mu();
    P = Tensor2Field(s_, d_);
    K = Tensor4Field(s_, d_);
    for (std::size_t q = 0; q < F.nodes(); ++q) {
      const Tensor2 f = F.tensor(q);
      Tensor2 E = dot(f.transposed(), f) - Tensor2::identity(d_);
      E *= 0.5;
      Tensor2 S = 2.0 * mu * E;
      for (int i = 0; i < d_; ++i) S(i, i) += lam * E.trace();
      P.set_tensor(q, dot(f, S));
      const Tensor2 b = dot(f, f.transposed());
      for (int i = 0; i < d_; ++i)
        for (int j = 0; j < d_; ++j)
          for (int k = 0; k < d_; ++k)
            for (int l = 0; l < d_; ++l)
              K.at(q, i, j, k, l) = lam * f(j, i) * f(k, l) + mu * f(j, l) * f(k, i) + (i == l ? mu * b(j, k) : 0.0) +
                                    (j == k ? S(i, l) : 0.0);
    }
  }
  void commit(const Tensor2Field&) override {}
  ScalarField equivalent_stress_field(const Tensor2Field&, const Tensor2Field& P) const override {
    return equivalent_stress(P);
  }

 private:
  GridShape s_;
  int d_;
  ElasticParams p_;
};

static std::string slurp(const std::filesystem::path& p) {
  std::ifstream in(p, std::ios::binary);
  std::ostringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

static std::vector<std::vector<std::string>> csv_rows(const std::filesystem::path& p) {
  std::vector<std::vector<std::string>> rows;
  std::istringstream in(slurp(p));
  std::string line;
  while (std::getline(in, line)) {
    std::vector<std::string> cells;
    std::istringstream ls(line);
    std::string c;
    while (std::getline(ls, c, ',')) cells.push_back(c);
    rows.push_back(cells);
  }
  return rows;
}

// One reference run (execute_run's loop, run_config.cpp:497-524) written
// through SnapshotSink, then compared with the reference's own record
// directory: meta_<k>.json and VTK byte-for-byte, report.csv on every column
// but wall_ms (newton/cg exact, residual to 1e-6 relative -- the CG vectors'
// round-off -- and eps_bar to 1e-14).
static void check_run_against_record(const std::filesystem::path& golden, const std::string& rec,
                                     const GridShape& s, const std::vector<double>& fractions,
                                     const std::vector<ElasticParams>& phases, double gamma, int increments,
                                     OutputOptions opts) {
  namespace fs = std::filesystem;
  const fs::path out = fs::temp_directory_path() / ("fftmech_b200_" + rec);
  fs::remove_all(out);
  opts.directory = out;
  const PhaseGrid pg = make_laminate(s, fractions);
  std::vector<ElasticParams> used(phases.begin(), phases.begin() + pg.phase_count);
  const MaterialFields mf = bind_parameters(pg, used);
  HyperelasticModel model(s, s.dim, mf.lambda, mf.mu);
  const ProjectionOperator G = build_projection(s, s.dim);
  Tensor2Field F = identity2(s, s.dim);
  LoadProgram program;
  for (int t = 1; t <= increments; ++t) {
    Tensor2 f = Tensor2::identity(s.dim);
    f(0, 1) = gamma * static_cast<double>(t) / increments;
    program.push_back({f, std::to_string(t)});
  }
  SnapshotSink sink(opts);
  run_program(F, model, G, program, SolverParams{}, sink);
  sink.finish();
  const fs::path ref = golden / rec;
  for (const auto& e : fs::directory_iterator(ref)) {
    const std::string name = e.path().filename().string();
    if (name == "report.csv") continue;
    const bool same = slurp(out / name) == slurp(e.path());
    if (!same) std::printf("    %s/%s differs from the reference record\n", rec.c_str(), name.c_str());
    CHECK(same);
  }
  const auto got = csv_rows(out / "report.csv"), want = csv_rows(ref / "report.csv");
  CHECK(got.size() == want.size());
  for (size_t r = 0; r < std::min(got.size(), want.size()); ++r) {
    CHECK(got[r].size() == 6 && want[r].size() == 6);
    if (got[r].size() != 6 || want[r].size() != 6) continue;
    if (r == 0) {
      for (int c = 0; c < 6; ++c) CHECK(got[r][c] == want[r][c]);
      continue;
    }
    CHECK(got[r][0] == want[r][0] && got[r][1] == want[r][1] && got[r][2] == want[r][2]);
    const double rg = std::stod(got[r][3]), rw = std::stod(want[r][3]);
    CHECK(std::abs(rg - rw) <= 1e-6 * std::abs(rw));
    const double eg = std::stod(got[r][5]), ew = std::stod(want[r][5]);
    CHECK(std::abs(eg - ew) <= 1e-14 * std::abs(ew));
  }
  CHECK(list_snapshots(out).size() == size_t((increments) / opts.stride));
}

// parse_config behaviour (proj/tests/unit/test_config_io.cpp:40-133); host only.
static const char* kMinimalCube = R"({
  "grid": {"points": [3, 3, 3]},
  "microstructure": {"kind": "cube", "volume_fraction": 0.037},
  "model": {"kind": "hyperelastic",
            "phases": [{"youngs": 1.0, "poisson": 0.3},
                       {"youngs": 10.0, "poisson": 0.3}]},
  "loading": {"mode": "simple_shear", "gamma": 0.1, "increments": 1}
})";

static void config_cases() {
  run("config: minimal config picks up the documented defaults", [] {
    const RunConfig cfg = parse_config(kMinimalCube);
    CHECK(cfg.solver.eta_newton == 1e-5 && cfg.solver.eta_cg == 1e-8 && cfg.solver.max_newton == 30);
    CHECK(cfg.nyquist == NyquistMode::ZeroCompatible && cfg.snapshot_stride == 1 && cfg.tensor_dim() == 3);
    CHECK(cfg.output_fields == (std::vector<std::string>{"F", "P", "eq"}));
  });
  run("config: poisson = 0.5 is flagged at its config path", [] {
    std::string text = kMinimalCube;
    text.replace(text.find("0.3"), 3, "0.5");
    bool ok = false;
    try {
      parse_config(text);
    } catch (const ConfigInvalid& e) {
      ok = e.violations.size() == 1 && e.violations[0].find("model.phases[0].poisson") != std::string::npos;
    }
    CHECK(ok);
  });
  run("config: all violations are collected, not just the first", [] {
    const char* broken = R"({
      "grid": {"points": [3, 3, 3]},
      "microstructure": {"kind": "cube", "volume_fraction": 1.5},
      "model": {"kind": "hyperelastic",
                "phases": [{"youngs": -1.0, "poisson": 0.7}, {"youngs": 10.0, "poisson": 0.3}]},
      "loading": {"mode": "pure_shear", "lambda": -2.0, "increments": 0}
    })";
    size_t nv = 0;
    try {
      parse_config(broken);
    } catch (const ConfigInvalid& e) {
      nv = e.violations.size();
    }
    CHECK(nv >= 5);
  });
  run("config: pure shear expands to a uniform stretch ramp (plane strain Simo)", [] {
    const RunConfig cfg = parse_config(R"({
      "grid": {"points": [4, 4]},
      "microstructure": {"kind": "laminate", "fractions": [0.5, 0.5]},
      "model": {"kind": "simo", "contrast": 2.0,
                "phases": [{"youngs": 1.0, "poisson": 0.3, "tau_y0": 0.003, "hardening": 0.01}]},
      "loading": {"mode": "pure_shear", "lambda": 1.2, "increments": 250}
    })");
    CHECK(cfg.tensor_dim() == 3);
    const LoadProgram prog = expand_loading(cfg);
    CHECK(prog.size() == 250);
    double worst = 0.0;
    for (size_t t = 0; t < prog.size(); ++t) {
      const double lam = 1.0 + 0.2 * double(t + 1) / 250.0;
      worst = std::max({worst, std::abs(prog[t].fbar(0, 0) - lam) / lam,
                        std::abs(prog[t].fbar(1, 1) - 1.0 / lam) * lam});
      CHECK(prog[t].fbar(2, 2) == 1.0 && prog[t].label == std::to_string(t + 1));
    }
    CHECK(worst < 1e-14);
  });
  run("config: explicit loading lists are validated matrix by matrix", [] {
    bool ok = false;
    try {
      parse_config(R"({
        "grid": {"points": [3, 3]},
        "microstructure": {"kind": "laminate", "fractions": [1.0]},
        "model": {"kind": "hyperelastic", "phases": [{"youngs": 1.0, "poisson": 0.3}]},
        "loading": {"mode": "explicit", "fbar": [[[1.0, 0.1], [0.0, 1.0]], [[-1.0, 0.0], [0.0, 1.0]]]}
      })");
    } catch (const ConfigInvalid& e) {
      ok = e.violations.size() == 1 && e.violations[0].find("loading.fbar[1]") != std::string::npos;
    }
    CHECK(ok);
  });
  run("config: type errors, unknown kinds and cross-field checks", [] {
    std::vector<std::string> v;
    try {
      parse_config(R"({
        "grid": {"points": [4, "x"]},
        "microstructure": {"kind": "sphere"},
        "model": {"kind": "hyperelastic", "phases": [{"youngs": 1.0, "poisson": 0.3}]},
        "loading": {"mode": "simple_shear", "gamma": 0.1, "increments": 1},
        "output": {"fields": ["F", "epsp", "Q"], "stride": 0}
      })");
    } catch (const ConfigInvalid& e) {
      v = e.violations;
    }
    auto has = [&](const char* s) {
      for (const auto& x : v)
        if (x.find(s) != std::string::npos) return true;
      return false;
    };
    CHECK(has("grid.points: expected array of int") && has("microstructure.kind"));
    CHECK(has("'epsp' requires the simo model") && has("unknown field 'Q'") && has("output.stride"));
  });
}

static void snapshot_round_trip(const std::filesystem::path& golden) {
      namespace fs = std::filesystem;
      const fs::path dir = fs::temp_directory_path() / "fftmech_b200_unit_snapshot_out";
      fs::remove_all(dir);
      Snapshot snap;
      snap.increment = 7;
      snap.label = "7";
      snap.grid = grid_2d(3, 2);
      snap.tensor_dim = 2;
      snap.fbar = Tensor2::identity(2);
      snap.fbar(0, 1) = 0.25;
      SnapshotFieldData f;
      f.components = 4;
      for (int c = 0; c < 4; ++c)
        for (int k = 0; k < 6; ++k) f.values.push_back(0.1 * c + 1e-13 * k + (c == 0 || c == 3));
      snap.fields["F"] = f;
      SnapshotFieldData eq;
      eq.components = 1;
      for (int k = 0; k < 6; ++k) eq.values.push_back(std::sqrt(2.0) * k);
      snap.fields["eq"] = eq;
      write_snapshot(dir, snap);
      const Snapshot back = read_snapshot(dir, 7);
      CHECK(back.label == "7" && back.tensor_dim == 2 && back.grid.points[0] == 3 && back.fbar(0, 1) == 0.25);
      CHECK(back.fields.count("F") == 1 && back.fields.at("F").values == f.values);
      CHECK(back.fields.at("eq").values == eq.values);
      CHECK(list_snapshots(dir) == std::vector<int>{7});
      CHECK(slurp(dir / "meta_7.json") == slurp(golden / "unit_snapshot_out" / "meta_7.json"));
      const Tensor2Field T = snapshot_to_field(back, "F");
      CHECK(T.at(5, 1, 1) == f.values[3 * 6 + 5]);
    }

int main(int argc, char** argv) {
  const char* golden_env = std::getenv("FFTMECH_GOLDEN_RECORDS");
  const std::filesystem::path golden = argc > 1 ? argv[1] : (golden_env ? golden_env : "");
  if (argc > 2 && std::string(argv[2]) == "--no-device") {  // host-only cases (CPU test suite)
    run("output: snapshot round trip, bit-exact (test_config_io.cpp:135-164)", [&] { snapshot_round_trip(golden); });
    config_cases();
    std::printf("%d checks, %d failed\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
  }
  run("projection: constant fields project to zero", [] {
    const GridShape s = grid_3d(5, 5, 5);
    const ProjectionOperator G = build_projection(s, 3);
    Tensor2Field A(s, 3);
    Tensor2 c(3);
    c(0, 1) = 2.0;
    c(2, 2) = -0.7;
    A.add_uniform(c);
    CHECK(field_norm(apply_projection(G, A)) < 1e-12 * field_norm(A));
  });

  run("projection: idempotent, zero-mean, self-adjoint (5 shapes, both Nyquist modes)", [] {
    std::mt19937 rng(1234);
    const std::vector<std::pair<GridShape, NyquistMode>> cases = {
        {grid_3d(5, 5, 5), NyquistMode::ZeroCompatible},
        {grid_3d(5, 3, 7, 1.0, 2.0, 0.5), NyquistMode::ZeroCompatible},
        {grid_3d(4, 4, 4), NyquistMode::ZeroCompatible},
        {grid_3d(4, 4, 4), NyquistMode::IdentityEquilibrium},
        {grid_2d(6, 5), NyquistMode::ZeroCompatible},
    };
    for (const auto& [s, mode] : cases) {
      const int d = s.dim;
      const ProjectionOperator G = build_projection(s, d, mode);
      const Tensor2Field A = random_field(s, d, rng), B = random_field(s, d, rng);
      const Tensor2Field GA = apply_projection(G, A);
      Tensor2Field diff = apply_projection(G, GA);
      diff -= GA;
      CHECK(field_norm(diff) < 1e-10 * std::max(1.0, field_norm(GA)));
      const Tensor2 m = field_mean(GA);
      for (int c = 0; c < d * d; ++c) CHECK(std::abs(m.v[c]) < 1e-12);
      const double lhs = field_dot(A, apply_projection(G, B)), rhs = field_dot(GA, B);
      CHECK(std::abs(lhs - rhs) <= 1e-10 * std::abs(rhs));
    }
  });

  run("projection: ghat closed form and Nyquist handling", [] {
    const GridShape s = grid_3d(3, 3, 3);
    const ProjectionOperator G = build_projection(s, 3);
    const std::size_t node = s.node_index({1, 0, 0});
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        CHECK(G.ghat().at(0, i, j) == 0.0);
        CHECK(std::abs(G.ghat().at(node, i, j) - (i == 0 && j == 0 ? 1.0 : 0.0)) < 1e-15);
      }
    const GridShape e = grid_3d(4, 4, 4);
    const ProjectionOperator Gz = build_projection(e, 3, NyquistMode::ZeroCompatible);
    for (int qy = 0; qy < 4; ++qy)
      for (int qz = 0; qz < 4; ++qz)
        for (int c = 0; c < 9; ++c) CHECK(Gz.ghat().data()[c * 64 + e.node_index({2, qy, qz})] == 0.0);
  });

  run("projection: plane strain keeps the third column free of fluctuation", [] {
    const GridShape s = grid_2d(5, 7);
    const ProjectionOperator G = build_projection(s, 3);
    std::mt19937 rng(9);
    const Tensor2Field GA = apply_projection(G, random_field(s, 3, rng));
    for (std::size_t k = 0; k < GA.nodes(); ++k)
      for (int i = 0; i < 3; ++i) CHECK(std::abs(GA.at(k, i, 2)) < 1e-12);
  });

  run("projected tangent: identity tangent, zero update, composition", [] {
    const GridShape s = grid_2d(3, 3);
    const ProjectionOperator G = build_projection(s, 2);
    std::mt19937 rng(55);
    const Tensor2Field dF = random_field(s, 2, rng);
    Tensor2Field diff = apply_projected_tangent(G, identity4(s, 2), dF);
    const Tensor2Field direct = apply_projection(G, dF);
    diff -= direct;
    CHECK(field_norm(diff) < 1e-12 * std::max(1.0, field_norm(direct)));
    Tensor4Field K(s, 2);
    std::uniform_real_distribution<double> u(-1, 1);
    for (double& v : K.data()) v = u(rng);
    CHECK(field_norm(apply_projected_tangent(G, K, Tensor2Field(s, 2))) == 0.0);
    const GridShape s3 = grid_3d(3, 3, 3);
    const ProjectionOperator G3 = build_projection(s3, 3);
    Tensor4Field K3(s3, 3);
    for (double& v : K3.data()) v = u(rng);
    const Tensor2Field d3 = random_field(s3, 3, rng);
    Tensor2Field composed = apply_projection(G3, trans2(ddot42(K3, trans2(d3))));
    const Tensor2Field fused = apply_projected_tangent(G3, K3, d3);
    composed -= fused;
    CHECK(field_norm(composed) < 1e-12 * std::max(1.0, field_norm(fused)));
  });

  run("hyperelastic: F = I gives P = 0 and K = C; uniaxial closed form", [] {
    const GridShape s = grid_3d(2, 2, 2);
    const ElasticParams p{1.0, 0.3};
    Tensor2Field P;
    Tensor4Field K;
    hyperelastic_evaluate(identity2(s, 3), p, P, K);
    CHECK(field_norm(P) == 0.0);
    const double lam = p.lame_lambda(), mu = p.lame_mu();
    for (std::size_t q = 0; q < 8; ++q)
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
          for (int k = 0; k < 3; ++k)
            for (int l = 0; l < 3; ++l) {
              const double c = lam * (i == j) * (k == l) + mu * ((i == l) * (j == k) + (i == k) * (j == l));
              CHECK(std::abs(K.at(q, i, j, k, l) - c) <= 1e-14 * std::max(1.0, std::abs(c)));
            }
    const GridShape one = grid_3d(1, 1, 1);
    Tensor2Field F = identity2(one, 3);
    F.at(0, 0, 0) = 1.1;
    hyperelastic_evaluate(F, p, P, K);
    const double e11 = 0.5 * (1.1 * 1.1 - 1.0);
    CHECK(std::abs(P.at(0, 0, 0) - 1.1 * (lam + 2 * mu) * e11) < 1e-14);
    CHECK(std::abs(P.at(0, 1, 1) - lam * e11) < 1e-14);
  });

  run("hyperelastic: inverted node reports the first offending node", [] {
    const GridShape s = grid_3d(4, 1, 1);
    Tensor2Field F = identity2(s, 3);
    F.at(3, 0, 0) = -1.0;
    F.at(2, 0, 0) = -1.0;
    Tensor2Field P;
    Tensor4Field K;
    bool thrown = false;
    try {
      hyperelastic_evaluate(F, ElasticParams{}, P, K);
    } catch (const InvertedElement& e) {
      thrown = e.node == 2;
    }
    CHECK(thrown);
  });

  run("simo: virgin state, commit promotes trial, plane strain", [] {
    const PlasticParams pp{{1.0, 0.3}, 0.01, 0.05};
    const GridShape one = grid_3d(1, 1, 1);
    HistoryState committed(one, 3), trial;
    Tensor2Field P;
    Tensor4Field K;
    const Tensor2Field I = identity2(one, 3);
    simo_evaluate(I, I, committed, ScalarField(one, pp.elastic.lame_lambda()), ScalarField(one, pp.elastic.lame_mu()),
                  ScalarField(one, 0.01), ScalarField(one, 0.05), P, K, trial);
    CHECK(field_norm(P) < 1e-14);
    CHECK(trial.eps_p[0] == 0.0);
    const GridShape s = grid_2d(2, 2);
    SimoPlasticityModel model(s, pp);
    CHECK(model.tensor_dim() == 3);
    Tensor2Field F = identity2(s, 3);
    F.at(0, 0, 1) = 0.05;
    model.evaluate(F, P, K);
    CHECK(model.trial().eps_p[0] > 0.0);
    CHECK(model.committed().eps_p[0] == 0.0);
    model.commit(F);
    CHECK(std::abs(model.committed().eps_p[0] - model.trial().eps_p[0]) < 1e-15);
    const GridShape ps = grid_2d(3, 2);
    SimoPlasticityModel m2(ps, pp);
    Tensor2Field F2 = identity2(ps, 3);
    for (std::size_t q = 0; q < F2.nodes(); ++q) F2.at(q, 0, 1) = 0.03;
    m2.evaluate(F2, P, K);
    for (std::size_t q = 0; q < F2.nodes(); ++q) {
      CHECK(std::abs(P.at(q, 2, 0)) < 1e-14 && std::abs(P.at(q, 0, 2)) < 1e-14);
      CHECK(P.at(q, 2, 2) != 0.0);
    }
  });

  run("cg: zero rhs returns immediately; compatible rhs converges", [] {
    const GridShape s = grid_2d(5, 5);
    const ProjectionOperator G = build_projection(s, 2);
    const Tensor4Field C = stiffness(s, 2, 0.58, 0.38);
    const ProjectedTangentOperator op(G, C);
    Tensor2Field x;
    CHECK(cg_solve(op, Tensor2Field(s, 2), SolverParams{}, x).iterations == 0);
    CHECK(field_norm(x) == 0.0);
    std::mt19937 rng(8);
    const Tensor2Field b = apply_projection(G, random_field(s, 2, rng));
    SolverParams prm;
    prm.eta_cg = 1e-12;
    const CgResult r = cg_solve(op, b, prm, x);
    CHECK(r.iterations <= int(b.nodes()) * 4);
    Tensor2Field Ax = op.apply(x);
    Ax -= b;
    CHECK(field_norm(Ax) <= 1e-11 * field_norm(b));
  });

  run("cg: a user LinearOperator runs through the device CG", [] {
    struct Scaled : LinearOperator {
      const ProjectionOperator& G;
      explicit Scaled(const ProjectionOperator& g) : G(g) {}
      Tensor2Field apply(const Tensor2Field& x) const override {
        Tensor2Field y = apply_projection(G, x);
        y *= 2.5;
        return y;
      }
    };
    const GridShape s = grid_3d(4, 5, 3);
    const ProjectionOperator G = build_projection(s, 3);
    std::mt19937 rng(3);
    const Tensor2Field b = apply_projection(G, random_field(s, 3, rng));
    Tensor2Field x;
    const CgResult r = cg_solve(Scaled(G), b, SolverParams{}, x);
    x *= 2.5;
    x -= b;
    CHECK(r.iterations == 1);
    CHECK(field_norm(x) < 1e-10 * field_norm(b));
  });

  run("solver: homogeneous cell converges exactly in one equilibrium pass", [] {
    const GridShape s = grid_3d(4, 3, 5);
    HyperelasticModel model(s, 3, ElasticParams{1.0, 0.3});
    const ProjectionOperator G = build_projection(s, 3);
    Tensor2Field F = identity2(s, 3);
    Tensor2 fbar = Tensor2::identity(3);
    fbar(0, 1) = 0.37;
    fbar(0, 0) = 1.05;
    fbar(2, 0) = -0.11;
    const SolveReport rep = solve_increment(F, model, G, {fbar, "1"}, SolverParams{});
    CHECK(rep.converged && rep.equilibrium_iterations() == 1);
    double worst = 0.0;
    for (std::size_t q = 0; q < F.nodes(); ++q)
      for (int c = 0; c < 9; ++c) worst = std::max(worst, std::abs(F.data()[c * F.nodes() + q] - fbar.v[c]));
    CHECK(worst < 1e-12);
    CHECK(rep.max_mean_drift < 1e-12);
  });

  run("solver: golden laminate run (proj/unit_det_out1/report.csv)", [] {
    const GridShape s = grid_2d(5, 4);
    const PhaseGrid pg = make_laminate(s, {0.4, 0.6});
    const MaterialFields mf = bind_parameters(pg, std::vector<ElasticParams>{{1.0, 0.3}, {5.0, 0.25}});
    HyperelasticModel model(s, 2, mf.lambda, mf.mu);
    const ProjectionOperator G = build_projection(s, 2);
    Tensor2Field F = identity2(s, 2);
    const int newton[3] = {3, 3, 3};
    const long cg[3] = {5, 6, 6};
    const double res[3] = {9.9744016807068452e-08, 2.7431520407441979e-07, 5.4231097371528531e-07};
    for (int t = 1; t <= 3; ++t) {
      Tensor2 fbar = Tensor2::identity(2);
      fbar(0, 1) = 0.15 * t / 3;
      const SolveReport r = solve_increment(F, model, G, {fbar, std::to_string(t)}, SolverParams{});
      CHECK(r.newton_iterations() == newton[t - 1]);
      CHECK(r.total_cg_iterations() == cg[t - 1]);
      CHECK(std::abs(r.passes.back().rel_update - res[t - 1]) < 1e-6 * res[t - 1]);
    }
  });

  run("solver: converged inclusion state is in equilibrium, drift-free", [] {
    const GridShape s = grid_3d(5, 5, 5);
    const PhaseGrid pg = make_cubic_inclusion(s, std::pow(2.0 / 5.0, 3));
    const MaterialFields mf = bind_parameters(pg, std::vector<ElasticParams>{{1.0, 0.3}, {10.0, 0.3}});
    HyperelasticModel model(s, 3, mf.lambda, mf.mu);
    const ProjectionOperator G = build_projection(s, 3);
    Tensor2Field F = identity2(s, 3);
    Tensor2 fbar = Tensor2::identity(3);
    fbar(0, 1) = 0.2;
    const SolveReport rep = solve_increment(F, model, G, {fbar, "1"}, SolverParams{});
    CHECK(rep.converged);
    CHECK(rep.max_mean_drift < 1e-12);
    CHECK(rep.equilibrium_rel_residual < 10.0 * SolverParams{}.eta_newton);
  });

  run("solver: a host-side user MaterialModel matches the device model", [] {
    const GridShape s = grid_3d(6, 5, 4);
    const ProjectionOperator G = build_projection(s, 3);
    HyperelasticModel dev(s, 3, ElasticParams{1.0, 0.3});
    HostSvk host(s, 3, ElasticParams{1.0, 0.3});
    Tensor2 fbar = Tensor2::identity(3);
    fbar(0, 1) = 0.1;
    Tensor2Field F1 = identity2(s, 3), F2 = identity2(s, 3);
    const SolveReport a = solve_increment(F1, dev, G, {fbar, "1"}, SolverParams{});
    const SolveReport b = solve_increment(F2, host, G, {fbar, "1"}, SolverParams{});
    CHECK(a.newton_iterations() == b.newton_iterations());
    F1 -= F2;
    CHECK(field_norm(F1) < 1e-12 * field_norm(F2));
  });

  run("solver: elastic increment then its inverse returns to identity", [] {
    const GridShape s = grid_2d(4, 3);
    const PhaseGrid pg = make_laminate(s, {0.5, 0.5});
    const MaterialFields mf = bind_parameters(pg, std::vector<ElasticParams>{{1.0, 0.3}, {3.0, 0.3}});
    HyperelasticModel model(s, 2, mf.lambda, mf.mu);
    const ProjectionOperator G = build_projection(s, 2);
    SolverParams prm;
    prm.eta_newton = 1e-9;
    Tensor2Field F = identity2(s, 2);
    Tensor2 fbar = Tensor2::identity(2);
    fbar(0, 1) = 0.08;
    solve_increment(F, model, G, {fbar, "fwd"}, prm);
    solve_increment(F, model, G, {Tensor2::identity(2), "back"}, prm);
    Tensor2Field d = F;
    d -= identity2(s, 2);
    CHECK(field_norm(d) / field_norm(F) < 1e-8);
  });

  run("solver: run_program commits per increment (Simo, pure shear)", [] {
    const GridShape s = grid_2d(3, 3);
    SimoPlasticityModel model(s, PlasticParams{{1.0, 0.3}, 0.003, 0.01});
    const ProjectionOperator G = build_projection(s, 3);
    Tensor2Field F = identity2(s, 3);
    struct Counter : ProgramSink {
      int calls = 0;
      void on_increment(std::size_t, const Increment&, const SolveReport&, const Tensor2Field&, const Tensor2Field&,
                        MaterialModel&) override {
        ++calls;
      }
    } sink;
    run_program(F, model, G, {}, SolverParams{}, sink);
    CHECK(sink.calls == 0);
    LoadProgram prog;
    for (int t = 1; t <= 3; ++t) {
      Tensor2 f = Tensor2::identity(3);
      f(0, 0) = 1.0 + 0.02 * t;
      f(1, 1) = 1.0 / f(0, 0);
      prog.push_back({f, std::to_string(t)});
    }
    run_program(F, model, G, prog, SolverParams{}, sink);
    CHECK(sink.calls == 3);
    CHECK((*model.committed_eps_p())[0] > 0.0);
  });

  run("solver: Newton cap raises NewtonDiverged with the report attached", [] {
    const GridShape s = grid_3d(3, 3, 3);
    const PhaseGrid pg = make_cubic_inclusion(s, std::pow(1.5 / 3.0, 3));
    const MaterialFields mf = bind_parameters(pg, std::vector<ElasticParams>{{1.0, 0.3}, {10.0, 0.3}});
    HyperelasticModel model(s, 3, mf.lambda, mf.mu);
    const ProjectionOperator G = build_projection(s, 3);
    Tensor2 fbar = Tensor2::identity(3);
    fbar(0, 1) = 0.5;
    SolverParams prm;
    prm.max_newton = 1;
    Tensor2Field F = identity2(s, 3);
    bool ok = false;
    try {
      solve_increment(F, model, G, {fbar, "1"}, prm);
    } catch (const NewtonDiverged& e) {
      ok = e.report.passes.size() == 1 && !e.report.converged && e.report.label == "1";
    }
    CHECK(ok);
  });

  run("solver: invalid increments are rejected up front", [] {
    const GridShape s = grid_2d(2, 2);
    HyperelasticModel model(s, 2, ElasticParams{});
    const ProjectionOperator G = build_projection(s, 2);
    Tensor2Field F = identity2(s, 2);
    Tensor2 bad = Tensor2::identity(2);
    bad(0, 0) = -1.0;
    bool ok = false;
    try {
      solve_increment(F, model, G, {bad, "x"}, SolverParams{});
    } catch (const std::invalid_argument&) {
      ok = true;
    }
    CHECK(ok);
  });

  if (!golden.empty()) {
    run("output: homogeneous 4x4 run == proj/unit_run_out (meta, report)", [&] {
      check_run_against_record(golden, "unit_run_out", grid_2d(4, 4), {1.0}, {{1.0, 0.3}}, 0.2, 2, OutputOptions{});
    });
    run("output: 3x3 run with VTK == proj/unit_vtk_out (meta, VTK bytes, report)", [&] {
      OutputOptions o;
      o.vtk = true;
      check_run_against_record(golden, "unit_vtk_out", grid_2d(3, 3), {1.0}, {{1.0, 0.3}}, 0.05, 1, o);
    });
    run("output: laminate run == proj/unit_det_out1 (meta, report)", [&] {
      OutputOptions o;
      o.fields = {"F", "P", "eq"};
      check_run_against_record(golden, "unit_det_out1", grid_2d(5, 4), {0.4, 0.6}, {{1.0, 0.3}, {5.0, 0.25}}, 0.15,
                               3, o);
    });
    run("output: snapshot round trip, bit-exact (test_config_io.cpp:135-164)", [&] { snapshot_round_trip(golden); });
    run("output: equivalent stress on the device == host restatement", [] {
      const GridShape s = grid_3d(4, 3, 5);
      std::mt19937 rng(3);
      Tensor2Field F = random_field(s, 3, rng, 0.2);
      F.add_uniform(Tensor2::identity(3));
      const Tensor2Field P = random_field(s, 3, rng);
      const ScalarField eq = HyperelasticModel(s, 3, ElasticParams{}).equivalent_stress_field(F, P);
      const ScalarField eqs = equivalent_stress(dot22(P, trans2(F)));
      const ScalarField tau = SimoPlasticityModel(s, PlasticParams{}).equivalent_stress_field(F, P);
      double worst = 0.0;
      for (std::size_t q = 0; q < s.node_count(); ++q) {
        const Tensor2 S = dot(F.tensor(q).inverse(), P.tensor(q));
        const double m = S.trace() / 3.0;
        double ss = 0.0;
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) ss += (S(i, j) - (i == j ? m : 0.0)) * (S(i, j) - (i == j ? m : 0.0));
        worst = std::max(worst, std::abs(eq[q] - std::sqrt(1.5 * ss)) / std::max(1.0, eq[q]));
        worst = std::max(worst, std::abs(eqs[q] - tau[q]) / std::max(1.0, tau[q]));
      }
      CHECK(worst < 1e-13);
    });
  } else {
    std::printf("[SKIP] output records (pass the golden record directory as argv[1])\n");
  }

  std::printf("%d checks, %d failed\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
