#include <cstdio>
#include "fftmech/hyperelastic.hpp"
#include "fftmech/solver.hpp"
#include "fftmech/tensor_ops.hpp"
using namespace fftmech;
int main() {
  const GridShape s = grid_3d(6, 5, 4);
  const ProjectionOperator G = build_projection(s, 3);
  HyperelasticModel dev(s, 3, ElasticParams{1.0, 0.3});
  Tensor2 fbar = Tensor2::identity(3);
  fbar(0, 1) = 0.1;
  Tensor2Field F1 = identity2(s, 3);
  try {
    Tensor2Field P; Tensor4Field K;
    dev.evaluate(F1, P, K);
    std::printf("evaluate ok %g\n", field_norm(P));
    const SolveReport a = solve_increment(F1, dev, G, {fbar, "1"}, SolverParams{});
    std::printf("device solve ok passes=%d\n", a.newton_iterations());
  } catch (const std::exception& e) { std::printf("device path: %s\n", e.what()); }
  return 0;
}
