// Synthetic input streams of the benchmark configurations:
// std::mt19937_64 words mapped to u = (x >> 11) * 2^-53, computed explicitly
// (never through a std distribution, whose output is implementation-defined;
// reference oracles.cpp:313-319).  Config 4 fills 9 component slabs with
// 2u - 1 in node order.  C linkage so the Python layer can fill multi-GB
// inputs at native speed.
#include <cstdint>
#include <random>

extern "C" {

void fmh_mt19937_uniform(uint64_t seed, int64_t count, double* out) {
  std::mt19937_64 gen(seed);
  const double scale = 1.0 / 9007199254740992.0;  // 2^-53
  for (int64_t i = 0; i < count; ++i) out[i] = double(gen() >> 11) * scale;
}

void fmh_uniform_field(uint64_t seed, int64_t count, double* out) {
  std::mt19937_64 gen(seed);
  const double scale = 1.0 / 9007199254740992.0;
  for (int64_t i = 0; i < count; ++i) out[i] = 2.0 * (double(gen() >> 11) * scale) - 1.0;
}

}  // extern "C"
