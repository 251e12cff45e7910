// seq_sum_const (csrc/seqsum.h) against the plain sequential loop it emulates
// (masked_grid_plan's row-major sum, sparsify.cpp:53-63) and against the
// committed 10^12-term config-4 sum (tests/golden/c4_normaliser.json).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>

#include "seqsum.h"

int main(int argc, char** argv) {
  std::mt19937_64 g(7);
  int bad = 0;
  for (int it = 0; it < 4000; ++it) {
    double t = std::ldexp(1.0 + static_cast<double>(g() % 1000000) / 1e6, -static_cast<int>(g() % 45));
    if (it % 3 == 0) t = 1.0 / static_cast<double>(1 + g() % 1000);
    if (it % 7 == 0) t = std::ldexp(1.5, -20);  // exact ties on the way up
    const uint64_t N = 1 + g() % (it < 3000 ? 20000 : 2000000);
    double s = 0.0;
    for (uint64_t k = 0; k < N; ++k) s += t;
    if (s != spk::seq_sum_const(t, N)) ++bad;
  }
  std::printf("random cases: %d mismatches\n", bad);
  if (argc > 2) {  // the config-4 term and support count -> total
    const double t = std::strtod(argv[1], nullptr);
    const unsigned long long N = std::strtoull(argv[2], nullptr, 10);
    std::printf("%a\n", spk::seq_sum_const(t, N));
  }
  return bad;
}
