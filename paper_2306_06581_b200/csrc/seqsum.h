// seqsum.h -- the reference's sequential fp64 sum of N equal terms, exactly,
// in O(binades) steps.
//
// masked_grid_plan (proj/src/sparsify.cpp:53-63) sums the grid row-major one
// entry at a time. With uniform marginals every supported entry holds the
// same term t = ra_i * cb_j, so the sum is fl(...fl(fl(t + t) + t)...) over
// N = #support terms (the zeros add nothing). At config 4 (N = 10^12,
// t = 1e-12) that sum is 1.6e-5 relative BELOW the exact one (each add drops
// the same fraction of an ulp), so a tree sum -- or any other order -- gives a
// different 1/total, hence different p* and different sampled index sets.
//
// Emulation: inside a binade [2^E, 2^(E+1)) the running total is T * u
// (u = 2^(E-52), T an integer), and fl(T u + t) = (T + q + c) u with
// t / u = q + f, c = [f > 1/2] (f = 1/2: round half to even on T + q). So the
// increment is constant (after at most two steps when f = 1/2) until the
// total leaves the binade: jump there in one integer step, step across the
// binade edge with real fp adds, repeat. Exact: every jump reproduces the
// same sequence of roundings the sequential loop performs.
#pragma once

#include <cmath>
#include <cstdint>

namespace spk {

inline double seq_sum_const(double t, uint64_t N) {
  if (N == 0 || t == 0.0) return 0.0;
  double total = 0.0;
  while (N > 0) {
    if (!(total > 0.0) || total < 4.0 * t) {  // early terms: plain fp adds
      total += t;
      --N;
      continue;
    }
    int E;
    (void)std::frexp(total, &E);  // total in [2^(E-1), 2^E)
    const double u = std::ldexp(1.0, E - 53);
    // two real steps give the steady increment (absorbs the tie parity case)
    const double a1 = total + t;
    if (--N == 0) return a1;
    const double a2 = a1 + t;
    if (--N == 0) return a2;
    const double d1 = a1 - total, d2 = a2 - a1;  // exact (Sterbenz: same binade or its upper edge)
    total = a2;
    if (d1 != d2 || d2 <= 0.0) continue;  // still settling, or crossed into the next binade
    int E2;
    (void)std::frexp(total, &E2);
    if (E2 != E) continue;
    // jump: k more adds of d2 keep the total strictly inside the binade with
    // room for one more increment (so every skipped add rounds identically)
    const double top = std::ldexp(1.0, E);
    const uint64_t T = static_cast<uint64_t>(total / u), D = static_cast<uint64_t>(d2 / u),
                   TOP = static_cast<uint64_t>(top / u);
    if (T + 2 * D >= TOP) continue;
    uint64_t k = (TOP - T - 1) / D - 1;  // T + (k + 1) D < TOP
    if (k > N) k = N;
    total = static_cast<double>(T + k * D) * u;  // exact: T + k D < 2^53
    N -= k;
  }
  return total;
}

}  // namespace spk
