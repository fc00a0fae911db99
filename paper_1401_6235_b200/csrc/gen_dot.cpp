// gen_dot.cpp — host-side generator of ill-conditioned dot products (workload
// tool for the config-4 benchmark and the reduction tests).
//
// Restates the published GenDot method of Ogita, Rump & Oishi, "Accurate sum and
// dot product", SIAM J. Sci. Comput. 26(6), 2005, Algorithm 6.1 (the reference
// repository has no generator):
//   b = log2(cond); the first half of the pairs gets random exponents in
//   [0, b/2] (the first forced to b/2+1, the last to 0); the second half gets
//   exponents falling linearly from b/2 to 0 and y_i chosen so that x_i*y_i
//   cancels the running dot of everything before it.
// The running dot is carried in double-double (TwoProd + TwoSum), accurate to
// ~u^2 * sum|x_i y_i| — far below what the cancellation needs.  No final
// permutation is applied.  Compiled with -ffp-contract=off.
//
// One calibration beyond the published method: the LAST pair's target (the
// value the whole dot ends on) is +-2 * sum|x_i y_i| / cond instead of a random
// number of unit scale.  With unit-scale final targets the achieved condition
// number 2 sum|x_i y_i| / |sum x_i y_i| grows with n (sum|x_i y_i| ~ n 2^b /
// log2 cond): 2.5e24 at n = 2^30 for a 1e16 target.  Calibrated, it is the
// requested cond at every n (up to ~1/u^2, the double-double limit).
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

#include "../../include/twofold_b200.h"

namespace {

inline uint64_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
inline double u01(uint64_t key, uint64_t i) { return (double)(mix(key ^ i) >> 11) * 0x1p-53; }

struct DD {
  double s = 0, c = 0;
  double abs_sum = 0;  // sum |x_i y_i| (plain double; only scales the final target)
  void add(double p) {
    double t = s + p;
    double bv = t - s;
    double av = t - bv;
    double e = (s - av) + (p - bv);
    s = t;
    c += e;
  }
  void add_prod(double x, double y) {
    double p = x * y;
    double e = std::fma(x, y, -p);
    add(p);
    c += e;
    abs_sum += std::fabs(p);
  }
};

}  // namespace

extern "C" int tf_gen_dot_host(int64_t n, double cond, uint64_t seed, double* x, double* y) {
  if (n < 2 || !(cond > 1.0) || !x || !y) return TF_EINVAL;
  const double b = std::log2(cond);
  const int64_t n2 = n / 2;
  const uint64_t key = mix(seed);
  const double half = b / 2.0;
  // first half: independent, parallel over threads
  unsigned nth = std::thread::hardware_concurrency();
  if (nth < 1) nth = 1;
  if (nth > 64) nth = 64;
  std::vector<DD> part(nth);
  std::vector<std::thread> th;
  for (unsigned t = 0; t < nth; t++) {
    th.emplace_back([&, t]() {
      const int64_t lo = n2 * t / nth, hi = n2 * (t + 1) / nth;
      DD acc;
      for (int64_t i = lo; i < hi; i++) {
        double e = std::round(u01(key, 4 * (uint64_t)i) * half);
        if (i == 0) e = std::round(half) + 1;
        if (i == n2 - 1) e = 0;
        x[i] = (2 * u01(key, 4 * (uint64_t)i + 1) - 1) * std::ldexp(1.0, (int)e);
        y[i] = (2 * u01(key, 4 * (uint64_t)i + 2) - 1) * std::ldexp(1.0, (int)e);
        acc.add_prod(x[i], y[i]);
      }
      part[t] = acc;
    });
  }
  for (auto& t : th) t.join();
  DD run;
  for (auto& p : part) {
    run.add(p.s);
    run.c += p.c;
    run.abs_sum += p.abs_sum;
  }
  // second half: sequential cancellation
  const int64_t m = n - n2;
  for (int64_t j = 0; j < m; j++) {
    const int64_t i = n2 + j;
    const double frac = m > 1 ? (double)j / (double)(m - 1) : 1.0;
    const double e = std::round(half * (1.0 - frac));
    const double sc = std::ldexp(1.0, (int)e);
    double xi = (2 * u01(key, 4 * (uint64_t)i + 1) - 1) * sc;
    if (xi == 0) xi = sc;
    double target = (2 * u01(key, 4 * (uint64_t)i + 2) - 1) * sc;
    if (j == m - 1)  // the dot ends on this value: calibrated to the requested cond
      target = (target < 0 ? -2.0 : 2.0) * run.abs_sum / cond;
    const double cur = run.s + run.c;
    x[i] = xi;
    y[i] = (target - cur) / xi;
    run.add_prod(x[i], y[i]);
  }
  return TF_OK;
}
