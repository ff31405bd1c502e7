// Host side of csrc/glibc_exp.cuh against this host's std::exp (glibc), bit for bit.
// Built with -ffp-contract=off by tests/test_exp_glibc_cpu.py. Prints "n bad" and the first misses.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>

#include "glibc_exp.cuh"

int main(int argc, char** argv) {
  const long scale = argc > 1 ? std::atol(argv[1]) : 1;
  std::mt19937_64 g(20250919);
  long n = 0, bad = 0;
  auto check = [&](double x) {
    const double a = std::exp(x), b = cmoe::exp_glibc(x);
    ++n;
    if (cmoe::expd::asu(a) != cmoe::expd::asu(b) && !(std::isnan(a) && std::isnan(b))) {
      if (bad < 5) std::printf("miss x=%a std::exp=%a port=%a\n", x, a, b);
      ++bad;
    }
  };
  // softmax inputs: float logit - float row max, in double
  std::uniform_real_distribution<float> lf(-30.f, 30.f);
  for (long i = 0; i < 4000000 * scale; ++i) {
    const float a = lf(g), b = lf(g);
    check((double)a - (double)(a > b ? a : b));
  }
  std::uniform_real_distribution<double> mid(-60.0, 0.0), wide(-800.0, 800.0), sub(-746.0, -700.0),
      over(500.0, 710.0), tiny(-1e-15, 1e-15);
  for (long i = 0; i < 2000000 * scale; ++i) check(mid(g));
  for (long i = 0; i < 500000 * scale; ++i) check(wide(g));
  for (long i = 0; i < 500000 * scale; ++i) check(sub(g));
  for (long i = 0; i < 500000 * scale; ++i) check(over(g));
  for (long i = 0; i < 100000 * scale; ++i) check(tiny(g));
  const double special[] = {0.0, -0.0, 1.0, -1.0, 709.782712893384, 709.79, -745.1332191019411, -745.14, -708.4,
                            -708.39641853226408, 1e-300, -1e-300, INFINITY, -INFINITY, NAN, 0x1p-54, -0x1p-54,
                            0x1p-55, 512.0, -512.0, 1024.0, -1024.0};
  for (double x : special) check(x);
  std::printf("%ld %ld\n", n, bad);
  return bad != 0;
}
