// Host check of csrc/fexp.cuh against the C library exp (glibc), which is
// what CPython's math.exp — and so the reference — uses.
// usage: fexp_test N lo hi seed [tablesize 64|1024] -> prints "n equal max_ulp"
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>

#include "../paper_2003_04617_b200/csrc/fexp.cuh"

static const rl::Exp2Tab TAB[64] = RL_EXP2_TABLE_INIT;
static const rl::ExpConsts KC = RL_EXP_CONSTS_INIT;
static const rl::Exp2Tab TAB1024[1024] = RL_EXP2_TABLE_INIT_1024;
static const rl::ExpConsts1024 KC1024 = RL_EXP_CONSTS_1024_INIT;
static const rl::Exp2Tab TAB256[256] = RL_EXP2_TABLE_INIT_256;
static const rl::ExpConsts256 KC256 = RL_EXP_CONSTS_256_INIT;

int main(int argc, char **argv) {
  long n = atol(argv[1]);
  double lo = atof(argv[2]), hi = atof(argv[3]);
  std::mt19937_64 g(atol(argv[4]));
  const int ts = argc > 5 ? atoi(argv[5]) : 64;
  std::uniform_real_distribution<double> U(lo, hi);  // |x| < 708
  long eq = 0;
  double maxulp = 0;
  for (long i = 0; i < n; i++) {
    double x = U(g);
    double a = ts == 1024 ? rl::fexp1024_core(x, TAB1024, KC1024)
               : ts == 256 ? rl::fexp256_core(x, TAB256, KC256) : rl::fexp_core(x, TAB, KC);
    double b = exp(x);
    if (memcmp(&a, &b, 8) == 0) {
      eq++;
    } else {
      double u = fabs(a - b) / (nextafter(b, INFINITY) - b);
      if (u > maxulp) maxulp = u;
    }
  }
  printf("%ld %ld %.3f\n", n, eq, maxulp);
  return 0;
}
