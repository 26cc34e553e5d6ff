// Host check of paper_1201_3018_b200/csrc/pc_intfp.cuh against the host's IEEE binary64
// arithmetic (round to nearest even; C round() for Eq. (2)).  Built and run by
// tests/test_intfp.py.  Exit code 0 = every case bit-identical (or declined: false returned,
// where the kernels take the FP64 instruction).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>

#include "../paper_1201_3018_b200/csrc/pc_intfp.cuh"

using namespace pc::ifp;

static uint64_t bits(double x) {
  uint64_t u;
  std::memcpy(&u, &x, 8);
  return u;
}

static long fails = 0, declined = 0, checked = 0;
static void fail(const char* what, double a, double b, uint64_t got, uint64_t want) {
  if (fails++ < 20)
    std::printf("FAIL %s a=%.17g b=%.17g got=%016llx want=%016llx\n", what, a, b, (unsigned long long)got,
                (unsigned long long)want);
}

static void check_mul(double a, double b) {
  uint64_t r;
  ++checked;
  if (!dmul_rn_pos(bits(a), bits(b), r)) {
    const double p = a * b;
    if (a > 0 && b > 0 && std::isnormal(a) && std::isnormal(b) && std::isnormal(p)) fail("mul declined", a, b, 0, bits(p));
    ++declined;
    return;
  }
  if (r != bits(a * b)) fail("mul", a, b, r, bits(a * b));
}
static void check_div(double a, double b) {
  uint64_t r;
  ++checked;
  if (!ddiv_rn_pos(bits(a), bits(b), r)) {
    const double q = a / b;
    if (a > 0 && b > 0 && std::isnormal(a) && std::isnormal(b) && std::isnormal(q)) fail("div declined", a, b, 0, bits(q));
    ++declined;
    return;
  }
  if (r != bits(a / b)) fail("div", a, b, r, bits(a / b));
}
static void check_compand(double c, double x) {
  long long n;
  bool neg0;
  ++checked;
  const double want = std::round(c * x);
  if (!compand_int(bits(c), bits(x), n, neg0)) {
    if (std::isnormal(c * x) && std::fabs(c * x) < 1e15 && (x == 0 || std::isnormal(x))) fail("compand declined", c, x, 0, bits(want));
    ++declined;
    return;
  }
  const uint64_t got = i2d_scaled(n, 0, neg0);
  if (got != bits(want)) fail("compand", c, x, got, bits(want));
}
// Horner of Eq. (7) (M digits, eps = 2^-b, oracle order) vs the integer word
static void check_pack(const double* d, int M, int b) {
  const double eps = std::ldexp(1.0, -b);
  double a = d[M - 1];
  for (int q = M - 2; q >= 0; --q) a = d[q] + eps * a;
  long long N = 0;
  bool all_neg0 = true;
  for (int q = 0; q < M; ++q) {
    N = N * (1ll << b) + (long long)d[q];
    all_neg0 = all_neg0 && d[q] == 0 && std::signbit(d[q]);
  }
  ++checked;
  const uint64_t got = i2d_scaled(N, (M - 1) * b, all_neg0);
  if (got != bits(a)) fail("pack", d[0], d[1], got, bits(a));
}

int main() {
  std::mt19937_64 rng(12345);
  std::uniform_real_distribution<double> u01(0.0, 1.0);
  auto any_double = [&]() {   // random sign, exponent in [-60, 60], random significand
    const double m = 1.0 + u01(rng);
    const int e = (int)(rng() % 121) - 60;
    return std::ldexp(m, e) * ((rng() & 1) ? -1.0 : 1.0);
  };
  // products and quotients of positive normals, random and with short significands (exact ties)
  for (int i = 0; i < 2000000; ++i) {
    const double a = std::fabs(any_double()), b = std::fabs(any_double());
    check_mul(a, b);
    check_div(a, b);
    const double as = std::ldexp((double)(rng() % 100000 + 1), (int)(rng() % 40) - 20);
    const double bs = std::ldexp((double)(rng() % 100000 + 1), (int)(rng() % 40) - 20);
    check_mul(as, bs);
    check_div(as, bs);
    check_div(as, b);
  }
  // exponent extremes: overflow / underflow must decline, not return a wrong normal
  for (int i = 0; i < 200000; ++i) {
    const double a = std::ldexp(1.0 + u01(rng), (int)(rng() % 2046) - 1022);
    const double b = std::ldexp(1.0 + u01(rng), (int)(rng() % 2046) - 1022);
    check_mul(a, b);
    check_div(a, b);
  }
  // divisors whose significand is near 2^52 (the reciprocal seed's edge) or all ones
  for (long long k = 1; k < 4096; ++k) {
    const double lo = 1.0 + std::ldexp((double)k, -52), mid = 1.0 + std::ldexp((double)((1ll << 29) - 2048 + k), -52);
    const double top = 2.0 - std::ldexp((double)k, -52);
    for (double a : {511.0, 1.0, 3.0, 1.9999999999999998, 1.0000000000000002, 1234.5678}) {
      check_div(a, lo);
      check_div(a, mid);
      check_div(a, top);
      check_div(a, 0.5 * lo);
      check_div(a * 1.25, top);
    }
  }
  check_div(511.0, 0.999999999999);
  check_div(1.0, 3.0);
  check_mul(1.0 + std::ldexp(1.0, -52), 1.0 + std::ldexp(1.0, -52));
  // Eq. (2): c = Q / peak, x in [-peak, peak] (the kernel's operand range), and products landing
  // on / next to half-integers
  for (int i = 0; i < 3000000; ++i) {
    const double Q = (double)((rng() % 2047) + 1);
    const double peak = std::ldexp(1.0 + u01(rng), -(int)(rng() % 12));
    const double c = Q / peak;
    const double x = (2.0 * u01(rng) - 1.0) * peak;
    check_compand(c, x);
    // a sample whose product is (nearly) k + 1/2
    const double k = std::floor(u01(rng) * Q) + 0.5;
    const double xt = k / c;
    check_compand(c, xt);
    check_compand(c, -xt);
    check_compand(c, std::nextafter(xt, 0.0));
    check_compand(c, std::nextafter(xt, 2.0 * xt));
  }
  check_compand(3.0, -0.0);
  check_compand(3.0, 0.0);
  check_compand(3.0, -0.1);
  check_compand(0.5, 1.0);
  check_compand(0.5, -1.0);
  check_compand(1.5, 1.0);
  check_compand(2.5, 1.0);
  check_compand(1e300, 1e-310);   // subnormal operand: declined
  // packing: random balanced digits, incl. negative zeros, M = 2 and 3
  for (int i = 0; i < 1000000; ++i) {
    const int M = 2 + (int)(rng() % 2);
    const int b = 12 + (int)(rng() % (M == 2 ? 9 : 5));   // packed words exact: |N| < 2^53 (ModeP::exact_pack)
    const int Q = 1 << (b - 2);
    double d[3];
    for (int q = 0; q < M; ++q) {
      const long long v = (long long)(rng() % (2 * Q + 1)) - Q;
      d[q] = (double)v;
      if (v == 0 && (rng() & 1)) d[q] = -0.0;
    }
    if ((rng() % 50) == 0)
      for (int q = 0; q < M; ++q) d[q] = -0.0;
    check_pack(d, M, b);
  }
  std::printf("checked %ld declined %ld fails %ld\n", checked, declined, fails);
  return fails ? 1 : 0;
}
