// TEST INFRASTRUCTURE — csrc/fmt.cuh compiled as host code against std::to_chars
// / std::to_string (what the reference's report.cpp:42-47 calls): prints the
// number of mismatches over random bit patterns, decimal-looking values,
// integers, powers of ten and their neighbours, subnormals and edge values.
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>

#include "fmt.cuh"

static uint64_t s = 0x243F6A8885A308D3ull;
static uint64_t rnd() {
  uint64_t z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static long bad = 0, total = 0;
static void check(double x) {
  char a[64], b[64];
  auto r = std::to_chars(a, a + 64, x);
  const int na = (int)(r.ptr - a);
  const int nb = xsp::fmt_double(b, x);
  const int nc = xsp::fmt_double(nullptr, x);
  ++total;
  if (na != nb || nb != nc || memcmp(a, b, na) != 0) {
    if (bad < 10) printf("MISMATCH %.17g: std '%.*s' ours '%.*s' (count %d)\n", x, na, a, nb, b, nc);
    ++bad;
  }
}
static void check_i(uint64_t u) {
  char b[32];
  const std::string a = std::to_string(u);
  const int n = xsp::fmt_u64(b, u);
  ++total;
  if (a != std::string(b, n)) ++bad;
  const int64_t v = (int64_t)u;
  const std::string c = std::to_string(v);
  const int m = xsp::fmt_i64(b, v);
  ++total;
  if (c != std::string(b, m)) ++bad;
}

int main(int argc, char** argv) {
  const long n = argc > 1 ? atol(argv[1]) : 2000000;
  for (long i = 0; i < n; ++i) {
    uint64_t b = rnd();
    double d;
    memcpy(&d, &b, 8);
    if (std::isfinite(d)) check(d);
    check((double)(rnd() % 1000000000000ull) / std::pow(10.0, (int)(rnd() % 20)));
    check((double)(int64_t)(rnd() >> (rnd() % 64)));
    check(std::ldexp((double)(rnd() >> 11), (int)(rnd() % 2200) - 1100));
    check_i(rnd() >> (rnd() % 64));
  }
  for (int e = -330; e <= 310; ++e) {
    const double p = std::pow(10.0, e);
    check(p);
    check(std::nextafter(p, 0.0));
    check(std::nextafter(p, 1e308));
    check(-p);
  }
  const double edge[] = {0.0, -0.0, 1.0, 0.5, 0.1, 0.2, 0.3, 1e21, 1e22, 1e23, 123456789012345678.0,
                         std::numeric_limits<double>::max(), std::numeric_limits<double>::min(),
                         std::numeric_limits<double>::denorm_min(), 5e-324, 9007199254740993.0,
                         std::numeric_limits<double>::infinity(), -std::numeric_limits<double>::infinity()};
  for (double e : edge) check(e);
  printf("%ld of %ld mismatched\n", bad, total);
  return bad ? 1 : 0;
}
