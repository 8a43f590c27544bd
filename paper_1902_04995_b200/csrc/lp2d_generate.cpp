// lp2d_generate.cpp — host instance synthesis (include/lp2d_b200_gen.h).
//
// A restatement of the reference's generators (generate.hpp:60-91,174-189)
// and RNG streams (rng.hpp:13-68), written against the packed SoA layout and
// parallelised over LPs with std::thread. Compiled with -ffp-contract=off so
// b = a.interior + slack rounds exactly as the reference's x86-64 code; libm
// cos/sin are the same library the reference calls.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

#include "../../include/lp2d_b200_gen.h"

namespace {

uint64_t splitmix64(uint64_t& state) {
  uint64_t z = (state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

// rng.hpp:20-60
struct Rng {
  uint64_t s[4];
  explicit Rng(uint64_t seed) {
    uint64_t sm = seed;
    for (auto& w : s) w = splitmix64(sm);
  }
  uint64_t next() {
    const uint64_t result = rotl(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return result;
  }
  double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double in_range(double lo, double hi) { return lo + (hi - lo) * unit(); }
  uint64_t below(uint64_t n) {
    unsigned __int128 m = static_cast<unsigned __int128>(next()) * n;
    auto lo = static_cast<uint64_t>(m);
    if (lo < n) {
      const uint64_t threshold = -n % n;
      while (lo < threshold) {
        m = static_cast<unsigned __int128>(next()) * n;
        lo = static_cast<uint64_t>(m);
      }
    }
    return static_cast<uint64_t>(m >> 64);
  }
};

constexpr double kTwoPi = 2.0 * 3.141592653589793238462643383279502884;
constexpr double kDefaultBound = 1e7;  // serial.hpp:26

// generate.hpp:60-79 (kind feasible) and the builder's unbounded variant.
void gen_feasible(int64_t m, Rng& r, double margin, bool toward_minus_c, double* ax,
                  double* ay, double* b, double* c) {
  const double phi = kTwoPi * r.unit();
  c[0] = std::cos(phi);
  c[1] = std::sin(phi);
  const double half = kDefaultBound / 2.0;
  const double ix = r.in_range(-half, half);
  const double iy = r.in_range(-half, half);
  for (int64_t k = 0; k < m; ++k) {
    double theta = kTwoPi * r.unit();
    if (toward_minus_c) {
      // builder-defined: theta in (phi + pi) +- pi/3
      theta = phi + 3.141592653589793 + (theta / kTwoPi * 2.0 - 1.0) * (3.141592653589793 / 3.0);
    }
    const double a0 = std::cos(theta), a1 = std::sin(theta);
    const double slack = margin * (1.0 + 9.0 * r.unit());
    ax[k] = a0;
    ay[k] = a1;
    b[k] = (a0 * ix + a1 * iy) + slack;
  }
}

void gen_one(int64_t m, uint64_t seed, int kind, double margin, double* ax, double* ay,
             double* b, double* c) {
  Rng r(seed);
  if (kind == LP2D_GEN_INFEASIBLE && m >= 1) {
    // generate.hpp:81-91
    gen_feasible(m - 1, r, margin, false, ax, ay, b, c);
    const double theta = kTwoPi * r.unit();
    const double a0 = std::cos(theta), a1 = std::sin(theta);
    const double box_min = -(std::fabs(a0) + std::fabs(a1)) * kDefaultBound;
    ax[m - 1] = a0;
    ay[m - 1] = a1;
    b[m - 1] = box_min - 1.0;
    return;
  }
  gen_feasible(m, r, margin, kind == LP2D_GEN_UNBOUNDED, ax, ay, b, c);
}

}  // namespace

extern "C" {

uint64_t lp2dgen_derive_seed(uint64_t base, uint64_t stream) {
  uint64_t st = base ^ (0x9e3779b97f4a7c15ull * (stream + 1));
  splitmix64(st);
  return splitmix64(st);
}

void lp2dgen_shuffle(int64_t m, uint64_t seed, uint32_t* order) {
  for (int64_t i = 0; i < m; ++i) order[i] = static_cast<uint32_t>(i);
  Rng r(seed);
  for (int64_t i = m; i > 1; --i) {
    const uint64_t j = r.below(static_cast<uint64_t>(i));
    std::swap(order[i - 1], order[j]);
  }
}

int lp2dgen_gen(int64_t m, uint64_t seed, int kind, double margin, double* ax,
                double* ay, double* b, double* c, double* bound_m) {
  if (m < 0 || (kind == LP2D_GEN_INFEASIBLE && m < 1)) return -1;
  gen_one(m, seed, kind, margin, ax, ay, b, c);
  *bound_m = kDefaultBound;
  return 0;
}

int lp2dgen_fill(int64_t n, int64_t first, uint64_t seed, const int32_t* m,
                 const int64_t* offset, const uint8_t* kind, double margin,
                 double bscale, double* ax, double* ay, double* b, uint32_t* perm,
                 double* c, double* bound_m, int threads) {
  if (n < 0 || !m || !offset || !ax || !ay || !b || !c || !bound_m) return -1;
  for (int64_t j = 0; j < n; ++j) {
    if (m[j] < 0) return -2;
    if (kind && kind[j] == LP2D_GEN_INFEASIBLE && m[j] < 1) return -3;
  }
  unsigned hw = std::thread::hardware_concurrency();
  int nt = threads > 0 ? threads : static_cast<int>(hw ? hw : 1);
  nt = static_cast<int>(std::min<int64_t>(nt, std::max<int64_t>(1, n / 64)));
  std::atomic<int64_t> next{0};
  auto work = [&] {
    for (int64_t j0 = next.fetch_add(64); j0 < n; j0 = next.fetch_add(64)) {
      const int64_t j1 = std::min(n, j0 + 64);
      for (int64_t j = j0; j < j1; ++j) {
        const uint64_t g = static_cast<uint64_t>(first + j);
        const int64_t o = offset[j];
        const int k = kind ? static_cast<int>(kind[j]) : static_cast<int>(LP2D_GEN_FEASIBLE);
        gen_one(m[j], lp2dgen_derive_seed(seed, 2 * g), k, margin, ax + o, ay + o, b + o,
                c + 2 * j);
        bound_m[j] = kDefaultBound;
        if (bscale != 1.0) {
          for (int64_t q = 0; q < m[j]; ++q) b[o + q] *= bscale;
          bound_m[j] *= bscale;
        }
        if (perm) lp2dgen_shuffle(m[j], lp2dgen_derive_seed(seed, 2 * g + 1), perm + o);
      }
    }
  };
  if (nt <= 1) {
    work();
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t) pool.emplace_back(work);
    for (auto& t : pool) t.join();
  }
  return 0;
}

void lp2dgen_uniform(uint64_t seed, uint64_t stream, double lo, double hi, int64_t n,
                     double* out) {
  Rng r(lp2dgen_derive_seed(seed, stream));
  for (int64_t i = 0; i < n; ++i) out[i] = r.in_range(lo, hi);
}

int64_t lp2dgen_pareto_sizes(uint64_t seed, double xmin, double alpha, int32_t xmax,
                             int64_t target_total, int64_t n_max, int32_t* m) {
  Rng r(lp2dgen_derive_seed(seed, 0xB0));
  int64_t total = 0, n = 0;
  while (n < n_max && total < target_total) {
    const double u = r.unit();
    double v = u > 0.0 ? std::floor(xmin / std::pow(u, 1.0 / alpha)) : (double)xmax;
    v = std::min<double>(v, xmax);
    v = std::max<double>(v, xmin);
    m[n] = static_cast<int32_t>(v);
    total += m[n];
    ++n;
  }
  return n;
}

}  // extern "C"
