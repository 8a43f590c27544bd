// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// C-callable wrapper around the UNMODIFIED reference headers
// (/root/reference/proj/include/lp2d/*.hpp), compiled by oracle/Makefile into
// oracle/_ref/liblp2d_ref.so. It is the ground truth the restated oracle is
// pinned against, and the CPU baseline timed by bench.py (--impl reference and
// the cpu_baseline leg). Nothing in the product links it.
//
// Packed layout (same as the product C-ABI): LP j owns elements
// [offset[j], offset[j] + m[j]) of ax/ay/b/perm (perm widened to u32).

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <stdexcept>
#include <vector>

#include "lp2d/bench.hpp"
#include "lp2d/lp2d.hpp"

namespace {

lp2d::tolerance make_tol(double eps_par, double eps_feas) {
  lp2d::tolerance t;
  t.eps_parallel = eps_par;
  t.eps_feas = eps_feas;
  return t;
}

void fill_solution(const lp2d::solution& s, uint8_t* feasible, double* x,
                   double* y, double* v) {
  *feasible = s.feasible ? 1 : 0;
  *x = s.point.x;
  *y = s.point.y;
  *v = s.value;
}

}  // namespace

extern "C" {

uint64_t ref_derive_seed(uint64_t base, uint64_t stream) {
  return lp2d::derive_seed(base, stream);
}

void ref_xoshiro_first(uint64_t seed, int n, uint64_t* out) {
  lp2d::xoshiro256pp r(seed);
  for (int i = 0; i < n; ++i) out[i] = r.next();
}

void ref_shuffle(int64_t m, uint64_t seed, uint32_t* order) {
  const lp2d::permutation p = lp2d::shuffle(static_cast<std::size_t>(m), seed);
  std::memcpy(order, p.order.data(), sizeof(uint32_t) * p.order.size());
}

// gen({m, seed, kind, margin}); kind 0 feasible_random, 1 infeasible,
// 2 adversarial_ordered. Returns 0, or -1 on a thrown exception.
int ref_gen(int64_t m, uint64_t seed, int kind, double margin, double* ax,
            double* ay, double* b, double* c, double* bound_m) {
  try {
    lp2d::gen_spec spec{static_cast<std::size_t>(m), seed,
                        static_cast<lp2d::gen_kind>(kind), margin};
    const lp2d::problem p = lp2d::gen(spec);
    for (std::size_t k = 0; k < p.constraints.size(); ++k) {
      ax[k] = p.constraints[k].a.x;
      ay[k] = p.constraints[k].a.y;
      b[k] = p.constraints[k].b;
    }
    c[0] = p.obj.c.x;
    c[1] = p.obj.c.y;
    *bound_m = p.bound_m;
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// gen_mixed(sizes, count, seed, kind, margin) into the packed layout; the
// caller sized offset/m from sizes[i % nsizes].
int ref_gen_mixed(const int64_t* sizes, int64_t nsizes, int64_t count,
                  uint64_t seed, int kind, double margin,
                  const int64_t* offset, double* ax, double* ay, double* b,
                  uint32_t* perm, double* c, double* bound_m) {
  try {
    std::vector<std::size_t> sz(sizes, sizes + nsizes);
    const lp2d::batch bt = lp2d::gen_mixed(sz, static_cast<std::size_t>(count),
                                           seed,
                                           static_cast<lp2d::gen_kind>(kind),
                                           margin);
    for (int64_t j = 0; j < count; ++j) {
      const lp2d::problem& p = bt.problems[j];
      const int64_t o = offset[j];
      for (std::size_t k = 0; k < p.constraints.size(); ++k) {
        ax[o + k] = p.constraints[k].a.x;
        ay[o + k] = p.constraints[k].a.y;
        b[o + k] = p.constraints[k].b;
        perm[o + k] = bt.permutations[j].order[k];
      }
      c[2 * j] = p.obj.c.x;
      c[2 * j + 1] = p.obj.c.y;
      bound_m[j] = p.bound_m;
    }
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// The benchmark workloads built from the reference's own
// generator, independent of the product library: LP j (global index
// g = first + j) is gen({m[j], derive_seed(seed, 2g), kind[j], margin}) with
// insertion order shuffle(m[j], derive_seed(seed, 2g+1)) (generate.hpp:
// 174-189 streams), b and bound_m scaled by bscale. kind 3 is the builder's
// "unbounded" kind (no reference counterpart): feasible_random's draws with
// every normal within +-60 degrees of -c, restated here with the reference's
// xoshiro256pp. Returns 0, or -1 on a thrown exception / bad kind.
int ref_fill(int64_t n, int64_t first, uint64_t seed, const int32_t* m,
             const int64_t* offset, const uint8_t* kind, double margin, double bscale,
             double* ax, double* ay, double* b, uint32_t* perm, double* c,
             double* bound_m) {
  try {
    constexpr double two_pi = 2.0 * 3.141592653589793238462643383279502884;
    for (int64_t j = 0; j < n; ++j) {
      const uint64_t g = static_cast<uint64_t>(first + j);
      const int k = kind ? static_cast<int>(kind[j]) : 0;
      const int64_t o = offset[j];
      const uint64_t ps = lp2d::derive_seed(seed, 2 * g);
      if (k == 3) {
        lp2d::xoshiro256pp r(ps);
        const double phi = two_pi * r.unit();
        c[2 * j] = std::cos(phi);
        c[2 * j + 1] = std::sin(phi);
        const double half = 1e7 / 2.0;
        const double ix = r.in_range(-half, half), iy = r.in_range(-half, half);
        for (int64_t q = 0; q < m[j]; ++q) {
          double theta = two_pi * r.unit();
          theta = phi + 3.141592653589793 + (theta / two_pi * 2.0 - 1.0) * (3.141592653589793 / 3.0);
          const double a0 = std::cos(theta), a1 = std::sin(theta);
          const double slack = margin * (1.0 + 9.0 * r.unit());
          ax[o + q] = a0;
          ay[o + q] = a1;
          b[o + q] = (a0 * ix + a1 * iy) + slack;
        }
        bound_m[j] = 1e7;
      } else if (k == 0 || k == 1 || k == 2) {
        lp2d::gen_spec spec{static_cast<std::size_t>(m[j]), ps, static_cast<lp2d::gen_kind>(k),
                            margin};
        const lp2d::problem p = lp2d::gen(spec);
        for (std::size_t q = 0; q < p.constraints.size(); ++q) {
          ax[o + q] = p.constraints[q].a.x;
          ay[o + q] = p.constraints[q].a.y;
          b[o + q] = p.constraints[q].b;
        }
        c[2 * j] = p.obj.c.x;
        c[2 * j + 1] = p.obj.c.y;
        bound_m[j] = p.bound_m;
      } else {
        return -1;
      }
      if (bscale != 1.0) {
        for (int64_t q = 0; q < m[j]; ++q) b[o + q] *= bscale;
        bound_m[j] *= bscale;
      }
      if (perm) {
        const lp2d::permutation pm =
            lp2d::shuffle(static_cast<std::size_t>(m[j]), lp2d::derive_seed(seed, 2 * g + 1));
        std::memcpy(perm + o, pm.order.data(), sizeof(uint32_t) * pm.order.size());
      }
    }
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// Config 4 sizes: m = clamp(floor(xmin / u^(1/alpha)), xmin,
// xmax) with u from xoshiro256pp(derive_seed(seed, 0xB0)).unit(), until the
// sizes sum to target_total. Returns the count.
int64_t ref_pareto_sizes(uint64_t seed, double xmin, double alpha, int32_t xmax,
                         int64_t target_total, int64_t n_max, int32_t* m) {
  lp2d::xoshiro256pp r(lp2d::derive_seed(seed, 0xB0));
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

// serial.hpp solve on one LP, with stats.
void ref_solve(const double* ax, const double* ay, const double* b,
               const uint32_t* perm, int64_t m, double cx, double cy, double M,
               double eps_par, double eps_feas, uint8_t* feasible, double* x,
               double* y, double* value, uint64_t* viol, uint64_t* wu) {
  lp2d::problem p;
  p.obj.c = {cx, cy};
  p.bound_m = M;
  p.constraints.resize(static_cast<std::size_t>(m));
  for (int64_t k = 0; k < m; ++k) p.constraints[k] = {{ax[k], ay[k]}, b[k]};
  lp2d::permutation pm;
  pm.order.assign(perm, perm + m);
  lp2d::solve_stats st;
  const lp2d::solution s = lp2d::solve(p, pm, make_tol(eps_par, eps_feas), &st);
  fill_solution(s, feasible, x, y, value);
  *viol = st.violation_events;
  *wu = st.work_units;
}

int ref_bruteforce(const double* ax, const double* ay, const double* b,
                   int64_t m, double cx, double cy, double M, double eps_par,
                   double eps_feas, uint8_t* feasible, double* x, double* y,
                   double* value) {
  try {
    lp2d::problem p;
    p.obj.c = {cx, cy};
    p.bound_m = M;
    p.constraints.resize(static_cast<std::size_t>(m));
    for (int64_t k = 0; k < m; ++k) p.constraints[k] = {{ax[k], ay[k]}, b[k]};
    const lp2d::solution s =
        lp2d::solve_bruteforce(p, make_tol(eps_par, eps_feas));
    fill_solution(s, feasible, x, y, value);
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// A reference batch kept alive across timed solves (bench.hpp:101-119: the
// timed region is solve_batch alone; building the batch stays outside).
void* ref_batch_create(int64_t n, const int64_t* offset, const int32_t* m,
                       const double* ax, const double* ay, const double* b,
                       const uint32_t* perm, const double* c,
                       const double* bound_m) {
  auto* bt = new lp2d::batch;
  bt->problems.resize(static_cast<std::size_t>(n));
  bt->permutations.resize(static_cast<std::size_t>(n));
  for (int64_t j = 0; j < n; ++j) {
    lp2d::problem& p = bt->problems[j];
    const int64_t o = offset[j];
    p.obj.c = {c[2 * j], c[2 * j + 1]};
    p.bound_m = bound_m[j];
    p.constraints.resize(static_cast<std::size_t>(m[j]));
    for (int32_t k = 0; k < m[j]; ++k) {
      p.constraints[k] = {{ax[o + k], ay[o + k]}, b[o + k]};
    }
    bt->permutations[j].order.assign(perm + o, perm + o + m[j]);
  }
  return bt;
}

void ref_batch_free(void* h) { delete static_cast<lp2d::batch*>(h); }

// solve_batch(b, {block_width, scheduler, workers}, tol). Returns wall ns of
// the solve_batch call, or -1 on std::invalid_argument. Outputs may be NULL.
int64_t ref_batch_solve(void* h, int64_t block_width, int scheduler,
                        unsigned workers, double eps_par, double eps_feas,
                        uint8_t* feasible, double* x, double* y,
                        double* value, uint64_t* stats /* [5] */,
                        double* imbalance) {
  const auto* bt = static_cast<const lp2d::batch*>(h);
  lp2d::block_config cfg;
  cfg.block_width = static_cast<std::size_t>(block_width);
  cfg.scheduler = scheduler == 0 ? lp2d::scheduler_kind::naive
                                 : lp2d::scheduler_kind::balanced;
  cfg.workers = workers;
  try {
    const auto t0 = std::chrono::steady_clock::now();
    const lp2d::batch_result r =
        lp2d::solve_batch(*bt, cfg, make_tol(eps_par, eps_feas));
    const auto t1 = std::chrono::steady_clock::now();
    if (feasible) {
      for (std::size_t j = 0; j < r.solutions.size(); ++j) {
        fill_solution(r.solutions[j], &feasible[j], &x[j], &y[j], &value[j]);
      }
    }
    if (stats) {
      stats[0] = r.stats.total_wu;
      stats[1] = r.stats.violation_events;
      stats[2] = r.stats.masked_lane_iterations;
      stats[3] = r.stats.idle_wu_steps;
      stats[4] = r.stats.blocks;
    }
    if (imbalance) {
      *imbalance = r.stats.total_wu ? lp2d::lane_imbalance(r.stats) : 1.0;
    }
    return std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0)
        .count();
  } catch (const std::invalid_argument&) {
    return -1;
  }
}

// lane_stats of solve_batch (batch.hpp:94-107): lane_wu (nblocks * width
// entries) and [total_wu, violation_events, masked_lane_iterations,
// idle_wu_steps, blocks, iterations recorded]. Returns 0, -1 on error.
int ref_batch_lane_stats(void* h, int64_t block_width, int scheduler, int record,
                         uint64_t* lane_wu, uint64_t* stats, uint64_t* iter_wu) {
  const auto* bt = static_cast<const lp2d::batch*>(h);
  lp2d::block_config cfg;
  cfg.block_width = static_cast<std::size_t>(block_width);
  cfg.scheduler = scheduler == 0 ? lp2d::scheduler_kind::naive : lp2d::scheduler_kind::balanced;
  cfg.workers = 1;
  cfg.record_iterations = record != 0;
  try {
    const lp2d::batch_result r = lp2d::solve_batch(*bt, cfg, lp2d::tolerance{});
    std::memcpy(lane_wu, r.stats.lane_wu.data(), sizeof(uint64_t) * r.stats.lane_wu.size());
    stats[0] = r.stats.total_wu;
    stats[1] = r.stats.violation_events;
    stats[2] = r.stats.masked_lane_iterations;
    stats[3] = r.stats.idle_wu_steps;
    stats[4] = r.stats.blocks;
    stats[5] = r.stats.iterations.size();
    if (iter_wu)
      for (std::size_t k = 0; k < r.stats.iterations.size(); ++k) {
        const auto& it = r.stats.iterations[k];
        iter_wu[6 * k + 0] = it.block;
        iter_wu[6 * k + 1] = it.iteration;
        iter_wu[6 * k + 2] = it.active_lanes;
        iter_wu[6 * k + 3] = it.masked_lanes;
        iter_wu[6 * k + 4] = it.wu_count;
        iter_wu[6 * k + 5] = it.idle_steps;
      }
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// Serial solve of every LP across `threads` std::threads.
int64_t ref_batch_solve_serial_threads(void* h, unsigned threads,
                                       double eps_par, double eps_feas,
                                       uint8_t* feasible, double* x, double* y,
                                       double* value) {
  const auto* bt = static_cast<const lp2d::batch*>(h);
  const std::size_t n = bt->problems.size();
  const lp2d::tolerance tol = make_tol(eps_par, eps_feas);
  std::vector<lp2d::solution> out(n);
  if (threads < 1) threads = 1;
  const auto t0 = std::chrono::steady_clock::now();
  {
    std::atomic<std::size_t> next{0};
    std::vector<std::jthread> pool;
    for (unsigned w = 0; w < threads; ++w) {
      pool.emplace_back([&] {
        for (std::size_t j = next.fetch_add(64); j < n; j = next.fetch_add(64)) {
          const std::size_t e = std::min(n, j + 64);
          for (std::size_t i = j; i < e; ++i) {
            out[i] = lp2d::solve(bt->problems[i], bt->permutations[i], tol);
          }
        }
      });
    }
  }
  const auto t1 = std::chrono::steady_clock::now();
  if (feasible) {
    for (std::size_t j = 0; j < n; ++j) {
      fill_solution(out[j], &feasible[j], &x[j], &y[j], &value[j]);
    }
  }
  return std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
}

// bench::verify(count, max_size, opts) — the reference's own parity harness.
int64_t ref_verify(int64_t count, int64_t max_size, uint64_t seed,
                   int64_t block_width) {
  lp2d::bench::sweep_options opts;
  opts.seed = seed;
  opts.block_width = static_cast<std::size_t>(block_width);
  const auto rep = lp2d::bench::verify(static_cast<std::size_t>(count),
                                       static_cast<std::size_t>(max_size), opts);
  return static_cast<int64_t>(rep.disagreements);
}

// reduction.hpp:46 segmented_extremes; -1 when it throws invalid_argument.
int ref_segmented_extremes(const double* in, int64_t n, int64_t contention, int strategy,
                           double* out_min, double* out_max) {
  const std::size_t groups = contention > 0 ? static_cast<std::size_t>(n / contention) : 0;
  try {
    lp2d::segmented_extremes(std::span<const double>(in, static_cast<std::size_t>(n)),
                             static_cast<std::size_t>(contention),
                             static_cast<lp2d::reduce_strategy>(strategy),
                             std::span<double>(out_min, groups), std::span<double>(out_max, groups));
  } catch (const std::invalid_argument&) {
    return -1;
  }
  return 0;
}

// bench.hpp:256-257 contention inputs.
void ref_uniform(uint64_t seed, uint64_t stream, double lo, double hi, int64_t n, double* out) {
  lp2d::xoshiro256pp rng(lp2d::derive_seed(seed, stream));
  for (int64_t i = 0; i < n; ++i) out[i] = rng.in_range(lo, hi);
}

// bench::contention_bench: the reference's own CPU timing of one strategy at
// one contention level (ns per pass, median of reps).
int64_t ref_contention_ns(int strategy, int64_t contention, int64_t reps, uint64_t seed,
                          int64_t values) {
  const lp2d::reduce_strategy s = static_cast<lp2d::reduce_strategy>(strategy);
  const std::size_t c = static_cast<std::size_t>(contention);
  const auto recs = lp2d::bench::contention_bench(std::span<const lp2d::reduce_strategy>(&s, 1),
                                                  std::span<const std::size_t>(&c, 1),
                                                  static_cast<std::size_t>(reps), seed,
                                                  static_cast<std::size_t>(values));
  std::vector<int64_t> t;
  for (const auto& r : recs) t.push_back(r.wall_time_ns);
  std::sort(t.begin(), t.end());
  return t.empty() ? 0 : t[t.size() / 2];
}

}  // extern "C"
