// Compiles the reference's own headers together with the C++ drop-in
// (include/lp2d_b200/solve_batch.hpp) and checks, the way the reference's
// test_batch.cpp:55-98 and :169-184 do, that the GPU solve_batch reproduces
// the reference serial solver bit for bit and validates its input. Built in
// the container (where /root/reference exists) by tests/cpp/Makefile; the GPU
// test runs the prebuilt binary.
#include <cstdio>
#include <stdexcept>

#include "lp2d/lp2d.hpp"
#include "lp2d_b200/solve_batch.hpp"

using namespace lp2d;

static int failures = 0;
#define CHECK(c)                                                     \
  do {                                                               \
    if (!(c)) {                                                      \
      std::printf("CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
      ++failures;                                                    \
    }                                                                \
  } while (0)

int main() {
  const tolerance tol{};
  {  // test_batch.cpp:55-74
    const batch b = replicate(gen({128, 77}), 96, 5);
    solve_stats st;
    for (const scheduler_kind sched : {scheduler_kind::naive, scheduler_kind::balanced}) {
      block_config cfg;
      cfg.scheduler = sched;
      const batch_result r = b200::solve_batch(b, cfg, tol);
      solve_stats s2;
      for (std::size_t i = 0; i < b.problems.size(); ++i) {
        CHECK(r.solutions[i] == solve(b.problems[i], b.permutations[i], tol, &s2));
      }
      CHECK(r.stats.violation_events == s2.violation_events);
      CHECK(r.stats.total_wu == s2.work_units);
    }
    (void)st;
  }
  {  // test_batch.cpp:76-98, mixed sizes + infeasible lanes
    batch b = gen_mixed(std::array<std::size_t, 3>{3, 40, 150}, 50, 123);
    for (std::size_t i : {7ul, 23ul, 48ul}) {
      b.problems[i] = gen({20, 1000 + i, gen_kind::infeasible});
      b.permutations[i] = shuffle(20, 2000 + i);
    }
    const batch_result r = b200::solve_batch(b, {}, tol);
    // lane_stats with the reference's block semantics, both schedulers and
    // an odd block width (rebuilt from the GPU's violation histogram)
    for (auto sched : {scheduler_kind::balanced, scheduler_kind::naive}) {
      block_config cfg;
      cfg.scheduler = sched;
      cfg.block_width = 7;
      cfg.record_iterations = true;
      const batch_result g = b200::solve_batch(b, cfg, tol);
      const batch_result c = solve_batch(b, cfg, tol);
      CHECK(g.stats.lane_wu == c.stats.lane_wu);
      CHECK(g.stats.blocks == c.stats.blocks);
      CHECK(g.stats.masked_lane_iterations == c.stats.masked_lane_iterations);
      CHECK(g.stats.idle_wu_steps == c.stats.idle_wu_steps);
      CHECK(g.stats.iterations.size() == c.stats.iterations.size());
      for (std::size_t k = 0; k < g.stats.iterations.size() && k < c.stats.iterations.size(); ++k) {
        CHECK(g.stats.iterations[k].active_lanes == c.stats.iterations[k].active_lanes);
        CHECK(g.stats.iterations[k].masked_lanes == c.stats.iterations[k].masked_lanes);
        CHECK(g.stats.iterations[k].idle_steps == c.stats.iterations[k].idle_steps);
        if (sched == scheduler_kind::balanced)
          CHECK(g.stats.iterations[k].lane_wu == c.stats.iterations[k].lane_wu);
      }
      CHECK(lane_imbalance(g.stats) == lane_imbalance(c.stats));
    }
    std::size_t infeasible = 0;
    for (std::size_t i = 0; i < b.problems.size(); ++i) {
      const solution s = solve(b.problems[i], b.permutations[i], tol);
      CHECK(r.solutions[i] == s);
      if (!s.feasible) ++infeasible;
    }
    CHECK(infeasible >= 3);
  }
  {  // the headline shape at a small count, fp64 bit-exact
    const batch b = gen_mixed(std::array<std::size_t, 1>{1024}, 64, 2);
    const batch_result g = b200::solve_batch(b);
    const batch_result c = solve_batch(b);  // the reference itself
    for (std::size_t i = 0; i < b.problems.size(); ++i) CHECK(g.solutions[i] == c.solutions[i]);
    CHECK(g.stats.total_wu == c.stats.total_wu);
  }
  {  // test_batch.cpp:169-184
    int thrown = 0;
    try { b200::solve_batch(batch{}); } catch (const std::invalid_argument&) { ++thrown; }
    batch b = replicate(gen({10, 1}), 2, 1);
    b.permutations.pop_back();
    try { b200::solve_batch(b); } catch (const std::invalid_argument&) { ++thrown; }
    batch c = replicate(gen({10, 1}), 2, 1);
    c.permutations[1].order.pop_back();
    try { b200::solve_batch(c); } catch (const std::invalid_argument&) { ++thrown; }
    block_config zero;
    zero.block_width = 0;
    try { b200::solve_batch(replicate(gen({10, 1}), 2, 1), zero); } catch (const std::invalid_argument&) { ++thrown; }
    batch d = replicate(gen({10, 1}), 2, 1);  // permutation entry out of range
    d.permutations[1].order[3] = 99;
    try { b200::solve_batch(d); } catch (const std::invalid_argument&) { ++thrown; }
    CHECK(thrown == 5);
  }
  std::printf(failures ? "shim_test: %d failures\n" : "shim_test: ok%d\n", failures);
  return failures ? 1 : 0;
}
