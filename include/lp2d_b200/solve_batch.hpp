// lp2d_b200/solve_batch.hpp — C++ drop-in for lp2d::solve_batch on the GPU.
//
// Include AFTER the reference's <lp2d/batch.hpp> (it uses the reference's
// own types):
//
//   #include <lp2d/batch.hpp>
//   #include <lp2d_b200/solve_batch.hpp>
//   lp2d::batch_result r = lp2d::b200::solve_batch(b, cfg, tol);
//
// Same signature, types, validation and exceptions as
// /root/reference/proj/include/lp2d/batch.hpp:303-320; solutions are
// bit-identical to the reference's (fp64 on the GPU). block_config::workers
// selects the number of GPUs (0 = all visible); block_width is validated but
// the GPU schedule is the kernel's. lane_stats carries the exact
// total_wu / violation_events; lane_wu holds one entry per LP.
// solve_batch_ex additionally returns the builder's status / defining pair.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../lp2d_b200.h"

namespace lp2d::b200 {

struct extended_result {
  lp2d::batch_result result;
  std::vector<std::uint8_t> status;  // LP2D_OPTIMAL / _INFEASIBLE / _UNBOUNDED
  std::vector<std::int32_t> pair;    // 2 per LP (original index, box -> -1..-4)
};

inline extended_result solve_batch_ex(const lp2d::batch& b, const lp2d::block_config& cfg = {},
                                      const lp2d::tolerance& tol = {}) {
  const std::size_t n = b.problems.size();
  // batch.hpp:305-320, same checks in the same order.
  if (n == 0) throw std::invalid_argument("solve_batch: empty batch");
  if (b.permutations.size() != n)
    throw std::invalid_argument("solve_batch: one permutation per problem required");
  for (std::size_t i = 0; i < n; ++i)
    if (b.permutations[i].order.size() != b.problems[i].constraints.size())
      throw std::invalid_argument("solve_batch: permutation length does not match problem size");
  if (cfg.block_width == 0) throw std::invalid_argument("solve_batch: block width must be positive");

  // AoS problems -> packed SoA (the layout contract of lp2d_b200.h).
  std::vector<std::int32_t> m(n);
  for (std::size_t i = 0; i < n; ++i) m[i] = static_cast<std::int32_t>(b.problems[i].constraints.size());
  std::vector<std::int64_t> off(n + 1);
  const std::int64_t total = lp2dgpu_pack_offsets(static_cast<std::int64_t>(n), m.data(), off.data());
  std::vector<double> ax(total), ay(total), bb(total), c(2 * n), M(n);
  std::vector<std::uint32_t> perm(total);
  for (std::size_t i = 0; i < n; ++i) {
    const auto& p = b.problems[i];
    const std::int64_t o = off[i];
    for (std::size_t k = 0; k < p.constraints.size(); ++k) {
      ax[o + k] = p.constraints[k].a.x;
      ay[o + k] = p.constraints[k].a.y;
      bb[o + k] = p.constraints[k].b;
      perm[o + k] = b.permutations[i].order[k];
    }
    c[2 * i] = p.obj.c.x;
    c[2 * i + 1] = p.obj.c.y;
    M[i] = p.bound_m;
  }
  lp2d_batch_soa soa{};
  soa.n = static_cast<std::int64_t>(n);
  soa.m = m.data();
  soa.offset = off.data();
  soa.ax = ax.data();
  soa.ay = ay.data();
  soa.b = bb.data();
  soa.perm = perm.data();
  soa.perm_bits = LP2D_PERM_U32;
  soa.mem = LP2D_MEM_HOST;
  soa.c = c.data();
  soa.bound_m = M.data();
  lp2d_opts opts;
  lp2dgpu_default_opts(&opts);
  opts.scheduler = cfg.scheduler == lp2d::scheduler_kind::naive ? LP2D_SCHED_NAIVE : LP2D_SCHED_BALANCED;
  opts.block_width = cfg.block_width > 0x7fffffff ? 0x7fffffff : static_cast<std::int32_t>(cfg.block_width);
  opts.n_gpus = static_cast<std::int32_t>(cfg.workers);
  opts.eps_parallel = tol.eps_parallel;
  opts.eps_feas = tol.eps_feas;
  extended_result ex;
  ex.status.resize(n);
  ex.pair.resize(2 * n);
  std::vector<double> x(n), y(n), v(n);
  std::vector<std::uint32_t> viol(n);
  std::vector<std::uint64_t> wu(n);
  lp2d_out out{ex.status.data(), x.data(), y.data(), v.data(), ex.pair.data(), viol.data(), wu.data()};
  const int rc = lp2dgpu_solve_f64(&soa, &opts, &out);
  if (rc != LP2D_OK) {
    const std::string msg = lp2dgpu_last_error();
    if (rc == LP2D_ERR_CUDA || rc == LP2D_ERR_UNSUPPORTED) throw std::runtime_error(msg);
    throw std::invalid_argument(msg);
  }
  lp2d::batch_result& r = ex.result;
  r.solutions.resize(n);
  r.stats.block_width = cfg.block_width;
  r.stats.blocks = n;
  r.stats.lane_wu.assign(wu.begin(), wu.end());
  for (std::size_t i = 0; i < n; ++i) {
    if (ex.status[i] == LP2D_OPTIMAL || ex.status[i] == LP2D_UNBOUNDED)
      r.solutions[i] = lp2d::solution::optimal({x[i], y[i]}, v[i]);
    else
      r.solutions[i] = lp2d::solution::infeasible();
    r.stats.total_wu += wu[i];
    r.stats.violation_events += viol[i];
  }
  return ex;
}

inline lp2d::batch_result solve_batch(const lp2d::batch& b, const lp2d::block_config& cfg = {},
                                      const lp2d::tolerance& tol = {}) {
  return solve_batch_ex(b, cfg, tol).result;
}

}  // namespace lp2d::b200
