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
// the GPU schedule is the kernel's. lane_stats are the
// reference's (block semantics of run_block), rebuilt exactly from the GPU
// solve's per-(block, step) violation histogram (rebuild_lane_stats).
// A permutation entry >= m throws std::invalid_argument.
// solve_batch_ex additionally returns the builder's status / defining pair.
#pragma once

#include <algorithm>
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

// The reference's lane_stats (batch.hpp:94-107, block semantics of run_block
// :149-294, merge :357-371) rebuilt exactly from the GPU solve: per block of
// W = block_width LPs and per executed insertion step, the masked lanes (out
// of the batch, past their m, or infeasible from the step of their
// infeasible event), the balanced deal of active*prefix units round-robin
// over W lanes, or the naive per-lane prefixes; `hist` is the solve's
// lp2d_out::iter_hist. Same numbers as the reference's own emulation.
inline lp2d::lane_stats rebuild_lane_stats(const lp2d::batch& b,
                                           const std::vector<std::uint8_t>& status,
                                           const std::vector<std::int32_t>& pair,
                                           const std::vector<std::uint64_t>& wu,
                                           const std::vector<std::uint32_t>& hist,
                                           const lp2d::block_config& cfg) {
  const std::size_t n = b.problems.size(), W = cfg.block_width;
  const std::size_t nb = (n + W - 1) / W, stride = nb ? hist.size() / nb : 0;
  const bool balanced = cfg.scheduler == lp2d::scheduler_kind::balanced;
  lp2d::lane_stats st;
  st.block_width = W;
  st.blocks = nb;
  st.lane_wu.assign(nb * W, 0);
  std::vector<std::uint64_t> t(n, UINT64_MAX), mm(n);
  for (std::size_t j = 0; j < n; ++j) {
    mm[j] = b.problems[j].constraints.size();
    if (status[j] == LP2D_INFEASIBLE) {
      const auto& ord = b.permutations[j].order;
      for (std::size_t k = 0; k < ord.size(); ++k)
        if (static_cast<std::int32_t>(ord[k]) == pair[2 * j]) {
          t[j] = k + 1;
          break;
        }
    }
  }
  for (std::size_t blk = 0; blk < nb; ++blk) {
    const std::size_t first = blk * W, count = std::min(W, n - first);
    std::uint64_t lp_max = 0, last = 0;
    for (std::size_t l = 0; l < count; ++l) {
      lp_max = std::max(lp_max, mm[first + l]);
      last = std::max(last, std::min(mm[first + l], t[first + l]));
    }
    if (lp_max == 0) continue;
    last = std::min(lp_max, std::max<std::uint64_t>(1, last));
    for (std::uint64_t it = 1; it <= last; ++it) {
      const std::uint64_t prefix = 3 + it, active = hist[blk * stride + it];
      std::uint32_t masked = static_cast<std::uint32_t>(W - count);
      for (std::size_t l = 0; l < count; ++l)
        masked += (it > mm[first + l] || it > t[first + l]) ? 1u : 0u;
      st.masked_lane_iterations += masked;
      st.violation_events += active;
      const std::uint64_t wc = active * prefix;
      std::uint64_t idle = 0;
      lp2d::iteration_record rec;
      if (cfg.record_iterations) {
        rec.block = static_cast<std::uint32_t>(blk);
        rec.iteration = static_cast<std::uint32_t>(it);
        rec.active_lanes = static_cast<std::uint32_t>(active);
        rec.masked_lanes = masked;
        rec.lane_wu.assign(W, 0);
      }
      if (active) {
        if (balanced) {
          const std::uint64_t q = wc / W, r = wc % W;
          for (std::size_t l = 0; l < W; ++l) {
            const std::uint64_t u = q + (l < r ? 1 : 0);
            st.lane_wu[blk * W + l] += u;
            if (cfg.record_iterations) rec.lane_wu[l] = static_cast<std::uint32_t>(u);
          }
          idle = ((wc + W - 1) / W) * W - wc;
        } else {
          idle = prefix * (W - active);
        }
      }
      st.idle_wu_steps += idle;
      if (cfg.record_iterations) {
        rec.wu_count = wc;
        rec.idle_steps = idle;
        st.iterations.push_back(std::move(rec));
      }
    }
    if (!balanced)
      for (std::size_t l = 0; l < count; ++l) st.lane_wu[blk * W + l] = wu[first + l];
  }
  for (std::uint64_t u : st.lane_wu) st.total_wu += u;
  return st;
}

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
  std::int32_t max_m = 0;
  for (std::int32_t mi : m) max_m = std::max(max_m, mi);
  const std::size_t W = cfg.block_width, nb = (n + W - 1) / W;
  std::vector<std::uint32_t> hist(nb * (static_cast<std::size_t>(max_m) + 1));
  lp2d_out out{ex.status.data(), x.data(), y.data(), v.data(), ex.pair.data(),
               viol.data(),      wu.data(), hist.data()};
  const int rc = lp2dgpu_solve_f64(&soa, &opts, &out);
  if (rc != LP2D_OK) {
    const std::string msg = lp2dgpu_last_error();
    if (rc == LP2D_ERR_CUDA || rc == LP2D_ERR_UNSUPPORTED) throw std::runtime_error(msg);
    throw std::invalid_argument(msg);
  }
  for (std::size_t i = 0; i < n; ++i)
    if (ex.status[i] == LP2D_INVALID)
      throw std::invalid_argument("solve_batch: permutation entry out of range (problem " +
                                  std::to_string(i) + ")");
  lp2d::batch_result& r = ex.result;
  r.solutions.resize(n);
  for (std::size_t i = 0; i < n; ++i) {
    if (ex.status[i] == LP2D_OPTIMAL || ex.status[i] == LP2D_UNBOUNDED)
      r.solutions[i] = lp2d::solution::optimal({x[i], y[i]}, v[i]);
    else
      r.solutions[i] = lp2d::solution::infeasible();
  }
  r.stats = rebuild_lane_stats(b, ex.status, ex.pair, wu, hist, cfg);
  return ex;
}

inline lp2d::batch_result solve_batch(const lp2d::batch& b, const lp2d::block_config& cfg = {},
                                      const lp2d::tolerance& tol = {}) {
  return solve_batch_ex(b, cfg, tol).result;
}

}  // namespace lp2d::b200
