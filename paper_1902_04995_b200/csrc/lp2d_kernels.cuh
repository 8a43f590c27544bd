// lp2d_kernels.cuh — the batch-solve kernels (sm_100a).
//
// K3 "warp" kernel (scheduler = balanced): one warp owns one LP at a time; the
// LP's constraints live in REGISTERS in insertion order (lane l, slot s holds
// user constraint perm[32 s + l]). Per LP:
//   * violation test (core.hpp:111-113) of 32 consecutive insertion positions
//     at once against the current optimum; __ballot_sync + __ffs finds the
//     first violated position. Because the optimum only moves at a violation,
//     this is exactly the serial order of serial.hpp:173-186.
//   * on a violation at insertion index i, the 1D re-solve over the considered
//     prefix (4 box positions + i user constraints, serial.hpp:114-122) is
//     dealt as work units round-robin over the 32 lanes (the reference's
//     balanced deal, batch.hpp:219-240, with the warp as the block), folded
//     per lane, then merged with REDUX max/min (order-independent exact
//     min/max, serial.hpp:60-63) and resolved (serial.hpp:95-111).
// LPs are claimed dynamically by warps (atomic ticket), and the next LP's
// constraints are prefetched into shared memory by 1D bulk TMA
// (cp.async.bulk + mbarrier) while the current LP is solved from registers.
//
// Naive kernel (scheduler = naive): one thread per LP, constraints gathered
// from global memory in insertion order — the paper's unbalanced baseline
// (PAPER.md "RGB Naive"; batch.hpp:241-256).
#pragma once

#include <type_traits>

#include "lp2d_device.cuh"
#include "lp2d_pair.cuh"
#include "lp2d_fold.cuh"

namespace lp2d_b200 {

constexpr int kWarpsPerCta = 4;
#ifndef LP2D_WU_GROUP
#define LP2D_WU_GROUP 2
#endif
constexpr int kWuGroup = LP2D_WU_GROUP;

struct KParams {
  int64_t n_list;        // LPs this launch solves
  const int32_t* list;   // LP ids (nullptr: 0..n_list-1)
  // Size-class binning (mixed batches): when bin_counts is set, this launch
  // solves the ids of bins [bin_lo, bin_hi), stored in `list` after the ids
  // of the lower bins (k_bin_* below). A class is one bin, except the tiny
  // class of the lane kernel, which has one bin per m (ids sorted by m).
  const int32_t* bin_counts;
  int32_t bin_lo, bin_hi;
  const int32_t* m;
  const int64_t* offset;
  const void* ax;
  const void* ay;
  const void* b;
  const void* perm;
  const void* c;
  const void* bound_m;
  uint8_t* status;
  void* x;
  void* y;
  void* value;
  int32_t* pair;
  uint32_t* viol;
  uint64_t* wu;
  uint32_t* counter;     // [0] LP ticket, [1] finished warps (self-resetting)
  double eps_par, eps_feas, eps_hi;   // tolerance rounded to the scalar type
  float eps_par_f, eps_feas_f, eps_hi_f;  // (float copies: constant-bank operands)
  int32_t total_warps;
  PairConsts pk;  // packed-fp32 constants (lp2d_pair.cuh)
  unsigned long long* fxstat;  // K4 path counters (LP2D_B200_FX_STATS; null normally)
  // K4 certificate factors (host-computed from the tolerance, lp2d_fx.cuh):
  // Ka = A*fx_ka, Tpar = A*fx_tp, Ec = (|cx|+|cy|)*fx_ec, eps_feas rounded up
  float fx_ka, fx_tp, fx_ec, fx_eps;
  // Optional per-(block, insertion step) violation histogram (lane_stats with
  // the reference's block semantics, batch.hpp:149-294, are rebuilt from it on
  // the host): iter_hist[((hist_lp0 + lp) / hist_w) * hist_stride + iter] +=
  // 1 per violation at insertion step iter = pi - 3 (1-based).
  uint32_t* iter_hist;
  int64_t hist_lp0;
  int32_t hist_w, hist_stride;
};

__device__ __forceinline__ void note_event(const KParams& p, int64_t lp, uint32_t pi) {
  if (p.iter_hist)
    atomicAdd(p.iter_hist + ((p.hist_lp0 + lp) / p.hist_w) * (int64_t)p.hist_stride + (pi - 3), 1u);
}

template <typename T>
struct Eps {
  static __device__ __forceinline__ T par(const KParams& p) { return (T)p.eps_par; }
  static __device__ __forceinline__ T feas(const KParams& p) { return (T)p.eps_feas; }
  static __device__ __forceinline__ T hi(const KParams& p) { return (T)p.eps_hi; }
};
template <>
struct Eps<float> {
  static __device__ __forceinline__ float par(const KParams& p) { return p.eps_par_f; }
  static __device__ __forceinline__ float feas(const KParams& p) { return p.eps_feas_f; }
  static __device__ __forceinline__ float hi(const KParams& p) { return p.eps_hi_f; }
};

__host__ __device__ constexpr uint32_t round16(uint32_t x) {
  return (x + 15u) & ~15u;
}

// Warp layout: considered positions P = 32*chunk + lane, P in [0, m+4);
// positions 0..3 are the box constraints (serial.hpp:47-52), P >= 4 is user
// constraint perm[P-4] (batch.hpp:137-139). Chunks 0..NS-1 live in REGISTERS
// (fully unrolled, compile-time slot indices); chunks NS..NS+NT-1 (the
// "tail", only for the largest class) live in a per-warp shared-memory copy
// in insertion order and are walked by rolled loops, which keeps the hot code
// under the SM's instruction cache. The staging buffer receives one LP of up
// to kCap constraints (original order + permutation) by 1D bulk TMA.
// CAP (late-TMA classes): a smaller data capacity for launches whose LPs all
// have m <= CAP (config 2: m = 1024 → 14.4 KB per warp, 16 warps/SM); the
// permutation array keeps the class capacity so every chunk index stays in it.
template <typename T, typename P, int NS, int NT, int CAP = 0>
struct WarpLayout {
  static constexpr int kChunks = NS + NT;
  static constexpr int kCap = CAP ? CAP : 32 * kChunks - 4;
  static constexpr int kPermCap = 32 * kChunks - 4;
  static constexpr uint32_t kArr = round16(kCap * sizeof(T));
  static constexpr uint32_t kPerm = round16(kPermCap * sizeof(P));
  static constexpr uint32_t kStage = 3 * kArr + kPerm;
  // The tail is read in place from the staging buffer (through the
  // permutation), so the buffer lives until the LP is solved and the next
  // LP's TMA is issued at the end of the solve instead of the start. That
  // keeps the big class at 14.7 KB of shared memory per warp (15 warps/SM).
  static constexpr bool kLateTma = NT > 0;
  static constexpr uint32_t kBuf = kStage;  // per warp
  // Warps per CTA maximising resident warps under 227 KB of smem (ties to
  // the smaller CTA): 4 or 5 for the register-only classes, up to 7 for the
  // tail classes whose staging buffers bound the CTAs per SM.
  static constexpr int blocks_for(int w) { return (int)((227u * 1024u) / (w * kBuf + w * 8u)); }
  static constexpr int best_warps() {
    int bw = 4;
    // (fp64: 4, so 3 CTAs/SM leave 170 registers per thread)
    for (int w = 5; w <= (NT > 0 ? 7 : (sizeof(T) == 8 ? 4 : 5)); ++w)
      if (blocks_for(w) * w > blocks_for(bw) * bw) bw = w;
    return bw;
  }
  static constexpr int kWarps = best_warps();
#ifndef LP2D_MIN_BLOCKS
#define LP2D_MIN_BLOCKS 4
#endif
#ifndef LP2D_MIN_BLOCKS_F64
#define LP2D_MIN_BLOCKS_F64 3
#endif
  static constexpr int kMinB = sizeof(T) == 8 ? LP2D_MIN_BLOCKS_F64 : LP2D_MIN_BLOCKS;
  static constexpr int kMinBlocks =
      blocks_for(kWarps) < 1 ? 1 : (blocks_for(kWarps) < kMinB ? blocks_for(kWarps) : kMinB);
  // Late-TMA classes are launched with a run-time CTA shape (4..8 warps, the
  // most resident warps for this layout): launch bounds of the widest shape,
  // with the register budget of the best compile-time shape.
  static constexpr int kMaxWarpsRt = kLateTma ? 8 : kWarps;
  static constexpr int kMinBlocksRt =
      kLateTma ? ((kWarps * kMinBlocks + 7) / 8 < 1 ? 1
                  : ((kWarps * kMinBlocks + 7) / 8 > 2 ? 2 : (kWarps * kMinBlocks + 7) / 8))
               : kMinBlocks;
  static constexpr uint32_t kSmem = kWarps * kBuf + kWarps * 8;
  // Register chunks below this index are never past the end of an LP of this
  // size class (m + 4 > 32 * previous class's chunks), so their test needs
  // no bound check.
  static constexpr int kAlwaysValid =
      NT > 0 ? NS
             : (NS == 2 ? 1 : NS == 4 ? 2 : NS == 5 ? 4 : NS == 6 ? 5 : NS == 9 ? 6 : NS == 10 ? 9 : NS == 18 ? 10 : 0);
};

// Per-LP header held by lane 0 between claim and solve.
template <typename T>
struct Header {
  int64_t lp;
  int64_t off;
  int32_t m;
  int32_t ok;
  T cx, cy, M;
};

// This launch's LP list (see KParams::bin_counts).
__device__ __forceinline__ void resolve_list(const KParams& p, const int32_t*& list,
                                             int64_t& n) {
  list = p.list;
  n = p.n_list;
  if (p.bin_counts) {
    int64_t base = 0, cnt = 0;
    for (int c = 0; c < p.bin_lo; ++c) base += p.bin_counts[c];
    for (int c = p.bin_lo; c < p.bin_hi; ++c) cnt += p.bin_counts[c];
    list = p.list + base;
    n = cnt;
  }
}

template <typename L, typename T, typename P>
__device__ __forceinline__ void issue_lp(const KParams& p, const int32_t* list,
                                         int64_t j, unsigned char* buf, uint64_t* bar,
                                         uint64_t policy, Header<T>& h) {
  const int64_t lp = list ? (int64_t)list[j] : j;
  const int32_t mj = p.m[lp];
  const int64_t o = p.offset[lp];
  const int64_t o1 = p.offset[lp + 1];
  const int64_t cap8 = ((int64_t)mj + 7) & ~int64_t(7);
  const bool ok = mj >= 0 && mj <= L::kCap && (o & 7) == 0 && o1 - o >= cap8;
  const uint32_t bt = ok ? round16((uint32_t)mj * sizeof(T)) : 0u;
  const uint32_t bp = ok ? round16((uint32_t)mj * sizeof(P)) : 0u;
  mbar_arrive_expect_tx(bar, 3 * bt + bp);
  if (bt) {
    bulk_g2s(buf, static_cast<const T*>(p.ax) + o, bt, bar, policy);
    bulk_g2s(buf + L::kArr, static_cast<const T*>(p.ay) + o, bt, bar, policy);
    bulk_g2s(buf + 2 * L::kArr, static_cast<const T*>(p.b) + o, bt, bar,
             policy);
    bulk_g2s(buf + 3 * L::kArr, static_cast<const P*>(p.perm) + o, bp, bar,
             policy);
  }
  const T* c = static_cast<const T*>(p.c);
  h.lp = lp;
  h.off = o;
  h.m = mj;
  h.ok = ok;
  h.cx = c[2 * lp];
  h.cy = c[2 * lp + 1];
  h.M = static_cast<const T*>(p.bound_m)[lp];
}

// Predicated loads / atomics in inline PTX: issued exactly where written and
// never merged through a branch, so a pipeline stage's request does not make
// the warp wait for its result (the consumer is one LP later).
__device__ __forceinline__ uint32_t ldg_u32_if(const void* addr, bool pred) {
  uint32_t v = 0;
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.global.nc.u32 %0, [%1];\n\t}"
      : "+r"(v)
      : "l"(addr), "r"((uint32_t)pred)
      : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ldg_u16_if(const void* addr, bool pred) {
  uint32_t v = 0;
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t"
      "@q ld.global.nc.u16 %0, [%1];\n\t}"
      : "+r"(v)
      : "l"(addr), "r"((uint32_t)pred)
      : "memory");
  return v;
}
// Ticket claim by the predicated lane. The address carries a lane-dependent
// zero (lane * zero, zero = a run-time 0 such as KParams::pk.zero) so ptxas
// cannot prove it warp-uniform: a uniform-address atomic is rewritten into the
// warp-aggregated form (VOTEU/POPC/leader ATOMG + an immediate SHFL of the
// result), which stalls on the atomic's round trip right here instead of where
// the ticket is consumed, one LP later.
__device__ __forceinline__ uint32_t atomic_add_if(uint32_t* addr, bool pred, uint64_t zero) {
  uint32_t v = 0;
  const uint32_t* a = addr + (uint64_t)(threadIdx.x & 31) * zero;
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q atom.global.add.u32 %0, [%1], 1;\n\t}"
      : "+r"(v)
      : "l"(a), "r"((uint32_t)pred)
      : "memory");
  return v;
}

// Lane-distributed LP header: lane w holds 32-bit word w of one LP's header
// (0 m; 1,2 offset[lp]; 3,4 offset[lp+1]; then cx, cy, M as raw words), one
// register per lane, all words requested by a single predicated load.
template <typename T>
__device__ __forceinline__ uint32_t load_header_word(const KParams& p, int64_t lp, int lane) {
  constexpr int WT = sizeof(T) / 4;  // words per scalar
  const uint32_t* base;
  int64_t wi;
  if (lane == 0) {
    base = reinterpret_cast<const uint32_t*>(p.m);
    wi = lp;
  } else if (lane < 5) {
    base = reinterpret_cast<const uint32_t*>(p.offset);
    wi = 2 * lp + (lane - 1);  // offset[lp], offset[lp+1] as lo/hi words
  } else if (lane < 5 + 2 * WT) {
    base = reinterpret_cast<const uint32_t*>(p.c);
    wi = 2 * WT * lp + (lane - 5);
  } else {
    base = reinterpret_cast<const uint32_t*>(p.bound_m);
    wi = WT * lp + (lane - 5 - 2 * WT);
  }
  const bool on = lp >= 0 && lane < 5 + 3 * WT;
  return ldg_u32_if(base + (on ? wi : 0), on);
}

template <typename T>
__device__ __forceinline__ T word_scalar(uint32_t w, int src) {
  if constexpr (sizeof(T) == 4) {
    return __uint_as_float(__shfl_sync(kFull, w, src));
  } else {
    const uint32_t lo = __shfl_sync(kFull, w, src), hi = __shfl_sync(kFull, w, src + 1);
    return __longlong_as_double((long long)(((unsigned long long)hi << 32) | lo));
  }
}

template <typename L, typename T>
__device__ __forceinline__ Header<T> unpack_header(uint32_t w, int64_t lp) {
  constexpr int WT = sizeof(T) / 4;
  Header<T> h;
  h.lp = lp;
  h.m = (int32_t)__shfl_sync(kFull, w, 0);
  h.off = (int64_t)(((uint64_t)__shfl_sync(kFull, w, 2) << 32) | __shfl_sync(kFull, w, 1));
  const int64_t o1 = (int64_t)(((uint64_t)__shfl_sync(kFull, w, 4) << 32) | __shfl_sync(kFull, w, 3));
  h.cx = word_scalar<T>(w, 5);
  h.cy = word_scalar<T>(w, 5 + WT);
  h.M = word_scalar<T>(w, 5 + 2 * WT);
  const int64_t cap8 = ((int64_t)h.m + 7) & ~int64_t(7);
  h.ok = h.m >= 0 && h.m <= L::kCap && (h.off & 7) == 0 && o1 - h.off >= cap8;
  return h;
}

// Stage an LP's ax/ay/b/perm segments into the warp's buffer with 1D bulk
// copies completing on the warp's mbarrier (no bytes if !ok). Called by the
// whole warp: the operands are made warp-uniform by REDUX (results in uniform
// registers), so lane 0 issues the bulk copies with them directly instead of
// ptxas's per-lane waterfall loop around each UBLKCP (the header values are
// equal on every lane already).
template <typename L, typename T, typename P>
__device__ __forceinline__ void issue_tma_warp(const KParams& p, const Header<T>& h,
                                               unsigned char* buf, uint64_t* bar,
                                               uint64_t policy, uint32_t arr, int lane) {
  const bool go = h.lp >= 0;
  const uint32_t m = __reduce_max_sync(kFull, h.ok ? (uint32_t)h.m : 0u);
  const uint32_t olo = __reduce_max_sync(kFull, (uint32_t)(uint64_t)h.off);
  const uint32_t ohi = __reduce_max_sync(kFull, (uint32_t)((uint64_t)h.off >> 32));
  const uint32_t sbuf = __reduce_max_sync(kFull, smem_u32(buf));
  const uint32_t sbar = __reduce_max_sync(kFull, smem_u32(bar));
  const uint32_t plo = __reduce_max_sync(kFull, (uint32_t)policy);
  const uint32_t phi = __reduce_max_sync(kFull, (uint32_t)(policy >> 32));
  const int64_t off = (int64_t)(((uint64_t)ohi << 32) | olo);
  const uint64_t pol = ((uint64_t)phi << 32) | plo;
  const uint32_t bt = round16(m * (uint32_t)sizeof(T));
  const uint32_t bp = round16(m * (uint32_t)sizeof(P));
  if (lane == 0 && go) {
    mbar_arrive_expect_tx_u(sbar, 3 * bt + bp);
    if (bt) {
      bulk_g2s_u(sbuf, static_cast<const T*>(p.ax) + off, bt, sbar, pol);
      bulk_g2s_u(sbuf + arr, static_cast<const T*>(p.ay) + off, bt, sbar, pol);
      bulk_g2s_u(sbuf + 2 * arr, static_cast<const T*>(p.b) + off, bt, sbar, pol);
      bulk_g2s_u(sbuf + 3 * arr, static_cast<const P*>(p.perm) + off, bp, sbar, pol);
    }
  }
}

// Defining-pair export: box k -> -(k+1), user position 4+i -> perm[i].
__device__ __forceinline__ int32_t pair_code(uint32_t pos, uint32_t orig) {
  if (pos == kNone) return (int32_t)0x80000000;
  if (pos < 4) return -(int32_t)pos - 1;
  return (int32_t)orig;
}

template <typename T>
__device__ __forceinline__ Header<T> bcast(const Header<T>& h) {
  Header<T> r;
  r.lp = __shfl_sync(kFull, h.lp, 0);
  r.off = __shfl_sync(kFull, h.off, 0);
  r.m = __shfl_sync(kFull, h.m, 0);
  r.ok = __shfl_sync(kFull, h.ok, 0);
  r.cx = __shfl_sync(kFull, h.cx, 0);
  r.cy = __shfl_sync(kFull, h.cy, 0);
  r.M = __shfl_sync(kFull, h.M, 0);
  return r;
}

template <typename T>
__device__ __forceinline__ void write_main(const KParams& p, const Header<T>& h, uint8_t st,
                                           T px, T py, uint32_t viol, uint64_t wu) {
  const int64_t lp = h.lp;
  p.status[lp] = st;
  T vx = T(0), vy = T(0), vv = T(0);
  if (st == 0 || st == 2) {
    vx = px;
    vy = py;
    vv = h.cx * px + h.cy * py;  // serial.hpp:187 objective_value
  }
  static_cast<T*>(p.x)[lp] = vx;
  static_cast<T*>(p.y)[lp] = vy;
  static_cast<T*>(p.value)[lp] = vv;
  if (p.viol) p.viol[lp] = viol;
  if (p.wu) p.wu[lp] = wu;
}

template <typename T, typename P>
__device__ __forceinline__ void write_result(const KParams& p,
                                             const Header<T>& h, uint8_t st,
                                             T px, T py, uint32_t pos0,
                                             uint32_t pos1, uint32_t viol,
                                             uint64_t wu) {
  const P* perm = static_cast<const P*>(p.perm) + h.off;
  auto exp = [&](uint32_t pos) -> int32_t {
    if (pos == kNone) return (int32_t)0x80000000;
    if (pos < 4) return -(int32_t)pos - 1;
    return (int32_t)perm[pos - 4];
  };
  const int64_t lp = h.lp;
  p.status[lp] = st;
  T vx = T(0), vy = T(0), vv = T(0);
  if (st == 0 || st == 2) {
    vx = px;
    vy = py;
    vv = h.cx * px + h.cy * py;  // serial.hpp:187 objective_value
  }
  static_cast<T*>(p.x)[lp] = vx;
  static_cast<T*>(p.y)[lp] = vy;
  static_cast<T*>(p.value)[lp] = vv;
  if (p.pair) {
    const bool valid = st != 255;
    p.pair[2 * lp] = valid ? exp(pos0) : (int32_t)0x80000000;
    p.pair[2 * lp + 1] = valid ? exp(pos1) : (int32_t)0x80000000;
  }
  if (p.viol) p.viol[lp] = viol;
  if (p.wu) p.wu[lp] = wu;
}

// Exact 1D fold over considered positions [0, pi) straight from global
// memory with the reference's classify (wu_apply). Taken only when a unit of
// the register fold hit the parallel bound (essentially parallel constraints),
// so speed is irrelevant; out of line to keep the hot code small.
// S: the storage type of the scalars (float storage is widened exactly, the
// fp32 configs' semantics).
template <typename T, typename P, typename S = T>
__device__ __noinline__ Acc<T> fold_exact_global(const KParams& p, int64_t off,
                                                 uint32_t pi, Line<T> l, T M,
                                                 T eps_par, T eps_feas, T eps_hi) {
  const int lane = threadIdx.x & 31;
  const S* ax = static_cast<const S*>(p.ax) + off;
  const S* ay = static_cast<const S*>(p.ay) + off;
  const S* b = static_cast<const S*>(p.b) + off;
  const P* perm = static_cast<const P*>(p.perm) + off;
  Acc<T> acc;
  acc.uL = -T(INFINITY);
  acc.uR = T(INFINITY);
  acc.oL = acc.oR = acc.par = kNone;
  for (uint32_t k = lane; k < pi; k += 32) {
    T vax, vay, vb;
    if (k < 4) {
      vax = k == 0 ? T(1) : (k == 1 ? T(-1) : T(0));
      vay = k == 2 ? T(1) : (k == 3 ? T(-1) : T(0));
      vb = M;
    } else {
      const uint32_t o = perm[k - 4];
      vax = (T)ax[o];
      vay = (T)ay[o];
      vb = (T)b[o];
    }
    wu_apply(vax, vay, vb, l, eps_par, eps_feas, eps_hi, k, acc);
  }
  return acc;
}

// Per-LP running state of the incremental loop (serial.hpp:159-188) plus the
// builder's defining pair (considered positions) and the solve_stats.
template <typename T>
struct LPState {
  T px, py;
  uint32_t pos0, pos1;
  uint32_t viol;
  uint64_t wu;
  uint8_t st;  // 0 running/optimal, 1 infeasible, 255 invalid
};

template <typename T>
__device__ __forceinline__ void lp_init(LPState<T>& S, const Header<T>& h) {
  const T M = h.M;
  S.px = h.cx < T(0) ? -M : M;  // serial.hpp:56-58
  S.py = h.cy < T(0) ? -M : M;
  S.pos0 = h.cx < T(0) ? 1u : 0u;  // the box corner's two edges
  S.pos1 = h.cy < T(0) ? 3u : 2u;
  S.viol = 0;
  S.wu = 0;
  S.st = 0;
}

// Lanes' folded intervals merged over the warp (order-independent exact
// min/max, serial.hpp:60-63; owners tie to the smallest position).
template <typename T>
struct Merged {
  T uL, uR;
  uint32_t oL, oR, par;
};

template <typename T>
__device__ __forceinline__ Merged<T> merge_lanes(const Acc<T>& acc, bool with_par) {
  Merged<T> mg;
  T nuR;
  // The reductions are independent: issued back to back, no branch between.
  warp_best(acc.uL, acc.oL, mg.uL, mg.oL);
  warp_best(-acc.uR, acc.oR, nuR, mg.oR);
  mg.uR = -nuR;
  mg.par = with_par ? __reduce_min_sync(kFull, acc.par) : kNone;
  return mg;
}

// Resolve the 1D program on l (serial.hpp:95-111) for the violation at
// considered position pi. Returns false when the LP turned out infeasible.
template <typename T>
__device__ __forceinline__ bool resolve_merged(LPState<T>& S, const Merged<T>& mg,
                                               const Line<T>& l, uint32_t pi,
                                               const Header<T>& h, T cthr, T eps_feas) {
  if (mg.par != kNone) {  // serial.hpp:97 parallel-infeasible
    S.st = 1;
    S.pos0 = pi;
    S.pos1 = mg.par;
    return false;
  }
  const T scale = fmax(fabs(mg.uL), fabs(mg.uR));
  if (mg.uL > mg.uR + feas_slack(eps_feas, scale)) {  // serial.hpp:98-101
    S.st = 1;
    S.pos0 = pi;
    S.pos1 = mg.oL;
    return false;
  }
  const T along = h.cx * l.dx + h.cy * l.dy;  // serial.hpp:102-108
  const bool take_right = !(fabs(along) <= cthr) && along > T(0);
  const T t = take_right ? mg.uR : mg.uL;
  S.px = l.ox + t * l.dx;
  S.py = l.oy + t * l.dy;
  S.pos0 = pi;
  S.pos1 = take_right ? mg.oR : mg.oL;
  return true;
}

template <typename T>
__device__ __forceinline__ bool resolve_event(LPState<T>& S, const Acc<T>& acc,
                                              const Line<T>& l, uint32_t pi,
                                              const Header<T>& h, T cthr,
                                              T eps_feas) {
  return resolve_merged(S, merge_lanes(acc, true), l, pi, h, cthr, eps_feas);
}

// Whole-LP exact solve straight from global memory (no register staging):
// the reference loop with warp-parallel tests and folds. Used for LPs whose
// magnitudes leave the fast path's proven range (non-finite or huge
// coefficients, a non-finite running optimum); rare, so simple.
template <typename T, typename P, typename SS = T>
// skip_note: events already noted by a partial fast solve of this LP (the
// exact re-solve repeats them; note_event records each event once).
__device__ __noinline__ void solve_exact_global(const KParams& p, const Header<T>& h,
                                                T eps_par, T eps_feas, T eps_hi,
                                                LPState<T>& S, uint32_t skip_note = 0) {
  const int lane = threadIdx.x & 31;
  const SS* ax = static_cast<const SS*>(p.ax) + h.off;
  const SS* ay = static_cast<const SS*>(p.ay) + h.off;
  const SS* b = static_cast<const SS*>(p.b) + h.off;
  const P* perm = static_cast<const P*>(p.perm) + h.off;
  lp_init(S, h);
  const T cthr = eps_par * sqrt(h.cx * h.cx + h.cy * h.cy);
  const int m = h.m;
  int start = 0;
  while (start < m) {
    const int i = start + lane;
    bool v = false;
    if (i < m) {
      const uint32_t o = perm[i];
      v = !satisfied((T)ax[o], (T)ay[o], (T)b[o], S.px, S.py, eps_feas);
    }
    const uint32_t vm = __ballot_sync(kFull, v);
    if (!vm) {
      start += 32;
      continue;
    }
    const int iv = start + __ffs(vm) - 1;
    const uint32_t o = perm[iv];
    const uint32_t pi = 4u + (uint32_t)iv;
    S.viol += 1;
    S.wu += pi;
    if (lane == 0 && S.viol > skip_note) note_event(p, h.lp, pi);
    const Line<T> l = boundary_of((T)ax[o], (T)ay[o], (T)b[o]);
    const Acc<T> acc = fold_exact_global<T, P, SS>(p, h.off, pi, l, h.M, eps_par, eps_feas, eps_hi);
    if (!resolve_event(S, acc, l, pi, h, cthr, eps_feas)) return;
    start = iv + 1;
  }
}

// k_solve_warp (the balanced warp-per-LP solver) lives in lp2d_warp.cuh.

// Naive: thread per LP, the serial loop with global-memory gathers.
template <typename T, typename P>
__global__ void __launch_bounds__(128) k_solve_naive(const __grid_constant__ KParams p) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int32_t* list;
  int64_t n_list;
  resolve_list(p, list, n_list);
  if (j >= n_list) return;
  const T eps_par = (T)p.eps_par;
  const T eps_feas = (T)p.eps_feas;
  const T eps_hi = (T)p.eps_hi;
  Header<T> h;
  h.lp = list ? (int64_t)list[j] : j;
  h.m = p.m[h.lp];
  h.off = p.offset[h.lp];
  h.ok = h.m >= 0;
  h.cx = static_cast<const T*>(p.c)[2 * h.lp];
  h.cy = static_cast<const T*>(p.c)[2 * h.lp + 1];
  h.M = static_cast<const T*>(p.bound_m)[h.lp];
  const T* ax = static_cast<const T*>(p.ax) + h.off;
  const T* ay = static_cast<const T*>(p.ay) + h.off;
  const T* b = static_cast<const T*>(p.b) + h.off;
  const P* perm = static_cast<const P*>(p.perm) + h.off;
  const T M = h.M;
  T px = h.cx < T(0) ? -M : M;
  T py = h.cy < T(0) ? -M : M;
  uint32_t pos0 = h.cx < T(0) ? 1u : 0u;
  uint32_t pos1 = h.cy < T(0) ? 3u : 2u;
  const T cthr = eps_par * sqrt(h.cx * h.cx + h.cy * h.cy);
  uint32_t viol = 0;
  uint64_t wu = 0;
  uint8_t st = h.ok ? 0 : 255;
  for (int32_t i = 0; i < h.m && st == 0; ++i) {
    const uint32_t oi = perm[i];
    if (oi >= (uint32_t)h.m) {
      st = 255;
      break;
    }
    const T hx = ax[oi], hy = ay[oi], hb = b[oi];
    if (satisfied(hx, hy, hb, px, py, eps_feas)) continue;
    viol += 1;
    wu += 4 + (uint32_t)i;
    note_event(p, h.lp, 4u + (uint32_t)i);
    const Line<T> l = boundary_of(hx, hy, hb);
    Acc<T> acc;
    acc.uL = -T(INFINITY);
    acc.uR = T(INFINITY);
    acc.oL = acc.oR = acc.par = kNone;
    for (int k = 0; k < 4; ++k) {
      const T bx = k == 0 ? T(1) : (k == 1 ? T(-1) : T(0));
      const T by = k == 2 ? T(1) : (k == 3 ? T(-1) : T(0));
      wu_apply(bx, by, M, l, eps_par, eps_feas, eps_hi, (uint32_t)k, acc);
    }
    for (int32_t k = 0; k < i; ++k) {
      const uint32_t ok = min((uint32_t)perm[k], (uint32_t)(h.m - 1));
      wu_apply(ax[ok], ay[ok], b[ok], l, eps_par, eps_feas, eps_hi, 4u + k, acc);
    }
    if (acc.par != kNone) {
      st = 1;
      pos0 = 4 + i;
      pos1 = acc.par;
      break;
    }
    const T scale = fmax(fabs(acc.uL), fabs(acc.uR));
    if (acc.uL > acc.uR + feas_slack(eps_feas, scale)) {
      st = 1;
      pos0 = 4 + i;
      pos1 = acc.oL;
      break;
    }
    const T along = h.cx * l.dx + h.cy * l.dy;
    T t;
    uint32_t own;
    if (fabs(along) <= cthr) {
      t = acc.uL;
      own = acc.oL;
    } else if (along > T(0)) {
      t = acc.uR;
      own = acc.oR;
    } else {
      t = acc.uL;
      own = acc.oL;
    }
    px = l.ox + t * l.dx;
    py = l.oy + t * l.dy;
    pos0 = 4 + i;
    pos1 = own;
  }
  if (st == 0 && (pos0 < 4 || pos1 < 4)) st = 2;
  write_result<T, P>(p, h, st, px, py, pos0, pos1, viol, wu);
}

// ---------------------------------------------------------------------------
// Small LPs (m <= MAXM): one LP per LANE, 32 LPs per warp in lockstep — the
// paper's RGB layout (thread per LP, block-wide work-unit deal). Each lane
// gathers its LP's constraints through the permutation into a shared tile
// (element (position k, lane l) at [(k-4)*33 + l]: conflict-free both for
// all lanes reading their own position k and for all lanes reading one
// lane's positions). The warp sweeps positions 4, 5, ...: every lane tests
// position i of its own LP (one test per lane per step). The lanes that
// violated position i need a 1D fold over their positions 0..i-1; per step
// the warp picks the cheaper deal:
//   * lane-serial: each violated lane folds its own i units (cost ~ i);
//   * pooled: for each violated lane in turn the whole warp folds that LP's
//     i units (ceil(i/32) per lane) and merges them with REDUX — the balanced
//     deal of batch.hpp:219-240 with the warp as the block (cost ~ #violated).
// Both folds are wu_fold (fast division, per-LP parallel bound) with the
// exact reference fold (wu_apply) redone when a unit is undecided, as in the
// warp kernel. Box positions 0..3 are constants, not stored.
constexpr int kLaneWarps = 4;
constexpr int kLaneMaxM = 28;
#ifndef LP2D_LANE_MINB
#define LP2D_LANE_MINB 4  // resident CTAs per SM the lane kernel's registers allow
#endif

template <typename T, int MAXM>
struct LaneTile {
  static constexpr int kStride = 33;
  static constexpr size_t kWarpBytes = 3 * sizeof(T) * MAXM * kStride;
  static constexpr size_t kSmem = kLaneWarps * kWarpBytes;
};

template <typename T>
__device__ __forceinline__ void box_unit(int k, T M, T& bx, T& by, T& bb) {
  bx = k == 0 ? T(1) : (k == 1 ? T(-1) : T(0));  // serial.hpp:47-52
  by = k == 2 ? T(1) : (k == 3 ? T(-1) : T(0));
  bb = M;
}

template <typename T>
__device__ __forceinline__ Line<T> shfl_line(const Line<T>& l, int src) {
  Line<T> r;
  r.ox = __shfl_sync(kFull, l.ox, src);
  r.oy = __shfl_sync(kFull, l.oy, src);
  r.dx = __shfl_sync(kFull, l.dx, src);
  r.dy = __shfl_sync(kFull, l.dy, src);
  return r;
}

// S: storage type of the batch's scalars (float storage is widened exactly on
// load; the arithmetic is T's, the fp32 configs' double semantics).
template <typename T, typename P, int MAXM, typename S = T>
__global__ void __launch_bounds__(kLaneWarps * 32, LP2D_LANE_MINB) k_solve_lanes(const __grid_constant__ KParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  // the tile holds the STORED scalars (float storage: half the shared memory
  // of a double tile, so twice the resident warps); reads widen exactly
  using LT = LaneTile<S, MAXM>;
  constexpr int ST = LT::kStride;
  const int lane = threadIdx.x & 31, wic = threadIdx.x >> 5;
  S* sx = reinterpret_cast<S*>(smem + wic * LT::kWarpBytes);
  S* sy = sx + MAXM * ST;
  S* sb = sy + MAXM * ST;
  // user constraint at considered position k (>= 4) of lane c's LP
  auto at = [&](int k, int c) { return (k - 4) * ST + c; };
  const int32_t* list;
  int64_t n_list;
  resolve_list(p, list, n_list);
  const T eps_par = Eps<T>::par(p);
  const T eps_feas = Eps<T>::feas(p);
  const T eps_hi = Eps<T>::hi(p);
  const int64_t groups = (n_list + 31) / 32;
  const int64_t TW = p.total_warps;
  int64_t g = (int64_t)blockIdx.x * kLaneWarps + wic;
  while (g < groups) {
    // next group's ticket now; consumed after this group (one group ahead)
    const uint32_t ticket = atomic_add_if(p.counter, lane == 0, p.pk.zero);
    const int64_t j = g * 32 + lane;
    Header<T> h;
    h.lp = j < n_list ? (list ? (int64_t)list[j] : j) : -1;
    const bool live = h.lp >= 0;
    h.m = live ? p.m[h.lp] : 0;
    h.off = live ? p.offset[h.lp] : 0;
    h.ok = h.m >= 0 && h.m <= MAXM;
    h.cx = live ? (T) static_cast<const S*>(p.c)[2 * h.lp] : T(0);
    h.cy = live ? (T) static_cast<const S*>(p.c)[2 * h.lp + 1] : T(0);
    h.M = live ? (T) static_cast<const S*>(p.bound_m)[h.lp] : T(0);
    const int mj = live && h.ok ? h.m : 0;
    // ---- gather through the permutation (serial.hpp:28-32 insertion order)
    const S* gx = static_cast<const S*>(p.ax) + h.off;
    const S* gy = static_cast<const S*>(p.ay) + h.off;
    const S* gb = static_cast<const S*>(p.b) + h.off;
    const P* gp = static_cast<const P*>(p.perm) + h.off;
    uint32_t pmax = 0;
    decltype(float_bits(T(0))) sbits = float_bits(T(1));
    // The whole permutation by 16-byte loads (segments start 8-element
    // aligned and are padded to 8 elements: the layout contract), then every
    // constraint copied straight into the tile with cp.async (no registers,
    // one round trip for the data), then the magnitude bound from the tile.
    constexpr int PV = 16 / (int)sizeof(P);  // permutation entries per vector
    constexpr int NV = (MAXM + PV - 1) / PV;
    uint4 wv[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v)
      wv[v] = v * PV < mj ? __ldg(reinterpret_cast<const uint4*>(gp) + v) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const uint32_t ww[4] = {wv[v].x, wv[v].y, wv[v].z, wv[v].w};
#pragma unroll
      for (int e = 0; e < PV; ++e) {
        const int k = v * PV + e;
        if (k < MAXM && k < mj) {
          const uint32_t o = sizeof(P) == 2 ? ((ww[e / 2] >> (16 * (e & 1))) & 0xffffu) : ww[e];
          pmax = max(pmax, o);
          const uint32_t oc = min(o, (uint32_t)(mj - 1));
          cp_async_elem(&sx[at(4 + k, lane)], gx + oc);
          cp_async_elem(&sy[at(4 + k, lane)], gy + oc);
          cp_async_elem(&sb[at(4 + k, lane)], gb + oc);
        }
      }
    }
    cp_async_wait_all();
#pragma unroll
    for (int k = 0; k < MAXM; ++k)
      if (k < mj) sbits = max(sbits, float_bits(fabs((T)sx[at(4 + k, lane)]) + fabs((T)sy[at(4 + k, lane)])));
    __syncwarp();
    const bool bad = live && (!h.ok || (mj > 0 && pmax >= (uint32_t)mj));
    const T m_all = float_from_bits<T>(sbits);
    // Outside the fast path's proven range every unit is undecided, so the
    // folds below are the exact reference fold for this LP.
    const bool wild = !(m_all < Limits<T>::kBig) || !(fabs(h.M) < T(INFINITY));
    const T lpbnd = wild ? T(INFINITY)
                         : fmax(fmax(m_all, Limits<T>::kSmall) * eps_hi, FastDiv<T>::kDLo);
    LPState<T> St;
    lp_init(St, h);
    St.st = bad ? 255 : 0;
    const T cthr = eps_par * sqrt(h.cx * h.cx + h.cy * h.cy);
    bool alive = live && !bad;
    const int mpos = mj + 4;
    const int pend = __reduce_max_sync(kFull, alive ? (uint32_t)mpos : 0u);
    // ---- lockstep sweep (serial.hpp:168-186 per lane) ----------------------
    for (int i = 4; i < pend; ++i) {
      const bool v = alive && i < mpos &&
                     !satisfied((T)sx[at(i, lane)], (T)sy[at(i, lane)], (T)sb[at(i, lane)], St.px, St.py,
                                eps_feas);
      uint32_t vm = __ballot_sync(kFull, v);
      if (!vm) continue;
      Line<T> l;
      if (v) {
        St.viol += 1;
        St.wu += (uint32_t)i;
        note_event(p, h.lp, (uint32_t)i);
        l = boundary_of((T)sx[at(i, lane)], (T)sy[at(i, lane)], (T)sb[at(i, lane)]);
      }
      const int nv = __popc(vm);
      if (nv * (((i + 31) >> 5) * 26 + 64) >= i * 22) {
        // ---- lane-serial folds ----------------------------------------------
        if (v) {
          Acc<T> acc;
          acc.uL = -T(INFINITY);
          acc.uR = T(INFINITY);
          acc.oL = acc.oR = acc.par = kNone;
          bool rare = false;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            T bx, by, bb;
            box_unit(k, h.M, bx, by, bb);
            wu_fold(bx, by, bb, l, lpbnd, (uint32_t)k, true, acc, rare);
          }
#pragma unroll 4
          for (int k = 4; k < i; ++k)
            wu_fold((T)sx[at(k, lane)], (T)sy[at(k, lane)], (T)sb[at(k, lane)], l, lpbnd, (uint32_t)k,
                    true, acc, rare);
          if (rare) {  // exact reference fold for this lane (rare)
            acc.uL = -T(INFINITY);
            acc.uR = T(INFINITY);
            acc.oL = acc.oR = acc.par = kNone;
            for (int k = 0; k < 4; ++k) {
              T bx, by, bb;
              box_unit(k, h.M, bx, by, bb);
              wu_apply(bx, by, bb, l, eps_par, eps_feas, eps_hi, (uint32_t)k, acc);
            }
            for (int k = 4; k < i; ++k)
              wu_apply((T)sx[at(k, lane)], (T)sy[at(k, lane)], (T)sb[at(k, lane)], l, eps_par, eps_feas,
                       eps_hi, (uint32_t)k, acc);
          }
          Merged<T> mg;
          mg.uL = acc.uL;
          mg.uR = acc.uR;
          mg.oL = acc.oL;
          mg.oR = acc.oR;
          mg.par = acc.par;
          if (!resolve_merged(St, mg, l, (uint32_t)i, h, cthr, eps_feas)) alive = false;
        }
      } else {
        // ---- pooled: the warp folds each violated LP in turn ----------------
        while (vm) {
          const int c = __ffs(vm) - 1;
          vm &= vm - 1;
          const Line<T> lc = shfl_line(l, c);
          const T Mc = __shfl_sync(kFull, h.M, c);
          const T bnd = __shfl_sync(kFull, lpbnd, c);
          Acc<T> acc;
          acc.uL = -T(INFINITY);
          acc.uR = T(INFINITY);
          acc.oL = acc.oR = acc.par = kNone;
          bool rare = false;
          for (int k = lane; k < i; k += 32) {
            T x, y, bb;
            if (k < 4) {
              box_unit(k, Mc, x, y, bb);
            } else {
              x = (T)sx[at(k, c)];
              y = (T)sy[at(k, c)];
              bb = (T)sb[at(k, c)];
            }
            wu_fold(x, y, bb, lc, bnd, (uint32_t)k, true, acc, rare);
          }
          const bool rare_any = __any_sync(kFull, rare);
          if (rare_any) {  // exact reference fold, pooled the same way
            acc.uL = -T(INFINITY);
            acc.uR = T(INFINITY);
            acc.oL = acc.oR = acc.par = kNone;
            for (int k = lane; k < i; k += 32) {
              T x, y, bb;
              if (k < 4) {
                box_unit(k, Mc, x, y, bb);
              } else {
                x = (T)sx[at(k, c)];
                y = (T)sy[at(k, c)];
                bb = (T)sb[at(k, c)];
              }
              wu_apply(x, y, bb, lc, eps_par, eps_feas, eps_hi, (uint32_t)k, acc);
            }
          }
          const Merged<T> mg = merge_lanes(acc, rare_any);
          if (lane == c && !resolve_merged(St, mg, l, (uint32_t)i, h, cthr, eps_feas))
            alive = false;
        }
      }
    }
    if (live) {
      uint8_t st = St.st;
      if (st == 0 && (St.pos0 < 4 || St.pos1 < 4)) st = 2;
      write_result<T, P>(p, h, st, St.px, St.py, St.pos0, St.pos1, St.viol, St.wu);
    }
    __syncwarp();  // the tile is rewritten by the next group
    g = (int64_t)__shfl_sync(kFull, ticket, 0) + TW;
  }
  if (lane == 0) {
    __threadfence();
    const uint32_t t = atomicAdd(p.counter + 1, 1u);
    if (t == (uint32_t)p.total_warps - 1) {
      p.counter[0] = 0;
      p.counter[1] = 0;
    }
  }
}

// ---------------------------------------------------------------------------
// Large LPs: one CTA (THREADS threads) per LP, the LP resident in shared
// memory in its ORIGINAL order (ax, ay, b, perm: 14 B per constraint in fp32,
// so two m = 8192 LPs fit an SM and one CTA's event latency hides behind the
// other's work). Per LP:
//   * warp 0 stages the raw segments with 1D bulk TMA (contiguous in HBM);
//   * positions are read through the staged permutation (position k >= 4 is
//     element perm[k-4]; 0..3 are the box constants);
//   * the violation test sweeps THREADS positions per step (warp ballots
//     through a double-buffered shared array: one barrier per step, first
//     violated position found with one more ballot);
//   * a violation's 1D re-solve deals the prefix round-robin over ALL threads
//     (the reference's balanced deal with the CTA as the block,
//     batch.hpp:219-240), folded branch-free (wu_fold), merged with REDUX per
//     warp and once more across the warps' results;
//   * every thread resolves the event redundantly (identical inputs and
//     operations), so the new optimum needs no broadcast.
// Warp 0 keeps the next LP's ticket and header one LP ahead. The class's LPs
// come sorted by decreasing m (LPT). LPs larger than the launch's capacity,
// or outside the fast path's range, are solved by warp 0 with
// solve_exact_global.
constexpr int kCtaMaxWarps = 16;

template <typename T>
struct CtaShared {
  uint64_t bar;
  Header<T> hdr;
  uint32_t bal[2][kCtaMaxWarps];   // per-warp ballots, double-buffered by step
  T vL[kCtaMaxWarps], vR[kCtaMaxWarps];  // per-warp merged interval endpoints
  uint32_t oL[kCtaMaxWarps], oR[kCtaMaxWarps], par[kCtaMaxWarps];
  uint32_t redk[kCtaMaxWarps][3];  // per-warp pmax / |a| bound words
};

// S: the staged (stored) scalar type, T: the arithmetic's.
template <typename T, typename P, typename S = T>
struct CtaBuffers {
  static __host__ __device__ size_t head() { return (sizeof(CtaShared<T>) + 127) & ~size_t(127); }
  static __host__ __device__ size_t bytes(int64_t cap) {
    return head() + (3 * sizeof(S) + sizeof(P)) * (size_t)cap;
  }
};

template <typename T, typename S = T>
__device__ __forceinline__ Header<T> unpack_header_cap(uint32_t w, int64_t lp, int64_t cap,
                                                       bool& fits) {
  constexpr int WT = sizeof(S) / 4;
  Header<T> h;
  h.lp = lp;
  h.m = (int32_t)__shfl_sync(kFull, w, 0);
  h.off = (int64_t)(((uint64_t)__shfl_sync(kFull, w, 2) << 32) | __shfl_sync(kFull, w, 1));
  const int64_t o1 = (int64_t)(((uint64_t)__shfl_sync(kFull, w, 4) << 32) | __shfl_sync(kFull, w, 3));
  h.cx = (T)word_scalar<S>(w, 5);
  h.cy = (T)word_scalar<S>(w, 5 + WT);
  h.M = (T)word_scalar<S>(w, 5 + 2 * WT);
  const int64_t cap8 = ((int64_t)h.m + 7) & ~int64_t(7);
  h.ok = h.m >= 0 && (h.off & 7) == 0 && o1 - h.off >= cap8;
  fits = h.ok && h.m <= cap;
  return h;
}

template <typename T, typename P, int THREADS, typename S = T>
__global__ void __launch_bounds__(THREADS) k_solve_cta(const __grid_constant__ KParams p, int32_t cap) {
  static_assert(sizeof(T) == 4 || sizeof(T) == 8, "scalar");
  constexpr int W = THREADS / 32;
  static_assert(W <= kCtaMaxWarps, "warps per CTA");
  extern __shared__ __align__(128) unsigned char smem[];
  CtaShared<T>& sh = *reinterpret_cast<CtaShared<T>*>(smem);
  S* rax = reinterpret_cast<S*>(smem + CtaBuffers<T, P, S>::head());
  S* ray = rax + cap;
  S* rb = ray + cap;
  P* rperm = reinterpret_cast<P*>(rb + cap);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int32_t* list;
  int64_t n_list;
  resolve_list(p, list, n_list);
  const T eps_par = Eps<T>::par(p);
  const T eps_feas = Eps<T>::feas(p);
  const T eps_hi = Eps<T>::hi(p);
  const int64_t G = gridDim.x;
  auto lp_of = [&](int64_t t) -> int64_t { return t < n_list ? (list ? (int64_t)list[t] : t) : -1; };
  // considered position k: box constants for k < 4, else staged element perm[k-4]
  auto pos = [&](int k, T M, T& x, T& y, T& bb) {
    const bool box = k < 4;
    const uint32_t o = rperm[box ? 0 : k - 4];
    x = box ? (k == 0 ? T(1) : (k == 1 ? T(-1) : T(0))) : (T)rax[o];
    y = box ? (k == 2 ? T(1) : (k == 3 ? T(-1) : T(0))) : (T)ray[o];
    bb = box ? M : (T)rb[o];
  };
  // warp 0's pipeline registers: the next LP's header words and ticket
  uint32_t hwN = 0, ticket = 0;
  int64_t lpN = -1;
  uint64_t policy = 0;
  if (wid == 0) {
    policy = policy_evict_first();
    lpN = lp_of(blockIdx.x);
    hwN = load_header_word<S>(p, lpN, lane);
    ticket = atomic_add_if(p.counter, lane == 0, p.pk.zero);
    if (lane == 0) mbar_init(&sh.bar, 1);
  }
  uint32_t phase = 0;
  int step = 0;  // test steps so far (selects the ballot buffer)
  while (true) {
    // ---- warp 0: stage the LP (header loaded an LP ago) -------------------
    if (wid == 0) {
      bool fits;
      const Header<T> hn = unpack_header_cap<T, S>(hwN, lpN, cap, fits);
      if (lane == 0) {
        sh.hdr = hn;
        if (hn.lp >= 0) {
          const uint32_t bt = fits ? round16((uint32_t)hn.m * sizeof(S)) : 0u;
          const uint32_t bp = fits ? round16((uint32_t)hn.m * sizeof(P)) : 0u;
          mbar_arrive_expect_tx(&sh.bar, 3 * bt + bp);
          if (bt) {
            bulk_g2s(rax, static_cast<const S*>(p.ax) + hn.off, bt, &sh.bar, policy);
            bulk_g2s(ray, static_cast<const S*>(p.ay) + hn.off, bt, &sh.bar, policy);
            bulk_g2s(rb, static_cast<const S*>(p.b) + hn.off, bt, &sh.bar, policy);
            bulk_g2s(rperm, static_cast<const P*>(p.perm) + hn.off, bp, &sh.bar, policy);
          }
        }
      }
      lpN = lp_of((int64_t)__shfl_sync(kFull, ticket, 0) + G);
      hwN = load_header_word<S>(p, lpN, lane);
      ticket = atomic_add_if(p.counter, lane == 0, p.pk.zero);
    }
    __syncthreads();  // header visible (and the previous LP's reads are done)
    const Header<T> h = sh.hdr;
    if (h.lp < 0) break;
    const int mpos = h.m + 4;
    const bool fits = h.ok && h.m <= cap;
    mbar_wait(&sh.bar, phase);
    phase ^= 1u;
    // ---- validate the permutation, bound |a| (original order, contiguous) -
    uint32_t pmax = 0;
    decltype(float_bits(T(0))) sbits = float_bits(T(1));  // the box's |a|
    if (fits) {
      for (int i = tid; i < h.m; i += THREADS) {
        pmax = max(pmax, (uint32_t)rperm[i]);
        sbits = max(sbits, float_bits(fabs((T)rax[i]) + fabs((T)ray[i])));
      }
    } else if (h.ok) {
      const P* gperm = static_cast<const P*>(p.perm) + h.off;
      for (int i = tid; i < h.m; i += THREADS) pmax = max(pmax, (uint32_t)gperm[i]);
    }
    pmax = __reduce_max_sync(kFull, pmax);
    const auto sb_w = reduce_max_bits(sbits);
    if (lane == 0) {
      sh.redk[wid][0] = pmax;
      sh.redk[wid][1] = (uint32_t)((unsigned long long)sb_w >> (sizeof(T) == 8 ? 32 : 0));
      sh.redk[wid][2] = (uint32_t)(unsigned long long)sb_w;
    }
    __syncthreads();
    uint32_t pm_all;
    decltype(float_bits(T(0))) sb_all;
    {
      pm_all = __reduce_max_sync(kFull, lane < W ? sh.redk[lane][0] : 0u);
      if constexpr (sizeof(T) == 8) {
        const unsigned long long v =
            lane < W ? (((unsigned long long)sh.redk[lane][1] << 32) | sh.redk[lane][2]) : 0ull;
        sb_all = reduce_max_bits(v);
      } else {
        sb_all = __reduce_max_sync(kFull, lane < W ? sh.redk[lane][2] : 0u);
      }
    }
    const bool bad = !h.ok || (h.m > 0 && pm_all >= (uint32_t)h.m);
    const T m_all = float_from_bits<T>(sb_all);
    const bool wild = !(m_all < Limits<T>::kBig) || !(fabs(h.M) < T(INFINITY)) || !fits;
    const T lpbnd = fmax(fmax(m_all, Limits<T>::kSmall) * eps_hi, FastDiv<T>::kDLo);
    LPState<T> St;
    lp_init(St, h);
    St.st = bad ? 255 : 0;
    const T cthr = eps_par * sqrt(h.cx * h.cx + h.cy * h.cy);
    bool need_exact = !bad && wild;
    // ---- sweep (serial.hpp:168-186) ----------------------------------------
    int start = 4;  // first position to test
    bool running = !bad && !wild;
    while (running) {
      int pi = -1;
      for (int base = start & ~(THREADS - 1); base < mpos; base += THREADS) {
        const int P_ = base + tid;
        bool v = false;
        if (P_ >= start && P_ < mpos) {
          T x, y, bb;
          pos(P_, h.M, x, y, bb);
          v = !satisfied(x, y, bb, St.px, St.py, eps_feas);
        }
        const uint32_t bm = __ballot_sync(kFull, v);
        uint32_t* bal = sh.bal[step & 1];
        ++step;
        if (lane == 0) bal[wid] = bm;
        __syncthreads();
        const uint32_t wb = lane < W ? bal[lane] : 0u;
        const uint32_t nz = __ballot_sync(kFull, wb != 0u);
        if (nz) {
          const int w = __ffs(nz) - 1;
          pi = base + 32 * w + __ffs(__shfl_sync(kFull, wb, w)) - 1;
          break;
        }
      }
      if (pi < 0) break;
      // ---- event at position pi ------------------------------------------
      St.viol += 1;
      St.wu += (uint32_t)pi;
      if (tid == 0) note_event(p, h.lp, (uint32_t)pi);
      T hx, hy, hb;
      pos(pi, h.M, hx, hy, hb);
      const Line<T> l = boundary_fast(hx, hy, hb);
      // The thread's units k = tid + i*THREADS, two per packed fold (k,
      // k + THREADS), owners = positions; the same range trackers as the
      // warp kernel certify the fast arithmetic against the per-LP bound.
      LineP<T> lpair;
      lpair.ox = splat2(l.ox);
      lpair.oy = splat2(l.oy);
      lpair.dx = splat2(l.dx);
      lpair.dy = splat2(l.dy);
      FoldAcc<T> fa;
      acc_init(fa);
      fa.lbv = lpbnd;
      int k = tid;
#pragma unroll 1
      for (; k + THREADS < pi; k += 2 * THREADS) {
        T x0, y0, b0, x1, y1, b1;
        pos(k, h.M, x0, y0, b0);
        pos(k + THREADS, h.M, x1, y1, b1);
        fold2s<T, false>(mk2(x0, x1), mk2(y0, y1), mk2(b0, b1), lpair, (uint32_t)k,
                         (uint32_t)(k + THREADS), true, true, fa, p.pk);
      }
      if (k < pi) {
        T x0, y0, b0;
        pos(k, h.M, x0, y0, b0);
        fold2s<T, true>(mk2(x0, x0), mk2(y0, y0), mk2(b0, b0), lpair, (uint32_t)k, kNone, true,
                        false, fa, p.pk);
      }
      Acc<T> acc;
      acc.uL = fa.uL;
      acc.uR = fa.uR;
      acc.oL = fa.oL;
      acc.oR = fa.oR;
      acc.par = kNone;
      const bool rare = !FastRange<T>::ok(fa, lpbnd);
      if (__syncthreads_or(rare)) {  // exact reference classify for every unit (rare)
        acc.uL = -T(INFINITY);
        acc.uR = T(INFINITY);
        acc.oL = acc.oR = acc.par = kNone;
        for (int k = tid; k < pi; k += THREADS) {
          T x, y, bb;
          pos(k, h.M, x, y, bb);
          wu_apply(x, y, bb, l, eps_par, eps_feas, eps_hi, (uint32_t)k, acc);
        }
      }
      const Merged<T> mw = merge_lanes(acc, true);
      if (lane == 0) {
        sh.vL[wid] = mw.uL;
        sh.vR[wid] = mw.uR;
        sh.oL[wid] = mw.oL;
        sh.oR[wid] = mw.oR;
        sh.par[wid] = mw.par;
      }
      __syncthreads();
      // Merge the warps' extremes the same way (value ties keep the smaller
      // position, as the serial fold does). The slots are rewritten only
      // after the next test step's barrier.
      Acc<T> aw;
      aw.uL = lane < W ? sh.vL[lane] : -T(INFINITY);
      aw.uR = lane < W ? sh.vR[lane] : T(INFINITY);
      aw.oL = lane < W ? sh.oL[lane] : kNone;
      aw.oR = lane < W ? sh.oR[lane] : kNone;
      aw.par = lane < W ? sh.par[lane] : kNone;
      const Merged<T> mg = merge_lanes(aw, true);
      if (!resolve_merged(St, mg, l, (uint32_t)pi, h, cthr, eps_feas)) break;
      if (!(fabs(St.px) < T(INFINITY) && fabs(St.py) < T(INFINITY))) {
        need_exact = true;
        break;
      }
      start = pi + 1;
    }
    if (need_exact) {
      if (wid == 0) solve_exact_global<T, P, S>(p, h, eps_par, eps_feas, eps_hi, St, St.viol);
    }
    if (tid == 0) {
      uint8_t st = St.st;
      if (st == 0 && (St.pos0 < 4 || St.pos1 < 4)) st = 2;
      write_result<T, P>(p, h, st, St.px, St.py, St.pos0, St.pos1, St.viol, St.wu);
    }
    fence_proxy_async_smem();  // this LP's reads before the next LP's TMA
  }
  if (tid == 0) {
    __threadfence();
    const uint32_t t = atomicAdd(p.counter + 1, 1u);
    if (t == gridDim.x - 1) {
      p.counter[0] = 0;
      p.counter[1] = 0;
    }
  }
}


// Large LPs (m above the register classes) and any other LP: one warp per
// LP straight from global memory (solve_exact_global), claimed dynamically.
template <typename T, typename P>
__global__ void __launch_bounds__(kWarpsPerCta * 32) k_solve_global(const __grid_constant__ KParams p) {
  const int lane = threadIdx.x & 31;
  const int32_t* list;
  int64_t n_list;
  resolve_list(p, list, n_list);
  const T eps_par = Eps<T>::par(p);
  const T eps_feas = Eps<T>::feas(p);
  const T eps_hi = Eps<T>::hi(p);
  int64_t j = (int64_t)blockIdx.x * kWarpsPerCta + (threadIdx.x >> 5);
  while (j < n_list) {
    Header<T> h;
    h.lp = list ? (int64_t)list[j] : j;
    h.m = p.m[h.lp];
    h.off = p.offset[h.lp];
    h.ok = h.m >= 0;
    h.cx = static_cast<const T*>(p.c)[2 * h.lp];
    h.cy = static_cast<const T*>(p.c)[2 * h.lp + 1];
    h.M = static_cast<const T*>(p.bound_m)[h.lp];
    LPState<T> S;
    lp_init(S, h);
    bool bad = !h.ok;
    if (!bad) {  // validate the permutation entries
      const P* perm = static_cast<const P*>(p.perm) + h.off;
      uint32_t pm = 0;
      for (int i = lane; i < h.m; i += 32) pm = max(pm, (uint32_t)perm[i]);
      bad = h.m > 0 && __reduce_max_sync(kFull, pm) >= (uint32_t)h.m;
    }
    if (bad) {
      S.st = 255;
    } else {
      solve_exact_global<T, P>(p, h, eps_par, eps_feas, eps_hi, S);
    }
    uint8_t st = S.st;
    if (st == 0 && (S.pos0 < 4 || S.pos1 < 4)) st = 2;
    if (lane == 0) write_result<T, P>(p, h, st, S.px, S.py, S.pos0, S.pos1, S.viol, S.wu);
    int64_t jn = 0;
    if (lane == 0) jn = (int64_t)atomicAdd(p.counter, 1u) + p.total_warps;
    j = __shfl_sync(kFull, jn, 0);
  }
  if (lane == 0) {
    __threadfence();
    const uint32_t t = atomicAdd(p.counter + 1, 1u);
    if (t == (uint32_t)p.total_warps - 1) {
      p.counter[0] = 0;
      p.counter[1] = 0;
    }
  }
}

// Size-class binning for mixed batches: class of LP j is the first register
// class whose 32*NS slots hold m+4 positions, else the large class
// (nclass - 1). Two passes: count, then scatter ids into class-contiguous
// segments of `list` (order within a class is irrelevant: LPs are
// independent).
// Branch-free: the class is the number of classes too small for m (slots
// ascend), counted over a fixed-size unrolled table (no dynamic indexing of
// the parameter array, no loop-carried branch).
constexpr int kMaxSlotClasses = 12;  // BinSpec::slots capacity (static_assert in lp2d_capi.cu)

__device__ __forceinline__ int size_class(int32_t m, const int32_t* slots, int nreg) {
  int c = 0;
#pragma unroll
  for (int k = 0; k < kMaxSlotClasses; ++k) c += (k < nreg && m + 4 > 32 * slots[k]) ? 1 : 0;
  return c;
}

constexpr int kMaxBins = 128;

struct BinSpec {
  int32_t slots[kMaxSlotClasses];
  int32_t nreg;
  int32_t lane_bins;  // > 0: class 0 is split into one bin per m in [0, lane_bins)
  int32_t cta_bins;   // > 1: the large class is split by m, largest first
  int32_t cta_lo, cta_width;
};

// Bin of an LP. Bins in list order: class 0 (one bin per m when the lane
// kernel runs it, ascending), classes 1..nreg-1 (one bin each), the large
// class (cta_bins bins of cta_width sizes, DEScending m: longest LPs first).
__device__ __forceinline__ int bin_of(int32_t m, const BinSpec& spec) {
  const int c = size_class(m, spec.slots, spec.nreg);
  const int b0 = spec.lane_bins ? spec.lane_bins : 1;
  if (c == 0) return spec.lane_bins ? min(max(m, 0), spec.lane_bins - 1) : 0;
  if (c < spec.nreg) return b0 + c - 1;
  const int base = b0 + spec.nreg - 1;
  if (spec.cta_bins <= 1) return base;
  const int q = min((max(m, spec.cta_lo) - spec.cta_lo) / spec.cta_width, spec.cta_bins - 1);
  return base + spec.cta_bins - 1 - q;
}

// Bin histogram: warp-aggregated shared-memory counts (one shared atomic
// per (warp, bin)), then one global atomic per (block, non-empty bin). The
// grid is a small multiple of the SM count, so the hot bins of a skewed size
// distribution see a few hundred global atomics, not one per warp.
__global__ void k_bin_count(int64_t n, const int32_t* m, BinSpec spec, int32_t* counts) {
  __shared__ int32_t local[kMaxBins];
  for (int i = threadIdx.x; i < kMaxBins; i += blockDim.x) local[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j0 = (int64_t)blockIdx.x * blockDim.x; j0 < n; j0 += stride) {
    const int64_t j = j0 + threadIdx.x;
    const int c = j < n ? bin_of(m[j], spec) : -1;
    const uint32_t peers = __match_any_sync(kFull, c);
    if (c >= 0 && lane == __ffs(peers) - 1) atomicAdd(&local[c], __popc(peers));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kMaxBins; i += blockDim.x)
    if (local[i]) atomicAdd(&counts[i], local[i]);
}

// Scatter of LP indices into per-bin lists. Each block owns one contiguous
// chunk of LPs: it counts its chunk per bin (warp-aggregated shared atomics),
// reserves one range per non-empty bin with a single global atomic, then
// hands out slots inside its ranges with shared atomics. Order inside a bin
// is unspecified (scheduling only; results are per LP).
__global__ void k_bin_scatter(int64_t n, const int32_t* m, BinSpec spec, const int32_t* counts,
                              int32_t* cursors, int32_t* list) {
  __shared__ int32_t base[kMaxBins];  // global bin start + this block's range
  __shared__ int32_t cnt[kMaxBins];
  const int lane = threadIdx.x & 31;
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = (int64_t)blockIdx.x * chunk, hi = min(n, lo + chunk);
  for (int i = threadIdx.x; i < kMaxBins; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  for (int64_t j0 = lo; j0 < hi; j0 += blockDim.x) {
    const int64_t j = j0 + threadIdx.x;
    const int c = j < hi ? bin_of(m[j], spec) : -1;
    const uint32_t peers = __match_any_sync(kFull, c);
    if (c >= 0 && lane == __ffs(peers) - 1) atomicAdd(&cnt[c], __popc(peers));
  }
  __syncthreads();
  if (threadIdx.x < 32) {  // exclusive prefix of the global counts, one warp
    int32_t carry = 0;
    for (int q0 = 0; q0 < kMaxBins; q0 += 32) {
      const int32_t v = counts[q0 + lane];
      int32_t x = v;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int32_t y = __shfl_up_sync(kFull, x, d);
        if (lane >= d) x += y;
      }
      base[q0 + lane] = carry + x - v;
      carry += __shfl_sync(kFull, x, 31);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kMaxBins; i += blockDim.x) {
    if (cnt[i]) base[i] += atomicAdd(&cursors[i], cnt[i]);
    cnt[i] = 0;
  }
  __syncthreads();
  for (int64_t j0 = lo; j0 < hi; j0 += blockDim.x) {
    const int64_t j = j0 + threadIdx.x;
    const int c = j < hi ? bin_of(m[j], spec) : -1;
    const uint32_t peers = __match_any_sync(kFull, c);
    const int leader = __ffs(peers) - 1;
    int32_t slot = 0;
    if (c >= 0 && lane == leader) slot = atomicAdd(&cnt[c], __popc(peers));
    slot = __shfl_sync(kFull, slot, leader) + __popc(peers & ((1u << lane) - 1u));
    if (c >= 0) list[base[c] + slot] = (int32_t)j;
  }
}

// fp32-stored batches are solved with the reference's double arithmetic
// (the fp32 configs' semantics: the reference applied to the fp32-rounded
// instance). Every float is exactly a double, so widening is exact; this is
// the staging step for the size classes without an fp32-storage kernel.
__global__ void k_widen(int64_t n, const float* __restrict__ in, double* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t n4 = n / 4;
  const float4* in4 = reinterpret_cast<const float4*>(in);
  double2* out2 = reinterpret_cast<double2*>(out);
  const bool vec = ((reinterpret_cast<uintptr_t>(in) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (vec) {
    for (int64_t i = i0; i < n4; i += stride) {
      const float4 v = __ldcs(in4 + i);
      __stcs(out2 + 2 * i, make_double2((double)v.x, (double)v.y));
      __stcs(out2 + 2 * i + 1, make_double2((double)v.z, (double)v.w));
    }
    for (int64_t i = 4 * n4 + i0; i < n; i += stride) out[i] = (double)in[i];
  } else {
    for (int64_t i = i0; i < n; i += stride) out[i] = (double)in[i];
  }
}

// K1: device Fisher-Yates (serial.hpp:138-146), one thread per LP, in place.
template <typename P>
__global__ void k_shuffle(int64_t n, const int32_t* m, const int64_t* offset,
                          const uint64_t* seeds, P* perm) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int32_t mj = m[j];
  P* o = perm + offset[j];
  for (int32_t i = 0; i < mj; ++i) o[i] = (P)i;
  Xoshiro r(seeds[j]);
  for (int64_t i = mj; i > 1; --i) {
    const uint64_t q = r.below((uint64_t)i);
    const P tmp = o[i - 1];
    o[i - 1] = o[q];
    o[q] = tmp;
  }
}

// Permutations from seeds inside a solve (lp2d_batch_soa::perm_from_seed):
// LP j's order is shuffle(m[j], derive_seed(seed, mul * (first + j) + add))
// (serial.hpp:138-146, rng.hpp:64-68; integer-only, so bit-identical to the
// host). One thread per LP; the array is built in the thread's shared-memory
// slice (ps entries, ps >= m) and streamed out in 16-byte vectors (segments
// are 8-element aligned and padded, the layout contract); LPs larger than ps
// shuffle in place in global memory.
__device__ __forceinline__ uint64_t derive_seed_dev(uint64_t base, uint64_t stream);

template <typename P>
__global__ void k_shuffle_seeded(int64_t n, const int32_t* m, const int64_t* offset, uint64_t seed,
                                 int64_t first, int32_t mul, int32_t add, P* perm, int32_t ps,
                                 int32_t big_lo, int32_t big_hi) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int32_t mj = m[j];
  if (mj > big_lo && mj <= big_hi) return;  // k_shuffle_seeded_big's
  P* g = perm + offset[j];
  Xoshiro r(derive_seed_dev(seed, (uint64_t)((int64_t)mul * (first + j) + add)));
  const bool in_smem = mj <= ps;
  P* o = in_smem ? reinterpret_cast<P*>(smem) + (size_t)threadIdx.x * ps : g;
  for (int32_t i = 0; i < mj; ++i) o[i] = (P)i;
  for (int64_t i = mj; i > 1; --i) {
    const uint64_t q = r.below((uint64_t)i);
    const P tmp = o[i - 1];
    o[i - 1] = o[q];
    o[q] = tmp;
  }
  if (in_smem) {
    constexpr int V = 16 / (int)sizeof(P);
    const uint4* src = reinterpret_cast<const uint4*>(o);
    uint4* dst = reinterpret_cast<uint4*>(g);
    for (int32_t v = 0; v < (mj + V - 1) / V; ++v) dst[v] = src[v];
  }
}

// LPs with big_lo < m <= big_hi: one CTA per LP (grid-stride over the
// batch), the whole permutation in shared memory. Fisher-Yates is one serial
// chain: thread 0 runs it against shared memory (no L2 round trip per swap),
// the other threads fill the identity and stream the result out. (Drawing
// the generator's raw outputs in batches ahead of the swap loop measured
// slower.)
template <typename P>
__global__ void __launch_bounds__(64) k_shuffle_seeded_big(int64_t n, const int32_t* m,
                                                           const int64_t* offset, uint64_t seed,
                                                           int64_t first, int32_t mul, int32_t add,
                                                           P* perm, int32_t big_lo, int32_t big_hi) {
  extern __shared__ __align__(128) unsigned char smem[];
  P* o = reinterpret_cast<P*>(smem);
  for (int64_t j = blockIdx.x; j < n; j += gridDim.x) {
    const int32_t mj = m[j];
    if (mj <= big_lo || mj > big_hi) continue;
    for (int32_t i = threadIdx.x; i < mj; i += blockDim.x) o[i] = (P)i;
    __syncthreads();
    if (threadIdx.x == 0) {
      Xoshiro r(derive_seed_dev(seed, (uint64_t)((int64_t)mul * (first + j) + add)));
      for (int64_t i = mj; i > 1; --i) {
        const uint64_t q = r.below((uint64_t)i);
        const P tmp = o[i - 1];
        o[i - 1] = o[q];
        o[q] = tmp;
      }
    }
    __syncthreads();
    constexpr int V = 16 / (int)sizeof(P);
    const uint4* src = reinterpret_cast<const uint4*>(o);
    uint4* dst = reinterpret_cast<uint4*>(perm + offset[j]);
    for (int32_t v = threadIdx.x; v < (mj + V - 1) / V; v += blockDim.x) dst[v] = src[v];
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Device-side instance synthesis: generate.hpp:60-91
// (feasible_random, infeasible) plus the builder's unbounded kind, LP j of
// global index g = first + j seeded derive_seed(seed, 2g) and its insertion
// order shuffle(m, derive_seed(seed, 2g+1)) — lp2d::gen_mixed streams,
// generate.hpp:174-189. Integer parts (seeds, draws, permutations) are
// bit-identical to the host generator; cos/sin are CUDA's (within an ulp or
// two of glibc's), so parity of a solve over a device-generated batch is
// checked against the oracle on the DOWNLOADED instance. One thread per LP
// (the per-LP draw stream is sequential); scalars stored as T.
__device__ __forceinline__ uint64_t derive_seed_dev(uint64_t base, uint64_t stream) {
  uint64_t st = base ^ (0x9e3779b97f4a7c15ull * (stream + 1));  // rng.hpp:64-68
  splitmix64(st);
  return splitmix64(st);
}

__device__ __forceinline__ double unit_dev(Xoshiro& r) {  // rng.hpp:39-41
  return (double)(r.next() >> 11) * 0x1.0p-53;
}

template <typename T, typename P>
__global__ void k_generate(int64_t n, int64_t first, uint64_t seed, const int32_t* m,
                           const int64_t* offset, const uint8_t* kind, double margin,
                           double bscale, T* ax, T* ay, T* b, P* perm, T* c, T* bound_m) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  constexpr double kTwoPi = 6.283185307179586;
  constexpr double kPi = 3.141592653589793;
  constexpr double kBound = 1e7;  // serial.hpp:26 default bound_m
  const uint64_t g = (uint64_t)(first + j);
  const int32_t mj = m[j];
  const int64_t o = offset[j];
  const int kd = kind ? (int)kind[j] : 0;
  Xoshiro r(derive_seed_dev(seed, 2 * g));
  // feasible_random core (generate.hpp:60-79) over mf constraints
  const int64_t mf = (kd == 1 && mj >= 1) ? mj - 1 : mj;
  const double phi = kTwoPi * unit_dev(r);
  c[2 * j] = (T)cos(phi);
  c[2 * j + 1] = (T)sin(phi);
  const double half = kBound / 2.0;
  const double ix = -half + (half - -half) * unit_dev(r);  // rng.hpp:42 in_range
  const double iy = -half + (half - -half) * unit_dev(r);
  for (int64_t k = 0; k < mf; ++k) {
    double theta = kTwoPi * unit_dev(r);
    if (kd == 3)  // builder-defined unbounded kind: theta in (phi + pi) +- pi/3
      theta = phi + kPi + (theta / kTwoPi * 2.0 - 1.0) * (kPi / 3.0);
    const double a0 = cos(theta), a1 = sin(theta);
    const double slack = margin * (1.0 + 9.0 * unit_dev(r));
    ax[o + k] = (T)a0;
    ay[o + k] = (T)a1;
    b[o + k] = (T)(((a0 * ix + a1 * iy) + slack) * bscale);
  }
  if (kd == 1 && mj >= 1) {  // generate.hpp:81-91: one constraint excluding the box
    const double theta = kTwoPi * unit_dev(r);
    const double a0 = cos(theta), a1 = sin(theta);
    const double box_min = -(fabs(a0) + fabs(a1)) * kBound;
    ax[o + mj - 1] = (T)a0;
    ay[o + mj - 1] = (T)a1;
    b[o + mj - 1] = (T)((box_min - 1.0) * bscale);
  }
  bound_m[j] = (T)(kBound * bscale);
  if (perm) {  // serial.hpp:138-146 shuffle
    P* q = perm + o;
    for (int32_t i = 0; i < mj; ++i) q[i] = (P)i;
    Xoshiro s(derive_seed_dev(seed, 2 * g + 1));
    for (int64_t i = mj; i > 1; --i) {
      const uint64_t t = s.below((uint64_t)i);
      const P tmp = q[i - 1];
      q[i - 1] = q[t];
      q[t] = tmp;
    }
  }
}

}  // namespace lp2d_b200

#include "lp2d_warp.cuh"
#include "lp2d_fx.cuh"
#include "lp2d_fs.cuh"
#include "lp2d_grp.cuh"
