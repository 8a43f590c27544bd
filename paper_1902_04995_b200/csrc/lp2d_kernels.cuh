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

#include "lp2d_device.cuh"

namespace lp2d_b200 {

constexpr int kWarpsPerCta = 4;

struct KParams {
  int64_t n_list;        // LPs this launch solves
  const int32_t* list;   // LP ids (nullptr: 0..n_list-1)
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
  double eps_par, eps_feas, eps_hi;
  int32_t total_warps;
};

__host__ __device__ constexpr uint32_t round16(uint32_t x) {
  return (x + 15u) & ~15u;
}

template <typename T, typename P, int NSLOT>
struct WarpLayout {
  static constexpr int kCap = 32 * NSLOT;
  static constexpr uint32_t kArr = round16(kCap * sizeof(T));
  static constexpr uint32_t kPerm = round16(kCap * sizeof(P));
  static constexpr uint32_t kBuf = 3 * kArr + kPerm;  // per warp
  static constexpr uint32_t kSmem = kWarpsPerCta * kBuf + kWarpsPerCta * 8;
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

template <typename T, typename P, int NSLOT>
__device__ __forceinline__ void issue_lp(const KParams& p, int64_t j,
                                         unsigned char* buf, uint64_t* bar,
                                         uint64_t policy, Header<T>& h) {
  using L = WarpLayout<T, P, NSLOT>;
  const int64_t lp = p.list ? (int64_t)p.list[j] : j;
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

template <typename T, typename P, int NSLOT>
__global__ void __launch_bounds__(kWarpsPerCta * 32)
    k_solve_warp(const KParams p) {
  using L = WarpLayout<T, P, NSLOT>;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int wic = threadIdx.x >> 5;
  unsigned char* buf = smem + wic * L::kBuf;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kWarpsPerCta * L::kBuf) + wic;
  const T* sax = reinterpret_cast<const T*>(buf);
  const T* say = reinterpret_cast<const T*>(buf + L::kArr);
  const T* sb = reinterpret_cast<const T*>(buf + 2 * L::kArr);
  const P* sperm = reinterpret_cast<const P*>(buf + 3 * L::kArr);

  const T eps_par = (T)p.eps_par;
  const T eps_feas = (T)p.eps_feas;
  const T eps_hi = (T)p.eps_hi;
  const uint64_t policy = policy_evict_first();

  if (lane == 0) mbar_init(bar, 1);
  __syncwarp();

  uint32_t phase = 0;
  int64_t j = (int64_t)blockIdx.x * kWarpsPerCta + wic;
  Header<T> hn{};
  if (lane == 0 && j < p.n_list) issue_lp<T, P, NSLOT>(p, j, buf, bar, policy, hn);

  // Box constraint folded by this lane at every event (positions 0..3,
  // serial.hpp:47-52); lanes 4..31 duplicate one of them harmlessly.
  const int bk = lane & 3;
  const T bax = bk == 0 ? T(1) : (bk == 1 ? T(-1) : T(0));
  const T bay = bk == 2 ? T(1) : (bk == 3 ? T(-1) : T(0));

  while (j < p.n_list) {
    const Header<T> h = bcast(hn);
    mbar_wait(bar, phase);
    phase ^= 1u;

    // ---- gather the LP into registers in insertion order ------------------
    T rax[NSLOT], ray[NSLOT], rb[NSLOT];
    bool bad = !h.ok;
    const int mj = h.ok ? h.m : 0;
#pragma unroll
    for (int s = 0; s < NSLOT; ++s) {
      const int k = 32 * s + lane;
      T vax = T(0), vay = T(0), vb = T(0);
      if (k < mj) {
        uint32_t o = sperm[k];
        if (o >= (uint32_t)mj) {
          bad = true;
          o = 0;
        }
        vax = sax[o];
        vay = say[o];
        vb = sb[o];
      }
      rax[s] = vax;
      ray[s] = vay;
      rb[s] = vb;
    }
    bad = __any_sync(kFull, bad);
    __syncwarp();
    fence_proxy_async_smem();

    // ---- claim + prefetch the next LP (overlaps this LP's solve) ----------
    int64_t jn = 0;
    if (lane == 0) jn = (int64_t)atomicAdd(p.counter, 1u) + p.total_warps;
    jn = __shfl_sync(kFull, jn, 0);
    if (lane == 0 && jn < p.n_list) issue_lp<T, P, NSLOT>(p, jn, buf, bar, policy, hn);

    // ---- solve (serial.hpp:159-188) ---------------------------------------
    const T M = h.M;
    T px = h.cx < T(0) ? -M : M;  // serial.hpp:56-58
    T py = h.cy < T(0) ? -M : M;
    uint32_t pos0 = h.cx < T(0) ? 1u : 0u;
    uint32_t pos1 = h.cy < T(0) ? 3u : 2u;
    const T cthr = eps_par * sqrt(h.cx * h.cx + h.cy * h.cy);
    uint32_t viol = 0;
    uint64_t wu = 0;
    uint8_t st = bad ? 255 : 0;
    int s = 0;
    uint32_t startmask = kFull;
    while (!bad) {
      // Speculative chunked violation test from slot s onward.
      bool ev = false;
      int f = 0;
      T hx = T(0), hy = T(0), hb = T(0);
#pragma unroll
      for (int S = 0; S < NSLOT; ++S) {
        if (S < s) continue;
        if (32 * S >= mj) break;
        const bool v = (32 * S + lane < mj) &&
                       !satisfied(rax[S], ray[S], rb[S], px, py, eps_feas);
        const uint32_t vm = __ballot_sync(kFull, v) & startmask;
        startmask = kFull;
        // Unconditional opaque copies (not a shuffle inside the branch): the
        // compiler cannot merge them into one dynamically indexed load after
        // the loop, so the slot index stays compile-time and the arrays stay
        // in registers.
        hx = opaque_copy(rax[S]);
        hy = opaque_copy(ray[S]);
        hb = opaque_copy(rb[S]);
        if (vm) {
          f = __ffs(vm) - 1;
          s = S;
          ev = true;
          break;
        }
      }
      if (!ev) break;
      hx = __shfl_sync(kFull, hx, f);
      hy = __shfl_sync(kFull, hy, f);
      hb = __shfl_sync(kFull, hb, f);

      // Violation at insertion index i: 1D LP over positions 0..i+3.
      const uint32_t i = 32u * (uint32_t)s + (uint32_t)f;
      viol += 1;
      wu += 4 + i;
      const Line<T> l = boundary_of(hx, hy, hb);
      Acc<T> acc;
      acc.uL = -T(INFINITY);
      acc.uR = T(INFINITY);
      acc.oL = acc.oR = acc.par = kNone;
      wu_apply(bax, bay, M, l, eps_par, eps_feas, eps_hi, (uint32_t)bk, acc);
#pragma unroll
      for (int S = 0; S < NSLOT; ++S) {
        if (S > s) break;
        const uint32_t k = 32u * S + lane;
        if (k < i) wu_apply(rax[S], ray[S], rb[S], l, eps_par, eps_feas, eps_hi, 4u + k, acc);
      }
      const uint32_t par = __reduce_min_sync(kFull, acc.par);
      if (par != kNone) {  // serial.hpp:97 parallel-infeasible
        st = 1;
        pos0 = 4 + i;
        pos1 = par;
        break;
      }
      T uL, nuR;
      uint32_t oL, oR;
      warp_best(acc.uL, acc.oL, uL, oL);
      warp_best(-acc.uR, acc.oR, nuR, oR);
      const T uR = -nuR;
      const T scale = fmax(fabs(uL), fabs(uR));
      if (uL > uR + feas_slack(eps_feas, scale)) {  // serial.hpp:98-101
        st = 1;
        pos0 = 4 + i;
        pos1 = oL;
        break;
      }
      const T along = h.cx * l.dx + h.cy * l.dy;
      T t;
      uint32_t own;
      if (fabs(along) <= cthr) {
        t = uL;
        own = oL;
      } else if (along > T(0)) {
        t = uR;
        own = oR;
      } else {
        t = uL;
        own = oL;
      }
      px = l.ox + t * l.dx;
      py = l.oy + t * l.dy;
      pos0 = 4 + i;
      pos1 = own;
      startmask = (f == 31) ? 0u : (kFull << (f + 1));
    }
    if (st == 0 && (pos0 < 4 || pos1 < 4)) st = 2;
    if (lane == 0) write_result<T, P>(p, h, st, px, py, pos0, pos1, viol, wu);
    j = jn;
  }

  // Self-reset of the ticket counter by the last warp to finish, so the next
  // launch on this counter slot starts from zero without a memset.
  if (lane == 0) {
    __threadfence();
    const uint32_t t = atomicAdd(p.counter + 1, 1u);
    if (t == (uint32_t)p.total_warps - 1) {
      p.counter[0] = 0;
      p.counter[1] = 0;
    }
  }
}

// Naive: thread per LP, the serial loop with global-memory gathers.
template <typename T, typename P>
__global__ void __launch_bounds__(128) k_solve_naive(const KParams p) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= p.n_list) return;
  const T eps_par = (T)p.eps_par;
  const T eps_feas = (T)p.eps_feas;
  const T eps_hi = (T)p.eps_hi;
  Header<T> h;
  h.lp = p.list ? (int64_t)p.list[j] : j;
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

}  // namespace lp2d_b200
