// lp2d_grp.cuh — K6: LANE GROUPS for the small warp classes of fp32-stored
// batches (29 <= m <= CAP). Included at the end of lp2d_kernels.cuh.
//
// A warp-per-LP kernel pays its per-event chain (detect, broadcast, line,
// fold, warp merge, resolve) once per violation of ONE LP; at m <= 188 that
// chain, not the fold, is most of the instructions (config 3: ~230 of ~360
// instructions per event, 9 events per LP). K6 splits the warp into 32/G
// groups of G lanes, each group solving its own LP, so one pass of the chain
// serves every group with a pending violation:
//   * each group's LP is staged in its own shared-memory slot in ORIGINAL
//     order (ax, ay, b as stored, the permutation), by 16-byte cp.async of
//     the contiguous segments; two slots per group, so the next LP's copy is
//     in flight while this one is solved (no permutation dependency: the
//     copy needs only the header);
//   * the sweep tests positions i .. i+G-1 of every group per step (one
//     ballot for the warp); a group whose window holds a violation takes the
//     event at its first violated position pi, the others advance by G;
//   * an event's 1D re-solve deals the positions [0, pi) round-robin over
//     the group's G lanes (the reference's balanced deal, batch.hpp:219-240,
//     with the group as the block) with wu_fold, the exact reference fold
//     (wu_apply) redone for a group whose bound could not decide a unit, and
//     the group's lanes merged by xor butterflies (owner ties to the smallest
//     position, as the reference's sequential apply_bound keeps the first);
//   * a group that finishes writes its result and takes the next LP from its
//     other slot at once (per-group tickets, claimed two LPs ahead; headers
//     loaded one LP ahead), so a warp's groups never wait for each other's LPs.
// The arithmetic is the reference's double on the exactly widened stored
// values, operation for operation (satisfied, boundary_of, classify,
// apply_bound, resolve_on_line: lp2d_device.cuh / lp2d_kernels.cuh), so the
// results are bit-identical to the reference on the stored instance.
#pragma once

namespace lp2d_b200 {

constexpr int kGrpWarps = 4;  // warps per CTA

template <typename P, int G, int CAP>
struct GrpLayout {
  static_assert(G == 4 || G == 8 || G == 16 || G == 32, "group width");
  static constexpr int kGroups = 32 / G;
  static constexpr uint32_t kArr = (uint32_t)((CAP + 3) & ~3) * 4u;                // float4 runs
  static constexpr uint32_t kPerm = ((uint32_t)(CAP * sizeof(P)) + 15u) & ~15u;   // 16-byte runs
  static constexpr uint32_t kSlot = 3 * kArr + kPerm;
  static constexpr size_t kWarpBytes = (size_t)2 * kGroups * kSlot;  // two slots per group
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}

// Butterflies over the G lanes of a group (all 32 lanes execute them; each
// group reduces its own values). best_*: value with the smallest owner among
// equal extremes (IEEE ==, so -0 ties +0 and the smaller owner keeps its own
// value — the reference's first-come apply_bound).
template <int G>
__device__ __forceinline__ void grp_best_max(double& v, uint32_t& o) {
#pragma unroll
  for (int s = G / 2; s >= 1; s >>= 1) {
    const double v2 = __shfl_xor_sync(kFull, v, s);
    const uint32_t o2 = __shfl_xor_sync(kFull, o, s);
    const bool take = (v2 > v) | ((v2 == v) & (o2 < o));
    v = take ? v2 : v;
    o = take ? o2 : o;
  }
}
template <int G>
__device__ __forceinline__ void grp_best_min(double& v, uint32_t& o) {
#pragma unroll
  for (int s = G / 2; s >= 1; s >>= 1) {
    const double v2 = __shfl_xor_sync(kFull, v, s);
    const uint32_t o2 = __shfl_xor_sync(kFull, o, s);
    const bool take = (v2 < v) | ((v2 == v) & (o2 < o));
    v = take ? v2 : v;
    o = take ? o2 : o;
  }
}
template <int G>
__device__ __forceinline__ uint32_t grp_min_u32(uint32_t v) {
#pragma unroll
  for (int s = G / 2; s >= 1; s >>= 1) v = min(v, (uint32_t)__shfl_xor_sync(kFull, v, s));
  return v;
}
template <int G>
__device__ __forceinline__ uint32_t grp_max_u32(uint32_t v) {
#pragma unroll
  for (int s = G / 2; s >= 1; s >>= 1) v = max(v, (uint32_t)__shfl_xor_sync(kFull, v, s));
  return v;
}
template <int G>
__device__ __forceinline__ unsigned long long grp_max_u64(unsigned long long v) {
#pragma unroll
  for (int s = G / 2; s >= 1; s >>= 1) {
    const unsigned long long o = __shfl_xor_sync(kFull, v, s);
    v = o > v ? o : v;
  }
  return v;
}

// Header of a group's next LP (loaded one LP ahead of its staging).
struct GrpNext {
  int64_t lp, off;
  int32_t m;
  bool ok;
  float cx, cy, M;
};

template <typename P, int G, int CAP>
__global__ void __launch_bounds__(kGrpWarps * 32, 4) k_solve_grp(const __grid_constant__ KParams p) {
  using L = GrpLayout<P, G, CAP>;
  using T = double;
  constexpr int NG = L::kGroups;
  constexpr uint32_t gbits = G == 32 ? kFull : (1u << G) - 1u;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wic = threadIdx.x >> 5;
  const int g = lane / G, r = lane % G;
  const int gl = g * G;  // the group's first lane
  unsigned char* const wb = smem + (size_t)wic * L::kWarpBytes;
  auto slot_ptr = [&](int b) { return wb + (size_t)(b * NG + g) * L::kSlot; };

  const int32_t* list;
  int64_t n_list;
  resolve_list(p, list, n_list);
  const T eps_par = Eps<T>::par(p);
  const T eps_feas = Eps<T>::feas(p);
  const T eps_hi = Eps<T>::hi(p);
  // tickets: group w takes LPs w, w + TG, w + 2 TG, then counter + 3 TG, ...
  const int64_t TG = (int64_t)p.total_warps * NG;
  const int64_t w = ((int64_t)blockIdx.x * kGrpWarps + wic) * NG + g;
  auto lp_of = [&](int64_t t) -> int64_t {
    return t < n_list ? (list ? (int64_t)list[t] : t) : -1;
  };
  auto load_hdr = [&](int64_t lp, GrpNext& q) {
    q.lp = lp;
    q.off = 0;
    q.m = 0;
    q.ok = false;
    q.cx = q.cy = q.M = 0.0f;
    if (lp >= 0) {
      const int32_t mm = p.m[lp];
      const int64_t o = p.offset[lp], o1 = p.offset[lp + 1];
      q.m = mm;
      q.off = o;
      // the layout contract (8-aligned, 8-padded segments) the 16-byte copies need
      q.ok = mm >= 0 && mm <= CAP && (o & 7) == 0 && o1 - o >= (((int64_t)mm + 7) & ~int64_t(7));
      q.cx = static_cast<const float*>(p.c)[2 * lp];
      q.cy = static_cast<const float*>(p.c)[2 * lp + 1];
      q.M = static_cast<const float*>(p.bound_m)[lp];
    }
  };
  // the group's lanes copy LP q's segments into slot b (asynchronous)
  auto stage = [&](const GrpNext& q, int b) {
    if (q.lp >= 0 && q.ok) {
      unsigned char* s = slot_ptr(b);
      const float* gx = static_cast<const float*>(p.ax) + q.off;
      const float* gy = static_cast<const float*>(p.ay) + q.off;
      const float* gb = static_cast<const float*>(p.b) + q.off;
      const int nv = (q.m + 3) >> 2;
      for (int v = r; v < nv; v += G) {
        cp_async16(s + 16 * v, gx + 4 * v);
        cp_async16(s + L::kArr + 16 * v, gy + 4 * v);
        cp_async16(s + 2 * L::kArr + 16 * v, gb + 4 * v);
      }
      const unsigned char* gp =
          reinterpret_cast<const unsigned char*>(static_cast<const P*>(p.perm) + q.off);
      const int np = (int)(((size_t)q.m * sizeof(P) + 15) / 16);
      for (int v = r; v < np; v += G) cp_async16(s + 3 * L::kArr + 16 * v, gp + 16 * v);
    }
  };

  // ---- prologue: LP w staged (slot 0), w + TG's header, w + 2 TG's id -----
  GrpNext nx, nn;
  load_hdr(lp_of(w), nx);
  stage(nx, 0);
  load_hdr(lp_of(w + TG), nn);
  int64_t lp3 = lp_of(w + 2 * TG);
  uint32_t tk_raw = (r == 0) ? atomicAdd(p.counter, 1u) : 0u;  // broadcast at the next refill

  int cur = 1;  // slot of the current LP (the first refill flips to slot 0)
  bool cur_live = false, active = false;
  Header<T> h;
  h.lp = -1;
  h.off = 0;
  h.m = 0;
  h.ok = 0;
  h.cx = h.cy = h.M = T(0);
  LPState<T> St;
  lp_init(St, h);
  T lpbnd = T(0), cthr = T(0);
  int i = 4, mpos = 4;

  for (;;) {
    // ---- refill: groups whose LP ended write it and take the staged one ----
    const bool rf = !active && (cur_live || nx.lp >= 0);
    if (__any_sync(kFull, rf)) {
      if (rf && cur_live && r == 0) {
        uint8_t st = St.st;
        if (st == 0 && (St.pos0 < 4 || St.pos1 < 4)) st = 2;
        write_result<T, P>(p, h, st, St.px, St.py, St.pos0, St.pos1, St.viol, St.wu);
      }
      if (rf) cp_async_wait_all();  // this lane's copies of the staged LP
      __syncwarp();                 // ... and the group's other lanes'
      if (rf) {
        cur ^= 1;
        h.lp = nx.lp;
        h.off = nx.off;
        h.m = nx.m;
        h.ok = nx.ok ? 1 : 0;
        h.cx = (T)nx.cx;
        h.cy = (T)nx.cy;
        h.M = (T)nx.M;
        cur_live = nx.lp >= 0;
      }
      // permutation bound and magnitude bound of the new LP
      const unsigned char* s = slot_ptr(cur);
      const float* sx = reinterpret_cast<const float*>(s);
      const float* sy = reinterpret_cast<const float*>(s + L::kArr);
      const P* sp = reinterpret_cast<const P*>(s + 3 * L::kArr);
      uint32_t pm = 0;
      unsigned long long mb = float_bits(T(1));
      if (rf && cur_live && h.ok) {
        for (int k = r; k < h.m; k += G) {
          pm = max(pm, (uint32_t)sp[k]);
          mb = max(mb, float_bits(fabs((T)sx[k]) + fabs((T)sy[k])));
        }
      }
      pm = grp_max_u32<G>(pm);
      mb = grp_max_u64<G>(mb);
      const int64_t t_next = (int64_t)__shfl_sync(kFull, tk_raw, gl) + 3 * TG;
      if (rf) {
        const bool bad = cur_live && (!h.ok || (h.m > 0 && pm >= (uint32_t)h.m));
        const T m_all = __longlong_as_double((long long)mb);
        // outside the fast path's proven range every unit is undecided, so
        // the folds are the exact reference fold for this LP
        const bool wild = !(m_all < Limits<T>::kBig) || !(fabs(h.M) < T(INFINITY));
        lpbnd = wild ? T(INFINITY)
                     : fmax(fmax(m_all, Limits<T>::kSmall) * eps_hi, FastDiv<T>::kDLo);
        lp_init(St, h);
        St.st = bad ? 255 : 0;
        cthr = eps_par * sqrt(h.cx * h.cx + h.cy * h.cy);
        i = 4;
        mpos = (h.ok ? h.m : 0) + 4;
        active = cur_live && !bad;
        // advance the group's pipeline: stage the next LP into the slot just
        // freed, load the header after it, resolve the id after that
        stage(nn, cur ^ 1);
        nx = nn;
        load_hdr(lp3, nn);
        lp3 = lp_of(t_next);
        if (r == 0) tk_raw = atomicAdd(p.counter, 1u);
      }
    }
    if (!__any_sync(kFull, active)) {
      if (!__any_sync(kFull, cur_live || nx.lp >= 0)) break;
      continue;
    }

    // ---- sweep step: every active group tests positions i .. i+G-1 ---------
    const unsigned char* s = slot_ptr(cur);
    const float* sx = reinterpret_cast<const float*>(s);
    const float* sy = reinterpret_cast<const float*>(s + L::kArr);
    const float* sb = reinterpret_cast<const float*>(s + 2 * L::kArr);
    const P* sp = reinterpret_cast<const P*>(s + 3 * L::kArr);
    const uint32_t lim = (uint32_t)max(h.m, 1) - 1u;
    const int pos = i + r;
    const bool inr = active && pos < mpos;
    T x = T(0), y = T(0), bb = T(0);
    if (inr) {
      const uint32_t o = min((uint32_t)sp[pos - 4], lim);
      x = (T)sx[o];
      y = (T)sy[o];
      bb = (T)sb[o];
    }
    const bool v = inr && !satisfied(x, y, bb, St.px, St.py, eps_feas);  // core.hpp:111-113
    const uint32_t bal = __ballot_sync(kFull, v);
    const uint32_t gv = (bal >> gl) & gbits;
    const bool ev = gv != 0;
    const int f = ev ? __ffs(gv) - 1 : 0;
    if (active && !ev) i += G;
    if (bal) {
      // ---- events: 1D LP over positions [0, pi) of each violated group ------
      const uint32_t pi = (uint32_t)(i + f);
      const int src = gl + f;
      const T hx = __shfl_sync(kFull, x, src);
      const T hy = __shfl_sync(kFull, y, src);
      const T hb = __shfl_sync(kFull, bb, src);
      if (ev) {
        St.viol += 1;
        St.wu += pi;  // considered.size() (serial.hpp:176-179)
        if (r == 0) note_event(p, h.lp, pi);
      }
      const Line<T> l = boundary_of(hx, hy, hb);
      const uint32_t pe = ev ? pi : 0u;
      const uint32_t kend = __reduce_max_sync(kFull, pe);
      Acc<T> acc;
      acc.uL = -T(INFINITY);
      acc.uR = T(INFINITY);
      acc.oL = acc.oR = acc.par = kNone;
      bool rare = false;
#pragma unroll 2
      for (uint32_t k = r; k < kend; k += G) {
        T ux, uy, ub;
        if (k < 4) {
          box_unit((int)k, h.M, ux, uy, ub);
        } else {
          const uint32_t o = min((uint32_t)sp[k - 4], lim);
          ux = (T)sx[o];
          uy = (T)sy[o];
          ub = (T)sb[o];
        }
        wu_fold(ux, uy, ub, l, lpbnd, k, k < pe, acc, rare);
      }
      const bool rare_g = ((__ballot_sync(kFull, rare) >> gl) & gbits) != 0;
      if (__any_sync(kFull, rare_g)) {
        // the exact reference fold for the groups the bound could not decide
        Acc<T> ex;
        ex.uL = -T(INFINITY);
        ex.uR = T(INFINITY);
        ex.oL = ex.oR = ex.par = kNone;
        for (uint32_t k = r; k < kend; k += G) {
          if (rare_g && k < pe) {
            T ux, uy, ub;
            if (k < 4) {
              box_unit((int)k, h.M, ux, uy, ub);
            } else {
              const uint32_t o = min((uint32_t)sp[k - 4], lim);
              ux = (T)sx[o];
              uy = (T)sy[o];
              ub = (T)sb[o];
            }
            wu_apply(ux, uy, ub, l, eps_par, eps_feas, eps_hi, k, ex);
          }
        }
        if (rare_g) acc = ex;
      }
      Merged<T> mg;
      mg.uL = acc.uL;
      mg.oL = acc.oL;
      mg.uR = acc.uR;
      mg.oR = acc.oR;
      grp_best_max<G>(mg.uL, mg.oL);
      grp_best_min<G>(mg.uR, mg.oR);
      mg.par = grp_min_u32<G>(acc.par);
      if (ev) {
        if (!resolve_merged(St, mg, l, pi, h, cthr, eps_feas)) active = false;  // serial.hpp:95-111
        i = (int)pi + 1;
      }
    }
    if (active && i >= mpos) active = false;
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

}  // namespace lp2d_b200
