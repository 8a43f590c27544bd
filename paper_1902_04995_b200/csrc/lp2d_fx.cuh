// lp2d_fx.cuh — K4: fp32-STORED batches solved with the reference's DOUBLE
// semantics (the fp32 configs). Included at the end of lp2d_kernels.cuh.
//
// The reference computes in double (core.hpp, serial.hpp); the fp32 configs
// store the instance in float (12 B per constraint in HBM), and the answer
// must be the reference's own answer on that instance: the same status,
// defining pair, violation/work-unit counts and bit-identical x, y, value.
// Plain fp32 arithmetic cannot decide the reference's comparisons for these
// workloads (coordinates ~5e6 with slacks ~1: relative margins ~1e-7, below
// fp32's 6e-8 resolution), and double arithmetic on every unit is 2-4x the
// issue cost. K4 therefore runs an fp32 FILTER whose every decision is
// CERTIFIED against the reference's double decision by an a-priori error
// bound, and falls back to the reference's double operations whenever a
// certificate fails:
//
//   * local frame: constraints are used as (a, b') with b' = b - a.s for a
//     per-LP shift s (fp32 point). b' is computed from the original b by fp32
//     error-free transformations (bshift), so |b'32 - (b - a.s)| <= u|b'| + Eb:
//     kept in registers for the register chunks and rewritten in place in the
//     staging buffer for the tail (originals re-read from L2). s starts at 0 and
//     is moved (reshift) to the current candidate point when a certificate
//     fails at an event, so coordinates near the optimum are small and fp32
//     resolves them.
//   * violation test (core.hpp:111-113): e = a.p' - b' in fp32 (p' = the
//     current optimum in the local frame, |p' - (p64 - s)| <= epp). The
//     reference violates iff D > S + eta (D = a.p64 - b exact, S = its slack,
//     |eta| <= Dr its rounding): e < -T proves "satisfied", e > Smax + T
//     proves "violated"; anything in between is re-tested exactly in double
//     with the exact optimum (rare).
//   * 1D re-solve (serial.hpp:114-122): on the violated line (fp32 local:
//     direction d = perp(a)/|a| by rsqrt, foot w of the perpendicular from s),
//     every unit's quotient q = (b' - a.w)/(a.d) is within
//     E(q) = (Kn + Ka|q|)/|a.d| of the reference's sigma64 - tau (tau a per-
//     event constant). The chosen endpoint's side is made the "max" side by
//     flipping d; per lane the fold keeps the top two quotients of that side
//     (with the owner slot of the first), the min of the other side and the
//     min |a.d|. The event is certified when (1) min |a.d| exceeds the
//     parallel/sign bound, (2) the top quotient beats the runner-up by more
//     than their error bounds (so the reference's argmax, i.e. the owner, is
//     ours and unique), (3) the interval is provably non-empty. Then the new
//     optimum is known EXACTLY as "the intersection of lines (pi, owner)" and
//     approximately as p' = w + q1 d; its double value is computed lazily
//     with the reference's operations (fx_exact_point) only when an exact
//     test needs it and at the end of the LP. A failed certificate reshifts
//     once to the candidate point and refolds; a second failure (or an
//     uncertain objective side, or an empty interval) runs the reference's
//     double fold for that event (fold_exact_global on the widened values).
//
// Exactness therefore rests on the error bounds (DESIGN.md §4 lists the
// error sources and constants); the constants are deliberately loose
// (factors 1.1-2). The bound model is not machine-checked: it is validated by
// the GPU parity tests against the unmodified reference (full-size c2 and c3,
// a heavy-tailed c4 subset, adversarial insertion orders, every size-class
// edge, K4 and K5 for every class), all bit-identical.
#pragma once

#ifndef LP2D_FX_COLD
#define LP2D_FX_COLD __forceinline__  // cold paths inline (measured faster than calls)
#endif

namespace lp2d_b200 {

#ifndef LP2D_FX_EXACT_BATCH
#define LP2D_FX_EXACT_BATCH 1
#endif
#ifndef LP2D_FX_SHIFT_BATCH
#define LP2D_FX_SHIFT_BATCH 2
#endif
// Loads in flight per lane in the exact fold and in a reshift's staged
// rewrite. Small on purpose: these paths are inlined (calls measured slower)
// and their unrolled bodies crowd the hot loops out of the instruction cache
// (B200, 8 -> 1/2: c2 0.231 -> 0.219 ms, c3 0.809 -> 0.698 ms, c4 0.804 ->
// 0.758 ms).
constexpr int kFxExactBatch = LP2D_FX_EXACT_BATCH;
constexpr int kFxShiftBatch = LP2D_FX_SHIFT_BATCH;
constexpr float kU32 = 0x1p-24f;   // fp32 unit roundoff
constexpr float kU64 = 0x1p-53f;   // fp64 unit roundoff (a normal float)
constexpr float kRho = 0x1p-21f;   // MUFU rcp/rsqrt relative error bound (PTX: <= 1 ulp / 2^-22.9)

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// Warp max of floats with NaN propagation (redux .NaN form): a NaN anywhere
// in the LP must reach the range guard.
__device__ __forceinline__ float warp_max_nan_f(float v) {
  float r;
  asm volatile("redux.sync.max.NaN.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}

// K4 path counters (debug/measurement builds of the statistics, see
// lp2dgpu_fx_stats): events, certified first pass, reshifts, exact events,
// uncertain tests, lazy exact points, whole-LP exact solves.
enum { kFxEvents, kFxCert1, kFxReshift, kFxExact, kFxTestFlag, kFxLazy, kFxWild, kFxNStat = 8 };
__device__ __forceinline__ void fx_count(const KParams& p, int which, int lane) {
  if (p.fxstat && lane == 0) atomicAdd(p.fxstat + which, 1ull);
}

__device__ __forceinline__ float rsqrt_approx(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// b - ax*sx - ay*sy rounded to float, through error-free transformations
// (TwoProduct by FMA, TwoSum): the exact value is v + ev + et - e1 - e2 with
// all five terms exact; only the final sum of the small terms and the last
// addition round, so |result - (b - a.s)| <= u|result| + 2u^2(|b| + 2|a.s|).
__device__ __forceinline__ float bshift(float ax, float ay, float b, float sx, float sy) {
  const float p1 = ax * sx, e1 = fmaf(ax, sx, -p1);
  const float p2 = ay * sy, e2 = fmaf(ay, sy, -p2);
  const float t = b - p1, z = t - b, et = (b - (t - z)) + (-p1 - z);
  const float v = t - p2, z2 = v - t, ev = (t - (v - z2)) + (-p2 - z2);
  return v + ((et + ev) - (e1 + e2));
}

// bshift of two values at once (packed FFMA2/FADD2; every packed lane is the
// scalar IEEE operation).
__device__ __forceinline__ Pair<float> bshift2(Pair<float> ax, Pair<float> ay, Pair<float> b,
                                               Pair<float> sx, Pair<float> sy,
                                               const PairConsts& k) {
  const Pair<float> p1 = mul2(ax, sx, k), e1 = fma2(ax, sx, sub2(konst2(k.nz), p1));
  const Pair<float> p2 = mul2(ay, sy, k), e2 = fma2(ay, sy, sub2(konst2(k.nz), p2));
  const Pair<float> t = sub2(b, p1), z = sub2(t, b);
  const Pair<float> et = add2(sub2(b, sub2(t, z)), sub2(sub2(konst2(k.nz), p1), z));
  const Pair<float> v = sub2(t, p2), z2 = sub2(v, t);
  const Pair<float> ev = add2(sub2(t, sub2(v, z2)), sub2(sub2(konst2(k.nz), p2), z2));
  return add2(v, sub2(add2(et, ev), add2(e1, e2)));
}

// Original (unshifted) constraint at considered position pos, widened to
// double, straight from global memory (exact paths only).
template <typename P>
__device__ __forceinline__ void fx_orig(const KParams& p, int64_t off, uint32_t pos, double M,
                                        double& x, double& y, double& b) {
  if (pos < 4) {
    x = pos == 0 ? 1.0 : (pos == 1 ? -1.0 : 0.0);  // serial.hpp:47-52
    y = pos == 2 ? 1.0 : (pos == 3 ? -1.0 : 0.0);
    b = M;
  } else {
    const uint32_t o = static_cast<const P*>(p.perm)[off + pos - 4];
    x = static_cast<const float*>(p.ax)[off + o];
    y = static_cast<const float*>(p.ay)[off + o];
    b = static_cast<const float*>(p.b)[off + o];
  }
}

// The reference's optimum after the event at position p0 whose chosen
// endpoint is owned by position p1: boundary_of (core.hpp:70-75), the owner's
// classify quotient (core.hpp:106) and origin + t*dir (serial.hpp:109) — the
// same double operations in the same order, hence the same bits.
__device__ LP2D_FX_COLD void fx_exact_point(double hx, double hy, double hb, double ox,
                                            double oy, double ob, double& px, double& py) {
  // (all arguments are floats widened exactly)
  const Line<double> l = boundary_of(hx, hy, hb);
  const double along = ox * l.dx + oy * l.dy;
  const double t = (ob - (ox * l.ox + oy * l.oy)) / along;
  px = l.ox + t * l.dx;
  py = l.oy + t * l.dy;
}

// Fold accumulator of one lane, with PER-UNIT error bounds: every unit's
// quotient q lies within e = (Kn + Ka |q|)/|a.d| of the reference's sigma64 -
// tau, so it is represented by [lo, hi] = [q - e, q + e]. Chosen side: the
// two largest hi (and the lo and owner slot of the first); other side: the
// smallest lo; all units: min |a.d| (parallel / sign certificate).
struct FxAcc {
  float h1, l1, h2, rl, mal;
  uint32_t own;
};

__device__ __forceinline__ void fx_acc_init(FxAcc& a) {
  a.h1 = -INFINITY;
  a.l1 = -INFINITY;
  a.h2 = -INFINITY;
  a.rl = INFINITY;
  a.mal = INFINITY;
  a.own = kNone;
}

// Two work units (classify, core.hpp:96-109, in the local flipped frame):
// alm = -(a.d'), nmn = -(b' - a.w) = a.w - b' (nb = -b'), q = nmn / alm.
// Chosen side (d' flipped so it is the max side): a.d' < 0  <=>  alm > 0.
// kn/ka: the event's numerator error and the LP's quotient error factor
// (pre-scaled by 1 + 2^-10 for the rounding of e itself).
template <bool MASKED>
__device__ __forceinline__ void fx_fold2(Pair<float> ax, Pair<float> ay, Pair<float> nb,
                                         Pair<float> ndx, Pair<float> ndy, Pair<float> wx,
                                         Pair<float> wy, float kn, float ka, uint32_t s0,
                                         uint32_t s1, bool act0, bool act1, FxAcc& a,
                                         const PairConsts& k) {
  const Pair<float> alm = fma2(ax, ndx, mul2(ay, ndy, k));
  const Pair<float> nmn = fma2(ax, wx, fma2(ay, wy, nb));
  const float r0 = rcp_approx(lo2(alm)), r1 = rcp_approx(hi2(alm));
  const Pair<float> q = mul2(nmn, mk2(r0, r1), k);
  const float a0 = lo2(alm), a1 = hi2(alm), q0 = lo2(q), q1 = hi2(q);
  const float e0 = fmaf(ka, fabsf(q0), kn) * fabsf(r0);
  const float e1 = fmaf(ka, fabsf(q1), kn) * fabsf(r1);
  const Pair<float> E = mk2(e0, e1);
  const Pair<float> hi = add2(q, E), lo = sub2(q, E);
  const float h0 = lo2(hi), hh1 = hi2(hi), w0 = lo2(lo), w1 = hi2(lo);
  const bool l0 = a0 > 0.0f, l1 = a1 > 0.0f;
  float hL0, hL1, lR0, lR1, m0 = a0, m1 = a1;
  if constexpr (MASKED) {
    hL0 = (act0 & l0) ? h0 : -INFINITY;
    hL1 = (act1 & l1) ? hh1 : -INFINITY;
    lR0 = (act0 & (a0 < 0.0f)) ? w0 : INFINITY;
    lR1 = (act1 & (a1 < 0.0f)) ? w1 : INFINITY;
    m0 = act0 ? m0 : INFINITY;
    m1 = act1 ? m1 : INFINITY;
  } else {
    hL0 = l0 ? h0 : -INFINITY;
    hL1 = l1 ? hh1 : -INFINITY;
    lR0 = (a0 < 0.0f) ? w0 : INFINITY;
    lR1 = (a1 < 0.0f) ? w1 : INFINITY;
  }
  a.mal = min3_abs(a.mal, m0, m1);  // NaN-propagating: a NaN unit fails the certificate
  float rr;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(rr) : "f"(a.rl), "f"(lR0), "f"(lR1));
  a.rl = rr;
  const float mx = fmaxf(hL0, hL1), mn = fminf(hL0, hL1);
  const bool first = hL0 >= hL1;
  float h2;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(h2) : "f"(a.h2), "f"(fminf(a.h1, mx)), "f"(mn));
  a.h2 = h2;
  const bool up = mx > a.h1;
  a.own = up ? (first ? s0 : s1) : a.own;
  a.l1 = up ? (first ? w0 : w1) : a.l1;
  a.h1 = fmaxf(a.h1, mx);
}

// Per-LP constants of the certificates (DESIGN.md §3 derives every bound).
struct FxLP {
  float A;     // max |a_x|,|a_y| over the LP (>= 1, the box)
  float B;     // max |b| (incl. M)
  float Ka;    // quotient error per unit |q| (times 1/|a.d|)
  float Tpar;  // min |a.d| that proves every unit non-parallel with an exact sign
  float Ec;    // error bound of the objective's c.d
  float eps;   // eps_feas rounded up
};

__device__ __forceinline__ FxLP fx_lp_consts(const KParams& p, float A, float B, float cx,
                                             float cy) {
  FxLP c;
  c.A = A;
  c.B = B;
  c.Ka = A * p.fx_ka;
  c.Tpar = A * p.fx_tp;
  c.Ec = fmaf(fabsf(cx) + fabsf(cy), p.fx_ec, 0x1p-120f);
  c.eps = p.fx_eps;
  return c;
}

// Constants of the current frame s (recomputed at every reshift).
struct FxFrame {
  float sx, sy;
  float Eb;   // |b'32 - (b - a.s)| - u|b'| bound (the bshift residual)
  float KT;   // frame part of the test threshold
  float Kn;   // frame part of the quotient numerator error
  float kE;   // per-event numerator error factor of 1/|a_h|
  float eF;   // frame part of the optimum's error
};

__device__ __forceinline__ FxFrame fx_frame(const FxLP& C, float sx, float sy) {
  FxFrame F;
  F.sx = sx;
  F.sy = sy;
  const float Sm = fabsf(sx) + fabsf(sy);
  F.Eb = sx == 0.0f && sy == 0.0f ? 0.0f
                                  : 2.2f * kU32 * kU32 * (C.B + 2.0f * C.A * Sm) + 0x1p-120f;
  // test: 1.05 (2A Eb + 4U A Sm + U (B + 2 Smax + 1)) + the slack estimate's
  // absolute error eps (3u A Sm + Eb)
  const float Smax = C.eps * (1.0f + C.B) * 1.001f;
  F.KT = 1.05f * (2.0f * C.A * F.Eb + 4.0f * kU64 * C.A * Sm + kU64 * (C.B + 2.0f * Smax + 1.0f)) +
         1.1f * C.eps * (3.0f * kU32 * C.A * Sm + F.Eb) + 0x1p-120f;
  F.Kn = C.A * (1.25f * 25.5f * kU64 * Sm + 2.5f * F.Eb) + 3.75f * kU64 * C.B + 0x1p-120f;
  F.kE = 3.75f * C.A * F.Eb;
  F.eF = 1.1f * 12.0f * kU64 * Sm + 0x1p-120f;
  return F;
}

// ---- cold paths (out of line: they run for a small fraction of events) ----

// The reference's double event at position pi (original values from global
// memory, fold_exact_global, resolve_merged): returns 1 if the LP turned
// infeasible, 2 if the new optimum is not finite, else 0 with the exact
// optimum in (xp, yp) and its defining positions in (pos0, pos1).
// The reference's fold (classify + apply_bound with owners, wu_apply) over
// considered positions [0, pi), lane-strided, on the widened original values:
// the permutation and a from the staging buffer when it is resident (sperm
// non-null), b (and everything else) from global memory, 8 positions per lane
// in flight so the loads overlap.
template <typename P>
__device__ __forceinline__ Acc<double> fx_fold_exact(const KParams& p, int64_t off, uint32_t pi,
                                                     const Line<double>& l, double M,
                                                     const P* sperm, const float* sax,
                                                     const float* say) {
  const int lane = threadIdx.x & 31;
  const float* gx = static_cast<const float*>(p.ax) + off;
  const float* gy = static_cast<const float*>(p.ay) + off;
  const float* gb = static_cast<const float*>(p.b) + off;
  const P* gp = static_cast<const P*>(p.perm) + off;
  Acc<double> acc;
  acc.uL = -INFINITY;
  acc.uR = INFINITY;
  acc.oL = acc.oR = acc.par = kNone;
#pragma unroll 1
  for (uint32_t k0 = lane; k0 < pi; k0 += 32 * kFxExactBatch) {
    float vx[kFxExactBatch], vy[kFxExactBatch], vb[kFxExactBatch];
#pragma unroll
    for (int u = 0; u < kFxExactBatch; ++u) {
      const uint32_t k = k0 + 32 * u;
      const bool in = k < pi && k >= 4;
      const uint32_t o = in ? (sperm ? (uint32_t)sperm[k - 4] : (uint32_t)gp[k - 4]) : 0u;
      vx[u] = in ? (sax ? sax[o] : gx[o]) : 0.0f;
      vy[u] = in ? (say ? say[o] : gy[o]) : 0.0f;
      vb[u] = in ? __ldg(gb + o) : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < kFxExactBatch; ++u) {
      const uint32_t k = k0 + 32 * u;
      if (k < pi) {
        double x = vx[u], y = vy[u], bb = vb[u];
        if (k < 4) {
          x = k == 0 ? 1.0 : (k == 1 ? -1.0 : 0.0);  // serial.hpp:47-52
          y = k == 2 ? 1.0 : (k == 3 ? -1.0 : 0.0);
          bb = M;
        }
        wu_apply(x, y, bb, l, p.eps_par, p.eps_feas, p.eps_hi, k, acc);
      }
    }
  }
  return acc;
}

template <typename P>
__device__ LP2D_FX_COLD int fx_exact_event(const KParams& p, int64_t lp, int64_t off, int m,
                                           uint32_t pi, float cxf, float cyf, float Mf,
                                           uint32_t& pos0, uint32_t& pos1, double& xp,
                                           double& yp, const P* sperm, const float* sax,
                                           const float* say) {
  const double M = Mf;
  double ox, oy, ob;
  fx_orig<P>(p, off, pi, M, ox, oy, ob);
  const Line<double> l = boundary_of(ox, oy, ob);
  const Acc<double> ex = fx_fold_exact<P>(p, off, pi, l, M, sperm, sax, say);
  Header<double> h64;
  h64.lp = lp;
  h64.off = off;
  h64.m = m;
  h64.ok = 1;
  h64.cx = cxf;
  h64.cy = cyf;
  h64.M = M;
  LPState<double> S;
  S.px = xp;
  S.py = yp;
  S.pos0 = pos0;
  S.pos1 = pos1;
  S.st = 0;
  const double cthr = p.eps_par * sqrt(h64.cx * h64.cx + h64.cy * h64.cy);
  const bool feasible = resolve_merged(S, merge_lanes(ex, true), l, pi, h64, cthr, p.eps_feas);
  pos0 = S.pos0;
  pos1 = S.pos1;
  if (!feasible) return 1;
  xp = S.px;
  yp = S.py;
  return (fabs(xp) < INFINITY && fabs(yp) < INFINITY) ? 0 : 2;
}

// The reference's violation test of position pos against the exact optimum
// of the event (p0, p1) (computed here with the reference's operations).
template <typename P>
__device__ LP2D_FX_COLD bool fx_exact_violates(const KParams& p, int64_t off, float Mf,
                                               uint32_t pos, uint32_t p0, uint32_t p1,
                                               bool stale, double& xp, double& yp) {
  const double M = Mf;
  if (stale) {
    double hx, hy, hb, ox, oy, ob;
    fx_orig<P>(p, off, p0, M, hx, hy, hb);
    fx_orig<P>(p, off, p1, M, ox, oy, ob);
    fx_exact_point(hx, hy, hb, ox, oy, ob, xp, yp);
  }
  double x, y, b;
  fx_orig<P>(p, off, pos, M, x, y, b);
  return !satisfied(x, y, b, xp, yp, p.eps_feas);
}

// One case of the fx violation-test dispatch (cf. LP2D_TEST_PAIR): stop at
// the first position whose filtered residual e = a.p' - b' is not provably
// below every slack (e >= -T).
#define LP2D_FX_TEST_PAIR(J)                                                     \
  case J:                                                                        \
    if constexpr (J < NP) {                                                      \
      if constexpr (2 * J + 1 >= L::kAlwaysValid)                                \
        if (64 * J >= mpos) break;                                               \
      const Pair<float> e = fma2(rax[J], PX, fma2(ray[J], PY, rnb[J]));          \
      const uint32_t v0 = __ballot_sync(kFull, lo2(e) >= nT) & m0;               \
      const uint32_t v1 = __ballot_sync(kFull, hi2(e) >= nT) & m1;               \
      m0 = m1 = kFull;                                                           \
      if (v0 | v1) {                                                             \
        sfound = v0 ? 2 * J : 2 * J + 1;                                         \
        vfound = v0 ? v0 : v1;                                                   \
        hx = v0 ? lo2(rax[J]) : hi2(rax[J]);                                     \
        hy = v0 ? lo2(ray[J]) : hi2(ray[J]);                                     \
        hnb = v0 ? lo2(rnb[J]) : hi2(rnb[J]);                                    \
        he = v0 ? lo2(e) : hi2(e);                                               \
        break;                                                                   \
      }                                                                          \
    }                                                                            \
    [[fallthrough]];

// Fold of register pairs (cf. fold_pairs): pairs wholly below the violated
// slot unmasked, the pair holding it masked; distinct asm markers keep the
// compiler from merging the masked tails (which would demote the register
// arrays to local memory).
template <int J, int NP>
__device__ __forceinline__ void fx_fold_pairs(const Pair<float> (&rax)[NP],
                                              const Pair<float> (&ray)[NP],
                                              const Pair<float> (&rnb)[NP], Pair<float> ndx,
                                              Pair<float> ndy, Pair<float> wx, Pair<float> wy,
                                              float kn, float ka, int s, int rel, FxAcc& a,
                                              const PairConsts& k) {
  if constexpr (J + 1 < NP) {
    if (2 * J + 3 < s) {
      fx_fold2<false>(rax[J], ray[J], rnb[J], ndx, ndy, wx, wy, kn, ka, 2 * J, 2 * J + 1, true, true, a, k);
      fx_fold2<false>(rax[J + 1], ray[J + 1], rnb[J + 1], ndx, ndy, wx, wy, kn, ka, 2 * J + 2, 2 * J + 3,
                      true, true, a, k);
      fx_fold_pairs<J + 2, NP>(rax, ray, rnb, ndx, ndy, wx, wy, kn, ka, s, rel, a, k);
    } else if (2 * J + 1 < s) {
      asm volatile("// fx masked pair %0" ::"n"(J + 1));
      fx_fold2<false>(rax[J], ray[J], rnb[J], ndx, ndy, wx, wy, kn, ka, 2 * J, 2 * J + 1, true, true, a, k);
      fx_fold2<true>(rax[J + 1], ray[J + 1], rnb[J + 1], ndx, ndy, wx, wy, kn, ka, 2 * J + 2, 2 * J + 3,
                     64 * J + 64 < rel, 64 * J + 96 < rel, a, k);
    } else {
      asm volatile("// fx masked pair %0" ::"n"(J));
      fx_fold2<true>(rax[J], ray[J], rnb[J], ndx, ndy, wx, wy, kn, ka, 2 * J, 2 * J + 1, 64 * J < rel,
                     64 * J + 32 < rel, a, k);
    }
  } else if constexpr (J < NP) {
    if (2 * J + 1 < s) {
      fx_fold2<false>(rax[J], ray[J], rnb[J], ndx, ndy, wx, wy, kn, ka, 2 * J, 2 * J + 1, true, true, a, k);
    } else {
      asm volatile("// fx masked pair %0" ::"n"(J));
      fx_fold2<true>(rax[J], ray[J], rnb[J], ndx, ndy, wx, wy, kn, ka, 2 * J, 2 * J + 1, 64 * J < rel,
                     64 * J + 32 < rel, a, k);
    }
  }
}

// Register budget: the register-only classes run 3 CTAs of kWarps warps
// (<= 128 registers; K4 keeps more per-LP state than the float kernel).
template <typename L>
struct FxBounds {
  static constexpr int kMinBlocks = L::kLateTma ? L::kMinBlocksRt : (L::kMinBlocks < 3 ? L::kMinBlocks : 3);
};

// DB (tail classes): two staging buffers per warp — the next LP's bulk copy
// is issued into the other buffer when an LP starts instead of when it ends,
// so short LPs do not wait on it.
template <typename P, int NS, int NT, int CAP = 0, bool DB = false>
__global__ void __launch_bounds__(WarpLayout<float, P, NS, NT, CAP>::kMaxWarpsRt * 32,
                                  (FxBounds<WarpLayout<float, P, NS, NT, CAP>>::kMinBlocks))
    k_solve_fx(const __grid_constant__ KParams p) {
  static_assert(NS >= 1 && NS <= 40, "slot count");
  static_assert(NT == 0 || NS % 2 == 0, "the tail starts at a pair boundary");
  static_assert(!DB || NT > 0, "double buffering is for the tail classes");
  using T = float;
  using L = WarpLayout<float, P, NS, NT, CAP>;
  constexpr bool LATE = L::kLateTma && !DB;  // next LP's TMA issued at the end of this one
  constexpr int NBUF = DB ? 2 : 1;
  const int W = L::kLateTma ? (int)(blockDim.x >> 5) : L::kWarps;
  constexpr uint32_t cap = (uint32_t)L::kCap;
  constexpr uint32_t arr = L::kArr;
  constexpr uint32_t bufb = L::kBuf;
  constexpr int NP = (NS + 1) / 2;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int wic = threadIdx.x >> 5;
  unsigned char* const buf0 = smem + (size_t)wic * NBUF * bufb;
  uint64_t* const bar0 = reinterpret_cast<uint64_t*>(smem + (size_t)W * NBUF * bufb) + wic * NBUF;
  int cur = 0;
  uint32_t phases = 0;  // mbarrier parity per buffer (bit)
  unsigned char* buf = buf0;
  uint64_t* bar = bar0;
  const float* sax = reinterpret_cast<const float*>(buf);
  const float* say = reinterpret_cast<const float*>(buf + arr);
  float* sb = reinterpret_cast<float*>(buf + 2 * arr);  // b, after a reshift b' (frame s)
  const P* sperm = reinterpret_cast<const P*>(buf + 3 * arr);
  auto tail_idx = [&](int c, uint32_t lim) -> uint32_t {
    return min((uint32_t)sperm[32 * min(c, NS + NT - 1) + lane - 4], lim);
  };
  const PairConsts pk = p.pk;
  const uint64_t policy = policy_evict_first();

  if (lane < NBUF) mbar_init(bar0 + lane, 1);
  __syncwarp();

  const int32_t* list;
  int64_t n_list;
  resolve_list(p, list, n_list);
  const int64_t TW = p.total_warps;
  const int64_t j0 = (int64_t)blockIdx.x * W + wic;
  auto lp_of = [&](int64_t t) -> int64_t { return t < n_list ? (list ? (int64_t)list[t] : t) : -1; };
  constexpr int64_t kAhead = LATE ? 1 : 2;
  int64_t lpA = lp_of(j0), lpB = LATE ? -1 : lp_of(j0 + TW);
  uint32_t hA = load_header_word<T>(p, lpA, lane);
  uint32_t hB = LATE ? 0u : load_header_word<T>(p, lpB, lane);
  uint32_t ticket = atomic_add_if(p.counter, lane == 0, p.pk.zero);
  Header<T> h = unpack_header<L, T>(hA, lpA);
  issue_tma_warp<L, T, P>(p, h, buf, bar, policy, arr, lane);
  int64_t pend_lp = -1;  // deferred pair export of the previous LP (register-only classes)
  uint32_t pend_pos = kNone, pend_q = 0;

  while (h.lp >= 0) {
    if constexpr (DB) {
      buf = buf0 + cur * bufb;
      bar = bar0 + cur;
      sax = reinterpret_cast<const float*>(buf);
      say = reinterpret_cast<const float*>(buf + arr);
      sb = reinterpret_cast<float*>(buf + 2 * arr);
      sperm = reinterpret_cast<const P*>(buf + 3 * arr);
    }
    mbar_wait(bar, (phases >> cur) & 1u);
    phases ^= 1u << cur;
#ifdef LP2D_FX_TIMELINE
    uint64_t tl0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tl0));
#endif

    // ---- gather (frame s = 0: b' = b) -------------------------------------
    Pair<T> rax[NP], ray[NP], rnb[NP];
    Pair<T> rbo[L::kLateTma ? 1 : NP];  // register-only classes: original b
    const int mj = h.ok ? h.m : 0;
    const int mpos = mj + 4;
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      T vx[2], vy[2], vb[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int K = 2 * j + e;
        const int P_ = 32 * K + lane;
        if (K >= NS) {
          vx[e] = 0.0f;
          vy[e] = 0.0f;
          vb[e] = INFINITY;
          continue;
        }
        const bool valid = (K < L::kAlwaysValid || P_ < mpos) && !(K == 0 && P_ < 4);
        const uint32_t o = min((uint32_t)sperm[K == 0 ? max(P_ - 4, 0) : P_ - 4], cap - 1u);
        T x = valid ? sax[o] : 0.0f;
        T y = valid ? say[o] : 0.0f;
        T bb = valid ? sb[o] : INFINITY;
        if (K == 0 && P_ < 4) {
          x = P_ == 0 ? 1.0f : (P_ == 1 ? -1.0f : 0.0f);
          y = P_ == 2 ? 1.0f : (P_ == 3 ? -1.0f : 0.0f);
          bb = h.M;
        }
        vx[e] = x;
        vy[e] = y;
        vb[e] = bb;
      }
      rax[j] = mk2(vx[0], vx[1]);
      ray[j] = mk2(vy[0], vy[1]);
      rnb[j] = mk2(-vb[0], -vb[1]);
      if constexpr (!L::kLateTma) rbo[j] = mk2(vb[0], vb[1]);
    }
    // Magnitudes over the whole LP (original order, vector reads) and the
    // permutation check.
    float amx = 1.0f, bmx = fabsf(h.M);
    {
      const int ng = (mj + 3) >> 2;
#pragma unroll 1
      for (int g = lane; g < ng; g += 32) {
        const float4 vx = reinterpret_cast<const float4*>(sax)[g];
        const float4 vy = reinterpret_cast<const float4*>(say)[g];
        const float4 vb = reinterpret_cast<const float4*>(sb)[g];
        const int rem = mj - 4 * g;
        const float x[4] = {vx.x, vx.y, vx.z, vx.w}, y[4] = {vy.x, vy.y, vy.z, vy.w},
                    b4[4] = {vb.x, vb.y, vb.z, vb.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (e < rem) {
            amx = max3_abs(amx, x[e], y[e]);
            bmx = max3_abs(bmx, b4[e], b4[e]);
          }
        }
      }
    }
    const bool bad = !h.ok || (mj > 0 && perm_max<P>(sperm, mj, lane) >= (uint32_t)mj);
    const float A = warp_max_nan_f(amx), B = warp_max_nan_f(bmx);  // NaN reaches the guard
    if constexpr (!L::kLateTma) {
      __syncwarp();
      fence_proxy_async_smem();
    }
    Header<T> hn;
    if constexpr (!LATE) {
      // register-only classes: the buffer was consumed by the gather; DB: the
      // other buffer's LP finished (and fenced) one LP ago
      hn = unpack_header<L, T>(hB, lpB);
      if constexpr (DB)
        issue_tma_warp<L, T, P>(p, hn, buf0 + (cur ^ 1) * bufb, bar0 + (cur ^ 1), policy, arr, lane);
      else
        issue_tma_warp<L, T, P>(p, hn, buf, bar, policy, arr, lane);
    }
    const int64_t tk = (int64_t)__shfl_sync(kFull, ticket, 0) + kAhead * TW;
    lpB = lp_of(tk);
    hB = load_header_word<T>(p, lpB, lane);
    if constexpr (!LATE) ticket = atomic_add_if(p.counter, lane == 0, p.pk.zero);

    // ---- solve (serial.hpp:159-188) -----------------------------------------
    // range guard: outside it the fp32 filter has no proven bounds (and
    // NaN/INF inputs), so the LP takes the reference's operations throughout
    const bool wild = !(A < 0x1p24f) || !(B < 0x1p62f) || !(fabsf(h.cx) < 0x1p100f) ||
                      !(fabsf(h.cy) < 0x1p100f) || !(fabsf(h.M) < 0x1p62f);
    const FxLP C = fx_lp_consts(p, A, B, h.cx, h.cy);
    FxFrame F = fx_frame(C, 0.0f, 0.0f);
    bool shifted = false;  // frame != 0 (late-TMA classes: the buffer holds b')
#ifdef LP2D_FX_LPSTATS
    uint32_t st_res = 0, st_exe = 0, st_tst = 0;  // debug: per-LP path counts
#endif
    // Move the frame to s = (nsx, nsy): b' of every constraint (register
    // chunks, and in place in the staging buffer for the late-TMA classes).
    auto reshift = [&](float nsx, float nsy) {
      fx_count(p, kFxReshift, lane);
#ifdef LP2D_FX_LPSTATS
      ++st_res;
#endif
      if constexpr (L::kLateTma) {
        // b' of every staged constraint rewritten in place (original
        // order): from the staged original b on the first reshift, else
        // from the original b in global memory (L2: streamed an LP ago)
        const Pair<T> SX = splat2(nsx), SY = splat2(nsy);
        const int nv = (mj + 3) >> 2;
        float4* sb4 = reinterpret_cast<float4*>(sb);
        const float4* gb4 = reinterpret_cast<const float4*>(static_cast<const float*>(p.b) + h.off);
#pragma unroll 1
        for (int g0 = lane; g0 < nv; g0 += 32 * kFxShiftBatch) {
          float4 vb[kFxShiftBatch];
#pragma unroll
          for (int u = 0; u < kFxShiftBatch; ++u) {
            const int g = g0 + 32 * u;
            vb[u] = g < nv ? (shifted ? __ldg(gb4 + g) : sb4[g]) : make_float4(0, 0, 0, 0);
          }
#pragma unroll
          for (int u = 0; u < kFxShiftBatch; ++u) {
            const int g = g0 + 32 * u;
            if (g < nv) {
              const float4 vx = reinterpret_cast<const float4*>(sax)[g];
              const float4 vy = reinterpret_cast<const float4*>(say)[g];
              const Pair<T> lo =
                  bshift2(mk2(vx.x, vx.y), mk2(vy.x, vy.y), mk2(vb[u].x, vb[u].y), SX, SY, pk);
              const Pair<T> hi =
                  bshift2(mk2(vx.z, vx.w), mk2(vy.z, vy.w), mk2(vb[u].z, vb[u].w), SX, SY, pk);
              sb4[g] = make_float4(lo2(lo), hi2(lo), lo2(hi), hi2(hi));
            }
          }
        }
        __syncwarp();
        // register chunks from the rewritten buffer (the box: M - (+-s))
#pragma unroll
        for (int j = 0; j < NP; ++j) {
          T v[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int K = 2 * j + e;
            const int P_ = 32 * K + lane;
            const bool valid = K < NS && (K < L::kAlwaysValid || P_ < mpos);
            const uint32_t o = min((uint32_t)sperm[K == 0 ? max(P_ - 4, 0) : P_ - 4], cap - 1u);
            v[e] = valid ? -sb[o] : -INFINITY;
            if (K == 0 && P_ < 4)
              v[e] = -bshift(P_ == 0 ? 1.0f : (P_ == 1 ? -1.0f : 0.0f),
                             P_ == 2 ? 1.0f : (P_ == 3 ? -1.0f : 0.0f), h.M, nsx, nsy);
          }
          rnb[j] = mk2(v[0], v[1]);
        }
      } else {
        const Pair<T> SX = splat2(nsx), SY = splat2(nsy);
#pragma unroll
        for (int j = 0; j < NP; ++j) {
          const Pair<T> bs = bshift2(rax[j], ray[j], rbo[j], SX, SY, pk);
          // (padding slots hold b = +INF: keep their b' at +INF)
          rnb[j] = mk2(lo2(rbo[j]) < INFINITY ? -lo2(bs) : -INFINITY,
                       hi2(rbo[j]) < INFINITY ? -hi2(bs) : -INFINITY);
        }
      }
      F = fx_frame(C, nsx, nsy);
      shifted = true;
    };
    uint8_t st = bad ? 255 : 0;
    uint32_t pos0 = h.cx < 0.0f ? 1u : 0u, pos1 = h.cy < 0.0f ? 3u : 2u;  // box corner's edges
    double xp = h.cx < 0.0f ? -(double)h.M : (double)h.M;  // serial.hpp:56-58
    double yp = h.cy < 0.0f ? -(double)h.M : (double)h.M;
    bool stale = false;                      // (xp, yp) is exact unless stale
    float ppx = (float)xp, ppy = (float)yp;  // local optimum (s = 0: exact)
    float epp = 0.0f;                        // its error bound
    uint32_t viol = 0, wu32 = 0;
    int ns = 0;
    uint32_t nmask = 0xfffffff0u;
    bool running = !bad && !wild;
    bool need_exact_lp = !bad && wild;
    constexpr float cP = 7.35f * kU32 + 8.4f * kU64;
    while (running) {
      const float pmag = fmaxf(fabsf(ppx), fabsf(ppy));
      const float T_ = fmaf(C.A, fmaf(2.11f, epp, cP * pmag), F.KT);
      const float nT = -T_;
      const Pair<T> PX = splat2(ppx), PY = splat2(ppy);
      int sfound = -1;
      uint32_t vfound = 0;
      T hx = 0.0f, hy = 0.0f, hnb = 0.0f, he = 0.0f;
      uint32_t m0 = (ns & 1) ? 0u : nmask;
      uint32_t m1 = (ns & 1) ? nmask : kFull;
      switch (ns >> 1) {
        LP2D_FX_TEST_PAIR(0) LP2D_FX_TEST_PAIR(1) LP2D_FX_TEST_PAIR(2) LP2D_FX_TEST_PAIR(3)
        LP2D_FX_TEST_PAIR(4) LP2D_FX_TEST_PAIR(5) LP2D_FX_TEST_PAIR(6) LP2D_FX_TEST_PAIR(7)
        LP2D_FX_TEST_PAIR(8) LP2D_FX_TEST_PAIR(9) LP2D_FX_TEST_PAIR(10) LP2D_FX_TEST_PAIR(11)
        LP2D_FX_TEST_PAIR(12) LP2D_FX_TEST_PAIR(13) LP2D_FX_TEST_PAIR(14) LP2D_FX_TEST_PAIR(15)
        LP2D_FX_TEST_PAIR(16) LP2D_FX_TEST_PAIR(17) LP2D_FX_TEST_PAIR(18) LP2D_FX_TEST_PAIR(19)
        default:
          if constexpr (NT > 0) {
            int c = NS;
            uint32_t t0 = kFull, t1 = kFull;
            if (ns >= NS) {
              c = ns & ~1;
              t0 = (ns & 1) ? 0u : nmask;
              t1 = (ns & 1) ? nmask : kFull;
            }
            const int cend = min(NS + NT, (mpos + 31) >> 5);
            const uint32_t lim = (uint32_t)(mj - 1);
            uint32_t o0 = tail_idx(c, lim), o1 = tail_idx(c + 1, lim);
#pragma unroll 1
            for (; c < cend; c += 2) {
              const T x0 = sax[o0], y0 = say[o0], b0 = sb[o0];
              const T x1 = sax[o1], y1 = say[o1], b1 = sb[o1];
              o0 = tail_idx(c + 2, lim);
              o1 = tail_idx(c + 3, lim);
              const Pair<T> e = fma2(mk2(x0, x1), PX, fma2(mk2(y0, y1), PY, mk2(-b0, -b1)));
              const uint32_t v0 = __ballot_sync(kFull, lo2(e) >= nT && 32 * c + lane < mpos) & t0;
              const uint32_t v1 =
                  __ballot_sync(kFull, hi2(e) >= nT && 32 * c + 32 + lane < mpos) & t1;
              t0 = t1 = kFull;
              if (v0 | v1) {
                sfound = v0 ? c : c + 1;
                vfound = v0 ? v0 : v1;
                hx = v0 ? x0 : x1;
                hy = v0 ? y0 : y1;
                hnb = v0 ? -b0 : -b1;
                he = v0 ? lo2(e) : hi2(e);
                break;
              }
            }
          }
          break;
      }
      if (sfound < 0) break;
      const int s = sfound;
      const int f = __ffs(vfound) - 1;
      hx = __shfl_sync(kFull, hx, f);
      hy = __shfl_sync(kFull, hy, f);
      hnb = __shfl_sync(kFull, hnb, f);
      he = __shfl_sync(kFull, he, f);
      const uint32_t pi = 32u * (uint32_t)s + (uint32_t)f;
      ns = (int)(pi + 1) >> 5;  // resume right after pi (test or event)
      nmask = kFull << ((pi + 1) & 31);
      {
        // The candidate's own slack S = eps (1 + |b|) (core.hpp:65-67), |b|
        // from b' and the frame: proves "satisfied" or "violated" unless the
        // residual lies within the bound of it.
        const float bo = fmaf(hx, F.sx, fmaf(hy, F.sy, -hnb));
        const float Sk = fmaf(C.eps, fabsf(bo), C.eps);
        const float tol = T_ + 6.0f * kU32 * fabsf(he) + 16.0f * kU32 * Sk;
        if (he < Sk - tol) continue;  // satisfied: resume the sweep after pi
        if (!(he > Sk + tol)) {
          fx_count(p, kFxTestFlag, lane);
#ifdef LP2D_FX_LPSTATS
          ++st_tst;
#endif
          if (stale) fx_count(p, kFxLazy, lane);
          const bool v = fx_exact_violates<P>(p, h.off, h.M, pi, pos0, pos1, stale, xp, yp);
          stale = false;
          if (T_ > 16.0f * Sk) {
            // the band is wide (the optimum is far from the frame): move the
            // frame onto the exact optimum so the next tests are sharp
            reshift((float)xp, (float)yp);
            ppx = (float)(xp - (double)F.sx);
            ppy = (float)(yp - (double)F.sy);
            epp = kU32 * fmaxf(fabsf(ppx), fabsf(ppy)) +
                  2.0f * kU64 * (float)fmax(fabs(xp), fabs(yp)) + 0x1p-120f;
            // the candidate's b' in the new frame (the event below uses it)
            if constexpr (L::kLateTma) {
              hnb = -sb[min((uint32_t)sperm[pi - 4], cap - 1u)];
            } else {
              const int sl = (int)(pi >> 5);
              float vb = 0.0f;
#pragma unroll
              for (int j = 0; j < NP; ++j)
                vb = sl == 2 * j ? lo2(rbo[j]) : (sl == 2 * j + 1 ? hi2(rbo[j]) : vb);
              hnb = -bshift(hx, hy, __shfl_sync(kFull, vb, f), F.sx, F.sy);
            }
          }
          if (!v) continue;
        }
      }
      // ---- event at position pi: 1D LP over positions [0, pi) ----------------
      viol += 1;
      wu32 += pi;  // considered.size() (serial.hpp:176-179)
      if (lane == 0) note_event(p, h.lp, pi);
      const float len2 = fmaf(hx, hx, hy * hy);
      const bool line_ok = (len2 >= 0x1p-100f) & (len2 <= 0x1p100f);
      const float rs = rsqrt_approx(len2), rl2 = rcp_approx(len2);
      const float dx = -hy * rs, dy = hx * rs;
      const float ac = fmaf(h.cx, dx, h.cy * dy);
      bool fast = line_ok && fabsf(ac) > C.Ec;
      const bool take_right = ac > 0.0f;  // serial.hpp:102-108 (proved when fast)
      const float fdx = take_right ? -dx : dx, fdy = take_right ? -dy : dy;
      const Pair<T> NDX = splat2(-fdx), NDY = splat2(-fdy);
      const float Obig = 1.5f * C.B * rs;  // >= |o64| = |b_h|/|a_h|
      float hbp = -hnb;
      const int rel = (int)pi - lane;
      bool done = false;
#pragma unroll 1
      for (int pass = 0; fast; ++pass) {
        const float scl = hbp * rl2;
        const float wx = hx * scl, wy = hy * scl;
        const float Wm = fmaxf(fabsf(wx), fabsf(wy));
        const float kn = fmaf(C.A, fmaf(1.25f * (30.0f * kU32 + 16.5f * kU64), Wm,
                                        fmaf(1.25f * 23.0f * kU64, Obig, F.kE * rs)),
                              F.Kn) * (1.0f + 0x1p-10f);
        const float ka = C.Ka * (1.0f + 0x1p-10f);
        FxAcc acc;
        fx_acc_init(acc);
        const Pair<T> WX = splat2(wx), WY = splat2(wy);
        fx_fold_pairs<0, NP>(rax, ray, rnb, NDX, NDY, WX, WY, kn, ka, s, rel, acc, pk);
        if constexpr (NT > 0) {
          const uint32_t lim = (uint32_t)(mj - 1);
          uint32_t o0 = tail_idx(NS, lim), o1 = tail_idx(NS + 1, lim);
#pragma unroll 1
          for (int c = NS; c <= s; c += 2) {
            const T x0 = sax[o0], y0 = say[o0], b0 = sb[o0];
            const T x1 = sax[o1], y1 = say[o1], b1 = sb[o1];
            o0 = tail_idx(c + 2, lim);
            o1 = tail_idx(c + 3, lim);
            const Pair<T> X = mk2(x0, x1), Y = mk2(y0, y1), NB = mk2(-b0, -b1);
            if (c + 1 < s)
              fx_fold2<false>(X, Y, NB, NDX, NDY, WX, WY, kn, ka, (uint32_t)c, (uint32_t)c + 1, true,
                              true, acc, pk);
            else
              fx_fold2<true>(X, Y, NB, NDX, NDY, WX, WY, kn, ka, (uint32_t)c, (uint32_t)c + 1,
                             32 * c < rel, 32 * (c + 1) < rel, acc, pk);
          }
        }
        // ---- merge and certify ---------------------------------------------
        const float G1 = warp_max_f(acc.h1);
        const uint32_t hold = __ballot_sync(kFull, acc.h1 == G1);
        const int hl = __ffs(hold) - 1;
        const int src = hl < 0 ? 0 : hl;
        const float G2 = warp_max_f(lane == hl ? acc.h2 : acc.h1);
        const float RL = warp_min_f(acc.rl);
        const float MAL = warp_min_f(acc.mal);
        const uint32_t oslot = __shfl_sync(kFull, acc.own, src);
        const float L1 = __shfl_sync(kFull, acc.l1, src);
        // the winner's lo beats every other unit's hi (unique owner, the
        // reference's argmax) and the chosen side's hi is below the other
        // side's lo (non-empty interval); 4u margins cover hi/lo rounding
        const bool cert = (MAL > C.Tpar) && __popc(hold) == 1 && oslot != kNone &&
                          fabsf(G1) < INFINITY && fabsf(L1) < INFINITY &&
                          (L1 > G2 + 4.0f * kU32 * (fabsf(L1) + fabsf(G2))) &&
                          (G1 + 4.0f * kU32 * (fabsf(G1) + fabsf(RL)) <= RL);
        const float q1 = 0.5f * (G1 + L1);          // the winner's quotient
        const float aG1 = fabsf(q1);
        if (cert) {
          // the reference's event resolves to the owner at (oslot, hl): the
          // optimum is that pair's intersection, exactly known, computed lazily
          const float E1 = 0.505f * (G1 - L1);
          pos0 = pi;
          pos1 = 32u * oslot + (uint32_t)hl;
          stale = true;
          ppx = fmaf(q1, fdx, wx);
          ppy = fmaf(q1, fdy, wy);
          epp = fmaf(1.1f, E1,
                     fmaf(1.1f * (kRho + 6.0f * kU32 + 2.0f * kU64), aG1,
                          fmaf(1.1f * (11.0f * kU32 + 7.5f * kU64), Wm,
                               fmaf(1.65f * F.Eb + 9.0f * kU64 * C.B * 1.5f, rs, F.eF))));
          done = true;
          break;
        }
        if (pass > 0 || !(aG1 < INFINITY) || hl < 0 || !(fabsf(L1) < INFINITY)) break;
        // reshift the frame to the candidate point and refold once
        const float nsx = F.sx + fmaf(q1, fdx, wx), nsy = F.sy + fmaf(q1, fdy, wy);
        reshift(nsx, nsy);
        // the violated constraint's b' in the new frame
        if constexpr (L::kLateTma) {
          hbp = sb[min((uint32_t)sperm[pi - 4], cap - 1u)];
        } else {
          const int sl = (int)(pi >> 5);
          float vb = 0.0f;
#pragma unroll
          for (int j = 0; j < NP; ++j)
            vb = sl == 2 * j ? lo2(rbo[j]) : (sl == 2 * j + 1 ? hi2(rbo[j]) : vb);
          hbp = bshift(hx, hy, __shfl_sync(kFull, vb, f), nsx, nsy);
        }
      }
      if (!done) {
        // the reference's double operations for this event
        fx_count(p, kFxExact, lane);
#ifdef LP2D_FX_LPSTATS
        ++st_exe;
#endif
        const int r = fx_exact_event<P>(p, h.lp, h.off, mj, pi, h.cx, h.cy, h.M, pos0, pos1, xp, yp,
                                        L::kLateTma ? sperm : nullptr, L::kLateTma ? sax : nullptr,
                                        L::kLateTma ? say : nullptr);
        stale = false;
        if (r == 1) {
          st = 1;
          break;
        }
        if (r == 2) {
          need_exact_lp = true;  // non-finite optimum: whole-LP reference path
          break;
        }
        reshift((float)xp, (float)yp);  // the frame onto the exact optimum
        ppx = (float)(xp - (double)F.sx);
        ppy = (float)(yp - (double)F.sy);
        epp = kU32 * fmaxf(fabsf(ppx), fabsf(ppy)) +
              2.0f * kU64 * (float)fmax(fabs(xp), fabs(yp)) + 0x1p-120f;
      }
    }
    // ---- results ------------------------------------------------------------
    if (need_exact_lp) {
      fx_count(p, kFxWild, lane);
      Header<double> h64;
      h64.lp = h.lp;
      h64.off = h.off;
      h64.m = h.m;
      h64.ok = h.ok;
      h64.cx = h.cx;
      h64.cy = h.cy;
      h64.M = h.M;
      LPState<double> S64;
      solve_exact_global<double, P, float>(p, h64, p.eps_par, p.eps_feas, p.eps_hi, S64, viol);
      st = S64.st;
      pos0 = S64.pos0;
      pos1 = S64.pos1;
      xp = S64.px;
      yp = S64.py;
      viol = S64.viol;
      wu32 = (uint32_t)S64.wu;
      stale = false;
    }
    if (st == 0 && stale) {
      // the final optimum with the reference's operations, from the
      // resident staging buffer (late-TMA classes: b from global) or the
      // registers (register-only classes, broadcast from the owning lanes)
      float v[6];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const uint32_t pos = q ? pos1 : pos0;
        float x, y, bb;
        if (pos < 4) {
          x = pos == 0 ? 1.0f : (pos == 1 ? -1.0f : 0.0f);  // serial.hpp:47-52
          y = pos == 2 ? 1.0f : (pos == 3 ? -1.0f : 0.0f);
          bb = h.M;
        } else if constexpr (L::kLateTma) {
          const uint32_t o = min((uint32_t)sperm[pos - 4], cap - 1u);
          x = sax[o];
          y = say[o];
          bb = shifted ? __ldg(static_cast<const float*>(p.b) + h.off + o) : sb[o];
        } else {
          const int sl = (int)(pos >> 5), ln = (int)(pos & 31);
          float vx = 0.0f, vy = 0.0f, vb = 0.0f;
#pragma unroll
          for (int j = 0; j < NP; ++j) {
            vx = sl == 2 * j ? lo2(rax[j]) : (sl == 2 * j + 1 ? hi2(rax[j]) : vx);
            vy = sl == 2 * j ? lo2(ray[j]) : (sl == 2 * j + 1 ? hi2(ray[j]) : vy);
            vb = sl == 2 * j ? lo2(rbo[j]) : (sl == 2 * j + 1 ? hi2(rbo[j]) : vb);
          }
          x = __shfl_sync(kFull, vx, ln);
          y = __shfl_sync(kFull, vy, ln);
          bb = __shfl_sync(kFull, vb, ln);
        }
        v[3 * q] = x;
        v[3 * q + 1] = y;
        v[3 * q + 2] = bb;
      }
      fx_exact_point(v[0], v[1], v[2], v[3], v[4], v[5], xp, yp);
    }
    if (st == 0 && (pos0 < 4 || pos1 < 4)) st = 2;
    if constexpr (L::kLateTma) {
      // defining pair from the still-resident staged permutation
      if (lane < 2 && p.pair) {
        uint32_t pos = lane == 0 ? pos0 : pos1;
        if (st == 255) pos = kNone;
        const uint32_t q =
            (pos != kNone && pos >= 4) ? (uint32_t)sperm[min(pos - 4, cap - 1u)] : 0u;
        p.pair[2 * h.lp + lane] = pair_code(pos, q);
      }
      __syncwarp();
      fence_proxy_async_smem();  // (DB: this buffer is restaged one LP from now)
      if constexpr (LATE) {
        hn = unpack_header<L, T>(hB, lpB);
        issue_tma_warp<L, T, P>(p, hn, buf, bar, policy, arr, lane);
        ticket = atomic_add_if(p.counter, lane == 0, p.pk.zero);
      }
    } else {
      // pair export: lanes 0/1 request perm[pos-4] now, store one LP later
      if (pend_lp >= 0 && lane < 2 && p.pair)
        p.pair[2 * pend_lp + lane] = pair_code(pend_pos, pend_q);
      pend_lp = h.lp;
      pend_pos = lane == 0 ? pos0 : pos1;
      if (st == 255) pend_pos = kNone;
      const bool need = lane < 2 && pend_pos != kNone && pend_pos >= 4;
      const P* pa = static_cast<const P*>(p.perm) + h.off + (need ? pend_pos - 4 : 0);
      pend_q = sizeof(P) == 2 ? ldg_u16_if(pa, need) : ldg_u32_if(pa, need);
    }
    if (lane == 0) {
      const int64_t lp = h.lp;
      p.status[lp] = st;
      const bool feas = st == 0 || st == 2;
      static_cast<double*>(p.x)[lp] = feas ? xp : 0.0;
      static_cast<double*>(p.y)[lp] = feas ? yp : 0.0;
      // serial.hpp:187 objective_value
      static_cast<double*>(p.value)[lp] = feas ? (double)h.cx * xp + (double)h.cy * yp : 0.0;
      if (p.viol) p.viol[lp] = viol;
      if (p.wu) p.wu[lp] = wu32;
#ifdef LP2D_FX_LPSTATS  // debug: pair[2lp+1] = reshifts | exact events << 10 | exact tests << 20
      if (p.pair) p.pair[2 * lp + 1] = (int32_t)(st_res | (st_exe << 10) | (st_tst << 20));
#endif
#ifdef LP2D_FX_TIMELINE
      uint64_t tl1;  // debug: wu = start (ns), pair[2lp] = duration (ns)
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tl1));
      if (p.wu) p.wu[lp] = tl0;
      if (p.pair) p.pair[2 * lp] = (int32_t)min(tl1 - tl0, (uint64_t)0x7fffffff);
#endif
    }
    h = hn;
    if constexpr (DB) cur ^= 1;
  }
  if (pend_lp >= 0 && lane < 2 && p.pair) p.pair[2 * pend_lp + lane] = pair_code(pend_pos, pend_q);

  // Self-reset of the ticket counter by the last warp to finish. The fence
  // orders this warp's last ticket claim (whose value may be unread) before
  // the finish count.
  if (lane == 0) {
    __threadfence();
    const uint32_t t = atomicAdd(p.counter + 1, 1u);
    if (t == (uint32_t)p.total_warps - 1) {
      p.counter[0] = 0;
      p.counter[1] = 0;
    }
  }
}
#undef LP2D_FX_TEST_PAIR

}  // namespace lp2d_b200
