// lp2d_fs.cuh — K5: fp32-STORED batches with the reference's DOUBLE semantics,
// insertion-order shared-memory layout. Included after lp2d_fx.cuh (it reuses
// K4's certificate machinery: FxLP / FxFrame constants, fx_fold2, bshift2,
// fx_exact_point, fx_exact_violates — the bounds are derived once, DESIGN.md
// §3, and shared by both kernels).
//
// Why a second kernel: K4 keeps the first NS chunks of an LP in registers and
// walks the rest through the permutation in the staging buffer. That costs a
// size-class template per chunk count, a 20-way resume dispatch, masked-pair
// variants per slot and an indirection (LDS.U16 + 3 conflicting LDS) per tail
// unit — 129 KB of SASS per instantiation (ncu: 35% of warp stalls were
// `no_instruction`) and ~360 instructions of fixed cost per violation event.
//
// K5 applies the permutation ONCE per LP, in place, in shared memory: the bulk
// TMA lands the LP's original-order ax / ay / b / perm segments in a per-warp
// buffer whose three scalar regions are sized for the considered positions
// (box + constraints, rounded to 64); each lane gathers its positions through
// the permutation into registers, and after a __syncwarp writes them back in
// INSERTION order (position k = 4 + i holds constraint perm[i]; positions
// 0..3 hold the box, serial.hpp:47-52; b is stored negated, NB = -b' with b'
// the frame-shifted bound). From then on:
//   * a test step is 64 consecutive positions: three LDS.64 per lane (positions
//     64c + 2 lane + {0, 1}), two packed FFMA2, two ballots;
//   * the 1D re-solve over [0, pi) is a plain loop over whole 64-position
//     chunks (+ one masked chunk): the same three LDS.64 feed fx_fold2;
//   * the violated constraint is read back with three broadcast loads (no
//     shuffles), and owners are positions (no slot bookkeeping).
// The permutation region stays resident for the defining pair's export and for
// the exact paths (which read the original b from global memory).
#pragma once

namespace lp2d_b200 {

// Per-warp buffer of one LP of up to CAP constraints.
template <typename P, int CAP>
struct FsLayout {
  static constexpr int kCap = CAP;
  static constexpr int kPos = ((CAP + 4 + 63) / 64) * 64;  // considered positions, padded
  static constexpr int kChunks = kPos / 64;                // 64-position chunks
  static constexpr uint32_t kArr = (uint32_t)kPos * 4u;    // one scalar region (float)
  // (kPos entries: the permute pass reads an index pair per position pair)
  static constexpr uint32_t kPerm = round16((uint32_t)kPos * (uint32_t)sizeof(P));
  static constexpr uint32_t kBuf = 3 * kArr + kPerm;
};

__device__ __forceinline__ Pair<float> neg2(Pair<float> v) { return Pair<float>{v.v ^ 0x8000000080000000ull}; }

__device__ __forceinline__ Pair<float> lds2(const float* base, int idx2) {
  return Pair<float>{reinterpret_cast<const unsigned long long*>(base)[idx2]};
}
__device__ __forceinline__ void sts2(float* base, int idx2, Pair<float> v) {
  reinterpret_cast<unsigned long long*>(base)[idx2] = v.v;
}

// Issue the bulk copies of one LP into a K5 buffer (whole warp calls; the
// operands are made warp-uniform first, cf. issue_tma_warp).
template <typename L, typename P>
__device__ __forceinline__ void fs_issue(const KParams& p, const Header<float>& h,
                                         unsigned char* buf, uint64_t* bar, uint64_t policy,
                                         int lane) {
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
  const uint32_t bt = round16(m * 4u);
  const uint32_t bp = round16(m * (uint32_t)sizeof(P));
  if (lane == 0 && go) {
    mbar_arrive_expect_tx_u(sbar, 3 * bt + bp);
    if (bt) {
      bulk_g2s_u(sbuf, static_cast<const float*>(p.ax) + off, bt, sbar, pol);
      bulk_g2s_u(sbuf + L::kArr, static_cast<const float*>(p.ay) + off, bt, sbar, pol);
      bulk_g2s_u(sbuf + 2 * L::kArr, static_cast<const float*>(p.b) + off, bt, sbar, pol);
      bulk_g2s_u(sbuf + 3 * L::kArr, static_cast<const P*>(p.perm) + off, bp, sbar, pol);
    }
  }
}

// In-place permutation of a landed LP into insertion order (see the header).
// Returns the LP's magnitude bounds A = max(1, |ax|, |ay|), B = max(|M|, |b|)
// over its constraints (original order, vector reads; NaN-propagating: a NaN
// coefficient reaches the range guard) and the largest permutation entry
// (>= m: invalid LP). m >= 1.
template <typename P, int CAP>
__device__ __forceinline__ void fs_permute(unsigned char* buf, int m, float M, int lane, float& A,
                                           float& B, uint32_t& pmax) {
  using L = FsLayout<P, CAP>;
  constexpr int NC = L::kChunks;
  float* X = reinterpret_cast<float*>(buf);
  float* Y = reinterpret_cast<float*>(buf + L::kArr);
  float* NB = reinterpret_cast<float*>(buf + 2 * L::kArr);
  const P* perm = reinterpret_cast<const P*>(buf + 3 * L::kArr);
  const int mpos = m + 4;
  {
    float amx = 1.0f, bmx = fabsf(M);
    const int ng = (m + 3) >> 2;
#pragma unroll 1
    for (int g = lane; g < ng; g += 32) {
      const float4 vx = reinterpret_cast<const float4*>(X)[g];
      const float4 vy = reinterpret_cast<const float4*>(Y)[g];
      const float4 vb = reinterpret_cast<const float4*>(NB)[g];
      if (4 * g + 4 <= m) {
        amx = max3_abs(amx, vx.x, vx.y);
        amx = max3_abs(amx, vx.z, vx.w);
        amx = max3_abs(amx, vy.x, vy.y);
        amx = max3_abs(amx, vy.z, vy.w);
        bmx = max3_abs(bmx, vb.x, vb.y);
        bmx = max3_abs(bmx, vb.z, vb.w);
      } else {
        const int rem = m - 4 * g;
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
    A = warp_max_nan_f(amx);
    B = warp_max_nan_f(bmx);
  }
  pmax = perm_max<P>(perm, m, lane);
  // Byte offsets of the constraints at this lane's positions k0 = 64 j +
  // 2 lane and k0 + 1 (entries k0 - 4, k0 - 3: one aligned index pair). Box
  // rows (chunk 0, lanes 0-1) and rows past m read some entry of the buffer
  // (clamped in range) and are overwritten below; chunks past the LP's last
  // are never read.
  const int nc = (mpos + 63) >> 6;
  uint32_t o[2 * NC];
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    const int e0 = max(64 * j + 2 * lane - 4, 0);
    uint32_t i0, i1;
    if constexpr (sizeof(P) == 2) {
      const uint32_t w = *reinterpret_cast<const uint32_t*>(perm + e0);
      i0 = w & 0xffffu;
      i1 = w >> 16;
    } else {
      const uint2 w = *reinterpret_cast<const uint2*>(perm + e0);
      i0 = w.x;
      i1 = w.y;
    }
    o[2 * j] = 4u * min(i0, (uint32_t)CAP - 1u);
    o[2 * j + 1] = 4u * min(i1, (uint32_t)CAP - 1u);
  }
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    unsigned char* R = buf + r * L::kArr;
    float v[2 * NC];
#pragma unroll
    for (int i = 0; i < 2 * NC; ++i) v[i] = *reinterpret_cast<const float*>(R + o[i]);
    __syncwarp();
    float* RF = reinterpret_cast<float*>(R);
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      if (j < nc || j == 0) {
        RF[64 * j + 2 * lane] = r == 2 ? -v[2 * j] : v[2 * j];
        RF[64 * j + 2 * lane + 1] = r == 2 ? -v[2 * j + 1] : v[2 * j + 1];
      }
    }
  }
  __syncwarp();
}

// The box (positions 0..3: lanes 0 and 1 of chunk 0, serial.hpp:47-52, NB =
// -M in frame 0) and the padding positions [mpos, 64 nc): never-violated
// zero rows with NB = -INF.
__device__ __forceinline__ void fs_fixup(float* X, float* Y, float* NB, int mpos, float M,
                                         int lane) {
  if (lane < 2) {
    sts2(X, lane, lane == 0 ? mk2(1.0f, -1.0f) : mk2(0.0f, 0.0f));
    sts2(Y, lane, lane == 0 ? mk2(0.0f, 0.0f) : mk2(1.0f, -1.0f));
    sts2(NB, lane, splat2(-M));
  }
  const int nc = (mpos + 63) >> 6;
  const int k = (mpos & ~1) + 2 * lane;  // pairs from the one holding mpos
  if (k < 64 * nc) {
    if (k >= mpos) {  // (mpos odd: the pair's first entry is real)
      X[k] = 0.0f;
      Y[k] = 0.0f;
      NB[k] = -INFINITY;
    }
    X[k + 1] = 0.0f;
    Y[k + 1] = 0.0f;
    NB[k + 1] = -INFINITY;
  }
  __syncwarp();
}

// The reference's fold (classify + apply_bound with owners, wu_apply) over
// positions [0, pi) on the widened original values: a from the insertion-order
// buffer (exact floats, box included), b from global memory through the
// staged permutation. Exact paths only.
template <typename P>
__device__ __forceinline__ Acc<double> fs_fold_exact(const KParams& p, int64_t off, uint32_t pi,
                                                     const Line<double>& l, double M,
                                                     const float* X, const float* Y,
                                                     const P* sperm) {
  const int lane = threadIdx.x & 31;
  const float* gb = static_cast<const float*>(p.b) + off;
  Acc<double> acc;
  acc.uL = -INFINITY;
  acc.uR = INFINITY;
  acc.oL = acc.oR = acc.par = kNone;
#pragma unroll 1
  for (uint32_t k0 = lane; k0 < pi; k0 += 32 * 8) {
    float vb[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t k = k0 + 32 * u;
      vb[u] = (k < pi && k >= 4) ? __ldg(gb + (uint32_t)sperm[k - 4]) : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t k = k0 + 32 * u;
      if (k < pi) {
        const double bb = k < 4 ? M : (double)vb[u];
        wu_apply((double)X[k], (double)Y[k], bb, l, p.eps_par, p.eps_feas, p.eps_hi, k, acc);
      }
    }
  }
  return acc;
}

// The reference's double event at position pi (cf. fx_exact_event).
template <typename P>
__device__ __noinline__ int fs_exact_event(const KParams& p, int64_t lp, int64_t off, int m,
                                           uint32_t pi, float cxf, float cyf, float Mf,
                                           uint32_t& pos0, uint32_t& pos1, double& xp, double& yp,
                                           const float* X, const float* Y, const P* sperm) {
  const double M = Mf;
  const double ob = pi < 4 ? M : (double)__ldg(static_cast<const float*>(p.b) + off + sperm[pi - 4]);
  const Line<double> l = boundary_of((double)X[pi], (double)Y[pi], ob);
  const Acc<double> ex = fs_fold_exact<P>(p, off, pi, l, M, X, Y, sperm);
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

// Move the frame to s: NB of every real position rewritten in place, from NB
// itself on the first reshift (-b exactly), else from the original b in
// global memory (streamed an LP ago: L2). Out of line: about one call per LP.
template <typename P>
__device__ __noinline__ void fs_reshift(const KParams& p, const float* X, const float* Y, float* NB,
                                        const P* sperm, int64_t off, float M, int mpos,
                                        bool shifted, float nsx, float nsy, PairConsts pk) {
  const int lane = threadIdx.x & 31;
  const Pair<float> SX = splat2(nsx), SY = splat2(nsy);
  const int nc = (mpos + 63) >> 6;
  const float* gbl = static_cast<const float*>(p.b) + off;
#pragma unroll 1
  for (int j0c = 0; j0c < nc; j0c += 4) {
    Pair<float> bo[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = j0c + u;
      const int k0 = 64 * j + 2 * lane;
      if (j < nc) {
        if (!shifted) {
          bo[u] = neg2(lds2(NB, 32 * j + lane));
        } else {
          float b0 = M, b1 = M;  // (box rows: b = M)
          if (k0 >= 4 && k0 < mpos) b0 = __ldg(gbl + (uint32_t)sperm[k0 - 4]);
          if (k0 + 1 >= 4 && k0 + 1 < mpos) b1 = __ldg(gbl + (uint32_t)sperm[k0 - 3]);
          bo[u] = mk2(b0, b1);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = j0c + u;
      const int k0 = 64 * j + 2 * lane;
      if (j < nc) {
        const Pair<float> bs =
            neg2(bshift2(lds2(X, 32 * j + lane), lds2(Y, 32 * j + lane), bo[u], SX, SY, pk));
        // padding rows keep NB = -INF
        sts2(NB, 32 * j + lane,
             mk2(k0 < mpos ? lo2(bs) : -INFINITY, k0 + 1 < mpos ? hi2(bs) : -INFINITY));
      }
    }
  }
  __syncwarp();
}

// Out-of-line forms of K4's exact helpers (K5 keeps its hot loop small).
template <typename P>
__device__ __noinline__ bool fs_exact_violates(const KParams& p, int64_t off, float Mf, uint32_t pos,
                                               uint32_t p0, uint32_t p1, bool stale, double& xp,
                                               double& yp) {
  return fx_exact_violates<P>(p, off, Mf, pos, p0, p1, stale, xp, yp);
}
__device__ __noinline__ void fs_exact_point(float hx, float hy, float hb, float ox, float oy,
                                            float ob, double& px, double& py) {
  fx_exact_point(hx, hy, hb, ox, oy, ob, px, py);
}

// Register budget: REGW warps per SM worth of registers (65536 / (32 REGW),
// rounded down to the allocation granule of 8); CTAs of at most REGW warps.
constexpr int fs_regs(int regw) { return (65536 / (32 * regw)) / 8 * 8 > 255 ? 255 : (65536 / (32 * regw)) / 8 * 8; }

template <typename P, int CAP, int NBUF, int REGW>
__global__ void __maxnreg__(fs_regs(REGW)) k_solve_fs(const __grid_constant__ KParams p) {
  using L = FsLayout<P, CAP>;
  constexpr int NC = L::kChunks;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int wic = threadIdx.x >> 5;
  const int W = (int)(blockDim.x >> 5);
  unsigned char* wbuf = smem + (size_t)wic * NBUF * L::kBuf;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)W * NBUF * L::kBuf) + wic * NBUF;
  const PairConsts pk = p.pk;
  const uint64_t policy = policy_evict_first();
  const float* gb = static_cast<const float*>(p.b);
  const bool hist = p.iter_hist != nullptr;

  if (lane < NBUF) mbar_init(bars + lane, 1);
  __syncwarp();

  const int32_t* list;
  int64_t n_list;
  resolve_list(p, list, n_list);
  const int64_t TW = p.total_warps;
  const int64_t j0 = (int64_t)blockIdx.x * W + wic;
  auto lp_of = [&](int64_t t) -> int64_t { return t < n_list ? (list ? (int64_t)list[t] : t) : -1; };
  // LPs [0, NBUF*TW) are dealt statically (warp w: w, w + TW, ...), the rest by ticket
  constexpr int64_t kStatic = NBUF;
  Header<float> h = unpack_header<L, float>(load_header_word<float>(p, lp_of(j0), lane), lp_of(j0));
  fs_issue<L, P>(p, h, wbuf, bars, policy, lane);
  int64_t lpB = NBUF == 2 ? lp_of(j0 + TW) : -1;
  uint32_t hB = NBUF == 2 ? load_header_word<float>(p, lpB, lane) : 0u;
  uint32_t ticket = atomic_add_if(p.counter, lane == 0, pk.zero);
  uint32_t phases = 0;  // mbarrier parity per buffer (bit q)
  int cur = 0;

  while (h.lp >= 0) {
    unsigned char* buf = wbuf + (NBUF == 2 ? cur * L::kBuf : 0);
    uint64_t* bar = bars + (NBUF == 2 ? cur : 0);
    mbar_wait(bar, (phases >> cur) & 1u);
    phases ^= 1u << cur;
    Header<float> hn;
    if constexpr (NBUF == 2) {
      // the other buffer held the previous LP: stage the next one now
      hn = unpack_header<L, float>(hB, lpB);
      fs_issue<L, P>(p, hn, wbuf + (cur ^ 1) * L::kBuf, bars + (cur ^ 1), policy, lane);
    }
    // claim one LP further ahead (its header is consumed one LP later)
    lpB = lp_of((int64_t)__shfl_sync(kFull, ticket, 0) + kStatic * TW);
    hB = load_header_word<float>(p, lpB, lane);
    ticket = atomic_add_if(p.counter, lane == 0, pk.zero);

    float* X = reinterpret_cast<float*>(buf);
    float* Y = reinterpret_cast<float*>(buf + L::kArr);
    float* NB = reinterpret_cast<float*>(buf + 2 * L::kArr);
    const P* sperm = reinterpret_cast<const P*>(buf + 3 * L::kArr);
    const int mj = h.ok ? h.m : 0;
    const int mpos = mj + 4;
    float A = 1.0f, B = fabsf(h.M);
    uint32_t pmax = 0;
    if (mj > 0) fs_permute<P, CAP>(buf, mj, h.M, lane, A, B, pmax);
    fs_fixup(X, Y, NB, mpos, h.M, lane);
    const bool bad = !h.ok || (mj > 0 && pmax >= (uint32_t)mj);

    // ---- solve (serial.hpp:159-188) -----------------------------------------
    const bool wild = !(A < 0x1p24f) || !(B < 0x1p62f) || !(fabsf(h.cx) < 0x1p100f) ||
                      !(fabsf(h.cy) < 0x1p100f) || !(fabsf(h.M) < 0x1p62f);
    const FxLP C = fx_lp_consts(p, A, B, h.cx, h.cy);
    FxFrame F = fx_frame(C, 0.0f, 0.0f);
    bool shifted = false;  // NB holds -b (exact) until the first reshift
    auto reshift = [&](float nsx, float nsy) {
      fx_count(p, kFxReshift, lane);
      fs_reshift<P>(p, X, Y, NB, sperm, h.off, h.M, mpos, shifted, nsx, nsy, pk);
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
    int c = 0;                                     // test cursor (64-position chunk)
    uint32_t mlo = 0xfffffffcu, mhi = 0xfffffffcu;  // resume masks of chunk c (the box: never tested)
    const int ncp = (mpos + 63) >> 6;
    bool running = !bad && !wild;
    bool need_exact_lp = !bad && wild;
    constexpr float cP = 7.35f * kU32 + 8.4f * kU64;
    while (running) {
      const float pmag = fmaxf(fabsf(ppx), fabsf(ppy));
      const float T_ = fmaf(C.A, fmaf(2.11f, epp, cP * pmag), F.KT);
      const float nT = -T_;
      const Pair<float> PX = splat2(ppx), PY = splat2(ppy);
      // ---- violation tests (core.hpp:111-113): stop at the first position
      // whose filtered residual e = a.p' - b' is not provably below the slack
      int pi = -1;
      auto hit = [&](int cc, uint32_t vlo, uint32_t vhi) {
        const int f = __ffs(vlo | vhi) - 1;
        const int odd = (vlo >> f) & 1u ? 0 : 1;
        pi = 64 * cc + 2 * f + odd;
        // resume inside this chunk right after pi
        const uint32_t above = f == 31 ? 0u : (kFull << (f + 1));
        mlo = above;
        mhi = odd ? above : (kFull << f);
        c = cc;
      };
      if (c < ncp) {
        // the resume chunk (masked), then two unmasked chunks per step
        const Pair<float> e =
            fma2(lds2(X, 32 * c + lane), PX, fma2(lds2(Y, 32 * c + lane), PY, lds2(NB, 32 * c + lane)));
        const uint32_t vlo = __ballot_sync(kFull, lo2(e) >= nT) & mlo;
        const uint32_t vhi = __ballot_sync(kFull, hi2(e) >= nT) & mhi;
        if (vlo | vhi) {
          hit(c, vlo, vhi);
        } else {
          int cc = c + 1;
#pragma unroll 1
          for (; cc + 1 < ncp; cc += 2) {
            const Pair<float> e0 = fma2(lds2(X, 32 * cc + lane), PX,
                                        fma2(lds2(Y, 32 * cc + lane), PY, lds2(NB, 32 * cc + lane)));
            const Pair<float> e1 = fma2(lds2(X, 32 * cc + 32 + lane), PX,
                                        fma2(lds2(Y, 32 * cc + 32 + lane), PY, lds2(NB, 32 * cc + 32 + lane)));
            const uint32_t a0 = __ballot_sync(kFull, lo2(e0) >= nT);
            const uint32_t a1 = __ballot_sync(kFull, hi2(e0) >= nT);
            const uint32_t b0 = __ballot_sync(kFull, lo2(e1) >= nT);
            const uint32_t b1 = __ballot_sync(kFull, hi2(e1) >= nT);
            if (a0 | a1 | b0 | b1) {
              if (a0 | a1) hit(cc, a0, a1);
              else hit(cc + 1, b0, b1);
              break;
            }
          }
          if (pi < 0 && cc < ncp) {
            const Pair<float> e0 = fma2(lds2(X, 32 * cc + lane), PX,
                                        fma2(lds2(Y, 32 * cc + lane), PY, lds2(NB, 32 * cc + lane)));
            const uint32_t a0 = __ballot_sync(kFull, lo2(e0) >= nT);
            const uint32_t a1 = __ballot_sync(kFull, hi2(e0) >= nT);
            if (a0 | a1) hit(cc, a0, a1);
          }
        }
      }
      if (pi < 0) break;
      const uint32_t upi = (uint32_t)pi;
      const float hx = X[pi], hy = Y[pi];
      float hnb = NB[pi];
      const float he = fmaf(hx, ppx, fmaf(hy, ppy, hnb));
      {
        // The candidate's own slack S = eps (1 + |b|) (core.hpp:65-67), |b|
        // from b' and the frame: proves "satisfied" or "violated" unless the
        // residual lies within the bound of it (cf. k_solve_fx).
        const float bo = fmaf(hx, F.sx, fmaf(hy, F.sy, -hnb));
        const float Sk = fmaf(C.eps, fabsf(bo), C.eps);
        const float tol = T_ + 6.0f * kU32 * fabsf(he) + 16.0f * kU32 * Sk;
        if (he < Sk - tol) continue;  // satisfied: resume after pi
        if (!(he > Sk + tol)) {
          fx_count(p, kFxTestFlag, lane);
          if (stale) fx_count(p, kFxLazy, lane);
          const bool v = fs_exact_violates<P>(p, h.off, h.M, upi, pos0, pos1, stale, xp, yp);
          stale = false;
          if (T_ > 16.0f * Sk) {
            // the band is wide (the optimum is far from the frame): move the
            // frame onto the exact optimum so the next tests are sharp
            reshift((float)xp, (float)yp);
            ppx = (float)(xp - (double)F.sx);
            ppy = (float)(yp - (double)F.sy);
            epp = kU32 * fmaxf(fabsf(ppx), fabsf(ppy)) +
                  2.0f * kU64 * (float)fmax(fabs(xp), fabs(yp)) + 0x1p-120f;
            hnb = NB[pi];  // the candidate's b' in the new frame
          }
          if (!v) continue;
        }
      }
      // ---- event at position pi: 1D LP over positions [0, pi) ----------------
      viol += 1;
      wu32 += upi;  // considered.size() (serial.hpp:176-179)
      if (hist && lane == 0) note_event(p, h.lp, upi);
      const float len2 = fmaf(hx, hx, hy * hy);
      const bool line_ok = (len2 >= 0x1p-100f) & (len2 <= 0x1p100f);
      const float rs = rsqrt_approx(len2), rl2 = rcp_approx(len2);
      const float dx = -hy * rs, dy = hx * rs;
      const float ac = fmaf(h.cx, dx, h.cy * dy);
      const bool fast = line_ok && fabsf(ac) > C.Ec;
      const bool take_right = ac > 0.0f;  // serial.hpp:102-108 (proved when fast)
      const float fdx = take_right ? -dx : dx, fdy = take_right ? -dy : dy;
      const Pair<float> NDX = splat2(-fdx), NDY = splat2(-fdy);
      const float Obig = 1.5f * C.B * rs;  // >= |o64| = |b_h|/|a_h|
      float hbp = -hnb;
      bool done = false;
      const int nfull = pi >> 6;
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
        const Pair<float> WX = splat2(wx), WY = splat2(wy);
#pragma unroll 2
        for (int j = 0; j < nfull; ++j) {
          const uint32_t k0 = 64u * (uint32_t)j + 2u * (uint32_t)lane;
          fx_fold2<false>(lds2(X, 32 * j + lane), lds2(Y, 32 * j + lane), lds2(NB, 32 * j + lane),
                          NDX, NDY, WX, WY, kn, ka, k0, k0 + 1, true, true, acc, pk);
        }
        if (pi & 63) {
          const int j = nfull;
          const uint32_t k0 = 64u * (uint32_t)j + 2u * (uint32_t)lane;
          fx_fold2<true>(lds2(X, 32 * j + lane), lds2(Y, 32 * j + lane), lds2(NB, 32 * j + lane),
                         NDX, NDY, WX, WY, kn, ka, k0, k0 + 1, k0 < upi, k0 + 1 < upi, acc, pk);
        }
        // ---- merge and certify (cf. k_solve_fx) ------------------------------
        const float G1 = warp_max_f(acc.h1);
        const uint32_t hold = __ballot_sync(kFull, acc.h1 == G1);
        const int hl = __ffs(hold) - 1;
        const int src = hl < 0 ? 0 : hl;
        const float G2 = warp_max_f(lane == hl ? acc.h2 : acc.h1);
        const float RL = warp_min_f(acc.rl);
        const float MAL = warp_min_f(acc.mal);
        const uint32_t own = __shfl_sync(kFull, acc.own, src);
        const float L1 = __shfl_sync(kFull, acc.l1, src);
        const bool cert = (MAL > C.Tpar) && __popc(hold) == 1 && own != kNone &&
                          fabsf(G1) < INFINITY && fabsf(L1) < INFINITY &&
                          (L1 > G2 + 4.0f * kU32 * (fabsf(L1) + fabsf(G2))) &&
                          (G1 + 4.0f * kU32 * (fabsf(G1) + fabsf(RL)) <= RL);
        const float q1 = 0.5f * (G1 + L1);  // the winner's quotient
        const float aG1 = fabsf(q1);
        if (cert) {
          // the reference's event resolves to the owner: the optimum is that
          // pair's intersection, exactly known, computed lazily
          const float E1 = 0.505f * (G1 - L1);
          pos0 = upi;
          pos1 = own;
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
        reshift(F.sx + fmaf(q1, fdx, wx), F.sy + fmaf(q1, fdy, wy));
        hbp = -NB[pi];  // the violated constraint's b' in the new frame
      }
      if (!done) {
        // the reference's double operations for this event
        fx_count(p, kFxExact, lane);
        const int r = fs_exact_event<P>(p, h.lp, h.off, mj, upi, h.cx, h.cy, h.M, pos0, pos1, xp,
                                        yp, X, Y, sperm);
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
      // the final optimum with the reference's operations: a from the buffer,
      // b from global memory (box rows: M)
      const float* gbl = gb + h.off;
      const float b0 = pos0 < 4 ? h.M : __ldg(gbl + (uint32_t)sperm[pos0 - 4]);
      const float b1 = pos1 < 4 ? h.M : __ldg(gbl + (uint32_t)sperm[pos1 - 4]);
      fs_exact_point(X[pos0], Y[pos0], b0, X[pos1], Y[pos1], b1, xp, yp);
    }
    if (st == 0 && (pos0 < 4 || pos1 < 4)) st = 2;
    // defining pair from the resident permutation
    int32_t pc = 0;
    if (lane < 2) {
      uint32_t pos = lane == 0 ? pos0 : pos1;
      if (st == 255) pos = kNone;
      const uint32_t q = (pos != kNone && pos >= 4) ? (uint32_t)sperm[min(pos - 4, (uint32_t)CAP - 1u)] : 0u;
      pc = pair_code(pos, q);
    }
    if constexpr (NBUF == 1) {
      // the buffer is free: stage the next LP into it
      __syncwarp();
      fence_proxy_async_smem();
      hn = unpack_header<L, float>(hB, lpB);
      fs_issue<L, P>(p, hn, wbuf, bars, policy, lane);
    } else {
      __syncwarp();
      fence_proxy_async_smem();  // (this buffer is restaged one LP from now)
    }
    if (lane < 2 && p.pair) p.pair[2 * h.lp + lane] = pc;
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
    }
    h = hn;
    if constexpr (NBUF == 2) cur ^= 1;
  }

  // Self-reset of the ticket counter by the last warp to finish (the fence
  // orders this warp's last, possibly unread, ticket claim before the count).
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
