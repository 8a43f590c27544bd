/* ORACLE — test infrastructure only (see oracle/lp2d_oracle.c header).
 *
 * Scalar-generic body of the CPU restatement of the reference's serial
 * Seidel solver. Included twice by lp2d_oracle.c: arithmetic type T=double
 * always (the reference computes in double), storage type S=double (fp64
 * configs) or S=float (fp32 configs: the fp32-stored instance, widened
 * exactly to double on load, so the result is the reference's own result on
 * the fp32-rounded instance). Every expression follows the reference
 * operation by operation (no FMA contraction: the file is compiled with
 * -ffp-contract=off), so it is bit-identical to
 * /root/reference/proj/include/lp2d.
 *
 * Macros expected: T, S, SUF, SQRT, FABS, FMAX, FMIN.
 */

#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)
#define FN(name) CAT(name, SUF)

/* core.hpp:65-67  tolerance::feas_slack(bound) = eps_feas * (1 + |bound|) */
static inline T FN(feas_slack_)(T eps_feas, T bound) {
  return eps_feas * ((T)1 + FABS(bound));
}

/* core.hpp:111-113  satisfied(h, p) = a.x*p.x + a.y*p.y <= b + feas_slack(b) */
static inline int FN(satisfied_)(T ax, T ay, T b, T px, T py, T eps_feas) {
  return ax * px + ay * py <= b + FN(feas_slack_)(eps_feas, b);
}

typedef struct {
  T ox, oy, dx, dy;
} FN(line_);

/* core.hpp:70-75  boundary_of: len2 = a.a; len = sqrt(len2);
 * origin = (b/len2) * a; dir = (1/len) * perp(a), perp(v) = (-v.y, v.x). */
static inline FN(line_) FN(boundary_of_)(T ax, T ay, T b) {
  FN(line_) l;
  const T len2 = ax * ax + ay * ay;
  const T len = SQRT(len2);
  const T s = b / len2;
  const T r = (T)1 / len;
  l.ox = s * ax;
  l.oy = s * ay;
  l.dx = r * (-ay);
  l.dy = r * ax;
  return l;
}

/* Folded 1D interval (serial.hpp:64-90) extended with the owning positions
 * of both endpoints (builder extension).
 * Ties keep the smallest position: positions are visited in increasing
 * order and only a strict improvement moves the owner. */
typedef struct {
  T u_left, u_right;
  int infeasible;
  int64_t own_left, own_right; /* -1 = none */
  int64_t first_par_infeasible; /* smallest parallel-infeasible position */
} FN(interval_);

/* core.hpp:96-109 classify + serial.hpp:64-81 apply_bound, for the
 * constraint at considered position k. */
static inline void FN(classify_apply_)(FN(interval_) * acc, T ax, T ay, T b,
                                       const FN(line_) * l, T eps_par,
                                       T eps_feas, int64_t k) {
  const T along = ax * l->dx + ay * l->dy;
  if (FABS(along) <= eps_par * SQRT(ax * ax + ay * ay)) {
    const int inside = ax * l->ox + ay * l->oy <= b + FN(feas_slack_)(eps_feas, b);
    if (!inside) {
      acc->infeasible = 1;
      if (acc->first_par_infeasible < 0) acc->first_par_infeasible = k;
    }
    return;
  }
  const T sigma = (b - (ax * l->ox + ay * l->oy)) / along;
  if (along > (T)0) {
    if (sigma < acc->u_right) acc->own_right = k;
    acc->u_right = FMIN(acc->u_right, sigma);
  } else {
    if (sigma > acc->u_left) acc->own_left = k;
    acc->u_left = FMAX(acc->u_left, sigma);
  }
}

/* serial.hpp:47-52 box_constraints: x<=M, -x<=M, y<=M, -y<=M. */
static inline void FN(box_)(int k, T M, T* ax, T* ay, T* b) {
  static const double bx[4] = {1.0, -1.0, 0.0, 0.0};
  static const double by[4] = {0.0, 0.0, 1.0, -1.0};
  *ax = (T)bx[k];
  *ay = (T)by[k];
  *b = M;
}

/* serial.hpp:159-188 solve (plus the builder's status/pair extension).
 * Inputs are one LP in the original constraint order, with the insertion
 * order perm (indices 0..m-1). perm may be NULL for identity order.
 * Returns 0 on success, -1 if perm is not a permutation index set. */
static int FN(solve_hist_)(const S* cax, const S* cay, const S* cb,
                           const uint32_t* perm, int64_t m, S cx_s, S cy_s, S M_s,
                           double eps_par_d, double eps_feas_d,
                           lp2d_oracle_result* out, uint32_t* hist_row);

int FN(lp2d_oracle_solve_)(const S* cax, const S* cay, const S* cb,
                           const uint32_t* perm, int64_t m, S cx_s, S cy_s, S M_s,
                           double eps_par_d, double eps_feas_d,
                           lp2d_oracle_result* out) {
  return FN(solve_hist_)(cax, cay, cb, perm, m, cx_s, cy_s, M_s, eps_par_d, eps_feas_d, out,
                         NULL);
}

/* The same solve, additionally counting each violation at its 1-based
 * insertion step into hist_row[step] (lane_stats reconstruction tests). */
static int FN(solve_hist_)(const S* cax, const S* cay, const S* cb,
                           const uint32_t* perm, int64_t m, S cx_s, S cy_s, S M_s,
                           double eps_par_d, double eps_feas_d,
                           lp2d_oracle_result* out, uint32_t* hist_row) {
  const T eps_par = (T)eps_par_d;
  const T eps_feas = (T)eps_feas_d;
  const T cx = (T)cx_s, cy = (T)cy_s, M = (T)M_s;
  /* serial.hpp:56-58 initial_optimum: zero components tie toward +M. */
  T px = cx < (T)0 ? -M : M;
  T py = cy < (T)0 ? -M : M;
  /* initial defining pair: the two box positions through the start corner */
  int64_t pair0 = cx < (T)0 ? 1 : 0;
  int64_t pair1 = cy < (T)0 ? 3 : 2;
  uint64_t viol = 0, wu = 0;
  int infeasible = 0;
  const T cnorm_thr = eps_par * SQRT(cx * cx + cy * cy);

  for (int64_t i = 0; i < m; ++i) {
    const int64_t oi = perm ? (int64_t)perm[i] : i;
    if (oi < 0 || oi >= m) return -1;
    const T hx = (T)cax[oi], hy = (T)cay[oi], hb = (T)cb[oi];
    if (FN(satisfied_)(hx, hy, hb, px, py, eps_feas)) continue;
    viol += 1;
    wu += (uint64_t)(4 + i);
    if (hist_row) hist_row[i + 1] += 1;
    const FN(line_) l = FN(boundary_of_)(hx, hy, hb);
    FN(interval_) acc;
    acc.u_left = -(T)INFINITY;
    acc.u_right = (T)INFINITY;
    acc.infeasible = 0;
    acc.own_left = acc.own_right = -1;
    acc.first_par_infeasible = -1;
    /* considered positions 0..3 = box, 4+k = user constraint perm[k] */
    for (int k = 0; k < 4; ++k) {
      T bx, by, bb;
      FN(box_)(k, M, &bx, &by, &bb);
      FN(classify_apply_)(&acc, bx, by, bb, &l, eps_par, eps_feas, k);
    }
    for (int64_t k = 0; k < i; ++k) {
      const int64_t ok = perm ? (int64_t)perm[k] : k;
      FN(classify_apply_)(&acc, (T)cax[ok], (T)cay[ok], (T)cb[ok], &l, eps_par, eps_feas,
                          4 + k);
    }
    /* serial.hpp:95-111 resolve_on_line */
    if (acc.infeasible) {
      infeasible = 1;
      pair0 = 4 + i;
      pair1 = acc.first_par_infeasible;
      break;
    }
    const T scale = FMAX(FABS(acc.u_left), FABS(acc.u_right));
    if (acc.u_left > acc.u_right + FN(feas_slack_)(eps_feas, scale)) {
      infeasible = 1;
      pair0 = 4 + i;
      pair1 = acc.own_left;
      break;
    }
    const T along = cx * l.dx + cy * l.dy;
    T t;
    int64_t owner;
    if (FABS(along) <= cnorm_thr) {
      t = acc.u_left;
      owner = acc.own_left;
    } else if (along > (T)0) {
      t = acc.u_right;
      owner = acc.own_right;
    } else {
      t = acc.u_left;
      owner = acc.own_left;
    }
    px = l.ox + t * l.dx;
    py = l.oy + t * l.dy;
    pair0 = 4 + i;
    pair1 = owner;
  }

  out->violation_events = viol;
  out->work_units = wu;
  /* export positions: box k -> -(k+1); user position 4+j -> perm[j] */
  {
    int64_t pr[2] = {pair0, pair1};
    int32_t ex[2];
    for (int q = 0; q < 2; ++q) {
      if (pr[q] < 0)
        ex[q] = LP2D_ORACLE_NONE;
      else if (pr[q] < 4)
        ex[q] = (int32_t)(-(pr[q] + 1));
      else
        ex[q] = (int32_t)(perm ? perm[pr[q] - 4] : (uint32_t)(pr[q] - 4));
    }
    out->pair[0] = ex[0];
    out->pair[1] = ex[1];
  }
  if (infeasible) {
    out->status = LP2D_ORACLE_INFEASIBLE;
    out->x = 0.0;
    out->y = 0.0;
    out->value = 0.0;
    return 0;
  }
  {
    const int unbounded = (pair0 >= 0 && pair0 < 4) || (pair1 >= 0 && pair1 < 4);
    out->status = unbounded ? LP2D_ORACLE_UNBOUNDED : LP2D_ORACLE_OPTIMAL;
  }
  out->x = (double)px;
  out->y = (double)py;
  /* serial.hpp:187 objective_value(c, x) */
  out->value = (double)(cx * px + cy * py);
  return 0;
}

/* Violation histogram per (block of W LPs, insertion step): the input of the
 * reference's lane_stats (batch.hpp:149-294), see include/lp2d_b200.h. */
int FN(lp2d_oracle_iter_hist_)(int64_t n, const int64_t* offset, const int32_t* m,
                               const S* ax, const S* ay, const S* b,
                               const uint32_t* perm, const S* c, const S* M,
                               double eps_par, double eps_feas, int64_t W,
                               int64_t stride, uint32_t* hist) {
  for (int64_t j = 0; j < n; ++j) {
    const int64_t o = offset[j];
    lp2d_oracle_result r;
    const int rc = FN(solve_hist_)(ax + o, ay + o, b + o, perm ? perm + o : NULL, m[j],
                                   c[2 * j], c[2 * j + 1], M[j], eps_par, eps_feas, &r,
                                   hist + (j / W) * stride);
    if (rc) return rc;
  }
  return 0;
}

/* Batch over the packed SoA layout (offsets into ax/ay/b/perm). */
static int FN(serial_batch_)(int64_t n, const int64_t* offset,
                                 const int32_t* m, const S* ax, const S* ay,
                                 const S* b, const uint32_t* perm, const S* c,
                                 const S* M, double eps_par, double eps_feas,
                                 lp2d_oracle_result* out) {
  for (int64_t j = 0; j < n; ++j) {
    const int64_t o = offset[j];
    const int rc = FN(lp2d_oracle_solve_)(ax + o, ay + o, b + o,
                                          perm ? perm + o : NULL, m[j],
                                          c[2 * j], c[2 * j + 1], M[j],
                                          eps_par, eps_feas, &out[j]);
    if (rc) return rc;
  }
  return 0;
}

#undef FN
#undef CAT
#undef CAT2
