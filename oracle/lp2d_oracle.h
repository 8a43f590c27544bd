/* ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference's batch 2D-LP solve path
 * (/root/reference/proj/include/lp2d/{core,rng,serial,generate,oracle}.hpp),
 * used as the parity checker for the CUDA path. Only tests/, the smoke() check
 * in __graft_entry__.py and bench.py's cpu_baseline / --impl reference leg may
 * load it. The product (paper_1902_04995_b200/) never links or calls it.
 *
 * Parity pinning: the solver is checked bit-for-bit against the unmodified
 * reference compiled from /root/reference (oracle/_ref, see oracle/Makefile)
 * and against the reference's own golden values (tests/golden/,
 * tests/test_oracle.py). Both entry points compute in double exactly like the
 * reference: *_d reads double inputs, *_f reads float inputs (the fp32
 * configs' storage) and widens them exactly, so *_f IS the reference applied
 * to the fp32-rounded instance (pinned against oracle/_ref on such instances
 * too). The status/defining-pair extension has no reference counterpart; it
 * follows the same operation order, is cross-checked against the reference's
 * brute-force vertex oracle (oracle.hpp:38-70) for m <= 512, and is pinned by
 * the committed fixtures.
 */
#ifndef LP2D_ORACLE_H
#define LP2D_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  LP2D_ORACLE_OPTIMAL = 0,
  LP2D_ORACLE_INFEASIBLE = 1,
  LP2D_ORACLE_UNBOUNDED = 2,
};
#define LP2D_ORACLE_NONE ((int32_t)0x80000000)

typedef struct lp2d_oracle_result {
  double x, y, value;          /* point and objective (0 when infeasible) */
  uint64_t violation_events;   /* serial.hpp:148-151 solve_stats */
  uint64_t work_units;
  int32_t pair[2];             /* defining pair: original index, box -> -1..-4 */
  int32_t status;              /* LP2D_ORACLE_* */
  int32_t pad;
} lp2d_oracle_result;

/* rng.hpp */
uint64_t lp2d_oracle_derive_seed(uint64_t base, uint64_t stream);
void lp2d_oracle_xoshiro_first(uint64_t seed, int n, uint64_t* out);
void lp2d_oracle_shuffle(int64_t m, uint64_t seed, uint32_t* order);
uint64_t lp2d_oracle_below(uint64_t seed, uint64_t n, int draws, uint64_t* out);

/* generate.hpp: one instance of kind 0 (feasible_random) or 1 (infeasible).
 * Writes m constraints, c[2], bound; witness[2] may be NULL. */
int lp2d_oracle_gen(int64_t m, uint64_t seed, int kind, double margin,
                    double* ax, double* ay, double* b, double* c,
                    double* bound_m, double* witness);

/* serial.hpp solve; single LP, original order + insertion order perm. */
int lp2d_oracle_solve_d(const double* ax, const double* ay, const double* b,
                        const uint32_t* perm, int64_t m, double cx, double cy,
                        double M, double eps_par, double eps_feas,
                        lp2d_oracle_result* out);
int lp2d_oracle_solve_f(const float* ax, const float* ay, const float* b,
                        const uint32_t* perm, int64_t m, float cx, float cy,
                        float M, double eps_par, double eps_feas,
                        lp2d_oracle_result* out);

/* Packed-SoA batch (same layout as the product's C-ABI, perm widened to u32),
 * solved with `threads` POSIX threads (1 = serial). */
int lp2d_oracle_solve_batch_d(int64_t n, const int64_t* offset,
                              const int32_t* m, const double* ax,
                              const double* ay, const double* b,
                              const uint32_t* perm, const double* c,
                              const double* M, double eps_par, double eps_feas,
                              int threads, lp2d_oracle_result* out);
int lp2d_oracle_solve_batch_f(int64_t n, const int64_t* offset,
                              const int32_t* m, const float* ax,
                              const float* ay, const float* b,
                              const uint32_t* perm, const float* c,
                              const float* M, double eps_par, double eps_feas,
                              int threads, lp2d_oracle_result* out);

/* Per-(block of W LPs, 1-based insertion step) violation counts, hist[(j /
 * W) * stride + step] (stride >= max m + 1): the input from which the
 * reference's lane_stats are rebuilt (the GPU's lp2d_out::iter_hist). */
int lp2d_oracle_iter_hist_d(int64_t n, const int64_t* offset, const int32_t* m,
                            const double* ax, const double* ay, const double* b,
                            const uint32_t* perm, const double* c, const double* M,
                            double eps_par, double eps_feas, int64_t W, int64_t stride,
                            uint32_t* hist);

/* oracle.hpp solve_bruteforce (O(m^3), m <= 512). Returns -2 above the cap. */
int lp2d_oracle_bruteforce(const double* ax, const double* ay, const double* b,
                           int64_t m, double cx, double cy, double M,
                           double eps_par, double eps_feas,
                           lp2d_oracle_result* out);

/* reduction.hpp:46-129 segmented_extremes (strategy 0 serialized, 1 tree,
 * 2 private-then-merge); -1 on the reference's invalid_argument cases. */
int lp2d_oracle_segmented_extremes(const double* in, int64_t n, int64_t contention,
                                   int strategy, double* out_min, double* out_max);
/* bench.hpp:256-257 inputs: xoshiro256pp(derive_seed(seed, stream)).in_range */
void lp2d_oracle_uniform(uint64_t seed, uint64_t stream, double lo, double hi, int64_t n,
                         double* out);

#ifdef __cplusplus
}
#endif
#endif
