/* lp2d_b200_gen.h — host-side instance synthesis for the batch solver.
 *
 * Restates the reference's seeded generators and permutation streams
 * (/root/reference/proj/include/lp2d/generate.hpp:60-91,174-189,
 * rng.hpp:13-68, serial.hpp:138-146) so that batches of the benchmark shapes
 * are produced bit-identically to lp2d::gen_mixed, multi-threaded, directly in
 * the packed layout of lp2d_b200.h. Builder-defined kinds (SURVEY.md §8(d)
 * configs 3 and 5) are marked as such; they have no reference counterpart.
 */
#ifndef LP2D_B200_GEN_H
#define LP2D_B200_GEN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  LP2D_GEN_FEASIBLE = 0,   /* generate.hpp:60-79 feasible_random          */
  LP2D_GEN_INFEASIBLE = 1, /* generate.hpp:81-91 infeasible               */
  /* builder-defined: feasible_random whose normals all lie within +-60
   * degrees of -c, so the optimum sits on the box (status unbounded). */
  LP2D_GEN_UNBOUNDED = 3,
};

/* rng.hpp:64-68 derive_seed */
uint64_t lp2dgen_derive_seed(uint64_t base, uint64_t stream);

/* serial.hpp:138-146 shuffle(m, seed) into order[0..m-1]. */
void lp2dgen_shuffle(int64_t m, uint64_t seed, uint32_t* order);

/* generate.hpp:143-155 gen({m, seed, kind, margin}) for one instance
 * (the instance seed is used directly, not derived). */
int lp2dgen_gen(int64_t m, uint64_t seed, int kind, double margin, double* ax,
                double* ay, double* b, double* c, double* bound_m);

/* Fill n LPs of the packed layout. LP j (global index g = first + j) is
 * generate.hpp gen({m[j], derive_seed(seed, 2g), kind[j], margin}) and its
 * insertion order shuffle(m[j], derive_seed(seed, 2g+1)) — exactly
 * lp2d::gen_mixed (generate.hpp:174-189) when kind is uniform and the sizes
 * cycle. kind may be NULL (all feasible). b and bound_m are multiplied by
 * bscale afterwards when bscale != 1 (covariant rescale, SURVEY.md §8(d)
 * config 3). perm may be NULL (no permutation work). threads <= 0 means all
 * hardware threads. Returns 0 or a negative code. */
int lp2dgen_fill(int64_t n, int64_t first, uint64_t seed, const int32_t* m,
                 const int64_t* offset, const uint8_t* kind, double margin,
                 double bscale, double* ax, double* ay, double* b,
                 uint32_t* perm, double* c, double* bound_m, int threads);

/* n draws of xoshiro256pp(derive_seed(seed, stream)).in_range(lo, hi)
 * (rng.hpp:42) — the contention benchmark's inputs with stream 0xC0
 * (bench.hpp:256-257). */
void lp2dgen_uniform(uint64_t seed, uint64_t stream, double lo, double hi, int64_t n,
                     double* out);

/* Heavy-tailed sizes: m_j = clamp(floor(xmin /
 * u^(1/alpha)), xmin, xmax) with u = xoshiro256pp(derive_seed(seed, 0xB0))
 * .unit() drawn in sequence, until sum(m) >= target or n_max reached.
 * Returns the count written to m. */
int64_t lp2dgen_pareto_sizes(uint64_t seed, double xmin, double alpha,
                             int32_t xmax, int64_t target_total, int64_t n_max,
                             int32_t* m);

#ifdef __cplusplus
}
#endif
#endif
