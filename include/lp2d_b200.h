/* lp2d_b200.h — C ABI of the B200-native batch 2D-LP solver.
 *
 * Drop-in boundary for the reference's batch-solve path:
 *
 *   lp2d::batch_result lp2d::solve_batch(const batch&, const block_config&,
 *                                        const tolerance&)
 *     /root/reference/proj/include/lp2d/batch.hpp:303-371
 *
 * The reference is header-only C++ with no ABI (proj/README.md:15); this
 * header is what a reference-side binding calls. Plain
 * pointers and sizes only: no exceptions, no C++ or torch types cross it.
 *
 * Semantics per LP (serial.hpp:159-188): maximise c.x subject to the four box
 * constraints x<=M, -x<=M, y<=M, -y<=M (positions 0..3, never permuted) and the
 * user constraints a.x <= b inserted in the order perm[0..m-1]. Results are
 * bit-identical to the reference's serial solver (double arithmetic) on the
 * stored instance: lp2dgpu_solve_f64 reads double inputs, lp2dgpu_solve_f32
 * reads float inputs (12 B per constraint in HBM), which are widened exactly,
 * so both return the reference's own doubles.
 */
#ifndef LP2D_B200_H
#define LP2D_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- return codes (0 = ok) ---------------------------------------------- */
enum {
  LP2D_OK = 0,
  LP2D_ERR_EMPTY_BATCH = -1,    /* batch.hpp:306   "empty batch"            */
  LP2D_ERR_PERM_COUNT = -2,     /* batch.hpp:307-310 one permutation per LP */
  LP2D_ERR_PERM_LENGTH = -3,    /* batch.hpp:311-316 length mismatch        */
  LP2D_ERR_BLOCK_WIDTH = -4,    /* batch.hpp:317-319 zero block width       */
  LP2D_ERR_LAYOUT = -5,         /* offsets not 8-aligned / segment too short */
  LP2D_ERR_BAD_PERM = -6,       /* a perm entry >= m: the C ABI reports it per
                                   LP (status LP2D_INVALID); the C++ and Python
                                   front-ends throw std::invalid_argument /
                                   ValueError on it                          */
  LP2D_ERR_ARG = -7,            /* null pointer / bad enum                  */
  LP2D_ERR_UNSUPPORTED = -8,    /* size class not built                     */
  LP2D_ERR_CUDA = -9,           /* CUDA runtime error (see last_error)      */
};

/* ---- per-LP status (the builder's extension of serial.hpp:34-43) -------- */
enum {
  LP2D_OPTIMAL = 0,     /* feasible, both defining constraints are user ones */
  LP2D_INFEASIBLE = 1,  /* solution::infeasible()                            */
  LP2D_UNBOUNDED = 2,   /* feasible, optimum held by a box edge (k < 4)      */
  LP2D_INVALID = 255,   /* malformed input for this LP (perm out of range)   */
  LP2D_MOCK = 254,      /* test-only mock devices (LP2D_B200_MOCK_DEVICES=N):
                           the host-mode shard/chunk driver ran without CUDA;
                           x = global LP index, y = shard, value = the chunk's
                           first LP, work_units = m. Not a solution.        */
};
/* pair entries: original constraint index, box position k -> -(k+1),
 * LP2D_PAIR_NONE when no constraint owns the endpoint. */
#define LP2D_PAIR_NONE ((int32_t)0x80000000)

enum { LP2D_MEM_HOST = 0, LP2D_MEM_DEVICE = 1 };
enum { LP2D_SCHED_NAIVE = 0, LP2D_SCHED_BALANCED = 1 };
enum { LP2D_PERM_U16 = 16, LP2D_PERM_U32 = 32 };

/* Packed structure-of-arrays batch (replaces the AoS std::vector<problem> of
 * serial.hpp:28-32 + batch.hpp:45-48).
 *   LP j owns elements [offset[j], offset[j] + m[j]) of ax, ay, b and perm.
 *   offset[j] must be a multiple of 8 and offset[j+1] - offset[j] >=
 *   round_up(m[j], 8) (16-byte bulk-copy granularity); lp2dgpu_pack_offsets()
 *   computes such offsets.
 *   perm[offset[j] + i] is the original index (0..m[j]-1) of the constraint
 *   inserted i-th (serial.hpp:126-146 permutation::order).
 *   c[2j], c[2j+1] is the objective, bound_m[j] the box half-width M.
 * Scalars are float for lp2dgpu_solve_f32 and double for lp2dgpu_solve_f64.
 * mem says whether every array is host or device memory. In device mode
 * max_m must be given (host scalar, max over m[j]) and min_m should be (a
 * lower bound; 0 if unknown): when both fall in one size class the batch is
 * solved by a single kernel, otherwise LPs are first binned by size class on
 * the device. In host mode both are computed. */
typedef struct lp2d_batch_soa {
  int64_t n;
  const int32_t* m;
  const int64_t* offset; /* [n+1] */
  const void* ax;
  const void* ay;
  const void* b;
  const void* perm;
  int32_t perm_bits; /* LP2D_PERM_U16 (needs m <= 65536) or LP2D_PERM_U32 */
  int32_t mem;       /* LP2D_MEM_HOST / LP2D_MEM_DEVICE */
  const void* c;     /* [2n] */
  const void* bound_m; /* [n] */
  int64_t max_m;
  int64_t min_m;
  /* Permutations from seeds (perm_from_seed != 0): LP j's insertion order is
   * shuffle(m[j], derive_seed(perm_seed, perm_mul * (perm_first + j) +
   * perm_add)) (serial.hpp:138-146 with rng.hpp:64-68), generated on the
   * device instead of copied in: (mul, add) = (2, 1) are gen_mixed's /
   * verify's streams (generate.hpp:186, bench.hpp:312), (1, 0) replicate's
   * (generate.hpp:165-166). Host mode: perm may be NULL (nothing is read);
   * device mode: perm is a device buffer the library fills (offset[n]
   * entries of perm_bits). Zero-initialised callers keep explicit perms. */
  int32_t perm_from_seed;
  int32_t perm_mul;
  int32_t perm_add;
  int32_t _pad;
  uint64_t perm_seed;
  int64_t perm_first;
} lp2d_batch_soa;

/* block_config (batch.hpp:50-58) + tolerance (core.hpp:59-68). */
typedef struct lp2d_opts {
  int32_t scheduler;   /* LP2D_SCHED_BALANCED (warp-cooperative work units,
                          default) or LP2D_SCHED_NAIVE (thread per LP) */
  int32_t block_width; /* must be > 0 (validated like batch.hpp:317); the GPU
                          schedule is fixed by the kernel, see DESIGN.md */
  int32_t n_gpus;      /* host mode: shard over this many visible devices
                          (0 = all); replaces block_config::workers */
  int32_t device;      /* device mode: device ordinal of the pointers; host
                          mode with n_gpus == 1: the device that solves (e.g.
                          a rank's local GPU; out of range = device 0) */
  void* stream;        /* device mode: cudaStream_t (NULL = legacy stream) */
  double eps_parallel; /* core.hpp:60 (1e-12) */
  double eps_feas;     /* core.hpp:61 (1e-9)  */
} lp2d_opts;

/* Outputs, n entries each (host or device per batch->mem). Optional members
 * may be NULL. x/y/value are double for both entry points (the reference's
 * solution::point / value type, serial.hpp:34-43). */
typedef struct lp2d_out {
  uint8_t* status;
  void* x;
  void* y;
  void* value;
  int32_t* pair;              /* [2n], optional */
  uint32_t* violation_events; /* optional, serial.hpp:148-151 */
  uint64_t* work_units;       /* optional */
  /* optional: violations per (block, insertion step), the input of the
   * reference's lane_stats (batch.hpp:84-120, block semantics of run_block,
   * :149-294) rebuilt on the host (lane_stats.hpp). Block b holds LPs
   * [b*W, (b+1)*W) for W = opts->block_width; entry b*(max_m+1) + iter
   * counts the LPs of block b that violated at 1-based insertion step iter.
   * ceil(n/W) * (max_m+1) entries, max_m = the batch's largest m; the library
   * zeroes it. */
  uint32_t* iter_hist;
} lp2d_out;

void lp2dgpu_default_opts(lp2d_opts* opts);

/* Solve a batch. Host mode: shards the batch over n_gpus devices (LP ranges
 * balanced by sum(m + 4), one host thread per device); each shard is cut into
 * chunks (LP2D_B200_CHUNK_ELEMS elements, default 4 Mi) pipelined over two
 * device slots (H2D of the next chunk overlaps the solve of the current one;
 * pageable inputs are staged through pinned buffers, pinned ones are DMA'd
 * directly; results return on a second copy stream); returns when every
 * result is in place. The layout contract is checked before any LP of a
 * chunk is sent (single-GPU calls check chunk by chunk, so on an error the
 * outputs of earlier chunks may already be written: outputs are unspecified
 * after any error). Device mode: enqueues on opts->stream and returns
 * without synchronising. */
int lp2dgpu_solve_f32(const lp2d_batch_soa* batch, const lp2d_opts* opts,
                      lp2d_out* out);
int lp2dgpu_solve_f64(const lp2d_batch_soa* batch, const lp2d_opts* opts,
                      lp2d_out* out);

/* Offsets for a batch of sizes m[0..n-1] satisfying the layout contract;
 * writes offset[0..n] and returns the total element count. */
int64_t lp2dgpu_pack_offsets(int64_t n, const int32_t* m, int64_t* offset);

/* Multi-GPU partitioner used by host mode: contiguous LP
 * ranges [cut[g], cut[g+1]) balanced by sum(m + 4); cut has parts+1 entries.
 * Pure host code (no CUDA). Returns 0 or LP2D_ERR_ARG. */
int lp2dgpu_partition(int64_t n, const int32_t* m, int32_t parts, int64_t* cut);

/* Device-side permutation generation (serial.hpp:138-146 shuffle with
 * rng.hpp:64-68 seeds): perm for LP j is shuffle(m[j], seeds[j]). Device
 * pointers, enqueued on stream. perm_bits as in lp2d_batch_soa. */
int lp2dgpu_shuffle_device(int64_t n, const int32_t* m, const int64_t* offset,
                           const uint64_t* seeds, void* perm, int32_t perm_bits,
                           int32_t device, void* stream);

/* Device-side instance synthesis (replaces the host
 * path of lp2d::gen_mixed, /root/reference/proj/include/lp2d/generate.hpp:
 * 60-91, 174-189, for batches that should not cross PCIe). LP j (global index
 * g = first + j) is gen({m[j], derive_seed(seed, 2g), kind[j], margin}) with
 * insertion order shuffle(m[j], derive_seed(seed, 2g+1)), written in the
 * packed layout at offset[j]; b and bound_m scaled by bscale. kind as in
 * lp2d_b200_gen.h (NULL: all feasible; an infeasible LP needs m >= 1, else it
 * is generated feasible). The integer streams (seeds, draws, permutations)
 * are bit-identical to lp2dgen_fill; cos/sin are the device's (an ulp or two
 * from glibc's). scalar_bits 32 stores the fp64 instance rounded to float
 * (as lp2dgen_fill + a cast). perm may be NULL. Device pointers, enqueued on
 * stream. */
int lp2dgpu_generate_device(int64_t n, int64_t first, uint64_t seed, const int32_t* m,
                            const int64_t* offset, const uint8_t* kind, double margin,
                            double bscale, int32_t scalar_bits, void* ax, void* ay, void* b,
                            void* perm, int32_t perm_bits, void* c, void* bound_m,
                            int32_t device, void* stream);

/* ---- contention microbenchmark -------------------
 * Segmented extremes: out_min[g] / out_max[g] = min / max of the g-th
 * consecutive group of `contention` values of in[0..n) — replaces
 * lp2d::segmented_extremes (reduction.hpp:46-129) with the GPU update
 * disciplines of the paper's Fig. atomicComp. Every strategy returns the
 * same values (min/max are exact); NaNs are ignored like std::fmin/fmax.
 * Device pointers, enqueued on `stream`. Errors as reduction.hpp:52-64
 * (contention < 1, n not a multiple of contention: LP2D_ERR_ARG). */
enum {
  LP2D_REDUCE_SHARED_ATOMIC = 0, /* shared-memory atomics (serialized update) */
  LP2D_REDUCE_TREE = 1,          /* halving-stride tree in shared memory      */
  LP2D_REDUCE_PRIVATE_MERGE = 2, /* private partials, merged per warp         */
  LP2D_REDUCE_GLOBAL_ATOMIC = 3, /* global-memory atomics                     */
  LP2D_REDUCE_CUB = 4,           /* cub::DeviceSegmentedReduce (library)      */
};
int lp2dgpu_segmented_extremes(const double* in, int64_t n, int64_t contention,
                               int32_t strategy, double* out_min, double* out_max,
                               int32_t device, void* stream);

/* Measurement hook of the fp32-storage kernel (K4): with the environment
 * variable LP2D_B200_FX_STATS=1 the kernels count events, first-pass
 * certificates, frame shifts, exact (double) events, uncertain tests, lazy
 * exact optima, whole-LP exact solves (8 counters, summed over calls).
 * Copies them into out[0..7] (reset if reset != 0) and returns 8, or 0 when
 * counting is off. */
int lp2dgpu_fx_stats(uint64_t* out, int reset);

/* Number of visible CUDA devices (0 when none). */
int lp2dgpu_device_count(void);

/* Number of kernels this library has enqueued so far (all devices, all
 * calls; monotonic). A solve of a uniform batch is one launch; a mixed batch
 * adds the two binning kernels and one launch per non-empty size class. */
uint64_t lp2dgpu_kernel_launches(void);

/* Thread-local message for the last non-zero return code. */
const char* lp2dgpu_last_error(void);

/* Library build identification string. */
const char* lp2dgpu_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LP2D_B200_H */
