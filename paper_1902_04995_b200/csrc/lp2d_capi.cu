// lp2d_capi.cu — C ABI (include/lp2d_b200.h) over the sm_100a kernels.
//
// Replaces lp2d::solve_batch (/root/reference/proj/include/lp2d/batch.hpp:
// 303-371): same validation and error cases (:305-320, returned as codes, not
// exceptions), the reference's jthread block pool (:335-351) replaced by
// LP-index sharding over GPUs (one host thread per device) and, inside a GPU,
// by warps claiming LPs from an atomic ticket.
#include <algorithm>
#include <cmath>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/lp2d_b200.h"
#include "lp2d_kernels.cuh"
#include "lp2d_reduce.cuh"

using namespace lp2d_b200;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(expr)                                                     \
  do {                                                                     \
    cudaError_t e_ = (expr);                                               \
    if (e_ != cudaSuccess) {                                               \
      return fail(LP2D_ERR_CUDA, std::string(#expr) + ": " +               \
                                     cudaGetErrorString(e_));              \
    }                                                                      \
  } while (0)

// Kernels enqueued by this library (all devices), lp2dgpu_kernel_launches().
std::atomic<uint64_t> g_launches{0};
inline void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// Ticket counter pairs, handed out round robin; a kernel leaves its pair at
// zero when its last warp finishes. A pair is reused after kCounterSlots
// launches on the device, so two launches could only share one if 2^16
// launches were in flight at once (each solve issues at most ~16).
constexpr int kCounterSlots = 1 << 16;

// Per-device state: ticket counters (self-resetting, round-robin slots) and a
// grow-only scratch arena for host-mode calls.
struct DeviceState {
  std::mutex mu;
  bool init = false;
  int sm_count = 0;
  uint32_t* counters = nullptr;
  std::atomic<uint32_t> next_slot{0};
  void* arena = nullptr;
  size_t arena_bytes = 0;
  cudaStream_t stream = nullptr;
  // fork/join of size-class launches (mixed batches)
  std::mutex fork_mu;
  cudaStream_t cls_stream[16] = {};
  cudaEvent_t cls_event[17] = {};
  // Host mode with perm_from_seed: the large LPs' permutations are shuffled
  // on aux while the rest of the chunk proceeds (see PermWait).
  cudaStream_t aux = nullptr;
  cudaEvent_t perm_ev = nullptr;
  // Stream-ordered workspace pool (binning lists) that keeps its memory:
  // the default pool returns freed memory at every synchronisation, making
  // the next allocation remap it (milliseconds, randomly).
  cudaMemPool_t pool = nullptr;
};

DeviceState g_dev[64];

// The pending wait of a split shuffle (shuffle_seeded with split): only size
// classes that can hold an LP with m > wait_m wait for the device's perm_ev.
// Set and consumed by the same host thread (the shard's, holding the
// device's mu), so a concurrent device-mode call on another thread never
// sees it.
struct PermWait {
  int dev = -1;
  int64_t wait_m = INT64_MAX;
};
thread_local PermWait t_perm_wait;

// Restores the caller's current device (torch and others rely on it).
struct DeviceGuard {
  int prev = -1;
  DeviceGuard() { cudaGetDevice(&prev); }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

int ensure_device(int dev) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || dev < 0 || dev >= ndev || dev >= 64)
    return fail(LP2D_ERR_ARG, "bad device ordinal " + std::to_string(dev));
  DeviceState& d = g_dev[dev];
  std::lock_guard<std::mutex> lock(d.mu);
  if (d.init) return 0;
  CUDA_TRY(cudaSetDevice(dev));
  CUDA_TRY(cudaDeviceGetAttribute(&d.sm_count, cudaDevAttrMultiProcessorCount, dev));
  CUDA_TRY(cudaMalloc(&d.counters, sizeof(uint32_t) * 2 * kCounterSlots));
  CUDA_TRY(cudaMemset(d.counters, 0, sizeof(uint32_t) * 2 * kCounterSlots));
  CUDA_TRY(cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking));
  for (auto& cs : d.cls_stream) CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  for (auto& ce : d.cls_event) CUDA_TRY(cudaEventCreateWithFlags(&ce, cudaEventDisableTiming));
  CUDA_TRY(cudaStreamCreateWithFlags(&d.aux, cudaStreamNonBlocking));
  CUDA_TRY(cudaEventCreateWithFlags(&d.perm_ev, cudaEventDisableTiming));
  cudaMemPoolProps props = {};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  CUDA_TRY(cudaMemPoolCreate(&d.pool, &props));
  uint64_t keep = UINT64_MAX;
  CUDA_TRY(cudaMemPoolSetAttribute(d.pool, cudaMemPoolAttrReleaseThreshold, &keep));
  CUDA_TRY(cudaDeviceSynchronize());
  d.init = true;
  return 0;
}

uint32_t* take_counter(int dev) {
  DeviceState& d = g_dev[dev];
  const uint32_t s = d.next_slot.fetch_add(1) % kCounterSlots;
  return d.counters + 2 * s;
}

// Register slot classes: NS slots hold m + 4 positions (box included).
constexpr int kSlotClasses[] = {1, 2, 4, 5, 6, 9, 10, 18, 33, 65, 129};
constexpr int kNumSlotClasses = (int)(sizeof(kSlotClasses) / sizeof(kSlotClasses[0]));
static_assert(kNumSlotClasses <= kMaxSlotClasses, "BinSpec::slots holds every register class");
static_assert(kNumSlotClasses + 1 <= 16, "host_counts holds every class + the large class");
static_assert(kLaneMaxM + 1 + kNumSlotClasses + 64 <= kMaxBins, "bins fit kMaxBins");

template <typename T>
constexpr int max_nslot() {
  // warp classes up to m <= 2076; larger LPs: the CTA kernel (one LP per CTA,
  // every thread of the CTA dealt its work units). Measured per uniform batch
  // (B200, per 2^13 LPs / 2^12 at m = 4000): fp32 storage m = 2100 459 vs 520
  // us, 3000 533 vs 577, 4000 339 vs 412; fp64 m = 2100 449 vs 688, 3000 859
  // vs 886, 4000 505 vs 572; at m <= 2000 the warp classes win (m = 2000: 356
  // vs 450 fp32, 366 vs 435 fp64).
  return 65;
}

// Eps_par rounded up by 2^-10 (relative), in T: the parallel-filter factor.
template <typename T>
double eps_hi_of(double eps_par) {
  const T e = (T)eps_par;
  T hi = (T)((double)e * (1.0 + 1.0 / 1024.0));
  if ((double)hi < (double)e * (1.0 + 1.0 / 1024.0)) hi = std::nextafter(hi, (T)INFINITY);
  return (double)hi;
}

// Late-TMA classes: the CTA shape (1..8 warps) with the most resident warps
// under the shared-memory and register limits is picked at launch, and a
// launch whose LPs all have m <= 1024 uses the CAP = 1024 layout of the
// config-2 class (14.4 KB per warp: 16 warps/SM instead of 15).
template <typename T, typename P, int NS, int NT, int CAP>
int launch_late_tma_cap(KParams kp, int dev, cudaStream_t stream) {
  using L = WarpLayout<T, P, NS, NT, CAP>;
  auto kern = k_solve_warp<T, P, NS, NT, CAP>;
  struct Shape {
    int warps = 0, blocks = 0;
  };
  static Shape shape[64];
  static std::mutex mu;  // host threads of a multi-GPU solve initialise concurrently
  std::unique_lock<std::mutex> lock(mu);
  if (!shape[dev].warps) {
    int optin = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    Shape best;
    for (int w = 1; w <= L::kMaxWarpsRt; ++w) {
      int b = 0;
      CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, w * 32,
                                                             (size_t)w * (L::kBuf + 8)));
      if (b * w > best.blocks * best.warps) best = Shape{w, b};
    }
    if (best.blocks < 1) return fail(LP2D_ERR_CUDA, "warp kernel does not fit on an SM");
    shape[dev] = best;
  }
  const Shape sh = shape[dev];
  lock.unlock();
  const size_t smem = (size_t)sh.warps * (L::kBuf + 8);
  const int64_t want = (kp.n_list + sh.warps - 1) / sh.warps;
  const int64_t maxb = (int64_t)sh.blocks * g_dev[dev].sm_count;
  const int grid = (int)std::max<int64_t>(1, std::min(want, maxb));
  kp.total_warps = grid * sh.warps;
  kp.counter = take_counter(dev);
  kern<<<grid, sh.warps * 32, smem, stream>>>(kp);
  note_launch();
  CUDA_TRY(cudaGetLastError());
  return 0;
}

template <typename T, typename P, int NS, int NT>
int launch_late_tma(KParams kp, int64_t max_m, int dev, cudaStream_t stream) {
  if constexpr (NS + NT == 33) {
    if (max_m > 0 && max_m <= 1024) return launch_late_tma_cap<T, P, NS, NT, 1024>(kp, dev, stream);
  }
  return launch_late_tma_cap<T, P, NS, NT, 0>(kp, dev, stream);
}

template <typename T, typename P, int NS, int NT = 0>
int launch_warp_kernel(KParams kp, int dev, cudaStream_t stream, int64_t max_m = 0) {
  using L = WarpLayout<T, P, NS, NT>;
  if constexpr (L::kLateTma) return launch_late_tma<T, P, NS, NT>(kp, max_m, dev, stream);
  constexpr int kWarpsPerCta = L::kWarps;
  auto kern = k_solve_warp<T, P, NS, NT>;
  static int blocks_per_sm[64] = {0};
  static std::mutex mu;  // concurrent first use from multi-GPU host threads
  std::lock_guard<std::mutex> lock(mu);
  // (experiment knob: LP2D_B200_SMEM_PAD bytes of extra shared memory per CTA
  // lower the resident warps, for occupancy-sensitivity measurements)
  static const size_t pad = [] {
    const char* e = std::getenv("LP2D_B200_SMEM_PAD");
    return e ? (size_t)std::atol(e) : (size_t)0;
  }();
  const size_t smem = L::kSmem + pad;
  if (!blocks_per_sm[dev]) {
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    int b = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, kWarpsPerCta * 32,
                                                           smem));
    if (b < 1) return fail(LP2D_ERR_CUDA, "warp kernel does not fit on an SM");
    blocks_per_sm[dev] = b;
  }
  const int64_t want = (kp.n_list + kWarpsPerCta - 1) / kWarpsPerCta;
  const int64_t maxb = (int64_t)blocks_per_sm[dev] * g_dev[dev].sm_count;
  const int grid = (int)std::max<int64_t>(1, std::min(want, maxb));
  kp.total_warps = grid * kWarpsPerCta;
  kp.counter = take_counter(dev);
  kern<<<grid, kWarpsPerCta * 32, smem, stream>>>(kp);
  note_launch();
  CUDA_TRY(cudaGetLastError());
  return 0;
}

// Tiny class (m <= 28): lane-per-LP kernel (k_solve_lanes), 32 LPs per warp.
// LP2D_B200_TINY=warp selects the warp-per-LP kernel instead (A/B switch).
bool tiny_uses_lanes() {
  static const bool lanes = [] {
    const char* e = std::getenv("LP2D_B200_TINY");
    return !(e && std::strcmp(e, "warp") == 0);
  }();
  return lanes;
}

template <typename T, typename P, int MAXM = kLaneMaxM, typename S = T>
int launch_lane_kernel(KParams kp, int dev, cudaStream_t stream) {
  auto kern = k_solve_lanes<T, P, MAXM, S>;
  constexpr size_t smem = LaneTile<S, MAXM>::kSmem;
  static int blocks_per_sm[64] = {0};
  static std::mutex mu;  // concurrent first use from multi-GPU host threads
  std::lock_guard<std::mutex> lock(mu);
  if (!blocks_per_sm[dev]) {
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int b = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, kLaneWarps * 32, smem));
    if (b < 1) return fail(LP2D_ERR_CUDA, "lane kernel does not fit on an SM");
    blocks_per_sm[dev] = b;
  }
  const int64_t groups = (kp.n_list + 31) / 32;
  const int64_t want = (groups + kLaneWarps - 1) / kLaneWarps;
  const int64_t maxb = (int64_t)blocks_per_sm[dev] * g_dev[dev].sm_count;
  const int grid = (int)std::max<int64_t>(1, std::min(want, maxb));
  kp.total_warps = grid * kLaneWarps;
  kp.counter = take_counter(dev);
  kern<<<grid, kLaneWarps * 32, smem, stream>>>(kp);
  note_launch();
  CUDA_TRY(cudaGetLastError());
  return 0;
}

template <typename T>
constexpr int n_reg_classes() {
  int n = 0;
  for (int ns : kSlotClasses)
    if (ns <= max_nslot<T>()) ++n;
  return n;
}

// Size class of an LP of m constraints: index into kSlotClasses, or
// n_reg_classes<T>() for the large (global-memory) class.
template <typename T>
int class_of(int64_t m) {
  for (int c = 0; c < n_reg_classes<T>(); ++c)
    if (m + 4 <= 32 * kSlotClasses[c]) return c;
  return n_reg_classes<T>();
}

template <typename T, typename P>
int launch_global_kernel(KParams kp, int dev, cudaStream_t stream) {
  auto kern = k_solve_global<T, P>;
  static int blocks_per_sm[64] = {0};
  static std::mutex mu;  // concurrent first use from multi-GPU host threads
  std::lock_guard<std::mutex> lock(mu);
  if (!blocks_per_sm[dev]) {
    int b = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, kWarpsPerCta * 32, 0));
    blocks_per_sm[dev] = std::max(b, 1);
  }
  const int64_t want = (kp.n_list + kWarpsPerCta - 1) / kWarpsPerCta;
  const int64_t maxb = (int64_t)blocks_per_sm[dev] * g_dev[dev].sm_count;
  const int grid = (int)std::max<int64_t>(1, std::min(want, maxb));
  kp.total_warps = grid * kWarpsPerCta;
  kp.counter = take_counter(dev);
  kern<<<grid, kWarpsPerCta * 32, 0, stream>>>(kp);
  note_launch();
  CUDA_TRY(cudaGetLastError());
  return 0;
}

// Large class: CTA per LP with the LP resident in shared memory
// (k_solve_cta). Capacity = the class's largest LP, bounded by the opt-in
// shared memory per block; bigger LPs are solved by the CTA's warp 0 from
// global memory. 512 threads when one CTA fills the SM, else 256.
template <typename T, typename P, int THREADS, typename S = T>
int launch_cta_t(KParams kp, int64_t cap, size_t smem, int dev, cudaStream_t stream) {
  auto kern = k_solve_cta<T, P, THREADS, S>;
  CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int b = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, THREADS, smem));
  b = std::max(b, 1);
  const int64_t maxb = (int64_t)b * g_dev[dev].sm_count;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(kp.n_list, maxb));
  kp.total_warps = grid;
  kp.counter = take_counter(dev);
  kern<<<grid, THREADS, smem, stream>>>(kp, (int32_t)cap);
  note_launch();
  CUDA_TRY(cudaGetLastError());
  return 0;
}

template <typename T, typename P, typename S = T>
int launch_cta_kernel(KParams kp, int64_t max_m, int dev, cudaStream_t stream) {
  int optin = 0, per_sm = 0;
  CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  CUDA_TRY(cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
  int64_t cap = std::max<int64_t>(16, ((max_m + 15) / 16) * 16);
  while (cap > 16 && CtaBuffers<T, P, S>::bytes(cap) > (size_t)optin) cap -= 16;
  const size_t smem = CtaBuffers<T, P, S>::bytes(cap);
  // 16 warps per SM, split over as many CTAs (LPs) as shared memory allows
  const int ctas = (int)std::max<size_t>(1, (size_t)per_sm / (smem + 1024));
  if (ctas >= 3) return launch_cta_t<T, P, 128, S>(kp, cap, smem, dev, stream);
  if (ctas >= 2) return launch_cta_t<T, P, 256, S>(kp, cap, smem, dev, stream);
  return launch_cta_t<T, P, 512, S>(kp, cap, smem, dev, stream);
}

template <typename T, typename P>
int launch_class(const KParams& kp, int cls, int dev, cudaStream_t s, int64_t max_m) {
  // (experiment knob: LP2D_B200_FORCE_CTA=1 sends every class to the CTA kernel)
  static const bool force_cta = std::getenv("LP2D_B200_FORCE_CTA") &&
                                std::getenv("LP2D_B200_FORCE_CTA")[0] == '1';
  if (cls >= n_reg_classes<T>() || force_cta) return launch_cta_kernel<T, P>(kp, max_m, dev, s);
  // <NS, NT>: NS register chunks + NT shared-memory tail chunks (late TMA).
  // fp64 classes above m = 28 keep 2 register chunks and a tail (16 warps/SM at
  // 128 registers instead of 12 at 168: 10-48% faster per class); fp32 keeps
  // register-only classes up to m = 316 (measured faster there) and tails above.
  switch (kSlotClasses[cls]) {
    case 1:
      if (tiny_uses_lanes()) return launch_lane_kernel<T, P>(kp, dev, s);
      return launch_warp_kernel<T, P, 1>(kp, dev, s);
    case 2: return launch_warp_kernel<T, P, 2>(kp, dev, s);
    case 4:
      if constexpr (sizeof(T) == 8) return launch_warp_kernel<T, P, 2, 2>(kp, dev, s, max_m);
      else return launch_warp_kernel<T, P, 4>(kp, dev, s);
    case 5:
      if constexpr (sizeof(T) == 8) return launch_warp_kernel<T, P, 2, 3>(kp, dev, s, max_m);
      else return launch_warp_kernel<T, P, 5>(kp, dev, s);
    case 6:
      if constexpr (sizeof(T) == 8) return launch_warp_kernel<T, P, 2, 4>(kp, dev, s, max_m);
      else return launch_warp_kernel<T, P, 6>(kp, dev, s);
    case 9:
      if constexpr (sizeof(T) == 8) return launch_warp_kernel<T, P, 2, 7>(kp, dev, s, max_m);
      else return launch_warp_kernel<T, P, 9>(kp, dev, s);
    case 10:
      if constexpr (sizeof(T) == 8) return launch_warp_kernel<T, P, 2, 8>(kp, dev, s, max_m);
      else return launch_warp_kernel<T, P, 10>(kp, dev, s);
    case 18:
      if constexpr (sizeof(T) == 8) return launch_warp_kernel<T, P, 2, 16>(kp, dev, s, max_m);
      else return launch_warp_kernel<T, P, 10, 8>(kp, dev, s, max_m);
    case 33:  // 14 register chunks + 19 shared-memory tail chunks (fp64: 2 + 31)
      if constexpr (sizeof(T) == 8) return launch_warp_kernel<T, P, 2, 31>(kp, dev, s, max_m);
      else return launch_warp_kernel<T, P, 14, 19>(kp, dev, s, max_m);
    case 65:  // 16 register chunks + 49 tail chunks (m <= 2076, 29 KB per warp; fp64 2 + 63)
      if constexpr (sizeof(T) == 8) return launch_warp_kernel<T, P, 2, 63>(kp, dev, s, max_m);
      else return launch_warp_kernel<T, P, 16, 49>(kp, dev, s, max_m);
  }
  return fail(LP2D_ERR_UNSUPPORTED, "size class not built");
}

// may_sync: host mode (which synchronises anyway) reads the class counts back
// and launches only the non-empty classes with right-sized grids; device
// mode stays asynchronous and launches every class in [min_m, max_m].
// ---- fp32 storage: K4 (k_solve_fx, lp2d_fx.cuh) for the warp classes ------
// Same staging geometry and CTA-shape selection as the double/float warp
// kernels (WarpLayout<float, ...>): register-only classes at a compile-time
// CTA shape, late-TMA classes at the run-time shape with the most resident
// warps.
template <typename P, int NS, int NT, int CAP, bool DB = false>
int launch_fx_cap(KParams kp, int dev, cudaStream_t stream) {
  using L = WarpLayout<float, P, NS, NT, CAP>;
  auto kern = k_solve_fx<P, NS, NT, CAP, DB>;
  constexpr size_t nbuf = DB ? 2 : 1;
  struct Shape {
    int warps = 0, blocks = 0;
  };
  static Shape shape[64];
  static std::mutex mu;
  Shape sh;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (!shape[dev].warps) {
      Shape best;
      if constexpr (L::kLateTma) {
        int optin = 0;
        CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
        for (int w = 1; w <= L::kMaxWarpsRt; ++w) {
          int b = 0;
          CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, w * 32,
                                                                 (size_t)w * nbuf * (L::kBuf + 8)));
          if (b * w > best.blocks * best.warps) best = Shape{w, b};
        }
      } else {
        CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)L::kSmem));
        int b = 0;
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, L::kWarps * 32, L::kSmem));
        best = Shape{L::kWarps, b};
      }
      if (best.blocks < 1) return fail(LP2D_ERR_CUDA, "fx warp kernel does not fit on an SM");
      shape[dev] = best;
    }
    sh = shape[dev];
  }
  const size_t smem = L::kLateTma ? (size_t)sh.warps * nbuf * (L::kBuf + 8) : (size_t)L::kSmem;
  const int64_t want = (kp.n_list + sh.warps - 1) / sh.warps;
  const int64_t maxb = (int64_t)sh.blocks * g_dev[dev].sm_count;
  const int grid = (int)std::max<int64_t>(1, std::min(want, maxb));
  kp.total_warps = grid * sh.warps;
  kp.counter = take_counter(dev);
  kern<<<grid, sh.warps * 32, smem, stream>>>(kp);
  note_launch();
  CUDA_TRY(cudaGetLastError());
  return 0;
}

template <typename P, int NS, int NT, bool DB = false>
int launch_fx(KParams kp, int64_t max_m, int dev, cudaStream_t s) {
  if constexpr (NS + NT == 33) {
    if (max_m > 0 && max_m <= 1024) return launch_fx_cap<P, NS, NT, 1024, DB>(kp, dev, s);
  }
  return launch_fx_cap<P, NS, NT, 0, DB>(kp, dev, s);
}

// K4/K5 cover the warp classes (29 <= m <= 2076); the lane class and the CTA
// class read the float storage directly (their kernels' S = float).
bool fx_class(int cls) { return cls >= 1 && cls < n_reg_classes<double>(); }

// ---- fp32 storage: K5 (k_solve_fs, lp2d_fs.cuh) ---------------------------
// Run-time CTA shape: the most resident warps for the buffer size, at most
// REGW warps per CTA (the kernel's register budget).
template <typename P, int CAP, int NBUF, int REGW>
int launch_fs(KParams kp, int dev, cudaStream_t stream) {
  using L = FsLayout<P, CAP>;
  auto kern = k_solve_fs<P, CAP, NBUF, REGW>;
  constexpr size_t per_warp = (size_t)NBUF * (L::kBuf + 8);
  struct Shape {
    int warps = 0, blocks = 0;
  };
  static Shape shape[64];
  static std::mutex mu;
  Shape sh;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (!shape[dev].warps) {
      int optin = 0;
      CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
      CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
      Shape best;
      for (int w = 1; w <= std::min(REGW, 32) && (size_t)w * per_warp <= (size_t)optin; ++w) {
        int b = 0;
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, w * 32, (size_t)w * per_warp));
        if (b * w > best.blocks * best.warps) best = Shape{w, b};
      }
      if (best.blocks < 1) return fail(LP2D_ERR_CUDA, "fs kernel does not fit on an SM");
      shape[dev] = best;
    }
    sh = shape[dev];
  }
  const size_t smem = (size_t)sh.warps * per_warp;
  const int64_t want = (kp.n_list + sh.warps - 1) / sh.warps;
  const int64_t maxb = (int64_t)sh.blocks * g_dev[dev].sm_count;
  const int grid = (int)std::max<int64_t>(1, std::min(want, maxb));
  kp.total_warps = grid * sh.warps;
  kp.counter = take_counter(dev);
  kern<<<grid, sh.warps * 32, smem, stream>>>(kp);
  note_launch();
  CUDA_TRY(cudaGetLastError());
  return 0;
}

// 0 or 1: K4 (the default), 2 ("all"): K5 for every class <= 1052 (A/B).
int fs_mode() {
  static const int mode = [] {
    const char* e = std::getenv("LP2D_B200_FS");
    if (!e) return 1;
    if (e[0] == '0') return 0;
    return std::strcmp(e, "all") == 0 ? 2 : 1;
  }();
  return mode;
}

template <typename P>
int launch_fx_class(const KParams& kp, int cls, int dev, cudaStream_t s, int64_t max_m) {
  // K5 (insertion-order shared memory) for every class <= 1052 only on
  // request (LP2D_B200_FS=all; the default and =0 run K4): K4 measured
  // faster everywhere once its tail classes keep 2 register chunks (B200,
  // m = 500: 293 vs 345 us per 2^15 LPs, m = 1024: 235 vs 283 per 2^14).
  const int fs = fs_mode();
  if (fs == 2) {
    switch (kSlotClasses[cls]) {
      case 2: return launch_fs<P, 60, 2, 20>(kp, dev, s);
      case 4: return launch_fs<P, 124, 2, 20>(kp, dev, s);
      case 5: return launch_fs<P, 156, 2, 20>(kp, dev, s);
      case 6: return launch_fs<P, 188, 2, 20>(kp, dev, s);
      case 9: return launch_fs<P, 284, 2, 20>(kp, dev, s);
      case 10: return launch_fs<P, 316, 2, 20>(kp, dev, s);
      case 18: return launch_fs<P, 572, 1, 20>(kp, dev, s);
      case 33: return launch_fs<P, 1052, 1, 15>(kp, dev, s);
    }
  }
  // Every class above m = 60 keeps 2 register chunks + a shared-memory tail
  // walked through the staged permutation (more register chunks hold more
  // registers and unrolled code: m = 1100 284 vs 211 us per 2^13 LPs with 16
  // vs 2, c2 0.284 vs 0.228 ms with 8 vs 2). Up to m = 188 the tail classes
  // are double-buffered (the next LP's bulk copy overlaps this LP: m = 64 584
  // -> 515 us per 2^17, m = 100 339 -> 305 per 2^16, c3 0.705 -> 0.635 ms);
  // above, one buffer and the late copy (m = 250: 375 vs 387 us per 2^16,
  // m = 500: 264 vs 292 per 2^15: more resident warps win).
  switch (kSlotClasses[cls]) {
    case 2: return launch_fx<P, 2, 0>(kp, max_m, dev, s);
    case 4: return launch_fx<P, 2, 2, true>(kp, max_m, dev, s);
    case 5: return launch_fx<P, 2, 3, true>(kp, max_m, dev, s);
    case 6: return launch_fx<P, 2, 4, true>(kp, max_m, dev, s);
    case 9: return launch_fx<P, 2, 7>(kp, max_m, dev, s);
    case 10: return launch_fx<P, 2, 8>(kp, max_m, dev, s);
    case 18: return launch_fx<P, 2, 16>(kp, max_m, dev, s);
    case 33: return launch_fx<P, 2, 31>(kp, max_m, dev, s);
    case 65: return launch_fx<P, 2, 63>(kp, max_m, dev, s);
  }
  return fail(LP2D_ERR_UNSUPPORTED, "fx size class not built");
}

// ---- fp32 storage: K6 lane groups (k_solve_grp, lp2d_grp.cuh) -------------
template <typename P, int G, int CAP>
int launch_grp(KParams kp, int dev, cudaStream_t stream) {
  using L = GrpLayout<P, G, CAP>;
  auto kern = k_solve_grp<P, G, CAP>;
  constexpr size_t smem = kGrpWarps * L::kWarpBytes;
  static int blocks_per_sm[64] = {0};
  static std::mutex mu;  // concurrent first use from multi-GPU host threads
  int b = 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (!blocks_per_sm[dev]) {
      CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      int q = 0;
      CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&q, kern, kGrpWarps * 32, smem));
      if (q < 1) return fail(LP2D_ERR_CUDA, "group kernel does not fit on an SM");
      blocks_per_sm[dev] = q;
    }
    b = blocks_per_sm[dev];
  }
  const int64_t per_warp = L::kGroups;
  const int64_t warps = (kp.n_list + per_warp - 1) / per_warp;
  const int64_t want = (warps + kGrpWarps - 1) / kGrpWarps;
  const int64_t maxb = (int64_t)b * g_dev[dev].sm_count;
  const int grid = (int)std::max<int64_t>(1, std::min(want, maxb));
  kp.total_warps = grid * kGrpWarps;
  kp.counter = take_counter(dev);
  kern<<<grid, kGrpWarps * 32, smem, stream>>>(kp);
  note_launch();
  CUDA_TRY(cudaGetLastError());
  return 0;
}

// Largest register-slot count whose class runs K6 (0: none, the default).
// K6 is an opt-in variant: it beats K4 only on large batches of m <= ~45
// (m = 40: 3.01 vs 3.26 ns/LP over 2^17 LPs) and loses on config 4's own
// m <= 60 LPs solved alone (38,863 LPs: 191 vs 143 us: ~2 LPs per group, and
// its per-LP latency is 4-8 lanes' worth), at m = 60 (4.15 vs 3.51 ns/LP) and
// above (the double fold: m = 128 7.56 vs 4.64 ns/LP); inside the
// whole config-4 solve it is a wash under the final launch order (0.672/0.700
// vs 0.682/0.680 ms). LP2D_B200_GRP=2 runs it on the m <= 60 class, =6 on
// every class up to m = 188 (A/B, parity tests); LP2D_B200_FS=all keeps K5.
int grp_max_slots() {
  static const int v = [] {
    const char* e = std::getenv("LP2D_B200_GRP");
    if (!e) return 0;
    return std::atoi(e);
  }();
  return v;
}

bool grp_class(int cls) {
  return cls >= 1 && cls < n_reg_classes<double>() && kSlotClasses[cls] <= grp_max_slots() &&
         kSlotClasses[cls] <= 6 && fs_mode() != 2;
}

template <typename P>
int launch_grp_class(const KParams& kp, int cls, int dev, cudaStream_t s) {
  switch (kSlotClasses[cls]) {
    case 2: return launch_grp<P, 4, 60>(kp, dev, s);
    case 4: return launch_grp<P, 8, 124>(kp, dev, s);
    case 5: return launch_grp<P, 8, 156>(kp, dev, s);
    case 6: return launch_grp<P, 8, 188>(kp, dev, s);
  }
  return fail(LP2D_ERR_UNSUPPORTED, "group size class not built");
}

template <typename T, typename F>
int launch_binned(KParams kp, int64_t min_m, int64_t max_m, int dev, cudaStream_t s,
                  bool may_sync, F&& launch_cls);

template <typename T, typename P>
int launch_balanced(KParams kp, int64_t min_m, int64_t max_m, int dev, cudaStream_t s,
                    bool may_sync) {
  return launch_binned<T>(kp, min_m, max_m, dev, s, may_sync,
                          [](const KParams& kc, int c, int d, cudaStream_t cs, int64_t cap_m) {
                            return launch_class<T, P>(kc, c, d, cs, cap_m);
                          });
}

// Size-class dispatch: a uniform batch is one launch; a mixed batch is binned
// on the device and launched one class per stream. launch_cls(kp, class, dev,
// stream, max_m) launches one class.
template <typename T, typename F>
int launch_binned(KParams kp, int64_t min_m, int64_t max_m, int dev, cudaStream_t s,
                  bool may_sync, F&& launch_cls) {
  const int cmin = class_of<T>(std::max<int64_t>(min_m, 0));
  const int cmax = class_of<T>(max_m);
  DeviceState& dv = g_dev[dev];
  const bool perm_wait = t_perm_wait.dev == dev && t_perm_wait.wait_m != INT64_MAX;
  const int64_t perm_wait_m = t_perm_wait.wait_m;
  t_perm_wait = PermWait{};
  if (cmin == cmax) {
    if (perm_wait) CUDA_TRY(cudaStreamWaitEvent(s, dv.perm_ev, 0));
    return launch_cls(kp, cmax, dev, s, max_m);
  }
  // Mixed sizes: bin LP ids by class on the device, one launch per class.
  BinSpec spec{};
  spec.nreg = n_reg_classes<T>();
  for (int c = 0; c < spec.nreg; ++c) spec.slots[c] = kSlotClasses[c];
  // The lane kernel's class is split by m, so its LP list comes out sorted
  // by m and a warp's 32 LPs have similar sizes (its sweep runs to the
  // largest of them).
  static const bool sort_tiny = !(std::getenv("LP2D_B200_SORT") && std::getenv("LP2D_B200_SORT")[0] == '0');
  spec.lane_bins = tiny_uses_lanes() && sort_tiny ? kLaneMaxM + 1 : 0;
  // The large class is split by m (256 per bin, largest first): LPT order.
  spec.cta_bins = 64;
  spec.cta_lo = 32 * kSlotClasses[spec.nreg - 1] - 3;
  spec.cta_width = 256;
  auto bin_range = [&](int c, int& lo, int& hi) {
    const int b0 = spec.lane_bins ? spec.lane_bins : 1;
    if (c == 0) {
      lo = 0;
      hi = b0;
    } else if (c < spec.nreg) {
      lo = b0 + c - 1;
      hi = lo + 1;
    } else {
      lo = b0 + spec.nreg - 1;
      hi = lo + spec.cta_bins;
    }
  };
  const size_t ws_bytes = 2 * kMaxBins * sizeof(int32_t) + sizeof(int32_t) * (size_t)kp.n_list;
  void* ws = nullptr;
  CUDA_TRY(cudaMallocFromPoolAsync(&ws, ws_bytes, g_dev[dev].pool, s));
  int32_t* counts = static_cast<int32_t*>(ws);
  int32_t* cursors = counts + kMaxBins;
  int32_t* list = counts + 2 * kMaxBins;
  CUDA_TRY(cudaMemsetAsync(counts, 0, 2 * kMaxBins * sizeof(int32_t), s));
  const int threads = 512;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((kp.n_list + threads - 1) / threads,
                                                               (int64_t)g_dev[dev].sm_count * 2));
  k_bin_count<<<grid, threads, 0, s>>>(kp.n_list, kp.m, spec, counts);
  note_launch();
  k_bin_scatter<<<grid, threads, 0, s>>>(kp.n_list, kp.m, spec, counts, cursors, list);
  note_launch();
  CUDA_TRY(cudaGetLastError());
  kp.list = list;
  kp.bin_counts = counts;
  int32_t host_bins[kMaxBins] = {0};
  if (may_sync) {
    CUDA_TRY(cudaMemcpyAsync(host_bins, counts, sizeof(host_bins), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
  }
  int64_t host_counts[16] = {0};
  for (int c = 0; c <= spec.nreg; ++c) {
    int lo, hi;
    bin_range(c, lo, hi);
    for (int q = lo; q < hi; ++q) host_counts[c] += host_bins[q];
  }
  int rc = 0;
  // One stream per class, forked from and joined back into s: a class's
  // tail (few long LPs) overlaps the next classes instead of idling the GPU.
  {
    DeviceState& d = g_dev[dev];
    std::lock_guard<std::mutex> lock(d.fork_mu);
    CUDA_TRY(cudaEventRecord(d.cls_event[16], s));
    // The large (CTA) class is launched in two capacity tiers: LPs up to
    // kCtaTierM share an SM three at a time (57 KB each), only the larger
    // ones get the whole-batch capacity (up to one LP per SM).
    constexpr int kTierBins = 8;  // bins holding m < cta_lo + 8 * cta_width
    const int64_t tier_m = (int64_t)spec.cta_lo + kTierBins * spec.cta_width - 1;
    auto launch_one = [&](int c, int lo, int hi, int64_t n_host, int64_t cap_m, int sidx) {
      KParams kc = kp;
      kc.bin_lo = lo;
      kc.bin_hi = hi;
      if (may_sync) kc.n_list = n_host;
      cudaStream_t cs = d.cls_stream[sidx];
      CUDA_TRY(cudaStreamWaitEvent(cs, d.cls_event[16], 0));
      // (LPs above perm_wait_m get their permutations from the aux stream)
      if (perm_wait && (c >= spec.nreg || 32 * kSlotClasses[c] - 4 > perm_wait_m))
        CUDA_TRY(cudaStreamWaitEvent(cs, d.perm_ev, 0));
      int r = launch_cls(kc, c, dev, cs, cap_m);
      CUDA_TRY(cudaEventRecord(d.cls_event[sidx], cs));
      CUDA_TRY(cudaStreamWaitEvent(s, d.cls_event[sidx], 0));
      return r;
    };
    // Launch order: the large (CTA) class first (its LPs are the longest and
    // latency-bound, so they start earliest), then the register classes from
    // the smallest up (B200, config 4 isolated solve: 0.708/0.712 ms largest
    // first, 0.674/0.696 this order; 0.682/0.685 with the tiny classes next and
    // the warp classes largest first; 0.697/0.698 smallest first throughout).
    // LP2D_B200_ORDER = 0 / 2 / 3 selects those alternatives (A/B).
    static const int order = std::getenv("LP2D_B200_ORDER") ? std::atoi(std::getenv("LP2D_B200_ORDER")) : 1;
    std::vector<int> seq;
    if (order == 1 && cmax == spec.nreg) {
      seq.push_back(cmax);
      for (int c = cmin; c < cmax; ++c) seq.push_back(c);
    } else if (order == 2 && cmax == spec.nreg) {
      seq.push_back(cmax);
      for (int c = cmin; c < std::min(cmax, 2); ++c) seq.push_back(c);
      for (int c = cmax - 1; c >= std::max(cmin, 2); --c) seq.push_back(c);
    } else if (order == 3) {
      for (int c = cmin; c <= cmax; ++c) seq.push_back(c);
    } else {
      for (int c = cmax; c >= cmin; --c) seq.push_back(c);
    }
    for (size_t si = 0; si < seq.size() && rc == 0; ++si) {
      const int c = seq[si];
      if (may_sync && host_counts[c] == 0) continue;
      int lo, hi;
      bin_range(c, lo, hi);
      if (c == spec.nreg && max_m > tier_m) {
        const int mid = hi - kTierBins;
        int64_t n_big = 0, n_small = 0;
        for (int q = lo; q < hi; ++q) (q < mid ? n_big : n_small) += host_bins[q];
        if (!may_sync || n_big) rc = launch_one(c, lo, mid, n_big, max_m, c);
        if (rc == 0 && (!may_sync || n_small))
          rc = launch_one(c, mid, hi, n_small, std::min<int64_t>(max_m, tier_m), c + 1);
        continue;
      }
      rc = launch_one(c, lo, hi, host_counts[c], max_m, c);
    }
  }
  if (perm_wait) CUDA_TRY(cudaStreamWaitEvent(s, dv.perm_ev, 0));
  CUDA_TRY(cudaFreeAsync(ws, s));
  return rc;
}

template <typename T>
int launch_solve(const KParams& kp, int64_t min_m, int64_t max_m, int perm_bits, int sched,
                 int dev, cudaStream_t s, bool may_sync = false) {
  if (kp.n_list == 0) return 0;
  if (sched == LP2D_SCHED_NAIVE) {
    const int threads = 128;
    const int64_t grid = (kp.n_list + threads - 1) / threads;
    if (perm_bits == 16)
      k_solve_naive<T, uint16_t><<<(unsigned)grid, threads, 0, s>>>(kp);
    else
      k_solve_naive<T, uint32_t><<<(unsigned)grid, threads, 0, s>>>(kp);
    note_launch();
    CUDA_TRY(cudaGetLastError());
    return 0;
  }
  if (perm_bits == 16) return launch_balanced<T, uint16_t>(kp, min_m, max_m, dev, s, may_sync);
  return launch_balanced<T, uint32_t>(kp, min_m, max_m, dev, s, may_sync);
}

int validate_common(const lp2d_batch_soa* b, const lp2d_opts* o, const lp2d_out* out) {
  if (!b || !o || !out) return fail(LP2D_ERR_ARG, "null argument");
  if (b->n <= 0) return fail(LP2D_ERR_EMPTY_BATCH, "solve_batch: empty batch");
  if (o->block_width <= 0)
    return fail(LP2D_ERR_BLOCK_WIDTH, "solve_batch: block width must be positive");
  if (b->perm_bits != 16 && b->perm_bits != 32)
    return fail(LP2D_ERR_ARG, "perm_bits must be 16 or 32");
  if (b->mem != LP2D_MEM_HOST && b->mem != LP2D_MEM_DEVICE)
    return fail(LP2D_ERR_ARG, "mem must be LP2D_MEM_HOST or LP2D_MEM_DEVICE");
  if (o->scheduler != LP2D_SCHED_NAIVE && o->scheduler != LP2D_SCHED_BALANCED)
    return fail(LP2D_ERR_ARG, "unknown scheduler");
  if (!b->m || !b->offset || !b->ax || !b->ay || !b->b || !b->c || !b->bound_m)
    return fail(LP2D_ERR_ARG, "null batch array");
  if (!b->perm && !(b->perm_from_seed && b->mem == LP2D_MEM_HOST))
    return fail(LP2D_ERR_ARG, b->perm_from_seed ? "device mode: perm_from_seed needs the perm buffer to fill"
                                                : "null batch array");
  if (!out->status || !out->x || !out->y || !out->value)
    return fail(LP2D_ERR_ARG, "null output array");
  return 0;
}

// K4 path counters (LP2D_B200_FX_STATS=1): a device buffer of kFxNStat
// counters on device 0, read back by lp2dgpu_fx_stats.
unsigned long long* g_fxstat = nullptr;
unsigned long long* fx_stats_ptr() {
  static const bool on = std::getenv("LP2D_B200_FX_STATS") && std::getenv("LP2D_B200_FX_STATS")[0] == '1';
  if (!on) return nullptr;
  if (!g_fxstat) {
    if (cudaMalloc(&g_fxstat, sizeof(unsigned long long) * kFxNStat) != cudaSuccess) return nullptr;
    cudaMemset(g_fxstat, 0, sizeof(unsigned long long) * kFxNStat);
  }
  return g_fxstat;
}

template <typename T>
KParams make_params(const lp2d_opts* o) {
  KParams kp{};
  kp.eps_par = (double)(T)o->eps_parallel;
  kp.eps_feas = (double)(T)o->eps_feas;
  kp.eps_hi = eps_hi_of<T>(o->eps_parallel);
  kp.eps_par_f = (float)kp.eps_par;
  kp.eps_feas_f = (float)kp.eps_feas;
  kp.eps_hi_f = (float)kp.eps_hi;
  kp.pk.nz = 0x8000000080000000ull;    // (-0.f, -0.f)
  kp.pk.one = 0x3f8000003f800000ull;   // (1.f, 1.f)
  kp.pk.zero = 0;                      // (+0.f, +0.f)
  kp.fxstat = fx_stats_ptr();
  {
    // K4 certificate factors (lp2d_fx.cuh / DESIGN.md §3): u = 2^-24 (fp32),
    // U = 2^-53 (fp64), rho = 2^-21 (MUFU rcp/rsqrt relative error bound),
    // ed = rho + 3u + 3U (error of the fp32 line direction); the tolerances
    // rounded up to float.
    const double u = 0x1p-24, U = 0x1p-53, rho = 0x1p-21, ed = rho + 3 * u + 3 * U;
    const double ep = (double)(float)o->eps_parallel * (1 + 0x1p-20);
    kp.fx_ka = (float)(1.25 * (2 * ed + 2 * (rho + u) + 8 * u + 5 * U) * (1 + 0x1p-20));
    kp.fx_tp = (float)((16 * (ed + 2 * u) + 3 * ep) * (1 + 0x1p-20) + 0x1p-100);
    kp.fx_ec = (float)((1.25 * (2 * ed + 2 * u) + 1.02 * ep) * (1 + 0x1p-20));
    kp.fx_eps = (float)o->eps_feas * (1.0f + 0x1p-20f);
  }
  return kp;
}

// fp32 storage: widen the batch's scalars into double copies on the device
// (k_widen), the input of the double kernels for those classes. kp's scalar
// pointers are redirected to the copies carved from ws (5 arrays). The
// element arrays cover offsets [e0, e0 + E) (a host-mode chunk addresses its
// slot through pointers biased by -e0, so its offsets stay absolute).
size_t widen_bytes(int64_t E, int64_t n) {
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  return 3 * al(sizeof(double) * E) + al(sizeof(double) * 2 * n) + al(sizeof(double) * n);
}

int widen_batch(KParams& kp, int64_t E, int64_t e0, int64_t n, char* ws, int dev, cudaStream_t s) {
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const void* src[5] = {static_cast<const float*>(kp.ax) + e0, static_cast<const float*>(kp.ay) + e0,
                        static_cast<const float*>(kp.b) + e0, kp.c, kp.bound_m};
  const int64_t cnt[5] = {E, E, E, 2 * n, n};
  void* dst[5];
  size_t o = 0;
  for (int k = 0; k < 5; ++k) {
    dst[k] = ws + o;
    o += al(sizeof(double) * cnt[k]);
    if (cnt[k] == 0) continue;
    const int threads = 256;
    const int64_t want = (cnt[k] / 4 + threads - 1) / threads;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)g_dev[dev].sm_count * 8));
    k_widen<<<grid, threads, 0, s>>>(cnt[k], static_cast<const float*>(src[k]),
                                     static_cast<double*>(dst[k]));
    note_launch();
  }
  CUDA_TRY(cudaGetLastError());
  kp.ax = static_cast<double*>(dst[0]) - e0;
  kp.ay = static_cast<double*>(dst[1]) - e0;
  kp.b = static_cast<double*>(dst[2]) - e0;
  kp.c = dst[3];
  kp.bound_m = dst[4];
  return 0;
}

// Solve of a device-resident batch with scalars stored as S (float or
// double); the arithmetic is the reference's double in both cases and the
// outputs are double. E = scalar elements (offset[n] - offset[0]), e0 = offset[0].
template <typename P>
int solve_f32_balanced(KParams kp, int64_t E, int64_t min_m, int64_t max_m, int dev,
                       cudaStream_t s, bool may_sync) {
  (void)E;
  return launch_binned<double>(
      kp, min_m, max_m, dev, s, may_sync,
      [&](const KParams& kc, int c, int d, cudaStream_t cs, int64_t cap_m) {
        // (experiment knob: LP2D_B200_FORCE_CTA=1 sends every class above the
        // lane class to the CTA kernel)
        static const bool force_cta = std::getenv("LP2D_B200_FORCE_CTA") &&
                                      std::getenv("LP2D_B200_FORCE_CTA")[0] == '1';
        if (force_cta && c >= 1) return launch_cta_kernel<double, P, float>(kc, cap_m, d, cs);
        if (grp_class(c)) return launch_grp_class<P>(kc, c, d, cs);
        if (fx_class(c)) return launch_fx_class<P>(kc, c, d, cs, cap_m);
        // the lane class (m <= 28) and the CTA class (large LPs) read the
        // float storage directly and widen on load (exact)
        if (c >= n_reg_classes<double>()) return launch_cta_kernel<double, P, float>(kc, cap_m, d, cs);
        if (tiny_uses_lanes()) return launch_lane_kernel<double, P, kLaneMaxM, float>(kc, d, cs);
        return fail(LP2D_ERR_UNSUPPORTED, "fp32 storage: the warp tiny class needs LP2D_B200_TINY unset");
      });
}

template <typename S>
int solve_device_batch(KParams kp, int64_t E, int64_t e0, int64_t min_m, int64_t max_m,
                       int perm_bits, int sched, int dev, cudaStream_t s, bool may_sync) {
  if constexpr (sizeof(S) == 4) {
    if (sched == LP2D_SCHED_BALANCED) {
      if (perm_bits == 16) return solve_f32_balanced<uint16_t>(kp, E, min_m, max_m, dev, s, may_sync);
      return solve_f32_balanced<uint32_t>(kp, E, min_m, max_m, dev, s, may_sync);
    }
    void* ws = nullptr;
    CUDA_TRY(cudaMallocFromPoolAsync(&ws, widen_bytes(E, kp.n_list), g_dev[dev].pool, s));
    int rc = widen_batch(kp, E, e0, kp.n_list, static_cast<char*>(ws), dev, s);
    if (rc == 0) rc = launch_solve<double>(kp, min_m, max_m, perm_bits, sched, dev, s, may_sync);
    CUDA_TRY(cudaFreeAsync(ws, s));
    return rc;
  } else {
    return launch_solve<double>(kp, min_m, max_m, perm_bits, sched, dev, s, may_sync);
  }
}

// Permutations of LPs [0, n) of a (sub)batch from seeds, global index
// first + j (k_shuffle_seeded), into perm (device), on stream s.
int shuffle_seeded(bool split, int64_t n, const int32_t* m, const int64_t* offset, int64_t max_m,
                   uint64_t seed, int64_t first, int32_t mul, int32_t add, void* perm,
                   int32_t perm_bits, cudaStream_t s) {
  if (n <= 0) return 0;
  const size_t es = perm_bits / 8;
  // shared-memory slices of up to 1024 entries per thread, so a few large
  // LPs do not push a mixed batch out of smem; LPs above get a CTA each
  // (k_shuffle_seeded_big, the whole permutation in smem), and LPs beyond
  // 200 KB of entries shuffle in place in global memory
  int32_t ps = (int32_t)(((std::min<int64_t>(std::max<int64_t>(max_m, 1), 1024) + 7) / 8) * 8);
  int threads = (int)std::min<int64_t>(128, (int64_t)(200 * 1024 / (ps * es)) & ~int64_t(31));
  if (threads < 32) {  // large LPs: in place in global memory
    ps = 0;
    threads = 128;
  }
  const size_t smem = (size_t)threads * ps * es;
  const unsigned grid = (unsigned)((n + threads - 1) / threads);
  // (the dynamic shared-memory opt-in, once per device and kernel: 200 KB)
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  {
    static bool done[64] = {};
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    if (dev >= 0 && dev < 64 && !done[dev]) {
      CUDA_TRY(cudaFuncSetAttribute(k_shuffle_seeded<uint16_t>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      CUDA_TRY(cudaFuncSetAttribute(k_shuffle_seeded<uint32_t>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      CUDA_TRY(cudaFuncSetAttribute(k_shuffle_seeded_big<uint16_t>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      CUDA_TRY(cudaFuncSetAttribute(k_shuffle_seeded_big<uint32_t>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      done[dev] = true;
    }
  }
  const int32_t big_lo = ps;
  const int32_t big_hi =
      (int32_t)std::min<int64_t>(max_m, (int64_t)(200 * 1024 / es) & ~int64_t(7));
  if (ps > 0 && big_hi > big_lo) {
    const size_t bsm = ((size_t)big_hi * es + 15) & ~size_t(15);
    const unsigned bgrid = (unsigned)std::min<int64_t>(n, 64 * (int64_t)std::max(1, g_dev[dev].sm_count));
    DeviceState& dv = g_dev[dev];
    cudaStream_t bs = s;
    if (split) {  // fork onto aux; launch_binned makes the large classes wait
      CUDA_TRY(cudaEventRecord(dv.perm_ev, s));
      CUDA_TRY(cudaStreamWaitEvent(dv.aux, dv.perm_ev, 0));
      bs = dv.aux;
    }
    if (perm_bits == 16)
      k_shuffle_seeded_big<uint16_t><<<bgrid, 64, bsm, bs>>>(n, m, offset, seed, first, mul, add,
                                                              static_cast<uint16_t*>(perm), big_lo, big_hi);
    else
      k_shuffle_seeded_big<uint32_t><<<bgrid, 64, bsm, bs>>>(n, m, offset, seed, first, mul, add,
                                                              static_cast<uint32_t*>(perm), big_lo, big_hi);
    note_launch();
    if (split) {
      CUDA_TRY(cudaEventRecord(dv.perm_ev, dv.aux));
      t_perm_wait = PermWait{dev, big_lo};
    }
  }
  const int32_t skip_hi = (ps > 0 && big_hi > big_lo) ? big_hi : big_lo;
  if (perm_bits == 16)
    k_shuffle_seeded<uint16_t><<<grid, threads, smem, s>>>(n, m, offset, seed, first, mul, add,
                                                           static_cast<uint16_t*>(perm), ps, big_lo, skip_hi);
  else
    k_shuffle_seeded<uint32_t><<<grid, threads, smem, s>>>(n, m, offset, seed, first, mul, add,
                                                           static_cast<uint32_t*>(perm), ps, big_lo, skip_hi);
  note_launch();
  CUDA_TRY(cudaGetLastError());
  return 0;
}

// ---- host mode: one shard [lo, hi) on one device ----------------------------
// The shard is cut into chunks of at most chunk_elems() constraint elements
// and pipelined over two device slots: H2D of chunk k+1 (copy stream) runs
// while chunk k is solved (compute stream), and chunk k's results come back
// on a third stream (the link is full duplex). Inputs in pageable memory are
// staged through two pinned buffers (filled by this shard's host thread while
// the previous chunk's DMA runs); pinned (page-locked / registered) inputs are
// DMA'd directly. Results go to pinned staging (one copy per chunk) and are
// copied out after their D2H completes, or, for large pinned result arrays,
// straight into them.

int64_t chunk_elems() {
  static const int64_t v = [] {
    const char* e = std::getenv("LP2D_B200_CHUNK_ELEMS");
    const long long x = e ? std::atoll(e) : 0;
    return x > 0 ? (int64_t)x : (int64_t)(4 << 20);
  }();
  return v;
}

// Chunk boundaries of [lo, hi): consecutive LP ranges spanning at most
// max_elems elements of the packed arrays (at least one LP each).
std::vector<int64_t> plan_chunks(const int64_t* offset, int64_t lo, int64_t hi, int64_t max_elems) {
  std::vector<int64_t> cut{lo};
  int64_t start = lo;
  while (start < hi) {
    // last j in (start, hi] with offset[j] - offset[start] <= max_elems
    const int64_t* f = std::upper_bound(offset + start + 1, offset + hi + 1, offset[start] + max_elems);
    int64_t j = (int64_t)(f - offset) - 1;
    if (j <= start) j = start + 1;
    cut.push_back(j);
    start = j;
  }
  // Taper: only the last chunk's solve is not hidden behind a transfer, so a
  // large last chunk is cut at 3/4 of its elements.
  const size_t k = cut.size();
  if (k >= 2 && max_elems >= 4) {
    const int64_t a = cut[k - 2], b = cut[k - 1];
    const int64_t target = offset[a] + (offset[b] - offset[a]) * 3 / 4;
    if (offset[b] - offset[a] > max_elems / 4) {
      int64_t j = (int64_t)(std::upper_bound(offset + a + 1, offset + b + 1, target) - offset) - 1;
      if (j > a && j < b) cut.insert(cut.end() - 1, j);
    }
  }
  return cut;
}

// Test-only mock devices (LP2D_B200_MOCK_DEVICES=N, N >= 1): host mode runs
// the threaded shard driver and the chunk planner without CUDA, and every LP
// gets status LP2D_MOCK with x = its global index, y = its shard, value = its
// chunk's first LP, work_units = its m (the gather order is checkable on a
// machine without a GPU). Never set in production: results are not solutions.
int mock_devices() {
  static const int v = [] {
    const char* e = std::getenv("LP2D_B200_MOCK_DEVICES");
    return e ? std::max(0, std::atoi(e)) : 0;
  }();
  return v;
}

bool host_pinned(const void* p) {
  if (!p) return true;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Per-device host-mode resources (grown on demand, kept across calls).
// LP2D_B200_TRACE=1: per-chunk timeline of the host pipeline on stderr
// (device events on the three streams, relative to the call's first H2D).
struct PipeTrace {
  bool on = false;
  std::vector<cudaEvent_t> ev;
  std::vector<std::string> what;
  void mark(cudaStream_t s, const std::string& w) {
    if (!on) return;
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    cudaEventRecord(e, s);
    ev.push_back(e);
    what.push_back(w);
  }
  void dump() {
    if (!on || ev.empty()) return;
    cudaEventSynchronize(ev.back());
    for (size_t i = 0; i < ev.size(); ++i) {
      float ms = 0;
      cudaEventElapsedTime(&ms, ev[0], ev[i]);
      std::fprintf(stderr, "[lp2d trace] %8.3f ms  %s\n", ms, what[i].c_str());
    }
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
    ev.clear();
  }
};
bool trace_on() {
  static const bool on = std::getenv("LP2D_B200_TRACE") && std::getenv("LP2D_B200_TRACE")[0] == '1';
  return on;
}
double host_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}
void trace_host(const char* what, double t0) {
  if (trace_on()) std::fprintf(stderr, "[lp2d trace] host %8.3f ms  %s\n", host_ms() - t0, what);
}

struct HostPipe {
  cudaStream_t copy = nullptr;  // host -> device
  cudaStream_t back = nullptr;  // device -> host (the link is full duplex)
  cudaEvent_t h2d[2] = {}, solved[2] = {}, d2h[2] = {};
  void* pin_in[2] = {};
  size_t pin_in_bytes = 0;
  void* pin_out[2] = {};
  size_t pin_out_bytes = 0;
};
HostPipe g_pipe[64];

int ensure_pinned(void** slot, size_t& have, size_t want) {
  if (have >= want) return 0;
  for (int q = 0; q < 2; ++q) {
    if (slot[q]) CUDA_TRY(cudaFreeHost(slot[q]));
    slot[q] = nullptr;
  }
  have = 0;
  for (int q = 0; q < 2; ++q) CUDA_TRY(cudaHostAlloc(&slot[q], want, cudaHostAllocDefault));
  have = want;
  return 0;
}

// The host-mode layout contract over LPs [lo, hi) (one branch-free pass; the
// slow scan only runs to name the first offending LP), with the range's
// smallest and largest m.
int scan_layout(const lp2d_batch_soa* b, int64_t lo, int64_t hi, int64_t& min_m, int64_t& max_m) {
  int32_t mx = 0, mn = INT32_MAX;
  uint64_t bad = 0;
  for (int64_t j = lo; j < hi; ++j) {
    const int32_t mj = b->m[j];
    const int64_t o0 = b->offset[j], o1 = b->offset[j + 1];
    bad |= (uint64_t)(mj < 0) | (uint64_t)(o0 & 7) | (uint64_t)(o1 - o0 < (((int64_t)mj + 7) & ~int64_t(7)));
    mx = std::max(mx, mj);
    mn = std::min(mn, mj);
  }
  if (bad) {
    for (int64_t j = lo; j < hi; ++j) {
      const int64_t mj = b->m[j];
      if (mj < 0) return fail(LP2D_ERR_PERM_LENGTH, "negative constraint count");
      const int64_t cap8 = (mj + 7) & ~int64_t(7);
      if ((b->offset[j] & 7) != 0 || b->offset[j + 1] - b->offset[j] < cap8)
        return fail(LP2D_ERR_LAYOUT, "offset[" + std::to_string(j) +
                                         "] violates the 8-element layout contract");
    }
  }
  if (b->perm_bits == 16 && mx > 65536) return fail(LP2D_ERR_ARG, "u16 permutations need m <= 65536");
  min_m = mn;
  max_m = mx;
  return 0;
}

template <typename S>
int solve_shard_mock(int dev, const lp2d_batch_soa* b, lp2d_out* out, int64_t lo, int64_t hi) {
  const std::vector<int64_t> cut = plan_chunks(b->offset, lo, hi, chunk_elems());
  for (size_t k = 0; k + 1 < cut.size(); ++k)
    for (int64_t j = cut[k]; j < cut[k + 1]; ++j) {
      out->status[j] = LP2D_MOCK;
      static_cast<double*>(out->x)[j] = (double)j;
      static_cast<double*>(out->y)[j] = (double)dev;
      static_cast<double*>(out->value)[j] = (double)cut[k];
      if (out->work_units) out->work_units[j] = (uint64_t)b->m[j];
    }
  return 0;
}

template <typename S>
int solve_shard_host(int dev, const lp2d_batch_soa* b, const lp2d_opts* o, lp2d_out* out,
                     int64_t lo, int64_t hi, int64_t min_m, int64_t max_m) {
  using T = double;  // outputs
  const double th0 = host_ms();
  // min_m < 0: the caller left the layout check to the pipeline (per chunk)
  const bool lazy = min_m < 0;
  if (mock_devices()) {
    if (lazy)
      if (int rc = scan_layout(b, lo, hi, min_m, max_m)) return rc;
    return solve_shard_mock<S>(dev, b, out, lo, hi);
  }
  if (int rc = ensure_device(dev)) return rc;
  DeviceState& d = g_dev[dev];
  std::lock_guard<std::mutex> lock(d.mu);
  CUDA_TRY(cudaSetDevice(dev));
  HostPipe& hp = g_pipe[dev];
  if (!hp.copy) {
    CUDA_TRY(cudaStreamCreateWithFlags(&hp.copy, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&hp.back, cudaStreamNonBlocking));
    for (int q = 0; q < 2; ++q) {
      CUDA_TRY(cudaEventCreateWithFlags(&hp.h2d[q], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&hp.solved[q], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&hp.d2h[q], cudaEventDisableTiming));
    }
  }
  const std::vector<int64_t> cut = plan_chunks(b->offset, lo, hi, chunk_elems());
  const int nk = (int)cut.size() - 1;
  int64_t cmax = 0, emax = 0;
  for (int k = 0; k < nk; ++k) {
    cmax = std::max(cmax, cut[k + 1] - cut[k]);
    emax = std::max(emax, b->offset[cut[k + 1]] - b->offset[cut[k]]);
  }
  const size_t ps = b->perm_bits / 8;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  // one slot: inputs (the contiguous pinned/staged part first) + outputs
  size_t o_in = 0;
  const size_t o_ax = 0, o_ay = o_ax + al(sizeof(S) * emax), o_b = o_ay + al(sizeof(S) * emax);
  const size_t o_perm = o_b + al(sizeof(S) * emax), o_c = o_perm + al(ps * emax);
  const size_t o_M = o_c + al(sizeof(S) * 2 * cmax), o_m = o_M + al(sizeof(S) * cmax);
  const size_t o_off = o_m + al(sizeof(int32_t) * cmax);
  const size_t in_bytes = o_off + al(sizeof(int64_t) * (cmax + 1));
  o_in = in_bytes;
  const size_t r_st = 0, r_x = r_st + al(cmax), r_y = r_x + al(sizeof(T) * cmax);
  const size_t r_v = r_y + al(sizeof(T) * cmax), r_pair = r_v + al(sizeof(T) * cmax);
  const size_t r_viol = r_pair + al(sizeof(int32_t) * 2 * cmax);
  const size_t r_wu = r_viol + al(sizeof(uint32_t) * cmax);
  const size_t out_bytes = r_wu + al(sizeof(uint64_t) * cmax);
  // (lane_stats histogram rows of the blocks one chunk touches)
  const int64_t W = o->block_width;
  const int64_t hstride = max_m + 1;
  const int64_t hrows = out->iter_hist ? cmax / W + 2 : 0;
  const size_t hist_bytes = al(sizeof(uint32_t) * hrows * hstride);
  const size_t slot_bytes = in_bytes + out_bytes + hist_bytes;
  if (d.arena_bytes < 2 * slot_bytes) {
    if (d.arena) CUDA_TRY(cudaFree(d.arena));
    d.arena = nullptr;
    d.arena_bytes = 0;
    CUDA_TRY(cudaMalloc(&d.arena, 2 * slot_bytes));
    d.arena_bytes = 2 * slot_bytes;
  }
  const bool in_pinned = host_pinned(b->ax) && host_pinned(b->ay) && host_pinned(b->b) &&
                         (b->perm_from_seed || host_pinned(b->perm)) && host_pinned(b->c) &&
                         host_pinned(b->bound_m);
  const bool out_pinned = host_pinned(out->status) && host_pinned(out->x) && host_pinned(out->y) &&
                          host_pinned(out->value) && host_pinned(out->pair) &&
                          host_pinned(out->violation_events) && host_pinned(out->work_units);
  trace_host("pinned checks", th0);
  // Results come back through the pinned staging slot (ONE copy of the
  // chunk's result block, then host copies) when the caller's arrays are
  // pageable or the block is small (per-copy latency beats bandwidth there);
  // otherwise straight into the caller's pinned arrays.
  const bool direct_out = out_pinned && out_bytes + hist_bytes > (size_t(1) << 20);
  // m and the offsets go to the device as they are (the chunk's element
  // arrays are addressed through pointers biased by -offset[c0]); staged only
  // when the caller's copies are pageable
  const bool mo_pinned = host_pinned(b->m) && host_pinned(b->offset);
  // Small chunks with pinned inputs: the four per-LP arrays (c, M, m, offset)
  // go up as ONE copy through the pinned staging slot (host memcpy of a few
  // KB) instead of four DMAs — at config 1 the copy engine's per-transfer
  // cost, not the bytes, sets the H2D time.
  const bool hdr_packed = in_pinned && o_in - o_c <= (size_t(256) << 10);
  const size_t stage_bytes = hdr_packed ? al(o_in - o_c)
                                        : (in_pinned ? (mo_pinned ? 0 : al(o_in - o_m)) : in_bytes);
  if (stage_bytes)
    if (int rc = ensure_pinned(hp.pin_in, hp.pin_in_bytes, stage_bytes)) return rc;
  if (!direct_out)
    if (int rc = ensure_pinned(hp.pin_out, hp.pin_out_bytes, out_bytes + hist_bytes)) return rc;
  cudaStream_t cs = d.stream, cp = hp.copy, cb = hp.back;
  char* arena = static_cast<char*>(d.arena);
  std::vector<std::vector<uint32_t>> hist_host(2);

  // stage + enqueue the H2D of chunk k into slot k % 2
  std::vector<int64_t> kmin(nk, min_m), kmax(nk, max_m);
  auto upload = [&](int k) -> int {
    const int q = k & 1;
    const int64_t c0 = cut[k], c1 = cut[k + 1], cnt = c1 - c0;
    if (lazy)
      if (int rc = scan_layout(b, c0, c1, kmin[k], kmax[k])) {
        // (earlier chunks are in flight: drain them before reporting)
        cudaStreamSynchronize(cp);
        cudaStreamSynchronize(cs);
        cudaStreamSynchronize(cb);
        return rc;
      }
    const int64_t e0 = b->offset[c0], E = b->offset[c1] - e0;
    char* D = arena + q * slot_bytes;
    char* H = static_cast<char*>(hp.pin_in[q]);
    CUDA_TRY(cudaEventSynchronize(hp.h2d[q]));  // the staging slot's previous DMA is done
    CUDA_TRY(cudaStreamWaitEvent(cp, hp.solved[q], 0));  // chunk k-2 no longer reads device slot q
    // staged area: from o_c (packed per-LP arrays), o_m (pinned inputs), else 0
    const size_t sm_base = hdr_packed ? o_c : (in_pinned ? o_m : 0);
    const void* src[8] = {static_cast<const S*>(b->ax) + e0, static_cast<const S*>(b->ay) + e0,
                          static_cast<const S*>(b->b) + e0,
                          b->perm ? static_cast<const char*>(b->perm) + ps * e0 : nullptr,
                          static_cast<const S*>(b->c) + 2 * c0,
                          static_cast<const S*>(b->bound_m) + c0, b->m + c0, b->offset + c0};
    const size_t dst[8] = {o_ax, o_ay, o_b, o_perm, o_c, o_M, o_m, o_off};
    const size_t len[8] = {sizeof(S) * E, sizeof(S) * E, sizeof(S) * E, ps * E,
                           sizeof(S) * 2 * cnt, sizeof(S) * cnt, sizeof(int32_t) * cnt,
                           sizeof(int64_t) * (cnt + 1)};
    for (int a = 0; a < 8; ++a) {
      if (!len[a] || (a == 3 && b->perm_from_seed)) continue;  // (perms generated on the device)
      if (hdr_packed && a >= 4) {
        std::memcpy(H + (dst[a] - sm_base), src[a], len[a]);
        continue;
      }
      if (a < 6 ? in_pinned : mo_pinned) {
        CUDA_TRY(cudaMemcpyAsync(D + dst[a], src[a], len[a], cudaMemcpyHostToDevice, cp));
      } else {
        char* h = H + (dst[a] - sm_base);
        std::memcpy(h, src[a], len[a]);
        CUDA_TRY(cudaMemcpyAsync(D + dst[a], h, len[a], cudaMemcpyHostToDevice, cp));
      }
    }
    if (hdr_packed)
      CUDA_TRY(cudaMemcpyAsync(D + o_c, H, o_off + len[7] - o_c, cudaMemcpyHostToDevice, cp));
    CUDA_TRY(cudaEventRecord(hp.h2d[q], cp));
    return 0;
  };
  // copy chunk k's results (slot k % 2) to the caller
  auto gather = [&](int k) -> int {
    const int q = k & 1;
    const int64_t c0 = cut[k], cnt = cut[k + 1] - c0;
    CUDA_TRY(cudaEventSynchronize(hp.d2h[q]));
    const int64_t row0 = c0 / W, rows = out->iter_hist ? (cut[k + 1] - 1) / W - row0 + 1 : 0;
    if (!direct_out) {
      const char* R = static_cast<const char*>(hp.pin_out[q]);
      std::memcpy(out->status + c0, R + r_st, cnt);
      std::memcpy(static_cast<T*>(out->x) + c0, R + r_x, sizeof(T) * cnt);
      std::memcpy(static_cast<T*>(out->y) + c0, R + r_y, sizeof(T) * cnt);
      std::memcpy(static_cast<T*>(out->value) + c0, R + r_v, sizeof(T) * cnt);
      if (out->pair) std::memcpy(out->pair + 2 * c0, R + r_pair, sizeof(int32_t) * 2 * cnt);
      if (out->violation_events)
        std::memcpy(out->violation_events + c0, R + r_viol, sizeof(uint32_t) * cnt);
      if (out->work_units) std::memcpy(out->work_units + c0, R + r_wu, sizeof(uint64_t) * cnt);
    }
    if (rows) {
      // chunks and shards may share a block row: accumulate (zeroed by the caller)
      const uint32_t* hsrc = direct_out ? hist_host[q].data()
                                        : reinterpret_cast<const uint32_t*>(
                                              static_cast<const char*>(hp.pin_out[q]) + out_bytes);
      static std::mutex hist_mu;
      std::lock_guard<std::mutex> hl(hist_mu);
      for (int64_t t = 0; t < rows * hstride; ++t) out->iter_hist[row0 * hstride + t] += hsrc[t];
    }
    return 0;
  };

  // Every wait is an event between the three streams except two host waits:
  // staging reuse (upload k+2 waits for chunk k's H2D, which is queued behind
  // nothing but other H2D) and the gather of chunk k-2 before chunk k's
  // results land in the same host slot. Inputs stream back to back on the
  // copy stream while the results go back on their own stream.
  trace_host("shard setup", th0);
  PipeTrace tr;
  tr.on = trace_on();
  tr.mark(cp, "start");
  if (nk > 0)
    if (int rc = upload(0)) return rc;
  trace_host("h2d 0 enqueued", th0);
  tr.mark(cp, "h2d 0 done");
  for (int k = 0; k < nk; ++k) {
    const int q = k & 1;
    if (k + 1 < nk) {
      if (int rc = upload(k + 1)) return rc;
      tr.mark(cp, "h2d " + std::to_string(k + 1) + " done");
    }
    if (k >= 2)
      if (int rc = gather(k - 2)) return rc;  // frees host result slot q
    const int64_t c0 = cut[k], cnt = cut[k + 1] - c0;
    const int64_t e0 = b->offset[c0], E = b->offset[cut[k + 1]] - e0;
    char* D = arena + q * slot_bytes;
    char* R = D + in_bytes;
    // element arrays addressed by the chunk's absolute offsets
    char* const dax = D + o_ax - (int64_t)sizeof(S) * e0;
    char* const day = D + o_ay - (int64_t)sizeof(S) * e0;
    char* const db = D + o_b - (int64_t)sizeof(S) * e0;
    char* const dperm = D + o_perm - (int64_t)ps * e0;
    CUDA_TRY(cudaStreamWaitEvent(cs, hp.h2d[q], 0));
    CUDA_TRY(cudaStreamWaitEvent(cs, hp.d2h[q], 0));  // chunk k-2's results are out of slot q
    tr.mark(cs, "solve " + std::to_string(k) + " start");
    if (b->perm_from_seed)
      if (int rc = shuffle_seeded(o->scheduler == LP2D_SCHED_BALANCED, cnt, reinterpret_cast<const int32_t*>(D + o_m),
                                  reinterpret_cast<const int64_t*>(D + o_off), kmax[k], b->perm_seed,
                                  b->perm_first + c0, b->perm_mul, b->perm_add, dperm,
                                  b->perm_bits, cs))
        return rc;
    KParams kp = make_params<T>(o);
    kp.n_list = cnt;
    kp.list = nullptr;
    kp.m = reinterpret_cast<const int32_t*>(D + o_m);
    kp.offset = reinterpret_cast<const int64_t*>(D + o_off);
    kp.ax = dax;
    kp.ay = day;
    kp.b = db;
    kp.perm = dperm;
    kp.c = D + o_c;
    kp.bound_m = D + o_M;
    kp.status = reinterpret_cast<uint8_t*>(R + r_st);
    kp.x = R + r_x;
    kp.y = R + r_y;
    kp.value = R + r_v;
    kp.pair = reinterpret_cast<int32_t*>(R + r_pair);
    kp.viol = reinterpret_cast<uint32_t*>(R + r_viol);
    kp.wu = reinterpret_cast<uint64_t*>(R + r_wu);
    const int64_t row0 = c0 / W, rows = out->iter_hist ? (cut[k + 1] - 1) / W - row0 + 1 : 0;
    if (rows) {
      kp.iter_hist = reinterpret_cast<uint32_t*>(R + out_bytes);
      kp.hist_lp0 = c0 - row0 * W;  // local LP 0 sits at this offset within row 0
      kp.hist_w = (int32_t)W;
      kp.hist_stride = (int32_t)hstride;
      CUDA_TRY(cudaMemsetAsync(kp.iter_hist, 0, sizeof(uint32_t) * rows * hstride, cs));
    }
    if (int rc = solve_device_batch<S>(kp, E, e0, kmin[k], kmax[k], b->perm_bits, o->scheduler, dev,
                                       cs, true))
      return rc;
    if (t_perm_wait.dev == dev) {  // (not consumed by a binned launch)
      t_perm_wait = PermWait{};
      CUDA_TRY(cudaStreamWaitEvent(cs, d.perm_ev, 0));
    }
    CUDA_TRY(cudaEventRecord(hp.solved[q], cs));
    trace_host("solve enqueued", th0);
    tr.mark(cs, "solve " + std::to_string(k) + " done");
    CUDA_TRY(cudaStreamWaitEvent(cb, hp.solved[q], 0));
    // results: D2H on the return stream
    char* dstp = static_cast<char*>(hp.pin_out[q]);
    auto d2h = [&](void* dst_user, size_t roff, size_t len) -> int {
      if (!len || !direct_out) return 0;
      CUDA_TRY(cudaMemcpyAsync(dst_user, R + roff, len, cudaMemcpyDeviceToHost, cb));
      return 0;
    };
    if (!direct_out) CUDA_TRY(cudaMemcpyAsync(dstp, R, out_bytes, cudaMemcpyDeviceToHost, cb));
    int rc = d2h(out->status + c0, r_st, cnt);
    if (!rc) rc = d2h(static_cast<T*>(out->x) + c0, r_x, sizeof(T) * cnt);
    if (!rc) rc = d2h(static_cast<T*>(out->y) + c0, r_y, sizeof(T) * cnt);
    if (!rc) rc = d2h(static_cast<T*>(out->value) + c0, r_v, sizeof(T) * cnt);
    if (!rc && out->pair) rc = d2h(out->pair + 2 * c0, r_pair, sizeof(int32_t) * 2 * cnt);
    if (!rc && out->violation_events)
      rc = d2h(out->violation_events + c0, r_viol, sizeof(uint32_t) * cnt);
    if (!rc && out->work_units) rc = d2h(out->work_units + c0, r_wu, sizeof(uint64_t) * cnt);
    if (rc) return rc;
    if (rows) {
      void* hdst;
      if (direct_out) {
        hist_host[q].assign((size_t)(rows * hstride), 0u);
        hdst = hist_host[q].data();  // (pageable: this copy completes before returning)
      } else {
        hdst = dstp + out_bytes;
      }
      CUDA_TRY(cudaMemcpyAsync(hdst, kp.iter_hist, sizeof(uint32_t) * rows * hstride,
                               cudaMemcpyDeviceToHost, cb));
    }
    CUDA_TRY(cudaEventRecord(hp.d2h[q], cb));
    tr.mark(cb, "d2h " + std::to_string(k) + " done");
  }
  trace_host("d2h enqueued", th0);
  for (int k = std::max(0, nk - 2); k < nk; ++k)
    if (int rc = gather(k)) return rc;
  trace_host("gathered", th0);
  CUDA_TRY(cudaStreamSynchronize(cb));
  CUDA_TRY(cudaStreamSynchronize(cp));
  trace_host("pipeline enqueued", th0);
  CUDA_TRY(cudaStreamSynchronize(cs));
  trace_host("pipeline done", th0);
  tr.dump();
  return 0;
}

template <typename S>
int solve_impl(const lp2d_batch_soa* b, const lp2d_opts* o, lp2d_out* out) {
  if (int rc = validate_common(b, o, out)) return rc;
  DeviceGuard guard;
  int ndev = 0;
  const int mock = b->mem == LP2D_MEM_HOST ? mock_devices() : 0;
  if (mock) {
    ndev = mock;  // test-only (see mock_devices): no CUDA, no solutions
  } else if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    return fail(LP2D_ERR_CUDA, "no CUDA device visible (the solver has no CPU fallback)");
  }
  if (b->mem == LP2D_MEM_DEVICE) {
    if (b->max_m < 0) return fail(LP2D_ERR_ARG, "device mode needs max_m");
    if (b->perm_bits == 16 && b->max_m > 65536)
      return fail(LP2D_ERR_ARG, "u16 permutations need m <= 65536");
    const int dev = o->device;
    if (dev < 0 || dev >= ndev || dev >= 64) return fail(LP2D_ERR_ARG, "bad device ordinal");
    if (int rc = ensure_device(dev)) return rc;
    CUDA_TRY(cudaSetDevice(dev));
    KParams kp = make_params<double>(o);
    kp.n_list = b->n;
    kp.m = b->m;
    kp.offset = b->offset;
    kp.ax = b->ax;
    kp.ay = b->ay;
    kp.b = b->b;
    kp.perm = b->perm;
    kp.c = b->c;
    kp.bound_m = b->bound_m;
    kp.status = out->status;
    kp.x = out->x;
    kp.y = out->y;
    kp.value = out->value;
    kp.pair = out->pair;
    kp.viol = out->violation_events;
    kp.wu = out->work_units;
    if (out->iter_hist) {
      const int64_t W = o->block_width;
      const int64_t rows = (b->n + W - 1) / W;
      CUDA_TRY(cudaMemsetAsync(out->iter_hist, 0, sizeof(uint32_t) * rows * (b->max_m + 1),
                               static_cast<cudaStream_t>(o->stream)));
      kp.iter_hist = out->iter_hist;
      kp.hist_lp0 = 0;
      kp.hist_w = (int32_t)W;
      kp.hist_stride = (int32_t)(b->max_m + 1);
    }
    if (b->perm_from_seed)
      if (int rc = shuffle_seeded(false, b->n, b->m, b->offset, b->max_m, b->perm_seed, b->perm_first,
                                  b->perm_mul, b->perm_add, const_cast<void*>(b->perm), b->perm_bits,
                                  static_cast<cudaStream_t>(o->stream)))
        return rc;
    // scalar elements (offset[n]): only the naive scheduler on fp32 storage
    // widens the batch and needs it; the balanced path stays asynchronous
    // (no host round trip per call)
    int64_t E = 0;
    if constexpr (sizeof(S) == 4) {
      if (o->scheduler != LP2D_SCHED_BALANCED) {
        const cudaStream_t st = static_cast<cudaStream_t>(o->stream);
        CUDA_TRY(cudaMemcpyAsync(&E, b->offset + b->n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
      }
    }
    return solve_device_batch<S>(kp, E, 0, b->min_m, b->max_m, b->perm_bits, o->scheduler, dev,
                                 static_cast<cudaStream_t>(o->stream), false);
  }
  const double th0 = host_ms();
  // host mode: validate the layout contract, then shard. A single-GPU solve
  // without lane histograms validates chunk by chunk inside the pipeline
  // (overlapped with the previous chunk's transfer); otherwise up front.
  int use = o->n_gpus > 0 ? std::min(o->n_gpus, ndev) : ndev;
  use = (int)std::min<int64_t>(std::min(use, 64), b->n);
  // a single-device call solves on opts.device (one process per GPU, e.g.
  // a torchrun rank's local GPU); shards of a multi-device call on 0..use-1
  const int dev1 = (use == 1 && !mock && o->device >= 0 && o->device < std::min(ndev, 64)) ? o->device : 0;
  if (use == 1 && !out->iter_hist) return solve_shard_host<S>(dev1, b, o, out, 0, b->n, -1, -1);
  int64_t min_m = 0, max_m = 0;
  if (int rc = scan_layout(b, 0, b->n, min_m, max_m)) return rc;
  trace_host("validated", th0);
  if (out->iter_hist)
    std::memset(out->iter_hist, 0,
                sizeof(uint32_t) * ((b->n + o->block_width - 1) / o->block_width) * (max_m + 1));
  if (use == 1) return solve_shard_host<S>(dev1, b, o, out, 0, b->n, min_m, max_m);
  std::vector<int64_t> cut(use + 1, 0);
  lp2dgpu_partition(b->n, b->m, use, cut.data());
  std::vector<int> rcs(use, 0);
  std::vector<std::string> errs(use);
  std::vector<std::thread> th;
  for (int g = 0; g < use; ++g) {
    th.emplace_back([&, g] {
      if (cut[g + 1] > cut[g]) rcs[g] = solve_shard_host<S>(g, b, o, out, cut[g], cut[g + 1], min_m, max_m);
      if (rcs[g]) errs[g] = g_err;
    });
  }
  for (auto& t : th) t.join();
  for (int g = 0; g < use; ++g)
    if (rcs[g]) return fail(rcs[g], "device " + std::to_string(g) + ": " + errs[g]);
  return 0;
}

}  // namespace

extern "C" {

void lp2dgpu_default_opts(lp2d_opts* o) {
  std::memset(o, 0, sizeof(*o));
  o->scheduler = LP2D_SCHED_BALANCED;
  o->block_width = 512;
  o->eps_parallel = 1e-12;
  o->eps_feas = 1e-9;
}

int lp2dgpu_solve_f32(const lp2d_batch_soa* b, const lp2d_opts* o, lp2d_out* out) {
  return solve_impl<float>(b, o, out);
}

int lp2dgpu_solve_f64(const lp2d_batch_soa* b, const lp2d_opts* o, lp2d_out* out) {
  return solve_impl<double>(b, o, out);
}

int lp2dgpu_partition(int64_t n, const int32_t* m, int32_t parts, int64_t* cut) {
  if (n < 0 || parts < 1 || !cut || (n > 0 && !m)) return fail(LP2D_ERR_ARG, "bad partition arguments");
  // cut k: the first prefix whose weight sum(m + 4) reaches total * k / parts
  // (integer sums; the thresholds are the double quotients rounded up)
  int64_t tot = 0;
  for (int64_t j = 0; j < n; ++j) tot += (int64_t)std::max(m[j], 0) + 4;
  const double total = (double)tot;
  std::vector<int64_t> thr(parts + 1);
  for (int k = 1; k < parts; ++k) thr[k] = (int64_t)std::ceil(total * k / parts);
  cut[0] = 0;
  int k = 1;
  int64_t acc = 0;
  for (int64_t j = 0; j < n && k < parts; ++j) {
    acc += (int64_t)std::max(m[j], 0) + 4;
    while (k < parts && acc >= thr[k]) cut[k++] = j + 1;
  }
  for (; k <= parts; ++k) cut[k] = n;
  return 0;
}

int64_t lp2dgpu_pack_offsets(int64_t n, const int32_t* m, int64_t* offset) {
  int64_t acc = 0;
  for (int64_t j = 0; j < n; ++j) {
    offset[j] = acc;
    acc += ((int64_t)std::max(m[j], 0) + 7) & ~int64_t(7);
  }
  offset[n] = acc;
  return acc;
}

int lp2dgpu_shuffle_device(int64_t n, const int32_t* m, const int64_t* offset,
                           const uint64_t* seeds, void* perm, int32_t perm_bits,
                           int32_t device, void* stream) {
  if (n <= 0) return 0;
  if (!m || !offset || !seeds || !perm) return fail(LP2D_ERR_ARG, "null argument");
  DeviceGuard guard;
  if (int rc = ensure_device(device)) return rc;
  CUDA_TRY(cudaSetDevice(device));
  const int threads = 128;
  const unsigned grid = (unsigned)((n + threads - 1) / threads);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (perm_bits == 16)
    k_shuffle<uint16_t><<<grid, threads, 0, s>>>(n, m, offset, seeds, static_cast<uint16_t*>(perm));
  else if (perm_bits == 32)
    k_shuffle<uint32_t><<<grid, threads, 0, s>>>(n, m, offset, seeds, static_cast<uint32_t*>(perm));
  else
    return fail(LP2D_ERR_ARG, "perm_bits must be 16 or 32");
  note_launch();
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int lp2dgpu_generate_device(int64_t n, int64_t first, uint64_t seed, const int32_t* m,
                            const int64_t* offset, const uint8_t* kind, double margin,
                            double bscale, int32_t scalar_bits, void* ax, void* ay, void* b,
                            void* perm, int32_t perm_bits, void* c, void* bound_m,
                            int32_t device, void* stream) {
  if (n < 0) return fail(LP2D_ERR_ARG, "generate: negative count");
  if (n == 0) return 0;
  if (!m || !offset || !ax || !ay || !b || !c || !bound_m)
    return fail(LP2D_ERR_ARG, "generate: null argument");
  if (scalar_bits != 32 && scalar_bits != 64)
    return fail(LP2D_ERR_ARG, "generate: scalar_bits must be 32 or 64");
  if (perm && perm_bits != 16 && perm_bits != 32)
    return fail(LP2D_ERR_ARG, "generate: perm_bits must be 16 or 32");
  DeviceGuard guard;
  if (int rc = ensure_device(device)) return rc;
  CUDA_TRY(cudaSetDevice(device));
  const int threads = 64;
  const unsigned grid = (unsigned)((n + threads - 1) / threads);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto go = [&](auto tag_t, auto tag_p) {
    using T = decltype(tag_t);
    using Pt = decltype(tag_p);
    k_generate<T, Pt><<<grid, threads, 0, s>>>(
        n, first, seed, m, offset, kind, margin, bscale, static_cast<T*>(ax), static_cast<T*>(ay),
        static_cast<T*>(b), static_cast<Pt*>(perm), static_cast<T*>(c), static_cast<T*>(bound_m));
  };
  const bool p16 = perm_bits == 16;
  if (scalar_bits == 32) {
    if (p16) go(float(), uint16_t()); else go(float(), uint32_t());
  } else {
    if (p16) go(double(), uint16_t()); else go(double(), uint32_t());
  }
  note_launch();
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int lp2dgpu_segmented_extremes(const double* in, int64_t n, int64_t contention, int32_t strategy,
                               double* out_min, double* out_max, int32_t device, void* stream) {
  // reduction.hpp:52-64 validation, as codes
  if (contention <= 0) return fail(LP2D_ERR_ARG, "segmented_extremes: contention must be >= 1");
  if (n < 0 || n % contention != 0)
    return fail(LP2D_ERR_ARG, "segmented_extremes: input size must be a multiple of contention");
  if (strategy < LP2D_REDUCE_SHARED_ATOMIC || strategy > LP2D_REDUCE_CUB)
    return fail(LP2D_ERR_ARG, "segmented_extremes: unknown strategy");
  const int64_t groups = n / contention;
  if (groups == 0) return 0;
  if (!in || !out_min || !out_max) return fail(LP2D_ERR_ARG, "null argument");
  DeviceGuard guard;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(LP2D_ERR_CUDA, "no CUDA device visible (the solver has no CPU fallback)");
  if (device < 0 || device >= ndev) return fail(LP2D_ERR_ARG, "bad device");
  CUDA_TRY(cudaSetDevice(device));
  if (int rc = ensure_device(device)) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t c = contention;
  const int64_t cap = (int64_t)g_dev[device].sm_count * 4;
  switch (strategy) {
    case LP2D_REDUCE_SHARED_ATOMIC: {
      const int64_t G = groups_per_block(c);
      const int grid = (int)std::min<int64_t>((groups + G - 1) / G, cap);
      k_ext_shared_atomic<<<grid, kReduceThreads, 0, s>>>(in, groups, c, out_min, out_max);
      note_launch();
      break;
    }
    case LP2D_REDUCE_TREE: {
      const int64_t G = groups_per_block(c);
      const int grid = (int)std::min<int64_t>((groups + G - 1) / G, cap);
      k_ext_tree<<<grid, kReduceThreads, 0, s>>>(in, groups, c, out_min, out_max);
      note_launch();
      break;
    }
    case LP2D_REDUCE_PRIVATE_MERGE: {
      const int64_t lanes = std::min<int64_t>(c, 32);
      if (32 % lanes == 0) {
        const int grid = (int)std::min<int64_t>((groups * lanes + kReduceThreads - 1) / kReduceThreads, cap);
        k_ext_private_shfl<<<grid, kReduceThreads, 0, s>>>(in, groups, c, out_min, out_max);
      } else {
        const int64_t per = kReduceThreads / lanes;
        const int grid = (int)std::min<int64_t>((groups + per - 1) / per, cap);
        k_ext_private<<<grid, kReduceThreads, 0, s>>>(in, groups, c, out_min, out_max);
      }
      note_launch();
      break;
    }
    case LP2D_REDUCE_GLOBAL_ATOMIC: {
      const int gg = (int)std::min<int64_t>((groups + 255) / 256, cap);
      const int gn = (int)std::min<int64_t>((n + 255) / 256, cap * 2);
      k_ext_global_init<<<gg, 256, 0, s>>>(groups, out_min, out_max);
      k_ext_global_atomic<<<gn, 256, 0, s>>>(in, n, c, out_min, out_max);
      k_ext_global_fini<<<gg, 256, 0, s>>>(groups, out_min, out_max);
      note_launch();
      note_launch();
      note_launch();
      break;
    }
    case LP2D_REDUCE_CUB: {
      cub::CountingInputIterator<int64_t> count(0);
      cub::TransformInputIterator<int64_t, GroupOffset, cub::CountingInputIterator<int64_t>> begin(
          count, GroupOffset{c});
      const double qnan = std::numeric_limits<double>::quiet_NaN();  // fmin/fmax identity
      size_t b1 = 0, b2 = 0;
      CUDA_TRY(cub::DeviceSegmentedReduce::Reduce(nullptr, b1, in, out_min, groups, begin, begin + 1,
                                                  NanMinOp{}, qnan, s));
      CUDA_TRY(cub::DeviceSegmentedReduce::Reduce(nullptr, b2, in, out_max, groups, begin, begin + 1,
                                                  NanMaxOp{}, qnan, s));
      void* tmp = nullptr;
      const size_t tb = std::max<size_t>(std::max(b1, b2), 16);
      CUDA_TRY(cudaMallocFromPoolAsync(&tmp, tb, g_dev[device].pool, s));
      CUDA_TRY(cub::DeviceSegmentedReduce::Reduce(tmp, b1, in, out_min, groups, begin, begin + 1,
                                                  NanMinOp{}, qnan, s));
      CUDA_TRY(cub::DeviceSegmentedReduce::Reduce(tmp, b2, in, out_max, groups, begin, begin + 1,
                                                  NanMaxOp{}, qnan, s));
      CUDA_TRY(cudaFreeAsync(tmp, s));
      break;
    }
  }
  CUDA_TRY(cudaGetLastError());
  return 0;
}

// Debug/measurement: copy (and optionally reset) the K4 path counters
// (enabled by LP2D_B200_FX_STATS=1; returns the counter count, 0 if off).
int lp2dgpu_fx_stats(uint64_t* out, int reset) {
  if (!g_fxstat) return 0;
  if (cudaMemcpy(out, g_fxstat, sizeof(unsigned long long) * kFxNStat, cudaMemcpyDeviceToHost) !=
      cudaSuccess)
    return 0;
  if (reset) cudaMemset(g_fxstat, 0, sizeof(unsigned long long) * kFxNStat);
  return kFxNStat;
}

int lp2dgpu_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

const char* lp2dgpu_last_error(void) { return g_err.c_str(); }

uint64_t lp2dgpu_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

const char* lp2dgpu_version(void) {
  return "lp2d_b200 0.1 (sm_100a; warp-register Seidel/RGB, TMA bulk prefetch)";
}

}  // extern "C"
