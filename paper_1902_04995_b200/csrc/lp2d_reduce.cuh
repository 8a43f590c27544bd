// lp2d_reduce.cuh — segmented min/max reductions under the contention
// disciplines of the paper's Fig. atomicComp.
//
// Reference: /root/reference/proj/include/lp2d/reduction.hpp:46-129
// (segmented_extremes: each consecutive group of `contention` values reduced
// to its minimum and maximum) and bench.hpp:244-274 (contention_bench). The
// reference models three CPU update disciplines; on the GPU they become the
// alternatives the paper measured for the 1D-LP fold's interval update:
//
//   SHARED_ATOMIC   every value is an atomic min/max on its group's slot in
//                   shared memory (the paper's choice; "serialized shared
//                   update");
//   TREE            halving-stride tree per group in shared memory, the same
//                   pairing as reduction.hpp:77-97;
//   PRIVATE_MERGE   min(contention, 32) lanes fold private partials, merged
//                   with warp REDUX (reduction.hpp:99-125);
//   GLOBAL_ATOMIC   atomic min/max on the group's slot in global memory;
//   CUB             cub::DeviceSegmentedReduce (the paper's library baseline).
//
// min/max are exact, so every strategy returns the reference's values
// bit for bit. NaN inputs are ignored as std::fmin/fmax ignore them (a group
// of NaNs gives NaN); the atomic strategies order doubles by an
// order-preserving 64-bit key.
#pragma once

#include <cub/device/device_segmented_reduce.cuh>
#include <cub/iterator/counting_input_iterator.cuh>
#include <cub/iterator/transform_input_iterator.cuh>

#include "lp2d_device.cuh"

namespace lp2d_b200 {

constexpr int kReduceThreads = 512;  // the paper's block size (max contention)
constexpr unsigned long long kKeyNoneMin = ~0ull;  // "no value" for min keys
constexpr unsigned long long kKeyNoneMax = 0ull;   // "no value" for max keys

__device__ __forceinline__ unsigned long long dkey(double v) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(v);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double dkey_inv(unsigned long long k) {
  const unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)u);
}
__device__ __forceinline__ double key_out_min(unsigned long long k) {
  return k == kKeyNoneMin ? __longlong_as_double(0x7ff8000000000000ll) : dkey_inv(k);
}
__device__ __forceinline__ double key_out_max(unsigned long long k) {
  return k == kKeyNoneMax ? __longlong_as_double(0x7ff8000000000000ll) : dkey_inv(k);
}
// std::fmin / std::fmax: a NaN operand is ignored.
__device__ __forceinline__ double nan_min(double a, double b) { return fmin(a, b); }
__device__ __forceinline__ double nan_max(double a, double b) { return fmax(a, b); }

// Groups handled by one block: whole groups, up to kReduceThreads values.
__host__ __device__ inline int64_t groups_per_block(int64_t c) {
  return c >= kReduceThreads ? 1 : kReduceThreads / c;
}

// ---- SHARED_ATOMIC ----------------------------------------------------------
__global__ void __launch_bounds__(kReduceThreads)
    k_ext_shared_atomic(const double* __restrict__ in, int64_t groups, int64_t c,
                        double* __restrict__ out_min, double* __restrict__ out_max) {
  __shared__ unsigned long long smin[kReduceThreads], smax[kReduceThreads];
  const int64_t G = groups_per_block(c);
  for (int64_t g0 = (int64_t)blockIdx.x * G; g0 < groups; g0 += (int64_t)gridDim.x * G) {
    const int64_t ng = min(G, groups - g0);
    for (int t = threadIdx.x; t < ng; t += blockDim.x) {
      smin[t] = kKeyNoneMin;
      smax[t] = kKeyNoneMax;
    }
    __syncthreads();
    const int64_t base = g0 * c, nv = ng * c;
    for (int64_t i = threadIdx.x; i < nv; i += blockDim.x) {
      const double v = in[base + i];
      if (v == v) {
        const unsigned long long k = dkey(v);
        const int slot = (int)(i / c);
        atomicMin(&smin[slot], k);
        atomicMax(&smax[slot], k);
      }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < ng; t += blockDim.x) {
      out_min[g0 + t] = key_out_min(smin[t]);
      out_max[g0 + t] = key_out_max(smax[t]);
    }
    __syncthreads();
  }
}

// ---- GLOBAL_ATOMIC ----------------------------------------------------------
// Keys live in the output arrays themselves (same width), converted in place.
__global__ void k_ext_global_init(int64_t groups, double* out_min, double* out_max) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups;
       g += (int64_t)gridDim.x * blockDim.x) {
    reinterpret_cast<unsigned long long*>(out_min)[g] = kKeyNoneMin;
    reinterpret_cast<unsigned long long*>(out_max)[g] = kKeyNoneMax;
  }
}
__global__ void k_ext_global_atomic(const double* __restrict__ in, int64_t n, int64_t c,
                                    double* out_min, double* out_max) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = in[i];
    if (v == v) {
      const unsigned long long k = dkey(v);
      atomicMin(reinterpret_cast<unsigned long long*>(out_min) + i / c, k);
      atomicMax(reinterpret_cast<unsigned long long*>(out_max) + i / c, k);
    }
  }
}
__global__ void k_ext_global_fini(int64_t groups, double* out_min, double* out_max) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups;
       g += (int64_t)gridDim.x * blockDim.x) {
    out_min[g] = key_out_min(reinterpret_cast<unsigned long long*>(out_min)[g]);
    out_max[g] = key_out_max(reinterpret_cast<unsigned long long*>(out_max)[g]);
  }
}

// ---- TREE -------------------------------------------------------------------
// Halving strides from bit_ceil(c)/2 over each group's values in shared
// memory (reduction.hpp:81-95); groups larger than the block are first folded
// to kReduceThreads partials per group by a strided pass.
__global__ void __launch_bounds__(kReduceThreads)
    k_ext_tree(const double* __restrict__ in, int64_t groups, int64_t c,
               double* __restrict__ out_min, double* __restrict__ out_max) {
  __shared__ double smn[kReduceThreads], smx[kReduceThreads];
  const int64_t G = groups_per_block(c);
  const int cw = (int)min(c, (int64_t)kReduceThreads);  // tree width per group
  int stride0 = 1;
  while (stride0 < cw) stride0 <<= 1;
  stride0 >>= 1;
  for (int64_t g0 = (int64_t)blockIdx.x * G; g0 < groups; g0 += (int64_t)gridDim.x * G) {
    const int64_t ng = min(G, groups - g0);
    const int t = threadIdx.x;
    const int gl = t / cw, li = t % cw;  // group in block, index in group
    const bool on = gl < ng;
    if (on) {
      const double* v = in + (g0 + gl) * c;
      double mn = v[li], mx = v[li];
      for (int64_t i = li + cw; i < c; i += cw) {  // only when c > block
        mn = nan_min(mn, v[i]);
        mx = nan_max(mx, v[i]);
      }
      smn[t] = mn;
      smx[t] = mx;
    }
    __syncthreads();
    for (int s = stride0; s >= 1; s >>= 1) {
      if (on && li < s && li + s < cw) {
        smn[t] = nan_min(smn[t], smn[t + s]);
        smx[t] = nan_max(smx[t], smx[t + s]);
      }
      __syncthreads();
    }
    if (on && li == 0) {
      out_min[g0 + gl] = smn[t];
      out_max[g0 + gl] = smx[t];
    }
    __syncthreads();
  }
}

// ---- PRIVATE_MERGE ----------------------------------------------------------
// min(c, 32) lanes per group fold strided private partials, then merge with
// REDUX on the keys (two 32-bit halves). Lanes of a group are consecutive
// threads; a group never straddles a warp when lanes divides 32, otherwise
// the merge goes through shared memory.
__global__ void __launch_bounds__(kReduceThreads)
    k_ext_private(const double* __restrict__ in, int64_t groups, int64_t c,
                  double* __restrict__ out_min, double* __restrict__ out_max) {
  __shared__ unsigned long long smin[kReduceThreads], smax[kReduceThreads];
  const int lanes = (int)min(c, (int64_t)32);
  const int per_block = kReduceThreads / lanes;  // groups per block
  const int t = threadIdx.x;
  const int gl = t / lanes, l = t % lanes;
  for (int64_t g0 = (int64_t)blockIdx.x * per_block; g0 < groups;
       g0 += (int64_t)gridDim.x * per_block) {
    const int64_t g = g0 + gl;
    const bool on = gl < per_block && g < groups;
    unsigned long long kmn = kKeyNoneMin, kmx = kKeyNoneMax;
    if (on) {
      const double* v = in + g * c;
      for (int64_t i = l; i < c; i += lanes) {
        const double x = v[i];
        if (x == x) {
          const unsigned long long k = dkey(x);
          kmn = min(kmn, k);
          kmx = max(kmx, k);
        }
      }
    }
    smin[t] = kmn;
    smax[t] = kmx;
    __syncthreads();
    if (on && l == 0) {
      for (int q = 1; q < lanes; ++q) {
        kmn = min(kmn, smin[t + q]);
        kmx = max(kmx, smax[t + q]);
      }
      out_min[g] = key_out_min(kmn);
      out_max[g] = key_out_max(kmx);
    }
    __syncthreads();
  }
}

// Warp-shuffle variant used when lanes divides 32 (power-of-two contention):
// each group's lanes are an aligned sub-warp, merged with xor shuffles.
__global__ void __launch_bounds__(kReduceThreads)
    k_ext_private_shfl(const double* __restrict__ in, int64_t groups, int64_t c,
                       double* __restrict__ out_min, double* __restrict__ out_max) {
  const int lanes = (int)min(c, (int64_t)32);
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // warp-uniform trip count: whole warps step together (shuffles below)
  for (int64_t wb = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31);
       wb < groups * lanes; wb += stride) {
    const int64_t t = wb + lane;
    const int64_t g = t / lanes;
    const int l = (int)(t % lanes);
    unsigned long long kmn = kKeyNoneMin, kmx = kKeyNoneMax;
    if (g < groups) {
      const double* v = in + g * c;
      for (int64_t i = l; i < c; i += lanes) {
        const double x = v[i];
        if (x == x) {
          const unsigned long long k = dkey(x);
          kmn = min(kmn, k);
          kmx = max(kmx, k);
        }
      }
    }
    for (int s = lanes >> 1; s >= 1; s >>= 1) {
      kmn = min(kmn, (unsigned long long)__shfl_xor_sync(kFull, (long long)kmn, s));
      kmx = max(kmx, (unsigned long long)__shfl_xor_sync(kFull, (long long)kmx, s));
    }
    if (g < groups && l == 0) {
      out_min[g] = key_out_min(kmn);
      out_max[g] = key_out_max(kmx);
    }
  }
}

// ---- CUB (library baseline) -------------------------------------------------
struct GroupOffset {
  int64_t c;
  __host__ __device__ int64_t operator()(int64_t g) const { return g * c; }
};
struct NanMinOp {
  __device__ double operator()(double a, double b) const { return nan_min(a, b); }
};
struct NanMaxOp {
  __device__ double operator()(double a, double b) const { return nan_max(a, b); }
};

}  // namespace lp2d_b200
