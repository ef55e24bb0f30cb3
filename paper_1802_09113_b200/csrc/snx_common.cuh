// Shared device helpers for libsnx (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/snx.h"

namespace snx {

constexpr int kDotBlocks = SNX_DOT_BLOCKS;
constexpr int kDotThreads = 256;

// ---------------------------------------------------------------- vector loads
template <typename T> struct Vec;
template <> struct Vec<double> { static constexpr int N = 2; };  // 16 B
template <> struct Vec<float> { static constexpr int N = 4; };   // 16 B

__device__ __forceinline__ void ldv(const double *p, double (&o)[2]) {
  const double2 v = __ldg(reinterpret_cast<const double2 *>(p));
  o[0] = v.x;
  o[1] = v.y;
}
__device__ __forceinline__ void ldv(const float *p, float (&o)[4]) {
  const float4 v = __ldg(reinterpret_cast<const float4 *>(p));
  o[0] = v.x;
  o[1] = v.y;
  o[2] = v.z;
  o[3] = v.w;
}

// numpy rounding for `x + a * y` / `x - a * y` (two roundings, never an FMA).
__device__ __forceinline__ double np_axpy(double x, double a, double y) {
  return __dadd_rn(x, __dmul_rn(a, y));
}
__device__ __forceinline__ double np_axmy(double x, double a, double y) {
  return __dsub_rn(x, __dmul_rn(a, y));
}

// ---------------------------------------------------------------- reductions
// All reductions have a fixed shape: xor-butterfly inside a warp (every lane
// ends with the same bits: fp add is commutative), then warps in index order.
__device__ __forceinline__ double warp_allsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_allsum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Sum of one double per thread over the block; result valid in thread 0.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double *sh) {
  v = warp_allsum(v);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NT / 32; ++i) t += sh[i];
  }
  __syncthreads();
  return t;
}

// Fixed-order sum of n partials by one block of NT threads; valid in thread 0.
template <int NT>
__device__ __forceinline__ double block_sum_array(const double *a, int n, double *sh) {
  double t = 0.0;
  for (int i = threadIdx.x; i < n; i += NT) t += a[i];
  return block_sum<NT>(t, sh);
}

// Every thread (of any block) reduces the kDotBlocks partials in the same
// order: lane i sums partials i, i+32, ... then the butterfly.
__device__ __forceinline__ double warp_sum_partials(const double *a) {
  const int lane = threadIdx.x & 31;
  double t = 0.0;
#pragma unroll
  for (int i = 0; i < kDotBlocks / 32; ++i) t += a[lane + 32 * i];
  return warp_allsum(t);
}

// The same, reading through L2 (partials written by other CTAs of a running
// persistent kernel).
__device__ __forceinline__ double warp_sum_partials_cg(const double *a) {
  const int lane = threadIdx.x & 31;
  double t = 0.0;
#pragma unroll
  for (int i = 0; i < kDotBlocks / 32; ++i) t += __ldcg(a + lane + 32 * i);
  return warp_allsum(t);
}

// CG state slot layout (SNX_CG_SLOT doubles per iteration)
enum { kRs = 0, kBest = 1, kDone = 2, kIters = 3, kConv = 4, kThr = 5, kErr = 6, kCurv = 7 };

__device__ __forceinline__ double *slot(double *state, int t) { return state + t * SNX_CG_SLOT; }

// scratch after the slots: [0, B) g.g / r.r partials
__device__ __forceinline__ double *scratch(double *state, int max_iters) {
  return state + (max_iters + 2) * SNX_CG_SLOT;
}

}  // namespace snx
