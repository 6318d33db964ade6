// common.cuh -- shared device helpers for libdstack (product path; no oracle code here).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "dstack.h"

#ifndef DSTACK_SMALL_CODE
#define DSTACK_SMALL_CODE 0
#endif
#if DSTACK_SMALL_CODE
#define DSTACK_UNROLL_SMALL _Pragma("unroll 1")
#else
#define DSTACK_UNROLL_SMALL _Pragma("unroll")
#endif

namespace dstack {

typedef unsigned __int128 u128;

constexpr unsigned FULL = 0xffffffffu;
constexpr uint64_t X_LIMIT = 1ull << 56;   // exact-arithmetic bound on X = E_t * S * M

// S(l) = ceil(l * S_tot / L)  (GPU% level -> SMs)
__device__ __forceinline__ int32_t s_of(int32_t l, int32_t S_tot, int32_t L) {
  return (l * S_tot + L - 1) / L;
}

// 64-bit warp shuffles
__device__ __forceinline__ uint64_t shfl_xor_u64(uint64_t v, int m) {
  uint32_t lo = __shfl_xor_sync(FULL, (uint32_t)v, m), hi = __shfl_xor_sync(FULL, (uint32_t)(v >> 32), m);
  return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ uint64_t shfl_u64(uint64_t v, int src) {
  uint32_t lo = __shfl_sync(FULL, (uint32_t)v, src), hi = __shfl_sync(FULL, (uint32_t)(v >> 32), src);
  return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ uint64_t shfl_up_u64(uint64_t v, int d) {
  uint32_t lo = __shfl_up_sync(FULL, (uint32_t)v, d), hi = __shfl_up_sync(FULL, (uint32_t)(v >> 32), d);
  return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
  DSTACK_UNROLL_SMALL
  for (int m = 16; m; m >>= 1) v += shfl_xor_u64(v, m);
  return v;
}
__device__ __forceinline__ uint32_t warp_or(uint32_t v) { return __reduce_or_sync(FULL, v); }

#ifndef DSTACK_DYN_SCEN
#define DSTACK_DYN_SCEN 1   // 1: k_ideal_sim, k_compare, k_cluster pull scenarios from a work counter (A/B switch)
#endif

// Work distribution of warp-per-item kernels: with a counter (a resident wave of warps, each taking the next item
// when it finishes one -- items of very different cost balance themselves) or else a grid stride.  The item index
// is delivered by a reduction, not a shuffle: it lands in a uniform register, so the compiler can prove that every
// loop and branch derived from it is warp-uniform and emits no divergence check (BRA.DIV) at the collectives of
// the item's body (items < 2^31, so the index fits the u32 reduction).
__device__ __forceinline__ int64_t warp_next_item(uint32_t *ctr, int64_t prev, int64_t gwarp, int64_t nwarps,
                                                  int lane) {
  uint32_t v = 0;
  if (ctr) {
    if (lane == 0) v = atomicAdd(ctr, 1u);
  } else {
    v = (uint32_t)(prev < 0 ? gwarp : prev + nwarps);
  }
  return (int64_t)__reduce_max_sync(FULL, v);
}

// bulk L2 prefetch of [ptr, ptr+bytes) (TMA engine, no registers / no wait): 16-byte aligned chunks
__device__ __forceinline__ void prefetch_l2(const void *ptr, int64_t bytes) {
  if (bytes <= 0) return;
  uintptr_t a0 = (uintptr_t)ptr & ~(uintptr_t)15;
  uintptr_t a1 = ((uintptr_t)ptr + (uintptr_t)bytes + 15) & ~(uintptr_t)15;
  while (a0 < a1) {
    uint32_t sz = (uint32_t)((a1 - a0) > (1u << 20) ? (1u << 20) : (a1 - a0));
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"(sz) : "memory");
    a0 += sz;
  }
}

// saturating add (sticky at >= 2^63)
__device__ __forceinline__ uint64_t sat_add(uint64_t a, uint64_t b) {
  uint64_t s = a + b;
  return (s < a || s >= (1ull << 63)) ? (1ull << 63) : s;
}
__device__ __forceinline__ uint64_t warp_sum_sat(uint64_t v) {
  DSTACK_UNROLL_SMALL
  for (int m = 16; m; m >>= 1) v = sat_add(v, shfl_xor_u64(v, m));
  return v;
}

// Exact comparison of scores  p1 / X1^2  vs  p2 / X2^2  (p = b*S <= 2^14, X < 2^56):
// returns sign(p1 * X2^2 - p2 * X1^2).  A float filter decides all but near-ties; near-ties
// (relative gap < 2^-18) fall back to exact 128-bit products (< 2^126).
__device__ __forceinline__ int cmp_score(uint32_t p1, uint64_t X1, float X1f, uint32_t p2, uint64_t X2, float X2f) {
  float l = (float)p1 * X2f * X2f;
  float r = (float)p2 * X1f * X1f;
  if (l > r * 1.0000038f) return 1;     // 1 + 2^-18
  if (r > l * 1.0000038f) return -1;
  u128 L = (u128)p1 * ((u128)X2 * X2);
  u128 R = (u128)p2 * ((u128)X1 * X1);
  return L > R ? 1 : (L < R ? -1 : 0);
}

}  // namespace dstack
