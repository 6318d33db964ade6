// agg.cu -- a8: per-call aggregate statistics, deterministic two-level reduction.
//
// Stage 1: a FIXED grid of AGG_BLOCKS blocks (independent of the device) each owns a contiguous
// scenario range; f64 sums are reduced in a fixed tree order, integer counts / histograms with
// shared-memory atomics (order-free).  Stage 2: one warp per struct word folds the partials in a fixed order.
// The multi-GPU combine is one NCCL all-reduce of this struct (python side).
#include "kernels.cuh"

namespace dstack {

#ifndef DSTACK_AGG_BLOCKS
#define DSTACK_AGG_BLOCKS 1024   // the fixed stage-1 grid (device-independent, so deterministic); A/B: 256 -> 0.44, 1024 -> 0.35, 2048 -> 0.50 ms
#endif
constexpr int AGG_BLOCKS = DSTACK_AGG_BLOCKS;
constexpr int AGG_THREADS = 256;



__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return x;
}

__device__ __forceinline__ double block_sum_f64(double v, double *red) {
#pragma unroll
  for (int m = 16; m; m >>= 1) v += __shfl_xor_sync(FULL, v, m);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
  return t;   // valid in thread 0
}

// shared-memory histogram increment (native 32-bit atomics)
__device__ __forceinline__ void hist_inc(uint32_t *h, uint32_t key, bool on) {
  if (on) atomicAdd(&h[key], 1u);   // (merging equal keys with __match_any_sync first: measured no faster)
}

// per-block u32 histograms (a block covers < 2^32 items), widened into the u64 partial at the end
struct AggHist {
  uint32_t n_st[5], n_scen_st[5], batch[DSTACK_MAX_BATCH + 1], demand[256];
};

__global__ void __launch_bounds__(AGG_THREADS) k_agg1(AggArgs a) {
  __shared__ AggHist hs;
  __shared__ double red[AGG_THREADS / 32];
  __shared__ unsigned long long cnt[7];
  uint32_t *hz = reinterpret_cast<uint32_t *>(&hs);
  for (int i = threadIdx.x; i < (int)(sizeof(AggHist) / 4); i += blockDim.x) hz[i] = 0;
  if (threadIdx.x < 7) cnt[threadIdx.x] = 0;
  __syncthreads();
  const int64_t per = ((int64_t)a.num_scen + AGG_BLOCKS - 1) / AGG_BLOCKS;
  const int64_t s0 = (int64_t)blockIdx.x * per;
  const int64_t s1 = s0 + per < a.num_scen ? s0 + per : a.num_scen;
  double f[5] = {0, 0, 0, 0, 0};
  uint64_t sched = 0, misses = 0, cks = 0, runs = 0, served = 0, ndnn = 0, nok = 0;
  // loop bounds rounded up to whole blocks so every warp reaches the warp-collective histogram updates
  for (int64_t s = s0 + threadIdx.x; s - threadIdx.x < s1; s += blockDim.x) {
    const bool in = s < s1;
    const uint8_t ss = in ? (a.scen_status ? a.scen_status[s] : 0) : 0;
    hist_inc(hs.n_scen_st, ss, in && ss < 5);
    const uint32_t T = in && a.T_us ? a.T_us[s] : 0;
    if (T > 0) {
      sched++;
      if (a.u_static) f[0] += a.u_static[s];
      if (a.u) f[1] += a.u[s];
      if (a.thr) f[2] += a.thr[s];
      if (a.u_ideal) f[3] += a.u_ideal[s];
      if (a.thr_ideal) f[4] += a.thr_ideal[s];
    }
    if (in && a.misses) misses += a.misses[s];
  }
  // DNN range of this block's scenarios
  const int64_t k0 = s0 < s1 ? a.off[s0] : 0, k1 = s0 < s1 ? a.off[s1] : 0;
  for (int64_t k = k0 + threadIdx.x; k - threadIdx.x < k1; k += blockDim.x) {
    const bool in = k < k1;
    const uint8_t st = in ? (a.status ? a.status[k] : 0) : 0xFF;
    const uint32_t dm = in && a.demand ? a.demand[k] : 0, bt = in && a.batch ? a.batch[k] : 0;
    hist_inc(hs.n_st, st, st < 5);
    const bool ok = st == DSTACK_ST_OK;
    hist_inc(hs.batch, bt <= DSTACK_MAX_BATCH ? bt : 0, ok);
    hist_inc(hs.demand, dm & 255, ok);
    if (in) {
      ndnn++;
      nok += ok;
      const uint32_t rn = a.runs ? a.runs[k] : 0, sv = a.served ? a.served[k] : 0;
      runs += rn; served += sv;
      // no DNN index in the mix: the checksum is a sum over the multiset of per-DNN outputs, so shards of the
      // problem (any GPU count, any chunking) add up to the whole problem's checksum
      const uint64_t v = ((uint64_t)dm << 24) ^ ((uint64_t)bt << 16) ^
                         ((uint64_t)(a.knee ? a.knee[k] : 0)) ^ ((uint64_t)(a.alloc ? a.alloc[k] : 0) << 8) ^
                         ((uint64_t)rn << 44) ^ ((uint64_t)sv << 20) ^ ((uint64_t)st << 60);
      cks += mix64(v);
    }
  }
  const uint64_t vals[7] = {sched, misses, cks, runs, served, ndnn, nok};
#pragma unroll
  for (int i = 0; i < 7; ++i) {
    uint64_t v = vals[i];
#pragma unroll
    for (int m = 16; m; m >>= 1) v += __shfl_xor_sync(FULL, v, m);
    if ((threadIdx.x & 31) == 0) atomicAdd(&cnt[i], (unsigned long long)v);
  }
  double tot[5];
  for (int i = 0; i < 5; ++i) tot[i] = block_sum_f64(f[i], red);
  __syncthreads();
  dstack_agg_t *dst = &a.partials[blockIdx.x];
  if (threadIdx.x == 0) {
    dst->sum_u_static = tot[0]; dst->sum_u = tot[1]; dst->sum_thr = tot[2]; dst->sum_u_ideal = tot[3];
    dst->sum_thr_ideal = tot[4];
    dst->n_scen = (uint64_t)(s1 > s0 ? s1 - s0 : 0);
    dst->n_scen_scheduled = cnt[0]; dst->misses = cnt[1]; dst->checksum = cnt[2]; dst->runs = cnt[3];
    dst->served = cnt[4]; dst->n_dnn = cnt[5]; dst->n_dnn_ok = cnt[6];
  }
  for (int i = threadIdx.x; i < 5; i += blockDim.x) { dst->n_st[i] = hs.n_st[i]; dst->n_scen_st[i] = hs.n_scen_st[i]; }
  for (int i = threadIdx.x; i <= DSTACK_MAX_BATCH; i += blockDim.x) dst->batch_hist[i] = hs.batch[i];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) dst->demand_hist[i] = hs.demand[i];
}

// Stage 2: one warp per word of the struct; lane i folds partials i, i + 32, ... in index order, then a fixed
// butterfly combines the lanes (a fixed order: deterministic)
__global__ void __launch_bounds__(AGG_THREADS) k_agg2(AggArgs a) {
  const int nwords = (int)(sizeof(dstack_agg_t) / 8);
  const int w = (int)(blockIdx.x * (AGG_THREADS / 32) + (threadIdx.x >> 5)), lane = threadIdx.x & 31;
  if (w >= nwords) return;
  if (w < 5) {   // the doubles
    double t = 0.0;
#pragma unroll 8
    for (int b = lane; b < AGG_BLOCKS; b += 32) t += reinterpret_cast<const double *>(&a.partials[b])[w];
#pragma unroll
    for (int m = 16; m; m >>= 1) t += __shfl_xor_sync(FULL, t, m);
    if (lane == 0) reinterpret_cast<double *>(a.out)[w] = t;
  } else {
    uint64_t t = 0;
#pragma unroll 8
    for (int b = lane; b < AGG_BLOCKS; b += 32) t += reinterpret_cast<const uint64_t *>(&a.partials[b])[w];
#pragma unroll
    for (int m = 16; m; m >>= 1) t += __shfl_xor_sync(FULL, t, m);
    if (lane == 0) reinterpret_cast<uint64_t *>(a.out)[w] = t;
  }
}

size_t agg_ws_bytes() { return sizeof(dstack_agg_t) * AGG_BLOCKS; }

int launch_agg(const AggArgs &a, cudaStream_t s, int *launches) {
  k_agg1<<<AGG_BLOCKS, AGG_THREADS, 0, s>>>(a);
  const int nwords = (int)(sizeof(dstack_agg_t) / 8), wpb = AGG_THREADS / 32;
  k_agg2<<<(nwords + wpb - 1) / wpb, AGG_THREADS, 0, s>>>(a);
  *launches += 2;
  return cudaGetLastError() == cudaSuccess ? 0 : DSTACK_ELAUNCH;
}

}  // namespace dstack
