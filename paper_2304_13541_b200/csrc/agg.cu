// agg.cu -- a8: per-call aggregate statistics, deterministic two-level reduction.
//
// Stage 1: a FIXED grid of AGG_BLOCKS blocks (independent of the device) each owns a contiguous
// scenario range; f64 sums are reduced in a fixed tree order, integer counts / histograms with
// shared-memory atomics (order-free).  Stage 2: one block folds the partials in index order.
// The multi-GPU combine is one NCCL all-reduce of this struct (python side).
#include "kernels.cuh"

namespace dstack {

constexpr int AGG_BLOCKS = 256;
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

__global__ void __launch_bounds__(AGG_THREADS) k_agg1(AggArgs a) {
  __shared__ dstack_agg_t sa;
  __shared__ double red[AGG_THREADS / 32];
  uint64_t *z = reinterpret_cast<uint64_t *>(&sa);
  for (int i = threadIdx.x; i < (int)(sizeof(dstack_agg_t) / 8); i += blockDim.x) z[i] = 0;
  __syncthreads();
  const int64_t per = ((int64_t)a.num_scen + AGG_BLOCKS - 1) / AGG_BLOCKS;
  const int64_t s0 = (int64_t)blockIdx.x * per;
  const int64_t s1 = s0 + per < a.num_scen ? s0 + per : a.num_scen;
  double f[5] = {0, 0, 0, 0, 0};
  uint64_t sched = 0, misses = 0, cks = 0, runs = 0, served = 0, ndnn = 0, nok = 0;
  for (int64_t s = s0 + threadIdx.x; s < s1; s += blockDim.x) {
    const uint8_t ss = a.scen_status ? a.scen_status[s] : 0;
    if (ss < 5) atomicAdd((unsigned long long *)&sa.n_scen_st[ss], 1ull);
    const uint32_t T = a.T_us ? a.T_us[s] : 0;
    if (T > 0) {
      sched++;
      if (a.u_static) f[0] += a.u_static[s];
      if (a.u) f[1] += a.u[s];
      if (a.thr) f[2] += a.thr[s];
      if (a.u_ideal) f[3] += a.u_ideal[s];
      if (a.thr_ideal) f[4] += a.thr_ideal[s];
    }
    if (a.misses) misses += a.misses[s];
  }
  // DNN range of this block's scenarios
  const int64_t k0 = s0 < s1 ? a.off[s0] : 0, k1 = s0 < s1 ? a.off[s1] : 0;
  for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
    ndnn++;
    const uint8_t st = a.status ? a.status[k] : 0;
    if (st < 5) atomicAdd((unsigned long long *)&sa.n_st[st], 1ull);
    const uint32_t dm = a.demand ? a.demand[k] : 0, bt = a.batch ? a.batch[k] : 0;
    if (st == DSTACK_ST_OK) {
      nok++;
      atomicAdd((unsigned long long *)&sa.batch_hist[bt <= DSTACK_MAX_BATCH ? bt : 0], 1ull);
      atomicAdd((unsigned long long *)&sa.demand_hist[dm & 255], 1ull);
    }
    const uint32_t rn = a.runs ? a.runs[k] : 0, sv = a.served ? a.served[k] : 0;
    runs += rn; served += sv;
    const uint64_t v = ((uint64_t)k << 40) ^ ((uint64_t)dm << 24) ^ ((uint64_t)bt << 16) ^
                       ((uint64_t)(a.knee ? a.knee[k] : 0)) ^ ((uint64_t)(a.alloc ? a.alloc[k] : 0) << 8) ^
                       ((uint64_t)rn << 44) ^ ((uint64_t)sv << 20) ^ ((uint64_t)st << 60);
    cks += mix64(v);
  }
  atomicAdd((unsigned long long *)&sa.n_scen_scheduled, (unsigned long long)sched);
  atomicAdd((unsigned long long *)&sa.misses, (unsigned long long)misses);
  atomicAdd((unsigned long long *)&sa.checksum, (unsigned long long)cks);
  atomicAdd((unsigned long long *)&sa.runs, (unsigned long long)runs);
  atomicAdd((unsigned long long *)&sa.served, (unsigned long long)served);
  atomicAdd((unsigned long long *)&sa.n_dnn, (unsigned long long)ndnn);
  atomicAdd((unsigned long long *)&sa.n_dnn_ok, (unsigned long long)nok);
  double tot[5];
  for (int i = 0; i < 5; ++i) tot[i] = block_sum_f64(f[i], red);
  __syncthreads();
  if (threadIdx.x == 0) {
    sa.sum_u_static = tot[0]; sa.sum_u = tot[1]; sa.sum_thr = tot[2]; sa.sum_u_ideal = tot[3];
    sa.sum_thr_ideal = tot[4];
    sa.n_scen = (uint64_t)(s1 > s0 ? s1 - s0 : 0);
  }
  __syncthreads();
  uint64_t *dst = reinterpret_cast<uint64_t *>(&a.partials[blockIdx.x]);
  for (int i = threadIdx.x; i < (int)(sizeof(dstack_agg_t) / 8); i += blockDim.x) dst[i] = z[i];
}

__global__ void __launch_bounds__(AGG_THREADS) k_agg2(AggArgs a) {
  // field-wise fold of the partials in index order: doubles first (5), then u64 words
  const int nwords = (int)(sizeof(dstack_agg_t) / 8);
  for (int w = threadIdx.x; w < nwords; w += blockDim.x) {
    if (w < 5) {
      double t = 0.0;
      for (int b = 0; b < AGG_BLOCKS; ++b) t += reinterpret_cast<const double *>(&a.partials[b])[w];
      reinterpret_cast<double *>(a.out)[w] = t;
    } else {
      uint64_t t = 0;
      for (int b = 0; b < AGG_BLOCKS; ++b) t += reinterpret_cast<const uint64_t *>(&a.partials[b])[w];
      reinterpret_cast<uint64_t *>(a.out)[w] = t;
    }
  }
}

size_t agg_ws_bytes() { return sizeof(dstack_agg_t) * AGG_BLOCKS; }

int launch_agg(const AggArgs &a, cudaStream_t s, int *launches) {
  k_agg1<<<AGG_BLOCKS, AGG_THREADS, 0, s>>>(a);
  k_agg2<<<1, AGG_THREADS, 0, s>>>(a);
  *launches += 2;
  return cudaGetLastError() == cudaSuccess ? 0 : DSTACK_ELAUNCH;
}

}  // namespace dstack
