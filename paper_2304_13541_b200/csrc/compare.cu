// compare.cu -- O9, the comparison schedulers of §6.3 on the same a1-a4 outputs:
// one warp per scenario evaluates, from the rows, d_j(b) at the session level g_j, the b* run time at 100% GPU
// (temporal) and at the knee level (static spatial), then
//   c = 0 D-STACK, 1 Max-Min fair fill, 2 max-throughput fill   three sessions of cycle_core (fill orders)
//   c = 3 temporal sharing (slices proportional to SLO)
//   c = 4 GSLICE-style static spatial sharing
// and writes U, throughput and Jain's fairness index of per-model GPU time, out[s * 5 + c].  Readings:
// DESIGN.md §3.2; the oracle's O9 (oracle/oracle.c) is the parity reference.
#include "cycle.cuh"
#include "kernels.cuh"
#include "prof.cuh"

namespace dstack {

constexpr int CMP_WARPS = 8;
#ifndef DSTACK_CMP_GRID
#define DSTACK_CMP_GRID 64   // grid: blocks per SM (A/B ms: 8 -> 95.3, 32 -> 94.2, 64 -> 93.1)
#endif
#ifndef DSTACK_CMP_MINB
#define DSTACK_CMP_MINB 4   // resident blocks per SM the register allocation targets (A/B: 1 -> 120, 3 -> 102, 4 -> 95 ms)
#endif

__device__ __forceinline__ double jain_idx(uint64_t x, bool act) {
  const uint64_t s1 = warp_sum_u64(act ? x : 0ull), s2 = warp_sum_u64(act ? x * x : 0ull);
  const uint64_t na = (uint64_t)__popc(__ballot_sync(FULL, act));
  const uint64_t den = na * s2;
  return den ? (double)(s1 * s1) / (double)den : 0.0;
}

__global__ void __launch_bounds__(CMP_WARPS * 32, DSTACK_CMP_MINB) k_compare(CmpArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  CycSmem &sm = reinterpret_cast<CycSmem *>(smem_raw)[warp];
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int32_t L = a.p.L, slot = a.p.slot_us, b_lo = a.p.b_min;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (int64_t s = warp_next_item(a.work_ctr, -1, gwarp, nwarps, lane); s < a.pb.num_scen;
       s = warp_next_item(a.work_ctr, s, gwarp, nwarps, lane)) {
    const int32_t k0 = a.pb.scen_dnn_off[s], nd = a.pb.scen_dnn_off[s + 1] - k0;
    double ou = 0.0, othr = 0.0, oj = 0.0;   // lane c < 5 holds scheduler c's results
    const bool mine = lane < nd && nd <= DSTACK_MAX_DNN_PER_SCEN;
    const int k = k0 + lane;
    uint32_t dem = 0, bs = 0, g = 0, slo = 0, sl = 1, rep = 0;
    if (mine) {
      dem = a.demand[k]; bs = a.batch[k]; slo = (uint32_t)a.pb.slo_us[k];
      const uint32_t al = a.alloc[k] >> 16;
      g = dem == 0 ? 0u : (dem > al ? dem : al);
    }
    const bool active = mine && dem > 0;
    uint32_t T = __reduce_max_sync(FULL, active ? slo : 0u);   // 0 when nd > DSTACK_MAX_DNN_PER_SCEN (no lane active); unconditional: see sim.cu
    int32_t nslots = 0;
    if (T > 0) {
      nslots = (int32_t)(T / (uint32_t)slot);
      if (active) { sl = slo / (uint32_t)slot; rep = (uint32_t)nslots / sl; }
      const uint32_t njobs = __reduce_add_sync(FULL, rep);
      if (nslots > DSTACK_MAX_SLOTS || njobs > DSTACK_MAX_JOBS) T = 0;
    }
    if (T > 0) {
      // ---- run times from the rows: d_j(b) at g_j (b in [b_lo, b*]), b* at 100% GPU, b* at the knee level ----
      uint16_t *dtab = a.dtab_rows + (int64_t)k0 * DTAB_ROW;
      uint32_t dL = 0, dk = 0;
      uint32_t todo = __ballot_sync(FULL, active);
      while (todo) {
        const int j = __ffs(todo) - 1;
        todo &= todo - 1;
        const int64_t kj = k0 + j;
        // broadcast by reductions (uniform registers): the conditional out-of-line call below then needs no
        // divergence checks at the collectives that follow it
        const int32_t gj = (int32_t)__reduce_max_sync(FULL, lane == j ? g : 0u);
        const int32_t bj = (int32_t)__reduce_max_sync(FULL, lane == j ? bs : 0u);
        const int32_t dj = (int32_t)__reduce_max_sync(FULL, lane == j ? dem : 0u);
        const uint64_t M = a.p.mem_mode == 0 ? 1ull : (uint64_t)a.pb.mem_bw[kj];
        const uint64_t SL = (uint64_t)a.p.S_tot, Sk = (uint64_t)s_of(dj, a.p.S_tot, L);
        const uint64_t Sg = (uint64_t)s_of(gj, a.p.S_tot, L);
        // one row pass: the sums, X(g, b*), X(L, b*), X(knee, b*); d_j(b) for b < b* (rare) one pass each
        uint64_t RT, D, Vg, VL, Vk;
        rows_pass3(a.pb, a.p, kj, bj, Sg, SL, Sk, RT, D, Vg, VL, Vk, lane);
        if (bj > b_lo) dtab_from_rows(a.pb, a.p, kj, RT, D, gj, b_lo, bj - 1, dtab + j * DTAB_ROW, lane);
        if (lane == 0)
          dtab[j * DTAB_ROW + bj - 1] = ceil_div_clamp16(x_of_v(a.pb, a.p, kj, RT, D, Sg, bj, Vg), Sg * M * (uint64_t)slot);
        const uint64_t XL = x_of_v(a.pb, a.p, kj, RT, D, SL, bj, VL);
        const uint64_t Xk = x_of_v(a.pb, a.p, kj, RT, D, Sk, bj, Vk);
        if (lane == j) {
          dL = ceil_div_clamp16(XL, SL * M * (uint64_t)slot);
          dk = ceil_div_clamp16(Xk, Sk * M * (uint64_t)slot);
        }
      }
      __syncwarp();
      const double NL = (double)nslots * (double)L;
      // ---- c = 0, 1, 2: the session with each fill order ----
      for (int c = 0; c < 3; ++c) {
        uint32_t runs = 0, served = 0, busy = 0;
        const CycRes cr = cycle_core(sm, dtab, lane, active, g, bs, sl, rep, nslots, L, b_lo, false, runs, served, 0,
                                     nullptr, 0, nullptr, c, &busy);
        const double jn = jain_idx(busy, active);
        if (lane == c) {
          ou = (double)cr.occ_all / NL;
          othr = (double)cr.served_tot * 1e6 / (double)T;
          oj = jn;
        }
        __syncwarp();
      }
      // ---- c = 3: temporal sharing ----
      {
        const uint64_t tot = warp_sum_u64(active ? (uint64_t)sl : 0ull);
        const uint64_t slice = active ? (uint64_t)nslots * sl / tot : 0ull;
        const uint64_t truns = active && dL ? slice / dL : 0ull;
        const uint64_t occn = warp_sum_u64(slice * dem), srv = warp_sum_u64(truns * bs);
        const double jn = jain_idx(slice, active);
        if (lane == 3) { ou = (double)occn / NL; othr = (double)srv * 1e6 / (double)T; oj = jn; }
      }
      // ---- c = 4: static spatial sharing (residents + first-fit decreasing time slots) ----
      {
        const uint32_t lv = active ? dem : 0u;
        const uint32_t key = (lv << 5) | (uint32_t)lane;
        uint32_t rank = 0, pre_lt = 0;
#pragma unroll 4
        for (int q = 0; q < 32; ++q) {   // ascending (level, index) rank among the active models
          const uint32_t kq = __shfl_sync(FULL, key, q);
          const bool aq = __shfl_sync(FULL, (int)active, q) != 0;
          if (aq && kq < key) { ++rank; pre_lt += kq >> 5; }
        }
        const uint32_t na = (uint32_t)__popc(__ballot_sync(FULL, active));
        const uint32_t mx = __reduce_max_sync(FULL, lv);
        const bool cond = active && pre_lt + lv + (rank + 1 < na ? mx : 0u) <= (uint32_t)L;
        const uint32_t np = (uint32_t)__popc(__ballot_sync(FULL, cond));   // residents: rank < np
        const bool res = active && rank < np;
        const uint32_t pre = __reduce_add_sync(FULL, res ? lv : 0u);
        const bool rest = active && !res;
        uint32_t rank2 = 0;   // (level desc, index asc) among the rest
#pragma unroll 4
        for (int q = 0; q < 32; ++q) {
          const uint32_t lq = __shfl_sync(FULL, lv, q);
          const bool rq = __shfl_sync(FULL, (int)rest, q) != 0;
          if (rq && (lq > lv || (lq == lv && q < lane))) ++rank2;
        }
        const uint32_t nrest = na - np;
        uint32_t resid = 0, K = 0;   // lane b holds slot b's residual capacity
        for (uint32_t q2 = 0; q2 < nrest; ++q2) {
          const int own = __ffs(__ballot_sync(FULL, rest && rank2 == q2)) - 1;
          const uint32_t lq = __shfl_sync(FULL, lv, own);
          const uint32_t fit = __ballot_sync(FULL, (uint32_t)lane < K && resid >= lq);
          uint32_t b = K;
          if (fit) b = (uint32_t)(__ffs(fit) - 1);
          else { if ((uint32_t)lane == K) resid = (uint32_t)L - pre; ++K; }
          if ((uint32_t)lane == b) resid -= lq;
        }
        if (K == 0) K = 1;
        const uint64_t w = (uint64_t)nslots / K;
        const uint64_t gr = active && dk ? (uint64_t)(res ? K : 1u) * (w / dk) : 0ull;
        const uint64_t gb = gr * dk;
        const uint64_t occn = warp_sum_u64(gb * lv), srv = warp_sum_u64(gr * bs);
        const double jn = jain_idx(gb, active);
        if (lane == 4) { ou = (double)occn / NL; othr = (double)srv * 1e6 / (double)T; oj = jn; }
      }
    }
    if (lane < DSTACK_NCMP) {
      a.u[s * DSTACK_NCMP + lane] = ou; a.thr[s * DSTACK_NCMP + lane] = othr; a.jain[s * DSTACK_NCMP + lane] = oj;
    }
    __syncwarp();
  }
}

int launch_compare(const CmpArgs &a, cudaStream_t s, int *launches) {
  if (a.pb.num_scen <= 0) return 0;
  const size_t smem = sizeof(CycSmem) * CMP_WARPS;
  int64_t blocks = (a.pb.num_scen + CMP_WARPS - 1) / CMP_WARPS;
  const int64_t cap = (int64_t)num_sms() * DSTACK_CMP_GRID;
  if (blocks > cap) blocks = cap;
  cudaFuncSetAttribute(k_compare, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  CmpArgs b = a;
  if (!DSTACK_DYN_SCEN) b.work_ctr = nullptr;
  if (b.work_ctr) {
    if (cudaMemsetAsync(b.work_ctr, 0, sizeof(uint32_t), s) != cudaSuccess) return DSTACK_ELAUNCH;
    blocks = resident_wave(k_compare, CMP_WARPS * 32, smem, blocks);
  }
  k_compare<<<(unsigned)blocks, CMP_WARPS * 32, smem, s>>>(b);
  ++*launches;
  return cudaGetLastError() == cudaSuccess ? 0 : DSTACK_ELAUNCH;
}

}  // namespace dstack
