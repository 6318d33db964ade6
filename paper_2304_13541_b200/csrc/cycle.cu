// cycle.cu -- standalone a4 (dstack_wmaxmin) and a5 (dstack_schedule_cycle) kernels, warp per scenario.
// Device code in cycle.cuh; the fused path (a1-a5 in one kernel) is fused.cu.
#include <type_traits>

#include "cycle.cuh"
#include "kernels.cuh"
#include "prof.cuh"

namespace dstack {

constexpr int CYC_WARPS = 8;

__global__ void __launch_bounds__(256) k_wmaxmin(int32_t num_scen, const int32_t *__restrict__ off, int32_t L,
                                                 const uint16_t *__restrict__ demand, uint32_t *__restrict__ alloc) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < num_scen; s += nwarps) {
    const int32_t k0 = off[s], nd = off[s + 1] - k0;
    if (nd > DSTACK_MAX_DNN_PER_SCEN) {
      for (int j = lane; j < nd; j += 32) alloc[k0 + j] = 0;
      continue;
    }
    const uint32_t dem = lane < nd ? demand[k0 + lane] : 0u;
    const uint32_t a = wmaxmin_lane(dem, lane, nd, L);
    if (lane < nd) alloc[k0 + lane] = a;
  }
}

#ifndef DSTACK_CYC_GRID
#define DSTACK_CYC_GRID 64   // k_cycle grid: blocks per SM (4 resident; A/B ms: 4 -> 18.7, 8 -> 17.86, 16 -> 17.15, 32 -> 16.85, 64 -> 16.73, 128 -> 16.8, 256 -> 17.2)
#endif
#ifndef DSTACK_CYC_DYN
#define DSTACK_CYC_DYN 1   // 1: k_cycle takes scenarios from a work counter (A/B switch)
#endif
#ifndef DSTACK_CYC_BK_MINB
#define DSTACK_CYC_BK_MINB 3   // k_cycle<true> resident blocks per SM (A/B: 4 -> 23.98 ms F1 leg, 3 -> 23.38)
#endif
#ifndef DSTACK_CYC_BK_GRID
#define DSTACK_CYC_BK_GRID 8   // k_cycle<true> (F1) grid: blocks per SM (A/B leg: 8 -> 49.5, 64 -> 53.0 ms)
#endif
#ifndef DSTACK_CYC_MINB
#define DSTACK_CYC_MINB 4
#endif
#ifndef DSTACK_CYC_SMALL
#define DSTACK_CYC_SMALL 1   // 1: the eval / schedule path runs the small-buffer pass first (A/B switch)
#endif
#ifndef DSTACK_CYC_SMALL_WARPS
#define DSTACK_CYC_SMALL_WARPS 8   // small-buffer pass: warps per block
#endif
#ifndef DSTACK_CYC_SMALL_MINB
#define DSTACK_CYC_SMALL_MINB 5   // small-buffer pass: resident blocks per SM (40 warps, 48 registers)
#endif
// Small-buffer pass: 1.6 KB of session buffers per warp instead of 6.3 KB, so 40 warps fit an SM (A/B at config 3,
// where every session qualifies: 9.38 -> 9.23 ms); a longer session is queued for the full-buffer pass.
constexpr int CYC_SMALL_SLOTS = 1024, CYC_SMALL_JOBS = 128;
using CycSmemSmall = CycSmemT<CYC_SMALL_SLOTS, CYC_SMALL_JOBS>;

// BK: F1 below-knee fallback compiled in (DSTACK_FLAG_BELOW_KNEE); the default instantiation has no trace of it.
// SMALL: the small-buffer pass (sessions over CYC_SMALL_SLOTS slots or CYC_SMALL_JOBS static jobs go to a.big_q);
// !SMALL with a.big_q set: the full-buffer pass over the queued scenarios only.
template <bool BK, bool SMALL>
__global__ void __launch_bounds__((SMALL ? DSTACK_CYC_SMALL_WARPS : CYC_WARPS) * 32,
                                  BK ? DSTACK_CYC_BK_MINB : (SMALL ? DSTACK_CYC_SMALL_MINB : DSTACK_CYC_MINB))
k_cycle(const __grid_constant__ CycArgs a) {
  using SM = typename std::conditional<SMALL, CycSmemSmall, CycSmem>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  SM &sm = reinterpret_cast<SM *>(smem_raw)[warp];
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int32_t L = a.p.L, slot = a.p.slot_us, b_lo = a.p.b_min;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // scenario order: a work counter (one resident wave of warps, each takes the next scenario when it finishes one)
  // or a grid stride; the queued pass walks the queue instead
  const bool queued = !SMALL && a.big_q != nullptr;
  const int64_t nitems = queued ? (int64_t)__ldcg(a.big_q) : (int64_t)a.pb.num_scen;
  auto fetch = [&](int64_t prev) -> int64_t { return warp_next_item(a.work_ctr, prev, gwarp, nwarps, lane); };
  for (int64_t item = fetch(-1); item < nitems; item = fetch(item)) {
    const int64_t s = queued ? (int64_t)__ldcg(a.big_q + 2 + item) : item;
    const int32_t k0 = a.pb.scen_dnn_off[s], nd = a.pb.scen_dnn_off[s + 1] - k0;
    uint8_t sst = DSTACK_ST_OK;
    uint32_t T = 0;
    CycRes cr; cr.occ_static = cr.occ_all = cr.served_tot = cr.misses = cr.below = 0; cr.oversub = false;
    const bool mine = lane < nd && nd <= DSTACK_MAX_DNN_PER_SCEN;
    const int k = k0 + lane;
    uint32_t dem = 0, bs = 0, g = 0, sl = 1, rep = 0, slo = 0, runs = 0, served = 0;
    if (mine) {
      slo = (uint32_t)a.pb.slo_us[k];
      bs = a.batch[k];
      if (a.hook_level) {
        g = a.hook_level[k] > 0 ? (uint32_t)a.hook_level[k] : 0u;
        dem = g;
      } else {
        dem = a.demand[k];
      }
    }
    if (!a.hook_level) {
      uint32_t al = 0;
      if (a.alloc_out) {   // a4 fused (the eval path): WMAX-MIN over this scenario's demands, written out
        if (nd <= DSTACK_MAX_DNN_PER_SCEN) {
          al = wmaxmin_lane(dem, lane, nd, L);
          if (mine) a.alloc_out[k] = al;
        } else {
          for (int j = lane; j < nd; j += 32) a.alloc_out[k0 + j] = 0;
        }
      } else if (mine) {
        al = a.alloc[k];
      }
      al >>= 16;
      g = dem == 0 ? 0u : (dem > al ? dem : al);
    }
    const bool active = mine && dem > 0;
    if (nd > DSTACK_MAX_DNN_PER_SCEN) {
      sst = DSTACK_ST_INVALID;
    } else {
      T = __reduce_max_sync(FULL, active ? slo : 0u);
      if (T == 0) sst = DSTACK_ST_INFEASIBLE;
    }
    int32_t nslots = 0;
    if (sst == DSTACK_ST_OK) {
      nslots = (int32_t)(T / (uint32_t)slot);
      if (active) { sl = slo / (uint32_t)slot; rep = (uint32_t)nslots / sl; }
      const uint32_t njobs = __reduce_add_sync(FULL, rep);
      if (nslots > DSTACK_MAX_SLOTS || njobs > DSTACK_MAX_JOBS) { sst = DSTACK_ST_INVALID; T = 0; }
      else if (SMALL && (nslots > CYC_SMALL_SLOTS || njobs > CYC_SMALL_JOBS)) {   // to the full-buffer pass
        if (lane == 0) a.big_q[2 + atomicAdd(a.big_q, 1u)] = (uint32_t)s;
        __syncwarp();
        continue;
      }
    }
    if (sst == DSTACK_ST_OK) {
      // runtimes d_j(b) = ceil(X(g_j, b) / (S(g_j) M Delta)), b in [b_lo, b*_j], one u16 row per DNN.
      // On the eval path k_prof already wrote them at g = demand (exact whenever WMAX-MIN did not raise
      // the level, i.e. every oversubscribed scenario); only raised levels are recomputed from the rows.
      uint16_t *dtab = a.dtab_rows + (int64_t)k0 * DTAB_ROW;
      const bool need = active && (a.hook_level != nullptr || a.ws_RT == nullptr || g != dem);
      uint32_t redo = __ballot_sync(FULL, need);
      while (redo) {
        const int j = __ffs(redo) - 1;
        redo &= redo - 1;
        const uint32_t gj = __shfl_sync(FULL, g, j), bsj = __shfl_sync(FULL, bs, j);
        if (a.hook_level) {
          if (lane == 0) {
            const int32_t hd = a.hook_d[k0 + j];
            dtab[j * DTAB_ROW + bsj - 1] = (uint16_t)(hd > 0xFFFF ? 0xFFFF : (hd < 0 ? 0 : hd));
          }
          __syncwarp();
          continue;
        }
        uint64_t RT = 0, D = 0;
        if (a.ws_RT) {
          RT = a.ws_RT[k0 + j]; D = a.ws_D[k0 + j];
        } else {
          const int64_t r0 = a.pb.dnn_row_off[k0 + j];
          const int32_t K = (int32_t)(a.pb.dnn_row_off[k0 + j + 1] - r0);
          for (int i = lane; i < K; i += 32) { RT += a.pb.r[r0 + i]; D += (uint64_t)a.pb.r[r0 + i] * a.pb.d[r0 + i]; }
          RT = warp_sum_u64(RT); D = warp_sum_u64(D);
        }
        dtab_from_rows(a.pb, a.p, k0 + j, RT, D, (int32_t)gj, b_lo, (int32_t)bsj, dtab + j * DTAB_ROW, lane);
      }
      // d_j(b*) per lane: the dense array k_prof wrote, or the row just recomputed (then stored back for a6)
      uint32_t dst = 0;
      if (active) {
        if (need) {
          dst = dtab[lane * DTAB_ROW + bs - 1];
          if (a.dstar) a.dstar[k] = (uint16_t)dst;
        } else {
          dst = a.dstar[k];
        }
      }
      BelowKnee bk;
      const bool use_bk = BK && a.hook_level == nullptr;
      if (use_bk) {
        bk.pb = &a.pb; bk.p = &a.p; bk.k0 = k0; bk.ws_RT = a.ws_RT; bk.ws_D = a.ws_D;
        bk.c_slots = ((uint64_t)a.p.reconf_us + (uint64_t)slot - 1) / (uint64_t)slot;
      }
      cr = cycle_core(sm, dtab, lane, active, g, bs, sl, rep, nslots, L, b_lo, a.hook_level != nullptr, runs, served,
                      0, nullptr, 0, nullptr, 0, nullptr, use_bk ? &bk : nullptr, active ? dst : 0xFFFFFFFFu);
      if (cr.oversub) sst = DSTACK_ST_OVERSUBSCRIBED;
    }
    if (mine) {
      if (a.level) a.level[k] = (uint16_t)(sst == DSTACK_ST_OK || sst == DSTACK_ST_OVERSUBSCRIBED ? g : 0u);
      if (a.runs) a.runs[k] = (uint16_t)runs;
      if (a.served) a.served[k] = served;
    } else if (nd > DSTACK_MAX_DNN_PER_SCEN) {
      for (int j = lane; j < nd; j += 32) {
        if (a.level) a.level[k0 + j] = 0;
        if (a.runs) a.runs[k0 + j] = 0;
        if (a.served) a.served[k0 + j] = 0;
      }
    }
    if (lane == 0) {
      const bool sch = T > 0;
      if (a.scen_status) a.scen_status[s] = sst;
      if (a.T_us) a.T_us[s] = T;
      if (a.u_static) a.u_static[s] = sch ? (double)cr.occ_static / ((double)nslots * (double)L) : 0.0;
      if (a.u) a.u[s] = sch ? (double)cr.occ_all / ((double)nslots * (double)L) : 0.0;
      if (a.thr) a.thr[s] = sch ? (double)cr.served_tot * 1e6 / (double)T : 0.0;
      if (a.misses) a.misses[s] = cr.misses;
      if (a.below) a.below[s] = cr.below;
    }
    __syncwarp();
  }
}

int launch_wmaxmin(int32_t num_scen, const int32_t *off, int32_t L, const uint16_t *demand, uint32_t *alloc,
                   cudaStream_t s, int *launches) {
  if (num_scen <= 0) return 0;
  int64_t blocks = ((int64_t)num_scen * 32 + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  k_wmaxmin<<<(unsigned)blocks, 256, 0, s>>>(num_scen, off, L, demand, alloc);
  ++*launches;
  return cudaGetLastError() == cudaSuccess ? 0 : DSTACK_ELAUNCH;
}

int launch_cycle(const CycArgs &a, cudaStream_t s, int *launches) {
  if (a.pb.num_scen <= 0) return 0;
  const size_t smem = sizeof(CycSmem) * CYC_WARPS;
  if (DSTACK_CYC_SMALL && DSTACK_CYC_DYN && a.work_ctr && a.big_q && !(a.p.flags & DSTACK_FLAG_BELOW_KNEE)) {
    // small-buffer pass over every scenario, then the full-buffer pass over the queued long sessions (usually none:
    // its warps read an empty queue and exit)
    CycArgs b = a;
    b.big_q = a.big_q;
    if (cudaMemsetAsync(a.work_ctr, 0, sizeof(uint32_t), s) != cudaSuccess ||
        cudaMemsetAsync(a.big_q, 0, 2 * sizeof(uint32_t), s) != cudaSuccess) return DSTACK_ELAUNCH;
    const size_t smem_s = sizeof(CycSmemSmall) * DSTACK_CYC_SMALL_WARPS;
    const int64_t blocks_s = (a.pb.num_scen + DSTACK_CYC_SMALL_WARPS - 1) / DSTACK_CYC_SMALL_WARPS;
    const int64_t blocks = (a.pb.num_scen + CYC_WARPS - 1) / CYC_WARPS;
    const int64_t wave_s = (int64_t)num_sms() * DSTACK_CYC_SMALL_MINB;
    cudaFuncSetAttribute(k_cycle<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_s);
    k_cycle<false, true><<<(unsigned)(blocks_s < wave_s ? blocks_s : wave_s), DSTACK_CYC_SMALL_WARPS * 32, smem_s, s>>>(b);
    if (cudaMemsetAsync(a.work_ctr, 0, sizeof(uint32_t), s) != cudaSuccess) return DSTACK_ELAUNCH;
    const int64_t wave = (int64_t)num_sms() * DSTACK_CYC_MINB;
    cudaFuncSetAttribute(k_cycle<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_cycle<false, false><<<(unsigned)(blocks < wave ? blocks : wave), CYC_WARPS * 32, smem, s>>>(b);
    *launches += 2;
    return cudaGetLastError() == cudaSuccess ? 0 : DSTACK_ELAUNCH;
  }
  int64_t blocks = (a.pb.num_scen + CYC_WARPS - 1) / CYC_WARPS;
  const int64_t cap = (int64_t)num_sms() * DSTACK_CYC_GRID;
  if (blocks > cap) blocks = cap;
  if (a.p.flags & DSTACK_FLAG_BELOW_KNEE) {
    CycArgs b = a;
    b.big_q = nullptr;
    int64_t bk_blocks = blocks < (int64_t)num_sms() * DSTACK_CYC_BK_GRID ? blocks : (int64_t)num_sms() * DSTACK_CYC_BK_GRID;
    cudaFuncSetAttribute(k_cycle<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (DSTACK_CYC_DYN && b.work_ctr) {   // retries make F1 sessions very uneven: one resident wave pulling scenarios
      if (cudaMemsetAsync(b.work_ctr, 0, sizeof(uint32_t), s) != cudaSuccess) return DSTACK_ELAUNCH;
      bk_blocks = resident_wave(k_cycle<true, false>, CYC_WARPS * 32, smem, blocks);
    } else {
      b.work_ctr = nullptr;
    }
    k_cycle<true, false><<<(unsigned)bk_blocks, CYC_WARPS * 32, smem, s>>>(b);
  } else if (DSTACK_CYC_DYN && a.work_ctr) {
    // one resident wave (DSTACK_CYC_MINB blocks per SM) pulling scenarios from the work counter
    if (cudaMemsetAsync(a.work_ctr, 0, sizeof(uint32_t), s) != cudaSuccess) return DSTACK_ELAUNCH;
    const int64_t wave = (int64_t)num_sms() * DSTACK_CYC_MINB;
    CycArgs b = a;
    b.big_q = nullptr;
    cudaFuncSetAttribute(k_cycle<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_cycle<false, false><<<(unsigned)(blocks < wave ? blocks : wave), CYC_WARPS * 32, smem, s>>>(b);
  } else {
    CycArgs b = a;
    b.work_ctr = nullptr;
    b.big_q = nullptr;
    cudaFuncSetAttribute(k_cycle<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_cycle<false, false><<<(unsigned)blocks, CYC_WARPS * 32, smem, s>>>(b);
  }
  ++*launches;
  return cudaGetLastError() == cudaSuccess ? 0 : DSTACK_ELAUNCH;
}

}  // namespace dstack

#if DSTACK_PROF_STATS
extern "C" int dstack_debug_stats_cycle(unsigned long long *out16, int reset) {
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(out16, dstack::g_cstats, sizeof(unsigned long long) * 16) != cudaSuccess) return -1;
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(dstack::g_cstats, z, sizeof(z));
  }
  return 0;
}
#endif
