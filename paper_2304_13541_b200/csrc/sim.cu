// sim.cu -- a7: long-horizon D-STACK simulation (config 5), one warp per scenario, persistent grid.
//
// Per scenario the warp keeps, per lane (= DNN), two cursors into the DNN's Poisson arrival stream
// (the shared counter-based sampler of synth/synth_core.h: arrival k's gap is a pure function of
// (seed, scenario, dnn, k), so no request queue is stored): `arr` = first arrival not yet counted,
// `head` = oldest queued request.  Each cycle: active DNNs = queued requests at the cycle start;
// WMAX-MIN over their demands; d_j(b) at the granted level (recomputed from the rows only when the
// level changes); one session (cycle.cuh) with the fill ordered by the 10-session scoreboard and every
// fill run logged; then each lane executes its DNN's runs in start order (static windows merged with
// its fill runs), serving FIFO min(batch, queue) requests, classifying each as in-SLO or late, and
// voiding runs that find an empty queue.  Readings: DESIGN.md §3 O7.
#include "../../synth/synth_core.h"   // shared input generator: the arrival sampler only
#include "cycle.cuh"
#include "kernels.cuh"
#include "prof.cuh"

namespace dstack {

constexpr int SIM_WARPS = 8;
#ifndef DSTACK_SIM_MINB
#define DSTACK_SIM_MINB 2   // resident blocks per SM (and the grid: one wave); A/B config 5: grid 4/SM at 2 resident 155 ms, 2 -> 95, 3 -> 96, 4 -> 133 ms
#endif

struct ArrCursor {
  uint64_t idx, time;
};

__device__ __forceinline__ void arr_next(ArrCursor &a, const SimArgs &s, int64_t gs, uint32_t j, uint64_t mq) {
  a.idx++;
  a.time += sy_arrival_gap(mq, sy_arrival_word(s.seed, s.cfg_tag, gs, j, (uint32_t)a.idx));
}

__global__ void __launch_bounds__(SIM_WARPS * 32, DSTACK_SIM_MINB) k_sim(SimArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  CycSmem &sm = reinterpret_cast<CycSmem *>(smem_raw)[warp];
  uint32_t *ring = reinterpret_cast<uint32_t *>(smem_raw + sizeof(CycSmem) * SIM_WARPS) + warp * 10 * 32;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  uint64_t *fill_log = a.fill_log + gwarp * DSTACK_MAX_FILL_RUNS;
  const int32_t L = a.p.L, slot = a.p.slot_us, b_lo = a.p.b_min;
  for (int64_t s = warp_next_item(a.work_ctr, -1, gwarp, nwarps, lane); s < a.pb.num_scen;
       s = warp_next_item(a.work_ctr, s, gwarp, nwarps, lane)) {
    const int32_t k0 = a.pb.scen_dnn_off[s], nd = a.pb.scen_dnn_off[s + 1] - k0;
    const int64_t gs = a.scen_base + s;
    uint8_t sst = DSTACK_ST_OK;
    uint32_t T = 0;
    uint64_t arrived = 0, in_slo = 0, late = 0, unserved = 0, occ_tot = 0, nruns = 0, misses = 0, realloc = 0;
    const bool mine = lane < nd && nd <= DSTACK_MAX_DNN_PER_SCEN;
    const int k = k0 + lane;
    uint32_t dem = 0, bs = 0, slo = 0, sl = 1, rep = 0;
    bool ok = false;
    if (mine) {
      ok = a.status[k] == DSTACK_ST_OK;
      dem = ok ? a.demand[k] : 0u; bs = ok ? a.batch[k] : 0u; slo = (uint32_t)a.pb.slo_us[k];
    }
    T = __reduce_max_sync(FULL, ok ? slo : 0u);   // 0 when nd <= 0 (no lane owns a DNN)
    if (nd > DSTACK_MAX_DNN_PER_SCEN) { sst = DSTACK_ST_INVALID; T = 0; }
    else if (T == 0) sst = DSTACK_ST_INFEASIBLE;
    int32_t nslots = 0;
    if (sst == DSTACK_ST_OK) {
      nslots = (int32_t)(T / (uint32_t)slot);
      if (ok) { sl = slo / (uint32_t)slot; rep = (uint32_t)nslots / sl; }
      const uint32_t njobs = __reduce_add_sync(FULL, rep);
      if (nslots > DSTACK_MAX_SLOTS || njobs > DSTACK_MAX_JOBS) { sst = DSTACK_ST_INVALID; T = 0; }
    }
    if (sst == DSTACK_ST_OK) {
      // mean gap (us, Q32) = f_L(l*, b*) * 100 / (lam_pct * b*), f_L = X / (S M); capped at 2^30 us
      uint64_t mq = 0;
      for (int j = 0; j < nd; ++j) {
        if (!__shfl_sync(FULL, (int)ok, j)) continue;
        const int64_t kj = k0 + j;
        const int32_t dj = (int32_t)__shfl_sync(FULL, dem, j), bj = (int32_t)__shfl_sync(FULL, bs, j);
        const int32_t ls = dj - a.p.margin > 0 ? dj - a.p.margin : 1;
        const uint64_t S = (uint64_t)s_of(ls, a.p.S_tot, L);
        const uint64_t M = a.p.mem_mode == 0 ? 1ull : (uint64_t)a.pb.mem_bw[kj];
        const uint64_t X = x_from_rows(a.pb, a.p, kj, a.ws_RT[kj], a.ws_D[kj], S, bj, lane);
        if (lane == j) {
          const int32_t lam = a.lam_pct[kj];                      // <= 0: no requests (R25)
          const u128 den = lam > 0 ? (u128)S * M * (u128)lam * (u128)bj : (u128)0;
          u128 q = den ? ((((u128)X * 100u) << 32) / den) : ((u128)1 << 62);
          mq = q > ((u128)1 << 62) ? (1ull << 62) : (uint64_t)q;
        }
      }
      ArrCursor arr = {0, 0}, head = {0, 0};
      if (ok) {
        arr.time = sy_arrival_gap(mq, sy_arrival_word(a.seed, a.cfg_tag, gs, (uint32_t)lane, 0));
        head = arr;
      }
      uint64_t served = 0;
      uint32_t sb = 0, gcache = 0, prev_act = 0;
      for (int i = 0; i < 10; ++i) ring[i * 32 + lane] = 0;
      uint16_t *dtab = a.dtab_rows + (int64_t)k0 * DTAB_ROW;
      const uint32_t dstar_slo = slo;
      for (int32_t c = 0; c < a.cycles; ++c) {
        const uint64_t t0 = (uint64_t)c * T;
        if (ok) while (arr.time <= t0) arr_next(arr, a, gs, (uint32_t)lane, mq);
        const bool active = ok && arr.idx > served;
        const uint32_t act_mask = __ballot_sync(FULL, active);   // a changed set: WMAX-MIN re-allocates
        const uint32_t prev_mask = prev_act;
        if (c > 0 && act_mask != prev_act) ++realloc;
        prev_act = act_mask;
        const uint32_t dm = active ? dem : 0u;
        const uint32_t al = wmaxmin_lane(dm, lane, nd, L);
        const uint32_t g = active ? (dm > (al >> 16) ? dm : (al >> 16)) : 0u;
        // d_j(b) at level g: recompute from the rows when the level changed
        uint32_t redo = __ballot_sync(FULL, active && g != gcache);
        while (redo) {
          const int j = __ffs(redo) - 1;
          redo &= redo - 1;
          dtab_from_rows(a.pb, a.p, k0 + j, a.ws_RT[k0 + j], a.ws_D[k0 + j], (int32_t)__shfl_sync(FULL, g, j), b_lo,
                         (int32_t)__shfl_sync(FULL, bs, j), dtab + j * DTAB_ROW, lane);
        }
        if (active) gcache = g;
        uint32_t runs = 0, srv = 0, nfill = 0;
        const CycRes cr = cycle_core(sm, dtab, lane, active, g, bs, sl, active ? rep : 0u, nslots, L, b_lo, false, runs,
                                     srv, sb, fill_log, DSTACK_MAX_FILL_RUNS, &nfill);
        misses += cr.misses;
        if (nfill > DSTACK_MAX_FILL_RUNS) { sst = DSTACK_ST_INVALID; break; }
        const uint64_t in0 = in_slo, late0 = late, sv0 = served, occ0 = occ_tot, nr0 = nruns;   // per-cycle series
        // ---- execute this lane's runs in start order: static windows merged with its fill runs ----
        uint32_t cnt = 0;
        uint32_t jo = active ? rep : 0u;   // this lane's static-run offset (as in cycle_core)
#pragma unroll
        for (int dlt = 1; dlt < 32; dlt <<= 1) {
          const uint32_t v = __shfl_up_sync(FULL, jo, dlt);
          if (lane >= dlt) jo += v;
        }
        jo -= active ? rep : 0u;
        if (active) {
          uint32_t r = 0, f = 0;
          while (true) {
            // next static run of this DNN
            uint32_t ss = 0xFFFFFFFFu, sd = 0;
            while (r < rep) {
              const uint32_t v = sm.sr[jo + r];
              if (v != NONE32) { ss = v & 0xFFFFu; sd = v >> 16; break; }
              ++r;
            }
            // next fill run of this DNN
            uint64_t fr = 0;
            uint32_t fsv = 0xFFFFFFFFu;
            while (f < nfill) {
              const uint64_t e = fill_log[f];
              if ((uint32_t)(e >> 56) == (uint32_t)lane) { fr = e; fsv = (uint32_t)(e >> 32) & 0xFFFFFFu; break; }
              ++f;
            }
            if (ss == 0xFFFFFFFFu && fsv == 0xFFFFFFFFu) break;
            uint32_t st, d, b;
            if (ss <= fsv) { st = ss; d = sd; b = bs; ++r; }
            else { st = fsv; d = (uint32_t)(fr >> 8) & 0xFFFFFFu; b = (uint32_t)fr & 0xFFu; ++f; }
            const uint64_t ts = t0 + (uint64_t)st * slot, te = t0 + (uint64_t)(st + d) * slot;
            while (arr.time <= ts) arr_next(arr, a, gs, (uint32_t)lane, mq);
            uint64_t q = arr.idx - served;
            if (q > b) q = b;
            if (q == 0) continue;   // empty queue: the run is void
            for (uint64_t i = 0; i < q; ++i) {
              if (te - head.time > (uint64_t)dstar_slo) late++; else in_slo++;
              arr_next(head, a, gs, (uint32_t)lane, mq);
            }
            served += q;
            cnt++;
            occ_tot += (uint64_t)g * d;
            nruns++;
          }
        }
        if (a.out.series) {   // this session's row of the per-cycle aggregate series
          const uint64_t v_in = warp_sum_u64(in_slo - in0), v_late = warp_sum_u64(late - late0);
          const uint64_t v_sv = warp_sum_u64(served - sv0), v_occ = warp_sum_u64(occ_tot - occ0);
          const uint64_t v_runs = warp_sum_u64(nruns - nr0);
          if (lane == 0) {
            unsigned long long *row = reinterpret_cast<unsigned long long *>(a.out.series) + (int64_t)c * DSTACK_SIM_SERIES;
            atomicAdd(row + DSTACK_SIM_ACTIVE, (unsigned long long)__popc(act_mask));
            if (c > 0 && act_mask != prev_mask) atomicAdd(row + DSTACK_SIM_REALLOC, 1ull);
            if (v_runs) atomicAdd(row + DSTACK_SIM_RUNS, (unsigned long long)v_runs);
            if (v_sv) atomicAdd(row + DSTACK_SIM_SERVED, (unsigned long long)v_sv);
            if (v_in) atomicAdd(row + DSTACK_SIM_IN_SLO, (unsigned long long)v_in);
            if (v_late) atomicAdd(row + DSTACK_SIM_LATE, (unsigned long long)v_late);
            if (v_occ) atomicAdd(row + DSTACK_SIM_OCC, (unsigned long long)v_occ);
            if (cr.misses) atomicAdd(row + DSTACK_SIM_MISSES, (unsigned long long)cr.misses);
          }
        }
        sb += cnt - ring[(c % 10) * 32 + lane];
        ring[(c % 10) * 32 + lane] = cnt;
        __syncwarp();
      }
      if (sst == DSTACK_ST_OK) {
        const uint64_t tend = (uint64_t)a.cycles * T;
        if (ok) {
          while (arr.time <= tend) arr_next(arr, a, gs, (uint32_t)lane, mq);
          arrived = arr.idx;
          unserved = arr.idx - served;
        }
      }
    }
    if (sst == DSTACK_ST_INVALID) { arrived = in_slo = late = unserved = occ_tot = nruns = misses = realloc = 0; T = 0; }
    arrived = warp_sum_u64(arrived); in_slo = warp_sum_u64(in_slo); late = warp_sum_u64(late);
    unserved = warp_sum_u64(unserved); occ_tot = warp_sum_u64(occ_tot); nruns = warp_sum_u64(nruns);
    if (lane == 0) {
      a.out.status[s] = sst; a.out.T_us[s] = T; a.out.arrived[s] = arrived; a.out.in_slo[s] = in_slo;
      a.out.late[s] = late; a.out.unserved[s] = unserved; a.out.occ_sum[s] = occ_tot; a.out.runs[s] = nruns;
      a.out.misses[s] = misses; a.out.realloc[s] = realloc;
    }
    __syncwarp();
  }
}

size_t sim_fill_log_bytes() { return (size_t)SIM_MAX_WARPS * DSTACK_MAX_FILL_RUNS * 8; }

int launch_sim(const SimArgs &a, cudaStream_t s, int *launches) {
  if (a.pb.num_scen <= 0) return 0;
  const size_t smem = (sizeof(CycSmem) + 10 * 32 * 4) * SIM_WARPS;
  int64_t blocks = (a.pb.num_scen + SIM_WARPS - 1) / SIM_WARPS;
  int64_t cap = (int64_t)num_sms() * (DSTACK_SIM_MINB > 1 ? DSTACK_SIM_MINB : 4);   // one wave of resident blocks
  if (cap * SIM_WARPS > SIM_MAX_WARPS) cap = SIM_MAX_WARPS / SIM_WARPS;
  if (blocks > cap) blocks = cap;
  cudaFuncSetAttribute(k_sim, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  SimArgs b = a;
  if (!DSTACK_DYN_SCEN) b.work_ctr = nullptr;
  if (b.work_ctr && cudaMemsetAsync(b.work_ctr, 0, sizeof(uint32_t), s) != cudaSuccess) return DSTACK_ELAUNCH;
  k_sim<<<(unsigned)blocks, SIM_WARPS * 32, smem, s>>>(b);
  ++*launches;
  return cudaGetLastError() == cudaSuccess ? 0 : DSTACK_ELAUNCH;
}

}  // namespace dstack
