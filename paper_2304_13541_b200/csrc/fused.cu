// fused.cu -- dstack_eval_batch's a1-a5 in ONE kernel, one warp per scenario (persistent grid).
//
// Per scenario the warp (i) analyses its DNNs one after the other (prof.cuh: row pass, coefficient
// tables, exact branch-and-bound) keeping each DNN's result in lane j's registers; while a DNN's
// tables are still in shared memory it also evaluates d_j(b) at g = demand_j, which is the level the
// schedule uses whenever the scenario is oversubscribed (WMAX-MIN then grants at most the demand);
// (ii) runs WMAX-MIN across the lanes; (iii) recomputes d_j(b) from the rows -- an L2 re-read of a
// scenario the warp has just streamed -- only for DNNs whose level WMAX-MIN raised; (iv) simulates
// the session (cycle.cuh) in a shared-memory region that overlays the dead coefficient tables.
// The rows are read from HBM once; per-DNN intermediates never leave the SM.
#include "cycle.cuh"
#include "kernels.cuh"
#include "prof.cuh"

namespace dstack {

constexpr int FUSED_WARPS = 8;

__host__ __device__ inline size_t fused_warp_bytes(int S_tot) {
  size_t t = (size_t)16 * (S_tot + 1);
  size_t c = sizeof(CycSmem);
  size_t m = t > c ? t : c;
  return (m + 15) & ~(size_t)15;
}

template <int PAR>
__global__ void __launch_bounds__(FUSED_WARPS * 32, 3) k_fused(FusedArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int L = a.p.L, S_tot = a.p.S_tot, slot = a.p.slot_us, b_lo = a.p.b_min;
  uint16_t *Stab = (uint16_t *)smem;
  const size_t stab_bytes = ((size_t)(L + 1) * 2 + 15) & ~(size_t)15;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char *wreg = smem + stab_bytes + (size_t)warp * fused_warp_bytes(S_tot);
  uint64_t *cA = (uint64_t *)wreg;
  uint64_t *cU = cA + (S_tot + 1);
  CycSmem &sm = *reinterpret_cast<CycSmem *>(wreg);
  fill_stab(Stab, L, S_tot);
  __syncthreads();
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  uint16_t *dtab = a.dtab_slab + gwarp * DTAB_WORDS;

  for (int64_t s = gwarp; s < a.pb.num_scen; s += nwarps) {
    const int32_t k0 = a.pb.scen_dnn_off[s], nd = a.pb.scen_dnn_off[s + 1] - k0;
    const bool fits = nd <= DSTACK_MAX_DNN_PER_SCEN;
    // stage the rows of this warp's NEXT scenario into L2 while this one is analysed and simulated
    if (lane == 0 && s + nwarps < a.pb.num_scen) {
      const int64_t sn = s + nwarps;
      const int64_t q0 = a.pb.dnn_row_off[a.pb.scen_dnn_off[sn]], q1 = a.pb.dnn_row_off[a.pb.scen_dnn_off[sn + 1]];
      prefetch_l2(a.pb.n + q0, (q1 - q0) * 4);
      prefetch_l2(a.pb.r + q0, (q1 - q0) * 2);
      prefetch_l2(a.pb.d + q0, (q1 - q0) * 4);
    }
    // ---- (i) a1-a3 per DNN; lane j keeps DNN j's results ----
    uint32_t dem = 0, bs = 0;
    uint64_t RT = 0, D = 0;
    for (int j = 0; j < nd; ++j) {
      const int64_t k = k0 + j;
      const DnnRes r = analyze_dnn<PAR>(a.pb, a.p, k, Stab, cA, cU, lane, 0, 0);
      const bool ok = r.st == DSTACK_ST_OK;
      if (lane == (j & 31)) {
        dem = ok ? r.demand : 0u; bs = ok ? r.b : 0u; RT = r.RT; D = r.D;
        a.demand[k] = (uint16_t)dem;
        a.batch[k] = (uint8_t)bs;
        a.knee[k] = ok ? r.knee : 0;
        a.status[k] = r.st;
      }
      if (PAR == 0 && ok && fits)   // speculative d_j(b) at g = demand_j from the live tables
        dtab_from_tables(a.pb, a.p, k, cA, cU, r.RT, r.D, r.demand, b_lo, r.b, dtab + j * DSTACK_MAX_BATCH, lane);
      __syncwarp();
    }
    uint8_t sst = DSTACK_ST_OK;
    uint32_t T = 0, g = 0, sl = 1, rep = 0, slo = 0, runs = 0, served = 0;
    int32_t nslots = 0;
    CycRes cr; cr.occ_static = cr.occ_all = cr.served_tot = cr.misses = 0; cr.oversub = false;
    const bool mine = lane < nd && fits;
    if (!fits) {
      sst = DSTACK_ST_INVALID;
      for (int j = lane; j < nd; j += 32) {
        a.alloc[k0 + j] = 0;
        if (a.level) a.level[k0 + j] = 0;
        if (a.runs) a.runs[k0 + j] = 0;
        if (a.served) a.served[k0 + j] = 0;
      }
    } else {
      // ---- (ii) a4 WMAX-MIN ----
      const uint32_t al = wmaxmin_lane(mine ? dem : 0u, lane, nd, L);
      if (mine) a.alloc[k0 + lane] = al;
      const bool active = mine && dem > 0;
      g = active ? (dem > (al >> 16) ? dem : (al >> 16)) : 0u;
      if (mine) slo = (uint32_t)a.pb.slo_us[k0 + lane];
      T = __reduce_max_sync(FULL, active ? slo : 0u);
      if (T == 0) sst = DSTACK_ST_INFEASIBLE;
      if (sst == DSTACK_ST_OK) {
        nslots = (int32_t)(T / (uint32_t)slot);
        if (active) { sl = slo / (uint32_t)slot; rep = (uint32_t)nslots / sl; }
        const uint32_t njobs = __reduce_add_sync(FULL, rep);
        if (nslots > DSTACK_MAX_SLOTS || njobs > DSTACK_MAX_JOBS) { sst = DSTACK_ST_INVALID; T = 0; }
      }
      if (sst == DSTACK_ST_OK) {
        // ---- (iii) d_j(b) at the final level where WMAX-MIN raised it (or threads mode) ----
        uint32_t redo = __ballot_sync(FULL, active && (PAR == 1 || g != dem));
        while (redo) {
          const int j = __ffs(redo) - 1;
          redo &= redo - 1;
          dtab_from_rows(a.pb, a.p, k0 + j, shfl_u64(RT, j), shfl_u64(D, j), (int32_t)__shfl_sync(FULL, g, j), b_lo,
                         (int32_t)__shfl_sync(FULL, bs, j), dtab + j * DSTACK_MAX_BATCH, lane);
        }
        // ---- (iv) a5 the session ----
        cr = cycle_core(sm, dtab, lane, active, g, bs, sl, rep, nslots, L, b_lo, false, runs, served);
        if (cr.oversub) sst = DSTACK_ST_OVERSUBSCRIBED;
      }
      if (mine) {
        if (a.level) a.level[k0 + lane] = (uint16_t)(sst == DSTACK_ST_OK || sst == DSTACK_ST_OVERSUBSCRIBED ? g : 0u);
        if (a.runs) a.runs[k0 + lane] = (uint16_t)runs;
        if (a.served) a.served[k0 + lane] = served;
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
    }
    __syncwarp();
  }
}

int launch_fused(const FusedArgs &a, cudaStream_t s, int *launches) {
  if (a.pb.num_scen <= 0) return 0;
  const size_t smem = (((size_t)(a.p.L + 1) * 2 + 15) & ~(size_t)15) + FUSED_WARPS * fused_warp_bytes(a.p.S_tot);
  int64_t blocks = (a.pb.num_scen + FUSED_WARPS - 1) / FUSED_WARPS;
  int64_t cap = (int64_t)num_sms() * 8;
  if (cap * FUSED_WARPS > DTAB_MAX_WARPS) cap = DTAB_MAX_WARPS / FUSED_WARPS;
  if (blocks > cap) blocks = cap;
  if (a.p.par_mode == 0) {
    cudaFuncSetAttribute(k_fused<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_fused<0><<<(unsigned)blocks, FUSED_WARPS * 32, smem, s>>>(a);
  } else {
    cudaFuncSetAttribute(k_fused<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_fused<1><<<(unsigned)blocks, FUSED_WARPS * 32, smem, s>>>(a);
  }
  ++*launches;
  return cudaGetLastError() == cudaSuccess ? 0 : DSTACK_ELAUNCH;
}

}  // namespace dstack
