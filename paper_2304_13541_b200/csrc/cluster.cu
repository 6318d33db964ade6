// cluster.cu -- F4, the multi-GPU cluster of §7.1 (reading R23 in DESIGN.md
// §3.5): G modelled GPUs serve each scenario's active models under four policies, one warp per scenario:
//   c = 0 exclusive: the q-th active model on GPU q mod G, temporal sharing within a GPU;
//   c = 1 temporal on every GPU (G replicas of the whole mix);
//   c = 2 D-STACK on every GPU (G replicas: WMAX-MIN over the whole mix + one session);
//   c = 3 D-STACK with placement: first-fit decreasing by demand onto GPUs of L levels, overflow to the least
//         loaded; per GPU WMAX-MIN over its subset and one session (cycle_core with the subset active).
// U = mean over the G GPUs of occupied level-slots / (nslots_i L), throughput = sum of served * 1e6 / T_i.
// The oracle's F4 (oracle/oracle.c, cluster_scenario) is the parity reference.
#include "cycle.cuh"
#include "kernels.cuh"
#include "prof.cuh"

namespace dstack {

constexpr int CLU_WARPS = 8;
#ifndef DSTACK_CLU_GRID
#define DSTACK_CLU_GRID 64   // grid: blocks per SM (A/B ms: 8 -> 203, 32 -> 201, 64 -> 197)
#endif
#ifndef DSTACK_CLU_MINB
#define DSTACK_CLU_MINB 3   // resident blocks per SM the register allocation targets (A/B, current code: 2 -> 89.5,
                            // 3 -> 81.3, 4 -> 89.8 ms; at 64 registers lane / smem addresses were rematerialised)
#endif

struct CluArgs {
  dstack_problem_t pb;
  dstack_params_t p;
  int32_t G;
  const uint16_t *demand;
  const uint8_t *batch;
  uint16_t *dtab_rows;   // workspace
  double *u, *thr;       // [num_scen * DSTACK_NCLU]
  uint32_t *work_ctr;    // workspace word: scenario counter (NULL: grid stride)
};

__global__ void __launch_bounds__(CLU_WARPS * 32, DSTACK_CLU_MINB) k_cluster(const __grid_constant__ CluArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  CycSmem &sm = reinterpret_cast<CycSmem *>(smem_raw)[warp];
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int32_t L = a.p.L, slot = a.p.slot_us, b_lo = a.p.b_min, G = a.G;
  const double NLg = (double)L;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (int64_t s = warp_next_item(a.work_ctr, -1, gwarp, nwarps, lane); s < a.pb.num_scen;
       s = warp_next_item(a.work_ctr, s, gwarp, nwarps, lane)) {
    const int32_t k0 = a.pb.scen_dnn_off[s], nd = a.pb.scen_dnn_off[s + 1] - k0;
    double ou = 0.0, othr = 0.0;   // lane c < 4 holds policy c's results
    const bool mine = lane < nd && nd <= DSTACK_MAX_DNN_PER_SCEN;
    const int k = k0 + lane;
    uint32_t dem = 0, bs = 0, slo = 0, sl = 1;
    if (mine) { dem = a.demand[k]; bs = a.batch[k]; slo = (uint32_t)a.pb.slo_us[k]; sl = slo / (uint32_t)slot; }
    const bool active = mine && dem > 0;
    uint32_t T = __reduce_max_sync(FULL, active ? slo : 0u);   // 0 when nd > DSTACK_MAX_DNN_PER_SCEN (no lane active); unconditional: see sim.cu
    int32_t nslots = 0;
    if (T > 0) {
      nslots = (int32_t)(T / (uint32_t)slot);
      const uint32_t njobs = __reduce_add_sync(FULL, active ? (uint32_t)nslots / sl : 0u);
      if (nslots > DSTACK_MAX_SLOTS || njobs > DSTACK_MAX_JOBS) T = 0;
    }
    if (T > 0) {
      uint16_t *dtab = a.dtab_rows + (int64_t)k0 * DTAB_ROW;
      // ---- placements: home0 = (rank among active, index order) mod G; home3 = first-fit decreasing ----
      const uint32_t below = __ballot_sync(FULL, active) & ((1u << lane) - 1u);
      const int32_t home0 = active ? (int32_t)((uint32_t)__popc(below) % (uint32_t)G) : -1;
      int32_t home3 = -1;
      {
        uint32_t rank = 0;   // (demand desc, index asc) among the active
#pragma unroll 4
        for (int q = 0; q < 32; ++q) {
          const uint32_t dq = __shfl_sync(FULL, dem, q);
          const bool aq = __shfl_sync(FULL, (int)active, q) != 0;
          if (aq && (dq > dem || (dq == dem && q < lane))) ++rank;
        }
        const uint32_t na = (uint32_t)__popc(__ballot_sync(FULL, active));
        uint32_t load = 0;   // lane i < G: GPU i's summed demand
        for (uint32_t q = 0; q < na; ++q) {
          const int own = __ffs(__ballot_sync(FULL, active && rank == q)) - 1;
          const uint32_t dq = __shfl_sync(FULL, dem, own);
          const uint32_t fit = __ballot_sync(FULL, lane < G && load + dq <= (uint32_t)L);
          int gi;
          if (fit) gi = __ffs(fit) - 1;
          else gi = (int)(__reduce_min_sync(FULL, lane < G ? (load << 5) | (uint32_t)lane : 0xFFFFFFFFu) & 31u);
          if (lane == gi) load += dq;
          if (lane == own) home3 = gi;
        }
      }
      // ---- session levels: g over the whole mix (c = 2) and on the model's own GPU under FFD (c = 3) ----
      uint32_t gW, gG = 0;
      {
        const uint32_t al = wmaxmin_lane(active ? dem : 0u, lane, nd, L) >> 16;
        gW = active ? (dem > al ? dem : al) : 0u;
#pragma unroll 1
        for (int gi = 0; gi < G; ++gi) {
          const bool m3 = home3 == gi;
          const uint32_t ali = wmaxmin_lane(m3 ? dem : 0u, lane, nd, L) >> 16;
          if (m3) gG = dem > ali ? dem : ali;
        }
      }
      // ---- per active model, one row pass: sum R, sum R d and the b* runs at 100% GPU (d^L), at gW and at gG ----
      uint64_t RTl = 0, Dl = 0;
      uint32_t dL = 0, dW = 0, dG = 0;
      {
        uint32_t todo = __ballot_sync(FULL, active);
        while (todo) {
          const int j = __ffs(todo) - 1;
          todo &= todo - 1;
          const int64_t kj = k0 + j;
          const int32_t bj = (int32_t)__shfl_sync(FULL, bs, j);
          const uint64_t M = a.p.mem_mode == 0 ? 1ull : (uint64_t)a.pb.mem_bw[kj];
          const uint64_t SL = (uint64_t)a.p.S_tot;
          const uint64_t SW = (uint64_t)s_of((int32_t)__shfl_sync(FULL, gW, j), a.p.S_tot, L);
          const uint64_t SG = (uint64_t)s_of((int32_t)__shfl_sync(FULL, gG, j), a.p.S_tot, L);
          uint64_t RT, D, VL, VW, VG;
          rows_pass3(a.pb, a.p, kj, bj, SL, SW, SG, RT, D, VL, VW, VG, lane);
          if (lane == j) {
            RTl = RT; Dl = D;
            dL = ceil_div_clamp16(x_of_v(a.pb, a.p, kj, RT, D, SL, bj, VL), SL * M * (uint64_t)slot);
            dW = ceil_div_clamp16(x_of_v(a.pb, a.p, kj, RT, D, SW, bj, VW), SW * M * (uint64_t)slot);
            dG = ceil_div_clamp16(x_of_v(a.pb, a.p, kj, RT, D, SG, bj, VG), SG * M * (uint64_t)slot);
          }
        }
      }
      // one D-STACK session over the members at levels g (WMAX-MIN over their demands, above) with d_j(b*) = dstar;
      // d_j(b) for b < b* (rare) from one row pass each.  Returns occ | served << 32.
      auto session = [&](bool member, int32_t ns, uint32_t g, uint32_t dstar) -> uint64_t {
        if (member) dtab[lane * DTAB_ROW + bs - 1] = (uint16_t)dstar;
        uint32_t todo = __ballot_sync(FULL, member && bs > (uint32_t)b_lo);
        while (todo) {
          const int j = __ffs(todo) - 1;
          todo &= todo - 1;
          dtab_lower(a.pb, a.p, k0 + j, shfl_u64(RTl, j), shfl_u64(Dl, j), (int32_t)__shfl_sync(FULL, g, j), b_lo,
                         (int32_t)__shfl_sync(FULL, bs, j) - 1, dtab + j * DTAB_ROW, lane);
        }
        __syncwarp();
        const uint32_t rep = member ? (uint32_t)ns / sl : 0u;
        uint32_t runs = 0, served = 0;
        const CycRes cr = cycle_core(sm, dtab, lane, member, member ? g : 0u, bs, sl, rep, ns, L, b_lo, false, runs,
                                     served);
        return (uint64_t)cr.occ_all | ((uint64_t)cr.served_tot << 32);
      };
      // temporal sharing over the members (O9): slices proportional to SLO, back-to-back b* runs at 100%
      auto temporal = [&](bool member, int32_t ns, uint64_t &occn, uint64_t &srv) {
        const uint64_t tot = warp_sum_u64(member ? (uint64_t)sl : 0ull);
        const uint64_t slice = member ? (uint64_t)ns * sl / tot : 0ull;
        const uint64_t truns = member && dL ? slice / dL : 0ull;
        occn = warp_sum_u64(slice * dem);
        srv = warp_sum_u64(truns * bs);
      };
      const double NL = (double)nslots * (double)L;
      // ---- gi = -1: the whole mix on every GPU (c = 1, 2); gi >= 0: GPU gi under c = 0 and c = 3.  One call site
      // of the session and of temporal keeps one copy of each in the instruction cache. ----
      double u0 = 0.0, t0 = 0.0, u3 = 0.0, t3 = 0.0;
#pragma unroll 1
      for (int gi = -1; gi < G; ++gi) {
        const bool m0 = gi < 0 ? active : home0 == gi, m3 = gi < 0 ? active : home3 == gi;
        const uint32_t T0 = gi < 0 ? T : __reduce_max_sync(FULL, m0 ? slo : 0u);
        const uint32_t T3 = gi < 0 ? T : __reduce_max_sync(FULL, m3 ? slo : 0u);
        if (T0 > 0) {   // temporal over m0 (c = 1 for the whole mix, c = 0 on GPU gi)
          const int32_t ns = (int32_t)(T0 / (uint32_t)slot);
          uint64_t occn, srv;
          temporal(m0, ns, occn, srv);
          const double thr = (double)srv * 1e6 / (double)T0;
          if (gi < 0) {
            if (lane == 1) { ou = (double)occn / NL; othr = (double)G * thr; }
          } else {
            u0 += (double)occn / ((double)ns * NLg) / (double)G;
            t0 += thr;
          }
        }
        if (T3 > 0) {   // D-STACK over m3 (c = 2 for the whole mix, c = 3 on GPU gi)
          const int32_t ns = (int32_t)(T3 / (uint32_t)slot);
          const uint64_t r = session(m3, ns, gi < 0 ? gW : gG, gi < 0 ? dW : dG);
          const double thr = (double)(r >> 32) * 1e6 / (double)T3;
          if (gi < 0) {
            if (lane == 2) { ou = (double)(uint32_t)r / NL; othr = (double)G * thr; }
          } else {
            u3 += (double)(uint32_t)r / ((double)ns * NLg) / (double)G;
            t3 += thr;
          }
        }
      }
      if (lane == 0) { ou = u0; othr = t0; }
      if (lane == 3) { ou = u3; othr = t3; }
    }
    if (lane < DSTACK_NCLU) { a.u[s * DSTACK_NCLU + lane] = ou; a.thr[s * DSTACK_NCLU + lane] = othr; }
    __syncwarp();
  }
}

int launch_cluster(const dstack_problem_t &pb, const dstack_params_t &p, int32_t G, const uint16_t *demand,
                   const uint8_t *batch, uint16_t *dtab_rows, double *u, double *thr, uint32_t *work_ctr, cudaStream_t s,
                   int *launches) {
  if (pb.num_scen <= 0) return 0;
  CluArgs a;
  a.pb = pb; a.p = p; a.G = G; a.demand = demand; a.batch = batch; a.dtab_rows = dtab_rows; a.u = u; a.thr = thr;
  a.work_ctr = DSTACK_DYN_SCEN ? work_ctr : nullptr;
  const size_t smem = sizeof(CycSmem) * CLU_WARPS;
  int64_t blocks = (pb.num_scen + CLU_WARPS - 1) / CLU_WARPS;
  const int64_t cap = (int64_t)num_sms() * DSTACK_CLU_GRID;
  if (blocks > cap) blocks = cap;
  cudaFuncSetAttribute(k_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (a.work_ctr) {
    if (cudaMemsetAsync(a.work_ctr, 0, sizeof(uint32_t), s) != cudaSuccess) return DSTACK_ELAUNCH;
    blocks = resident_wave(k_cluster, CLU_WARPS * 32, smem, blocks);
  }
  k_cluster<<<(unsigned)blocks, CLU_WARPS * 32, smem, s>>>(a);
  ++*launches;
  return cudaGetLastError() == cudaSuccess ? 0 : DSTACK_ELAUNCH;
}

}  // namespace dstack
