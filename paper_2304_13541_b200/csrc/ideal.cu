// ideal.cu -- a6: the ideal per-kernel-GPU% scheduler (§6.2, Eqs. 13-14).
//
// k_ideal_rows (warp per DNN, lane per kernel row): execution demand g_e = Eq. 6 knee of the one-row
// DNN {n_i, R = 1, d_i} at b*_j ("we computed the knee of each kernel") and duration
// tau_e = ceil(f_e(g_e)) us.  Per lane the one-row latency has only two regimes (S < N_i and
// S >= N_i), so the knee scan is a register loop over the L levels with the same exact comparison
// as the batch search.
//
// k_ideal_sim (thread per scenario): event-driven preemptive schedule.  Each active DNN runs batches
// of b* back-to-back; at every event the eligible set is each DNN's current kernel execution (chain
// constraint of Eq. 14); the subset maximising sum g <= L (Eq. 13's per-slot maximisation, slot -> 0
// limit) is found with a 256-bit subset-sum bitset DP over the items in priority order (batch
// deadline, index), and the lexicographically-first optimal subset is read back from the suffix
// reachability sets.  Selected executions progress to the first completion.
#include "kernels.cuh"

namespace dstack {



__global__ void __launch_bounds__(256) k_ideal_rows(IdealArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int32_t L = a.p.L, S_tot = a.p.S_tot;
  const int mem_mode = a.p.mem_mode;
  for (int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < a.pb.num_dnn; k += nwarps) {
    if (a.demand[k] == 0) continue;
    const int64_t r0 = a.pb.dnn_row_off[k], r1 = a.pb.dnn_row_off[k + 1];
    const uint64_t b = a.batch[k];
    const uint64_t M = mem_mode == 0 ? 1ull : (uint64_t)a.pb.mem_bw[k];
    const uint64_t t_p = (uint64_t)a.pb.t_p[k], t_np = (uint64_t)a.pb.t_np[k];
    const uint64_t wC = (a.p.wse_mode == 0 ? b : 1ull) * t_np * M;
    for (int64_t i = r0 + lane; i < r1; i += 32) {
      const uint64_t nn = a.pb.n[i];
      const uint64_t N = a.p.par_mode == 0 ? b * nn : (b * nn + 2047) >> 11;
      const uint64_t dd = a.pb.d[i];
      uint32_t bestS = 0, bestl = 0;
      uint64_t bestX = 0;
      for (int32_t l = 1; l <= L; ++l) {
        const uint64_t S = (uint64_t)s_of(l, S_tot, L);
        uint64_t X = wC * S + (N >= 1 ? M * t_p * (N > S ? N : S) : 0ull);
        if (mem_mode == 1) X += b * dd;
        else if (mem_mode == 2) X += b * dd * S * S;
        if (bestl == 0 || cmp_score((uint32_t)S, X, (float)X, bestS, bestX, (float)bestX) > 0) {
          bestS = (uint32_t)S; bestl = (uint32_t)l; bestX = X;
        }
      }
      const uint64_t den = (uint64_t)bestS * M;
      const uint64_t tau = (bestX + den - 1) / den;
      a.ex_g[i] = (uint16_t)bestl;
      a.ex_tau[i] = (uint32_t)(tau > 0xFFFFFFFFull ? 0xFFFFFFFFull : tau);
    }
  }
}

struct Bits256 { uint64_t w[4]; };

__device__ __forceinline__ Bits256 shl_or(const Bits256 &x, int g, int L) {
  // x | (x << g), truncated to bits 0..L
  Bits256 y;
  const int ws = g >> 6, bs = g & 63;
#pragma unroll
  for (int i = 3; i >= 0; --i) {
    uint64_t v = 0;
    const int src = i - ws;
    if (src >= 0) {
      v = x.w[src] << bs;
      if (bs && src - 1 >= 0) v |= x.w[src - 1] >> (64 - bs);
    }
    y.w[i] = x.w[i] | v;
  }
  // truncate above L
  const int lw = L >> 6, lb = L & 63;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (i > lw) y.w[i] = 0;
    else if (i == lw && lb < 63) y.w[i] &= (2ull << lb) - 1ull;
  }
  return y;
}

__device__ __forceinline__ bool bit_at(const Bits256 &x, int s) { return (x.w[s >> 6] >> (s & 63)) & 1ull; }

__global__ void __launch_bounds__(128) k_ideal_sim(IdealArgs a) {
  const int32_t L = a.p.L, slot = a.p.slot_us;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < a.pb.num_scen;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int32_t k0 = a.pb.scen_dnn_off[s], nd = a.pb.scen_dnn_off[s + 1] - k0;
    double ui = 0.0, ti = 0.0;
    bool run = nd >= 1 && nd <= DSTACK_MAX_DNN_PER_SCEN;
    uint32_t T = 0;
    if (run) {
      uint32_t njobs = 0;
      for (int j = 0; j < nd; ++j)
        if (a.demand[k0 + j] > 0 && (uint32_t)a.pb.slo_us[k0 + j] > T) T = (uint32_t)a.pb.slo_us[k0 + j];
      if (T == 0) run = false;
      else {
        const uint32_t nslots = T / (uint32_t)slot;
        for (int j = 0; j < nd; ++j)
          if (a.demand[k0 + j] > 0) njobs += nslots / ((uint32_t)a.pb.slo_us[k0 + j] / (uint32_t)slot);
        if (nslots > DSTACK_MAX_SLOTS || njobs > DSTACK_MAX_JOBS) run = false;
      }
    }
    if (run) {
      int64_t rowpos[DSTACK_MAX_DNN_PER_SCEN];   // current row (absolute index)
      uint32_t rep[DSTACK_MAX_DNN_PER_SCEN];     // executions of the current row done
      uint64_t rem[DSTACK_MAX_DNN_PER_SCEN];
      uint32_t dline[DSTACK_MAX_DNN_PER_SCEN];   // batch start + SLO
      uint32_t comp[DSTACK_MAX_DNN_PER_SCEN];
      uint8_t ord[DSTACK_MAX_DNN_PER_SCEN];
      Bits256 reach[DSTACK_MAX_DNN_PER_SCEN + 1];
      int no = 0;
      for (int j = 0; j < nd; ++j) {
        comp[j] = 0;
        const int k = k0 + j;
        if (a.demand[k] == 0) continue;
        const int64_t r0 = a.pb.dnn_row_off[k], r1 = a.pb.dnn_row_off[k + 1];
        int64_t i = r0;
        while (i < r1 && a.ex_tau[i] == 0) ++i;
        if (i >= r1) continue;                 // all-zero chain: never runs
        rowpos[j] = i; rep[j] = 0; rem[j] = a.ex_tau[i];
        dline[j] = (uint32_t)a.pb.slo_us[k];
        ord[no++] = (uint8_t)j;
      }
      uint64_t util = 0, t = 0;
      while (no > 0 && t < T) {
        // priority order: (deadline, index) -- insertion sort (nearly sorted between events)
        for (int q = 1; q < no; ++q) {
          const uint8_t v = ord[q];
          int p = q - 1;
          while (p >= 0 && (dline[ord[p]] > dline[v] || (dline[ord[p]] == dline[v] && ord[p] > v))) {
            ord[p + 1] = ord[p]; --p;
          }
          ord[p + 1] = v;
        }
        reach[no].w[0] = 1; reach[no].w[1] = reach[no].w[2] = reach[no].w[3] = 0;
        for (int q = no - 1; q >= 0; --q) reach[q] = shl_or(reach[q + 1], a.ex_g[rowpos[ord[q]]], L);
        int target = L;
        while (target > 0 && !bit_at(reach[0], target)) --target;
        const uint64_t gsum = (uint64_t)target;
        uint64_t dt = ~0ull;
        uint32_t selmask = 0;
        for (int q = 0; q < no; ++q) {
          const int j = ord[q];
          const int gk = a.ex_g[rowpos[j]];
          if (gk <= target && bit_at(reach[q + 1], target - gk)) {
            selmask |= 1u << j; target -= gk;
            if (rem[j] < dt) dt = rem[j];
          }
        }
        if (selmask == 0 || dt == 0) break;
        if (dt > (uint64_t)T - t) dt = (uint64_t)T - t;
        util += gsum * dt;
        t += dt;
        for (int q = 0; q < no; ++q) {
          const int j = ord[q];
          if (!((selmask >> j) & 1u)) continue;
          rem[j] -= dt;
          if (rem[j] > 0) continue;
          const int k = k0 + j;
          const int64_t r0 = a.pb.dnn_row_off[k], r1 = a.pb.dnn_row_off[k + 1];
          int64_t i = rowpos[j];
          uint32_t rp = rep[j] + 1;
          if (rp >= a.pb.r[i]) { rp = 0; ++i; while (i < r1 && a.ex_tau[i] == 0) ++i; }
          if (i >= r1) {                       // batch complete: next batch back-to-back
            comp[j]++;
            dline[j] = (uint32_t)t + (uint32_t)a.pb.slo_us[k];
            i = r0;
            while (a.ex_tau[i] == 0) ++i;
            rp = 0;
          }
          rowpos[j] = i; rep[j] = rp; rem[j] = a.ex_tau[i];
        }
      }
      uint64_t bsum = 0;
      for (int j = 0; j < nd; ++j) bsum += (uint64_t)comp[j] * a.batch[k0 + j];
      ui = (double)util / ((double)L * (double)T);
      ti = (double)bsum * 1e6 / (double)T;
    }
    if (a.u_ideal) a.u_ideal[s] = ui;
    if (a.thr_ideal) a.thr_ideal[s] = ti;
  }
}

size_t ideal_ws_bytes(int64_t num_rows) {
  size_t g = ((size_t)(num_rows + 8) * 2 + 255) & ~(size_t)255;
  size_t t = ((size_t)(num_rows + 8) * 4 + 255) & ~(size_t)255;
  return g + t;
}

int launch_ideal(IdealArgs a, void *ws, cudaStream_t s, int *launches) {
  if (a.pb.num_scen <= 0) return 0;
  const int64_t num_rows = a.pb.num_rows;
  a.ex_g = (uint16_t *)ws;
  a.ex_tau = (uint32_t *)((char *)ws + (((size_t)(num_rows + 8) * 2 + 255) & ~(size_t)255));
  if (a.pb.num_dnn > 0) {
    int64_t blocks = ((int64_t)a.pb.num_dnn * 32 + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_ideal_rows<<<(unsigned)blocks, 256, 0, s>>>(a);
    ++*launches;
  }
  int64_t blocks = (a.pb.num_scen + 127) / 128;
  if (blocks > 148 * 64) blocks = 148 * 64;
  k_ideal_sim<<<(unsigned)blocks, 128, 0, s>>>(a);
  ++*launches;
  return cudaGetLastError() == cudaSuccess ? 0 : DSTACK_ELAUNCH;
}

}  // namespace dstack
