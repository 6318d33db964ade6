// cycle.cu -- a4 WMAX-MIN and a5 one D-STACK session, one warp per scenario.
//
// a4 (Algorithm WMAX-MIN): lane j holds DNN j's demand; the ascending (demand, index) order
// of "Fulfill Lowest Demand First" is realised as a per-lane rank + exclusive sum of the demands
// ranked before it, so grant_j = min(k_j, max(0, L - sum_before)) in O(32) lane-parallel steps;
// the surplus is split in Q16.16 exactly as the oracle's definition.
//
// a5 (Alg. 1 / Alg. 3 / Dynamic-schedule; §6.1): the session timeline of
// nslots = T/Delta slots lives in shared memory as one u8 occupancy per slot (levels <= 255).  Static
// jobs are generated in EDF order by a warp min-reduction over the per-DNN next repeat (deadline,
// d(b*), index); each window query is a ballot scan over 32-slot chunks that computes, per lane,
// the length of the run of fitting slots ending (Start-Early) or starting (Start-Late) at its slot,
// so a whole chunk is resolved with two ballots.  The opportunistic fill walks the decision times
// kept as a bitmask, evaluates every DNN's eligibility in parallel (lane = DNN), then serves the
// eligible ones in (runs so far, index) order by repeated min-reductions.
#include "kernels.cuh"

namespace dstack {

constexpr int CYC_WARPS = 4;
constexpr uint16_t NONE16 = 0xFFFF;



struct CycSmem {
  uint8_t occ[DSTACK_MAX_SLOTS];
  uint32_t dmask[DSTACK_MAX_SLOTS / 32];
  uint16_t dtab[DSTACK_MAX_DNN_PER_SCEN * DSTACK_MAX_BATCH];
  uint16_t starts[DSTACK_MAX_JOBS];
};

// ---------------------------------------------------------------- a4 ---
__device__ __forceinline__ uint32_t wmaxmin_lane(uint32_t dem, int lane, int nd, int32_t L) {
  // dem == 0 for lanes >= nd
  const uint32_t key = (dem << 5) | (uint32_t)lane;
  uint32_t before = 0;
#pragma unroll 8
  for (int q = 0; q < 32; ++q) {
    uint32_t kq = __shfl_sync(FULL, key, q);
    if (q < nd && kq < key) before += kq >> 5;
  }
  const uint32_t tot = __reduce_add_sync(FULL, dem);
  const int64_t rem_before = (int64_t)L - (int64_t)before;
  const uint32_t grant = rem_before <= 0 ? 0u : (uint32_t)((int64_t)dem < rem_before ? (int64_t)dem : rem_before);
  const uint64_t rem = tot >= (uint32_t)L ? 0ull : (uint64_t)(L - (int32_t)tot);
  uint64_t share = 0;
  if (tot > 0) share = (((uint64_t)dem * rem) << 16) / tot;
  return (uint32_t)(((uint64_t)grant << 16) + share);
}

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

// ---------------------------------------------------------------- a5 ---

// Start-Early: smallest s in [rel, dl-d] with occ[u] + g <= L for u in [s, s+d); -1 if none.
__device__ __forceinline__ int find_early(const uint8_t *occ, int rel, int dl, int d, int g, int L, int lane) {
  if (d > dl - rel) return -1;
  int run = 0;
  for (int base = rel; base < dl; base += 32) {
    const int u = base + lane;
    const bool fit = u < dl && (int)occ[u] + g <= L;
    const uint32_t mask = __ballot_sync(FULL, fit);
    const uint32_t z = (~mask) & ((2u << lane) - 1u);
    const int len = z == 0 ? run + lane + 1 : lane - (31 - __clz(z));
    const uint32_t hit = __ballot_sync(FULL, fit && len >= d);
    if (hit) return base + (__ffs(hit) - 1) - d + 1;
    run = mask == FULL ? run + 32 : __clz(~mask);
  }
  return -1;
}

// Start-Late: largest s in [rel, dl-d] with occ[u] + g <= L for u in [s, s+d); -1 if none.
__device__ __forceinline__ int find_late(const uint8_t *occ, int rel, int dl, int d, int g, int L, int lane) {
  if (d > dl - rel) return -1;
  int run = 0;
  for (int base = dl - 32; base + 32 > rel; base -= 32) {
    const int u = base + lane;
    const bool fit = u >= rel && u < dl && (int)occ[u] + g <= L;
    const uint32_t mask = __ballot_sync(FULL, fit);
    const uint32_t z = (~mask) & ~((1u << lane) - 1u);
    const int len = z == 0 ? (32 - lane) + run : (__ffs(z) - 1) - lane;
    const uint32_t hit = __ballot_sync(FULL, fit && len >= d);
    if (hit) return base + (31 - __clz(hit));
    run = mask == FULL ? run + 32 : __ffs(~mask) - 1;
  }
  return -1;
}

__device__ __forceinline__ void occ_add(uint8_t *occ, int s, int d, int g, int lane) {
  for (int u = s + lane; u < s + d; u += 32) occ[u] = (uint8_t)(occ[u] + g);
  __syncwarp();
}

__global__ void __launch_bounds__(CYC_WARPS * 32) k_cycle(CycArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  CycSmem &sm = reinterpret_cast<CycSmem *>(smem_raw)[warp];
  const int32_t L = a.p.L, S_tot = a.p.S_tot, slot = a.p.slot_us, b_lo = a.p.b_min;
  const int mem_mode = a.p.mem_mode;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;

  for (int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < a.pb.num_scen; s += nwarps) {
    const int32_t k0 = a.pb.scen_dnn_off[s], nd = a.pb.scen_dnn_off[s + 1] - k0;
    uint8_t sst = DSTACK_ST_OK;
    uint32_t T = 0, misses = 0;
    double us = 0.0, uu = 0.0, th = 0.0;
    // per-lane DNN state
    const bool mine = lane < nd && nd <= DSTACK_MAX_DNN_PER_SCEN;
    const int k = k0 + lane;
    uint32_t dem = 0, bs = 0, g = 0, sl = 1, rep = 0, slo = 0;
    uint32_t runs = 0, served = 0;
    if (mine) {
      slo = (uint32_t)a.pb.slo_us[k];
      bs = a.batch[k];
      if (a.hook_level) {
        g = a.hook_level[k] > 0 ? (uint32_t)a.hook_level[k] : 0u;
        dem = g;
      } else {
        dem = a.demand[k];
        const uint32_t al = a.alloc[k] >> 16;
        g = dem == 0 ? 0u : (dem > al ? dem : al);
      }
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
    }
    if (sst == DSTACK_ST_OK) {
      // ---- runtimes d_j(b) = ceil(X(g_j, b) / (S(g_j) M Delta)) for b in [b_lo, b*_j] ----
      for (int j = 0; j < nd; ++j) {
        const uint32_t gj = __shfl_sync(FULL, g, j), bsj = __shfl_sync(FULL, bs, j);
        if (gj == 0) continue;
        const int kj = k0 + j;
        if (a.hook_level) {
          if (lane == 0) {
            int32_t hd = a.hook_d[kj];
            sm.dtab[j * DSTACK_MAX_BATCH + bsj - 1] = (uint16_t)(hd > 0xFFFF ? 0xFFFF : (hd < 0 ? 0 : hd));
          }
          continue;
        }
        const int64_t r0 = a.pb.dnn_row_off[kj];
        const int32_t K = (int32_t)(a.pb.dnn_row_off[kj + 1] - r0);
        const uint64_t M = mem_mode == 0 ? 1ull : (uint64_t)a.pb.mem_bw[kj];
        const uint64_t t_p = (uint64_t)a.pb.t_p[kj], t_np = (uint64_t)a.pb.t_np[kj];
        const uint64_t S = (uint64_t)s_of((int32_t)gj, S_tot, L);
        const uint32_t *n = a.pb.n + r0;
        const uint16_t *r = a.pb.r + r0;
        const uint32_t *dd = a.pb.d + r0;
        uint64_t RT = 0, D = 0;
        for (int i = lane; i < K; i += 32) { RT += r[i]; D += (uint64_t)r[i] * dd[i]; }
        RT = warp_sum_u64(RT); D = warp_sum_u64(D);
        const uint64_t den = S * M * (uint64_t)slot;
        for (int32_t b = b_lo; b <= (int32_t)bsj; ++b) {
          uint64_t V = 0;   // sum_i R_i * max(S, N_i(b)) over N_i >= 1  (= S*A + U)
          for (int i = lane; i < K; i += 32) {
            const uint64_t nn = n[i];
            const uint64_t N = a.p.par_mode == 0 ? (uint64_t)b * nn : ((uint64_t)b * nn + 2047) >> 11;
            if (N >= 1) V += (uint64_t)r[i] * (N > S ? N : S);
          }
          V = warp_sum_u64(V);
          uint64_t X = (a.p.wse_mode == 0 ? (uint64_t)b : 1ull) * t_np * RT * S * M + M * t_p * V;
          if (mem_mode == 1) X += (uint64_t)b * D;
          else if (mem_mode == 2) X += (uint64_t)b * D * S * S;
          const uint64_t dslots = (X + den - 1) / den;
          if (lane == 0) sm.dtab[j * DSTACK_MAX_BATCH + b - 1] = (uint16_t)(dslots > 0xFFFF ? 0xFFFF : dslots);
        }
      }
      // ---- clear timeline ----
      for (int u = lane; u < nslots; u += 32) sm.occ[u] = 0;
      for (int w = lane; w < DSTACK_MAX_SLOTS / 32; w += 32) sm.dmask[w] = 0;
      __syncwarp();
      // per-lane static job bookkeeping
      uint32_t joff = rep;   // exclusive prefix of rep over lanes
#pragma unroll
      for (int dlt = 1; dlt < 32; dlt <<= 1) {
        uint32_t v = __shfl_up_sync(FULL, joff, dlt);
        if (lane >= dlt) joff += v;
      }
      joff -= rep;
      const uint32_t njobs = __reduce_add_sync(FULL, rep);
      const uint32_t dstar = active ? sm.dtab[lane * DSTACK_MAX_BATCH + bs - 1] : 0u;
      uint32_t nextr = 0;
      // ---- static placement in EDF order (Alg. 1 l.5; even repeats Start-Early, odd Start-Late) ----
      for (uint32_t q = 0; q < njobs; ++q) {
        const bool has = active && nextr < rep;
        const uint32_t dl = has ? (nextr + 1) * sl : 0xFFFFFFFFu;
        const uint32_t mindl = __reduce_min_sync(FULL, dl);
        const uint32_t key2 = (has && dl == mindl) ? (((dstar > 0xFFFF ? 0xFFFFu : dstar) << 5) | (uint32_t)lane) : 0xFFFFFFFFu;
        const uint32_t mk = __reduce_min_sync(FULL, key2);
        const int j = (int)(mk & 31u);
        const int rj = (int)__shfl_sync(FULL, nextr, j);
        const int slj = (int)__shfl_sync(FULL, sl, j);
        const int gj = (int)__shfl_sync(FULL, g, j);
        const int dj = (int)__shfl_sync(FULL, dstar, j);
        const int offj = (int)__shfl_sync(FULL, joff, j);
        const int rel = rj * slj, dlv = rel + slj;
        const int st = (rj & 1) ? find_late(sm.occ, rel, dlv, dj, gj, L, lane) : find_early(sm.occ, rel, dlv, dj, gj, L, lane);
        if (st >= 0) {
          occ_add(sm.occ, st, dj, gj, lane);
          if (lane == 0) {
            sm.starts[offj + rj] = (uint16_t)st;
            const int e = st + dj;
            if (e < nslots) sm.dmask[e >> 5] |= 1u << (e & 31);
          }
          if (lane == j) { runs++; served += bs; }
        } else {
          if (lane == 0) sm.starts[offj + rj] = NONE16;
          misses++;
          sst = DSTACK_ST_OVERSUBSCRIBED;
        }
        if (lane == j) nextr++;
        __syncwarp();
      }
      // U_static
      uint32_t osum = 0;
      for (int u = lane; u < nslots; u += 32) osum += sm.occ[u];
      const uint32_t occ_static = __reduce_add_sync(FULL, osum);
      // ---- opportunistic fill at decision times {0} u {run ends} ----
      if (lane == 0) sm.dmask[0] |= 1u;
      __syncwarp();
      uint32_t count = runs;
      int fs = -1, fe = -1;
      const int nwords = (nslots + 31) >> 5;
      int t = -1;
      while (true) {
        // next decision time > t
        const int start = t + 1;
        int nt = -1;
        for (int wb = start >> 5; wb < nwords; wb += 32) {
          const int w = wb + lane;
          uint32_t v = w < nwords ? sm.dmask[w] : 0u;
          if (w == (start >> 5)) v &= ~((1u << (start & 31)) - 1u);
          const uint32_t bal = __ballot_sync(FULL, v != 0);
          if (bal) {
            const int p = __ffs(bal) - 1;
            const uint32_t word = __shfl_sync(FULL, v, p);
            nt = (wb + p) * 32 + __ffs(word) - 1;
            break;
          }
        }
        if (nt < 0 || nt >= nslots) break;
        t = nt;
        int occ_t = sm.occ[t];
        // per-lane eligibility: not running at t, fits at t
        bool elig = false;
        int ns = nslots;
        if (active) {
          const int rr = t / (int)sl;
          bool covered = (fs <= t && t < fe);
          if (rr < (int)rep) {
            const uint16_t s0 = sm.starts[joff + rr];
            if (s0 != NONE16) {
              if ((int)s0 <= t && t < (int)s0 + (int)dstar) covered = true;
              if ((int)s0 > t) ns = s0;
            }
            if (ns == nslots) {
              for (int r2 = rr + 1; r2 < (int)rep; ++r2) {
                const uint16_t s2 = sm.starts[joff + r2];
                if (s2 != NONE16) { ns = s2; break; }
              }
            }
          }
          elig = !covered && occ_t + (int)g <= L;
        }
        uint32_t key = elig ? ((count << 5) | (uint32_t)lane) : 0xFFFFFFFFu;
        while (true) {
          const uint32_t mk = __reduce_min_sync(FULL, key);
          if (mk == 0xFFFFFFFFu) break;
          const int j = (int)(mk & 31u);
          if (lane == j) key = 0xFFFFFFFFu;
          const int gj = (int)__shfl_sync(FULL, g, j);
          if (occ_t + gj > L) continue;
          const int nsj = (int)__shfl_sync(FULL, ns, j);
          const int bsj = (int)__shfl_sync(FULL, bs, j);
          const int limit = nsj < nslots ? nsj : nslots;
          // slice: first u in [t, limit) with occ[u] + g > L
          int kslice = limit - t;
          for (int base = t; base < limit; base += 32) {
            const int u = base + lane;
            const bool blocked = u < limit && (int)sm.occ[u] + gj > L;
            const uint32_t bal = __ballot_sync(FULL, blocked);
            if (bal) { kslice = base + __ffs(bal) - 1 - t; break; }
          }
          // largest b in [b_lo, b*] with d(b) <= slice
          int bsel = 0;
          for (int b0 = b_lo + 32 * ((bsj - b_lo) >> 5); b0 >= b_lo; b0 -= 32) {
            const int b = b0 + lane;
            bool ok = false;
            if (b <= bsj) {
              if (a.hook_level) ok = (b == bsj) && (int)sm.dtab[j * DSTACK_MAX_BATCH + b - 1] <= kslice;
              else ok = (int)sm.dtab[j * DSTACK_MAX_BATCH + b - 1] <= kslice;
            }
            const uint32_t bal = __ballot_sync(FULL, ok);
            if (bal) { bsel = b0 + 31 - __clz(bal); break; }
          }
          if (bsel == 0) continue;
          const int dsel = sm.dtab[j * DSTACK_MAX_BATCH + bsel - 1];
          occ_add(sm.occ, t, dsel, gj, lane);
          occ_t += gj;
          if (lane == 0 && t + dsel < nslots) sm.dmask[(t + dsel) >> 5] |= 1u << ((t + dsel) & 31);
          __syncwarp();
          if (lane == j) { count++; runs++; served += (uint32_t)bsel; fs = t; fe = t + dsel; }
        }
      }
      osum = 0;
      for (int u = lane; u < nslots; u += 32) osum += sm.occ[u];
      const uint32_t occ_all = __reduce_add_sync(FULL, osum);
      const uint32_t served_tot = __reduce_add_sync(FULL, served);
      us = (double)occ_static / ((double)nslots * (double)L);
      uu = (double)occ_all / ((double)nslots * (double)L);
      th = (double)served_tot * 1e6 / (double)T;
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
      if (a.scen_status) a.scen_status[s] = sst;
      if (a.T_us) a.T_us[s] = T;
      if (a.u_static) a.u_static[s] = us;
      if (a.u) a.u[s] = uu;
      if (a.thr) a.thr[s] = th;
      if (a.misses) a.misses[s] = misses;
    }
    __syncwarp();
  }
}

int launch_wmaxmin(int32_t num_scen, const int32_t *off, int32_t L, const uint16_t *demand, uint32_t *alloc,
                   cudaStream_t s, int *launches) {
  if (num_scen <= 0) return 0;
  int64_t blocks = ((int64_t)num_scen * 32 + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_wmaxmin<<<(unsigned)blocks, 256, 0, s>>>(num_scen, off, L, demand, alloc);
  ++*launches;
  return cudaGetLastError() == cudaSuccess ? 0 : DSTACK_ELAUNCH;
}

int launch_cycle(const CycArgs &a, cudaStream_t s, int *launches) {
  if (a.pb.num_scen <= 0) return 0;
  const size_t smem = sizeof(CycSmem) * CYC_WARPS;
  int64_t blocks = (a.pb.num_scen + CYC_WARPS - 1) / CYC_WARPS;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
  cudaFuncSetAttribute(k_cycle, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_cycle<<<(unsigned)blocks, CYC_WARPS * 32, smem, s>>>(a);
  ++*launches;
  return cudaGetLastError() == cudaSuccess ? 0 : DSTACK_ELAUNCH;
}

}  // namespace dstack
