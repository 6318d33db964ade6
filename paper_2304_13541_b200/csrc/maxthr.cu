// maxthr.cu -- O9b, the max-throughput comparison scheduler of §6.3 ("a schedule that maximizes the sum
// of the throughput across all the models"), reading R24: over one session of nslots slots every
// active model j runs at its session level g_j as non-overlapping runs of a batch b in [b_lo, b*_j] lasting
// d_j(b) slots (O1 at g_j), starting at slot boundaries, inside the session, with the summed level of the runs in
// progress <= L at every slot; the value is the number of requests served.
//
// One block per scenario (work counter).  Warp 0 derives the session (g_j from a3/a4, T = max SLO, d_j(b) from the
// rows) and the state space: r_j = slots left of model j's run in progress, mixed radix over (max_b d_j(b) + 1).
// Then the block runs the exact backward recursion V_t(r) = max over the starts at t (each idle model: none, or one
// batch -- per distinct run length only its largest batch, the others are dominated) whose occupancy stays <= L
// of (sum b) + V_{t+1}(r - 1), threads over states, the two layers of V in shared memory.
#include "kernels.cuh"
#include "prof.cuh"

namespace dstack {

constexpr int MT_THREADS = 256;
constexpr int MT_MAX_ACT = 8;
constexpr int MT_MAX_STATES = 8192;   // the state-space cap (the oracle applies the same rule)

struct MtShared {
  uint32_t V[2][MT_MAX_STATES];
  uint16_t dtab[MT_MAX_ACT][DSTACK_MAX_BATCH];
  uint32_t g[MT_MAX_ACT], D[MT_MAX_ACT], radix[MT_MAX_ACT], nopt[MT_MAX_ACT];
  uint16_t od[MT_MAX_ACT][DSTACK_MAX_BATCH], ob[MT_MAX_ACT][DSTACK_MAX_BATCH];   // options: run length, batch
  int32_t n, nslots, nst, status;
  uint32_t scen;
};

__global__ void __launch_bounds__(MT_THREADS) k_maxthr(const __grid_constant__ MtArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  MtShared &sm = *reinterpret_cast<MtShared *>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int32_t L = a.p.L, slot = a.p.slot_us, b_lo = a.p.b_min;
  while (true) {
    if (tid == 0) sm.scen = atomicAdd(a.work_ctr, 1u);
    __syncthreads();
    const int64_t s = sm.scen;
    if (s >= a.pb.num_scen) break;
    if (warp == 0) {
      // ---- the session (eval-path quantities) and the state space ----
      const int32_t k0 = a.pb.scen_dnn_off[s], nd = a.pb.scen_dnn_off[s + 1] - k0;
      int32_t status = DSTACK_ST_OK, n = 0, nslots = 0, nst = 1;
      if (nd > DSTACK_MAX_DNN_PER_SCEN) {
        status = DSTACK_ST_INVALID;
      } else {
        const bool mine = lane < nd;
        const uint32_t dem = mine ? a.demand[k0 + lane] : 0u;
        const bool act = dem > 0;
        const uint32_t al = mine ? a.alloc[k0 + lane] >> 16 : 0u;
        const uint32_t g = act ? (dem > al ? dem : al) : 0u;
        const uint32_t T = __reduce_max_sync(FULL, act ? (uint32_t)a.pb.slo_us[k0 + lane] : 0u);
        const uint32_t am = __ballot_sync(FULL, act);
        n = __popc(am);
        if (T == 0) status = DSTACK_ST_INFEASIBLE;
        else {
          nslots = (int32_t)(T / (uint32_t)slot);
          if (n > MT_MAX_ACT || nslots > DSTACK_MAX_SLOTS) status = DSTACK_ST_INVALID;
        }
        if (status == DSTACK_ST_OK) {
          const int rank = __popc(am & ((1u << lane) - 1u));
          if (act) { sm.g[rank] = g; }
          uint32_t rem = am;
          for (int i = 0; i < n; ++i) {   // d_j(b) at g_j for b in [b_lo, b*_j], from the rows (O1)
            const int j = __ffs(rem) - 1;
            rem &= rem - 1;
            const int64_t k = k0 + j;
            const int32_t gj = (int32_t)__shfl_sync(FULL, g, j);
            const int32_t bs = (int32_t)a.batch[k];
            const int64_t r0 = a.pb.dnn_row_off[k];
            const int32_t K = (int32_t)(a.pb.dnn_row_off[k + 1] - r0);
            uint64_t RT = 0, D = 0;
            for (int q = lane; q < K; q += 32) { RT += a.pb.r[r0 + q]; D += (uint64_t)a.pb.r[r0 + q] * a.pb.d[r0 + q]; }
            RT = warp_sum_u64(RT); D = warp_sum_u64(D);
            dtab_from_rows(a.pb, a.p, k, RT, D, gj, b_lo, bs, sm.dtab[i], lane);
            if (lane == 0) {
              // options: per distinct run length the largest batch (a smaller one with the same d is dominated)
              uint32_t Dmax = 0, no = 0;
              for (int b = b_lo; b <= bs; ++b) {
                const uint32_t d = sm.dtab[i][b - 1];
                if (d > Dmax) Dmax = d;
                bool merged = false;
                for (uint32_t o = 0; o < no; ++o)
                  if (sm.od[i][o] == d) { sm.ob[i][o] = (uint16_t)b; merged = true; }
                if (!merged) { sm.od[i][no] = (uint16_t)d; sm.ob[i][no] = (uint16_t)b; ++no; }
              }
              sm.D[i] = Dmax; sm.nopt[i] = no;
            }
            __syncwarp();
          }
          if (lane == 0) {
            int64_t p = 1;
            for (int i = 0; i < n; ++i) {
              sm.radix[i] = (uint32_t)p;
              if ((int64_t)sm.D[i] + 1 > MT_MAX_STATES) { p = MT_MAX_STATES + 1; break; }
              p *= (int64_t)sm.D[i] + 1;
              if (p > MT_MAX_STATES) break;
            }
            if (p > MT_MAX_STATES) status = DSTACK_ST_INVALID;
            nst = (int32_t)(p > MT_MAX_STATES ? 1 : p);
          }
          status = __shfl_sync(FULL, status, 0);
          nst = __shfl_sync(FULL, nst, 0);
        }
      }
      if (lane == 0) { sm.status = status; sm.n = n; sm.nslots = nslots; sm.nst = nst; }
    }
    __syncthreads();
    const int32_t status = sm.status, n = sm.n, nslots = sm.nslots, nst = sm.nst;
    uint32_t result = 0;
    if (status == DSTACK_ST_OK) {
      for (int st = tid; st < nst; st += MT_THREADS) sm.V[0][st] = 0u;   // V_nslots = 0
      __syncthreads();
      int cur = 0;
      for (int32_t t = nslots - 1; t >= 0; --t) {
        const uint32_t *Vn = sm.V[cur];
        uint32_t *Vt = sm.V[cur ^ 1];
        for (int st = tid; st < nst; st += MT_THREADS) {
          uint32_t r[MT_MAX_ACT];
          uint32_t occ0 = 0, nx0 = 0, idle = 0;
#pragma unroll
          for (int i = 0; i < MT_MAX_ACT; ++i) {
            r[i] = 0;
            if (i < n) {
              r[i] = ((uint32_t)st / sm.radix[i]) % (sm.D[i] + 1);
              if (r[i] > 0) { occ0 += sm.g[i]; nx0 += (r[i] - 1) * sm.radix[i]; }
              else idle |= 1u << i;
            }
          }
          int64_t best = -1;
          if (occ0 <= (uint32_t)L) {
            // odometer over the idle models' choices (0 = no start, o + 1 = option o)
            uint32_t c[MT_MAX_ACT];
#pragma unroll
            for (int i = 0; i < MT_MAX_ACT; ++i) c[i] = 0;
            while (true) {
              uint32_t occ = occ0, nx = nx0, gain = 0;
              bool ok = true;
#pragma unroll
              for (int i = 0; i < MT_MAX_ACT; ++i) {
                if (c[i]) {
                  const uint32_t d = sm.od[i][c[i] - 1];
                  if (d < 1 || t + (int32_t)d > nslots) ok = false;
                  occ += sm.g[i]; nx += (d - 1) * sm.radix[i]; gain += sm.ob[i][c[i] - 1];
                }
              }
              if (ok && occ <= (uint32_t)L) {
                const int64_t v = (int64_t)gain + Vn[nx];
                if (v > best) best = v;
              }
              int i = 0;
              for (; i < n; ++i) {
                if (!((idle >> i) & 1u)) continue;
                if (c[i] < sm.nopt[i]) { ++c[i]; break; }
                c[i] = 0;
              }
              if (i == n) break;
            }
          }
          Vt[st] = best < 0 ? 0u : (uint32_t)best;   // unreachable states (running levels > L) hold 0
        }
        __syncthreads();
        cur ^= 1;
      }
      result = sm.V[cur][0];
    }
    if (tid == 0) {
      if (a.served) a.served[s] = result;
      if (a.st) a.st[s] = (uint8_t)status;
    }
    __syncthreads();
  }
}

int launch_maxthr(const MtArgs &a, cudaStream_t s, int *launches) {
  if (a.pb.num_scen <= 0) return 0;
  if (cudaMemsetAsync(a.work_ctr, 0, sizeof(uint32_t), s) != cudaSuccess) return DSTACK_ELAUNCH;
  const size_t smem = sizeof(MtShared);
  if (cudaFuncSetAttribute(k_maxthr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return DSTACK_ELAUNCH;
  const int64_t blocks = resident_wave(k_maxthr, MT_THREADS, smem, a.pb.num_scen);
  k_maxthr<<<(unsigned)blocks, MT_THREADS, smem, s>>>(a);
  ++*launches;
  return cudaGetLastError() == cudaSuccess ? 0 : DSTACK_ELAUNCH;
}

}  // namespace dstack
