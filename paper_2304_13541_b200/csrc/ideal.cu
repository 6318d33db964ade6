// ideal.cu -- a6: the ideal per-kernel-GPU% scheduler (§6.2, Eqs. 13-14).
//
// k_ideal_rows (warp per DNN, lane per kernel row): execution demand g_e = Eq. 6 knee of the one-row
// DNN {n_i, R = 1, d_i} at b*_j ("we computed the knee of each kernel") and duration
// tau_e = ceil(f_e(g_e)) us.  Per lane the one-row latency has only two regimes (S < N_i and
// S >= N_i), so the knee scan is a register loop over the L levels with the same exact comparison
// as the batch search.
//
// k_ideal_sim (warp per scenario, lane per DNN): event-driven preemptive schedule.  Each active DNN runs
// batches of b* back-to-back; at every event the eligible set is each DNN's current kernel execution
// (chain constraint of Eq. 14); the subset maximising sum g <= L (Eq. 13's per-slot maximisation, slot -> 0
// limit) is found with a 256-bit subset-sum DP over the items in priority order (batch deadline, index),
// and the lexicographically-first optimal subset is read back from the suffix reachability sets.
// Selected executions progress to the first completion.
#include "kernels.cuh"

namespace dstack {



#ifndef DSTACK_IDEAL_ROW_CANDIDATES
#define DSTACK_IDEAL_ROW_CANDIDATES 1   // per-row knee from each regime's ends and real maximum (0: scan every level)
#endif

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
      auto consider = [&](int32_t l) {   // exact; ties -> the smaller level (the brute-force scan's rule)
        if (l < 1 || l > L) return;
        const uint64_t S = (uint64_t)s_of(l, S_tot, L);
        l = (int32_t)(((S - 1) * (uint64_t)L) / (uint64_t)S_tot) + 1;   // the smallest level granting these S SMs
        uint64_t X = wC * S + (N >= 1 ? M * t_p * (N > S ? N : S) : 0ull);
        if (mem_mode == 1) X += b * dd;
        else if (mem_mode == 2) X += b * dd * S * S;
        const int c = bestl == 0 ? 1 : cmp_score((uint32_t)S, X, (float)X, bestS, bestX, (float)bestX);
        if (c > 0 || (c == 0 && (uint32_t)l < bestl)) { bestS = (uint32_t)S; bestl = (uint32_t)l; bestX = X; }
      };
#if DSTACK_IDEAL_ROW_CANDIDATES
      // One row has two latency regimes, S < N (X = a S^2 + (wC) S + M t_p N + m) and S >= N (X = a S^2 +
      // (wC + M t_p) S + m); on each, g = S / X^2 is unimodal in S with its real maximum at the positive root of
      // -3a S^2 - beta S + gamma = 0.  The exact argmax over the levels is therefore among each regime's ends and
      // the levels adjacent to that maximum (checked with a +-2 margin).
      const int64_t lmax_lt_N = N >= 1 ? (int64_t)((N - 1 < (uint64_t)S_tot ? N - 1 : (uint64_t)S_tot) * (uint64_t)L / (uint64_t)S_tot) : 0;
      const double vb = mem_mode == 2 ? (double)(b * dd) : 0.0, m1 = mem_mode == 1 ? (double)(b * dd) : 0.0;
      for (int seg = 0; seg < 2; ++seg) {
        // seg 0: S < N (levels 1..lmax_lt_N); seg 1: S >= N (levels lmax_lt_N+1..L)
        const int64_t l0 = seg == 0 ? 1 : lmax_lt_N + 1, l1 = seg == 0 ? lmax_lt_N : L;
        if (l0 > l1) continue;
        consider((int32_t)l0);
        consider((int32_t)l1);
        const double beta = (double)wC + (seg == 1 && N >= 1 ? (double)(M * t_p) : 0.0);
        const double gamma = m1 + (seg == 0 ? (double)(M * t_p * N) : 0.0);
        double sst;
        if (vb > 0.0) sst = (-beta + sqrt(beta * beta + 12.0 * vb * gamma)) / (6.0 * vb);
        else if (beta > 0.0) sst = gamma / beta;
        else sst = (double)S_tot;   // g increasing: the regime's end
        if (!(sst >= 0.0)) sst = 0.0;
        if (sst > (double)S_tot + 4.0) sst = (double)S_tot + 4.0;
        if (L <= S_tot) {   // levels sparse in S: the levels around S* L / S_tot
          const int64_t lc = (int64_t)floor(sst * (double)L / (double)S_tot);
          for (int64_t l = lc - 2; l <= lc + 3; ++l) if (l >= l0 && l <= l1) consider((int32_t)l);
        } else {            // every S attained: the smallest level of each S around S*
          const int64_t sc = (int64_t)floor(sst);
          for (int64_t S = sc - 2; S <= sc + 3; ++S) {
            if (S < 1 || S > S_tot) continue;
            const int64_t l = ((S - 1) * L) / S_tot + 1;   // smallest l with S(l) = S
            if (l >= l0 && l <= l1) consider((int32_t)l);
          }
        }
      }
#else
      for (int32_t l = 1; l <= L; ++l) consider(l);
#endif
      const uint64_t den = (uint64_t)bestS * M;
      const uint64_t tau = (bestX + den - 1) / den;
      // one 8-byte record per execution for k_ideal_sim: tau | g << 32 | R << 48
      a.ex_pk[i] = (tau > 0xFFFFFFFFull ? 0xFFFFFFFFull : tau) | ((uint64_t)bestl << 32) | ((uint64_t)a.pb.r[i] << 48);
    }
  }
}

// k_ideal_sim: one warp per scenario, lane j = DNN j.  Per event the subset-sum DP runs over the live
// executions in priority order with the 256 capacities distributed over the lanes (lane c holds capacities
// c, c+32, ..., c+224 as an 8-bit mask): adding an item of weight g = 32a + b is one shuffle from lane c-b and
// a shift by a (or a+1 across the wrap), so each item costs a handful of instructions.  The suffix sets stay
// in shared memory for the lexicographic read-back.  Each lane keeps its chain position in registers and
// prefetches its next row, so a completion does not wait on global memory.
constexpr int IDEAL_WARPS = 8;
#ifndef DSTACK_IDEAL_ENUM_MAX
#define DSTACK_IDEAL_ENUM_MAX 10   // live items up to which every subset is enumerated (else the DP; <= 12)
#endif
#ifndef DSTACK_IDEAL_MITM
#define DSTACK_IDEAL_MITM 1   // 11..16 live items: meet-in-the-middle enumeration instead of the DP (A/B switch)
#endif
#ifndef DSTACK_IDEAL_ORDER
#define DSTACK_IDEAL_ORDER 1   // heavy-first scenario order for k_ideal_sim (A/B switch)
#endif
#ifndef DSTACK_IDEAL_SMALL_MITM
#define DSTACK_IDEAL_SMALL_MITM 1   // 9-10 live items: 5 + 5 meet in the middle, one subset per lane (else enumeration)
#endif
#ifndef DSTACK_IDEAL_SHORTCUTS
#define DSTACK_IDEAL_SHORTCUTS 1   // all-fit shortcut: sum g <= L selects every live item (A/B switch)
#endif

// Execution runs (k_ideal_runs): the subset selection sees a chain only through its current item's demand g, so
// consecutive executions of equal g (the R repeats of a kernel, and successive kernels of the same knee) form one
// item whose duration is their sum; zero-duration rows complete instantly and are skipped.  Each run's record
// (at its first non-zero row; the chain's first run at the chain's first row) is tau | g << 32 | next << 48, next =
// rows to the following run's record (r1 - i: none); an all-zero chain has tau = 0 at its first row.  Merging
// removes exactly the events at which no item's (rank, g) changes: the selection, its sum and every item's
// progress are the same on both sides of such an event, so the schedule and util are unchanged.
__global__ void __launch_bounds__(256) k_ideal_runs(IdealArgs a) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < a.pb.num_dnn;
       k += (int64_t)gridDim.x * blockDim.x) {
    if (a.demand[k] == 0) continue;
    const int64_t r0 = a.pb.dnn_row_off[k], r1 = a.pb.dnn_row_off[k + 1];
    auto put = [&](int64_t i, uint64_t tau, uint32_t g, int64_t nx) {
      a.ex_pk[i] = (tau > 0xFFFFFFFFull ? 0xFFFFFFFFull : tau) | ((uint64_t)g << 32) | ((uint64_t)(nx - i) << 48);
    };
    int64_t nx = r1, first_nz = -1;   // the run being built backwards starts at first_nz; the following one at nx
    uint64_t acc = 0;
    uint32_t gcur = 0;
    for (int64_t i = r1 - 1; i >= r0; --i) {
      const uint64_t v = a.ex_pk[i];
      const uint64_t tz = (v & 0xFFFFFFFFull) * (v >> 48);   // tau x R (< 2^48)
      if (tz == 0) continue;
      const uint32_t g = (uint32_t)(v >> 32) & 0xFFFFu;
      if (first_nz >= 0 && g != gcur) { put(first_nz, acc, gcur, nx); nx = first_nz; acc = 0; }
      gcur = g; acc += tz; first_nz = i;
    }
    put(r0, acc, gcur, nx);   // the first run (or tau = 0: the chain never runs)
  }
}

struct IdealRow {
  int64_t i;      // row of the run's record (r1 = end of chain)
  uint32_t tau, g, nx;
};

// the run record at row i (tau = 0 past the chain's end): the prefetch of a chain's next run, whose load is only
// consumed at the next advance, so its latency overlaps the events in between
__device__ __forceinline__ IdealRow ideal_run_at(const IdealArgs &a, int64_t i, int64_t r1) {
  IdealRow w;
  w.i = i;
  w.tau = 0; w.g = 0; w.nx = 0;
  if (i < r1) {
    const uint64_t v = a.ex_pk[i];
    w.tau = (uint32_t)v; w.g = (uint32_t)(v >> 32) & 0xFFFFu; w.nx = (uint32_t)(v >> 48);
  }
  return w;
}

#ifndef DSTACK_IDEAL_MINB
#define DSTACK_IDEAL_MINB 4   // 64 registers (the meet-in-the-middle branch would take 109)
#endif
#ifndef DSTACK_IDEAL_FEW
#define DSTACK_IDEAL_FEW 32768   // below this many scenarios the 3-blocks-per-SM build (79 registers, shorter event
                                 // latency) runs: few scenarios per warp, the longest event chains set the time
                                 // (A/B: config 2 (10k) 14.7 -> 13.1 ms; config 4 (100k) 109.1 -> 114.8 ms)
#endif
template <int MINB>
__global__ void __launch_bounds__(IDEAL_WARPS * 32, MINB) k_ideal_sim(IdealArgs a) {
  __shared__ uint8_t reach_all[IDEAL_WARPS][DSTACK_MAX_DNN_PER_SCEN + 1][32];
  __shared__ __align__(16) uint8_t grank_all[IDEAL_WARPS][32];   // g of the live item of each priority rank
  __shared__ uint32_t mbb_all[IDEAL_WARPS][8];     // meet in the middle: achievable B sums (256-bit set)
  __shared__ int32_t mbl_all[IDEAL_WARPS][8];      // ... highest achievable B sum below each word
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t(*reach)[32] = reach_all[warp];
  uint8_t *grank = grank_all[warp];
  uint32_t *mb_bits = mbb_all[warp];
  int32_t *mb_below = mbl_all[warp];
  const int32_t L = a.p.L, slot = a.p.slot_us;
  uint32_t capmask = 0;   // bits k with capacity lane + 32 k <= L
  for (int k = 0; k < 8; ++k)
    if (lane + 32 * k <= L) capmask |= 1u << k;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (int64_t q = warp_next_item(a.work_ctr, -1, gwarp, nwarps, lane); q < a.pb.num_scen;
       q = warp_next_item(a.work_ctr, q, gwarp, nwarps, lane)) {
    const int64_t s = a.order ? (int64_t)a.order[q] : q;
    const int32_t k0 = a.pb.scen_dnn_off[s], nd = a.pb.scen_dnn_off[s + 1] - k0;
    double ui = 0.0, ti = 0.0;
    const bool mine = lane < nd && nd <= DSTACK_MAX_DNN_PER_SCEN;
    const int k = k0 + lane;
    const bool act = mine && a.demand[k] > 0;
    const uint32_t slo = mine ? (uint32_t)a.pb.slo_us[k] : 0u;
    uint32_t T = __reduce_max_sync(FULL, act ? slo : 0u);   // 0 when nd > DSTACK_MAX_DNN_PER_SCEN (no lane active)
    if (T > 0) {
      const uint32_t nslots = T / (uint32_t)slot;
      const uint32_t njobs = __reduce_add_sync(FULL, act ? nslots / (slo / (uint32_t)slot) : 0u);
      if (nslots > DSTACK_MAX_SLOTS || njobs > DSTACK_MAX_JOBS) T = 0;
    }
    if (T > 0) {
      int64_t r0 = 0, r1 = 0;
      IdealRow first, cur, nxt;
      first.i = cur.i = nxt.i = 0; first.nx = cur.nx = nxt.nx = 0; first.tau = cur.tau = nxt.tau = 0;
      first.g = cur.g = nxt.g = 0;
      bool live = false;
      if (act) {
        r0 = a.pb.dnn_row_off[k]; r1 = a.pb.dnn_row_off[k + 1];
        first = ideal_run_at(a, r0, r1);
        live = first.tau > 0;                 // an all-zero chain never runs
        cur = first;
        if (live) nxt = ideal_run_at(a, cur.i + cur.nx, r1);
      }
      uint32_t rem = cur.tau, dl = slo, comp = 0, rank = 0;
      const uint32_t n = (uint32_t)__popc(__ballot_sync(FULL, live));
      bool dirty = true;
      bool sel = false;
      uint32_t gsum = 0;
      uint64_t util = 0;
      uint32_t t = 0;   // < T <= 2^30 us
      uint32_t st_ev = 0, st_rs = 0, st_fit = 0, st_enum = 0, st_mitm = 0, st_dp = 0;   // a6 work counters
      while (n > 0 && t < T) {
        ++st_ev;
        if (dirty) {   // priority rank among the live DNNs: (batch deadline, index)
          const uint64_t key = ((uint64_t)dl << 5) | (uint32_t)lane;
          rank = 0;
          for (int q = 0; q < 32; ++q) {
            const uint64_t kq = shfl_u64(key, q);
            const bool lq = __shfl_sync(FULL, (int)live, q) != 0;
            if (lq && kq < key) ++rank;
          }
          dirty = false;
        }
        // Every event changes some live item's g (consecutive runs of a chain differ in g) or a rank, so the
        // selection is recomputed.  When every live item fits (sum g <= L) the unique optimum is all of them
        // (g >= 1).
        const uint32_t gtot = __reduce_add_sync(FULL, live ? cur.g : 0u);
        ++st_rs;
        if (DSTACK_IDEAL_SHORTCUTS && gtot <= (uint32_t)L) {
          ++st_fit;
          sel = live;
          gsum = gtot;
        } else if (n <= 5) {
          ++st_enum;
          // <= 32 subsets: one per lane (index bit p <-> rank n-1-p; the largest index among the max-sum subsets is
          // the lexicographically-first optimum)
          if (live) grank[rank] = (uint8_t)cur.g;
          __syncwarp();
          uint32_t sum = 0;
#pragma unroll
          for (int p = 0; p < 5; ++p)
            if (p < (int)n && ((lane >> p) & 1)) sum += grank[n - 1 - p];
          const uint32_t best = __reduce_max_sync(FULL, ((uint32_t)lane < (1u << n) && sum <= (uint32_t)L)
                                                            ? ((sum << 5) | (uint32_t)lane) : 0u);
          gsum = best >> 5;
          sel = live && (((best & 31u) >> (n - 1 - rank)) & 1u);
        } else if (DSTACK_IDEAL_SMALL_MITM && n >= 9 && n <= 10) {
          ++st_enum;
          // 9-10 live items: meet in the middle with one subset per lane on each side.  A = the nA = min(n, 5)
          // highest-priority items (A index bit p <-> rank nA-1-p), B = ranks nA..n-1 (nB <= 5; B index bit p <->
          // rank n-1-p); lane = subset index on both sides.  The lexicographically-first optimal subset has the
          // largest (A index, B index), exactly as in the 8 + 8 split below.
          if (live) grank[rank] = (uint8_t)cur.g;
          if (lane < 8) mb_bits[lane] = 0u;
          __syncwarp();
          const uint32_t nA = n < 5u ? n : 5u, nB = n - nA;
          uint32_t sA = 0, sB = 0;
#pragma unroll
          for (int p = 0; p < 5; ++p) {
            if (p < (int)nA && ((lane >> p) & 1)) sA += grank[nA - 1 - p];
            if (p < (int)nB && ((lane >> p) & 1)) sB += grank[n - 1 - p];
          }
          const bool bvalid_lane = (uint32_t)lane < (1u << nB);
          if (bvalid_lane && sB <= (uint32_t)L) atomicOr(&mb_bits[sB >> 5], 1u << (sB & 31));
          __syncwarp();
          {   // highest achievable B sum in the words below w (the empty B subset makes sum 0 achievable)
            const uint32_t wd = lane < 8 ? mb_bits[lane] : 0u;
            const int h = wd ? 32 * lane + 31 - __clz(wd) : -1;
            int ex = __shfl_up_sync(FULL, h, 1);
            if (lane == 0) ex = -1;
#pragma unroll
            for (int dd = 1; dd < 8; dd <<= 1) {
              const int o = __shfl_up_sync(FULL, ex, dd);
              if (lane >= dd) ex = max(ex, o);
            }
            if (lane < 8) mb_below[lane] = ex;
          }
          __syncwarp();
          uint32_t keyA = 0;   // (a + max{B sum <= L - a}, A index); the empty A subset always qualifies
          if ((uint32_t)lane < (1u << nA) && sA <= (uint32_t)L) {
            const uint32_t c = (uint32_t)L - sA, w = c >> 5;
            const uint32_t m = mb_bits[w] & (0xFFFFFFFFu >> (31u - (c & 31u)));
            const uint32_t mbs = m ? 32u * w + 31u - __clz(m) : (uint32_t)mb_below[w];
            keyA = ((sA + mbs) << 5) | (uint32_t)lane;
          }
          const uint32_t bestA = __reduce_max_sync(FULL, keyA);
          const uint32_t best = bestA >> 5, ia = bestA & 31u;
          const uint32_t tb = best - __shfl_sync(FULL, sA, (int)ia);
          const uint32_t ib = __reduce_max_sync(FULL, (bvalid_lane && sB == tb) ? (uint32_t)lane + 1u : 0u) - 1u;
          gsum = best;
          sel = live && (rank < nA ? ((ia >> (nA - 1 - rank)) & 1u) : ((ib >> (n - 1 - rank)) & 1u));
        } else if (n <= DSTACK_IDEAL_ENUM_MAX) {
          ++st_enum;
          sel = false;
          gsum = 0;
          // <= 1024 subsets: enumerate them all (8 per lane per round, 2^(n-8) rounds).  Subset index bit p <->
          // the item of rank n-1-p, so the largest index among the max-sum subsets is the lexicographically-
          // first (priority order) optimal subset -- the one the read-back below selects -- and one
          // max-reduction over (sum, index) decides.
          // grank reversed here: gp[p] = grank[p] (subset bit p <-> rank n-1-p); entries >= n are stale, but only
          // subsets of the first 2^n indices are ever kept
          if (live) grank[n - 1 - rank] = (uint8_t)cur.g;
          __syncwarp();
          constexpr int NE = DSTACK_IDEAL_ENUM_MAX > 8 ? DSTACK_IDEAL_ENUM_MAX : 8;   // items enumerable
          const uint32_t *gw = reinterpret_cast<const uint32_t *>(grank);
          uint32_t gp[NE];
#pragma unroll
          for (int p = 0; p < NE; ++p) gp[p] = (gw[p >> 2] >> (8 * (p & 3))) & 0xFFu;
          // key = (sum << NE) | index, built as (subset sum of bits 3..7 << NE | lane << 3) + (the low 3 bits' sum
          // << NE | lo): the fields never carry into each other, and sum <= L <=> key <= lim
          uint32_t lbase = 0;
#pragma unroll
          for (int p = 3; p < 8; ++p)
            if ((lane >> (p - 3)) & 1) lbase += gp[p];
          const uint32_t k1 = (gp[0] << NE) | 1u, k2 = (gp[1] << NE) | 2u, k4 = (gp[2] << NE) | 4u;
          const uint32_t kB[8] = {0u, k1, k2, k1 + k2, k4, k1 + k4, k2 + k4, k1 + k2 + k4};
          const uint32_t lim = (((uint32_t)L + 1u) << NE) - 1u;
          const uint32_t nsub = 1u << n;
          uint32_t best = 0;
          auto scan8 = [&](uint32_t base, uint32_t r) {
            const uint32_t kb = (base << NE) | (r << 8) | ((uint32_t)lane << 3);
            const uint32_t lm = (r << 8) + ((uint32_t)lane << 3) < nsub ? lim : 0u;   // this lane's indices exist
#pragma unroll
            for (int lo = 0; lo < 8; ++lo) {
              const uint32_t key = kb + kB[lo];
              if (key <= lm) best = max(best, key);
            }
          };
          if (n <= 8) {
            scan8(lbase, 0u);
          } else {
            for (uint32_t r = 0; r < (1u << (n - 8)); ++r) {
              uint32_t rb = lbase;
#pragma unroll
              for (int p = 8; p < NE; ++p)
                if ((r >> (p - 8)) & 1u) rb += gp[p];
              scan8(rb, r);
            }
          }
          best = __reduce_max_sync(FULL, best);   // the empty subset (key 0) is always feasible
          gsum = best >> NE;
          sel = live && ((best >> (n - 1 - rank)) & 1u);
        } else if (DSTACK_IDEAL_MITM && n <= 16) {
          ++st_mitm;
          // meet in the middle: A = ranks 0..7 (A index bit p <-> rank 7 - p), B = ranks 8..n-1 (B index bit p <->
          // rank n - 1 - p), 256 subsets each, 8 per lane.  The lexicographically-first optimal subset has the
          // largest (A index, B index): first the largest A index among the A subsets that complete to the
          // optimum (a + max{B sum <= L - a} maximal), then the largest B index whose sum completes it exactly.
          if (live) grank[rank] = (uint8_t)cur.g;
          if (lane < 8) mb_bits[lane] = 0u;
          __syncwarp();
          const uint32_t nB = n - 8;
          uint32_t gA[8], gB[8];
#pragma unroll
          for (int p = 0; p < 8; ++p) { gA[p] = grank[7 - p]; gB[p] = p < (int)nB ? grank[n - 1 - p] : 0u; }
          uint32_t baseA = 0, baseB = 0;
#pragma unroll
          for (int p = 3; p < 8; ++p)
            if ((lane >> (p - 3)) & 1) { baseA += gA[p]; baseB += gB[p]; }
          const bool bvalid_lane = ((uint32_t)lane << 3) < (1u << nB);
          uint32_t sA[8], sB[8];
#pragma unroll
          for (int lo = 0; lo < 8; ++lo) {
            sA[lo] = baseA + ((lo & 1) ? gA[0] : 0u) + ((lo & 2) ? gA[1] : 0u) + ((lo & 4) ? gA[2] : 0u);
            sB[lo] = baseB + ((lo & 1) ? gB[0] : 0u) + ((lo & 2) ? gB[1] : 0u) + ((lo & 4) ? gB[2] : 0u);
            if (bvalid_lane && sB[lo] <= (uint32_t)L) atomicOr(&mb_bits[sB[lo] >> 5], 1u << (sB[lo] & 31));
          }
          __syncwarp();
          // highest achievable B sum in the words below w (the empty B subset makes sum 0 always achievable):
          // an exclusive max-scan over the 8 words' highest set bits (lanes 0..7)
          {
            const uint32_t wd = lane < 8 ? mb_bits[lane] : 0u;
            int h = wd ? 32 * lane + 31 - __clz(wd) : -1;
            int ex = __shfl_up_sync(FULL, h, 1);
            if (lane == 0) ex = -1;
#pragma unroll
            for (int dd = 1; dd < 8; dd <<= 1) {
              const int o = __shfl_up_sync(FULL, ex, dd);
              if (lane >= dd) ex = max(ex, o);
            }
            if (lane < 8) mb_below[lane] = ex;
          }
          __syncwarp();
          uint32_t bestA = 0;
#pragma unroll
          for (int lo = 0; lo < 8; ++lo) {
            if (sA[lo] > (uint32_t)L) continue;
            const uint32_t c = (uint32_t)L - sA[lo], w = c >> 5;
            const uint32_t m = mb_bits[w] & (0xFFFFFFFFu >> (31u - (c & 31u)));
            const uint32_t mbs = m ? 32u * w + 31u - __clz(m) : (uint32_t)mb_below[w];
            const uint32_t key = ((sA[lo] + mbs) << 8) | ((uint32_t)lane << 3) | (uint32_t)lo;
            if (key > bestA) bestA = key;
          }
          bestA = __reduce_max_sync(FULL, bestA);   // the empty A subset always qualifies
          const uint32_t best = bestA >> 8, ia = bestA & 255u;
          uint32_t sa = 0;
#pragma unroll
          for (int p = 0; p < 8; ++p) if ((ia >> p) & 1u) sa += gA[p];
          const uint32_t tb = best - sa;
          uint32_t kb = 0;
#pragma unroll
          for (int lo = 0; lo < 8; ++lo)
            if (bvalid_lane && sB[lo] == tb) kb = ((uint32_t)lane << 3) + (uint32_t)lo + 1u;   // ascending lo
          const uint32_t ib = __reduce_max_sync(FULL, kb) - 1u;
          gsum = best;
          sel = live && (rank < 8 ? ((ia >> (7 - rank)) & 1u) : ((ib >> (n - 1 - rank)) & 1u));
        } else {
          ++st_dp;
          sel = false;
          gsum = 0;
          // suffix reachability: reach[q] = subset sums of the items of rank >= q; the items' weights by rank
          // come from shared memory (grank), so both passes are warp-uniform loops without owner look-ups
          if (live) grank[rank] = (uint8_t)cur.g;
          __syncwarp();
          uint32_t m = lane == 0 ? 1u : 0u;
          reach[n][lane] = (uint8_t)m;
          for (int q = (int)n - 1; q >= 0; --q) {
            const uint32_t gq = grank[q];
            const uint32_t sa = gq >> 5, sb = gq & 31u;
            const uint32_t v = __shfl_sync(FULL, m, (lane - (int)sb) & 31);
            m |= (v << ((uint32_t)lane >= sb ? sa : sa + 1u)) & 0xFFu;
            reach[q][lane] = (uint8_t)m;
          }
          // largest achievable sum <= L
          const uint32_t mm = m & capmask;
          const uint32_t top = mm ? (uint32_t)lane + 32u * (31u - __clz(mm)) + 1u : 0u;
          int target = (int)__reduce_max_sync(FULL, top) - 1;
          gsum = (uint64_t)(target > 0 ? target : 0);
          __syncwarp();
          // lexicographic read-back in priority order: include an item iff the rest can still complete target
          uint32_t selmask = 0;
          for (uint32_t q = 0; q < n; ++q) {
            const int gq = (int)grank[q];
            const int c = target - gq;
            if (c >= 0 && ((reach[q + 1][c & 31] >> (c >> 5)) & 1u)) {
              selmask |= 1u << q;
              target = c;
            }
          }
          sel = live && ((selmask >> rank) & 1u);
        }
        uint32_t dt = __reduce_min_sync(FULL, sel ? rem : 0xFFFFFFFFu);
        if (!__any_sync(FULL, sel) || dt == 0) break;
        if (dt > T - t) dt = T - t;
        util += (uint64_t)gsum * dt;
        t += dt;
        bool done_batch = false;
        if (sel) {
          rem -= dt;
          if (rem == 0) {   // next run of the chain
            if (nxt.i >= r1) {              // batch complete: next batch back-to-back
              comp++;
              dl = (uint32_t)t + slo;
              done_batch = true;
              cur = first;
            } else {
              cur = nxt;
            }
            nxt = ideal_run_at(a, cur.i + cur.nx, r1);
            rem = cur.tau;
          }
        }
        dirty = __any_sync(FULL, done_batch);
        __syncwarp();
      }
      if (a.stats && lane == 0) {
        atomicAdd(&a.stats[0], (unsigned long long)st_ev); atomicAdd(&a.stats[1], (unsigned long long)st_rs);
        atomicAdd(&a.stats[2], (unsigned long long)st_fit); atomicAdd(&a.stats[3], (unsigned long long)st_enum);
        atomicAdd(&a.stats[4], (unsigned long long)st_mitm); atomicAdd(&a.stats[5], (unsigned long long)st_dp);
        atomicAdd(&a.stats[6], 1ull);
      }
      const uint64_t bsum = warp_sum_u64(act ? (uint64_t)comp * a.batch[k] : 0ull);
      ui = (double)util / ((double)L * (double)T);
      ti = (double)bsum * 1e6 / (double)T;
    }
    if (lane == 0) {
      if (a.u_ideal) a.u_ideal[s] = ui;
      if (a.thr_ideal) a.thr_ideal[s] = ti;
    }
    __syncwarp();
  }
}

// a6 work counters of the last launch (events, re-selections, all-fit / enumeration / meet-in-the-middle / DP
// selections, scenarios simulated): 8 u64 at the end of the ideal workspace region
size_t ideal_stats_offset(int64_t num_rows, int64_t num_scen) {
  return (((size_t)(num_rows + 8) * 8 + 255) & ~(size_t)255) + (((size_t)(num_scen + 8) * 4 + 255) & ~(size_t)255) +
         48 * 4;
}

size_t ideal_ws_bytes(int64_t num_rows, int64_t num_scen) {
  size_t pk = ((size_t)(num_rows + 8) * 8 + 255) & ~(size_t)255;
  size_t o = ((size_t)(num_scen + 8) * 4 + 255) & ~(size_t)255;
  return pk + o + 256;
}

// Heavy-first scenario order for k_ideal_sim: its cost is the number of events, roughly sum over active DNNs of
// (executions per batch) x (batches per session) ~ sum_j rows_j * T / (run time of b*_j).  Scenarios are bucketed by
// floor(log2(estimate)) and listed heaviest bucket first (order inside a bucket arbitrary: the schedule, not the
// results, depends on it), so the longest event chains start first and the kernel's tail shrinks.
constexpr int IDEAL_BUCKETS = 40;
__device__ __forceinline__ uint32_t ideal_cost_bucket(const IdealArgs &a, int64_t s) {
  const int32_t k0 = a.pb.scen_dnn_off[s], k1 = a.pb.scen_dnn_off[s + 1];
  if (k1 - k0 > DSTACK_MAX_DNN_PER_SCEN) return 0;
  uint32_t T = 0;
  for (int32_t k = k0; k < k1; ++k)
    if (a.demand[k] > 0 && (uint32_t)a.pb.slo_us[k] > T) T = (uint32_t)a.pb.slo_us[k];
  double est = 0.0;
  for (int32_t k = k0; k < k1; ++k) {
    if (a.demand[k] == 0) continue;
    const double rows = (double)(a.pb.dnn_row_off[k + 1] - a.pb.dnn_row_off[k]);
    double d = 1.0;
    if (a.dstar) {
      const uint32_t v = a.batch[k] ? a.dstar[k] : 0u;
      d = v ? (double)v * (double)a.p.slot_us : 1.0;
    }
    est += rows * (double)T / d;
  }
  int e = 0;
  frexp(est + 1.0, &e);
  return (uint32_t)(e < 0 ? 0 : (e >= IDEAL_BUCKETS ? IDEAL_BUCKETS - 1 : e));
}

__global__ void __launch_bounds__(256) k_ideal_order_count(IdealArgs a) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < a.pb.num_scen; s += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&a.bucket_cnt[ideal_cost_bucket(a, s)], 1u);
}
__global__ void k_ideal_order_scan(IdealArgs a) {   // one thread: heaviest bucket first
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    uint32_t off = 0;
    for (int b = IDEAL_BUCKETS - 1; b >= 0; --b) { const uint32_t c = a.bucket_cnt[b]; a.bucket_cnt[b] = off; off += c; }
  }
}
__global__ void __launch_bounds__(256) k_ideal_order_scatter(IdealArgs a) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < a.pb.num_scen; s += (int64_t)gridDim.x * blockDim.x)
    a.order[atomicAdd(&a.bucket_cnt[ideal_cost_bucket(a, s)], 1u)] = (uint32_t)s;
}

int launch_ideal(IdealArgs a, void *ws, cudaStream_t s, int *launches) {
  if (a.pb.num_scen <= 0) return 0;
  const int64_t num_rows = a.pb.num_rows;
  a.ex_pk = (uint64_t *)ws;
  a.order = (uint32_t *)((char *)ws + (((size_t)(num_rows + 8) * 8 + 255) & ~(size_t)255));
  a.bucket_cnt = (uint32_t *)((char *)a.order + (((size_t)(a.pb.num_scen + 8) * 4 + 255) & ~(size_t)255));
  a.stats = (unsigned long long *)(a.bucket_cnt + 48);   // 8 u64 behind the 40 bucket counters (256 B slot)
  if (cudaMemsetAsync(a.stats, 0, 8 * sizeof(unsigned long long), s) != cudaSuccess) return DSTACK_ELAUNCH;
  if (a.pb.num_dnn > 0) {
    int64_t blocks = ((int64_t)a.pb.num_dnn * 32 + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_ideal_rows<<<(unsigned)blocks, 256, 0, s>>>(a);
    int64_t rb = (a.pb.num_dnn + 255) / 256;
    if (rb > (int64_t)num_sms() * 8) rb = (int64_t)num_sms() * 8;
    k_ideal_runs<<<(unsigned)rb, 256, 0, s>>>(a);
    *launches += 2;
  }
  int64_t blocks = (a.pb.num_scen + IDEAL_WARPS - 1) / IDEAL_WARPS;
  if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
  const bool few = a.pb.num_scen < DSTACK_IDEAL_FEW;
  if (!DSTACK_DYN_SCEN) a.work_ctr = nullptr;
  if (a.work_ctr) {   // one resident wave pulling scenarios (their event counts differ by orders of magnitude)
    if (cudaMemsetAsync(a.work_ctr, 0, sizeof(uint32_t), s) != cudaSuccess) return DSTACK_ELAUNCH;
    blocks = few ? resident_wave(k_ideal_sim<3>, IDEAL_WARPS * 32, 0, blocks)
                 : resident_wave(k_ideal_sim<DSTACK_IDEAL_MINB>, IDEAL_WARPS * 32, 0, blocks);
    if (DSTACK_IDEAL_ORDER) {   // heaviest estimated scenarios first
      if (cudaMemsetAsync(a.bucket_cnt, 0, sizeof(uint32_t) * IDEAL_BUCKETS, s) != cudaSuccess) return DSTACK_ELAUNCH;
      int64_t ob = (a.pb.num_scen + 255) / 256;
      if (ob > (int64_t)num_sms() * 8) ob = (int64_t)num_sms() * 8;
      k_ideal_order_count<<<(unsigned)ob, 256, 0, s>>>(a);
      k_ideal_order_scan<<<1, 32, 0, s>>>(a);
      k_ideal_order_scatter<<<(unsigned)ob, 256, 0, s>>>(a);
      *launches += 3;
    } else {
      a.order = nullptr;
    }
  } else {
    a.order = nullptr;
  }
  if (few) k_ideal_sim<3><<<(unsigned)blocks, IDEAL_WARPS * 32, 0, s>>>(a);
  else k_ideal_sim<DSTACK_IDEAL_MINB><<<(unsigned)blocks, IDEAL_WARPS * 32, 0, s>>>(a);
  ++*launches;
  return cudaGetLastError() == cudaSuccess ? 0 : DSTACK_ELAUNCH;
}

}  // namespace dstack
