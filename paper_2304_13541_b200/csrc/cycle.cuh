// cycle.cuh -- a4 (WMAX-MIN) and a5 (one D-STACK session) device code, one warp per scenario.
//
// a4, Algorithm WMAX-MIN: lane j holds DNN j's demand; the ascending (demand, index) order of
// "Fulfill Lowest Demand First" becomes a per-lane exclusive sum of the demands ranked before it, so
// grant_j = min(k_j, max(0, L - sum_before)); the surplus split is Q16.16, floored.
//
// a5, Alg. 1 / Alg. 3 / Dynamic-schedule (§6.1): the session of
// nslots = T/Delta slots is a shared-memory u8 occupancy array (levels <= 255), read as packed u32 words of 4 slots
// (one word per lane: a 128-slot window per warp instruction).  Static jobs come in EDF order from one warp
// min-reduction over a packed (deadline, d(b*), lane) key; Start-Early searches one window per step
// (find_early_win), Start-Late jumps over the first blocking slot of the candidate run (find_late_packed).  The
// opportunistic fill visits the decision times {0} u {run ends} (the next one is a min-reduction over the lanes' first
// run end after t), tests every DNN's eligibility in parallel (lane = DNN; including a necessary fit test of its
// shortest run) and serves the eligible ones in (runs so far, index) order by repeated min-reductions.
#pragma once
#include "common.cuh"
#include "prof.cuh"

namespace dstack {

#ifndef DSTACK_PROF_STATS
#define DSTACK_PROF_STATS 0
#endif
#if DSTACK_PROF_STATS
static __device__ unsigned long long g_cstats[16];   // per TU (instrumentation builds only)
#define CSTAT(i, v) atomicAdd(&g_cstats[i], (unsigned long long)(v))
#else
#define CSTAT(i, v) ((void)0)
#endif


#ifndef DSTACK_CYC_PACKED_MAX
#define DSTACK_CYC_PACKED_MAX 124   // static runs up to this length use the packed-word searches (A/B switch; <= 124;
                                    // 0 -> 32-slot ballot chunks: k_cycle 11.87 -> 12.59 ms at config 3)
#endif

#ifndef DSTACK_CYC_EARLY_WIN
#define DSTACK_CYC_EARLY_WIN 1   // 1: static Start-Early searches one 128-slot window per step (find_early_win)
#endif
#ifndef DSTACK_CYC_PRE_PTS
#define DSTACK_CYC_PRE_PTS 1   // slots of the shortest run tested lane-parallel before the serial fill loop (1, 2 or 4)
#endif

constexpr uint16_t NONE16 = 0xFFFF;
constexpr uint32_t NONE32 = 0xFFFFFFFFu;

// F1 below-knee fallback context (DSTACK_FLAG_BELOW_KNEE): where the scenario's DNN
// rows live, so that a static job that found no start at g_j can re-derive its run length at a lower level
// from O1 (32 levels per serial row pass, lanes over levels), plus the launch latency in slots.
struct BelowKnee {
  const dstack_problem_t *pb;
  const dstack_params_t *p;
  int64_t k0;              // first DNN of the scenario
  const uint32_t *ws_RT;   // per-DNN sum R and sum R d from k_prof (NULL: recomputed from the rows)
  const uint64_t *ws_D;
  uint64_t c_slots;        // ceil(reconf_us / Delta)
};


// one warp's session buffers: SLOTS >= nslots and JOBS >= the session's static jobs
template <int SLOTS, int JOBS>
struct CycSmemT {
  uint8_t occ[SLOTS + 128];   // + one register window of padding (never read as session slots)
  uint32_t sr[JOBS];          // static job (j, r): start | run slots << 16, or NONE32 (miss)
};
using CycSmem = CycSmemT<DSTACK_MAX_SLOTS, DSTACK_MAX_JOBS>;

// bytes of a lane's 4-slot word (first slot `base`) below slot x
__device__ __forceinline__ uint32_t bytes_below(int x, int base) {
  const int hb = min(x - base, 4);   // hb <= 0: shift >= 32, which the funnel shift clamps to 32 (no bytes)
  return __funnelshift_rc(0xFFFFFFFFu, 0u, (uint32_t)(32 - 8 * hb));
}

// dtab layout: one row of DSTACK_MAX_BATCH u16 per DNN of the scenario, entry b-1 = d_j(b) slots

__device__ __forceinline__ uint32_t wmaxmin_lane(uint32_t dem, int lane, int nd, int32_t L) {
  const uint32_t key = (dem << 5) | (uint32_t)lane;   // dem == 0 for lanes >= nd
  uint32_t before = 0;
#pragma unroll 4
  for (int q = 0; q < nd; ++q) {   // nd <= 32, warp-uniform
    const uint32_t kq = __shfl_sync(FULL, key, q);
    if (kq < key) before += kq >> 5;
  }
  const uint32_t tot = __reduce_add_sync(FULL, dem);
  const int64_t rem_before = (int64_t)L - (int64_t)before;
  const uint32_t grant = rem_before <= 0 ? 0u : (uint32_t)((int64_t)dem < rem_before ? (int64_t)dem : rem_before);
  const uint64_t rem = tot >= (uint32_t)L ? 0ull : (uint64_t)(L - (int32_t)tot);
  uint64_t share = 0;
  if (tot > 0) share = (((uint64_t)dem * rem) << 16) / tot;
  return (uint32_t)(((uint64_t)grant << 16) + share);
}

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

// byte mask of slots [lo, hi) of a 4-slot word starting at slot `base` (lo/hi are clamped to [0, 4])
__device__ __forceinline__ uint32_t bytes_mask(int s, int e, int base);

// Packed-word searches for runs of d <= 124 slots (the run [s, s+d) lies in the 128 slots from s & ~3, one u32
// word of 4 slots per lane): jump over the blocking slot nearest to the far end of the candidate run.
// Start-Early: smallest feasible s in [rel, dl-d]; -1 if none.
__device__ __forceinline__ int find_early_packed(const uint8_t *occ, int rel, int dl, int d, int g, int L, int lane) {
  const uint32_t *w32 = reinterpret_cast<const uint32_t *>(occ);
  const uint32_t th = (uint32_t)(L - g) * 0x01010101u;
  int s = rel;
  while (s + d <= dl) {
    const int bt = s & ~3, wi = (bt >> 2) + lane, mybase = bt + 4 * lane;
    const uint32_t word = w32[wi];   // padded array
    // blocking slots of [s & ~3, s + d): the last one + 1 is <= s iff none lies in the run [s, s + d)
    const uint32_t bb = __vcmpgtu4(word, th) & bytes_below(s + d, mybase);
    const uint32_t lb = bb ? (uint32_t)(mybase + ((31 - __clz(bb)) >> 3) + 1) : 0u;
    const uint32_t last = __reduce_max_sync(FULL, lb);   // (last blocking slot) + 1, or 0
    if (lane == 0) CSTAT(9, 1);
    if ((int)last <= s) return s;
    s = (int)last;
  }
  return -1;
}
// Start-Early over 128-slot windows for 4 <= d <= 124: the smallest feasible start s* >= s is s itself or x + 1 for a
// blocking slot x (s* - 1 >= s infeasible while [s*, s* + d) is free forces s* - 1 to block).  With d >= 4 only
// the last blocking slot of a lane's 4-slot word can open a gap of d, so one window costs a min-reduction for s,
// then per lane that slot, the next blocking slot after its word (ballot + one shuffle), and a min-reduction over
// the starts whose gap is known to reach d.  Otherwise the next window starts after the window's last blocking
// slot (every start before it is infeasible).  Slots >= dl may hold stale bytes: every accepted start has s + d <= dl,
// and a stale blocking slot >= dl only caps a gap at >= dl.
__device__ __forceinline__ int find_early_win(const uint8_t *occ, int rel, int dl, int d, int g, int L, int lane) {
  const uint32_t *w32 = reinterpret_cast<const uint32_t *>(occ);
  const uint32_t th = (uint32_t)(L - g) * 0x01010101u;
  int s = rel;
  while (s + d <= dl) {
    const int bt = s & ~3, mybase = bt + 4 * lane;
    const uint32_t word = w32[(bt >> 2) + lane];   // padded array
    const uint32_t bb = __vcmpgtu4(word, th) & ~bytes_below(s, mybase);   // blocking slots >= s
    const uint32_t fbl = bb ? (uint32_t)(mybase + ((__ffs(bb) - 1) >> 3)) : 0xFFFFFFFFu;
    const uint32_t first = __reduce_min_sync(FULL, fbl);
    if (lane == 0) CSTAT(9, 1);
    if (first >= (uint32_t)(s + d)) return s;   // none in the window: the gap is >= 125 > d
    const uint32_t later = __ballot_sync(FULL, bb != 0u) & ~((2u << lane) - 1u);   // lanes above with a blocking slot
    const uint32_t nbx = __shfl_sync(FULL, fbl, later ? __ffs(later) - 1 : 0);
    const int c = bb ? mybase + ((31 - __clz(bb)) >> 3) + 1 : 0;   // after this word's last blocking slot
    const bool feas = bb != 0u && c + d <= dl && (later ? (int)nbx >= c + d : c + d <= bt + 128);
    const uint32_t best = __reduce_min_sync(FULL, feas ? (uint32_t)c : 0xFFFFFFFFu);
    if (best != 0xFFFFFFFFu) return (int)best;
    s = (int)__reduce_max_sync(FULL, (uint32_t)c);
  }
  return -1;
}

// Start-Late: largest feasible s in [rel, dl-d]; -1 if none.
__device__ __forceinline__ int find_late_packed(const uint8_t *occ, int rel, int dl, int d, int g, int L, int lane) {
  const uint32_t *w32 = reinterpret_cast<const uint32_t *>(occ);
  const uint32_t th = (uint32_t)(L - g) * 0x01010101u;
  int s = dl - d;
  while (s >= rel) {
    const int bt = s & ~3, wi = (bt >> 2) + lane, mybase = bt + 4 * lane;
    const uint32_t word = w32[wi];   // padded array
    uint32_t bb = __vcmpgtu4(word, th) & bytes_below(s + d, mybase);
    if (lane == 0) bb &= 0xFFFFFFFFu << (8 * (s & 3));
    const uint32_t fb = bb ? (uint32_t)(mybase + ((__ffs(bb) - 1) >> 3)) : 0xFFFFFFFFu;
    const uint32_t first = __reduce_min_sync(FULL, fb);   // first blocking slot, or none
    if (lane == 0) CSTAT(10, 1);
    if (first == 0xFFFFFFFFu) return s;
    s = (int)first - d;
  }
  return -1;
}

__device__ __forceinline__ uint32_t bytes_mask(int s, int e, int base) {
  const int lo = min(max(s - base, 0), 4), hi = min(max(e - base, 0), 4);
  return __funnelshift_lc(0u, 0xFFFFFFFFu, (uint32_t)(8 * lo)) & __funnelshift_rc(0xFFFFFFFFu, 0u, (uint32_t)(32 - 8 * hi));
}

// occ[u] += g for u in [s, s+d): 4 slots per lane per step (packed u32; callers guarantee occ + g <= L <= 255,
// so no byte carries).
__device__ __forceinline__ void occ_add(uint8_t *occ, int s, int d, int g, int lane) {
  const int e = s + d;
  uint32_t *w32 = reinterpret_cast<uint32_t *>(occ);
  const uint32_t gg = (uint32_t)g * 0x01010101u;
  for (int w0 = s >> 2; (w0 << 2) < e; w0 += 32) {
    const int w = w0 + lane, base = w << 2;
    if (base < e) {
      w32[w] += gg & bytes_mask(s, e, base);
    }
  }
  __syncwarp();
}

// first u in [t, stop) with occ[u] > thr, or stop (4 slots per lane per step)
__device__ __forceinline__ int first_above(const uint8_t *occ, int t, int stop, int thr, int lane) {
  const uint32_t *w32 = reinterpret_cast<const uint32_t *>(occ);
  const uint32_t th = (uint32_t)thr * 0x01010101u;
  for (int w0 = t >> 2; (w0 << 2) < stop; w0 += 32) {
    const int w = w0 + lane, base = w << 2;
    const uint32_t bb = base < stop ? (__vcmpgtu4(w32[w], th) & bytes_mask(t, stop, base)) : 0u;
    const uint32_t bal = __ballot_sync(FULL, bb != 0);
    if (bal) {
      const int pl = __ffs(bal) - 1;
      const uint32_t b = __shfl_sync(FULL, bb, pl);
      return ((w0 + pl) << 2) + ((__ffs(b) - 1) >> 3);
    }
  }
  return stop;
}

__device__ __forceinline__ uint32_t occ_sum(const uint8_t *occ, int nslots, int lane) {
  const uint32_t *w32 = reinterpret_cast<const uint32_t *>(occ);
  uint32_t s = 0;
  for (int w = lane; (w << 2) < nslots; w += 32) {
    const int base = w << 2;
    s += __vsadu4(w32[w] & bytes_mask(0, nslots, base), 0u);
  }
  return __reduce_add_sync(FULL, s);
}

// F1 retry of static job (j, r) over the window [rel, dlv) at levels g_j - 1 .. 1 (warp-uniform arguments): the
// first level whose run ceil(X(S(l), b*) / (S(l) M Delta)) + launch latency has a feasible start under the job's
// rule.  Returns start | d << 16 | l << 32, or 0 if no level fits.  Out of line: only misses reach it.
static __device__ __noinline__ uint64_t below_knee_retry(const uint8_t *occ, const BelowKnee &bk, int j, int rj, int rel,
                                                         int dlv, int gj, int32_t bsj, int L, int lane) {
  const int64_t kj = bk.k0 + j;
  const dstack_problem_t &bpb = *bk.pb;
  const dstack_params_t &bp = *bk.p;
  uint64_t RT, D;
  if (bk.ws_RT) { RT = bk.ws_RT[kj]; D = bk.ws_D[kj]; }
  else {
    const int64_t r0 = bpb.dnn_row_off[kj];
    const int32_t K = (int32_t)(bpb.dnn_row_off[kj + 1] - r0);
    RT = 0; D = 0;
    for (int i = lane; i < K; i += 32) { RT += bpb.r[r0 + i]; D += (uint64_t)bpb.r[r0 + i] * bpb.d[r0 + i]; }
    RT = warp_sum_u64(RT); D = warp_sum_u64(D);
  }
  const uint64_t M = bp.mem_mode == 0 ? 1ull : (uint64_t)bpb.mem_bw[kj];
  const uint32_t win = (uint32_t)(dlv - rel);   // <= DSTACK_MAX_SLOTS < 0xFFFF: a clamped d never fits
  // 32 levels at a time, lane i holding level top - i: each lane sums V(S(l)) over all the DNN's rows itself
  // (the row loads are warp-wide broadcasts), so a chunk costs one serial row pass instead of 32 warp passes
  // with their reductions; the levels are then tried top-down exactly as one at a time.
  const int64_t r0 = bpb.dnn_row_off[kj];
  const int32_t K = (int32_t)(bpb.dnn_row_off[kj + 1] - r0);
  const uint32_t *nrow = bpb.n + r0;
  const uint16_t *rrow = bpb.r + r0;
  const uint64_t t_p = (uint64_t)bpb.t_p[kj], t_np = (uint64_t)bpb.t_np[kj];
  for (int top = gj - 1; top >= 1; top -= 32) {
    const int myl = top - lane;
    uint32_t dl = 0xFFFFFFFFu;
    if (myl >= 1) {
      const uint64_t S = (uint64_t)s_of(myl, bp.S_tot, bp.L);
      uint64_t V = 0;
#pragma unroll 4
      for (int i = 0; i < K; ++i) {
        const uint64_t nn = nrow[i];
        const uint64_t N = bp.par_mode == 0 ? (uint64_t)bsj * nn : ((uint64_t)bsj * nn + 2047) >> 11;
        if (N >= 1) V += (uint64_t)rrow[i] * (N > S ? N : S);
      }
      uint64_t X = (bp.wse_mode == 0 ? (uint64_t)bsj : 1ull) * t_np * RT * S * M + M * t_p * V;
      if (bp.mem_mode == 1) X += (uint64_t)bsj * D;
      else if (bp.mem_mode == 2) X += (uint64_t)bsj * D * S * S;
      dl = (uint32_t)ceil_div_clamp16(X, S * M * (uint64_t)bp.slot_us) + (uint32_t)bk.c_slots;
    }
    uint32_t cand = __ballot_sync(FULL, myl >= 1 && dl <= win);
    while (cand) {
      const int i = __ffs(cand) - 1;
      cand &= cand - 1;
      const int l = top - i;
      const int d = (int)__shfl_sync(FULL, dl, i);
      const int s = d <= 124 ? ((rj & 1) ? find_late_packed(occ, rel, dlv, d, l, L, lane)
                                         : find_early_packed(occ, rel, dlv, d, l, L, lane))
                             : ((rj & 1) ? find_late(occ, rel, dlv, d, l, L, lane) : find_early(occ, rel, dlv, d, l, L, lane));
      if (s >= 0) return (uint64_t)s | ((uint64_t)d << 16) | ((uint64_t)l << 32);
    }
  }
  return 0;
}

struct CycRes {
  uint32_t occ_static, occ_all, served_tot, misses, below;
  bool oversub;
};

// One D-STACK session for the scenario held by this warp.  Lane j (< nd) describes DNN j:
// active, g (level), bs (b*), sl (SLO in slots), rep (= nslots / sl); dtab rows hold d_j(b).
// hook_b_only: fill may only use b* (test hook).  runs/served are per-lane in/out.
// count0: per-lane initial fill priority (config-5 scoreboard; 0 for one session).  fill_log (nullable):
// every fill run appended as pack_run(j, t, d, b) up to fill_cap entries; *fill_n counts them (may exceed cap).
__device__ __forceinline__ uint64_t pack_run(uint32_t j, uint32_t t, uint32_t d, uint32_t b) {
  return ((uint64_t)j << 56) | ((uint64_t)t << 32) | ((uint64_t)d << 8) | b;
}

template <class SM>
__device__ __forceinline__ CycRes cycle_core(SM &sm, const uint16_t *dtab, int lane, bool active, uint32_t g,
                                            uint32_t bs, uint32_t sl, uint32_t rep, int32_t nslots, int32_t L,
                                            int32_t b_lo, bool hook_b_only, uint32_t &runs, uint32_t &served,
                                            uint32_t count0 = 0, uint64_t *fill_log = nullptr, uint32_t fill_cap = 0,
                                            uint32_t *fill_n = nullptr, int fill_order = 0, uint32_t *busy = nullptr,
                                            const BelowKnee *bk = nullptr, uint32_t dstar_in = 0xFFFFFFFFu) {
  // fill_order (O9 comparison schedulers): 0 D-STACK (runs so far), 1 Max-Min fair (smallest g
  // first), 2 max-throughput (shortest d(b*) first); ties by index.  busy (nullable): this lane's run slots.
  CycRes res; res.occ_static = 0; res.occ_all = 0; res.served_tot = 0; res.misses = 0; res.below = 0; res.oversub = false;
  for (int w = lane; (w << 2) < nslots; w += 32) reinterpret_cast<uint32_t *>(sm.occ)[w] = 0u;
  __syncwarp();
  uint32_t joff = rep;   // exclusive prefix of rep over lanes
#pragma unroll
  for (int dlt = 1; dlt < 32; dlt <<= 1) {
    const uint32_t v = __shfl_up_sync(FULL, joff, dlt);
    if (lane >= dlt) joff += v;
  }
  joff -= rep;
  const uint32_t njobs = __reduce_add_sync(FULL, rep);
  // d_j(b*): given by the caller (dstar_in) or from the dtab row
  const uint32_t dstar = active ? (dstar_in != 0xFFFFFFFFu ? dstar_in : (uint32_t)dtab[lane * DSTACK_MAX_BATCH + bs - 1]) : 0u;
  uint32_t nextr = 0;
  // ---- static placement in EDF order (Alg. 1 l.5; even repeats Start-Early, odd Start-Late) ----
  for (uint32_t q = 0; q < njobs; ++q) {
    const bool has = active && nextr < rep;
    // EDF key (deadline, d(b*), index) in one word: deadline <= nslots <= 4096 (13 bits), d(b*) clamped to 8191
    // (13 bits; every d >= 8191 > nslots misses its window, so their order among themselves changes nothing)
    const uint32_t key = has ? (((nextr + 1) * sl) << 18) | (min(dstar, 8191u) << 5) | (uint32_t)lane : 0xFFFFFFFFu;
    const uint32_t mk = __reduce_min_sync(FULL, key);
    const int j = (int)(mk & 31u);
    const int rj = (int)__shfl_sync(FULL, nextr, j);
    const int slj = (int)__shfl_sync(FULL, sl, j);
    const int gj = (int)__shfl_sync(FULL, g, j);
    const int dj = (int)__shfl_sync(FULL, dstar, j);
    const int offj = (int)__shfl_sync(FULL, joff, j);
    const int rel = rj * slj, dlv = rel + slj;
    int st;
    if (dj > dlv - rel) st = -1;
    else if (dj <= DSTACK_CYC_PACKED_MAX) st = (rj & 1) ? find_late_packed(sm.occ, rel, dlv, dj, gj, L, lane)
                                      : ((DSTACK_CYC_EARLY_WIN && dj >= 4) ? find_early_win(sm.occ, rel, dlv, dj, gj, L, lane)
                                                                           : find_early_packed(sm.occ, rel, dlv, dj, gj, L, lane));
    else st = (rj & 1) ? find_late(sm.occ, rel, dlv, dj, gj, L, lane) : find_early(sm.occ, rel, dlv, dj, gj, L, lane);
    if (lane == 0) CSTAT(1, 1);
    int lv = gj, dd = dj;
    if (st < 0 && bk != nullptr) {
      const uint64_t r = below_knee_retry(sm.occ, *bk, j, rj, rel, dlv, gj, (int32_t)__shfl_sync(FULL, bs, j), L, lane);
      if (r != 0) { st = (int)(r & 0xFFFFu); dd = (int)((r >> 16) & 0xFFFFu); lv = (int)(r >> 32); res.below++; }
    }
    if (st >= 0) {
      occ_add(sm.occ, st, dd, lv, lane);
      res.occ_static += (uint32_t)dd * (uint32_t)lv;   // sum of occ over the session = sum of d g over its runs
      if (lane == 0) sm.sr[offj + rj] = (uint32_t)st | ((uint32_t)dd << 16);
      if (lane == j) { runs++; served += bs; if (busy) *busy += (uint32_t)dd; }
    } else {
      if (lane == 0) sm.sr[offj + rj] = NONE32;
      res.misses++;
      res.oversub = true;
    }
    if (lane == j) nextr++;
    __syncwarp();
  }
  uint32_t occ_fill = 0;
  // ---- opportunistic fill at decision times {0} u {run ends} (Dynamic-schedule) ----
  // Per lane (DNN): free_at = end of its current run (static or fill); [ns, ne) = its next placed static run not
  // yet begun (ns = nslots when none).  Static runs that began by t are folded into free_at, so the DNN is
  // running at t <=> t < free_at, and ns is its next own static start after t (a fill run's slice stops there).
  // A DNN's runs are disjoint, so its first run end after t is free_at when it is running, else the end of its
  // next static run: the next decision time is the minimum of these over the DNNs (run ends >= nslots are none).
  // Per decision time t the warp holds the occupancy of slots [t & ~3, (t & ~3) + 128) in registers (one packed
  // word per lane); slice queries and placements inside that window touch no shared memory except the
  // write-through of placed runs.  Longer runs fall back to the shared-memory scans.
  __syncwarp();
  uint32_t count = runs + count0;
  uint32_t nfill = 0;
  int pnext = 0, ns = nslots, ne = 0x7FFFFFFF, free_at = 0;   // ne: no next static run -> never a run end
  auto next_static = [&]() {
    ns = nslots;
    ne = 0x7FFFFFFF;
    while (pnext < (int)rep) {
      const uint32_t v = sm.sr[joff + pnext];
      ++pnext;
      if (v != NONE32) { ns = (int)(v & 0xFFFFu); ne = ns + (int)(v >> 16); break; }
    }
  };
  if (active) next_static();
  const uint32_t pk = (g & 0xFFu) | ((bs & 0xFFu) << 8) | (dstar << 16);   // dstar <= 0xFFFF (u16 rows)
  // the shortest run the fill may place for this DNN: d(b_lo) when a batch below b* is allowed, else d(b*)
  // (d nondecreasing in b)
  const int dlo = !active ? 0 : ((!hook_b_only && (int)bs - 1 >= b_lo) ? (int)dtab[lane * DSTACK_MAX_BATCH + b_lo - 1]
                                                                        : (int)dstar);
  uint32_t *w32 = reinterpret_cast<uint32_t *>(sm.occ);
  // a candidate whose slice at t is too short for d(b_lo) stays too short at every later decision time
  // t' < blk: the slot that ended its slice never loses occupancy (or it was its own next static start)
  int blk = 0;
  for (int t = 0; t < nslots;) {
    if (lane == 0) CSTAT(3, 1);
    const int bt = t & ~3, mybase = bt + 4 * lane, wi = (t >> 2) + lane;
    uint32_t wv = w32[wi];   // occ is padded by 128 slots: the window never leaves the array
    const uint32_t lo_mask = lane == 0 ? (0xFFFFFFFFu << (8 * (t & 3))) : 0xFFFFFFFFu;
    uint32_t wvm = wv & lo_mask;   // the window's slots >= t
    int occ_t = (int)sm.occ[t];    // broadcast byte load
    // static runs begun by t folded into free_at (inactive lanes: ns = nslots > t, no iteration)
    while (t >= ns) { free_at = max(free_at, ne); next_static(); }
    // eligible: not running at t (static or fill run), not blocked, fits at t
    bool elig = active && t >= max(free_at, blk) && occ_t + (int)g <= L;
    // necessary for a placement (checked lane-parallel, so that most candidates that would be rejected never enter
    // the serial loop): its shortest run [t, t + dlo) ends by its next own static start and fits at its last slot.
    // Placements at t only raise occupancy, so a candidate failing here fails its serial test too.
    {
      const int xe = t + dlo;
      elig = elig && xe <= ns && (dlo == 0 || (int)sm.occ[xe - 1] + (int)g <= L);
#if DSTACK_CYC_PRE_PTS >= 2
      elig = elig && (int)sm.occ[t + (dlo >> 1)] + (int)g <= L;   // dlo >= 1 here (xe - 1 >= t)
#endif
#if DSTACK_CYC_PRE_PTS >= 3
      elig = elig && (int)sm.occ[t + (dlo >> 2)] + (int)g <= L && (int)sm.occ[t + ((3 * dlo) >> 2)] + (int)g <= L;
#endif
    }
    // candidates in (runs so far, index) order; a placement raises occ[t], so re-test the rest in parallel
    const uint32_t prio = fill_order == 0 ? count : (fill_order == 1 ? g : dstar);
    uint32_t key = elig ? ((prio << 5) | (uint32_t)lane) : 0xFFFFFFFFu;
#if DSTACK_PROF_STATS
    bool st_first = true;
#endif
    while (true) {
      const uint32_t mk = __reduce_min_sync(FULL, key);
      if (mk == 0xFFFFFFFFu) break;
      const int j = (int)(mk & 31u);
      if (lane == 0) CSTAT(4, 1);
#if DSTACK_PROF_STATS
      if (lane == 0 && st_first) CSTAT(8, 1);   // decision times with at least one candidate
      st_first = false;
#endif
      if (lane == j) key = 0xFFFFFFFFu;
      const uint32_t pj = __shfl_sync(FULL, pk, j);
      const int gj = (int)(pj & 0xFFu), bsj = (int)((pj >> 8) & 0xFFu), dsj = (int)(pj >> 16);
      const int limit = __shfl_sync(FULL, ns, j);
      // slice: first u in [t, stop) with occ[u] + g > L, else stop (stop = min(t + d(b*), next own static start))
      const int stop = min(t + dsj, limit);
      int kend;
      if (stop <= bt + 128) {   // first blocking slot of the window at or after t, capped at stop
        const uint32_t bb = __vcmpgtu4(wvm, (uint32_t)(L - gj) * 0x01010101u);
        const uint32_t bal = __ballot_sync(FULL, bb != 0u);
        kend = stop;
        if (bal) {
          const int pl = __ffs(bal) - 1;
          kend = min(stop, bt + 4 * pl + ((__ffs(__shfl_sync(FULL, bb, pl)) - 1) >> 3));
        }
      } else {
        kend = first_above(sm.occ, t, stop, L - gj, lane);
      }
      const int kslice = kend - t;
      int bsel = 0, dsel = 0;   // largest b in [b_lo, b*] with d(b) <= slice (d nondecreasing in b), and d(b)
      const uint16_t *dj = dtab + j * DSTACK_MAX_BATCH;
      if (kslice >= dsj) {
        bsel = bsj; dsel = dsj;
      } else if (!hook_b_only && bsj - 1 >= b_lo) {
        for (int b0 = b_lo + 32 * ((bsj - 1 - b_lo) >> 5); b0 >= b_lo; b0 -= 32) {
          const int b = b0 + lane;
          const int dv = b < bsj ? (int)dj[b - 1] : 0x7FFFFFFF;
          const uint32_t bal = __ballot_sync(FULL, dv <= kslice);
          if (bal) {
            const int src = 31 - __clz(bal);
            bsel = b0 + src; dsel = __shfl_sync(FULL, dv, src);
            break;
          }
        }
      }
      if (bsel == 0) {
        if (lane == j) blk = kend;
        continue;
      }
      if (lane == 0) { CSTAT(5, 1); CSTAT(6, bsel != bsj); CSTAT(7, kslice < dsj); }
      const int e = t + dsel;
      if (e <= bt + 128) {   // place inside the window: register word + write-through
        const uint32_t add = ((uint32_t)gj * 0x01010101u) & bytes_mask(t, e, mybase);
        if (add) { wv += add; w32[wi] = wv; }
        wvm += add;
      } else {
        occ_add(sm.occ, t, dsel, gj, lane);
        wv = w32[wi];
        wvm = wv & lo_mask;
      }
      if (dsel > 0) occ_t += gj;   // a zero-length run (d = 0, reachable through the test hook) occupies no slot
      occ_fill += (uint32_t)dsel * (uint32_t)gj;
      if (lane == 0 && fill_log && nfill < fill_cap) fill_log[nfill] = pack_run((uint32_t)j, (uint32_t)t, (uint32_t)dsel, (uint32_t)bsel);
      nfill++;
      __syncwarp();
      if (lane == j) {
        count++; runs++; served += (uint32_t)bsel; free_at = e;
        if (busy) *busy += (uint32_t)dsel;
      }
      if (occ_t + (int)g > L) key = 0xFFFFFFFFu;
    }
    const uint32_t nend = (uint32_t)(free_at > t ? free_at : ne);   // inactive lanes: free_at = 0, no static run
    t = (int)min(__reduce_min_sync(FULL, nend), (uint32_t)nslots);
  }
  res.occ_all = res.occ_static + occ_fill;   // every run lies inside [0, nslots)
  if (lane == 0) CSTAT(0, 1);
  if (fill_n) *fill_n = nfill;
  res.served_tot = __reduce_add_sync(FULL, served);
  return res;
}

}  // namespace dstack
