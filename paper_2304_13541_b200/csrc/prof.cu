// prof.cu -- a1-a3 kernels (dstack_batch_opt, dstack_knee, first stage of dstack_eval_batch / _simulate):
// one warp per DNN, grid-stride.
//
//  k_prof<PAR>     generic path, every mode (prof.cuh: row pass, coefficient tables, exact branch-and-bound
//                  over all batches).
//  k_prof_fast<CB> the printed model's defaults (linear N_i(b) = b n_i, per-request W_se, b_lo = 1;
//                  SURVEY §8(c) O1/O3), register-resident: the width histogram is scanned into per-lane
//                  registers (CB consecutive widths per lane), the b = 1 row is evaluated from them, and
//                  one b-independent certificate proves that no b >= 2 can beat it ("batch
//                  certificate").  A DNN whose certificate fails is re-analysed by the generic path.
#include "kernels.cuh"
#include "prof.cuh"

namespace dstack {

__host__ __device__ inline size_t prof_warp_bytes(int S_tot) {
  return (((size_t)20 * (S_tot + 1)) + 15) & ~(size_t)15;   // cA, cU u64 + hist u32
}

#ifndef DSTACK_PROF_MINB
#define DSTACK_PROF_MINB 4
#endif
#ifndef DSTACK_PROF_GRID
#define DSTACK_PROF_GRID 64   // k_prof grid: blocks per SM (4 resident; A/B ms: 4 -> 10.6, 8 -> 10.31, 16 -> 9.99, 32 -> 9.8, 64 -> 9.7, 128 -> 9.67, 256 -> 9.74)
#endif
#ifndef DSTACK_PROF_DYN
#define DSTACK_PROF_DYN 1   // 1: k_prof_fast takes groups of 32 DNNs from a work counter (A/B switch)
#endif
#ifndef DSTACK_PROF_ROWS_U
#define DSTACK_PROF_ROWS_U 7   // rows per lane in flight in the row pass (A/B at config 3, k_prof_lane ms: 4 -> 5.35, 5 -> 4.87, 6 -> 4.70, 7 -> 4.66, 8 -> 4.76)
#endif
#ifndef DSTACK_PROF_FAST
#define DSTACK_PROF_FAST 1   // 0: every launch takes the generic kernel (A/B switch)
#endif

// F3, online knee discovery: from the nominal level ceil(0.3 L), a binary search over
// l in [1, L] that compares the Eq. 6 objective g(l) = 1/(f_L(l,b)^2 S(l)) of adjacent levels m, m+1 (two latency
// measurements per step): g(m+1) > g(m) <=> S(m+1) X(m)^2 > S(m) X(m+1)^2 (exact, u128) moves right, else left.
// X from the DNN's O(1) tables (valid after analyze_dnn at batch b).  Warp-uniform; returns knee | steps << 16.
template <int PAR>
__device__ __forceinline__ uint32_t knee_probe_search(const dstack_problem_t &pb, const dstack_params_t &p, int64_t k,
                                                      const uint16_t *Stab, const uint64_t *cA, const uint64_t *cU,
                                                      uint64_t RT, uint64_t D, int32_t b) {
  const uint64_t M = p.mem_mode == 0 ? 1ull : (uint64_t)pb.mem_bw[k];
  const uint64_t wC1 = (p.wse_mode == 0 ? (uint64_t)b : 1ull) * (uint64_t)pb.t_np[k] * RT * M;
  const uint32_t magic = magic_of(b);
  int32_t lo = 1, hi = p.L, steps = 0;
  int32_t m = (3 * p.L + 9) / 10;   // ceil(0.3 L): the nominal 30% start
  while (lo < hi) {
    if (steps > 0) m = (lo + hi) >> 1;
    m = m < lo ? lo : (m > hi - 1 ? hi - 1 : m);
    const int32_t S0 = Stab[m], S1 = Stab[m + 1];
    const uint64_t X0 = cell_X<PAR>(S0, b, magic, wC1, cA, cU, p.mem_mode, D);
    const uint64_t X1 = cell_X<PAR>(S1, b, magic, wC1, cA, cU, p.mem_mode, D);
    const bool right = (u128)(uint32_t)S1 * ((u128)X0 * X0) > (u128)(uint32_t)S0 * ((u128)X1 * X1);
    if (right) lo = m + 1; else hi = m;
    ++steps;
  }
  return (uint32_t)lo | ((uint32_t)steps << 16);
}

// generic per-DNN analysis and its outputs
template <int PAR>
__device__ __forceinline__ void prof_one(const ProfArgs &a, int64_t k, const uint16_t *Stab, uint32_t *hist,
                                         uint64_t *cA, uint64_t *cU, int lane) {
  DnnRes r = analyze_dnn<PAR>(a.pb, a.p, k, Stab, hist, cA, cU, lane, a.probes ? 2 : a.knee_only, a.knee_b);
  if (a.probes) {   // F3: the probe's knee replaces Eq. 6's exact argmax
    uint32_t steps = 0;
    if (r.st == DSTACK_ST_OK) {
      const uint32_t v = knee_probe_search<PAR>(a.pb, a.p, k, Stab, cA, cU, r.RT, r.D, a.knee_b);
      r.knee = (uint16_t)(v & 0xFFFFu); steps = v >> 16;
    }
    if (lane == 0) a.probes[k] = (uint8_t)steps;
  }
  if (a.dtab_rows && r.st == DSTACK_ST_OK) {   // eval path: d_j(b) at g = demand, b in [b_lo, b*]
    if (PAR == 0)
      dtab_from_tables(a.pb, a.p, k, cA, cU, r.RT, r.D, r.demand, a.p.b_min, r.b, a.dtab_rows + k * DTAB_ROW, lane);
    else
      dtab_from_rows(a.pb, a.p, k, r.RT, r.D, r.demand, a.p.b_min, r.b, a.dtab_rows + k * DTAB_ROW, lane);
    if (a.dstar && lane == 0) a.dstar[k] = a.dtab_rows[k * DTAB_ROW + r.b - 1];
  }
  if (lane == 0) {
    if (a.ws_RT) { a.ws_RT[k] = (uint32_t)r.RT; a.ws_D[k] = r.D; }
    const bool ok = r.st == DSTACK_ST_OK;
    if (a.knee) a.knee[k] = ok ? r.knee : 0;
    if (a.status) a.status[k] = r.st;
    if (!a.knee_only) {
      if (a.demand) a.demand[k] = ok ? r.demand : 0;
      if (a.batch) a.batch[k] = ok ? r.b : 0;
    }
  }
  __syncwarp();
}

template <int PAR>
__global__ void __launch_bounds__(256, DSTACK_PROF_MINB) k_prof(ProfArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int L = a.p.L, S_tot = a.p.S_tot;
  uint16_t *Stab = (uint16_t *)smem;
  const int tab_bytes = ((L + 1 + S_tot + 1) * 2 + 15) & ~15;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char *wreg = smem + tab_bytes + (size_t)warp * prof_warp_bytes(S_tot);
  uint64_t *cA = (uint64_t *)wreg;
  uint64_t *cU = cA + (S_tot + 1);
  uint32_t *hist = (uint32_t *)(cU + (S_tot + 1));
  fill_stab(Stab, L, S_tot);
  __syncthreads();
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t gwarp = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  for (int64_t k = warp_next_item(a.work_ctr, -1, gwarp, nwarps, lane); k < a.pb.num_dnn;
       k = warp_next_item(a.work_ctr, k, gwarp, nwarps, lane))
    prof_one<PAR>(a, k, Stab, hist, cA, cU, lane);
}

// ------------------------------------------------------------------------------------------------------
// fast path
// ------------------------------------------------------------------------------------------------------

// cold: generic re-analysis of DNN k (certificate failed); leaves the histogram zeroed for the fast path
static __device__ __noinline__ void prof_one_cold(const ProfArgs *a, int64_t k, const uint16_t *Stab, uint32_t *hist,
                                                  uint64_t *cA, uint64_t *cU, int lane) {
  PSTAT(8, lane == 0);
  prof_one<0>(*a, k, Stab, hist, cA, cU, lane);
  for (int m = lane; m <= a->p.S_tot; m += 32) hist[m] = 0;
  __syncwarp();
}

// cold: exact argmax of S / X^2 (ties -> smaller S) over the candidates S in [1, S_tot] whose float score
// reaches `band` (X = scr[S]; candidate set: attained widths, and 2X <= S F when F != 0)
struct SX {
  uint64_t X;
  uint32_t S;
};
static __device__ __noinline__ SX band_exact(const uint64_t *scr, const uint16_t *lmin, int S_tot, uint64_t F, float band,
                                             int lane) {
  Best v = best_none();
  for (int S = 1 + lane; S <= S_tot; S += 32) {
    const uint64_t X = scr[S];
    const float f = score_f((uint32_t)S, X);
    if (!lmin[S] || f < band || (F != 0 && 2 * X > (uint64_t)S * F)) continue;
    Best c; c.found = 1; c.l = (uint32_t)S; c.b = 1; c.S = (uint32_t)S; c.X = X; c.sc = f;
    if (better(c, v)) v = c;
  }
  v = warp_best_exact(v);
  SX o;
  o.S = v.found ? v.S : 0u;
  o.X = v.X;
  return o;
}

// Per-lane top-2 tracker of float scores (t1 >= t2; s1 = width of t1, first occurrence).
struct Top2 {
  float t1, t2;
  uint32_t s1;
};
__device__ __forceinline__ void top2_add(Top2 &t, float f, uint32_t S) {   // branch-free
  const bool gt = f > t.t1;
  t.t2 = fmaxf(t.t2, fminf(t.t1, f));
  t.s1 = gt ? S : t.s1;
  t.t1 = fmaxf(t.t1, f);
}

// Warp argmax from the per-lane top-2 trackers: the float maximum decides unless a second candidate lies
// within 2^-19 of it (float scores are within 2^-21 of the exact ones, so the exact winner is always in
// that band); then the band is resolved exactly from the X values staged in scr[S].  F != 0: the
// feasible set (2X <= S F), else all attained widths.  One call site for both argmaxes (unroll 1).
__device__ __forceinline__ SX fast_argmax(const Top2 &t, const uint64_t *scr, const uint16_t *lmin, int S_tot,
                                          uint64_t F, int lane) {
  SX o;
  o.S = 0; o.X = 0;
  const uint32_t mx = __reduce_max_sync(FULL, __float_as_uint(t.t1));   // scores > 0: u32 order = float order
  if (mx == 0) return o;
  const float band = __uint_as_float(mx) * 0.99999809f;   // 1 - 2^-19 (score_f error <= 6 * 2^-24)
  const uint32_t cnt = (uint32_t)(t.t1 >= band) + (uint32_t)(t.t2 >= band);
  if (__reduce_add_sync(FULL, cnt) == 1) {
    o.S = __shfl_sync(FULL, t.s1, __ffs(__ballot_sync(FULL, cnt != 0)) - 1);
    o.X = scr[o.S];
    return o;
  }
  PSTAT(9, lane == 0);
  return band_exact(scr, lmin, S_tot, F, band, lane);
}

// cold: argmax of S / X^2 over the attained widths with 2X <= S F, from the staged X values (float filter, exact
// band resolution as fast_argmax)
static __device__ __noinline__ SX feasible_argmax(const uint64_t *scr, const uint16_t *lmin, int S_tot, uint64_t F,
                                                  int lane) {
  Top2 te = {0.f, 0.f, 0u};
  for (int S = 1 + lane; S <= S_tot; S += 32) {
    const uint64_t X = scr[S];
    const bool ok = lmin[S] != 0 && 2 * X <= (uint64_t)S * F;
    top2_add(te, ok ? score_f((uint32_t)S, X) : 0.f, (uint32_t)S);
  }
  return fast_argmax(te, scr, lmin, S_tot, F, lane);
}

// Exact sum over the warp of per-lane values < 2^59 from three 32-bit reductions (22/22/15-bit limbs).
// *top = the reduced top limb (the total is >= top * 2^44; the returned sum wraps only if top >= 2^20).
__device__ __forceinline__ uint64_t warp_sum_limbs(uint64_t v, uint32_t *top) {
  const uint32_t c0 = __reduce_add_sync(FULL, (uint32_t)v & 0x3FFFFFu);
  const uint32_t c1 = __reduce_add_sync(FULL, (uint32_t)(v >> 22) & 0x3FFFFFu);
  const uint32_t c2 = __reduce_add_sync(FULL, (uint32_t)(v >> 44));
  *top = c2;
  return (uint64_t)c0 + ((uint64_t)c1 << 22) + ((uint64_t)c2 << 44);
}

// min(ceil(X / den), 0xFFFF) for den >= 1: f32 quotient estimate (error < 0.05 below the clamp), exact fix-up
__device__ __forceinline__ uint32_t ceil_div_clamp16_fast(uint64_t X, uint64_t den) {
  const float qf = (float)X * rcp_approx((float)den);
  if (qf > 65600.f) return 0xFFFFu;
  uint64_t q = (uint64_t)qf;
  if (q * den > X) --q;
  else if ((q + 1) * den <= X) ++q;
  q += (q * den < X);
  return q > 0xFFFFu ? 0xFFFFu : (uint32_t)q;
}

// One DNN on the fast path.  Header values arrive warp-uniform (broadcast from the lane that loaded them).
// Returns false when the DNN must be decided by the generic path (the caller runs prof_one_cold).
template <int CB>
__device__ __forceinline__ bool fast_dnn(const ProfArgs &a, int64_t k, int64_t r0, int32_t K, uint32_t okb,
                                         uint32_t M, uint32_t t_np, uint64_t Mtp, uint64_t F, uint32_t vmask,
                                         const uint16_t *Stab, const uint16_t *lmin, uint32_t *hist, uint64_t *cA,
                                         uint64_t *cU, int lane, uint32_t &st, uint32_t &RT, uint64_t &D,
                                         uint32_t &knee, uint32_t &demand, uint32_t &dslots) {
  const dstack_problem_t &pb = a.pb;
  const dstack_params_t &p = a.p;
  const int L = p.L, S_tot = p.S_tot, mem_mode = p.mem_mode;
  st = DSTACK_ST_OK; RT = 0; D = 0; knee = demand = dslots = 0;
  if (!(okb & 1u)) { st = DSTACK_ST_INVALID; return true; }
  const int32_t b_hi = (int32_t)(okb >> 8);
  // ---- a1: one coalesced pass over the rows: RT, min R, D = sum R d, W> = sum_{n > S_tot} R n, and the
  //      width histogram of R over n <= S_tot (smem) ----
  uint32_t Rmin = 0xFFFFFFFFu;
  uint64_t Wb = 0;
  const uint32_t *n = pb.n + r0;
  const uint16_t *r = pb.r + r0;
  const uint32_t *d = pb.d + r0;
  // DSTACK_PROF_ROWS_U rows per lane in flight per iteration
  for (int i0 = lane; i0 < K; i0 += 32 * DSTACK_PROF_ROWS_U) {
    uint32_t nn[DSTACK_PROF_ROWS_U], dd[DSTACK_PROF_ROWS_U], RR[DSTACK_PROF_ROWS_U];
#pragma unroll
    for (int u = 0; u < DSTACK_PROF_ROWS_U; ++u) {
      const int i = i0 + 32 * u;
      nn[u] = 0; dd[u] = 0; RR[u] = 0;
      if (i < K) { nn[u] = __ldg(n + i); dd[u] = __ldg(d + i); RR[u] = __ldg(r + i); }
    }
#pragma unroll
    for (int u = 0; u < DSTACK_PROF_ROWS_U; ++u) {
      if (i0 + 32 * u < K) {
        RT += RR[u]; D += (uint64_t)RR[u] * dd[u]; Rmin = min(Rmin, RR[u]);
        if (nn[u] <= (uint32_t)S_tot) atomicAdd(&hist[nn[u]], RR[u]); else Wb += (uint64_t)RR[u] * nn[u];
      }
    }
  }
  RT = __reduce_add_sync(FULL, RT);
  Rmin = __reduce_min_sync(FULL, Rmin);
  uint32_t Dtop, Wtop;
  D = warp_sum_limbs(D, &Dtop);
  Wb = warp_sum_limbs(Wb, &Wtop);
  __syncwarp();
  // ---- scan of the histogram (lane owns widths m0..m0+CB-1, re-zeroing them): exclusive lane offsets;
  //      the per-width prefixes PA[m] = sum_{1<=n<=m} R, PW[m] = sum_{n<=m} n R (u32: RT < 2^24 here) are
  //      formed in the candidate pass below ----
  int m0 = lane * CB;
  asm volatile("" : "+r"(m0));   // per-DNN value: keeps the per-width constants out of the loop-invariant (spilled) set
  uint32_t h[CB], ra, rw, Wsm;
  {
    uint32_t sa = 0, sw = 0;
#pragma unroll
    for (int i = 0; i < CB; ++i) {
      const int m = m0 + i;
      h[i] = 0;
      if (m <= S_tot) { h[i] = hist[m]; hist[m] = 0; }
      if (m == 0) h[i] = 0;   // n = 0 rows: in neither PA nor sum n R
      sa += h[i]; sw += h[i] * (uint32_t)m;
    }
    uint32_t ia = sa, iw = sw;
#pragma unroll
    for (int dd = 1; dd < 32; dd <<= 1) {
      const uint32_t ua = __shfl_up_sync(FULL, ia, dd), uw = __shfl_up_sync(FULL, iw, dd);
      if (lane >= dd) { ia += ua; iw += uw; }
    }
    Wsm = __shfl_sync(FULL, iw, 31);
    ra = ia - sa; rw = iw - sw;
  }
  // ---- status (same order as the generic path) ----
  if (Rmin == 0 || (t_np == 0 && Wb == 0 && Wtop == 0 && Wsm == 0 && (mem_mode == 0 || (D == 0 && Dtop == 0)))) {
    st = DSTACK_ST_INVALID;
    return true;
  }
  if (b_hi < 1) { st = DSTACK_ST_INFEASIBLE; return true; }
  if (RT >= (1u << 24) || Wtop >= (1u << 19) || Dtop >= (1u << 19)) {   // outside the u32 / u64 fast ranges
    return false;
  }
  // ---- a2/a3 at b = 1: X(S, 1) = S C1 + Mtp (S PA[S] + Q[S]) + mem for every attained S (exact u64 once the
  //      overflow test below passes; staged in scr[S] for the argmax), per-lane top-2 trackers of the
  //      scores, and the batch certificate G over the segments m <= S_tot/2 ----
  const uint64_t C1 = (uint64_t)t_np * M * RT;
  const uint64_t memb = mem_mode == 1 ? D : 0ull;
  const uint64_t base = Mtp * Wb + memb;
  const float C1f2 = 2.f * (float)C1, Mtpf = (float)Mtp, Wbf = (float)Wb, membf = (float)memb;
  const float half = 0.5f * (float)S_tot;
  const int mh = S_tot >> 1;
  uint64_t *scr = cA;
  Top2 tk = {0.f, 0.f, 0u};
  float G = 0.f;
  {
    // overflow: X(L, b_hi) = b_hi t_np RT S_tot M + M t_p (S_tot PA[mb] + b_hi Q[mb]) + mem is the grid maximum;
    // with PA[mb] <= RT and Q[mb] <= W this bound (f64) settles it unless within 1e-4 of 2^56, where the
    // generic path decides exactly
    const double bd = (double)b_hi, Sd = (double)S_tot;
    double xe = bd * (double)t_np * (double)M * (double)RT * Sd +
                (double)Mtp * (Sd * (double)RT + bd * ((double)Wb + (double)Wsm));
    if (mem_mode == 1) xe += bd * (double)D;
    else if (mem_mode == 2) xe += bd * (double)D * Sd * Sd;
    if (xe >= 72057594037927936.0 * 0.9999) return false;
  }
#pragma unroll
  for (int i = 0; i < CB; ++i) {
    const uint32_t S = (uint32_t)(m0 + i);
    ra += h[i]; rw += h[i] * S;                          // PA[S], PW[S]
    const uint32_t q = Wsm - rw;                         // Q[S] - W>
    uint64_t X = (uint64_t)S * C1 + Mtp * ((uint64_t)S * ra + q) + base;
    if (mem_mode == 2) X += D * (uint64_t)(S * S);
    if ((int)S <= S_tot) scr[S] = X;
    const float f = score_f(S, X);
    const bool valid = (vmask >> i) & 1u;
    top2_add(tk, valid ? f : 0.f, S);
    // Batch certificate: for b >= 2 and s = S/b in segment m = floor(s),
    // X(S, b) >= b (alpha s + beta), alpha = 2 C1 + Mtp PA[m], beta = Mtp Q[m] + mem, hence
    // eta(S, b) <= s / (alpha s + beta)^2; G = max over m <= S_tot/2 of its supremum on [m, m+1).
    if ((int)S <= mh) cU[S] = ((uint64_t)q << 32) | ra;   // (PA[m], Q[m] - W>) for the certificate pass below
  }
  __syncwarp();
  uint32_t Sk = 0, Se = 0;
  uint64_t Xe = 0;
  {
    // knee = the exact argmax over every attained width (ties -> smaller S); when that width is feasible
    // (Eqs. 11-12: 2X <= S F) it is also the exact argmax over the feasible widths (a subset containing it),
    // else the feasible argmax is searched over the staged X values (cold)
    const SX r = fast_argmax(tk, scr, lmin, S_tot, 0ull, lane);
    Sk = r.S;
    if (F != 0 && 2 * r.X <= (uint64_t)r.S * F) { Se = r.S; Xe = r.X; }
    else { const SX e = feasible_argmax(scr, lmin, S_tot, F == 0 ? 1ull : F, lane); Se = e.S; Xe = e.X; }
  }
  if (Se == 0) { st = DSTACK_ST_INFEASIBLE; return true; }   // b = 1 is feasible whenever any b is (O3)
  // b* = 1 is certified when the incumbent beats G with a 2^-12 margin (f32 rounding of both sides is
  // < 2^-19); otherwise the generic exact branch-and-bound decides this DNN.
  if (b_hi >= 2) {
    // lanes over the segments m = 0 .. S_tot/2 (instead of every lane's CB widths): the same bound per m
    for (int m = lane; m <= mh; m += 32) {
      const uint64_t pv = cU[m];
      const uint32_t ra = (uint32_t)pv, q = (uint32_t)(pv >> 32);
      const float af = fmaf(Mtpf, (float)ra, C1f2), bf = fmaf(Mtpf, (float)q + Wbf, membf);
      const float lo = (float)m, hi = fminf(lo + 1.f, half);
      const float sx = fminf(fmaxf(bf * rcp_approx(af), lo), hi);
      const float x = fmaf(af, sx, bf);
      const float v = bf == 0.f ? __int_as_float(0x7f800000) : sx * rcp_approx(x * x);
      G = fmaxf(G, v);
    }
    const float Gw = __uint_as_float(__reduce_max_sync(FULL, __float_as_uint(G)));
    if (!(score_f(Se, Xe) * 0.99975586f > Gw)) return false;
  }
  knee = lmin[Sk];
  const uint32_t le = lmin[Se];
  demand = le + (uint32_t)p.margin < (uint32_t)L ? le + (uint32_t)p.margin : (uint32_t)L;
  // d_j(1) = ceil(X(S(g), 1) / (S(g) M Delta)) at g = demand
  if (a.dtab_rows) {
    const uint32_t Sg = Stab[demand];
    dslots = ceil_div_clamp16_fast(Sg == Se ? Xe : scr[Sg], (uint64_t)Sg * M * (uint64_t)p.slot_us);
  }
  return true;
}

// per-warp staging of 32 DNN headers / results in shared memory (keeps them out of the register file)
struct __align__(16) FastHdr {
  int64_t r0;
  uint64_t Mtp, F;
  int32_t K;
  uint32_t okb, M, tnp;
};
struct __align__(8) FastOut {
  uint64_t D;
  uint32_t RT, kd, sd, pad;   // kd: knee | demand << 16; sd: d_j(1) | status << 16 | cold << 24
};
constexpr size_t FAST_STAGE_BYTES = 32 * (sizeof(FastHdr) + sizeof(FastOut));

// Fast-path kernel: each warp owns a contiguous range of DNNs and walks it 32 at a time; lane j loads and
// validates DNN kb+j's header (coalesced, one pass per 32 DNNs) and buffers its outputs, which are
// written back coalesced after the 32 analyses.
template <int CB>
__global__ void __launch_bounds__(256, DSTACK_PROF_MINB) k_prof_fast(const __grid_constant__ ProfArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const dstack_problem_t &pb = a.pb;
  const dstack_params_t &p = a.p;
  const int L = p.L, S_tot = p.S_tot;
  uint16_t *Stab = (uint16_t *)smem;
  uint16_t *lmin = Stab + (L + 1);
  const int tab_bytes = ((L + 1 + S_tot + 1) * 2 + 15) & ~15;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char *wreg = smem + tab_bytes + (size_t)warp * prof_warp_bytes(S_tot);
  uint64_t *cA = (uint64_t *)wreg;
  uint64_t *cU = cA + (S_tot + 1);
  uint32_t *hist = (uint32_t *)(cU + (S_tot + 1));
  FastHdr *shdr = reinterpret_cast<FastHdr *>(smem + tab_bytes + (size_t)(blockDim.x >> 5) * prof_warp_bytes(S_tot) +
                                              (size_t)warp * FAST_STAGE_BYTES);
  FastOut *sout = reinterpret_cast<FastOut *>(shdr + 32);
  fill_stab(Stab, L, S_tot);
  // lmin[S] = smallest level l with S(l) = S (0: S not attained); ties between levels -> smaller l
  for (int S = threadIdx.x; S <= S_tot; S += blockDim.x) {
    const int l = S == 0 ? 0 : ((S - 1) * L) / S_tot + 1;
    lmin[S] = (uint16_t)((S >= 1 && l <= L && s_of(l, S_tot, L) == S) ? l : 0);
  }
  for (int m = lane; m <= S_tot; m += 32) hist[m] = 0;
  __syncthreads();
  uint32_t vmask = 0;   // bit i: width S = lane*CB + i is attained by some level
#pragma unroll
  for (int i = 0; i < CB; ++i) {
    const int S = lane * CB + i;
    if (S >= 1 && S <= S_tot && lmin[S]) vmask |= 1u << i;
  }
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t per = (pb.num_dnn + nw - 1) / nw;
  const int64_t kbeg = ((int64_t)blockIdx.x * (blockDim.x >> 5) + warp) * per;
  // groups of 32 DNNs: taken from the work counter (one resident wave of warps) or the warp's contiguous range
  const bool dyn = a.work_ctr != nullptr;
  const int64_t kend = dyn ? pb.num_dnn : (kbeg + per < pb.num_dnn ? kbeg + per : pb.num_dnn);
  auto fetch = [&](int64_t prev) -> int64_t {   // a reduction: the index is provably warp-uniform (common.cuh)
    uint32_t v = 0;
    if (dyn) {
      if (lane == 0) v = atomicAdd(a.work_ctr, 32u);
    } else {
      v = (uint32_t)(prev < 0 ? kbeg : prev + 32);
    }
    return (int64_t)__reduce_max_sync(FULL, v);
  };
  for (int64_t kb = fetch(-1); kb < kend; kb = fetch(kb)) {
    const int nj = kend - kb < 32 ? (int)(kend - kb) : 32;
    const int64_t kl = kb + lane;
    const bool have = lane < nj;
    // ---- lane-parallel header: load + validate (DSTACK_ST_INVALID conditions, dstack.h) ----
    if (have) {
      FastHdr h;
      h.r0 = pb.dnn_row_off[kl];
      const int64_t K64 = pb.dnn_row_off[kl + 1] - h.r0;
      const int32_t t_p = pb.t_p[kl], t_np = pb.t_np[kl], slo = pb.slo_us[kl], asm_us = pb.asm_us[kl];
      const int32_t bmax = pb.bmax[kl], mbw = pb.mem_bw[kl];
      const bool ok = !(K64 < 1 || K64 > DSTACK_MAX_ROWS_PER_DNN || t_p < 1 || t_np < 0 || slo < 1 ||
                        slo > (1 << 30) || (slo % p.slot_us) != 0 || asm_us < 0 || asm_us > (1 << 24) || bmax < 1 ||
                        (p.mem_mode != 0 && (mbw < 1 || mbw > (1 << 24))));
      h.K = ok ? (int32_t)K64 : 0;
      h.M = p.mem_mode == 0 ? 1u : (uint32_t)mbw;
      h.tnp = (uint32_t)t_np;
      h.Mtp = (uint64_t)h.M * (uint32_t)t_p;
      // Eqs. 11-12 at b = 1 as one test 2X <= S F:  F = min(2 (SLO - a) M, SLO M)  (0 if a > SLO)
      const uint64_t SLOM = (uint64_t)slo * h.M, aM = (uint64_t)asm_us * h.M;
      h.F = SLOM < aM ? 0ull : (2 * (SLOM - aM) < SLOM ? 2 * (SLOM - aM) : SLOM);
      const int32_t b_hi = bmax < p.b_max ? bmax : p.b_max;
      h.okb = ok ? (1u | ((uint32_t)b_hi << 8)) : 0u;
      shdr[lane] = h;
    }
    __syncwarp();
    for (int jj = 0; jj < nj; ++jj) {
      const FastHdr h = shdr[jj];
      uint32_t st, RT, knee, dem, ds;
      uint64_t D;
      const bool done = fast_dnn<CB>(a, kb + jj, h.r0, h.K, h.okb, h.M, h.tnp, h.Mtp, h.F, vmask, Stab, lmin, hist, cA,
                                     cU, lane, st, RT, D, knee, dem, ds);
      if (!done) prof_one_cold(&a, kb + jj, Stab, hist, cA, cU, lane);
      if (lane == 0) {
        FastOut o;
        o.D = D; o.RT = RT; o.kd = knee | (dem << 16); o.sd = ds | (st << 16) | (done ? 0u : (1u << 24)); o.pad = 0;
        sout[jj] = o;
      }
    }
    __syncwarp();
    // ---- coalesced write-back of the 32 DNNs' outputs ----
    if (have) {
      const FastOut o = sout[lane];
      if (!(o.sd >> 24)) {
        const uint32_t st = (o.sd >> 16) & 0xFFu;
        const bool ok = st == DSTACK_ST_OK;
        if (a.ws_RT) { a.ws_RT[kl] = o.RT; a.ws_D[kl] = o.D; }
        if (ok) {   // d_j(1): the dense array on the eval path, else the row's b = 1 entry
          if (a.dstar) a.dstar[kl] = (uint16_t)(o.sd & 0xFFFFu);
          else if (a.dtab_rows) a.dtab_rows[kl * DTAB_ROW] = (uint16_t)(o.sd & 0xFFFFu);
        }
        if (a.knee) a.knee[kl] = ok ? (uint16_t)(o.kd & 0xFFFFu) : 0;
        if (a.status) a.status[kl] = (uint8_t)st;
        if (a.demand) a.demand[kl] = ok ? (uint16_t)(o.kd >> 16) : 0;
        if (a.batch) a.batch[kl] = ok ? 1 : 0;
      }
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------------------------------------------
// lane-per-DNN fast path (k_prof_lane): the same decisions as k_prof_fast, organised so that the per-DNN
// scalar work runs one DNN per lane
// ------------------------------------------------------------------------------------------------------
//  * a warp takes groups of 32 consecutive DNNs; lane j loads and validates DNN kb+j's header;
//  * a1 row pass, warp-cooperative and coalesced, one DNN after the other: per-lane partial sums (RT, min R,
//    D = sum R d, W> = sum_{n > S_tot} R n, Wsm = sum_{n <= S_tot} R n) reduced to the owning lane, and the width
//    histogram H[n] = sum_{n_i = n} R_i of n <= S_tot accumulated with shared-memory atomics into the owning
//    lane's row of a [32][HSTRIDE] u32 table, two u16 bins per word (the fast path requires RT < 2^16, so no bin
//    carries), HSTRIDE odd so that the lanes' rows start in distinct banks;
//  * a2/a3 per lane: one sequential scan of the widths S = 1..S_tot forms PA[S], PW[S] and the exact
//    X(S, 1) = S C1 + Mtp (S PA[S] + Wsm - PW[S]) + Mtp W> + mem (O1, b = 1) in u64, keeps the exact argmax of
//    S / X^2 over the attained widths (ties -> smaller S; an f32 score filters, near-ties within 2^-19 are
//    decided by the 128-bit comparison S' X^2 vs S X'^2), and the b >= 2 certificate G over the
//    segments m <= S_tot / 2 from the same PA / Q values;
//  * a DNN outside the fast ranges (RT >= 2^16, X near 2^56, certificate not won) is re-analysed by the generic
//    warp path (prof_one_cold) after the group -- identical outputs, more work.
#ifndef DSTACK_PROF_LANE
#define DSTACK_PROF_LANE 1   // 1: the default-model fast path is k_prof_lane (0: k_prof_fast; A/B switch)
#endif
#ifndef DSTACK_PLANE_MINB
#define DSTACK_PLANE_MINB 2   // resident blocks per SM
#endif
#ifndef DSTACK_PLANE_WARPS
#define DSTACK_PLANE_WARPS 8   // warps per block
#endif

#ifndef DSTACK_PLANE_SEARCH
#define DSTACK_PLANE_SEARCH 1   // 1: a2/a3 by exact searches over the unimodal b = 1 curve (0: the f32 width scan; A/B)
#endif
__host__ __device__ inline int plane_nw(int S_tot) { return (S_tot + 2) >> 1; }         // bin words (bins 0..S_tot)
__host__ __device__ inline int plane_nck(int S_tot) { return ((plane_nw(S_tot) - 1) >> 2) + 1; }   // PPA checkpoints
__host__ __device__ inline int plane_hstride(int S_tot) {   // odd word stride
#if DSTACK_PLANE_SEARCH
  // a lane's row: the bins (then PA, in place), the PPA checkpoints, and room for a 4-word read at any checkpoint
  const int a = plane_nw(S_tot) + plane_nck(S_tot), b = 4 * plane_nck(S_tot);
  return (a > b ? a : b) | 1;
#else
  return plane_nw(S_tot) | 1;
#endif
}
__host__ __device__ inline size_t plane_warp_bytes(int S_tot) {
  // the H table; the cold path's scratch (cA, cU, hist) reuses it once the group's lane scans are done
  const size_t h = (size_t)32 * plane_hstride(S_tot) * 4, c = prof_warp_bytes(S_tot);
  return h > c ? h : c;
}

// exact-with-filter update of the running argmax (Sb, Xb, fb) of S / X^2 by a later (larger) width S
__device__ __forceinline__ void lane_best(uint32_t S, uint64_t X, float f, uint32_t &Sb, uint64_t &Xb, float &fb) {
  bool take;
  if (Sb == 0 || f > fb * 1.0000020f) take = true;          // 1 + 2^-19: certainly larger (score error < 2^-21)
  else if (f < fb * 0.99999809f) take = false;              // 1 - 2^-19: certainly smaller
  else take = (u128)S * ((u128)Xb * Xb) > (u128)Sb * ((u128)X * X);   // near tie: exact, strict (ties -> smaller S)
  if (take) { Sb = S; Xb = X; fb = f; }
}

// Exact scan (cold within the fast path): the exact argmax (Sb, Xb) of S / X^2 over the attained widths, or over
// those with 2X <= S F when feas_only (Eqs. 11-12 at b = 1); no_cert: skip the certificate terms.
template <int SCAN_MEM>   // 0: memory term off / bw (in `base`), 2: verbatim (D S^2)
static __device__ __noinline__ void lane_scan(const uint32_t *H, const uint16_t *lmin, int S_tot, int mh, uint64_t C1,
                                              uint64_t Mtp, uint64_t base, uint64_t D, uint32_t Wsm, uint64_t F,
                                              bool no_cert, float C1f2, float Mtpf, float Wbf, float membf, float half,
                                              uint32_t &Sb, uint64_t &Xb, float &fb, float &G, bool feas_only) {
  uint32_t ra = 0, rw = 0;
  const int nw = (S_tot >> 1) + 1;
  for (int w = 0; w < nw; ++w) {
    const uint32_t hw = H[w];
#pragma unroll
    for (int hi = 0; hi < 2; ++hi) {
      const uint32_t S = (uint32_t)(2 * w + hi);
      if (S > (uint32_t)S_tot) break;
      const uint32_t h = S == 0 ? 0u : (hi ? (hw >> 16) : (hw & 0xFFFFu));   // n = 0 rows: in neither PA nor PW
      ra += h; rw += h * S;
      const uint32_t q = Wsm - rw;                                             // Q[S] - W>
      if (!no_cert && (int)S <= mh) {   // certificate segment m = S: eta(S', b >= 2) <= s / (alpha s + beta)^2
        const float af = fmaf(Mtpf, (float)ra, C1f2), bf = fmaf(Mtpf, (float)q + Wbf, membf);
        const float lo = (float)S, hiS = fminf(lo + 1.f, half);
        const float sx = fminf(fmaxf(bf * rcp_approx(af), lo), hiS);
        const float x = fmaf(af, sx, bf);
        G = fmaxf(G, bf == 0.f ? __int_as_float(0x7f800000) : sx * rcp_approx(x * x));
      }
      if (S == 0 || !lmin[S]) continue;
      uint64_t X = (uint64_t)S * C1 + Mtp * ((uint64_t)S * ra + q) + base;
      if (SCAN_MEM == 2) X += D * (uint64_t)(S * S);
      if (feas_only && 2 * X > (uint64_t)S * F) continue;
      lane_best(S, X, score_f(S, X), Sb, Xb, fb);
    }
  }
}

// X(S, 1) at one width from the lane's histogram (the demand level's width when a margin moves it off the argmax)
__device__ __forceinline__ uint64_t lane_X_at(const uint32_t *H, uint32_t Sg, uint64_t C1, uint64_t Mtp, uint64_t base,
                                             uint64_t D, uint32_t Wsm, int mem_mode) {
  uint32_t ra = 0, rw = 0;
  for (uint32_t S = 1; S <= Sg; ++S) {
    const uint32_t hw = H[S >> 1];
    const uint32_t h = (S & 1) ? (hw >> 16) : (hw & 0xFFFFu);
    ra += h; rw += h * S;
  }
  uint64_t X = (uint64_t)Sg * C1 + Mtp * ((uint64_t)Sg * ra + (Wsm - rw)) + base;
  if (mem_mode == 2) X += D * (uint64_t)(Sg * Sg);
  return X;
}

// ---- a2/a3 by search (DSTACK_PLANE_SEARCH) -------------------------------------------------------------------
// O1 at b = 1 over the rows with n_i <= S_tot:  S PA[S] + Q[S] = sum_i R_i max(n_i, S) = Wsm + PPA(S), with
// PA[S] = sum_{1 <= n_i <= S} R_i and PPA(S) = sum_{k < S} PA[k] (summation by parts: PW[S] = S PA[S] - PPA(S)), so
//   X(S, 1) = S C1 + Mtp (Wsm + PPA(S)) + base  (+ D S^2 verbatim).
// sum_i R_i max(n_i, s) is convex in s, so X is convex and positive and S / X^2 is unimodal in S: d/ds log(s / X^2)
// has the sign of X - 2 s X', and (2 s X' - X)' = X' + 2 s X'' >= 0.  Both argmaxes are then binary searches:
//  * the knee (Eq. 6 at b = 1, ties -> smaller S) over the attained widths: compare adjacent candidates, keep the
//    left one on >=.  Strictly increasing before the real peak, so the first i with f(i) >= f(i + 1) is the
//    leftmost maximum (at most two maxima, adjacent);
//  * the b >= 2 certificate G: on segment m, s / (alpha_m s + beta_m)^2 rises while beta_m > alpha_m s,
//    and K(s) = alpha(s) s - beta(s) is nondecreasing (it jumps by 2 Mtp h(m+1) (m+1) >= 0 at each breakpoint), so
//    the supremum over (0, S_tot / 2] lies in the first segment m with alpha_m (m + 1) >= beta_m (exact u64), else
//    in the last; the closed form is evaluated there (the maximum over all segments of the scan version).
// The lane's histogram row becomes PA in place (u16, exact: RT < 2^16 on the fast path) with PPA checkpoints every
// 8 widths after the bins; PPA(S) = checkpoint + at most 7 PA terms.

// Row conversion: bins -> PA (bin 0, n = 0 rows, is in no prefix sum), PPA(8c) -> CK[c].  Returns PA[S_tot + 1].
__device__ __forceinline__ uint32_t lane_prefix(uint32_t *H, int nw, int nck) {
  uint32_t *CK = H + nw;
  uint32_t pa = 0, ppa = 0;
  for (int c = 0; c < nck; ++c) {   // warp-uniform bounds
    CK[c] = ppa;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int w = 4 * c + q;
      if (w < nw) {
        const uint32_t hw = H[w];
        const uint32_t p0 = pa + (w == 0 ? 0u : (hw & 0xFFFFu)), p1 = p0 + (hw >> 16);
        H[w] = (p0 & 0xFFFFu) | (p1 << 16);
        ppa += p0 + p1;
        pa = p1;
      }
    }
  }
  return pa;
}

// PPA(S) and PA[S] from the converted row (S <= S_tot)
__device__ __forceinline__ uint32_t lane_ppa(const uint32_t *H, int nw, uint32_t S, uint32_t &paS) {
  const uint32_t c = S >> 3, jj = (S & 7u) >> 1;
  const uint32_t *wp = H + 4 * c;
  uint32_t s = H[nw + c];
#pragma unroll
  for (uint32_t q = 0; q < 3; ++q) {   // whole words below S's word
    const uint32_t w = wp[q];
    s += q < jj ? (w & 0xFFFFu) + (w >> 16) : 0u;
  }
  const uint32_t wj = wp[jj];
  if (S & 1u) { s += wj & 0xFFFFu; paS = wj >> 16; }
  else paS = wj & 0xFFFFu;
  return s;
}

// f(a) >= f(b) for f = S / X^2: S_a X_b^2 >= S_b X_a^2, an f32 filter (each side within 2^-22) and u128 when close
__device__ __forceinline__ bool score_ge(uint32_t Sa, uint64_t Xa, uint32_t Sb, uint64_t Xb) {
  const float xa = (float)Xa, xb = (float)Xb;
  const float pa = (float)Sa * (xb * xb), pb = (float)Sb * (xa * xa);
  if (pa > pb * 1.00000095f) return true;    // 1 + 2^-20
  if (pa < pb * 0.99999905f) return false;   // 1 - 2^-20
  return (u128)Sa * ((u128)Xb * Xb) >= (u128)Sb * ((u128)Xa * Xa);
}

// Exact scan of the feasible widths (2X <= S F) from the converted row: the knee was infeasible (rare)
template <int SCAN_MEM>
static __device__ __noinline__ void lane_scan_pa(const uint32_t *H, const uint16_t *lmin, int S_tot, uint64_t C1,
                                                 uint64_t Mtp, uint64_t base, uint64_t D, uint32_t Wsm, uint64_t F,
                                                 uint32_t &Sb, uint64_t &Xb) {
  uint32_t ppa = 0;   // PPA(S) at the top of iteration S (PPA(1) = PA[0] = 0)
  float fb = 0.f;
  for (int S = 1; S <= S_tot; ++S) {
    const uint32_t hw = H[S >> 1];
    const uint32_t pa = (S & 1) ? (hw >> 16) : (hw & 0xFFFFu);
    uint64_t X = (uint64_t)S * C1 + Mtp * ((uint64_t)Wsm + ppa) + base;
    if (SCAN_MEM == 2) X += D * (uint64_t)(S * S);
    ppa += pa;
    if (!lmin[S] || 2 * X > (uint64_t)S * F) continue;
    lane_best((uint32_t)S, X, score_f((uint32_t)S, X), Sb, Xb, fb);
  }
}

// One f32 pass over the widths: per attained width S the score S / X(S, 1)^2 from an f32 evaluation of X
// (all terms non-negative: relative error < 2^-20, so only scores within 2^-19 of each other can be misordered),
// a top-3 tracker (t1 >= t2 >= t3, with the widths and PA / Q - W> values of the top 2), and the b >= 2
// certificate G over the segments m <= S_tot / 2.  The caller takes s1 when t2 < t1 (1 - 2^-17), decides s1 vs s2
// exactly when only t2 is that close (adjacent widths around a smooth maximum: ~4 % of DNNs), and rescans
// exactly (lane_scan) when t3 is too.
template <int SCAN_MEM>
__device__ __forceinline__ void lane_scan_f(const uint32_t *H, const uint16_t *lmin, int S_tot, int mh, bool all_valid,
                                            float C1f, float Mtpf, float basef, float Df, uint32_t Wsm, float C1f2,
                                            float Wbf, float membf, float half, float &t1, float &t2, float &t3,
                                            uint32_t &s1, uint32_t &ra1, uint32_t &q1, uint32_t &s2, float &G) {
  uint32_t ra = 0, rw = 0;
  // the same integers as floats, carried (all < 2^24, so every value is exact and equals (float) of the integer)
  float raf = 0.f, rwf = 0.f;
  const float Wsmf = (float)Wsm;
  float Sw = 0.f;   // 2 w
  const int nw = (S_tot + 2) >> 1;   // words holding bins 0..S_tot (bin S_tot + 1 of an even S_tot is 0)
#pragma unroll 2
  for (int w = 0; w < nw; ++w, Sw += 2.f) {
    const uint32_t hw = H[w];
#pragma unroll
    for (int hi = 0; hi < 2; ++hi) {
      const uint32_t S = (uint32_t)(2 * w + hi);   // S_tot + 1 (even S_tot): h = 0, lmin = 0 -> no candidate
      const uint32_t h = S == 0 ? 0u : (hi ? (hw >> 16) : (hw & 0xFFFFu));
      const float Sf = hi ? Sw + 1.f : Sw, hf = (float)h;
      ra += h; rw += h * S;
      raf += hf; rwf = fmaf(hf, Sf, rwf);
      const uint32_t q = Wsm - rw;
      const float qf = Wsmf - rwf;
      if ((int)S <= mh) {
        const float af = fmaf(Mtpf, raf, C1f2), bf = fmaf(Mtpf, qf + Wbf, membf);
        const float hiS = fminf(Sf + 1.f, half);
        const float sx = fminf(fmaxf(bf * rcp_approx(af), Sf), hiS);
        const float x = fmaf(af, sx, bf);
        G = fmaxf(G, bf == 0.f ? __int_as_float(0x7f800000) : sx * rcp_approx(x * x));
      }
      // widths that are no level's S(l) (and S = 0, S_tot + 1) score 0: a no-op for the tracker (f > t strict,
      // t1 >= t2 >= t3 >= 0), so the loop body has no data-dependent branch
      const bool cand = S != 0 && S <= (uint32_t)S_tot && (all_valid || lmin[S] != 0);
      float xf = fmaf(Sf, C1f, fmaf(Mtpf, fmaf(Sf, raf, qf), basef));
      if (SCAN_MEM == 2) xf = fmaf(Df, Sf * Sf, xf);
      const float f = cand ? Sf * rcp_approx(xf * xf) : 0.f;
      // top-3 of the scores (strict: the first width keeps a float tie), payloads of the top 2; branch-free
      // (lanes hold different DNNs, so a branch on f > t1 diverges)
      const uint32_t m1 = 0u - (uint32_t)(f > t1), m2 = 0u - (uint32_t)(f > t2);
      t3 = fmaxf(t3, fminf(t2, f));
      s2 = (s1 & m1) | (((S & m2) | (s2 & ~m2)) & ~m1);
      t2 = fmaxf(t2, fminf(t1, f));
      s1 = (S & m1) | (s1 & ~m1); ra1 = (ra & m1) | (ra1 & ~m1); q1 = (q & m1) | (q1 & ~m1);
      t1 = fmaxf(t1, f);
    }
  }
}

// QUEUE: DNNs outside the fast ranges are queued for k_prof_cold instead of analysed in place: a call inside the
// group loop would make the compiler distrust the warp's convergence everywhere in it (a divergence check at every
// collective); with the queue the loop has none.
template <bool QUEUE>
__global__ void __launch_bounds__(DSTACK_PLANE_WARPS * 32, DSTACK_PLANE_MINB) k_prof_lane(const __grid_constant__ ProfArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const dstack_problem_t &pb = a.pb;
  const dstack_params_t &p = a.p;
  const int L = p.L, S_tot = p.S_tot, mem_mode = p.mem_mode;
  uint16_t *Stab = (uint16_t *)smem;
  uint16_t *lmin = Stab + (L + 1);
  const int tab_bytes = ((L + 1 + S_tot + 1) * 2 + 15) & ~15;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int HS = plane_hstride(S_tot);
  unsigned char *wreg = smem + tab_bytes + (size_t)warp * plane_warp_bytes(S_tot);
  uint32_t *Htab = (uint32_t *)wreg;                       // [32][HS]
  uint64_t *cA = (uint64_t *)wreg;                          // cold path scratch (aliases Htab, used after the scans)
  uint64_t *cU = cA + (S_tot + 1);
  uint32_t *hist = (uint32_t *)(cU + (S_tot + 1));
  fill_stab(Stab, L, S_tot);
  for (int S = threadIdx.x; S <= S_tot; S += blockDim.x) {
    const int l = S == 0 ? 0 : ((S - 1) * L) / S_tot + 1;
    lmin[S] = (uint16_t)((S >= 1 && l <= L && s_of(l, S_tot, L) == S) ? l : 0);
  }
  __syncthreads();
  const int mh = S_tot >> 1;
  const float half = 0.5f * (float)S_tot;
  const int hwords = 32 * HS;
#if !DSTACK_PLANE_SEARCH
  const bool all_valid = L == S_tot;   // every width is some level's S(l)
#endif
  // groups of 32 DNNs from the work counter (one resident wave) or a grid stride over groups
  const int64_t gwarp = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp, nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t g = warp_next_item(a.work_ctr, -1, gwarp, nwarps, lane); g * 32 < pb.num_dnn;
       g = warp_next_item(a.work_ctr, g, gwarp, nwarps, lane)) {
    const int64_t kb = g * 32;
    const int nj = pb.num_dnn - kb < 32 ? (int)(pb.num_dnn - kb) : 32;
    const int64_t kl = kb + lane;
    const bool have = lane < nj;
    // ---- lane-parallel header: load + validate (DSTACK_ST_INVALID conditions, dstack.h) ----
    int64_t r0 = 0;
    int32_t K = 0, b_hi = 0;
    uint32_t M = 1, t_np = 0;
    uint64_t Mtp = 0, F = 0;
    bool ok = false;
    if (have) {
      r0 = pb.dnn_row_off[kl];
      const int64_t K64 = pb.dnn_row_off[kl + 1] - r0;
      const int32_t t_p = pb.t_p[kl], tnp = pb.t_np[kl], slo = pb.slo_us[kl], asm_us = pb.asm_us[kl];
      const int32_t bmax = pb.bmax[kl], mbw = pb.mem_bw[kl];
      ok = !(K64 < 1 || K64 > DSTACK_MAX_ROWS_PER_DNN || t_p < 1 || tnp < 0 || slo < 1 || slo > (1 << 30) ||
             (slo % p.slot_us) != 0 || asm_us < 0 || asm_us > (1 << 24) || bmax < 1 ||
             (p.mem_mode != 0 && (mbw < 1 || mbw > (1 << 24))));
      K = ok ? (int32_t)K64 : 0;
      M = p.mem_mode == 0 ? 1u : (uint32_t)mbw;
      t_np = (uint32_t)tnp;
      Mtp = (uint64_t)M * (uint32_t)t_p;
      // Eqs. 11-12 at b = 1 as one test 2X <= S F:  F = min(2 (SLO - a) M, SLO M)  (0 if a > SLO)
      const uint64_t SLOM = (uint64_t)slo * M, aM = (uint64_t)asm_us * M;
      F = SLOM < aM ? 0ull : (2 * (SLOM - aM) < SLOM ? 2 * (SLOM - aM) : SLOM);
      b_hi = bmax < p.b_max ? bmax : p.b_max;
    }
    // ---- zero the 32 histogram rows (16-byte stores) ----
    {
      uint4 *hz = reinterpret_cast<uint4 *>(Htab);
      // warp-uniform loops (lane-dependent trip counts would make the compiler distrust convergence afterwards)
      for (int i0 = 0; i0 < (hwords >> 2); i0 += 32)
        if (i0 + lane < (hwords >> 2)) hz[i0 + lane] = make_uint4(0u, 0u, 0u, 0u);
      if ((hwords & ~3) + lane < hwords) Htab[(hwords & ~3) + lane] = 0u;
    }
    __syncwarp();
    // ---- a1: row pass, one DNN after the other (coalesced), results to the owning lane; the first
    //      32 * DSTACK_PROF_ROWS_U rows of the next DNN are loaded while the current one is reduced ----
    constexpr int U = DSTACK_PROF_ROWS_U;
    uint32_t myRT = 0, myRmin = 0, myWsm = 0, myDtop = 0, myWtop = 0;
    uint64_t myD = 0, myWb = 0;
    uint32_t cn[U], cd[U], cr[U], pn[U], pd[U], pr[U];
    auto load_batch = [&](int64_t rb, int32_t Kb, int i0, uint32_t *bn, uint32_t *bd, uint32_t *br) {
      const uint32_t *np = pb.n + rb + i0;
      const uint32_t *dp = pb.d + rb + i0;
      const uint16_t *rp = pb.r + rb + i0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        bn[u] = 0; bd[u] = 0; br[u] = 0;
        if (i0 + 32 * u < Kb) { bn[u] = __ldg(np + 32 * u); bd[u] = __ldg(dp + 32 * u); br[u] = __ldg(rp + 32 * u); }
      }
    };
    // row counts broadcast by a reduction (not a shuffle): warp-uniform to the compiler, so the row loops bounded by
    // them carry no divergence checks (K >= 0)
    int32_t Kc = (int32_t)__reduce_max_sync(FULL, lane == 0 ? (uint32_t)K : 0u);
    int64_t rc = nj > 0 ? (int64_t)shfl_u64((uint64_t)r0, 0) : 0;
    load_batch(rc, Kc, lane, cn, cd, cr);
    for (int jj = 0; jj < nj; ++jj) {
      const int32_t Kn = (int32_t)__reduce_max_sync(FULL, lane == jj + 1 ? (uint32_t)K : 0u);   // 0 past the group
      const int64_t rn = jj + 1 < nj ? (int64_t)shfl_u64((uint64_t)r0, jj + 1) : 0;
      load_batch(rn, Kn, lane, pn, pd, pr);   // prefetch (predicated off past the group / for invalid DNNs)
      if (Kc > 0) {
        uint32_t *Hj = Htab + jj * HS;
        uint32_t RT = 0, Rmin = 0xFFFFFFFFu, Wsm = 0;
        uint64_t D = 0, Wb = 0;
        auto accum = [&](const uint32_t *bn, const uint32_t *bd, const uint32_t *br, int i0) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if (i0 + 32 * u < Kc) {
              RT += br[u]; D += (uint64_t)br[u] * bd[u]; Rmin = min(Rmin, br[u]);
              if (bn[u] <= (uint32_t)S_tot) {
                atomicAdd(&Hj[bn[u] >> 1], br[u] << ((bn[u] & 1u) << 4));
                Wsm += br[u] * bn[u];
              } else {
                Wb += (uint64_t)br[u] * bn[u];
              }
            }
          }
        };
        accum(cn, cd, cr, lane);
        for (int b0 = 32 * U; b0 < Kc; b0 += 32 * U) {   // rows beyond the prefetched batch (a warp-uniform loop)
          uint32_t tn[U], td[U], tr[U];
          load_batch(rc, Kc, b0 + lane, tn, td, tr);
          accum(tn, td, tr, b0 + lane);
        }
        RT = __reduce_add_sync(FULL, RT);
        Rmin = __reduce_min_sync(FULL, Rmin);
        Wsm = __reduce_add_sync(FULL, Wsm);
        uint32_t Dtop, Wtop;
        D = warp_sum_limbs(D, &Dtop);
        Wb = warp_sum_limbs(Wb, &Wtop);
        if (lane == jj) { myRT = RT; myRmin = Rmin; myWsm = Wsm; myD = D; myWb = Wb; myDtop = Dtop; myWtop = Wtop; }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) { cn[u] = pn[u]; cd[u] = pd[u]; cr[u] = pr[u]; }
      Kc = Kn; rc = rn;
    }
    __syncwarp();
    // ---- a2/a3 for this lane's DNN ----
    uint32_t st = ok ? DSTACK_ST_OK : DSTACK_ST_INVALID, knee = 0, demand = 0, dslots = 0;
    bool cold = false;
    if (have && ok) {
      // status (same order as the generic path); the fast ranges (else the generic path decides)
      if (myRmin == 0 || (t_np == 0 && myWb == 0 && myWtop == 0 && myWsm == 0 &&
                          (mem_mode == 0 || (myD == 0 && myDtop == 0)))) {
        st = DSTACK_ST_INVALID;
      } else if (b_hi < 1) {
        st = DSTACK_ST_INFEASIBLE;
      } else if (myRT >= (1u << 16) || myWtop >= (1u << 19) || myDtop >= (1u << 19)) {
        cold = true;
      } else {
        // overflow: X(L, b_hi) <= b_hi t_np RT S_tot M + Mtp (S_tot RT + b_hi (W> + Wsm)) + mem bounds every cell;
        // within 1e-4 of 2^56 the generic path decides exactly
        const double bd = (double)b_hi, Sd = (double)S_tot;
        double xe = bd * (double)t_np * (double)M * (double)myRT * Sd +
                    (double)Mtp * (Sd * (double)myRT + bd * ((double)myWb + (double)myWsm));
        if (mem_mode == 1) xe += bd * (double)myD;
        else if (mem_mode == 2) xe += bd * (double)myD * Sd * Sd;
        if (xe >= 72057594037927936.0 * 0.9999) cold = true;
      }
    }
#if DSTACK_PLANE_SEARCH
    // a2/a3 by search on every lane (uniform trip counts; lanes without a fast-path DNN search their own zero or
    // partial row and drop the result)
    const uint64_t C1 = (uint64_t)t_np * M * myRT;
    const uint64_t memb = mem_mode == 1 ? myD : 0ull;
    const uint64_t base = Mtp * myWb + memb;
    const float C1f2 = 2.f * (float)C1, Mtpf = (float)Mtp, Wbf = (float)myWb, membf = (float)memb;
    const int nw = plane_nw(S_tot);
    lane_prefix(Htab + lane * HS, nw, plane_nck(S_tot));
    const uint32_t *H = Htab + lane * HS;
    auto x_of = [&](uint32_t S, uint32_t ppa) {   // X(S, 1) from PPA(S)
      uint64_t X = (uint64_t)S * C1 + Mtp * ((uint64_t)myWsm + ppa) + base;
      if (mem_mode == 2) X += myD * (uint64_t)(S * S);
      return X;
    };
    // knee: the leftmost maximum of S / X^2 over the candidates i = 1..N (widths i when every width is some level's
    // S(l), i.e. L >= S_tot; else S(i) = Stab[i], strictly increasing)
    const bool dense = L >= S_tot;
    const int N = dense ? S_tot : L;
    int ilo = 1, ihi = N;
    const int ksteps = N > 1 ? 32 - __clz(N - 1) : 0;
    for (int it = 0; it < ksteps; ++it) {
      const int mid = (ilo + ihi) >> 1;
      const uint32_t Sa = dense ? (uint32_t)mid : Stab[mid];
      uint32_t paA, ppaB;
      const uint32_t ppaA = lane_ppa(H, nw, Sa, paA);
      uint32_t Sb2;
      if (dense) { Sb2 = Sa + 1; ppaB = ppaA + paA; }
      else { Sb2 = Stab[mid + 1 <= N ? mid + 1 : N]; uint32_t t; ppaB = lane_ppa(H, nw, Sb2, t); }
      const bool left = score_ge(Sa, x_of(Sa, ppaA), Sb2, x_of(Sb2, ppaB));
      if (ilo < ihi) { if (left) ihi = mid; else ilo = mid + 1; }
    }
    uint32_t Sk = dense ? (uint32_t)ilo : Stab[ilo];
    uint64_t Xk;
    { uint32_t t; Xk = x_of(Sk, lane_ppa(H, nw, Sk, t)); }
    // certificate G: the closed-form supremum on the first segment m <= S_tot / 2 with alpha_m (m + 1) >= beta_m
    float G;
    {
      int mlo = 0, mhi = mh;
      const int csteps = mh > 0 ? 32 - __clz(mh) : 0;
      const uint64_t C12 = 2 * C1;
      for (int it = 0; it < csteps; ++it) {
        const int mid = (mlo + mhi) >> 1;
        uint32_t pam;
        const uint32_t ppam = lane_ppa(H, nw, (uint32_t)mid, pam);
        const uint32_t Qm = myWsm - (uint32_t)mid * pam + ppam;   // Q[m] = Wsm - PW[m]
        const uint64_t alpha = C12 + Mtp * pam, beta = Mtp * ((uint64_t)Qm + myWb) + memb;
        const bool peak_by = alpha * (uint64_t)(mid + 1) >= beta;
        if (mlo < mhi) { if (peak_by) mhi = mid; else mlo = mid + 1; }
      }
      uint32_t pam;
      const uint32_t ppam = lane_ppa(H, nw, (uint32_t)mlo, pam);
      const uint32_t Qm = myWsm - (uint32_t)mlo * pam + ppam;
      const float af = fmaf(Mtpf, (float)pam, C1f2), bf = fmaf(Mtpf, (float)Qm + Wbf, membf);
      const float Sf = (float)mlo, hiS = fminf(Sf + 1.f, half);
      const float sx = fminf(fmaxf(bf * rcp_approx(af), Sf), hiS);
      const float x = fmaf(af, sx, bf);
      G = bf == 0.f ? __int_as_float(0x7f800000) : sx * rcp_approx(x * x);
    }
    if (have && ok) {
      if (st == DSTACK_ST_OK && !cold) {
        // knee = the exact argmax over every attained width; when it is feasible (Eqs. 11-12: 2X <= S F) it is
        // also the feasible argmax, else the feasible widths are scanned exactly
        uint32_t Se = 0;
        uint64_t Xe = 0;
        if (F != 0 && 2 * Xk <= (uint64_t)Sk * F) { Se = Sk; Xe = Xk; }
        else {   // (F = 0: no width is feasible; scanned with F = 1 exactly as the generic fast path does)
          const uint64_t F1 = F == 0 ? 1ull : F;
          if (mem_mode == 2) lane_scan_pa<2>(H, lmin, S_tot, C1, Mtp, base, myD, myWsm, F1, Se, Xe);
          else lane_scan_pa<0>(H, lmin, S_tot, C1, Mtp, base, myD, myWsm, F1, Se, Xe);
        }
        if (Se == 0) {
          st = DSTACK_ST_INFEASIBLE;   // b = 1 is feasible whenever any b is (O3)
        } else if (b_hi >= 2 && !(score_f(Se, Xe) * 0.99975586f > G)) {
          cold = true;   // b* = 1 not certified: the generic exact branch-and-bound decides
        } else {
          knee = lmin[Sk];
          const uint32_t le = lmin[Se];
          demand = le + (uint32_t)p.margin < (uint32_t)L ? le + (uint32_t)p.margin : (uint32_t)L;
          if (a.dtab_rows) {   // d_j(1) = ceil(X(S(g), 1) / (S(g) M Delta)) at g = demand
            const uint32_t Sg = Stab[demand];
            uint32_t t;
            const uint64_t Xg = Sg == Se ? Xe : x_of(Sg, lane_ppa(H, nw, Sg, t));
            dslots = ceil_div_clamp16_fast(Xg, (uint64_t)Sg * M * (uint64_t)p.slot_us);
          }
        }
      }
    }
#else
    // The f32 width scan runs on every lane, outside any lane-dependent branch: its branches on the width are then
    // provably warp-uniform (no reconvergence regions in the loop).  Lanes without a fast-path DNN scan their
    // (zero or partial) histogram row with their own parameters and drop the result.
    const uint64_t C1 = (uint64_t)t_np * M * myRT;
    const uint64_t memb = mem_mode == 1 ? myD : 0ull;
    const uint64_t base = Mtp * myWb + memb;
    const float C1f2 = 2.f * (float)C1, Mtpf = (float)Mtp, Wbf = (float)myWb, membf = (float)memb;
    const uint32_t *H = Htab + lane * HS;
    uint32_t Sk = 0, ra1 = 0, q1 = 0, s2 = 0;
    float t1 = 0.f, t2 = 0.f, t3 = 0.f, G = 0.f;
    {
      const float C1f = (float)C1, basef = (float)base, Df = (float)myD;
      if (mem_mode == 2) lane_scan_f<2>(H, lmin, S_tot, mh, all_valid, C1f, Mtpf, basef, Df, myWsm, C1f2, Wbf, membf, half, t1, t2, t3, Sk, ra1, q1, s2, G);
      else lane_scan_f<0>(H, lmin, S_tot, mh, all_valid, C1f, Mtpf, basef, Df, myWsm, C1f2, Wbf, membf, half, t1, t2, t3, Sk, ra1, q1, s2, G);
    }
    if (have && ok) {
      if (st == DSTACK_ST_OK && !cold) {
        uint64_t Xk = 0;
        const float band = t1 * 0.99999237f;   // 1 - 2^-17 (twice the worst f32 misordering)
        auto x_at = [&](uint32_t S, uint32_t ra, uint32_t q) {
          uint64_t X = (uint64_t)S * C1 + Mtp * ((uint64_t)S * ra + q) + base;
          if (mem_mode == 2) X += myD * (uint64_t)(S * S);
          return X;
        };
        if (t3 >= band) {   // three widths within the band (rare): exact rescan
          float fk = 0.f, Gd = 0.f;
          Sk = 0;
          if (mem_mode == 2) lane_scan<2>(H, lmin, S_tot, mh, C1, Mtp, base, myD, myWsm, F, true, C1f2, Mtpf, Wbf, membf, half, Sk, Xk, fk, Gd, false);
          else lane_scan<0>(H, lmin, S_tot, mh, C1, Mtp, base, myD, myWsm, F, true, C1f2, Mtpf, Wbf, membf, half, Sk, Xk, fk, Gd, false);
        } else {
          Xk = x_at(Sk, ra1, q1);
          if (t2 >= band) {   // s1 vs s2 exactly: larger S / X^2, ties -> the smaller width
            const uint64_t X2 = lane_X_at(H, s2, C1, Mtp, base, myD, myWsm, mem_mode);
            const u128 l1 = (u128)Sk * ((u128)X2 * X2), l2 = (u128)s2 * ((u128)Xk * Xk);
            if (l2 > l1 || (l2 == l1 && s2 < Sk)) { Sk = s2; Xk = X2; }
          }
        }
        // knee = the exact argmax over every attained width; when it is feasible (Eqs. 11-12: 2X <= S F) it is
        // also the feasible argmax, else the feasible widths are scanned again
        uint32_t Se = 0;
        uint64_t Xe = 0;
        if (F != 0 && 2 * Xk <= (uint64_t)Sk * F) { Se = Sk; Xe = Xk; }
        else {   // (F = 0: no width is feasible; scanned with F = 1 exactly as the generic fast path does)
          const uint64_t F1 = F == 0 ? 1ull : F;
          float fe = 0.f, Gd = 0.f;
          if (mem_mode == 2) lane_scan<2>(H, lmin, S_tot, mh, C1, Mtp, base, myD, myWsm, F1, true, C1f2, Mtpf, Wbf, membf, half, Se, Xe, fe, Gd, true);
          else lane_scan<0>(H, lmin, S_tot, mh, C1, Mtp, base, myD, myWsm, F1, true, C1f2, Mtpf, Wbf, membf, half, Se, Xe, fe, Gd, true);
        }
        if (Se == 0) {
          st = DSTACK_ST_INFEASIBLE;   // b = 1 is feasible whenever any b is (O3)
        } else if (b_hi >= 2 && !(score_f(Se, Xe) * 0.99975586f > G)) {
          cold = true;   // b* = 1 not certified: the generic exact branch-and-bound decides
        } else {
          knee = lmin[Sk];
          const uint32_t le = lmin[Se];
          demand = le + (uint32_t)p.margin < (uint32_t)L ? le + (uint32_t)p.margin : (uint32_t)L;
          if (a.dtab_rows) {   // d_j(1) = ceil(X(S(g), 1) / (S(g) M Delta)) at g = demand
            const uint32_t Sg = Stab[demand];
            const uint64_t Xg = Sg == Se ? Xe : lane_X_at(H, Sg, C1, Mtp, base, myD, myWsm, mem_mode);
            dslots = ceil_div_clamp16_fast(Xg, (uint64_t)Sg * M * (uint64_t)p.slot_us);
          }
        }
      }
    }
#endif
    // ---- outputs of the lanes' DNNs (coalesced: lane j writes DNN kb + j) ----
    if (have && !cold) {
      const bool okst = st == DSTACK_ST_OK;
      if (a.ws_RT) { a.ws_RT[kl] = myRT; a.ws_D[kl] = myD; }
      if (okst) {
        if (a.dstar) a.dstar[kl] = (uint16_t)dslots;
        else if (a.dtab_rows) a.dtab_rows[kl * DTAB_ROW] = (uint16_t)dslots;
      }
      if (a.knee) a.knee[kl] = okst ? (uint16_t)knee : 0;
      if (a.status) a.status[kl] = (uint8_t)st;
      if (a.demand) a.demand[kl] = okst ? (uint16_t)demand : 0;
      if (a.batch) a.batch[kl] = okst ? 1 : 0;
    }
    // ---- the generic path for the DNNs outside the fast ranges ----
    if (QUEUE) {
      if (have && cold) a.cold_q[2 + atomicAdd(a.cold_q, 1u)] = (uint32_t)kl;
    } else {
      uint32_t colds = __ballot_sync(FULL, have && cold);
      if (colds) {   // the cold path expects a zeroed hist (its scratch overlays the H table)
        __syncwarp();
        for (int m = lane; m <= S_tot; m += 32) hist[m] = 0;
        __syncwarp();
      }
      while (colds) {
        const int j = __ffs(colds) - 1;
        colds &= colds - 1;
        prof_one_cold(&a, kb + j, Stab, hist, cA, cU, lane);
      }
    }
    __syncwarp();
  }
}

// The DNNs k_prof_lane<true> queued (outside its fast ranges, or b* = 1 not certified): the generic exact analysis,
// one warp per DNN pulled from the queue (usually none: the warps read the count and exit).
__global__ void __launch_bounds__(256) k_prof_cold(const __grid_constant__ ProfArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int L = a.p.L, S_tot = a.p.S_tot;
  uint16_t *Stab = (uint16_t *)smem;
  const int tab_bytes = ((L + 1 + S_tot + 1) * 2 + 15) & ~15;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t n = a.cold_q[0];
  if (n == 0) return;
  unsigned char *wreg = smem + tab_bytes + (size_t)warp * prof_warp_bytes(S_tot);
  uint64_t *cA = (uint64_t *)wreg;
  uint64_t *cU = cA + (S_tot + 1);
  uint32_t *hist = (uint32_t *)(cU + (S_tot + 1));
  fill_stab(Stab, L, S_tot);
  for (int m = lane; m <= S_tot; m += 32) hist[m] = 0;
  __syncthreads();
  for (;;) {
    uint32_t i = 0;
    if (lane == 0) i = atomicAdd(a.cold_q + 1, 1u);
    i = __shfl_sync(FULL, i, 0);
    if (i >= n) break;
    prof_one_cold(&a, (int64_t)a.cold_q[2 + i], Stab, hist, cA, cU, lane);
  }
}

size_t prof_smem_bytes(const dstack_params_t *p, int warps) {
  return (size_t)(((p->L + 1 + p->S_tot + 1) * 2 + 15) & ~15) + (size_t)warps * prof_warp_bytes(p->S_tot) +
         (size_t)warps * FAST_STAGE_BYTES;
}
size_t plane_smem_bytes(const dstack_params_t *p, int warps) {
  return (size_t)(((p->L + 1 + p->S_tot + 1) * 2 + 15) & ~15) + (size_t)warps * plane_warp_bytes(p->S_tot);
}

template <typename KernelT>
static void launch_k(KernelT kern, const ProfArgs &a, int64_t blocks, int threads, size_t smem, cudaStream_t s) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<(unsigned)blocks, threads, smem, s>>>(a);
}

int launch_prof(const ProfArgs &a, cudaStream_t s, int *launches) {
  if (a.pb.num_dnn <= 0) return 0;
  const int threads = 256, warps = threads / 32;
  const size_t smem = prof_smem_bytes(&a.p, warps);
  int64_t blocks = (a.pb.num_dnn + warps - 1) / warps;
  const int64_t cap = (int64_t)num_sms() * DSTACK_PROF_GRID;
  if (blocks > cap) blocks = cap;
  const bool fast = DSTACK_PROF_FAST && a.p.par_mode == 0 && a.p.wse_mode == 0 && a.p.b_min == 1 && !a.knee_only;
  ProfArgs b = a;
  if (!DSTACK_PROF_DYN) b.work_ctr = nullptr;
  if (b.work_ctr) {   // one resident wave (DSTACK_PROF_MINB blocks per SM) pulling groups of 32 DNNs (fast) or DNNs
    if (cudaMemsetAsync(b.work_ctr, 0, sizeof(uint32_t), s) != cudaSuccess) return DSTACK_ELAUNCH;
    const int64_t wave = (int64_t)num_sms() * DSTACK_PROF_MINB;
    if (blocks > wave) blocks = wave;
  }
  if (fast && DSTACK_PROF_LANE) {
    // k_prof_lane: one resident wave of warps pulling groups of 32 DNNs (grid stride over groups without a counter)
    const int pw = DSTACK_PLANE_WARPS;
    const size_t sm2 = plane_smem_bytes(&a.p, pw);
    const int64_t groups = (a.pb.num_dnn + 31) / 32;
    int64_t nb = (groups + pw - 1) / pw;
    if (b.cold_q) {
      cudaFuncSetAttribute(k_prof_lane<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
      const int64_t wave = resident_wave(k_prof_lane<true>, pw * 32, sm2, nb);
      if (b.work_ctr || nb > wave) nb = wave;
      if (cudaMemsetAsync(b.cold_q, 0, 2 * sizeof(uint32_t), s) != cudaSuccess) return DSTACK_ELAUNCH;
      k_prof_lane<true><<<(unsigned)nb, pw * 32, sm2, s>>>(b);
      const size_t smc = (size_t)(((a.p.L + 1 + a.p.S_tot + 1) * 2 + 15) & ~15) + 8 * prof_warp_bytes(a.p.S_tot);
      cudaFuncSetAttribute(k_prof_cold, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smc);
      k_prof_cold<<<(unsigned)num_sms(), 256, smc, s>>>(b);
      ++*launches;
    } else {
      cudaFuncSetAttribute(k_prof_lane<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
      const int64_t wave = resident_wave(k_prof_lane<false>, pw * 32, sm2, nb);
      if (b.work_ctr || nb > wave) nb = wave;
      k_prof_lane<false><<<(unsigned)nb, pw * 32, sm2, s>>>(b);
    }
  } else if (fast && a.p.S_tot < 5 * 32) launch_k(k_prof_fast<5>, b, blocks, threads, smem, s);
  else if (fast) launch_k(k_prof_fast<9>, b, blocks, threads, smem, s);
  else if (a.p.par_mode == 0) launch_k(k_prof<0>, b, blocks, threads, smem, s);
  else launch_k(k_prof<1>, b, blocks, threads, smem, s);
  ++*launches;
  return cudaGetLastError() == cudaSuccess ? 0 : DSTACK_ELAUNCH;
}

int launch_knee_probe(const ProfArgs &a, cudaStream_t s, int *launches) {
  if (a.pb.num_dnn <= 0) return 0;
  const int threads = 256, warps = threads / 32;
  const size_t smem = prof_smem_bytes(&a.p, warps);
  int64_t blocks = (a.pb.num_dnn + warps - 1) / warps;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  ProfArgs b = a;
  if (!DSTACK_PROF_DYN) b.work_ctr = nullptr;
  if (b.work_ctr) {
    if (cudaMemsetAsync(b.work_ctr, 0, sizeof(uint32_t), s) != cudaSuccess) return DSTACK_ELAUNCH;
    const int64_t wave = (int64_t)num_sms() * DSTACK_PROF_MINB;
    if (blocks > wave) blocks = wave;
  }
  if (a.p.par_mode == 0) launch_k(k_prof<0>, b, blocks, threads, smem, s);
  else launch_k(k_prof<1>, b, blocks, threads, smem, s);
  ++*launches;
  return cudaGetLastError() == cudaSuccess ? 0 : DSTACK_ELAUNCH;
}

}  // namespace dstack

#if DSTACK_PROF_STATS
extern "C" int dstack_debug_stats(unsigned long long *out16, int reset) {
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(out16, dstack::g_pstats, sizeof(unsigned long long) * 16) != cudaSuccess) return -1;
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(dstack::g_pstats, z, sizeof(z));
  }
  return 0;
}
#endif
