// prof.cuh -- a1-a3 device code: one warp analyses one DNN (knee, batch/GPU% search).
//
// Data path per DNN (warp-cooperative):
//  1. one coalesced pass over the kernel rows (n u32, R u16, d u32): totals RT, D, sum R*n, the
//     overflow bound X(L, b_hi), and (linear mode) a shared-memory histogram of R and R*n over the
//     widths n <= S_tot;
//  2. a chunked warp scan turns the histogram into the coefficient tables
//        cA[m] = M t_p sum_{1<=n_i<=m} R_i,   cU[m] = M t_p sum_{n_i>m} R_i n_i
//     so X(l,b) = S*(w_b*C1 + cA[m]) + b*cU[m] + mem, m = floor(S/b), in O(1) per cell;
//  3. EXACT branch-and-bound for argmax eta = b S / X^2 over feasible (l, b) (Eqs. 9-12):
//     the b_lo row is evaluated exactly (it is feasible whenever any row is: f_L and C grow with b);
//     every other b is first bounded by a Jensen relaxation (X >= w_b C1 S + M t_p max(S RT1, b Wn)),
//     then per run of constant m = floor(S/b) by the continuous supremum of b S/(alpha S + beta)^2,
//     and only rows whose bound reaches the incumbent are evaluated exactly.  Bounds use f64 with a
//     1e-9 safety margin; every decision between candidates is exact (float filter + 128-bit products).
//     Threads mode (N_i(b) = ceil(b theta/2048)) rebuilds the tables per b and evaluates every row.
//  4. the knee (Eq. 6) at b* is the unconstrained argmax of the b* row, tracked during its evaluation.
#pragma once
#include "common.cuh"

namespace dstack {

// Optional instrumentation build (-DDSTACK_PROF_STATS=1, never the default library): event counters of the
// branch-and-bound, read back by dstack_debug_stats().
#ifndef DSTACK_PROF_STATS
#define DSTACK_PROF_STATS 0
#endif
#if DSTACK_PROF_STATS
static __device__ unsigned long long g_pstats[16];   // per TU; k_prof's copy is prof.cu's
#define PSTAT(i, v) atomicAdd(&g_pstats[i], (unsigned long long)(v))
#else
#define PSTAT(i, v) ((void)0)
#endif

#ifndef DSTACK_GEN_ROWS_U
#define DSTACK_GEN_ROWS_U 6   // rows per lane in flight in the generic row pass (A/B knee probe: 2 -> 34.6, 4 -> 34.4, 6 -> 33.1 ms)
#endif

struct Best {
  uint32_t found, l, b, S;
  uint64_t X;
  float sc;        // float score b S / X^2 (filter only)
};

__device__ __forceinline__ Best best_none() {
  Best r; r.found = 0; r.l = 0; r.b = 0; r.S = 0; r.X = 0; r.sc = 0.f;
  return r;
}

// exact comparison of two candidates whose float scores are within the filter tolerance (rare)
static __device__ __noinline__ bool better_exact(uint32_t cb, uint32_t cS, uint64_t cX, uint32_t cl, uint32_t ob, uint32_t oS,
                                          uint64_t oX, uint32_t ol) {
  PSTAT(4, 1);
  const u128 L = (u128)(cb * cS) * ((u128)oX * oX);
  const u128 R = (u128)(ob * oS) * ((u128)cX * cX);
  if (L != R) return L > R;
  return cl < ol || (cl == ol && cb < ob);
}

// exact total order: higher eta = b S / X^2, then smaller l, then smaller b
__device__ __forceinline__ bool better(const Best &c, const Best &o) {
  if (!c.found) return false;
  if (!o.found) return true;
  if (c.sc > o.sc * 1.0000077f) return true;    // 1 + 2^-17
  if (o.sc > c.sc * 1.0000077f) return false;
  return better_exact(c.b, c.S, c.X, c.l, o.b, o.S, o.X, o.l);
}

__device__ __forceinline__ float score_f(uint32_t P, uint64_t X) {
  const float xf = (float)X;
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(xf * xf));
  return (float)P * r;   // relative error < 2^-21: far inside the 2^-17 filter band
}

__device__ __forceinline__ Best shfl_best(const Best &v, int src) {
  Best o;
  const uint32_t packed = (v.found << 31) | (v.b << 24) | (v.l << 12) | v.S;   // l <= 255, S <= 256 (< 4096), b <= 64
  const uint32_t pk = __shfl_sync(FULL, packed, src);
  o.found = pk >> 31; o.b = (pk >> 24) & 127; o.l = (pk >> 12) & 4095; o.S = pk & 4095;
  o.X = shfl_u64(v.X, src);
  o.sc = __shfl_sync(FULL, v.sc, src);
  return o;
}

static __device__ __noinline__ Best warp_best_exact(Best v) {
  if ((threadIdx.x & 31) == 0) PSTAT(5, 1);
#pragma unroll 1
  for (int m = 16; m; m >>= 1) {
    Best o = shfl_best(v, (threadIdx.x & 31) ^ m);
    if (better(o, v)) v = o;
  }
  return v;
}

// warp argmax: float max + uniqueness test decides almost always; exact butterfly otherwise
__device__ __forceinline__ Best warp_best(Best v) {
  const uint32_t sb = v.found ? __float_as_uint(v.sc) : 0u;
  const uint32_t mx = __reduce_max_sync(FULL, sb);
  if (mx == 0) return best_none();
  const float thr = __uint_as_float(mx) * 0.9999847f;   // 1 - 2^-16
  const uint32_t near = __ballot_sync(FULL, v.found && v.sc >= thr);
  if (__popc(near) == 1) return shfl_best(v, __ffs(near) - 1);
  return warp_best_exact(v);
}

struct DnnRes {
  uint8_t st;
  uint16_t demand, knee;
  uint8_t b;
  uint64_t RT, D;
};

template <int PAR>
__device__ __forceinline__ uint64_t cell_X(int32_t S, int32_t b, uint32_t magic, uint64_t wC1, const uint64_t *cA,
                                           const uint64_t *cU, int mem_mode, uint64_t D) {
  int32_t m;
  uint64_t ub;
  if (PAR == 0) { m = (b == 1) ? S : (int32_t)__umulhi((uint32_t)S, magic); ub = (uint64_t)b; }
  else { m = S; ub = 1; }
  uint64_t X = (uint64_t)S * (wC1 + cA[m]) + ub * cU[m];
  if (mem_mode == 1) X += (uint64_t)b * D;
  else if (mem_mode == 2) X += (uint64_t)b * D * (uint64_t)S * (uint64_t)S;
  return X;
}

__device__ __forceinline__ uint32_t magic_of(int32_t b) { return b == 1 ? 0u : (uint32_t)(0xFFFFFFFFu / (uint32_t)b) + 1u; }

// Warp scan of the width histogram hist[0..S_tot] (u32 sums of R_i by n_i) into the SCALED tables
//   cA[m] = Mtp * PA[m], PA[m] = sum_{1<=n<=m} R;   cU[m] = Mtp * Q[m], Q[m] = W - sum_{n<=m} n R
// (lane-chunked, one shuffle scan).  Returns the unscaled PA[mb], Q[mb] in *pa_mb, *q_mb (all lanes).
__device__ __forceinline__ void scan_hist(const uint32_t *hist, uint64_t *cA, uint64_t *cU, int S_tot, uint64_t W,
                                          uint64_t Mtp, int mb, uint64_t *pa_mb, uint64_t *q_mb, int lane) {
  __syncwarp();
  const int C = (S_tot + 32) >> 5;          // bins per lane (S_tot+1 bins)
  const int m0 = lane * C;
  uint64_t sa = 0, sw = 0;
  for (int i = 0; i < C; ++i) {
    const int m = m0 + i;
    if (m <= S_tot && m >= 1) { const uint64_t h = hist[m]; sa += h; sw += h * (uint64_t)m; }
  }
  uint64_t pa = sa, pw = sw;   // inclusive scan of lane totals
  DSTACK_UNROLL_SMALL
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t ua = shfl_up_u64(pa, d), uw = shfl_up_u64(pw, d);
    if (lane >= d) { pa += ua; pw += uw; }
  }
  pa -= sa; pw -= sw;          // exclusive
  uint64_t a_mb = 0, q_m = 0;
  for (int i = 0; i < C; ++i) {
    const int m = m0 + i;
    if (m <= S_tot) {
      if (m >= 1) { const uint64_t h = hist[m]; pa += h; pw += h * (uint64_t)m; }
      cA[m] = Mtp * pa; cU[m] = Mtp * (W - pw);
      if (m == mb) { a_mb = pa; q_m = W - pw; }
    }
  }
  const int owner = mb / C;
  *pa_mb = shfl_u64(a_mb, owner);
  *q_mb = shfl_u64(q_m, owner);
  __syncwarp();
}

// threads mode: tables of N = ceil(b theta / 2048) (rebuilt per b)
__device__ __forceinline__ void build_tables_threads(const uint32_t *__restrict__ n, const uint16_t *__restrict__ r,
                                                     int32_t K, int32_t S_tot, uint64_t Mtp, int32_t b,
                                                     uint32_t *hist, uint64_t *cA, uint64_t *cU, int lane) {
  for (int m = lane; m <= S_tot; m += 32) hist[m] = 0;
  __syncwarp();
  uint64_t W = 0;
  for (int i = lane; i < K; i += 32) {
    const uint64_t N = ((uint64_t)b * n[i] + 2047) >> 11;
    const uint32_t R = r[i];
    W += (uint64_t)R * N;
    if (N <= (uint64_t)S_tot) atomicAdd(&hist[N], R);
  }
  W = warp_sum_u64(W);
  uint64_t pa, q;
  scan_hist(hist, cA, cU, S_tot, W, Mtp, 0, &pa, &q, lane);
}

struct RowCtx {
  const uint16_t *Stab;
  const uint64_t *cA, *cU;
  int32_t L, mem_mode, wse;
  uint64_t C1, D, SLOM, aM;
};

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// Row b: feasible argmax (e) and unconstrained argmax (k) of b S / X^2 over the levels, warp-reduced,
// exact (per level: O(1) X from the tables, f32 score filter, 128-bit comparison only on near-ties).
template <int PAR>
__device__ __forceinline__ void eval_row(const RowCtx &c, int32_t b, int lane, Best &e, Best &k) {
  const uint32_t magic = magic_of(b);
  const uint64_t wC1 = (c.wse == 0 ? (uint64_t)b : 1ull) * c.C1;
  const uint64_t baM = (uint64_t)b * c.aM;
  e = best_none(); k = best_none();
  for (int32_t l = 1 + lane; l <= c.L; l += 32) {
    const int32_t S = c.Stab[l];
    const uint64_t X = cell_X<PAR>(S, b, magic, wC1, c.cA, c.cU, c.mem_mode, c.D);
    Best cand; cand.found = 1; cand.l = l; cand.b = b; cand.S = S; cand.X = X; cand.sc = score_f(b * S, X);
    if (better(cand, k)) k = cand;
    const uint64_t cap = (uint64_t)S * c.SLOM;
    if (X + (uint64_t)S * baM <= cap && 2 * X <= cap && better(cand, e)) e = cand;   // Eq. 11, Eq. 12
  }
  e = warp_best(e);
  k = warp_best(k);
}

// exact X(L, b_eval) >= 2^56 test (only when the f64 estimate is within 1e-4 of the limit)
static __device__ __noinline__ bool xub_exact_over(uint32_t w, uint64_t t_np, uint64_t RT, uint32_t S_tot, uint64_t M,
                                            uint64_t t_p, uint64_t Vmax, int mem_mode, uint32_t b, uint64_t D) {
  u128 Xub = (u128)w * t_np * RT * S_tot * M + (u128)M * t_p * Vmax;
  if (mem_mode == 1) Xub += (u128)b * D;
  else if (mem_mode == 2) Xub += (u128)b * D * (u128)(S_tot * S_tot);
  return Xub >= (u128)X_LIMIT;
}

// does sup over real S in [lo, hi] of b S / (alpha S + beta)^2 reach thr?
__device__ __forceinline__ bool sup_reaches(double b, double alpha, double beta, double lo, double hi, double thr) {
  if (hi < lo) return false;
  double S;
  if (beta <= alpha * lo) S = lo;
  else if (beta >= alpha * hi) S = hi;
  else return b >= 4.0 * alpha * beta * thr;            // peak b / (4 alpha beta) at S* = beta / alpha
  const double x = alpha * S + beta;
  return b * S >= thr * x * x;
}

// Branch-and-bound pruning for linear mode: which b in (b_lo, b_hi] can still beat the incumbent?
// First a Jensen bound per b (lane per b): X >= w_b C1 S + M t_p max(S RT1, b Wn) + mem_lb; then, for the
// b's that survive it, the continuous supremum of b S/(alpha S + beta)^2 over every run of constant
// m = floor(S/b) (lanes over m).  f64 with a 1e-9 safety margin; returns a bit mask (bit b-1).
#ifndef DSTACK_BOUND_NOINLINE
#define DSTACK_BOUND_NOINLINE 0
#endif
#if DSTACK_BOUND_NOINLINE
static __device__ __noinline__
#else
__device__ __forceinline__
#endif
uint64_t bound_survivors(const uint64_t *cA, const uint64_t *cU, double thr, uint64_t C1,
                                                        uint64_t D, int b_lo, int b_hi, int S_tot, int mem_mode, int wse,
                                                        uint64_t Mtp, uint64_t RT1, uint64_t Wn, int lane) {
  const double Mtpd = (double)Mtp, C1d = (double)C1, Dd = (double)D, RT1d = (double)RT1, Wnd = (double)Wn;
  const double WnR = RT1 ? Wnd / RT1d : 0.0;
  uint32_t cand_lo = 0, cand_hi = 0;
  for (int bb = b_lo + 1 + lane; bb <= b_hi; bb += 32) {
    const double bd = (double)bb;
    const double a1 = (wse == 0 ? bd : 1.0) * C1d;
    const double m0 = mem_mode == 1 ? bd * Dd : 0.0;
    bool ok;
    if (RT1 == 0) {
      ok = sup_reaches(bd, a1, m0, 1.0, (double)S_tot, thr);
    } else {
      const double Sc = bd * WnR;
      ok = sup_reaches(bd, a1, Mtpd * bd * Wnd + m0, 1.0, fmin(Sc, (double)S_tot), thr) ||
           sup_reaches(bd, a1 + Mtpd * RT1d, m0, fmax(Sc, 1.0), (double)S_tot, thr);
    }
    if (ok) {
      const int bit = bb - 1;
      if (bit < 32) cand_lo |= 1u << bit; else cand_hi |= 1u << (bit - 32);
    }
  }
  cand_lo = __reduce_or_sync(FULL, cand_lo);
  cand_hi = __reduce_or_sync(FULL, cand_hi);
  uint64_t cand = ((uint64_t)cand_hi << 32) | cand_lo, out = 0;
  while (cand) {
    const int bb = __ffsll((long long)cand);
    cand &= cand - 1;
    const double bd = (double)bb;
    const uint64_t wC1 = (wse == 0 ? (uint64_t)bb : 1ull) * C1;
    const int mmax = S_tot / bb;
    bool ok = false;
    for (int m = lane; m <= mmax; m += 32) {
      const int lo = m * bb > 1 ? m * bb : 1;
      const int hi = m * bb + bb - 1 < S_tot ? m * bb + bb - 1 : S_tot;
      const uint64_t alpha = wC1 + cA[m] + (mem_mode == 2 ? (uint64_t)bb * D * (uint64_t)lo : 0ull);
      const uint64_t beta = (uint64_t)bb * cU[m] + (mem_mode == 1 ? (uint64_t)bb * D : 0ull);
      ok = ok || sup_reaches(bd, (double)alpha, (double)beta, (double)lo, (double)hi, thr);
    }
    if (__any_sync(FULL, ok)) out |= 1ull << (bb - 1);
  }
  if (lane == 0) { PSTAT(2, __popcll(((uint64_t)cand_hi << 32) | cand_lo)); PSTAT(3, __popcll(out)); }
  return out;
}

// Analyse DNN k.  knee_only: 1 status + knee at knee_b, 2 status + the tables at knee_b only.  Otherwise (l*, b*),
// demand, knee(b*).
// Per-warp shared memory: hist[S_tot+1] u32, cA/cU[S_tot+1] u64 (tables stay valid on return).
template <int PAR>
__device__ DnnRes analyze_dnn(const dstack_problem_t &pb, const dstack_params_t &p, int64_t k, const uint16_t *Stab,
                              uint32_t *hist, uint64_t *cA, uint64_t *cU, int lane, int knee_only, int32_t knee_b) {
  DnnRes res; res.st = DSTACK_ST_OK; res.demand = 0; res.knee = 0; res.b = 0; res.RT = 0; res.D = 0;
  const int L = p.L, S_tot = p.S_tot;
  const int64_t r0 = pb.dnn_row_off[k], r1 = pb.dnn_row_off[k + 1];
  const int64_t K64 = r1 - r0;
  const int32_t t_p = pb.t_p[k], t_np = pb.t_np[k], slo = pb.slo_us[k], asm_us = pb.asm_us[k];
  const int32_t bmax = pb.bmax[k], mbw = pb.mem_bw[k];
  const int mem_mode = p.mem_mode;
  const uint64_t M = mem_mode == 0 ? 1 : (uint64_t)mbw;
  const int32_t b_lo = p.b_min, b_hi = bmax < p.b_max ? bmax : p.b_max;
  const int32_t b_eval = knee_only ? knee_b : b_hi;   // where the overflow bound is checked
  // ---- header validation (DSTACK_ST_INVALID conditions, dstack.h) ----
  if (K64 < 1 || K64 > DSTACK_MAX_ROWS_PER_DNN || t_p < 1 || t_np < 0 || slo < 1 || slo > (1 << 30) ||
      (slo % p.slot_us) != 0 || asm_us < 0 || asm_us > (1 << 24) || bmax < 1 ||
      (mem_mode != 0 && (mbw < 1 || mbw > (1 << 24)))) {
    res.st = DSTACK_ST_INVALID;
    return res;
  }
  const int32_t K = (int32_t)K64;
  const uint32_t *n = pb.n + r0;
  const uint16_t *r = pb.r + r0;
  const uint32_t *d = pb.d + r0;
  // ---- a1: one coalesced pass over the rows (two rows per lane in flight) ----
  if (PAR == 0) {
    for (int m = lane; m <= S_tot; m += 32) hist[m] = 0;
    __syncwarp();
  }
  uint32_t RT = 0, anyR0 = 0;
  uint64_t D = 0, Wn = 0, Vmax = 0;
  auto row = [&](uint32_t nn, uint32_t R, uint32_t dd) {
    RT += R; D += (uint64_t)R * dd; Wn += (uint64_t)R * nn;
    anyR0 |= (R == 0);
    if (PAR == 0) {
      if (nn <= (uint32_t)S_tot) atomicAdd(&hist[nn], R);   // width histogram incl. n = 0 (bin 0)
    } else {
      const uint64_t Nb = ((uint64_t)b_eval * nn + 2047) >> 11;
      if (Nb >= 1) Vmax = sat_add(Vmax, (uint64_t)R * (Nb > (uint64_t)S_tot ? Nb : (uint64_t)S_tot));
    }
  };
  for (int i0 = lane; i0 < K; i0 += 32 * DSTACK_GEN_ROWS_U) {   // DSTACK_GEN_ROWS_U rows per lane in flight
    uint32_t nn[DSTACK_GEN_ROWS_U], dd[DSTACK_GEN_ROWS_U], RR[DSTACK_GEN_ROWS_U];
#pragma unroll
    for (int u = 0; u < DSTACK_GEN_ROWS_U; ++u) {
      const int i = i0 + 32 * u;
      nn[u] = 0; dd[u] = 0; RR[u] = 0;
      if (i < K) { nn[u] = __ldg(n + i); dd[u] = __ldg(d + i); RR[u] = __ldg(r + i); }
    }
#pragma unroll
    for (int u = 0; u < DSTACK_GEN_ROWS_U; ++u)
      if (i0 + 32 * u < K) row(nn[u], RR[u], dd[u]);
  }
  RT = __reduce_add_sync(FULL, RT);
  D = warp_sum_u64(D); Wn = warp_sum_u64(Wn);
  if (PAR == 1) Vmax = warp_sum_sat(Vmax);
  anyR0 = warp_or(anyR0);
  res.RT = RT; res.D = D;
  // (R_i >= 1 for all rows) => "some n_i != 0" <=> Wn > 0
  if (anyR0 || (t_np == 0 && Wn == 0 && (mem_mode == 0 || D == 0))) { res.st = DSTACK_ST_INVALID; return res; }
  if (!knee_only && b_hi < b_lo) { res.st = DSTACK_ST_INFEASIBLE; return res; }
  const uint64_t Mtp = M * (uint64_t)t_p;
  if (PAR == 0) {
    // sum_{N_i >= 1} R_i max(S_tot, b n_i) = S_tot PA[S_tot/b] + b Q[S_tot/b]  (exact, from the scan)
    const int mb = S_tot / b_eval;
    uint64_t pa_mb, q_mb;
    scan_hist(hist, cA, cU, S_tot, Wn, Mtp, mb, &pa_mb, &q_mb, lane);
    const u128 v = (u128)S_tot * pa_mb + (u128)b_eval * q_mb;
    Vmax = v >= ((u128)1 << 63) ? (1ull << 63) : (uint64_t)v;
  }
  {
    // X(L, b_eval) = w t_np RT S_tot M + M t_p Vmax + mem  (the maximum of X over the grid).  An f64
    // estimate settles all but |X - 2^56| < 1e-4 X; those are decided in exact 128-bit arithmetic.
    const double wd = p.wse_mode == 0 ? (double)b_eval : 1.0;
    double xe = wd * (double)t_np * (double)RT * (double)S_tot * (double)M + (double)M * (double)t_p * (double)Vmax;
    if (mem_mode == 1) xe += (double)b_eval * (double)D;
    else if (mem_mode == 2) xe += (double)b_eval * (double)D * (double)(S_tot * S_tot);
    bool over;
    if (Vmax >= (1ull << 63) || xe >= 72057594037927936.0 * 1.0001) over = true;
    else if (xe < 72057594037927936.0 * 0.9999) over = false;
    else over = xub_exact_over(p.wse_mode == 0 ? (uint32_t)b_eval : 1u, (uint64_t)t_np, (uint64_t)RT, (uint32_t)S_tot,
                               M, (uint64_t)t_p, Vmax, mem_mode, (uint32_t)b_eval, D);
    if (over) { res.st = DSTACK_ST_OVERFLOW; return res; }
  }
  const uint64_t RT1 = PAR == 0 ? (uint64_t)RT - hist[0] : 0ull;   // sum R over n_i >= 1
  RowCtx c;
  c.Stab = Stab; c.cA = cA; c.cU = cU; c.L = L; c.mem_mode = mem_mode; c.wse = p.wse_mode;
  c.C1 = (uint64_t)t_np * RT * M; c.D = D; c.SLOM = (uint64_t)slo * M; c.aM = (uint64_t)asm_us * M;
  // ---- a2/a3: rows evaluated exactly, b_lo (or the knee batch) first, then the b's the bounds keep ----
  Best e, kk, best = best_none();
  uint32_t knee = 0;
  bool first = true;
  uint64_t todo = 1ull << ((knee_only ? knee_b : b_lo) - 1);
  while (todo) {
    const int b = __ffsll((long long)todo);   // b = bit index + 1
    todo &= todo - 1;
    if (PAR == 1) build_tables_threads(n, r, K, S_tot, Mtp, b, hist, cA, cU, lane);
    if (knee_only == 2) return res;   // tables only (F3 knee probe): cA / cU valid at knee_b, RT and D set
    eval_row<PAR>(c, b, lane, e, kk);
    if (first) {
      first = false;
      if (knee_only) { res.knee = (uint16_t)kk.l; return res; }
      if (!e.found) { res.st = DSTACK_ST_INFEASIBLE; return res; }   // b_lo row feasible iff any row is
      best = e; knee = kk.l;
      if (b_hi > b_lo) {
        if (PAR == 1) {
          todo = (b_hi >= 64 ? ~0ull : ((1ull << b_hi) - 1)) & ~((1ull << b_lo) - 1);
        } else {
          const double thr = (double)(best.b * best.S) / ((double)best.X * (double)best.X) * (1.0 - 1e-9);
          todo = bound_survivors(cA, cU, thr, c.C1, D, b_lo, b_hi, S_tot, mem_mode, p.wse_mode, Mtp, RT1, Wn, lane);
        }
      }
    } else if (better(e, best)) {
      best = e; knee = kk.l;
    }
  }
  if (lane == 0) { PSTAT(0, 1); PSTAT(1, b_hi > b_lo); PSTAT(6, best.b > b_lo); PSTAT(7, K); }
  const int32_t dm = (int32_t)best.l + p.margin;
  res.demand = (uint16_t)(dm < L ? dm : L);
  res.b = (uint8_t)best.b;
  res.knee = (uint16_t)knee;
  return res;
}

// min(ceil(a / b), 0xFFFF) without a 64-bit integer division: f64 quotient estimate, exact fix-up.
__device__ __forceinline__ uint16_t ceil_div_clamp16(uint64_t a, uint64_t b) {
  const double qd = (double)a / (double)b;
  if (qd > 65536.0) return 0xFFFF;
  uint64_t q = (uint64_t)qd;                 // |qd - a/b| < 1e-10 here
  while (q > 0 && q * b > a) --q;            // q = floor(a / b)
  while ((q + 1) * b <= a) ++q;
  q += (q * b < a);                          // ceil
  return (uint16_t)(q > 0xFFFF ? 0xFFFF : q);
}

// d_j(b) = ceil(X(g, b) / (S(g) M Delta)) for b in [b_lo, b_hi] from the (linear-mode) tables of the
// DNN just analysed; lanes over b.  Writes dtab[b-1] (u16, clamped).
__device__ __forceinline__ void dtab_from_tables(const dstack_problem_t &pb, const dstack_params_t &p, int64_t k,
                                                 const uint64_t *cA, const uint64_t *cU, uint64_t RT, uint64_t D,
                                                 int32_t g, int32_t b_lo, int32_t b_hi, uint16_t *dtab, int lane) {
  const uint64_t M = p.mem_mode == 0 ? 1ull : (uint64_t)pb.mem_bw[k];
  const int32_t S = s_of(g, p.S_tot, p.L);
  const uint64_t C1 = (uint64_t)pb.t_np[k] * RT * M;
  const uint64_t den = (uint64_t)S * M * (uint64_t)p.slot_us;
  for (int32_t b = b_lo + lane; b <= b_hi; b += 32) {
    const uint64_t X = cell_X<0>(S, b, magic_of(b), (p.wse_mode == 0 ? (uint64_t)b : 1ull) * C1, cA, cU, p.mem_mode, D);
    dtab[b - 1] = ceil_div_clamp16(X, den);
  }
  __syncwarp();
}

// X(l, b) = E_t S M at S = S(l) from the rows (any mode), warp-cooperative; RT, D given.
__device__ __forceinline__ uint64_t x_from_rows(const dstack_problem_t &pb, const dstack_params_t &p, int64_t k,
                                                uint64_t RT, uint64_t D, uint64_t S, int32_t b, int lane) {
  const int64_t r0 = pb.dnn_row_off[k];
  const int32_t K = (int32_t)(pb.dnn_row_off[k + 1] - r0);
  const uint64_t M = p.mem_mode == 0 ? 1ull : (uint64_t)pb.mem_bw[k];
  const uint64_t t_p = (uint64_t)pb.t_p[k], t_np = (uint64_t)pb.t_np[k];
  const uint32_t *n = pb.n + r0;
  const uint16_t *r = pb.r + r0;
  uint64_t V = 0;   // sum_i R_i max(S, N_i(b)) over N_i >= 1  (= S*A + U)
  for (int i = lane; i < K; i += 32) {
    const uint64_t nn = n[i];
    const uint64_t N = p.par_mode == 0 ? (uint64_t)b * nn : ((uint64_t)b * nn + 2047) >> 11;
    if (N >= 1) V += (uint64_t)r[i] * (N > S ? N : S);
  }
  V = warp_sum_u64(V);
  uint64_t X = (p.wse_mode == 0 ? (uint64_t)b : 1ull) * t_np * RT * S * M + M * t_p * V;
  if (p.mem_mode == 1) X += (uint64_t)b * D;
  else if (p.mem_mode == 2) X += (uint64_t)b * D * S * S;
  return X;
}

// X from the row sum V = sum_i R_i max(S, N_i(b)) over N_i >= 1 (the tail of x_from_rows).
__device__ __forceinline__ uint64_t x_of_v(const dstack_problem_t &pb, const dstack_params_t &p, int64_t k, uint64_t RT,
                                           uint64_t D, uint64_t S, int32_t b, uint64_t V) {
  const uint64_t M = p.mem_mode == 0 ? 1ull : (uint64_t)pb.mem_bw[k];
  uint64_t X = (p.wse_mode == 0 ? (uint64_t)b : 1ull) * (uint64_t)pb.t_np[k] * RT * S * M + M * (uint64_t)pb.t_p[k] * V;
  if (p.mem_mode == 1) X += (uint64_t)b * D;
  else if (p.mem_mode == 2) X += (uint64_t)b * D * S * S;
  return X;
}

// One warp-cooperative row pass: RT = sum R, D = sum R d and V_q = sum_i R_i max(S_q, N_i(b)) for three S_q at
// one batch b -- the four row passes (sums, x_from_rows x 3) a consumer of one b would otherwise make.
__device__ __forceinline__ void rows_pass3(const dstack_problem_t &pb, const dstack_params_t &p, int64_t k, int32_t b,
                                           uint64_t S0, uint64_t S1, uint64_t S2, uint64_t &RT, uint64_t &D,
                                           uint64_t &V0, uint64_t &V1, uint64_t &V2, int lane) {
  const int64_t r0 = pb.dnn_row_off[k];
  const int32_t K = (int32_t)(pb.dnn_row_off[k + 1] - r0);
  const uint32_t *n = pb.n + r0;
  const uint16_t *r = pb.r + r0;
  const uint32_t *d = pb.d + r0;
  uint64_t rt = 0, dd = 0, v0 = 0, v1 = 0, v2 = 0;
  for (int i = lane; i < K; i += 32) {
    const uint64_t ri = r[i], nn = n[i];
    const uint64_t N = p.par_mode == 0 ? (uint64_t)b * nn : ((uint64_t)b * nn + 2047) >> 11;
    rt += ri;
    dd += ri * d[i];
    if (N >= 1) {
      v0 += ri * (N > S0 ? N : S0);
      v1 += ri * (N > S1 ? N : S1);
      v2 += ri * (N > S2 ? N : S2);
    }
  }
  RT = warp_sum_u64(rt); D = warp_sum_u64(dd);
  V0 = warp_sum_u64(v0); V1 = warp_sum_u64(v1); V2 = warp_sum_u64(v2);
}

// d_j(b) at level g for b in [b_lo, b_hi] from the rows (any mode): one row pass per b.
__device__ __forceinline__ void dtab_from_rows(const dstack_problem_t &pb, const dstack_params_t &p, int64_t k,
                                               uint64_t RT, uint64_t D, int32_t g, int32_t b_lo, int32_t b_hi,
                                               uint16_t *dtab, int lane) {
  const uint64_t M = p.mem_mode == 0 ? 1ull : (uint64_t)pb.mem_bw[k];
  const uint64_t S = (uint64_t)s_of(g, p.S_tot, p.L);
  const uint64_t den = S * M * (uint64_t)p.slot_us;
  for (int32_t b = b_lo; b <= b_hi; ++b) {
    const uint64_t X = x_from_rows(pb, p, k, RT, D, S, b, lane);
    if (lane == 0) dtab[b - 1] = ceil_div_clamp16(X, den);
  }
  __syncwarp();
}

// The same out of line, for the kernels that need it only on a rare path (b < b*) and keep their session's
// instruction stream small (k_compare, k_cluster).
static __device__ __noinline__ void dtab_lower(const dstack_problem_t &pb, const dstack_params_t &p, int64_t k,
                                               uint64_t RT, uint64_t D, int32_t g, int32_t b_lo, int32_t b_hi,
                                               uint16_t *dtab, int lane) {
  dtab_from_rows(pb, p, k, RT, D, g, b_lo, b_hi, dtab, lane);
}

__device__ __forceinline__ void fill_stab(uint16_t *Stab, int L, int S_tot) {
  for (int l = threadIdx.x; l <= L; l += blockDim.x) Stab[l] = (uint16_t)s_of(l, S_tot, L);
}

}  // namespace dstack
