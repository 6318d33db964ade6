/* oracle.c -- CPU ORACLE (test infrastructure only; see oracle.h header comment).
 *
 * Plain, slow, obviously-correct definitions of what the D-STACK hot path
 * computes, written from PAPER.md (P:n = /root/reference/PAPER.md line n) in
 * the readings of SURVEY.md §8(c) O1-O6 (listed in DESIGN.md §3).  No
 * blocking, no fusion, no candidate pruning: every argmax is a full grid
 * scan, every schedule query is a slot-by-slot loop, every latency is the
 * per-kernel sum of Eqs. 2-5 evaluated from scratch.  Decisions use exact
 * integers (unsigned __int128); f64 appears only in the reported ratios.
 *
 * Shares no code with the CUDA path (paper_2304_13541_b200/csrc).
 */
#include "oracle.h"
#include "../synth/synth_core.h"   /* the shared input generator: arrival sampler only */
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;

/* One DNN: per-DNN constants and its kernel rows (Table "Notations for DNN Model"). */
typedef struct {
  int64_t K;
  const uint32_t *n;   /* n_i: parallel ops at batch 1 (linear mode) or threads theta_i (threads mode) */
  const uint16_t *r;   /* R_i: repetitions of kernel i */
  const uint32_t *d;   /* d_i: bytes the kernel waits for */
  int64_t t_p, t_np, M, slo, a, bmax, mem_bw_raw;
} dnn_t;

static dnn_t get_dnn(const or_problem_t *pb, const or_params_t *p, int64_t k) {
  dnn_t m;
  int64_t r0 = pb->dnn_row_off[k], r1 = pb->dnn_row_off[k + 1];
  m.K = r1 - r0;
  m.n = pb->n + r0; m.r = pb->r + r0; m.d = pb->d + r0;
  m.t_p = pb->t_p[k]; m.t_np = pb->t_np[k];
  m.mem_bw_raw = pb->mem_bw[k];
  /* M is forced to 1 when the memory term is off (it then cancels everywhere). */
  m.M = (p->mem_mode == 0) ? 1 : pb->mem_bw[k];
  m.slo = pb->slo_us[k]; m.a = pb->asm_us[k]; m.bmax = pb->bmax[k];
  return m;
}

/* S(l) = ceil(l * S_tot / L): SMs granted at GPU% level l (CUDA_MPS_ACTIVE_THREAD_PERCENTAGE
 * -> SM share; identity when L = S_tot). */
static int64_t S_of(const or_params_t *p, int64_t l) { return (l * p->S_tot + p->L - 1) / p->L; }

/* Eq. 1, tabulated reading: parallel ops of kernel i at batch b.
 * linear: N_i(b) = b * n_i (N_1 = p*b, decrement p*b/K: parallelism scales with b);
 * threads: N_i(b) = ceil(b * theta_i / 2048), the paper's threads -> SM-wave conversion. */
static u128 N_of(const or_params_t *p, uint32_t n, int64_t b) {
  if (p->par_mode == 0) return (u128)b * n;
  return ((u128)b * n + 2047) / 2048;
}

/* O1 -- Eqs. 2-5: X = E_t * S * M, exact.
 *   Eq. 2: E_i = W_i / max(1, min(S, N_i)), W_i = N_i t_p
 *   Eq. 3: E_m = d_i S / M (verbatim) | d_i / (M S) (bw, prose P:1517) | 0 (off)
 *   Eq. 4: W_se = b * sum_i R_i (t_np + E_m)  [per_request]
 *          W_se = sum_i R_i t_np + b * sum_i R_i E_m                  [per_launch reading, P:1515]
 *   Eq. 5: E_t = W_se + sum_i R_i E_i
 * Multiplying through by S*M makes every term an integer:
 *   E_i*S = t_p*S if 1 <= N_i <= S; t_p*N_i if N_i > S; 0 if N_i = 0.
 *   E_m*S*M = d_i*S^2 | d_i | 0.                                                           */
static u128 X_of(const dnn_t *m, const or_params_t *p, int64_t S, int64_t b) {
  u128 X = 0;
  const u128 w = (p->wse_mode == 0) ? (u128)b : (u128)1;
  for (int64_t i = 0; i < m->K; ++i) {
    const u128 R = m->r[i];
    const u128 N = N_of(p, m->n[i], b);
    u128 EiS = 0;
    if (N >= 1) EiS = (N <= (u128)S) ? (u128)m->t_p * (u128)S : (u128)m->t_p * N;
    u128 EmSM = 0;
    if (p->mem_mode == 1) EmSM = m->d[i];
    else if (p->mem_mode == 2) EmSM = (u128)m->d[i] * (u128)S * (u128)S;
    X += R * (w * (u128)m->t_np * (u128)S * (u128)m->M + (u128)b * EmSM + (u128)m->M * EiS);
  }
  return X;
}

#define X_LIMIT (((u128)1) << 56)

/* Validation (statuses documented in include/dstack.h).  Returns OR_OK, OR_INVALID,
 * OR_INFEASIBLE (empty batch range) or OR_OVERFLOW (X(L, b_hi) >= 2^56; X is nondecreasing
 * in S and b, so this bounds every cell). */
static int validate_basic(const dnn_t *m, const or_params_t *p) {
  if (m->K < 1 || m->K > OR_MAX_ROWS_PER_DNN) return OR_INVALID;
  if (m->t_p < 1 || m->t_np < 0) return OR_INVALID;
  if (m->slo < 1 || m->slo > (1LL << 30) || m->slo % p->slot_us != 0) return OR_INVALID;
  if (m->a < 0 || m->a > (1LL << 24)) return OR_INVALID;
  if (m->bmax < 1) return OR_INVALID;
  if (p->mem_mode != 0 && (m->mem_bw_raw < 1 || m->mem_bw_raw > (1LL << 24))) return OR_INVALID;
  for (int64_t i = 0; i < m->K; ++i)
    if (m->r[i] == 0) return OR_INVALID;
  if (X_of(m, p, S_of(p, 1), p->b_min) == 0) return OR_INVALID; /* latency identically 0: Eq. 6 undefined */
  return OR_OK;
}

static int validate(const dnn_t *m, const or_params_t *p, int64_t *b_lo, int64_t *b_hi) {
  int st = validate_basic(m, p);
  if (st != OR_OK) return st;
  *b_lo = p->b_min;
  *b_hi = m->bmax < p->b_max ? m->bmax : p->b_max;
  if (*b_hi < *b_lo) return OR_INFEASIBLE;
  if (X_of(m, p, S_of(p, p->L), *b_hi) >= X_LIMIT) return OR_OVERFLOW;
  return OR_OK;
}

/* O2 -- Eq. 6: knee(b) = argmax over l in 1..L of 1/(f_L(l,b)^2 * S(l)),
 * f_L = X/(S M); g = M^2 S / X^2.  g_1 > g_2  <=>  S_1 X_2^2 > S_2 X_1^2.  Ties -> smaller l. */
static int64_t knee_of(const dnn_t *m, const or_params_t *p, int64_t b) {
  int64_t best_l = 1, best_S = S_of(p, 1);
  u128 best_X = X_of(m, p, best_S, b);
  for (int64_t l = 2; l <= p->L; ++l) {
    const int64_t S = S_of(p, l);
    const u128 X = X_of(m, p, S, b);
    if ((u128)S * best_X * best_X > (u128)best_S * X * X) { best_l = l; best_S = S; best_X = X; }
  }
  return best_l;
}

/* O3 -- Eqs. 7-12.  Feasible(l, b) iff
 *   Eq. 10: b_lo <= b <= b_hi                      (1 <= b <= MaxBatch)
 *   Eq. 11: f_L + C <= SLO, C = b * a              (b = Rate * C; 481 us/image)
 *   Eq. 12: f_L <= SLO / 2
 * eta = b / (f_L^2 * GPU%) (Eq. 9) with GPU% = S(l)/S_tot; eta ∝ b S / X^2.
 * (l*, b*) = argmax over feasible cells, ties -> smaller l then smaller b (scan order, strict >).
 * The exact discrete argmax replaces fmincon. */
static void batch_opt_one(const dnn_t *m, const or_params_t *p, uint16_t *demand, uint8_t *batch,
                          uint16_t *knee, uint8_t *status) {
  int64_t b_lo, b_hi;
  int st = validate(m, p, &b_lo, &b_hi);
  *demand = 0; *batch = 0; *knee = 0;
  if (st != OR_OK) { *status = (uint8_t)st; return; }
  int found = 0;
  int64_t bl = 0, bb = 0, bS = 0;
  u128 bX = 0;
  const u128 SLO = (u128)m->slo, A = (u128)m->a, M = (u128)m->M;
  for (int64_t l = 1; l <= p->L; ++l) {
    const int64_t S = S_of(p, l);
    for (int64_t b = b_lo; b <= b_hi; ++b) {
      const u128 X = X_of(m, p, S, b);
      if (X + (u128)b * A * (u128)S * M > SLO * (u128)S * M) continue;   /* Eq. 11 */
      if (2 * X > SLO * (u128)S * M) continue;                            /* Eq. 12 */
      if (!found || (u128)b * (u128)S * bX * bX > (u128)bb * (u128)bS * X * X) {
        found = 1; bl = l; bb = b; bS = S; bX = X;
      }
    }
  }
  if (!found) { *status = OR_INFEASIBLE; return; }
  /* over-provisioning margin, default 0 */
  int64_t dm = bl + p->margin;
  *demand = (uint16_t)(dm < p->L ? dm : p->L);
  *batch = (uint8_t)bb;
  *knee = (uint16_t)knee_of(m, p, bb);
  *status = OR_OK;
}

int oracle_X(const or_problem_t *pb, const or_params_t *p, int64_t dnn, int32_t l, int32_t b,
             uint64_t *lo, uint64_t *hi) {
  if (!pb || !p || dnn < 0 || dnn >= pb->num_dnn || l < 1 || l > p->L || b < 1) return -1;
  dnn_t m = get_dnn(pb, p, dnn);
  u128 X = X_of(&m, p, S_of(p, l), b);
  *lo = (uint64_t)X; *hi = (uint64_t)(X >> 64);
  return 0;
}

int oracle_knee(const or_problem_t *pb, const or_params_t *p, int32_t b, uint16_t *knee_out, uint8_t *st_out) {
  if (!pb || !p || b < 1) return -1;
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t k = 0; k < pb->num_dnn; ++k) {
    dnn_t m = get_dnn(pb, p, k);
    int st = validate_basic(&m, p);                    /* the knee itself needs no batch range */
    if (st == OR_OK && X_of(&m, p, S_of(p, p->L), b) >= X_LIMIT) st = OR_OVERFLOW;
    st_out[k] = (uint8_t)st;
    knee_out[k] = (st == OR_OK) ? (uint16_t)knee_of(&m, p, b) : 0;
  }
  return 0;
}

/* F3 -- online knee discovery: "our platform initially provides it a nominal, 30%, GPU. The GPU% is
 * then readjusted ... to find the knee based on the inference latency using a simple binary search."
 * Reading R22: lo = 1, hi = L; step 1 probes m = ceil(0.3 L), later steps the midpoint
 * floor((lo + hi) / 2), m kept in [lo, hi - 1]; the latencies at m and m + 1 decide: Eq. 6's objective
 * g = 1/(f_L^2 S) larger at m + 1 (g(m+1) > g(m) <=> S(m+1) X(m)^2 > S(m) X(m+1)^2) => lo = m + 1, else hi = m.
 * trace (nullable, >= 16 entries): the probed m of every step. */
static int64_t knee_probe_of(const dnn_t *m, const or_params_t *p, int64_t b, int32_t *steps, int32_t *trace) {
  int64_t lo = 1, hi = p->L;
  int32_t n = 0;
  while (lo < hi) {
    int64_t mid = n == 0 ? (3 * (int64_t)p->L + 9) / 10 : (lo + hi) / 2;
    if (mid < lo) mid = lo;
    if (mid > hi - 1) mid = hi - 1;
    const int64_t S0 = S_of(p, mid), S1 = S_of(p, mid + 1);
    const u128 X0 = X_of(m, p, S0, b), X1 = X_of(m, p, S1, b);
    if (trace && n < 16) trace[n] = (int32_t)mid;
    if ((u128)S1 * X0 * X0 > (u128)S0 * X1 * X1) lo = mid + 1; else hi = mid;
    ++n;
  }
  *steps = n;
  return lo;
}

int oracle_knee_probe(const or_problem_t *pb, const or_params_t *p, int32_t b, uint16_t *knee_out, uint8_t *probes_out,
                      uint8_t *st_out, int32_t *trace) {
  if (!pb || !p || b < 1) return -1;
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t k = 0; k < pb->num_dnn; ++k) {
    dnn_t m = get_dnn(pb, p, k);
    int st = validate_basic(&m, p);
    if (st == OR_OK && X_of(&m, p, S_of(p, p->L), b) >= X_LIMIT) st = OR_OVERFLOW;
    st_out[k] = (uint8_t)st;
    int32_t steps = 0;
    knee_out[k] = (st == OR_OK) ? (uint16_t)knee_probe_of(&m, p, b, &steps, trace ? trace + 16 * k : NULL) : 0;
    probes_out[k] = (uint8_t)steps;
  }
  return 0;
}

int oracle_batch_opt(const or_problem_t *pb, const or_params_t *p, uint16_t *demand, uint8_t *batch,
                     uint16_t *knee, uint8_t *status) {
  if (!pb || !p) return -1;
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t k = 0; k < pb->num_dnn; ++k) {
    dnn_t m = get_dnn(pb, p, k);
    batch_opt_one(&m, p, demand + k, batch + k, knee + k, status + k);
  }
  return 0;
}

/* O4 -- Algorithm WMAX-MIN.  Readings: the loop "for i <- 1 to N,
 * Fulfill Lowest Demand First" visits demands in ascending (demand, index) order;
 * "retGPU[j] += knee[j]/totDemand x remGPU" is kept in Q16.16 fixed point, floored;
 * totDemand = 0 => no proportional share (0/0 guard). */
int oracle_wmaxmin(int32_t n, const uint16_t *demand, int32_t L, uint32_t *alloc_q16) {
  if (n < 0 || n > 4096) return -1;
  int32_t order[4096];
  int64_t ret[4096];
  int64_t rem = L;                                   /* P:29 remGPU <- maxGPU% */
  int64_t tot = 0;                                   /* P:31 totDemand <- sum knee[k] */
  for (int32_t i = 0; i < n; ++i) { ret[i] = 0; tot += demand[i]; order[i] = i; }
  for (int32_t i = 1; i < n; ++i) {                  /* stable insertion sort by demand */
    int32_t v = order[i], k = i - 1;
    while (k >= 0 && demand[order[k]] > demand[v]) { order[k + 1] = order[k]; --k; }
    order[k + 1] = v;
  }
  for (int32_t q = 0; q < n; ++q) {
    int32_t i = order[q];
    int64_t k = demand[i];
    if (rem >= k) { ret[i] = k; rem -= k; }
    else if (rem > 0) { ret[i] = rem; rem = 0; }
  }
  for (int32_t j = 0; j < n; ++j) {                  /* P:41-45 (remGPU >= 0 always holds) */
    uint64_t share = 0;
    if (tot > 0) share = (uint64_t)(((u128)demand[j] * (u128)rem << 16) / (u128)tot);
    alloc_q16[j] = (uint32_t)(((uint64_t)ret[j] << 16) + share);
  }
  return 0;
}

/* ---------------------------------------------------------------- O5 --- */

typedef struct { int32_t dl, d, j, r; } job_t;

static int job_cmp(const void *a, const void *b) {
  const job_t *x = (const job_t *)a, *y = (const job_t *)b;
  if (x->dl != y->dl) return x->dl < y->dl ? -1 : 1;   /* EDF: tightest deadline first (Alg.1 l.5) */
  if (x->d != y->d) return x->d < y->d ? -1 : 1;       /* ties: shorter runtime (SPEC S:375 reading) */
  if (x->j != y->j) return x->j < y->j ? -1 : 1;
  return x->r < y->r ? -1 : (x->r > y->r);
}

typedef struct { int32_t j, start, end, batch, kind, rep, level; } run_t;

/* occ[u] + g <= L for all u in [s, s+d)  (Eq. 14 `eq:constraints`: G_ui <= 100%) */
static int fits(const int32_t *occ, int32_t s, int64_t d, int32_t g, int32_t L) {
  for (int64_t u = s; u < s + d; ++u)
    if (occ[u] + g > L) return 0;
  return 1;
}

/* O5 -- one D-STACK session (Alg. 1, Alg. 3 Start-Late P:3597-3611, §6.1 P:2097-2161,
 * Fair Opportunistic Dynamic fill §6.1.2), reading of SURVEY §8(c) O5:
 *  - session T = max SLO (Alg.1 l.2), repeat_j = T / SLO_j (l.3), window (j,r) = [r SLO_j, (r+1) SLO_j)
 *  - static jobs in EDF order; even repeats Start-Early, odd repeats Start-Late ("STEP 2", P:3538;
 *    "as far apart as possible"); each job placed once on the whole run [s, s+d)
 *  - fill at decision times {0} u {run ends}: models by (runs so far, index) (scoreboard),
 *    not running at t, fits at t; slice to the next blocking slot / own next start; largest batch
 *    b <= b* whose runtime fits the slice ("a batch size that can complete within the time slice",
 *    P:2330-2331).                                                                                  */
static int cycle_core(int32_t n, const int32_t *g, const int32_t *sl, const int32_t *bstar,
                      const int64_t *dtab, int32_t b_lo, int32_t L, int32_t nslots, const int64_t *count0,
                      int32_t *runs, int64_t *served, int32_t *jmiss, or_cyc_sum_t *sum,
                      int32_t trace_cap, int32_t *tr_dnn, int32_t *tr_start, int32_t *tr_end,
                      int32_t *tr_batch, int32_t *tr_kind, int32_t *tr_rep, run_t **runs_out, int64_t *nrun_out,
                      int32_t fill_order, int64_t *busy, const int64_t *dlow, int32_t *tr_level) {
  if (n < 0 || n > 1024 || nslots < 0 || nslots > (1 << 20)) return -1;
  int32_t *occ = (int32_t *)calloc((size_t)nslots + 1, sizeof(int32_t));
  uint8_t *decide = (uint8_t *)calloc((size_t)nslots + 1, 1);
  int64_t njobs = 0;
  for (int32_t j = 0; j < n; ++j) if (g[j] > 0) njobs += nslots / sl[j];
  job_t *jobs = (job_t *)malloc(sizeof(job_t) * (size_t)(njobs + 1));
  int64_t runcap = njobs + 16 + 4 * (int64_t)nslots * (n + 1);
  run_t *rl = (run_t *)malloc(sizeof(run_t) * (size_t)runcap);
  int64_t nrun = 0;
  int64_t count[OR_MAX_DNN_PER_SCEN + 1024];
  memset(sum, 0, sizeof(*sum));
  for (int32_t j = 0; j < n; ++j) { runs[j] = 0; served[j] = 0; jmiss[j] = 0; count[j] = count0 ? count0[j] : 0; }

  /* Alg.1 l.3: repeat[] <- S-Length / SLO; jobs with EDF key */
  int64_t q = 0;
  for (int32_t j = 0; j < n; ++j) {
    if (g[j] <= 0) continue;
    int32_t rep = nslots / sl[j];
    for (int32_t r = 0; r < rep; ++r) {
      int64_t d = dtab[(int64_t)j * 64 + bstar[j] - 1];
      jobs[q].dl = (r + 1) * sl[j];
      jobs[q].d = d > 0x7FFFFFFF ? 0x7FFFFFFF : (int32_t)d;
      jobs[q].j = j; jobs[q].r = r;
      ++q;
    }
  }
  qsort(jobs, (size_t)q, sizeof(job_t), job_cmp);

  /* static placement */
  for (int64_t k = 0; k < q; ++k) {
    const int32_t j = jobs[k].j, r = jobs[k].r;
    const int64_t d = dtab[(int64_t)j * 64 + bstar[j] - 1];
    const int32_t rel = r * sl[j], dl = (r + 1) * sl[j];
    int32_t s_found = -1;
    if (d <= dl - rel) {
      if (r % 2 == 0) {                      /* Start-Early (struck helper) */
        for (int32_t s = rel; s + d <= dl; ++s)
          if (fits(occ, s, d, g[j], L)) { s_found = s; break; }
      } else {                               /* Start-Late (Alg. 3) */
        for (int32_t s = (int32_t)(dl - d); s >= rel; --s)
          if (fits(occ, s, d, g[j], L)) { s_found = s; break; }
      }
    }
    int32_t lv = g[j];
    int64_t dd = d;
    if (s_found < 0 && dlow) {
      /* F1 ("schedule a model with GPU% lower than its Knee, albeit with high inference latency
         when necessary", including "the additional latency of launching a new DNN model at lower GPU%"):
         levels g_j - 1 down to 1, the first one with a feasible start in the window, same start rule. */
      for (int32_t l = g[j] - 1; l >= 1 && s_found < 0; --l) {
        const int64_t dl_ = dlow[(int64_t)j * 256 + l];
        if (dl_ <= 0 || dl_ > dl - rel) continue;
        if (r % 2 == 0) {
          for (int32_t s = rel; s + dl_ <= dl; ++s)
            if (fits(occ, s, dl_, l, L)) { s_found = s; break; }
        } else {
          for (int32_t s = (int32_t)(dl - dl_); s >= rel; --s)
            if (fits(occ, s, dl_, l, L)) { s_found = s; break; }
        }
        if (s_found >= 0) { lv = l; dd = dl_; }
      }
    }
    if (s_found < 0) { jmiss[j]++; sum->misses++; sum->status = OR_OVERSUBSCRIBED; continue; }
    for (int64_t u = s_found; u < s_found + dd; ++u) occ[u] += lv;
    rl[nrun].j = j; rl[nrun].start = s_found; rl[nrun].end = (int32_t)(s_found + dd);
    rl[nrun].batch = bstar[j]; rl[nrun].kind = lv == g[j] ? 0 : 2; rl[nrun].rep = r; rl[nrun].level = lv; ++nrun;
    if (lv != g[j]) sum->below++;
    runs[j]++; served[j] += bstar[j]; count[j]++;
  }
  for (int32_t u = 0; u < nslots; ++u) sum->occ_static_sum += occ[u];

  /* Dynamic-schedule (Alg. 1): decision times {0} u {end of every run} */
  if (nslots > 0) decide[0] = 1;
  for (int64_t k = 0; k < nrun; ++k) if (rl[k].end < nslots) decide[rl[k].end] = 1;
  int32_t order[OR_MAX_DNN_PER_SCEN + 1024];
  for (int32_t t = 0; t < nslots; ++t) {
    if (!decide[t]) continue;
    /* priority, snapshot at time t: D-STACK fewest runs first (scoreboard); O9 comparison
       schedulers: Max-Min fair smallest GPU% first, max-throughput shortest run first;
       ties by index */
    int32_t no = 0;
    int64_t key[OR_MAX_DNN_PER_SCEN + 1024];
    for (int32_t j = 0; j < n; ++j) {
      if (g[j] <= 0) continue;
      key[j] = fill_order == 0 ? count[j] : fill_order == 1 ? (int64_t)g[j] : dtab[(int64_t)j * 64 + bstar[j] - 1];
      order[no++] = j;
    }
    for (int32_t i = 1; i < no; ++i) {
      int32_t v = order[i], k = i - 1;
      while (k >= 0 && (key[order[k]] > key[v] || (key[order[k]] == key[v] && order[k] > v))) {
        order[k + 1] = order[k]; --k;
      }
      order[k + 1] = v;
    }
    for (int32_t oi = 0; oi < no; ++oi) {
      const int32_t j = order[oi];
      int covered = 0;
      int64_t next_start = nslots;
      for (int64_t k = 0; k < nrun; ++k) {
        if (rl[k].j != j) continue;
        if (rl[k].start <= t && t < rl[k].end) covered = 1;
        if (rl[k].start > t && rl[k].start < next_start) next_start = rl[k].start;
      }
      if (covered) continue;                              /* model already active at t */
      if (occ[t] + g[j] > L) continue;                    /* "Remaining-GPU > model.GPU%" (fits) */
      int64_t k = 0;                                      /* Slice <- time(Schedule, GPU%) */
      while (t + k < next_start && occ[t + k] + g[j] <= L) ++k;
      int32_t b = 0;                                      /* Batch-Size(model, Slice) */
      for (int32_t bb = bstar[j]; bb >= b_lo; --bb)
        if (dtab[(int64_t)j * 64 + bb - 1] <= k) { b = bb; break; }
      if (b == 0) continue;
      const int64_t d = dtab[(int64_t)j * 64 + b - 1];   /* Run-Batch(model, batch) */
      for (int64_t u = t; u < t + d; ++u) occ[u] += g[j];
      rl[nrun].j = j; rl[nrun].start = t; rl[nrun].end = (int32_t)(t + d);
      rl[nrun].batch = b; rl[nrun].kind = 1; rl[nrun].rep = -1; rl[nrun].level = g[j]; ++nrun;
      runs[j]++; served[j] += b; count[j]++;
      if (t + d < nslots) decide[t + d] = 1;
    }
  }
  for (int32_t u = 0; u < nslots; ++u) sum->occ_sum += occ[u];
  for (int32_t j = 0; j < n; ++j) sum->served_total += served[j];
  if (busy) {
    for (int32_t j = 0; j < n; ++j) busy[j] = 0;
    for (int64_t k = 0; k < nrun; ++k) busy[rl[k].j] += rl[k].end - rl[k].start;
  }
  sum->trace_n = 0;
  for (int64_t k = 0; k < nrun && k < trace_cap; ++k) {
    tr_dnn[k] = rl[k].j; tr_start[k] = rl[k].start; tr_end[k] = rl[k].end;
    tr_batch[k] = rl[k].batch; tr_kind[k] = rl[k].kind; tr_rep[k] = rl[k].rep;
    if (tr_level) tr_level[k] = rl[k].level;
    sum->trace_n++;
  }
  free(occ); free(decide); free(jobs);
  if (runs_out) { *runs_out = rl; *nrun_out = nrun; } else free(rl);
  return 0;
}

int oracle_cycle_direct(int32_t n, const int32_t *g, const int32_t *sl, const int32_t *bstar,
                        const int64_t *dtab, int32_t b_lo, int32_t L, int32_t nslots, const int64_t *count0,
                        int32_t *runs, int64_t *served, int32_t *jmiss, or_cyc_sum_t *sum,
                        int32_t trace_cap, int32_t *tr_dnn, int32_t *tr_start, int32_t *tr_end,
                        int32_t *tr_batch, int32_t *tr_kind, int32_t *tr_rep) {
  return cycle_core(n, g, sl, bstar, dtab, b_lo, L, nslots, count0, runs, served, jmiss, sum, trace_cap, tr_dnn,
                    tr_start, tr_end, tr_batch, tr_kind, tr_rep, NULL, NULL, 0, NULL, NULL, NULL);
}

int oracle_cycle_direct_bk(int32_t n, const int32_t *g, const int32_t *sl, const int32_t *bstar, const int64_t *dtab,
                           const int64_t *dlow, int32_t b_lo, int32_t L, int32_t nslots, int32_t *runs,
                           int64_t *served, int32_t *jmiss, or_cyc_sum_t *sum, int32_t trace_cap, int32_t *tr_dnn,
                           int32_t *tr_start, int32_t *tr_end, int32_t *tr_batch, int32_t *tr_kind, int32_t *tr_rep,
                           int32_t *tr_level) {
  return cycle_core(n, g, sl, bstar, dtab, b_lo, L, nslots, NULL, runs, served, jmiss, sum, trace_cap, tr_dnn,
                    tr_start, tr_end, tr_batch, tr_kind, tr_rep, NULL, NULL, 0, NULL, dlow, tr_level);
}

int oracle_cycle_direct_ex(int32_t n, const int32_t *g, const int32_t *sl, const int32_t *bstar,
                           const int64_t *dtab, int32_t b_lo, int32_t L, int32_t nslots, const int64_t *count0,
                           int32_t fill_order, int32_t *runs, int64_t *served, int32_t *jmiss, int64_t *busy,
                           or_cyc_sum_t *sum, int32_t trace_cap, int32_t *tr_dnn, int32_t *tr_start, int32_t *tr_end,
                           int32_t *tr_batch, int32_t *tr_kind, int32_t *tr_rep) {
  if (fill_order < 0 || fill_order > 2) return -1;
  return cycle_core(n, g, sl, bstar, dtab, b_lo, L, nslots, count0, runs, served, jmiss, sum, trace_cap, tr_dnn,
                    tr_start, tr_end, tr_batch, tr_kind, tr_rep, NULL, NULL, fill_order, busy, NULL, NULL);
}

/* ---------------------------------------------------------------- O9 ---
 * Comparison schedulers of §6.3, readings in DESIGN.md §3.2.
 *
 * Temporal sharing: over the session of nslots slots, model j gets the contiguous slice
 * slice_j = floor(nslots * sl_j / sum sl) ("time slices proportional to the model's SLOs") holding the whole
 * GPU; in it it runs back-to-back batches of b*_j at 100% GPU, d^L_j slots each; the GPU utilization
 * counts its knee% over the slice ("We compute GPU utilization by using Knee% for each model").   */
int oracle_temporal_direct(int32_t n, const int32_t *lvl, const int32_t *sl, const int64_t *dL, int32_t nslots,
                           int64_t *slice_out, int64_t *runs_out, int64_t *occ_num) {
  int64_t tot = 0;
  *occ_num = 0;
  for (int32_t j = 0; j < n; ++j) if (lvl[j] > 0) tot += sl[j];
  for (int32_t j = 0; j < n; ++j) {
    slice_out[j] = 0; runs_out[j] = 0;
    if (lvl[j] <= 0 || tot == 0) continue;
    slice_out[j] = (int64_t)nslots * sl[j] / tot;
    runs_out[j] = dL[j] > 0 ? slice_out[j] / dL[j] : 0;
    *occ_num += slice_out[j] * lvl[j];
  }
  return 0;
}

/* Static spatial sharing, GSLICE-style CSS: models keep their knee GPU% for the
 * whole slot they run in.  When the knees do not fit together, the session is cut into K equal time slots:
 * the lightest models that fit beside every other model stay resident in all slots ("Alexnet and
 * Mobilenet concurrently in both time slots"), the others are packed first-fit decreasing into slots of the
 * remaining capacity ("VGG-19 in the first time slot, and ResNet-50 in the second").  In each of its
 * slots a model runs back-to-back batches of b*_j, dk_j slots each.  home[j] = -1 resident, else its slot. */
int oracle_gslice_direct(int32_t n, const int32_t *lvl, const int64_t *dk, int32_t nslots, int32_t L,
                         int32_t *home, int32_t *nbins, int64_t *runs_out, int64_t *busy_out, int64_t *occ_num) {
  if (n < 0 || n > 1024) return -1;
  int32_t ord[1024], na = 0;
  for (int32_t j = 0; j < n; ++j) { home[j] = -2; runs_out[j] = 0; busy_out[j] = 0; if (lvl[j] > 0) ord[na++] = j; }
  *occ_num = 0; *nbins = 0;
  if (na == 0) return 0;
  for (int32_t i = 1; i < na; ++i) {   /* ascending (level, index) */
    int32_t v = ord[i], k = i - 1;
    while (k >= 0 && (lvl[ord[k]] > lvl[v] || (lvl[ord[k]] == lvl[v] && ord[k] > v))) { ord[k + 1] = ord[k]; --k; }
    ord[k + 1] = v;
  }
  /* residents: the longest ascending prefix P with sum_P + (largest level outside P) <= L */
  int64_t pre = 0;
  int32_t np = 0;
  for (int32_t p = na; p >= 0; --p) {
    int64_t sp = 0;
    for (int32_t i = 0; i < p; ++i) sp += lvl[ord[i]];
    const int64_t mx = p < na ? lvl[ord[na - 1]] : 0;
    if (sp + mx <= L) { np = p; pre = sp; break; }
  }
  for (int32_t i = 0; i < np; ++i) home[ord[i]] = -1;
  /* the rest, first-fit decreasing (level desc, index asc) into slots of capacity L - sum_P */
  int32_t rest[1024], nr = 0;
  for (int32_t i = np; i < na; ++i) rest[nr++] = ord[i];
  for (int32_t i = 1; i < nr; ++i) {   /* (level desc, index asc) */
    int32_t v = rest[i], k = i - 1;
    while (k >= 0 && (lvl[rest[k]] < lvl[v] || (lvl[rest[k]] == lvl[v] && rest[k] > v))) { rest[k + 1] = rest[k]; --k; }
    rest[k + 1] = v;
  }
  int64_t resid[1024];
  int32_t K = 0;
  for (int32_t i = 0; i < nr; ++i) {
    const int32_t j = rest[i];
    int32_t b = 0;
    while (b < K && resid[b] < lvl[j]) ++b;   /* first fit */
    if (b == K) resid[K++] = L - pre;
    resid[b] -= lvl[j];
    home[j] = b;
  }
  if (K == 0) K = 1;
  *nbins = K;
  const int64_t w = nslots / K;
  for (int32_t j = 0; j < n; ++j) {
    if (lvl[j] <= 0 || dk[j] <= 0) continue;
    const int64_t nsl = home[j] == -1 ? K : 1;
    runs_out[j] = nsl * (w / dk[j]);
    busy_out[j] = runs_out[j] * dk[j];
    *occ_num += busy_out[j] * lvl[j];
  }
  return 0;
}

/* ---------------------------------------------------------------- O6 --- */

/* O6 setup (§6.2, "we computed the knee of each kernel"): execution demand g_e of row i
 * is the Eq. 6 knee of the one-row DNN {n_i, R = 1, d_i} at batch b (DNN's t_p, t_np, M, modes);
 * duration tau_e = ceil(f_e(g_e)) us with f_e = X_e / (S M). */
int oracle_ideal_rows(const or_problem_t *pb, const or_params_t *p, int64_t dnn, int32_t b,
                      int32_t *g_out, int64_t *tau_out) {
  dnn_t m = get_dnn(pb, p, dnn);
  for (int64_t i = 0; i < m.K; ++i) {
    dnn_t one = m;
    uint16_t rone = 1;
    one.K = 1; one.n = m.n + i; one.d = m.d + i; one.r = &rone;
    int64_t gl = knee_of(&one, p, b);
    int64_t S = S_of(p, gl);
    u128 X = X_of(&one, p, S, b);
    u128 den = (u128)S * (u128)one.M;
    g_out[i] = (int32_t)gl;
    tau_out[i] = (int64_t)((X + den - 1) / den);
  }
  return 0;
}

/* O6 -- ideal per-kernel scheduler (§6.2, Eqs. 13-14 `eq:maximization`/`eq:constraints`,
 * P:2373-2416): preemptive, instantaneous reallocation.  Event-driven (slot -> 0 limit of
 * the 100 us slots).  At each event the eligible set is every DNN's current kernel execution
 * (chain constraint k_i in E => k_{i-1} done); choose the subset maximising sum g <= L ("exhaustive
 * search"), ties broken lexicographically by priority (batch deadline, then index: "ordered
 * by their earliest deadline"); selected executions progress until the first completes. */
int oracle_ideal_direct(int32_t n, const int64_t *chain_off, const int32_t *ex_g, const int64_t *ex_tau,
                        const int64_t *slo_us, const int32_t *bstar, const uint8_t *active, int32_t L,
                        int64_t T_us, int64_t *util_out, int64_t *completed, int64_t *events_out) {
  (void)bstar;
  if (n < 0 || n > 1024 || L < 1) return -1;
  int64_t *pos = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
  int64_t *rem = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
  int64_t *bstart = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
  uint8_t *live = (uint8_t *)calloc((size_t)n + 1, 1);
  int32_t *ord = (int32_t *)calloc((size_t)n + 1, sizeof(int32_t));
  uint8_t *sel = (uint8_t *)calloc((size_t)n + 1, 1);
  uint8_t *reach = (uint8_t *)calloc((size_t)(n + 1) * (size_t)(L + 1), 1);
  int64_t util = 0, events = 0;
  for (int32_t j = 0; j < n; ++j) {
    completed[j] = 0;
    if (!active[j]) continue;
    for (int64_t e = chain_off[j]; e < chain_off[j + 1]; ++e)
      if (ex_tau[e] > 0) { live[j] = 1; pos[j] = e; rem[j] = ex_tau[e]; break; }
  }
  int64_t t = 0;
  while (t < T_us) {
    int32_t no = 0;
    for (int32_t j = 0; j < n; ++j) if (live[j]) ord[no++] = j;
    if (no == 0) break;
    for (int32_t i = 1; i < no; ++i) {            /* priority: (deadline, index) */
      int32_t v = ord[i], k = i - 1;
      while (k >= 0 && (bstart[ord[k]] + slo_us[ord[k]] > bstart[v] + slo_us[v] ||
                        (bstart[ord[k]] + slo_us[ord[k]] == bstart[v] + slo_us[v] && ord[k] > v))) {
        ord[k + 1] = ord[k]; --k;
      }
      ord[k + 1] = v;
    }
    /* reach[k][s] = items ord[k..no-1] can sum exactly to s (s <= L) */
    memset(reach, 0, (size_t)(no + 1) * (size_t)(L + 1));
    reach[(size_t)no * (L + 1) + 0] = 1;
    for (int32_t k = no - 1; k >= 0; --k) {
      const int32_t gk = ex_g[pos[ord[k]]];
      for (int32_t s = 0; s <= L; ++s) {
        uint8_t v = reach[(size_t)(k + 1) * (L + 1) + s];
        if (!v && s >= gk) v = reach[(size_t)(k + 1) * (L + 1) + s - gk];
        reach[(size_t)k * (L + 1) + s] = v;
      }
    }
    int32_t target = L;
    while (target > 0 && !reach[target]) --target;       /* max achievable sum <= L (row k = 0) */
    int64_t gsum = target, dt = -1;
    for (int32_t k = 0; k < no; ++k) {                   /* lexicographic: include if still completable */
      const int32_t j = ord[k];
      const int32_t gk = ex_g[pos[j]];
      sel[j] = 0;
      if (gk <= target && reach[(size_t)(k + 1) * (L + 1) + target - gk]) {
        sel[j] = 1; target -= gk;
        if (dt < 0 || rem[j] < dt) dt = rem[j];
      }
    }
    if (dt <= 0) break;
    if (dt > T_us - t) dt = T_us - t;
    util += gsum * dt;
    t += dt;
    ++events;
    for (int32_t k = 0; k < no; ++k) {
      const int32_t j = ord[k];
      if (!sel[j]) continue;
      rem[j] -= dt;
      if (rem[j] > 0) continue;
      /* next execution of the chain (zero-duration executions complete instantly) */
      int64_t e = pos[j] + 1;
      while (e < chain_off[j + 1] && ex_tau[e] == 0) ++e;
      if (e >= chain_off[j + 1]) {                        /* batch done: next batch back-to-back */
        completed[j]++;
        bstart[j] = t;
        e = chain_off[j];
        while (ex_tau[e] == 0) ++e;
      }
      pos[j] = e; rem[j] = ex_tau[e];
    }
  }
  *util_out = util;
  if (events_out) *events_out = events;
  free(pos); free(rem); free(bstart); free(live); free(ord); free(sel); free(reach);
  return 0;
}

/* ------------------------------------------------------------- driver --- */

static void eval_scenario(const or_problem_t *pb, const or_params_t *p, or_out_t *o, int64_t s) {
  const int32_t k0 = pb->scen_dnn_off[s], k1 = pb->scen_dnn_off[s + 1];
  const int32_t nd = k1 - k0;
  for (int32_t k = k0; k < k1; ++k) {
    dnn_t m = get_dnn(pb, p, k);
    batch_opt_one(&m, p, o->demand + k, o->batch + k, o->knee + k, o->status + k);
    o->alloc_q16[k] = 0; o->level[k] = 0; o->runs[k] = 0; o->served[k] = 0;
  }
  o->scen_status[s] = OR_OK; o->T_us[s] = 0; o->u_static[s] = 0; o->u[s] = 0; o->thr[s] = 0;
  o->misses[s] = 0;
  if (o->below) o->below[s] = 0;
  if (o->u_ideal) o->u_ideal[s] = 0;
  if (o->thr_ideal) o->thr_ideal[s] = 0;
  if (nd > OR_MAX_DNN_PER_SCEN) { o->scen_status[s] = OR_INVALID; return; }
  if (nd <= 0) { o->scen_status[s] = OR_INFEASIBLE; return; }
  uint16_t dem[OR_MAX_DNN_PER_SCEN];
  uint32_t alloc[OR_MAX_DNN_PER_SCEN];
  for (int32_t j = 0; j < nd; ++j) dem[j] = (o->status[k0 + j] == OR_OK) ? o->demand[k0 + j] : 0;
  oracle_wmaxmin(nd, dem, p->L, alloc);
  int64_t T = 0;
  for (int32_t j = 0; j < nd; ++j) {
    o->alloc_q16[k0 + j] = alloc[j];
    if (dem[j] > 0 && pb->slo_us[k0 + j] > T) T = pb->slo_us[k0 + j];
  }
  if (T == 0) { o->scen_status[s] = OR_INFEASIBLE; return; }
  const int64_t nslots = T / p->slot_us;
  int64_t njobs = 0;
  for (int32_t j = 0; j < nd; ++j) if (dem[j] > 0) njobs += nslots / (pb->slo_us[k0 + j] / p->slot_us);
  if (nslots > OR_MAX_SLOTS || njobs > OR_MAX_JOBS) { o->scen_status[s] = OR_INVALID; return; }
  o->T_us[s] = (uint32_t)T;

  int32_t g[OR_MAX_DNN_PER_SCEN], sl[OR_MAX_DNN_PER_SCEN], bst[OR_MAX_DNN_PER_SCEN];
  int64_t dtab[OR_MAX_DNN_PER_SCEN * 64];
  for (int32_t j = 0; j < nd; ++j) {
    const int32_t k = k0 + j;
    g[j] = 0; sl[j] = pb->slo_us[k] / p->slot_us; bst[j] = o->batch[k];
    if (dem[j] == 0) continue;
    /* WMAX-MIN's share feeds the run's GPU%: g = max(demand, floor(alloc)) (DESIGN.md §3 reading) */
    int32_t al = (int32_t)(alloc[j] >> 16);
    g[j] = dem[j] > al ? dem[j] : al;
    o->level[k] = (uint16_t)g[j];
    dnn_t m = get_dnn(pb, p, k);
    const int64_t S = S_of(p, g[j]);
    const u128 den = (u128)S * (u128)m.M * (u128)p->slot_us;
    for (int32_t b = p->b_min; b <= bst[j]; ++b) {
      /* d_j(b) = ceil(f_L(g_j, b) / Delta) slots */
      u128 X = X_of(&m, p, S, b);
      u128 dd = (X + den - 1) / den;
      dtab[j * 64 + b - 1] = dd > (u128)0x7FFFFFFFFFFFLL ? 0x7FFFFFFFFFFFLL : (int64_t)dd;
    }
  }
  /* F1: run slots of the b* batch at every level below g_j, plus the launch latency of the new
     instance, ceil(reconf_us / Delta) slots (P:2821 switchover) */
  int64_t *dlow = NULL;
  if (p->below_knee) {
    dlow = (int64_t *)calloc((size_t)nd * 256, sizeof(int64_t));
    const int64_t c = ((int64_t)p->reconf_us + p->slot_us - 1) / p->slot_us;
    for (int32_t j = 0; j < nd; ++j) {
      if (g[j] == 0) continue;
      dnn_t m = get_dnn(pb, p, k0 + j);
      for (int32_t l = 1; l < g[j]; ++l) {
        const int64_t S = S_of(p, l);
        const u128 den = (u128)S * (u128)m.M * (u128)p->slot_us;
        u128 dd = (X_of(&m, p, S, bst[j]) + den - 1) / den + (u128)c;
        dlow[(int64_t)j * 256 + l] = dd > (u128)0x7FFFFFFFFFFFLL ? 0x7FFFFFFFFFFFLL : (int64_t)dd;
      }
    }
  }
  int32_t runs[OR_MAX_DNN_PER_SCEN], jmiss[OR_MAX_DNN_PER_SCEN];
  int64_t served[OR_MAX_DNN_PER_SCEN];
  or_cyc_sum_t cs;
  oracle_cycle_direct_bk(nd, g, sl, bst, dtab, dlow, p->b_min, p->L, (int32_t)nslots, runs, served, jmiss, &cs, 0,
                         NULL, NULL, NULL, NULL, NULL, NULL, NULL);
  free(dlow);
  if (o->below) o->below[s] = (uint32_t)cs.below;
  for (int32_t j = 0; j < nd; ++j) {
    o->runs[k0 + j] = (uint16_t)runs[j];
    o->served[k0 + j] = (uint32_t)served[j];
  }
  o->misses[s] = (uint32_t)cs.misses;
  if (cs.status != OR_OK) o->scen_status[s] = (uint8_t)cs.status;
  /* reported ratios: U = sum occ / (nslots L) (§6.1 "GPU utilization by using Knee%");
     throughput = served requests per second of session (P:2827 saturating load). */
  o->u_static[s] = (double)cs.occ_static_sum / ((double)nslots * (double)p->L);
  o->u[s] = (double)cs.occ_sum / ((double)nslots * (double)p->L);
  o->thr[s] = (double)cs.served_total * 1e6 / (double)T;

  if (p->ideal && o->u_ideal && o->thr_ideal) {
    int64_t tot_rows = 0;
    for (int32_t j = 0; j < nd; ++j)
      if (dem[j] > 0) {
        dnn_t m = get_dnn(pb, p, k0 + j);
        for (int64_t i = 0; i < m.K; ++i) tot_rows += m.r[i];
      }
    int64_t chain_off[OR_MAX_DNN_PER_SCEN + 1];
    int32_t *exg = (int32_t *)malloc(sizeof(int32_t) * (size_t)(tot_rows + 1));
    int64_t *ext = (int64_t *)malloc(sizeof(int64_t) * (size_t)(tot_rows + 1));
    int64_t slo[OR_MAX_DNN_PER_SCEN];
    uint8_t act[OR_MAX_DNN_PER_SCEN];
    int64_t comp[OR_MAX_DNN_PER_SCEN];
    int64_t e = 0;
    for (int32_t j = 0; j < nd; ++j) {
      chain_off[j] = e;
      slo[j] = pb->slo_us[k0 + j];
      act[j] = dem[j] > 0;
      if (!act[j]) continue;
      dnn_t m = get_dnn(pb, p, k0 + j);
      int32_t *gr = (int32_t *)malloc(sizeof(int32_t) * (size_t)m.K);
      int64_t *tr = (int64_t *)malloc(sizeof(int64_t) * (size_t)m.K);
      oracle_ideal_rows(pb, p, k0 + j, bst[j], gr, tr);
      for (int64_t i = 0; i < m.K; ++i)           /* chain: row i repeated R_i times, profile order */
        for (int32_t q = 0; q < m.r[i]; ++q) { exg[e] = gr[i]; ext[e] = tr[i]; ++e; }
      free(gr); free(tr);
    }
    chain_off[nd] = e;
    int64_t util = 0;
    oracle_ideal_direct(nd, chain_off, exg, ext, slo, bst, act, p->L, T, &util, comp, NULL);
    int64_t bsum = 0;
    for (int32_t j = 0; j < nd; ++j) bsum += comp[j] * bst[j];
    o->u_ideal[s] = (double)util / ((double)p->L * (double)T);
    o->thr_ideal[s] = (double)bsum * 1e6 / (double)T;
    free(exg); free(ext);
  }
}

static int check_params(const or_params_t *p) {
  if (p->L < 1 || p->L > 255 || p->S_tot < 1 || p->S_tot > 256 || p->slot_us < 1) return -1;
  if (p->mem_mode < 0 || p->mem_mode > 2 || p->par_mode < 0 || p->par_mode > 1) return -1;
  if (p->wse_mode < 0 || p->wse_mode > 1 || p->b_min < 1 || p->b_max > 64 || p->b_min > p->b_max) return -1;
  if (p->margin < 0 || p->margin > p->L) return -1;
  if (p->below_knee < 0 || p->below_knee > 1 || p->reconf_us < 0) return -1;
  return 0;
}

int oracle_eval(const or_problem_t *pb, const or_params_t *p, or_out_t *o, int32_t nthreads) {
  if (!pb || !p || !o || check_params(p)) return -1;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t s = 0; s < pb->num_scen; ++s) eval_scenario(pb, p, o, s);
  return 0;
}

int oracle_eval_subset(const or_problem_t *pb, const or_params_t *p, or_out_t *o, const int64_t *idx,
                       int64_t count, int32_t nthreads) {
  if (!pb || !p || !o || check_params(p)) return -1;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t q = 0; q < count; ++q) eval_scenario(pb, p, o, idx[q]);
  return 0;
}

/* O9 over every scenario: the five schedulers on the same a1-a4 outputs.
 * out[s*5 + c], c = 0 D-STACK, 1 Max-Min fair fill, 2 max-throughput fill, 3 temporal, 4 static spatial. */
static uint64_t jain_num(const int64_t *x, int32_t n, const int32_t *act, uint64_t *den) {
  uint64_t s1 = 0, s2 = 0, na = 0;
  for (int32_t j = 0; j < n; ++j) if (act[j]) { s1 += (uint64_t)x[j]; s2 += (uint64_t)(x[j] * x[j]); ++na; }
  *den = na * s2;
  return s1 * s1;
}
static double jain_of(const int64_t *x, int32_t n, const int32_t *act) {
  uint64_t den, num = jain_num(x, n, act, &den);
  return den ? (double)num / (double)den : 0.0;   /* Jain's index (sum x)^2 / (n sum x^2) */
}

/* scenario s's five columns into u[0..4], thr[0..4], jain[0..4] */
static void compare_one(const or_problem_t *pb, const or_params_t *p, int64_t s, double *u, double *thr,
                        double *jain) {
  for (int c = 0; c < 5; ++c) { u[c] = 0; thr[c] = 0; jain[c] = 0; }
  const int32_t k0 = pb->scen_dnn_off[s], nd = pb->scen_dnn_off[s + 1] - k0;
  if (nd <= 0 || nd > OR_MAX_DNN_PER_SCEN) return;
  uint16_t dem[OR_MAX_DNN_PER_SCEN], knee[OR_MAX_DNN_PER_SCEN];
  uint8_t bt[OR_MAX_DNN_PER_SCEN], st[OR_MAX_DNN_PER_SCEN];
  uint32_t alloc[OR_MAX_DNN_PER_SCEN];
  for (int32_t j = 0; j < nd; ++j) {
    dnn_t m = get_dnn(pb, p, k0 + j);
    batch_opt_one(&m, p, dem + j, bt + j, knee + j, st + j);
    if (st[j] != OR_OK) dem[j] = 0;
  }
  oracle_wmaxmin(nd, dem, p->L, alloc);
  int64_t T = 0;
  for (int32_t j = 0; j < nd; ++j) if (dem[j] > 0 && pb->slo_us[k0 + j] > T) T = pb->slo_us[k0 + j];
  if (T == 0) return;
  const int64_t nslots = T / p->slot_us;
  int64_t njobs = 0;
  for (int32_t j = 0; j < nd; ++j) if (dem[j] > 0) njobs += nslots / (pb->slo_us[k0 + j] / p->slot_us);
  if (nslots > OR_MAX_SLOTS || njobs > OR_MAX_JOBS) return;
  int32_t g[OR_MAX_DNN_PER_SCEN], sl[OR_MAX_DNN_PER_SCEN], bst[OR_MAX_DNN_PER_SCEN], act[OR_MAX_DNN_PER_SCEN];
  int32_t lvl[OR_MAX_DNN_PER_SCEN];
  int64_t dtab[OR_MAX_DNN_PER_SCEN * 64], dL[OR_MAX_DNN_PER_SCEN], dk[OR_MAX_DNN_PER_SCEN];
  for (int32_t j = 0; j < nd; ++j) {
    const int32_t k = k0 + j;
    g[j] = 0; lvl[j] = 0; sl[j] = pb->slo_us[k] / p->slot_us; bst[j] = bt[j]; act[j] = dem[j] > 0;
    dL[j] = 0; dk[j] = 0;
    if (!act[j]) continue;
    const int32_t al = (int32_t)(alloc[j] >> 16);
    g[j] = dem[j] > al ? dem[j] : al;
    lvl[j] = dem[j];
    dnn_t m = get_dnn(pb, p, k);
    const int64_t S = S_of(p, g[j]);
    const u128 den = (u128)S * (u128)m.M * (u128)p->slot_us;
    for (int32_t b = p->b_min; b <= bst[j]; ++b) {
      u128 dd = (X_of(&m, p, S, b) + den - 1) / den;
      dtab[j * 64 + b - 1] = dd > (u128)0x7FFFFFFFFFFFLL ? 0x7FFFFFFFFFFFLL : (int64_t)dd;
    }
    /* run time of one b* batch at 100% GPU (temporal) and at the knee level (static spatial) */
    const u128 denL = (u128)p->S_tot * (u128)m.M * (u128)p->slot_us;
    dL[j] = (int64_t)((X_of(&m, p, p->S_tot, bst[j]) + denL - 1) / denL);
    const int64_t Sk = S_of(p, dem[j]);
    const u128 denk = (u128)Sk * (u128)m.M * (u128)p->slot_us;
    dk[j] = (int64_t)((X_of(&m, p, Sk, bst[j]) + denk - 1) / denk);
  }
  const double NL = (double)nslots * (double)p->L;
  for (int32_t c = 0; c < 3; ++c) {
    int32_t runs[OR_MAX_DNN_PER_SCEN], jmiss[OR_MAX_DNN_PER_SCEN];
    int64_t served[OR_MAX_DNN_PER_SCEN], busy[OR_MAX_DNN_PER_SCEN];
    or_cyc_sum_t cs;
    cycle_core(nd, g, sl, bst, dtab, p->b_min, p->L, (int32_t)nslots, NULL, runs, served, jmiss, &cs, 0, NULL, NULL,
               NULL, NULL, NULL, NULL, NULL, NULL, c, busy, NULL, NULL);
    u[c] = (double)cs.occ_sum / NL;
    thr[c] = (double)cs.served_total * 1e6 / (double)T;
    jain[c] = jain_of(busy, nd, act);
  }
  {
    int64_t slice[OR_MAX_DNN_PER_SCEN], runs[OR_MAX_DNN_PER_SCEN], occn = 0, srv = 0;
    oracle_temporal_direct(nd, lvl, sl, dL, (int32_t)nslots, slice, runs, &occn);
    for (int32_t j = 0; j < nd; ++j) srv += runs[j] * bst[j];
    u[3] = (double)occn / NL;
    thr[3] = (double)srv * 1e6 / (double)T;
    jain[3] = jain_of(slice, nd, act);
  }
  {
    int32_t home[OR_MAX_DNN_PER_SCEN], K = 0;
    int64_t runs[OR_MAX_DNN_PER_SCEN], busy[OR_MAX_DNN_PER_SCEN], occn = 0, srv = 0;
    oracle_gslice_direct(nd, lvl, dk, (int32_t)nslots, p->L, home, &K, runs, busy, &occn);
    for (int32_t j = 0; j < nd; ++j) srv += runs[j] * bst[j];
    u[4] = (double)occn / NL;
    thr[4] = (double)srv * 1e6 / (double)T;
    jain[4] = jain_of(busy, nd, act);
  }
}

static void compare_scenario(const or_problem_t *pb, const or_params_t *p, int64_t s, double *u, double *thr,
                             double *jain) {
  compare_one(pb, p, s, u + s * 5, thr + s * 5, jain + s * 5);
}

int oracle_compare(const or_problem_t *pb, const or_params_t *p, double *u, double *thr, double *jain,
                   const int64_t *idx, int64_t count, int32_t nthreads) {
  if (!pb || !p || !u || !thr || !jain || check_params(p)) return -1;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
  const int64_t n = idx ? count : pb->num_scen;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t q = 0; q < n; ++q) compare_scenario(pb, p, idx ? idx[q] : q, u, thr, jain);
  return 0;
}

/* ------------------------------------------------------------ O9b ---
 * Max-throughput (§6.3): "a schedule that maximizes the sum of the throughput across all the models".
 * Reading R24: over one session of nslots slots, every active model j runs at its session level
 * g_j (the level D-STACK's session uses), as any sequence of non-overlapping runs of a batch b in [b_lo, b*_j]
 * lasting d_j(b) slots, starting at slot boundaries and ending by the session end, with the summed level of the
 * runs in progress <= L at every slot (Eq. 14); the value is the number of requests served, sum of b over all runs
 * (throughput = served / T).  No SLO window: it is the throughput ceiling D-STACK is compared with (any D-STACK
 * session is one such schedule, so D-STACK <= max-throughput).
 * Exhaustive search over the schedules, memoised on the state: r_j = slots left of model j's run in progress
 * (0 = idle).  V_t(r) = max over the starts at t (each idle model: none, or one batch b with t + d_j(b) <= nslots)
 * whose occupancy at t stays <= L, of (sum b of the starts) + V_{t+1}(r - 1); V_nslots = 0; the answer is V_0(0).
 * Returns -1 when the state space prod_j (max_b d_j(b) + 1) exceeds max_states (the instance is too large). */
int oracle_maxthr_direct(int32_t n, const int32_t *g, const int32_t *bstar, const int64_t *dtab, int32_t b_lo,
                         int32_t L, int32_t nslots, int64_t max_states, int64_t *best) {
  if (n < 0 || n > 16 || nslots < 0) return -1;
  int64_t D[16], radix[16], nst = 1;
  for (int32_t j = 0; j < n; ++j) {
    D[j] = 0;
    if (g[j] > 0)
      for (int32_t b = b_lo; b <= bstar[j]; ++b) if (dtab[(int64_t)j * 64 + b - 1] > D[j]) D[j] = dtab[(int64_t)j * 64 + b - 1];
    radix[j] = nst;
    if (D[j] + 1 > max_states) return -1;
    nst *= D[j] + 1;
    if (nst > max_states) return -1;
  }
  int64_t *V = (int64_t *)calloc((size_t)nst, sizeof(int64_t));      /* V_{t+1} */
  int64_t *W = (int64_t *)calloc((size_t)nst, sizeof(int64_t));      /* V_t */
  int64_t r[16], c[16];
  for (int32_t t = nslots - 1; t >= 0; --t) {
    for (int64_t st = 0; st < nst; ++st) {
      for (int32_t j = 0; j < n; ++j) r[j] = (st / radix[j]) % (D[j] + 1);
      /* every combination of choices: c[j] = 0 (keep / idle) or a batch b (an idle active model starts b) */
      for (int32_t j = 0; j < n; ++j) c[j] = 0;
      int64_t bestv = -1;
      while (1) {
        int64_t occ = 0, gain = 0, nxt = 0;
        int ok = 1;
        for (int32_t j = 0; j < n && ok; ++j) {
          int64_t rr = r[j];
          if (c[j] > 0) {                                   /* start a run of batch c[j] */
            const int64_t d = dtab[(int64_t)j * 64 + c[j] - 1];
            if (d < 1 || t + d > nslots) ok = 0;
            rr = d; gain += c[j];
          }
          if (rr > 0) occ += g[j];
          nxt += (rr > 0 ? rr - 1 : 0) * radix[j];
        }
        if (ok && occ <= L) {
          const int64_t v = gain + V[nxt];
          if (v > bestv) bestv = v;
        }
        /* next combination (odometer over the idle active models' choices 0, b_lo..b*) */
        int32_t j = 0;
        for (; j < n; ++j) {
          if (r[j] > 0 || g[j] <= 0) continue;
          if (c[j] == 0) { c[j] = b_lo; break; }
          if (c[j] < bstar[j]) { ++c[j]; break; }
          c[j] = 0;
        }
        if (j == n) break;
      }
      W[st] = bestv < 0 ? 0 : bestv;   /* a state whose running models alone exceed L is unreachable */
    }
    int64_t *tmp = V; V = W; W = tmp;
  }
  *best = nslots > 0 ? V[0] : 0;
  free(V); free(W);
  return 0;
}

/* O9b per scenario on the eval path's quantities (O3 demand / b*, O4 levels g_j, session T = max SLO, d_j(b) at g_j
 * from O1): served_out[q] = the max-throughput served count, st_out[q] = OR_OK, OR_INFEASIBLE (nothing servable)
 * or OR_INVALID (more than 8 active models, a session over OR_MAX_SLOTS, or a state space over max_states). */
int oracle_maxthr(const or_problem_t *pb, const or_params_t *p, int64_t max_states, int64_t *served_out,
                  uint8_t *st_out, int64_t *T_out, const int64_t *idx, int64_t count, int32_t nthreads) {
  if (!pb || !p || !served_out || !st_out || check_params(p)) return -1;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
  const int64_t nq = idx ? count : pb->num_scen;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t q = 0; q < nq; ++q) {
    const int64_t s = idx ? idx[q] : q;
    served_out[q] = 0; st_out[q] = OR_INVALID; if (T_out) T_out[q] = 0;
    const int32_t k0 = pb->scen_dnn_off[s], nd = pb->scen_dnn_off[s + 1] - k0;
    if (nd > OR_MAX_DNN_PER_SCEN) continue;
    uint16_t dem[OR_MAX_DNN_PER_SCEN], knee[OR_MAX_DNN_PER_SCEN];
    uint8_t bt[OR_MAX_DNN_PER_SCEN], st[OR_MAX_DNN_PER_SCEN];
    uint32_t alloc[OR_MAX_DNN_PER_SCEN];
    for (int32_t j = 0; j < nd; ++j) {
      dnn_t m = get_dnn(pb, p, k0 + j);
      batch_opt_one(&m, p, dem + j, bt + j, knee + j, st + j);
      if (st[j] != OR_OK) dem[j] = 0;
    }
    oracle_wmaxmin(nd, dem, p->L, alloc);
    int64_t T = 0;
    int32_t nact = 0;
    for (int32_t j = 0; j < nd; ++j) if (dem[j] > 0) { ++nact; if (pb->slo_us[k0 + j] > T) T = pb->slo_us[k0 + j]; }
    if (T == 0) { st_out[q] = OR_INFEASIBLE; continue; }
    const int64_t nslots = T / p->slot_us;
    if (nact > 8 || nslots > OR_MAX_SLOTS) continue;
    int32_t g[8], bst[8];
    int64_t dtab[8 * 64];
    int32_t n = 0;
    for (int32_t j = 0; j < nd; ++j) {
      if (dem[j] == 0) continue;
      const int32_t al = (int32_t)(alloc[j] >> 16);
      g[n] = dem[j] > al ? dem[j] : al;
      bst[n] = bt[j];
      dnn_t m = get_dnn(pb, p, k0 + j);
      const int64_t S = S_of(p, g[n]);
      const u128 den = (u128)S * (u128)m.M * (u128)p->slot_us;
      for (int32_t b = p->b_min; b <= bst[n]; ++b) {
        const u128 dd = (X_of(&m, p, S, b) + den - 1) / den;
        dtab[n * 64 + b - 1] = dd > (u128)0x7FFFFFFF ? 0x7FFFFFFF : (int64_t)dd;
      }
      ++n;
    }
    int64_t best = 0;
    if (oracle_maxthr_direct(n, g, bst, dtab, p->b_min, p->L, (int32_t)nslots, max_states, &best) != 0) continue;
    served_out[q] = best; st_out[q] = OR_OK;
    if (T_out) T_out[q] = T;
  }
  return 0;
}

/* ---------------------------------------------------------------- F4 ---
 * Multi-GPU cluster of §7.1 (reading R23): G modelled GPUs
 * of L levels each serve the scenario's active models (status OK).  out[s*4 + c]:
 *  c = 0 exclusive ("one T4 GPU for each DNN model exclusively"): the q-th active model (index order) runs on
 *        GPU q mod G; a GPU holding several models shares them temporally (O9 temporal on its subset);
 *  c = 1 temporal ("all 4 models in each GPU, temporally sharing the GPU"): every GPU runs O9 temporal over all
 *        models, the load spread over the G replicas;
 *  c = 2 D-STACK on every GPU ("D-STACK with the 4 DNN models"): every GPU runs the O5 session over all models;
 *  c = 3 D-STACK with placement: models first-fit decreasing by demand (desc, index) onto GPUs of capacity L,
 *        a model that fits nowhere to the least-loaded GPU (lowest index on ties); each GPU runs WMAX-MIN (O4) and
 *        one O5 session over its subset.
 * Per GPU i with a non-empty subset: T_i = max SLO over it, nslots_i = T_i / Delta, U_i = occupied level-slots /
 * (nslots_i L), throughput_i = served * 1e6 / T_i.  Cluster: U = sum_i U_i / G (an idle GPU counts 0),
 * throughput = sum_i throughput_i. */
static void cluster_scenario(const or_problem_t *pb, const or_params_t *p, int32_t G, int64_t s, double *u,
                             double *thr) {
  for (int c = 0; c < 4; ++c) { u[s * 4 + c] = 0; thr[s * 4 + c] = 0; }
  const int32_t k0 = pb->scen_dnn_off[s], nd = pb->scen_dnn_off[s + 1] - k0;
  if (nd <= 0 || nd > OR_MAX_DNN_PER_SCEN) return;
  uint16_t dem[OR_MAX_DNN_PER_SCEN], knee[OR_MAX_DNN_PER_SCEN];
  uint8_t bt[OR_MAX_DNN_PER_SCEN], st[OR_MAX_DNN_PER_SCEN];
  int32_t sl[OR_MAX_DNN_PER_SCEN];
  for (int32_t j = 0; j < nd; ++j) {
    dnn_t m = get_dnn(pb, p, k0 + j);
    batch_opt_one(&m, p, dem + j, bt + j, knee + j, st + j);
    if (st[j] != OR_OK) dem[j] = 0;
    sl[j] = pb->slo_us[k0 + j] / p->slot_us;
  }
  int64_t T = 0;
  for (int32_t j = 0; j < nd; ++j) if (dem[j] > 0 && pb->slo_us[k0 + j] > T) T = pb->slo_us[k0 + j];
  if (T == 0) return;
  {
    const int64_t nslots = T / p->slot_us;
    int64_t njobs = 0;
    for (int32_t j = 0; j < nd; ++j) if (dem[j] > 0) njobs += nslots / sl[j];
    if (nslots > OR_MAX_SLOTS || njobs > OR_MAX_JOBS) return;   /* the scenario is INVALID for the session */
  }
  /* c = 1, 2: every GPU runs the whole mix: the single-GPU O9 temporal / D-STACK numbers, G replicas */
  {
    double cu[5], ct[5], cj[5];
    compare_one(pb, p, s, cu, ct, cj);
    u[s * 4 + 1] = cu[3]; thr[s * 4 + 1] = (double)G * ct[3];
    u[s * 4 + 2] = cu[0]; thr[s * 4 + 2] = (double)G * ct[0];
  }
  /* placements for c = 0 (round robin over active models) and c = 3 (first-fit decreasing by demand) */
  int32_t home0[OR_MAX_DNN_PER_SCEN], home3[OR_MAX_DNN_PER_SCEN];
  {
    int32_t q = 0;
    for (int32_t j = 0; j < nd; ++j) home0[j] = dem[j] > 0 ? (q++) % G : -1;
    int32_t ord[OR_MAX_DNN_PER_SCEN], na = 0;
    for (int32_t j = 0; j < nd; ++j) { home3[j] = -1; if (dem[j] > 0) ord[na++] = j; }
    for (int32_t i = 1; i < na; ++i) {   /* (demand desc, index asc) */
      int32_t v = ord[i], k = i - 1;
      while (k >= 0 && (dem[ord[k]] < dem[v] || (dem[ord[k]] == dem[v] && ord[k] > v))) { ord[k + 1] = ord[k]; --k; }
      ord[k + 1] = v;
    }
    int64_t load[64] = {0};
    for (int32_t i = 0; i < na; ++i) {
      const int32_t j = ord[i];
      int32_t gi = -1;
      for (int32_t c = 0; c < G; ++c) if (load[c] + dem[j] <= p->L) { gi = c; break; }   /* first fit */
      if (gi < 0) { gi = 0; for (int32_t c = 1; c < G; ++c) if (load[c] < load[gi]) gi = c; }   /* least loaded */
      home3[j] = gi;
      load[gi] += dem[j];
    }
  }
  for (int32_t gi = 0; gi < G; ++gi) {
    /* c = 0: O9 temporal over the models on GPU gi */
    {
      int64_t Ti = 0;
      for (int32_t j = 0; j < nd; ++j) if (home0[j] == gi && pb->slo_us[k0 + j] > Ti) Ti = pb->slo_us[k0 + j];
      if (Ti > 0) {
        const int32_t ns = (int32_t)(Ti / p->slot_us);
        int32_t lvl[OR_MAX_DNN_PER_SCEN];
        int64_t dL[OR_MAX_DNN_PER_SCEN], slice[OR_MAX_DNN_PER_SCEN], runs[OR_MAX_DNN_PER_SCEN], occn = 0, srv = 0;
        for (int32_t j = 0; j < nd; ++j) {
          lvl[j] = home0[j] == gi ? dem[j] : 0;
          dL[j] = 0;
          if (!lvl[j]) continue;
          dnn_t m = get_dnn(pb, p, k0 + j);
          const u128 denL = (u128)p->S_tot * (u128)m.M * (u128)p->slot_us;   /* b* batch at 100% GPU */
          dL[j] = (int64_t)((X_of(&m, p, p->S_tot, bt[j]) + denL - 1) / denL);
        }
        oracle_temporal_direct(nd, lvl, sl, dL, ns, slice, runs, &occn);
        for (int32_t j = 0; j < nd; ++j) srv += runs[j] * bt[j];
        u[s * 4 + 0] += (double)occn / ((double)ns * (double)p->L) / (double)G;
        thr[s * 4 + 0] += (double)srv * 1e6 / (double)Ti;
      }
    }
    /* c = 3: WMAX-MIN and one D-STACK session over the models placed on GPU gi */
    {
      int64_t Ti = 0;
      for (int32_t j = 0; j < nd; ++j) if (home3[j] == gi && pb->slo_us[k0 + j] > Ti) Ti = pb->slo_us[k0 + j];
      if (Ti > 0) {
        const int32_t ns = (int32_t)(Ti / p->slot_us);
        uint16_t sd[OR_MAX_DNN_PER_SCEN];
        uint32_t sa[OR_MAX_DNN_PER_SCEN];
        int32_t idx[OR_MAX_DNN_PER_SCEN], nsub = 0;
        for (int32_t j = 0; j < nd; ++j) if (home3[j] == gi) { idx[nsub] = j; sd[nsub] = dem[j]; ++nsub; }
        oracle_wmaxmin(nsub, sd, p->L, sa);
        int32_t g[OR_MAX_DNN_PER_SCEN], bst[OR_MAX_DNN_PER_SCEN];
        int64_t dtab[OR_MAX_DNN_PER_SCEN * 64];
        for (int32_t j = 0; j < nd; ++j) { g[j] = 0; bst[j] = bt[j] > 0 ? bt[j] : 1; }
        for (int32_t q = 0; q < nsub; ++q) {
          const int32_t j = idx[q];
          const int32_t al = (int32_t)(sa[q] >> 16);
          g[j] = dem[j] > al ? dem[j] : al;
          dnn_t m = get_dnn(pb, p, k0 + j);
          const int64_t S = S_of(p, g[j]);
          const u128 den = (u128)S * (u128)m.M * (u128)p->slot_us;
          for (int32_t b = p->b_min; b <= bt[j]; ++b) {
            const u128 dd = (X_of(&m, p, S, b) + den - 1) / den;
            dtab[j * 64 + b - 1] = dd > (u128)0x7FFFFFFFFFFFLL ? 0x7FFFFFFFFFFFLL : (int64_t)dd;
          }
        }
        int32_t runs[OR_MAX_DNN_PER_SCEN], jmiss[OR_MAX_DNN_PER_SCEN];
        int64_t served[OR_MAX_DNN_PER_SCEN];
        or_cyc_sum_t cs;
        cycle_core(nd, g, sl, bst, dtab, p->b_min, p->L, ns, NULL, runs, served, jmiss, &cs, 0, NULL, NULL, NULL, NULL,
                   NULL, NULL, NULL, NULL, 0, NULL, NULL, NULL);
        u[s * 4 + 3] += (double)cs.occ_sum / ((double)ns * (double)p->L) / (double)G;
        thr[s * 4 + 3] += (double)cs.served_total * 1e6 / (double)Ti;
      }
    }
  }
}

int oracle_cluster(const or_problem_t *pb, const or_params_t *p, int32_t G, double *u, double *thr,
                   const int64_t *idx, int64_t count, int32_t nthreads) {
  if (!pb || !p || !u || !thr || check_params(p) || G < 1 || G > 64) return -1;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
  const int64_t n = idx ? count : pb->num_scen;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t q = 0; q < n; ++q) cluster_scenario(pb, p, G, idx ? idx[q] : q, u, thr);
  return 0;
}

/* ---------------------------------------------------------------- O7 --- */

/* Arrival cursor of one DNN's Poisson stream (input generator, synth_core.h): index of the next arrival
 * and its absolute time in us. */
typedef struct { uint64_t idx, time, mean_q32; uint64_t seed; int32_t cfg; int64_t gs; uint32_t j; } arr_t;

static void arr_init(arr_t *a, uint64_t seed, int32_t cfg, int64_t gs, uint32_t j, uint64_t mean_q32) {
  a->seed = seed; a->cfg = cfg; a->gs = gs; a->j = j; a->mean_q32 = mean_q32; a->idx = 0;
  a->time = sy_arrival_gap(mean_q32, sy_arrival_word(seed, cfg, gs, j, 0));
}
static void arr_next(arr_t *a) {
  a->idx++;
  a->time += sy_arrival_gap(a->mean_q32, sy_arrival_word(a->seed, a->cfg, a->gs, a->j, (uint32_t)a->idx));
}
/* A(t): number of arrivals with time <= t */
static uint64_t arr_count(arr_t *a, uint64_t t) {
  while (a->time <= t) arr_next(a);
  return a->idx;
}

static int run_cmp(const void *x, const void *y) {
  const run_t *a = (const run_t *)x, *b = (const run_t *)y;
  if (a->j != b->j) return a->j < b->j ? -1 : 1;
  return a->start < b->start ? -1 : (a->start > b->start);
}

/* O7 -- long-horizon simulation (config 5, readings in DESIGN.md §3):
 *  cycle c spans [c T, (c+1) T), T = max SLO over the servable DNNs (status OK);
 *  Poisson arrivals, mean gap = f_L(l*, b*) / (lam_pct/100 * b_star) (load as a fraction of standalone
 *  capacity b_star / f_L); at each cycle start the active DNNs are those with queued requests; WMAX-MIN over
 *  their demands ("dynamic re-allocation"); one O5 session with the fill ordered by the scoreboard
 *  (runs in the last 10 sessions + this one); the runs then execute in time order, each serving
 *  FIFO min(planned batch, queue at its start) requests; a run that finds an empty queue is void (not
 *  counted, no occupancy).  A request is late iff completion - arrival > SLO; requests still queued at
 *  the horizon are unserved (both are SLO violations). */
static void simulate_scenario(const or_problem_t *pb, const or_params_t *p, const int32_t *lam_pct, int32_t cycles,
                              uint64_t seed, int32_t cfg_tag, int64_t scen_base, or_sim_out_t *o, int64_t s) {
  const int32_t k0 = pb->scen_dnn_off[s], k1 = pb->scen_dnn_off[s + 1];
  const int32_t nd = k1 - k0;
  o->status[s] = OR_OK; o->T_us[s] = 0; o->arrived[s] = 0; o->in_slo[s] = 0; o->late[s] = 0;
  o->unserved[s] = 0; o->occ_sum[s] = 0; o->runs[s] = 0; o->misses[s] = 0; o->realloc[s] = 0;
  if (nd > OR_MAX_DNN_PER_SCEN) { o->status[s] = OR_INVALID; return; }
  if (nd <= 0) { o->status[s] = OR_INFEASIBLE; return; }
  uint16_t dem[OR_MAX_DNN_PER_SCEN], knee[OR_MAX_DNN_PER_SCEN];
  uint8_t bst8[OR_MAX_DNN_PER_SCEN], st[OR_MAX_DNN_PER_SCEN];
  int64_t T = 0;
  for (int32_t j = 0; j < nd; ++j) {
    dnn_t m = get_dnn(pb, p, k0 + j);
    batch_opt_one(&m, p, dem + j, bst8 + j, knee + j, st + j);
    if (st[j] == OR_OK && pb->slo_us[k0 + j] > T) T = pb->slo_us[k0 + j];
  }
  if (T == 0) { o->status[s] = OR_INFEASIBLE; return; }
  const int64_t nslots = T / p->slot_us;
  int64_t njobs = 0;
  for (int32_t j = 0; j < nd; ++j) if (st[j] == OR_OK) njobs += nslots / (pb->slo_us[k0 + j] / p->slot_us);
  if (nslots > OR_MAX_SLOTS || njobs > OR_MAX_JOBS) { o->status[s] = OR_INVALID; return; }
  o->T_us[s] = (uint32_t)T;
  arr_t arr[OR_MAX_DNN_PER_SCEN], head[OR_MAX_DNN_PER_SCEN];
  uint64_t served[OR_MAX_DNN_PER_SCEN];
  int64_t ring[10][OR_MAX_DNN_PER_SCEN], sb[OR_MAX_DNN_PER_SCEN];
  memset(ring, 0, sizeof(ring)); memset(sb, 0, sizeof(sb));
  for (int32_t j = 0; j < nd; ++j) {
    served[j] = 0;
    if (st[j] != OR_OK) continue;
    /* mean gap (us) = f_L(l*, b*) * 100 / (lam_pct * b*),  f_L = X / (S M); Q32, capped at 2^30 us */
    dnn_t m = get_dnn(pb, p, k0 + j);
    const int64_t ls = dem[j] - p->margin > 0 ? dem[j] - p->margin : 1;   /* l* (demand = l* + margin) */
    const int64_t S = S_of(p, ls);
    const u128 X = X_of(&m, p, S, bst8[j]);
    /* lam_pct <= 0: no offered load, the gap is infinite and takes the 2^30 us cap (R25) */
    const int32_t lam = lam_pct[k0 + j];
    const u128 den = lam > 0 ? (u128)S * (u128)m.M * (u128)lam * (u128)bst8[j] : 0;
    u128 mq = den ? ((X * 100) << 32) / den : (u128)1 << 62;
    if (mq > ((u128)1 << 62)) mq = (u128)1 << 62;
    arr_init(arr + j, seed, cfg_tag, scen_base + s, (uint32_t)j, (uint64_t)mq);
    arr_init(head + j, seed, cfg_tag, scen_base + s, (uint32_t)j, (uint64_t)mq);
  }
  int32_t g[OR_MAX_DNN_PER_SCEN], sl[OR_MAX_DNN_PER_SCEN], bst[OR_MAX_DNN_PER_SCEN];
  int64_t dtab[OR_MAX_DNN_PER_SCEN * 64];
  uint16_t dm[OR_MAX_DNN_PER_SCEN];
  uint32_t alloc[OR_MAX_DNN_PER_SCEN];
  uint8_t prev_act[OR_MAX_DNN_PER_SCEN];
  memset(prev_act, 0, sizeof(prev_act));
  for (int32_t c = 0; c < cycles; ++c) {
    const uint64_t t0 = (uint64_t)c * (uint64_t)T;
    for (int32_t j = 0; j < nd; ++j) {
      dm[j] = 0;
      if (st[j] != OR_OK) continue;
      const uint64_t A = arr_count(arr + j, t0);
      if (A > served[j]) dm[j] = dem[j];                 /* active: requests queued at the cycle start */
    }
    int changed = 0;                                       /* the active set moved: WMAX-MIN re-allocates */
    uint64_t nact = 0;
    for (int32_t j = 0; j < nd; ++j) {
      changed |= (dm[j] > 0) != prev_act[j]; prev_act[j] = dm[j] > 0;
      nact += dm[j] > 0;
    }
    if (c > 0) o->realloc[s] += (uint64_t)changed;
    const uint64_t in0 = o->in_slo[s], late0 = o->late[s], occ0 = o->occ_sum[s], runs0 = o->runs[s];
    uint64_t srv0 = 0;
    for (int32_t j = 0; j < nd; ++j) srv0 += served[j];
    oracle_wmaxmin(nd, dm, p->L, alloc);
    for (int32_t j = 0; j < nd; ++j) {
      g[j] = 0; sl[j] = pb->slo_us[k0 + j] / p->slot_us; bst[j] = bst8[j];
      if (dm[j] == 0) continue;
      const int32_t al = (int32_t)(alloc[j] >> 16);
      g[j] = dm[j] > al ? dm[j] : al;
      dnn_t m = get_dnn(pb, p, k0 + j);
      const int64_t S = S_of(p, g[j]);
      const u128 den = (u128)S * (u128)m.M * (u128)p->slot_us;
      for (int32_t b = p->b_min; b <= bst[j]; ++b) {
        const u128 X = X_of(&m, p, S, b);
        const u128 dd = (X + den - 1) / den;
        dtab[j * 64 + b - 1] = dd > (u128)0x7FFFFFFFFFFFLL ? 0x7FFFFFFFFFFFLL : (int64_t)dd;
      }
    }
    int32_t runs[OR_MAX_DNN_PER_SCEN], jmiss[OR_MAX_DNN_PER_SCEN];
    int64_t srv[OR_MAX_DNN_PER_SCEN];
    or_cyc_sum_t cs;
    run_t *rl = NULL;
    int64_t nrun = 0;
    cycle_core(nd, g, sl, bst, dtab, p->b_min, p->L, (int32_t)nslots, sb, runs, srv, jmiss, &cs, 0, NULL, NULL,
               NULL, NULL, NULL, NULL, &rl, &nrun, 0, NULL, NULL, NULL);
    o->misses[s] += (uint64_t)cs.misses;
    int64_t nfill = 0;
    for (int64_t q = 0; q < nrun; ++q) nfill += rl[q].kind == 1;
    if (nfill > OR_MAX_FILL_RUNS) {                       /* ABI capacity limit: scenario INVALID */
      free(rl);
      o->status[s] = OR_INVALID; o->T_us[s] = 0; o->in_slo[s] = o->late[s] = o->occ_sum[s] = o->runs[s] = 0;
      o->misses[s] = 0; o->realloc[s] = 0;
      return;
    }
    qsort(rl, (size_t)nrun, sizeof(run_t), run_cmp);     /* per DNN, in start order */
    int64_t cnt[OR_MAX_DNN_PER_SCEN];
    for (int32_t j = 0; j < nd; ++j) cnt[j] = 0;
    for (int64_t q = 0; q < nrun; ++q) {
      const int32_t j = rl[q].j;
      const uint64_t ts = t0 + (uint64_t)rl[q].start * (uint64_t)p->slot_us;
      const uint64_t te = t0 + (uint64_t)rl[q].end * (uint64_t)p->slot_us;
      const uint64_t A = arr_count(arr + j, ts);
      uint64_t k = A - served[j];
      if (k > (uint64_t)rl[q].batch) k = (uint64_t)rl[q].batch;
      if (k == 0) continue;                               /* empty queue: the run is void */
      for (uint64_t i = 0; i < k; ++i) {
        if (te - head[j].time > (uint64_t)pb->slo_us[k0 + j]) o->late[s]++; else o->in_slo[s]++;
        arr_next(head + j);
      }
      served[j] += k;
      cnt[j]++;
      o->occ_sum[s] += (uint64_t)g[j] * (uint64_t)(rl[q].end - rl[q].start);
      o->runs[s]++;
    }
    free(rl);
    for (int32_t j = 0; j < nd; ++j) { sb[j] += cnt[j] - ring[c % 10][j]; ring[c % 10][j] = cnt[j]; }
    if (o->series) {   /* this session's row of the per-cycle series (a completed session only) */
      uint64_t srv = 0;
      for (int32_t j = 0; j < nd; ++j) srv += served[j];
      const uint64_t v[8] = {nact, (uint64_t)(c > 0 && changed), o->runs[s] - runs0, srv - srv0,
                             o->in_slo[s] - in0, o->late[s] - late0, o->occ_sum[s] - occ0, (uint64_t)cs.misses};
      for (int f = 0; f < 8; ++f) {
#pragma omp atomic
        o->series[(int64_t)c * 8 + f] += v[f];
      }
    }
  }
  const uint64_t tend = (uint64_t)cycles * (uint64_t)T;
  for (int32_t j = 0; j < nd; ++j) {
    if (st[j] != OR_OK) continue;
    const uint64_t A = arr_count(arr + j, tend);
    o->arrived[s] += A;
    o->unserved[s] += A - served[j];
  }
}

int oracle_simulate(const or_problem_t *pb, const or_params_t *p, const int32_t *lam_pct, int32_t cycles,
                    uint64_t seed, int32_t cfg_tag, int64_t scen_base, or_sim_out_t *o, const int64_t *scen_idx,
                    int64_t count, int32_t nthreads) {
  if (!pb || !p || !o || !lam_pct || cycles < 0 || check_params(p)) return -1;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
  const int64_t n = scen_idx ? count : pb->num_scen;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t q = 0; q < n; ++q)
    simulate_scenario(pb, p, lam_pct, cycles, seed, cfg_tag, scen_base, o, scen_idx ? scen_idx[q] : q);
  return 0;
}
