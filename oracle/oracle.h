/* oracle.h -- CPU ORACLE for the D-STACK batched scheduling-model path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2304_13541_b200/, libdstack.so) never links,
 * imports or executes anything under oracle/, and shares no code with it
 * (its own structs, constants and arithmetic are written independently).
 *
 * Every function is the plain definition from PAPER.md (P:n = line n), in
 * the reading fixed by SURVEY.md §8(c) O1-O6 and listed in DESIGN.md §3:
 * exact integer arithmetic (unsigned __int128) for every decision,
 * brute-force grids, slot-by-slot loops.  All pointers are HOST pointers.
 */
#ifndef DSTACK_ORACLE_H
#define DSTACK_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status values (same meaning as the product ABI, defined here independently). */
enum { OR_OK = 0, OR_INFEASIBLE = 1, OR_OVERFLOW = 2, OR_INVALID = 3, OR_OVERSUBSCRIBED = 4 };

/* Capacity limits that the ABI documents as INVALID conditions. */
#define OR_MAX_DNN_PER_SCEN 32
#define OR_MAX_SLOTS 4096
#define OR_MAX_JOBS 512
#define OR_MAX_ROWS_PER_DNN 65535
#define OR_MAX_FILL_RUNS 2048   /* O7: fill runs per session */

typedef struct {
  int32_t num_scen, num_dnn;
  const int32_t *scen_dnn_off;       /* [num_scen+1] */
  const int64_t *dnn_row_off;        /* [num_dnn+1] */
  const int32_t *t_p, *t_np, *mem_bw, *slo_us, *asm_us, *bmax;   /* [num_dnn] */
  const uint32_t *n; const uint16_t *r; const uint32_t *d;         /* [num_rows] */
} or_problem_t;

typedef struct {
  int32_t L, S_tot, slot_us;
  int32_t mem_mode;   /* 0 off, 1 bw (E_m = d/(M S)), 2 verbatim (E_m = d S / M) */
  int32_t margin;     /* over-provisioning in levels */
  int32_t par_mode;   /* 0 linear N_i(b) = b n_i; 1 threads N_i(b) = ceil(b theta_i / 2048) */
  int32_t wse_mode;   /* 0 per_request (Eq. 4 printed), 1 per_launch */
  int32_t b_min, b_max;
  int32_t ideal;      /* 1: run the ideal per-kernel scheduler (O6) */
  int32_t below_knee; /* 1: F1 below-knee fallback for unplaced static jobs */
  int32_t reconf_us;  /* F1: launch latency of an instance at a lower GPU% (switchover), us >= 0 */
} or_params_t;

typedef struct {
  /* per DNN [num_dnn] */
  uint16_t *demand; uint8_t *batch; uint16_t *knee; uint8_t *status;
  uint32_t *alloc_q16; uint16_t *level; uint16_t *runs; uint32_t *served;
  /* per scenario [num_scen] */
  uint8_t *scen_status; uint32_t *T_us; double *u_static; double *u; double *thr;
  uint32_t *misses; double *u_ideal; double *thr_ideal;
  uint32_t *below;    /* F1: static jobs placed below the knee (nullable) */
} or_out_t;

/* O1: X(l, b) = E_t * S * M for DNN `dnn` (Eqs. 1-5), returned as lo/hi 64-bit halves. */
int oracle_X(const or_problem_t *pb, const or_params_t *p, int64_t dnn, int32_t l, int32_t b,
             uint64_t *lo, uint64_t *hi);
/* O2: knee(b) for every DNN (Eq. 6); st_out gets the validation status (knee valid iff OK). */
int oracle_knee(const or_problem_t *pb, const or_params_t *p, int32_t b, uint16_t *knee_out, uint8_t *st_out);
/* F3: online knee discovery by binary search from 30%.  probes_out = steps;
 * trace (nullable): [num_dnn * 16] probed levels per step. */
int oracle_knee_probe(const or_problem_t *pb, const or_params_t *p, int32_t b, uint16_t *knee_out, uint8_t *probes_out,
                      uint8_t *st_out, int32_t *trace);
/* O3: batch/GPU% optimisation (Eqs. 7-12) for every DNN. */
int oracle_batch_opt(const or_problem_t *pb, const or_params_t *p, uint16_t *demand, uint8_t *batch,
                     uint16_t *knee, uint8_t *status);
/* O4: WMAX-MIN, Q16.16 fixed point. */
int oracle_wmaxmin(int32_t n, const uint16_t *demand, int32_t L, uint32_t *alloc_q16);

/* O5 with direct per-DNN inputs (test hook; also used internally).
 * dtab[j*64 + b-1] = d_j(b) in slots for b in [b_lo, bstar_j]. g_j == 0 => inactive.
 * count0 (nullable): initial fill-priority counts (config-5 scoreboard); NULL = 0.
 * Trace (optional, cap may be 0): one entry per placed run. kind 0 static, 1 fill. */
typedef struct {
  int64_t occ_static_sum, occ_sum, served_total;
  int32_t misses, status;
  int32_t trace_n;
  int32_t below;      /* F1: static jobs placed below the knee (kind 2 in the trace) */
} or_cyc_sum_t;
int oracle_cycle_direct(int32_t n, const int32_t *g, const int32_t *sl_slots, const int32_t *bstar,
                        const int64_t *dtab, int32_t b_lo, int32_t L, int32_t nslots, const int64_t *count0,
                        int32_t *runs, int64_t *served, int32_t *jmiss, or_cyc_sum_t *sum,
                        int32_t trace_cap, int32_t *tr_dnn, int32_t *tr_start, int32_t *tr_end,
                        int32_t *tr_batch, int32_t *tr_kind, int32_t *tr_rep);

/* O5 with a fill order (O9 comparison schedulers): 0 D-STACK (runs so far, index), 1 Max-Min fair (g, index),
 * 2 max-throughput (d_j(b*), index).  busy (nullable): per DNN, slots covered by its runs. */
int oracle_cycle_direct_ex(int32_t n, const int32_t *g, const int32_t *sl, const int32_t *bstar,
                           const int64_t *dtab, int32_t b_lo, int32_t L, int32_t nslots, const int64_t *count0,
                           int32_t fill_order, int32_t *runs, int64_t *served, int32_t *jmiss, int64_t *busy,
                           or_cyc_sum_t *sum, int32_t trace_cap, int32_t *tr_dnn, int32_t *tr_start, int32_t *tr_end,
                           int32_t *tr_batch, int32_t *tr_kind, int32_t *tr_rep);

/* O5 + F1 below-knee fallback.  dlow[j*256 + l] = run slots of DNN j's b* batch at
 * level l < g_j including the launch latency (0 = level unusable); an unplaced static job is retried at
 * l = g_j - 1 .. 1 and placed at the first level with a feasible start (trace kind 2, tr_level = l). */
int oracle_cycle_direct_bk(int32_t n, const int32_t *g, const int32_t *sl, const int32_t *bstar, const int64_t *dtab,
                           const int64_t *dlow, int32_t b_lo, int32_t L, int32_t nslots, int32_t *runs,
                           int64_t *served, int32_t *jmiss, or_cyc_sum_t *sum, int32_t trace_cap, int32_t *tr_dnn,
                           int32_t *tr_start, int32_t *tr_end, int32_t *tr_batch, int32_t *tr_kind, int32_t *tr_rep,
                           int32_t *tr_level);

/* O9 temporal sharing: lvl[j] > 0 active (knee level), sl[j] SLO in slots, dL[j] run slots at 100% GPU.
 * slice_out, runs_out per DNN; *occ_num = sum slice_j * lvl_j (utilisation numerator). */
int oracle_temporal_direct(int32_t n, const int32_t *lvl, const int32_t *sl, const int64_t *dL, int32_t nslots,
                           int64_t *slice_out, int64_t *runs_out, int64_t *occ_num);
/* O9 static spatial sharing (GSLICE CSS): home[j] = -1 resident in all slots, >= 0 its slot, -2 inactive. */
int oracle_gslice_direct(int32_t n, const int32_t *lvl, const int64_t *dk, int32_t nslots, int32_t L,
                         int32_t *home, int32_t *nbins, int64_t *runs_out, int64_t *busy_out, int64_t *occ_num);
/* O9 over every scenario (idx NULL) or the listed ones: out[s*5 + c], c = 0 D-STACK, 1 Max-Min fair,
 * 2 max-throughput, 3 temporal, 4 static spatial; U, throughput (req/s), Jain fairness of GPU time. */
int oracle_compare(const or_problem_t *pb, const or_params_t *p, double *u, double *thr, double *jain,
                   const int64_t *idx, int64_t count, int32_t nthreads);

/* F4 multi-GPU cluster of §7.1: G modelled GPUs; out[s*4 + c], c = 0 exclusive (round robin,
 * temporal within a GPU), 1 temporal on every GPU, 2 D-STACK on every GPU, 3 D-STACK with first-fit-decreasing
 * placement; U = mean over the G GPUs, throughput = sum (req/s). */
int oracle_maxthr_direct(int32_t n, const int32_t *g, const int32_t *bstar, const int64_t *dtab, int32_t b_lo,
                         int32_t L, int32_t nslots, int64_t max_states, int64_t *best);
int oracle_maxthr(const or_problem_t *pb, const or_params_t *p, int64_t max_states, int64_t *served_out,
                  uint8_t *st_out, int64_t *T_out, const int64_t *idx, int64_t count, int32_t nthreads);
int oracle_cluster(const or_problem_t *pb, const or_params_t *p, int32_t G, double *u, double *thr,
                   const int64_t *idx, int64_t count, int32_t nthreads);

/* O6 with direct per-DNN chains (test hook; also used internally).
 * chain_off[j]..chain_off[j+1] index executions (g_e levels, tau_e us) of DNN j's batch,
 * slo_us[j], bstar[j]; active[j] != 0.  Returns util (sum g*dt) and completed batches. */
int oracle_ideal_direct(int32_t n, const int64_t *chain_off, const int32_t *ex_g, const int64_t *ex_tau,
                        const int64_t *slo_us, const int32_t *bstar, const uint8_t *active, int32_t L,
                        int64_t T_us, int64_t *util_out, int64_t *completed /*[n]*/, int64_t *events_out);

/* Per-kernel ideal demand/duration for the rows of DNN `dnn` at batch b (O6 setup). */
int oracle_ideal_rows(const or_problem_t *pb, const or_params_t *p, int64_t dnn, int32_t b,
                      int32_t *g_out, int64_t *tau_out);

/* O7 long-horizon simulation (config 5).  Per scenario outputs [num_scen]. */
typedef struct {
  uint8_t *status; uint32_t *T_us;
  uint64_t *arrived, *in_slo, *late, *unserved, *occ_sum, *runs, *misses;
  uint64_t *realloc;   /* sessions 2..cycles whose active set differs from the previous session's */
  uint64_t *series;    /* optional [cycles][8] per-cycle sums over the scenarios (dstack_sim_out_t.series order):
                          active DNNs, realloc, runs, served, in SLO, late, occupied level-slots, misses */
} or_sim_out_t;
int oracle_simulate(const or_problem_t *pb, const or_params_t *p, const int32_t *lam_pct, int32_t cycles,
                    uint64_t seed, int32_t cfg_tag, int64_t scen_base, or_sim_out_t *out, const int64_t *scen_idx,
                    int64_t count, int32_t nthreads);

/* Whole path a1-a6 over every scenario (OpenMP over scenarios, nthreads <= 0 => default). */
int oracle_eval(const or_problem_t *pb, const or_params_t *p, or_out_t *out, int32_t nthreads);

/* Same, over an explicit list of scenario indices (stratified samples). Outputs indexed as in full arrays. */
int oracle_eval_subset(const or_problem_t *pb, const or_params_t *p, or_out_t *out, const int64_t *scen_idx,
                       int64_t count, int32_t nthreads);

#ifdef __cplusplus
}
#endif
#endif
