/* dstack.h -- C-ABI of libdstack: batched evaluation of D-STACK's scheduling models on B200.
 *
 * Paper: D-STACK (arXiv 2304.13541), /root/reference/PAPER.md; P:n = line n.
 * The library evaluates, for very many independent synthetic multi-DNN scenarios, the path
 *   a1-a2  knee model            Eqs. 1-6, §4.3
 *   a3     batch/GPU% search     Eqs. 7-12, §5
 *   a4     WMAX-MIN allocation   Algorithm WMAX-MIN
 *   a5     one D-STACK session   Alg. 1 + Alg. 3 + dynamic fill, §6.1
 *   a6     ideal per-kernel scheduler (optional)  §6.2, Eqs. 13-14
 *   a8     aggregate statistics
 * in the readings listed in DESIGN.md §3.
 *
 * CONVENTIONS (every call):
 *  - Pointers inside the structs and array arguments are DEVICE pointers, owned by the caller
 *    (e.g. torch tensor data_ptr()).  The structs themselves are host memory, read during the call.
 *  - Every call is asynchronous on `stream` (a cudaStream_t; NULL = legacy default stream).
 *    Inputs must stay alive and unmodified, outputs untouched, until the stream is synchronised.
 *  - No call allocates device memory.  Scratch comes from the caller's workspace of
 *    >= dstack_workspace_size() bytes (256-byte aligned); ws may be NULL when that size is 0.
 *    The workspace holds the calls' intermediate tables and work counters (reset by the call, on its stream),
 *    so one workspace must not serve two calls that may run concurrently (e.g. on different streams).
 *  - Return value: DSTACK_OK (0) or a negative DSTACK_E* code: a synchronous argument or launch
 *    error, in which case no work was enqueued (EINVAL/EWORKSPACE) or the launch failed (ELAUNCH).
 *  - Per-DNN / per-scenario data conditions are VALUES written to status arrays, not errors:
 *      DSTACK_ST_OK             computed
 *      DSTACK_ST_INFEASIBLE     no (level, batch) satisfies Eqs. 10-12 (or empty batch range);
 *                               scenario: no active DNN
 *      DSTACK_ST_OVERFLOW       X(L, b_hi) = E_t*S*M >= 2^56 (exact-arithmetic bound exceeded)
 *      DSTACK_ST_INVALID        DNN: K < 1 or K > 65535 rows, t_p < 1, t_np < 0, SLO < 1 or
 *                               SLO > 2^30 or SLO % slot_us != 0, a < 0 or a > 2^24, bmax < 1,
 *                               M outside [1, 2^24] (memory term on), some R_i = 0, or latency
 *                               identically 0 (t_np = 0, every n_i = 0, no memory bytes).
 *                               scenario: > DSTACK_MAX_DNN_PER_SCEN DNNs, session > DSTACK_MAX_SLOTS
 *                               slots, or > DSTACK_MAX_JOBS static jobs
 *      DSTACK_ST_OVERSUBSCRIBED scenario: some static job could not be placed (counted in misses)
 *  - Per-DNN and per-scenario results are deterministic: independent of GPU count, launch
 *    configuration and stream.  Integer outputs equal the oracle's bit for bit; f64 outputs are the
 *    documented ratios of exact integers, evaluated in the documented order.  The aggregate's integer
 *    words (counts, histograms, checksum) are sums, so shards add up exactly; its f64 sums depend on
 *    the summation order (fixed per call, but not across shardings: equal to ~1e-12 relative).
 *  - Row arrays n, r, d must be readable 16 bytes past their last element (vector loads).
 *  - There is no CPU fallback: without a CUDA device every compute call returns DSTACK_ELAUNCH.
 */
#ifndef DSTACK_H
#define DSTACK_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DSTACK_OK 0
#define DSTACK_EINVAL (-1)
#define DSTACK_EWORKSPACE (-2)
#define DSTACK_ELAUNCH (-3)

#define DSTACK_ST_OK 0
#define DSTACK_ST_INFEASIBLE 1
#define DSTACK_ST_OVERFLOW 2
#define DSTACK_ST_INVALID 3
#define DSTACK_ST_OVERSUBSCRIBED 4

#define DSTACK_MAX_DNN_PER_SCEN 32
#define DSTACK_MAX_SLOTS 4096
#define DSTACK_MAX_JOBS 512
#define DSTACK_MAX_ROWS_PER_DNN 65535
#define DSTACK_MAX_BATCH 64

#define DSTACK_MAX_FILL_RUNS 2048   /* dstack_simulate: fill runs per session (more => scenario INVALID) */

#define DSTACK_FLAG_IDEAL 1u   /* run a6, the ideal per-kernel scheduler */
/* F1 below-knee fallback ("D-STACK's scheduler can also schedule a model with
 * GPU% lower than its Knee, albeit with high inference latency when necessary ... also considers the
 * additional latency of launching a new DNN model at lower GPU%"; reading R21): a static
 * job with no feasible start at g_j is retried at levels g_j - 1 .. 1 and placed, under the same
 * Start-Early / Start-Late rule, at the first level whose run fits in its window; that run lasts
 * ceil(f_L(l, b*) / Delta) + ceil(reconf_us / Delta) slots at level l.  Only unplaced jobs count as misses.
 * Applies to dstack_schedule_cycle and dstack_eval_batch (not with a test hook); dstack_simulate and
 * dstack_compare reject it (DSTACK_EINVAL). */
#define DSTACK_FLAG_BELOW_KNEE 2u

/* Structure-of-arrays problem set, CSR-indexed.  Scenario s owns DNNs
 * [scen_dnn_off[s], scen_dnn_off[s+1]); DNN k owns kernel rows [dnn_row_off[k], dnn_row_off[k+1]). */
typedef struct {
  int32_t num_scen;
  int32_t num_dnn;                 /* == scen_dnn_off[num_scen] */
  int64_t num_rows;                /* == dnn_row_off[num_dnn] (host copy, sizes the workspace) */
  const int32_t *scen_dnn_off;     /* [num_scen+1], nondecreasing, [0] == 0 */
  const int64_t *dnn_row_off;      /* [num_dnn+1], nondecreasing, [0] == 0 */
  const int32_t *t_p;              /* [num_dnn] us per parallel op (Table) */
  const int32_t *t_np;             /* [num_dnn] us serialized launch time per kernel execution */
  const int32_t *mem_bw;           /* [num_dnn] M, bytes/us/SM (ignored when mem_mode = 0) */
  const int32_t *slo_us;           /* [num_dnn] SLO_j, multiple of slot_us */
  const int32_t *asm_us;           /* [num_dnn] a_j, request assembly us per request: C = b a */
  const int32_t *bmax;             /* [num_dnn] MaxBatchSize (Eq. 10) */
  const uint32_t *n;               /* [num_rows] n_i (linear) or theta_i threads/sample (threads mode) */
  const uint16_t *r;               /* [num_rows] R_i >= 1 */
  const uint32_t *d;               /* [num_rows] d_i bytes */
} dstack_problem_t;

typedef struct {
  int32_t L;          /* GPU% levels, 1..255 (100: 1% steps; 148: per-SM) */
  int32_t S_tot;      /* modelled SMs, 1..256; level l grants S(l) = ceil(l*S_tot/L) SMs */
  int32_t slot_us;    /* Delta, schedule slot width in us (>= 1) */
  int32_t mem_mode;   /* Eq. 3: 0 off, 1 bw E_m = d/(M S) (prose P:1517; default), 2 verbatim d S / M */
  int32_t margin;     /* over-provisioning in levels added to l* (P:2091), 0..L */
  int32_t par_mode;   /* Eq. 1: 0 linear N_i(b) = b n_i, 1 threads N_i(b) = ceil(b theta_i / 2048) */
  int32_t wse_mode;   /* Eq. 4: 0 per_request (printed), 1 per_launch (t_np once per kernel) */
  int32_t b_min, b_max;  /* batch range, 1 <= b_min <= b_max <= 64; per DNN b_hi = min(b_max, bmax_j) */
  uint32_t flags;     /* DSTACK_FLAG_IDEAL | DSTACK_FLAG_BELOW_KNEE */
  int32_t reconf_us;  /* F1 launch latency of an instance at a lower GPU%, us >= 0 (~100 us switchover
                         with active-standby overlap); read only with DSTACK_FLAG_BELOW_KNEE */
} dstack_params_t;

/* Aggregate statistics over the scenarios of one call (one struct, device memory). */
typedef struct {
  double sum_u_static, sum_u, sum_thr, sum_u_ideal, sum_thr_ideal;   /* over scenarios with T > 0 */
  uint64_t n_scen, n_scen_scheduled, n_dnn, n_dnn_ok;
  uint64_t n_st[5];          /* per-DNN status counts */
  uint64_t n_scen_st[5];     /* per-scenario status counts */
  uint64_t misses, runs, served;
  uint64_t batch_hist[DSTACK_MAX_BATCH + 1];   /* b* histogram over OK DNNs */
  uint64_t demand_hist[256];                   /* demand-level histogram over OK DNNs */
  uint64_t checksum;         /* sum over DNNs of a mix of (demand, batch, knee, alloc, runs, served, status):
                                position-free, so per-shard aggregates sum to the whole problem's */
} dstack_agg_t;

/* Outputs.  In dstack_eval_batch, demand/batch/knee/status/alloc_q16 are REQUIRED (the path reads
 * them back); every other pointer may be NULL (not written). */
typedef struct {
  /* per DNN [num_dnn] */
  uint16_t *demand;      /* l* + margin, capped at L; 0 unless status OK */
  uint8_t  *batch;       /* b* (0 unless OK) */
  uint16_t *knee;        /* knee(b*) (Eq. 6), 0 unless OK */
  uint8_t  *status;      /* DSTACK_ST_* */
  uint32_t *alloc_q16;   /* WMAX-MIN allocation, Q16.16 levels */
  uint16_t *level;       /* g_j = max(demand, alloc>>16) used by the schedule (0 if inactive) */
  uint16_t *runs;        /* runs placed in the session (static + fill) */
  uint32_t *served;      /* requests served = sum of batches of its runs */
  /* per scenario [num_scen] */
  uint8_t  *scen_status;
  uint32_t *T_us;        /* session length = max SLO over active DNNs (0 if none) */
  double   *u_static;    /* = (double)sum_slots occ_static / ((double)nslots * (double)L) */
  double   *u;           /* = (double)sum_slots occ / ((double)nslots * (double)L) */
  double   *thr;         /* = (double)sum_j served_j * 1e6 / (double)T_us  (requests/s) */
  uint32_t *misses;      /* static jobs not placed */
  double   *u_ideal;     /* = (double)sum_events(sum g * dt) / ((double)L * (double)T_us) */
  double   *thr_ideal;   /* = (double)sum_j(completed_j * b*_j) * 1e6 / (double)T_us */
  dstack_agg_t *agg;     /* optional, one struct */
  uint32_t *below;       /* per scenario: static jobs placed below the knee (DSTACK_FLAG_BELOW_KNEE; else 0) */
} dstack_out_t;

/* Optional test hook for dstack_schedule_cycle (Table 4 pins): per-DNN level g_j
 * (0 = inactive) and runtime in slots of one run at b*_j, replacing O1-O4; fill then uses b* only. */
typedef struct {
  const int32_t *level;      /* [num_dnn] */
  const int32_t *d_slots;    /* [num_dnn] */
} dstack_cycle_hook_t;

/* Bytes of device scratch the calls below need for this problem (0 is possible). */
size_t dstack_workspace_size(const dstack_problem_t *pb, const dstack_params_t *p);

/* a1-a2: knee(b) of every DNN at one batch b (Eq. 6): argmax over l in 1..L of
 * 1/(f_L(l,b)^2 S(l)), ties to the smaller l.  st_out: INVALID / OVERFLOW (X(L,b) >= 2^56) / OK. */
int dstack_knee(const dstack_problem_t *pb, const dstack_params_t *p, int32_t batch, uint16_t *knee_out,
                uint8_t *st_out, void *ws, size_t ws_bytes, void *stream);

/* F3, online knee discovery ("our platform initially provides it a nominal, 30%,
 * GPU. The GPU% is then readjusted using Dynamic GPU resource reconfiguration to find the knee based on the
 * inference latency using a simple binary search"; reading R22).  Per DNN at batch b: lo = 1,
 * hi = L; the first step probes m = ceil(0.3 L), later ones m = floor((lo + hi) / 2), m clamped to
 * [lo, hi - 1]; each step measures the latency at m and m + 1 and moves lo = m + 1 iff
 * 1/(f_L(m+1,b)^2 S(m+1)) > 1/(f_L(m,b)^2 S(m)) (Eq. 6's objective, exact), else hi = m; stops at lo == hi.
 * knee_out[k] = lo (0 unless st_out[k] is OK), probes_out[k] = the number of steps (<= ceil(log2 L) + 1).
 * The result is a discrete local maximum of Eq. 6's objective; it equals dstack_knee's exact argmax whenever
 * that objective is unimodal over the levels.  Statuses as dstack_knee.  Device arrays [num_dnn].  ws may be NULL;
 * with >= dstack_workspace_size() bytes the DNNs are distributed by a work counter in it (faster, same results). */
int dstack_knee_probe(const dstack_problem_t *pb, const dstack_params_t *p, int32_t batch, uint16_t *knee_out,
                      uint8_t *probes_out, uint8_t *st_out, void *ws, size_t ws_bytes, void *stream);

/* a1-a3: per DNN (l*, b*) = argmax of eta = b/(f_L^2 GPU%) (Eq. 9) over feasible cells (Eqs. 10-12),
 * ties to smaller l then smaller b; demand = min(L, l* + margin); knee = knee(b*). */
int dstack_batch_opt(const dstack_problem_t *pb, const dstack_params_t *p, uint16_t *demand, uint8_t *batch,
                     uint16_t *knee, uint8_t *status, void *ws, size_t ws_bytes, void *stream);

/* a4: WMAX-MIN per scenario over demand[] (0 = no demand), L levels; Q16.16 output. */
int dstack_wmaxmin(int32_t num_scen, const int32_t *scen_dnn_off, int32_t L, const uint16_t *demand,
                   uint32_t *alloc_q16, void *stream);

/* a5 (+ a6 when DSTACK_FLAG_IDEAL): one D-STACK session per scenario from a3/a4 results.
 * Active DNN <=> demand > 0.  hook may be NULL.  Writes out->level, runs, served, scen_status, T_us,
 * u_static, u, thr, misses (+ u_ideal, thr_ideal) where non-NULL. */
int dstack_schedule_cycle(const dstack_problem_t *pb, const dstack_params_t *p, const uint16_t *demand,
                          const uint8_t *batch, const uint32_t *alloc_q16, const dstack_cycle_hook_t *hook,
                          dstack_out_t *out, void *ws, size_t ws_bytes, void *stream);

/* a1-a6 + a8 fused path: batch_opt -> wmaxmin -> schedule_cycle (-> ideal) -> aggregate. */
int dstack_eval_batch(const dstack_problem_t *pb, const dstack_params_t *p, dstack_out_t *out, void *ws,
                      size_t ws_bytes, void *stream);

/* a8 alone: fold the per-DNN / per-scenario outputs already in `out` into out->agg (deterministic
 * two-level reduction, fixed grid).  Used when the path is driven call by call. */
int dstack_aggregate(const dstack_problem_t *pb, const dstack_params_t *p, dstack_out_t *out, void *ws,
                     size_t ws_bytes, void *stream);

/* a7: long-horizon simulation (config 5, readings in DESIGN.md §3).  Per scenario:
 * cycles sessions of T = max SLO over its servable DNNs; Poisson request arrivals per DNN with mean gap
 * f_L(l*, b*) * 100 / (lam_pct * b*) us (lam_pct <= 0: no requests, the gap takes its 2^30 us cap; reading R25)
 * drawn by the counter-based sampler of synth/synth_core.h keyed by
 * (seed, cfg_tag, scen_base + s, dnn, k); each session: active = queued requests at its start, WMAX-MIN
 * over their demands, one D-STACK session with the fill ordered by the runs of the last 10 sessions, then
 * every run serves FIFO min(batch, queue at its start) requests (void if the queue is empty).
 * Outputs per scenario (all device arrays [num_scen]): status, T_us, arrived, in_slo, late (completed
 * after arrival + SLO), unserved (queued at the horizon), occ_sum (sum over non-void runs of level x
 * slots; mean utilisation = occ_sum / (nslots L cycles)), runs (non-void), misses (unplaced static jobs),
 * realloc (sessions 2..cycles whose active DNN set differs from the previous session's: each is a per-cycle
 * WMAX-MIN re-allocation over a changed set).
 * series (optional, may be NULL): the per-cycle aggregate series, u64 [cycles][DSTACK_SIM_SERIES], zeroed by the
 * call; row c sums over the scenarios' session c: DSTACK_SIM_ACTIVE DNNs with requests queued at its start,
 * DSTACK_SIM_REALLOC scenarios whose active set changed at c (c >= 1), DSTACK_SIM_RUNS non-void runs,
 * DSTACK_SIM_SERVED requests served, DSTACK_SIM_IN_SLO / DSTACK_SIM_LATE of them in / after SLO,
 * DSTACK_SIM_OCC level-slots of the non-void runs, DSTACK_SIM_MISSES unplaced static jobs.  A scenario that turns
 * INVALID at session c (fill-run capacity) contributes its sessions before c.  Sums of integers: exact and
 * independent of the launch.  Workspace: dstack_sim_workspace_size(). */
#define DSTACK_SIM_ACTIVE 0
#define DSTACK_SIM_REALLOC 1
#define DSTACK_SIM_RUNS 2
#define DSTACK_SIM_SERVED 3
#define DSTACK_SIM_IN_SLO 4
#define DSTACK_SIM_LATE 5
#define DSTACK_SIM_OCC 6
#define DSTACK_SIM_MISSES 7
#define DSTACK_SIM_SERIES 8
typedef struct {
  uint8_t *status; uint32_t *T_us;
  uint64_t *arrived, *in_slo, *late, *unserved, *occ_sum, *runs, *misses, *realloc;
  uint64_t *series;
} dstack_sim_out_t;
size_t dstack_sim_workspace_size(const dstack_problem_t *pb, const dstack_params_t *p);
int dstack_simulate(const dstack_problem_t *pb, const dstack_params_t *p, const int32_t *lam_pct, int32_t cycles,
                    uint64_t seed, int32_t cfg_tag, int64_t scen_base, dstack_sim_out_t *out, void *ws,
                    size_t ws_bytes, void *stream);

/* O9 comparison schedulers of §6.3 (readings in DESIGN.md §3.2), evaluated on the
 * a3/a4 results (demand, batch, alloc_q16 as written by dstack_eval_batch / dstack_batch_opt +
 * dstack_wmaxmin).  For each scenario s and scheduler c (DSTACK_CMP_*), writes
 *   u[s*DSTACK_NCMP + c]    GPU utilisation: occupied level-slots / (nslots L)  (knee% accounting)
 *   thr[s*DSTACK_NCMP + c]  requests served per second of session (saturating load)
 *   jain[s*DSTACK_NCMP + c] Jain's index (sum x)^2 / (n sum x^2) of the per-model GPU time x_j (slots)
 * c = DSTACK_CMP_DSTACK: the D-STACK session (identical to dstack_schedule_cycle's u / thr);
 *     DSTACK_CMP_MAXMIN: same session, fill in ascending (GPU%, index) order (Max-Min fair);
 *     DSTACK_CMP_SRF_STRUCK: same session, fill in ascending (run time of b*, index) order -- "shortest run first",
 *     the procedure of the STRUCK text at P:2540 ("by prioritizing scheduling the model with the least runtime");
 *     the live definition of max-throughput is dstack_max_throughput (O9b);
 *     DSTACK_CMP_TEMPORAL: slices proportional to SLO at 100% GPU, knee% accounting;
 *     DSTACK_CMP_GSLICE: static spatial sharing at the knees, residents + first-fit decreasing time slots.
 * Scenarios that are INVALID / INFEASIBLE for the D-STACK session get zeros.  All pointers are device
 * pointers; u/thr/jain are [num_scen * DSTACK_NCMP] f64.  Workspace: dstack_workspace_size() (d_j(b) rows). */
#define DSTACK_CMP_DSTACK 0
#define DSTACK_CMP_MAXMIN 1
#define DSTACK_CMP_SRF_STRUCK 2
#define DSTACK_CMP_TEMPORAL 3
#define DSTACK_CMP_GSLICE 4
#define DSTACK_NCMP 5
int dstack_compare(const dstack_problem_t *pb, const dstack_params_t *p, const uint16_t *demand, const uint8_t *batch,
                   const uint32_t *alloc_q16, double *u, double *thr, double *jain, void *ws, size_t ws_bytes,
                   void *stream);

/* O9b max-throughput, the §6.3 comparison "a schedule that maximizes the sum of the throughput across all the
 * models" (reading R24; the paper's ">80%" comparison at P:2582).  Per scenario, on the
 * a3/a4 outputs (demand, batch = b*, alloc_q16, e.g. from dstack_eval_batch): the session T = max SLO over the active
 * DNNs (demand > 0) and their levels g_j = max(demand_j, floor(alloc_j)) as in D-STACK's session; every schedule of
 * non-overlapping runs of a batch b in [b_min, b*_j] lasting d_j(b) = ceil(X(S(g_j), b) / (S(g_j) M Delta)) slots per
 * DNN, starting at slot boundaries, ending by the session end, with the summed level of the runs in progress <= L at
 * every slot, is searched exactly (dynamic programming over the slots left of every DNN's run in progress).
 *   served_out[s] = the largest number of requests such a schedule serves (throughput = served * 1e6 / T_us);
 *   st_out[s] = DSTACK_ST_OK, DSTACK_ST_INFEASIBLE (no active DNN), or DSTACK_ST_INVALID (more than 8 active DNNs,
 *   more than DSTACK_MAX_SLOTS slots, or a state space prod_j (max_b d_j(b) + 1) above 8192): exact search is for
 *   small instances only.  Device u32 / u8 arrays [num_scen].  Workspace: dstack_workspace_size();
 *   DSTACK_FLAG_BELOW_KNEE is rejected (DSTACK_EINVAL). */
int dstack_max_throughput(const dstack_problem_t *pb, const dstack_params_t *p, const uint16_t *demand,
                          const uint8_t *batch, const uint32_t *alloc_q16, uint32_t *served_out, uint8_t *st_out,
                          void *ws, size_t ws_bytes, void *stream);

/* F4 multi-GPU cluster of §7.1 ("one T4 GPU for each DNN model exclusively",
 * "all 4 models in each GPU, temporally sharing the GPU", "D-STACK with the 4 DNN models"; reading R23,
 * DESIGN.md §3.5): `gpus` = G modelled GPUs of L levels (1 <= G <= 32) serve each scenario's active models
 * (demand > 0, from dstack_batch_opt / dstack_eval_batch).  For scenario s and policy c (DSTACK_CLU_*):
 *   u[s*DSTACK_NCLU + c]   = (1/G) sum over GPUs i with models of occ_i / (nslots_i L)  (idle GPUs count 0)
 *   thr[s*DSTACK_NCLU + c] = sum over GPUs i of served_i * 1e6 / T_i   (requests/s; T_i = max SLO on GPU i)
 * c = DSTACK_CLU_EXCLUSIVE: the q-th active model (index order) on GPU q mod G, temporal sharing (as
 *     DSTACK_CMP_TEMPORAL) among the models that share a GPU (one model per GPU when G >= their number);
 *     DSTACK_CLU_TEMPORAL: every GPU runs DSTACK_CMP_TEMPORAL over the whole mix (G replicas);
 *     DSTACK_CLU_DSTACK: every GPU runs the D-STACK session over the whole mix (G replicas);
 *     DSTACK_CLU_DSTACK_FFD: models first-fit decreasing by (demand desc, index) onto GPUs of L levels, one that
 *     fits nowhere to the least-loaded GPU (lowest index on ties); each GPU runs WMAX-MIN over its models and
 *     one D-STACK session.
 * Scenarios INVALID / INFEASIBLE for the single-GPU session get zeros.  u, thr: device f64 [num_scen * 4].
 * Workspace: dstack_workspace_size().  DSTACK_FLAG_BELOW_KNEE is rejected (DSTACK_EINVAL). */
#define DSTACK_CLU_EXCLUSIVE 0
#define DSTACK_CLU_TEMPORAL 1
#define DSTACK_CLU_DSTACK 2
#define DSTACK_CLU_DSTACK_FFD 3
#define DSTACK_NCLU 4
int dstack_cluster(const dstack_problem_t *pb, const dstack_params_t *p, int32_t gpus, const uint16_t *demand,
                   const uint8_t *batch, double *u, double *thr, void *ws, size_t ws_bytes, void *stream);

/* Live per-kernel timing of dstack_eval_batch (bench accounting): after dstack_profile_start, each
 * eval_batch call on this thread records CUDA events on its stream between its kernel launches
 * (slots: 0 k_prof, 1 k_wmaxmin, 2 k_cycle, 3 k_ideal, 4 k_agg).  dstack_profile_stop synchronises
 * those events and writes the summed milliseconds per slot into ms_out[DSTACK_PROF_SLOTS] and the
 * number of profiled calls into *calls.  At most max_calls calls are recorded. */
#define DSTACK_PROF_SLOTS 5
int dstack_profile_start(int32_t max_calls);
int dstack_profile_stop(double *ms_out, int32_t *calls);

/* Number of kernel launches the previous call on this thread enqueued (bench accounting). */
int dstack_last_launch_count(void);

/* a6 work counters of the last dstack_eval_batch / dstack_schedule_cycle call with DSTACK_FLAG_IDEAL that used this
 * workspace (§6.2 event-driven ideal scheduler, R15): out8[0] events (intervals between consecutive
 * completions), [1] events whose subset selection was recomputed, [2] of those decided by "every live item fits",
 * [3] by exhaustive subset enumeration, [4] by meet in the middle, [5] by the subset-sum DP, [6] scenarios
 * simulated, [7] reserved (0).  Host pointer out8; synchronises `stream`.  EINVAL without the IDEAL flag. */
int dstack_ideal_stats(const dstack_problem_t *pb, const dstack_params_t *p, const void *ws, size_t ws_bytes,
                       uint64_t *out8, void *stream);

/* Compact row transport (host -> device): a row whose n_i < 4096 and 1 <= R_i <= 15 travels as
 * nr = n_i | R_i << 12 (u16) beside its d_i (u32), 6 bytes instead of 10; this call expands nr[0..num_rows) into
 * the problem's n (u32) and r (u16) arrays on the device (pure data movement, results identical to copying the
 * wide arrays).  All three pointers must be 16-byte aligned; the output arrays need the ABI's 16 bytes of slack.
 * Rows outside that range must travel wide.  Used by the end-to-end path (bench.py e2e). */
int dstack_unpack_nr(int64_t num_rows, const uint16_t *nr, uint32_t *n_out, uint16_t *r_out, void *stream);
/* 5-byte variant of the compact transport for rows with n_i < 4096, 1 <= R_i <= 4 and d_i < 2^26:
 * w = d_i | (R_i - 1) << 26 | (n_i >> 8) << 28 (u32) and lo = n_i & 255 (u8); expands into n, r and d.  w, n_out,
 * d_out 16-byte aligned, lo 4-byte, r_out 8-byte aligned; outputs need the ABI's 16 bytes of slack. */
int dstack_unpack_w5(int64_t num_rows, const uint32_t *w, const uint8_t *lo, uint32_t *n_out, uint16_t *r_out,
                     uint32_t *d_out, void *stream);

const char *dstack_status_str(int code);
int dstack_version(void);

#ifdef __cplusplus
}
#endif
#endif
