// kernels.cuh -- argument blocks and launchers of the libdstack kernels (internal).
#pragma once
#include "common.cuh"

namespace dstack {

constexpr int DTAB_ROW = DSTACK_MAX_BATCH;   // d_j(b) row per DNN in the workspace: u16[64], entry b-1

inline int num_sms() {
  static thread_local int cached = 0;
  if (!cached) {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cached = n;
  }
  return cached;
}

struct ProfArgs {
  dstack_problem_t pb;
  dstack_params_t p;
  int32_t knee_only;   // 1: dstack_knee (knee at knee_b only)
  int32_t knee_b;
  uint16_t *demand;
  uint8_t *batch;
  uint16_t *knee;
  uint8_t *status;
  uint8_t *probes;     // dstack_knee_probe (F3): non-NULL => knee = the binary-search result, probes = its steps
  // eval path extras (workspace, may be NULL): d_j(b) at g = demand for b in [b_lo, b*], RT, D
  uint16_t *dtab_rows;
  uint16_t *dstar;      // d_j(b*) at g = demand, one u16 per DNN (dense: k_cycle's read of it is coalesced)
  uint32_t *ws_RT;
  uint64_t *ws_D;
  uint32_t *work_ctr;   // workspace word: k_prof_fast's DNN-group counter (NULL: contiguous ranges)
  uint32_t *cold_q;     // workspace [num_dnn + 2] (eval path): [0] count, [1] pull counter, then the DNNs k_prof_lane
                        // leaves to the generic path, which k_prof_cold then analyses (NULL: analysed in place)
};

struct CycArgs {
  dstack_problem_t pb;
  dstack_params_t p;
  const uint16_t *demand;
  const uint8_t *batch;
  const uint32_t *alloc;
  uint32_t *alloc_out;     // non-NULL (eval path): a4 fused -- WMAX-MIN computed here and written out; alloc unused
  const int32_t *hook_level;
  const int32_t *hook_d;
  uint16_t *level;
  uint16_t *runs;
  uint32_t *served;
  uint8_t *scen_status;
  uint32_t *T_us;
  double *u_static, *u, *thr;
  uint32_t *misses;
  uint32_t *below;         // F1: static jobs placed below the knee
  uint16_t *dtab_rows;     // workspace: num_dnn rows of DTAB_ROW u16
  uint16_t *dstar;         // workspace: d_j(b*) at the session level per DNN (read when k_prof wrote it, else written)
  const uint32_t *ws_RT;   // non-NULL => dtab_rows / dstar already hold d_j(b) at g = demand (from k_prof)
  const uint64_t *ws_D;
  uint32_t *work_ctr;      // workspace word: k_cycle's scenario counter (NULL: grid stride)
  uint32_t *big_q;         // workspace: [count, unused, scenario...] of the sessions too long for the small-buffer
                           // pass (NULL: one full-buffer pass)
};

constexpr int64_t SIM_MAX_WARPS = 148 * 32;   // persistent-grid cap (sizes the fill-run logs)

struct SimArgs {
  dstack_problem_t pb;
  dstack_params_t p;
  const int32_t *lam_pct;
  int32_t cycles;
  int32_t cfg_tag;
  uint64_t seed;
  int64_t scen_base;
  const uint16_t *demand;
  const uint8_t *batch;
  const uint8_t *status;
  const uint32_t *ws_RT;
  const uint64_t *ws_D;
  uint16_t *dtab_rows;
  uint64_t *fill_log;   // SIM_MAX_WARPS x DSTACK_MAX_FILL_RUNS
  dstack_sim_out_t out;
  uint32_t *work_ctr;   // workspace word: scenario counter (NULL: grid stride)
};

struct IdealArgs {
  dstack_problem_t pb;
  dstack_params_t p;
  const uint16_t *demand;
  const uint8_t *batch;
  uint64_t *ex_pk;    // [num_rows] workspace: tau | g << 32 | R << 48 per execution (k_ideal_rows -> k_ideal_sim)
  double *u_ideal, *thr_ideal;
  uint32_t *work_ctr;   // workspace word: k_ideal_sim's scenario counter (NULL: grid stride)
  const uint16_t *dstar;       // d_j(b*) of the session just computed, per DNN (cost estimate for the order; may be NULL)
  const uint32_t *ws_RT;       // sum R per DNN (may be NULL)
  uint32_t *order;             // [num_scen] scenarios, heaviest estimate first (set by launch_ideal)
  uint32_t *bucket_cnt;        // [64] workspace
  unsigned long long *stats;   // [8] workspace: work counters (ideal_stats_offset)
};

struct CmpArgs {
  dstack_problem_t pb;
  dstack_params_t p;
  const uint16_t *demand;
  const uint8_t *batch;
  const uint32_t *alloc;
  uint16_t *dtab_rows;      // workspace
  double *u, *thr, *jain;   // [num_scen * DSTACK_NCMP]
  uint32_t *work_ctr;       // workspace word: scenario counter (NULL: grid stride)
};

struct MtArgs {   // O9b max-throughput (maxthr.cu)
  dstack_problem_t pb;
  dstack_params_t p;
  const uint16_t *demand;
  const uint8_t *batch;
  const uint32_t *alloc;
  uint32_t *served;
  uint8_t *st;
  uint32_t *work_ctr;
};

struct AggArgs {
  int32_t num_scen;
  const int32_t *off;
  const uint16_t *demand, *knee, *level, *runs;
  const uint8_t *batch, *status, *scen_status;
  const uint32_t *alloc, *served, *T_us, *misses;
  const double *u_static, *u, *thr, *u_ideal, *thr_ideal;
  dstack_agg_t *partials;   // workspace
  dstack_agg_t *out;
};

int launch_prof(const ProfArgs &a, cudaStream_t s, int *launches);
int launch_knee_probe(const ProfArgs &a, cudaStream_t s, int *launches);
int launch_wmaxmin(int32_t num_scen, const int32_t *off, int32_t L, const uint16_t *demand, uint32_t *alloc,
                   cudaStream_t s, int *launches);
int launch_cycle(const CycArgs &a, cudaStream_t s, int *launches);
int launch_ideal(IdealArgs a, void *ws, cudaStream_t s, int *launches);
int launch_sim(const SimArgs &a, cudaStream_t s, int *launches);
size_t sim_fill_log_bytes();
int launch_agg(const AggArgs &a, cudaStream_t s, int *launches);
int launch_compare(const CmpArgs &a, cudaStream_t s, int *launches);
int launch_maxthr(const MtArgs &a, cudaStream_t s, int *launches);
int launch_unpack_nr(int64_t num_rows, const uint16_t *nr, uint32_t *n, uint16_t *r, cudaStream_t s, int *launches);
int launch_unpack_w5(int64_t num_rows, const uint32_t *w, const uint8_t *lo, uint32_t *n, uint16_t *r, uint32_t *d,
                     cudaStream_t s, int *launches);
int launch_cluster(const dstack_problem_t &pb, const dstack_params_t &p, int32_t G, const uint16_t *demand,
                   const uint8_t *batch, uint16_t *dtab_rows, double *u, double *thr, uint32_t *work_ctr, cudaStream_t s,
                   int *launches);

// one resident wave of `kern` (blocks per SM from the occupancy calculator x SMs), at most `blocks`
template <typename K>
inline int64_t resident_wave(K kern, int threads, size_t smem, int64_t blocks) {
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, threads, smem) != cudaSuccess || nb <= 0) nb = 1;
  const int64_t w = (int64_t)nb * num_sms();
  return blocks < w ? blocks : w;
}
size_t ideal_ws_bytes(int64_t num_rows, int64_t num_scen);
size_t ideal_stats_offset(int64_t num_rows, int64_t num_scen);
size_t agg_ws_bytes();

}  // namespace dstack
