// abi.cu -- the C-ABI entry points of libdstack (see include/dstack.h for the contract).
// Host side only: argument validation, workspace carving, launches on the caller's stream.
#include <cstring>

#include "kernels.cuh"

using namespace dstack;

namespace {

thread_local int g_launches = 0;

// live per-kernel event timing of eval_batch (dstack_profile_start/stop)
struct ProfState {
  bool on = false;
  int max_calls = 0, calls = 0;
  cudaEvent_t *ev = nullptr;        // [max_calls][DSTACK_PROF_SLOTS + 1]
  uint8_t *used = nullptr;          // [max_calls][DSTACK_PROF_SLOTS] slot launched?
};
thread_local ProfState g_prof;

inline void prof_mark(cudaStream_t s, int slot) {
  if (!g_prof.on || g_prof.calls >= g_prof.max_calls) return;
  const int base = g_prof.calls * (DSTACK_PROF_SLOTS + 1);
  cudaEventRecord(g_prof.ev[base + slot], s);
}

bool params_ok(const dstack_params_t *p) {
  return p && p->L >= 1 && p->L <= 255 && p->S_tot >= 1 && p->S_tot <= 256 && p->slot_us >= 1 &&
         p->mem_mode >= 0 && p->mem_mode <= 2 && p->par_mode >= 0 && p->par_mode <= 1 && p->wse_mode >= 0 &&
         p->wse_mode <= 1 && p->b_min >= 1 && p->b_max <= DSTACK_MAX_BATCH && p->b_min <= p->b_max &&
         p->margin >= 0 && p->margin <= p->L &&
         (p->flags & ~(DSTACK_FLAG_IDEAL | DSTACK_FLAG_BELOW_KNEE)) == 0 &&
         (!(p->flags & DSTACK_FLAG_BELOW_KNEE) || p->reconf_us >= 0);
}

bool problem_ok(const dstack_problem_t *pb) {
  if (!pb || pb->num_scen < 0 || pb->num_dnn < 0 || pb->num_rows < 0) return false;
  if (pb->num_scen > 0 && !pb->scen_dnn_off) return false;
  if (pb->num_dnn > 0 && (!pb->dnn_row_off || !pb->t_p || !pb->t_np || !pb->mem_bw || !pb->slo_us ||
                          !pb->asm_us || !pb->bmax))
    return false;
  if (pb->num_rows > 0 && (!pb->n || !pb->r || !pb->d)) return false;
  return true;
}

// outputs must not alias inputs
bool disjoint(const dstack_problem_t *pb, const void *o) {
  if (!o) return true;
  const void *in[] = {pb->scen_dnn_off, pb->dnn_row_off, pb->t_p, pb->t_np, pb->mem_bw, pb->slo_us,
                      pb->asm_us, pb->bmax, pb->n, pb->r, pb->d};
  for (const void *q : in)
    if (q == o) return false;
  return true;
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// workspace layout: [agg partials | counters | d_j(b) rows u16[num_dnn][64] | RT u32[num_dnn] | D u64[num_dnn] |
//                    d_j(b*) u16[num_dnn] | cold-DNN queue u32[num_dnn + 2] | ideal]
struct WsLayout {
  size_t ctr, dtab, rt, d, dst, cold, bigq, ideal, end;
};
WsLayout ws_layout(const dstack_problem_t *pb, const dstack_params_t *p) {
  WsLayout w;
  const size_t nd = (size_t)(pb->num_dnn > 0 ? pb->num_dnn : 0);
  w.ctr = align256(agg_ws_bytes());          // work counters (k_cycle)
  w.dtab = w.ctr + 256;
  w.rt = w.dtab + align256(nd * DTAB_ROW * 2);
  w.d = w.rt + align256(nd * 4);
  w.dst = w.d + align256(nd * 8);
  w.cold = w.dst + align256(nd * 2);
  w.bigq = w.cold + align256((nd + 2) * 4);   // k_cycle's queue of long sessions (count, unused, scenarios)
  w.ideal = w.bigq + align256(((size_t)(pb->num_scen > 0 ? pb->num_scen : 0) + 2) * 4);
  w.end = w.ideal + ((p->flags & DSTACK_FLAG_IDEAL) ? align256(ideal_ws_bytes(pb->num_rows, pb->num_scen)) : 0);
  return w;
}

int finish(int rc) {
  if (rc != 0) return rc;
  return cudaGetLastError() == cudaSuccess ? DSTACK_OK : DSTACK_ELAUNCH;
}

bool have_device() {
  int n = 0;
  return cudaGetDeviceCount(&n) == cudaSuccess && n > 0;
}

}  // namespace

static int aggregate_impl(const dstack_problem_t *pb, dstack_out_t *out, void *ws, cudaStream_t s) {
  AggArgs g;
  std::memset(&g, 0, sizeof(g));
  g.num_scen = pb->num_scen; g.off = pb->scen_dnn_off;
  g.demand = out->demand; g.knee = out->knee; g.level = out->level; g.runs = out->runs;
  g.batch = out->batch; g.status = out->status; g.scen_status = out->scen_status;
  g.alloc = out->alloc_q16; g.served = out->served; g.T_us = out->T_us; g.misses = out->misses;
  g.u_static = out->u_static; g.u = out->u; g.thr = out->thr; g.u_ideal = out->u_ideal; g.thr_ideal = out->thr_ideal;
  g.partials = (dstack_agg_t *)ws; g.out = out->agg;
  return launch_agg(g, s, &g_launches);
}

extern "C" {

int dstack_profile_start(int32_t max_calls) {
  if (max_calls < 1 || max_calls > 4096) return DSTACK_EINVAL;
  if (!have_device()) return DSTACK_ELAUNCH;
  ProfState &P = g_prof;
  P.ev = new cudaEvent_t[(size_t)max_calls * (DSTACK_PROF_SLOTS + 1)];
  for (int i = 0; i < max_calls * (DSTACK_PROF_SLOTS + 1); ++i) cudaEventCreate(&P.ev[i]);
  P.used = new uint8_t[(size_t)max_calls * DSTACK_PROF_SLOTS]();
  P.max_calls = max_calls; P.calls = 0; P.on = true;
  return DSTACK_OK;
}

int dstack_profile_stop(double *ms_out, int32_t *calls) {
  ProfState &P = g_prof;
  if (!P.on) return DSTACK_EINVAL;
  for (int k = 0; k < DSTACK_PROF_SLOTS; ++k) ms_out[k] = 0.0;
  for (int c = 0; c < P.calls; ++c) {
    cudaEvent_t *e = P.ev + c * (DSTACK_PROF_SLOTS + 1);
    cudaEventSynchronize(e[DSTACK_PROF_SLOTS]);
    for (int k = 0; k < DSTACK_PROF_SLOTS; ++k) {
      if (!P.used[c * DSTACK_PROF_SLOTS + k]) continue;
      // slot k spans from its own mark to the next recorded mark
      int nx = k + 1;
      while (nx < DSTACK_PROF_SLOTS && !P.used[c * DSTACK_PROF_SLOTS + nx]) ++nx;
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e[k], e[nx]);
      ms_out[k] += ms;
    }
  }
  if (calls) *calls = P.calls;
  for (int i = 0; i < P.max_calls * (DSTACK_PROF_SLOTS + 1); ++i) cudaEventDestroy(P.ev[i]);
  delete[] P.ev; delete[] P.used;
  P = ProfState();
  return DSTACK_OK;
}

int dstack_version(void) { return 1; }

int dstack_unpack_w5(int64_t num_rows, const uint32_t *w, const uint8_t *lo, uint32_t *n_out, uint16_t *r_out,
                     uint32_t *d_out, void *stream) {
  g_launches = 0;
  if (num_rows < 0 || (num_rows > 0 && (!w || !lo || !n_out || !r_out || !d_out))) return DSTACK_EINVAL;
  if ((((uintptr_t)w) | ((uintptr_t)n_out) | ((uintptr_t)d_out)) & 15u) return DSTACK_EINVAL;
  if ((((uintptr_t)lo) & 3u) || (((uintptr_t)r_out) & 7u)) return DSTACK_EINVAL;
  if (!have_device()) return DSTACK_ELAUNCH;
  return finish(launch_unpack_w5(num_rows, w, lo, n_out, r_out, d_out, (cudaStream_t)stream, &g_launches));
}

int dstack_unpack_nr(int64_t num_rows, const uint16_t *nr, uint32_t *n_out, uint16_t *r_out, void *stream) {
  g_launches = 0;
  if (num_rows < 0 || (num_rows > 0 && (!nr || !n_out || !r_out))) return DSTACK_EINVAL;
  if ((((uintptr_t)nr) | ((uintptr_t)n_out) | ((uintptr_t)r_out)) & 15u) return DSTACK_EINVAL;
  if (!have_device()) return DSTACK_ELAUNCH;
  return finish(launch_unpack_nr(num_rows, nr, n_out, r_out, (cudaStream_t)stream, &g_launches));
}

int dstack_last_launch_count(void) { return g_launches; }

int dstack_ideal_stats(const dstack_problem_t *pb, const dstack_params_t *p, const void *ws, size_t ws_bytes,
                       uint64_t *out8, void *stream) {
  if (!problem_ok(pb) || !params_ok(p) || !out8 || !(p->flags & DSTACK_FLAG_IDEAL)) return DSTACK_EINVAL;
  if (!ws || ws_bytes < dstack_workspace_size(pb, p)) return DSTACK_EWORKSPACE;
  if (!have_device()) return DSTACK_ELAUNCH;
  const char *src = (const char *)ws + ws_layout(pb, p).ideal + ideal_stats_offset(pb->num_rows, pb->num_scen);
  if (cudaMemcpyAsync(out8, src, 8 * sizeof(uint64_t), cudaMemcpyDeviceToHost, (cudaStream_t)stream) != cudaSuccess ||
      cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess)
    return DSTACK_ELAUNCH;
  return DSTACK_OK;
}

const char *dstack_status_str(int code) {
  switch (code) {
    case DSTACK_OK: return "OK";
    case DSTACK_EINVAL: return "EINVAL: bad argument";
    case DSTACK_EWORKSPACE: return "EWORKSPACE: workspace too small";
    case DSTACK_ELAUNCH: return "ELAUNCH: CUDA launch failed / no device";
    default: return "unknown";
  }
}

size_t dstack_workspace_size(const dstack_problem_t *pb, const dstack_params_t *p) {
  if (!problem_ok(pb) || !params_ok(p)) return 0;
  return ws_layout(pb, p).end;
}

int dstack_knee(const dstack_problem_t *pb, const dstack_params_t *p, int32_t batch, uint16_t *knee_out,
                uint8_t *st_out, void *ws, size_t ws_bytes, void *stream) {
  (void)ws; (void)ws_bytes;
  g_launches = 0;
  if (!problem_ok(pb) || !params_ok(p) || batch < 1 || batch > DSTACK_MAX_BATCH) return DSTACK_EINVAL;
  if (pb->num_dnn > 0 && (!knee_out || !st_out)) return DSTACK_EINVAL;
  if (!disjoint(pb, knee_out) || !disjoint(pb, st_out)) return DSTACK_EINVAL;
  if (!have_device()) return DSTACK_ELAUNCH;
  ProfArgs a;
  std::memset(&a, 0, sizeof(a));
  a.pb = *pb; a.p = *p; a.knee_only = 1; a.knee_b = batch; a.knee = knee_out; a.status = st_out;
  return finish(launch_prof(a, (cudaStream_t)stream, &g_launches));
}

int dstack_knee_probe(const dstack_problem_t *pb, const dstack_params_t *p, int32_t batch, uint16_t *knee_out,
                      uint8_t *probes_out, uint8_t *st_out, void *ws, size_t ws_bytes, void *stream) {
  g_launches = 0;
  if (!problem_ok(pb) || !params_ok(p) || batch < 1 || batch > DSTACK_MAX_BATCH) return DSTACK_EINVAL;
  if (pb->num_dnn > 0 && (!knee_out || !probes_out || !st_out)) return DSTACK_EINVAL;
  if (!disjoint(pb, knee_out) || !disjoint(pb, probes_out) || !disjoint(pb, st_out)) return DSTACK_EINVAL;
  if ((const void *)knee_out == (const void *)probes_out || (const void *)knee_out == (const void *)st_out ||
      (const void *)probes_out == (const void *)st_out)
    return DSTACK_EINVAL;
  if (!have_device()) return DSTACK_ELAUNCH;
  ProfArgs a;
  std::memset(&a, 0, sizeof(a));
  a.pb = *pb; a.p = *p; a.knee_only = 1; a.knee_b = batch; a.knee = knee_out; a.status = st_out;
  a.probes = probes_out;
  // with a workspace of dstack_workspace_size() bytes the DNNs are handed out by a counter, else grid stride
  if (ws && ws_bytes >= dstack_workspace_size(pb, p)) a.work_ctr = (uint32_t *)((char *)ws + ws_layout(pb, p).ctr) + 6;
  return finish(launch_knee_probe(a, (cudaStream_t)stream, &g_launches));
}

int dstack_batch_opt(const dstack_problem_t *pb, const dstack_params_t *p, uint16_t *demand, uint8_t *batch,
                     uint16_t *knee, uint8_t *status, void *ws, size_t ws_bytes, void *stream) {
  (void)ws; (void)ws_bytes;
  g_launches = 0;
  if (!problem_ok(pb) || !params_ok(p)) return DSTACK_EINVAL;
  if (pb->num_dnn > 0 && (!demand || !batch || !status)) return DSTACK_EINVAL;
  if (!disjoint(pb, demand) || !disjoint(pb, batch) || !disjoint(pb, knee) || !disjoint(pb, status))
    return DSTACK_EINVAL;
  if (!have_device()) return DSTACK_ELAUNCH;
  ProfArgs a;
  std::memset(&a, 0, sizeof(a));
  a.pb = *pb; a.p = *p; a.demand = demand; a.batch = batch; a.knee = knee; a.status = status;
  return finish(launch_prof(a, (cudaStream_t)stream, &g_launches));
}

int dstack_wmaxmin(int32_t num_scen, const int32_t *scen_dnn_off, int32_t L, const uint16_t *demand,
                   uint32_t *alloc_q16, void *stream) {
  g_launches = 0;
  if (num_scen < 0 || L < 1 || L > 255 || (num_scen > 0 && (!scen_dnn_off || !demand || !alloc_q16)))
    return DSTACK_EINVAL;
  if ((const void *)demand == (const void *)alloc_q16) return DSTACK_EINVAL;
  if (!have_device()) return DSTACK_ELAUNCH;
  return finish(launch_wmaxmin(num_scen, scen_dnn_off, L, demand, alloc_q16, (cudaStream_t)stream, &g_launches));
}

static int ideal_impl(const dstack_problem_t *pb, const dstack_params_t *p, const uint16_t *demand,
                      const uint8_t *batch, const dstack_cycle_hook_t *hook, dstack_out_t *out, void *ws,
                      cudaStream_t s);

static int schedule_impl(const dstack_problem_t *pb, const dstack_params_t *p, const uint16_t *demand,
                         const uint8_t *batch, const uint32_t *alloc_q16, const dstack_cycle_hook_t *hook,
                         dstack_out_t *out, void *ws, size_t ws_bytes, cudaStream_t s, bool pre_ws = false) {
  CycArgs c;
  std::memset(&c, 0, sizeof(c));
  c.pb = *pb; c.p = *p; c.demand = demand; c.batch = batch; c.alloc = alloc_q16;
  if (pre_ws && !hook) c.alloc_out = out->alloc_q16;   // eval path: a4 fused into k_cycle
  if (hook) { c.hook_level = hook->level; c.hook_d = hook->d_slots; }
  c.level = out->level; c.runs = out->runs; c.served = out->served; c.scen_status = out->scen_status;
  c.T_us = out->T_us; c.u_static = out->u_static; c.u = out->u; c.thr = out->thr; c.misses = out->misses;
  c.below = out->below;
  c.dtab_rows = (uint16_t *)((char *)ws + ws_layout(pb, p).dtab);
  c.dstar = (uint16_t *)((char *)ws + ws_layout(pb, p).dst);
  c.work_ctr = (uint32_t *)((char *)ws + ws_layout(pb, p).ctr);
  c.big_q = (uint32_t *)((char *)ws + ws_layout(pb, p).bigq);
  if (pre_ws) { c.ws_RT = (const uint32_t *)((char *)ws + ws_layout(pb, p).rt); c.ws_D = (const uint64_t *)((char *)ws + ws_layout(pb, p).d); }
  int rc = launch_cycle(c, s, &g_launches);
  if (rc) return rc;
  if (pre_ws && (p->flags & DSTACK_FLAG_IDEAL)) prof_mark(s, 3);
  return ideal_impl(pb, p, demand, batch, hook, out, ws, s);
}

static int ideal_impl(const dstack_problem_t *pb, const dstack_params_t *p, const uint16_t *demand,
                      const uint8_t *batch, const dstack_cycle_hook_t *hook, dstack_out_t *out, void *ws,
                      cudaStream_t s) {
  int rc = 0;
  if ((p->flags & DSTACK_FLAG_IDEAL) && !hook) {
    IdealArgs ia;
    std::memset(&ia, 0, sizeof(ia));
    ia.pb = *pb; ia.p = *p; ia.demand = demand; ia.batch = batch; ia.u_ideal = out->u_ideal;
    ia.thr_ideal = out->thr_ideal;
    ia.work_ctr = (uint32_t *)((char *)ws + ws_layout(pb, p).ctr) + 2;
    if (!hook) {   // the session's d_j(b) rows and sum R: a per-scenario cost estimate for the heavy-first order
      ia.dstar = (const uint16_t *)((char *)ws + ws_layout(pb, p).dst);
    }
    rc = launch_ideal(ia, (char *)ws + ws_layout(pb, p).ideal, s, &g_launches);
  }
  return rc;
}

int dstack_schedule_cycle(const dstack_problem_t *pb, const dstack_params_t *p, const uint16_t *demand,
                          const uint8_t *batch, const uint32_t *alloc_q16, const dstack_cycle_hook_t *hook,
                          dstack_out_t *out, void *ws, size_t ws_bytes, void *stream) {
  g_launches = 0;
  if (!problem_ok(pb) || !params_ok(p) || !out) return DSTACK_EINVAL;
  if (pb->num_dnn > 0 && (!batch || (!hook && (!demand || !alloc_q16)))) return DSTACK_EINVAL;
  if (hook && pb->num_dnn > 0 && (!hook->level || !hook->d_slots)) return DSTACK_EINVAL;
  if (ws_bytes < dstack_workspace_size(pb, p) || (dstack_workspace_size(pb, p) > 0 && !ws))
    return DSTACK_EWORKSPACE;
  if (!have_device()) return DSTACK_ELAUNCH;
  return finish(schedule_impl(pb, p, demand, batch, alloc_q16, hook, out, ws, ws_bytes, (cudaStream_t)stream));
}

int dstack_eval_batch(const dstack_problem_t *pb, const dstack_params_t *p, dstack_out_t *out, void *ws,
                      size_t ws_bytes, void *stream) {
  g_launches = 0;
  if (!problem_ok(pb) || !params_ok(p) || !out) return DSTACK_EINVAL;
  if (pb->num_dnn > 0 && (!out->demand || !out->batch || !out->knee || !out->status || !out->alloc_q16))
    return DSTACK_EINVAL;
  const void *outs[] = {out->demand, out->batch, out->knee, out->status, out->alloc_q16, out->level, out->runs,
                        out->served, out->scen_status, out->T_us, out->u_static, out->u, out->thr, out->misses,
                        out->u_ideal, out->thr_ideal, out->agg, out->below};
  for (const void *o : outs)
    if (!disjoint(pb, o)) return DSTACK_EINVAL;
  const size_t need = dstack_workspace_size(pb, p);
  if (ws_bytes < need || (need > 0 && !ws)) return DSTACK_EWORKSPACE;
  if (!have_device()) return DSTACK_ELAUNCH;
  cudaStream_t s = (cudaStream_t)stream;
  const WsLayout w = ws_layout(pb, p);
  ProfArgs a;
  std::memset(&a, 0, sizeof(a));
  a.pb = *pb; a.p = *p; a.demand = out->demand; a.batch = out->batch; a.knee = out->knee; a.status = out->status;
  a.dtab_rows = (uint16_t *)((char *)ws + w.dtab);
  a.dstar = (uint16_t *)((char *)ws + w.dst);
  a.ws_RT = (uint32_t *)((char *)ws + w.rt);
  a.ws_D = (uint64_t *)((char *)ws + w.d);
  a.work_ctr = (uint32_t *)((char *)ws + w.ctr) + 1;   // word 0: k_cycle's counter
  a.cold_q = (uint32_t *)((char *)ws + w.cold);
  const bool prof = g_prof.on && g_prof.calls < g_prof.max_calls;
  uint8_t *used = prof ? g_prof.used + g_prof.calls * DSTACK_PROF_SLOTS : nullptr;
  // slots: k_prof, (k_wmaxmin: a4 runs inside k_cycle on this path, slot unused), k_cycle, k_ideal, k_agg
  if (prof) { used[0] = used[2] = 1; used[1] = 0; used[3] = (p->flags & DSTACK_FLAG_IDEAL) ? 1 : 0; used[4] = out->agg ? 1 : 0; }
  prof_mark(s, 0);
  int rc = launch_prof(a, s, &g_launches);                                            // a1-a3
  prof_mark(s, 1);
  // a4 (WMAX-MIN) runs inside k_cycle on this path (CycArgs::alloc_out): the profile slot stays empty
  prof_mark(s, 2);
  if (!rc) rc = schedule_impl(pb, p, out->demand, out->batch, out->alloc_q16, nullptr, out, ws, ws_bytes, s, true);
  if (!rc && out->agg) { prof_mark(s, 4); rc = aggregate_impl(pb, out, ws, s); }
  if (prof) { prof_mark(s, DSTACK_PROF_SLOTS); g_prof.calls++; }
  return finish(rc);
}

// simulate workspace: [eval layout without ideal | demand u16 | knee u16 | batch u8 | status u8 | fill logs]
struct SimLayout {
  size_t dem, knee, bat, st, log, end;
};
static SimLayout sim_layout(const dstack_problem_t *pb, const dstack_params_t *p) {
  dstack_params_t q = *p;
  q.flags = 0;
  const size_t nd = (size_t)(pb->num_dnn > 0 ? pb->num_dnn : 0);
  SimLayout l;
  l.dem = ws_layout(pb, &q).end;
  l.knee = l.dem + align256(nd * 2);
  l.bat = l.knee + align256(nd * 2);
  l.st = l.bat + align256(nd);
  l.log = l.st + align256(nd);
  l.end = l.log + align256(sim_fill_log_bytes());
  return l;
}

size_t dstack_sim_workspace_size(const dstack_problem_t *pb, const dstack_params_t *p) {
  if (!problem_ok(pb) || !params_ok(p)) return 0;
  return sim_layout(pb, p).end;
}

int dstack_simulate(const dstack_problem_t *pb, const dstack_params_t *p, const int32_t *lam_pct, int32_t cycles,
                    uint64_t seed, int32_t cfg_tag, int64_t scen_base, dstack_sim_out_t *out, void *ws,
                    size_t ws_bytes, void *stream) {
  g_launches = 0;
  if (!problem_ok(pb) || !params_ok(p) || !out || cycles < 0 || (pb->num_dnn > 0 && !lam_pct)) return DSTACK_EINVAL;
  if (p->flags & DSTACK_FLAG_BELOW_KNEE) return DSTACK_EINVAL;
  if (pb->num_scen > 0 && (!out->status || !out->T_us || !out->arrived || !out->in_slo || !out->late ||
                           !out->unserved || !out->occ_sum || !out->runs || !out->misses || !out->realloc))
    return DSTACK_EINVAL;
  const size_t need = dstack_sim_workspace_size(pb, p);
  if (ws_bytes < need || !ws) return DSTACK_EWORKSPACE;
  if (!have_device()) return DSTACK_ELAUNCH;
  cudaStream_t s = (cudaStream_t)stream;
  const SimLayout sl = sim_layout(pb, p);
  dstack_params_t q = *p;
  q.flags = 0;
  const WsLayout w = ws_layout(pb, &q);
  char *base = (char *)ws;
  ProfArgs a;
  std::memset(&a, 0, sizeof(a));
  a.pb = *pb; a.p = q;
  a.demand = (uint16_t *)(base + sl.dem); a.knee = (uint16_t *)(base + sl.knee);
  a.batch = (uint8_t *)(base + sl.bat); a.status = (uint8_t *)(base + sl.st);
  a.ws_RT = (uint32_t *)(base + w.rt); a.ws_D = (uint64_t *)(base + w.d);
  a.cold_q = (uint32_t *)(base + w.cold);
  int rc = launch_prof(a, s, &g_launches);   // a1-a3 (RT, D for the arrival rates and d_j(b))
  if (rc) return finish(rc);
  SimArgs m;
  std::memset(&m, 0, sizeof(m));
  m.pb = *pb; m.p = q; m.lam_pct = lam_pct; m.cycles = cycles; m.cfg_tag = cfg_tag; m.seed = seed;
  m.scen_base = scen_base; m.demand = a.demand; m.batch = a.batch; m.status = a.status; m.ws_RT = a.ws_RT;
  m.ws_D = a.ws_D; m.dtab_rows = (uint16_t *)(base + w.dtab); m.fill_log = (uint64_t *)(base + sl.log);
  m.out = *out;
  m.work_ctr = (uint32_t *)(base + w.ctr) + 5;
  if (out->series && cycles > 0 &&
      cudaMemsetAsync(out->series, 0, (size_t)cycles * DSTACK_SIM_SERIES * sizeof(uint64_t), s) != cudaSuccess)
    return DSTACK_ELAUNCH;
  return finish(launch_sim(m, s, &g_launches));
}

int dstack_compare(const dstack_problem_t *pb, const dstack_params_t *p, const uint16_t *demand, const uint8_t *batch,
                   const uint32_t *alloc_q16, double *u, double *thr, double *jain, void *ws, size_t ws_bytes,
                   void *stream) {
  g_launches = 0;
  if (!problem_ok(pb) || !params_ok(p) || (p->flags & DSTACK_FLAG_BELOW_KNEE)) return DSTACK_EINVAL;
  if (pb->num_dnn > 0 && (!demand || !batch || !alloc_q16)) return DSTACK_EINVAL;
  if (pb->num_scen > 0 && (!u || !thr || !jain)) return DSTACK_EINVAL;
  const void *outs[] = {u, thr, jain};
  for (const void *o : outs)
    if (!disjoint(pb, o) || o == (const void *)demand || o == (const void *)batch || o == (const void *)alloc_q16)
      return DSTACK_EINVAL;
  const size_t need = dstack_workspace_size(pb, p);
  if (ws_bytes < need || (need > 0 && !ws)) return DSTACK_EWORKSPACE;
  if (!have_device()) return DSTACK_ELAUNCH;
  CmpArgs c;
  std::memset(&c, 0, sizeof(c));
  c.pb = *pb; c.p = *p; c.demand = demand; c.batch = batch; c.alloc = alloc_q16;
  c.dtab_rows = (uint16_t *)((char *)ws + ws_layout(pb, p).dtab);
  c.u = u; c.thr = thr; c.jain = jain;
  c.work_ctr = (uint32_t *)((char *)ws + ws_layout(pb, p).ctr) + 3;
  return finish(launch_compare(c, (cudaStream_t)stream, &g_launches));
}

int dstack_max_throughput(const dstack_problem_t *pb, const dstack_params_t *p, const uint16_t *demand,
                          const uint8_t *batch, const uint32_t *alloc_q16, uint32_t *served_out, uint8_t *st_out,
                          void *ws, size_t ws_bytes, void *stream) {
  g_launches = 0;
  if (!problem_ok(pb) || !params_ok(p) || (p->flags & DSTACK_FLAG_BELOW_KNEE)) return DSTACK_EINVAL;
  if (pb->num_dnn > 0 && (!demand || !batch || !alloc_q16)) return DSTACK_EINVAL;
  if (pb->num_scen > 0 && (!served_out || !st_out)) return DSTACK_EINVAL;
  if (!disjoint(pb, served_out) || !disjoint(pb, st_out) || (const void *)served_out == (const void *)st_out)
    return DSTACK_EINVAL;
  const size_t need = dstack_workspace_size(pb, p);
  if (ws_bytes < need || (need > 0 && !ws)) return DSTACK_EWORKSPACE;
  if (!have_device()) return DSTACK_ELAUNCH;
  MtArgs m;
  std::memset(&m, 0, sizeof(m));
  m.pb = *pb; m.p = *p; m.demand = demand; m.batch = batch; m.alloc = alloc_q16; m.served = served_out; m.st = st_out;
  m.work_ctr = (uint32_t *)((char *)ws + ws_layout(pb, p).ctr) + 10;
  return finish(launch_maxthr(m, (cudaStream_t)stream, &g_launches));
}

int dstack_cluster(const dstack_problem_t *pb, const dstack_params_t *p, int32_t gpus, const uint16_t *demand,
                   const uint8_t *batch, double *u, double *thr, void *ws, size_t ws_bytes, void *stream) {
  g_launches = 0;
  if (!problem_ok(pb) || !params_ok(p) || (p->flags & DSTACK_FLAG_BELOW_KNEE) || gpus < 1 || gpus > 32)
    return DSTACK_EINVAL;
  if (pb->num_dnn > 0 && (!demand || !batch)) return DSTACK_EINVAL;
  if (pb->num_scen > 0 && (!u || !thr || u == thr)) return DSTACK_EINVAL;
  const void *outs[] = {u, thr};
  for (const void *o : outs)
    if (!disjoint(pb, o) || o == (const void *)demand || o == (const void *)batch) return DSTACK_EINVAL;
  const size_t need = dstack_workspace_size(pb, p);
  if (ws_bytes < need || (need > 0 && !ws)) return DSTACK_EWORKSPACE;
  if (!have_device()) return DSTACK_ELAUNCH;
  return finish(launch_cluster(*pb, *p, gpus, demand, batch, (uint16_t *)((char *)ws + ws_layout(pb, p).dtab), u, thr,
                               (uint32_t *)((char *)ws + ws_layout(pb, p).ctr) + 4, (cudaStream_t)stream, &g_launches));
}

int dstack_aggregate(const dstack_problem_t *pb, const dstack_params_t *p, dstack_out_t *out, void *ws,
                     size_t ws_bytes, void *stream) {
  g_launches = 0;
  if (!problem_ok(pb) || !params_ok(p) || !out || !out->agg) return DSTACK_EINVAL;
  const size_t need = dstack_workspace_size(pb, p);
  if (ws_bytes < need || (need > 0 && !ws)) return DSTACK_EWORKSPACE;
  if (!have_device()) return DSTACK_ELAUNCH;
  return finish(aggregate_impl(pb, out, ws, (cudaStream_t)stream));
}

}  // extern "C"
