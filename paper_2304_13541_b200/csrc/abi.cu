// abi.cu -- the C-ABI entry points of libdstack (see include/dstack.h for the contract).
// Host side only: argument validation, workspace carving, launches on the caller's stream.
#include <cstring>

#include "kernels.cuh"

using namespace dstack;

namespace {

thread_local int g_launches = 0;

bool params_ok(const dstack_params_t *p) {
  return p && p->L >= 1 && p->L <= 255 && p->S_tot >= 1 && p->S_tot <= 256 && p->slot_us >= 1 &&
         p->mem_mode >= 0 && p->mem_mode <= 2 && p->par_mode >= 0 && p->par_mode <= 1 && p->wse_mode >= 0 &&
         p->wse_mode <= 1 && p->b_min >= 1 && p->b_max <= DSTACK_MAX_BATCH && p->b_min <= p->b_max &&
         p->margin >= 0 && p->margin <= p->L && (p->flags & ~DSTACK_FLAG_IDEAL) == 0;
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

// workspace layout: [agg partials | d_j(b) slabs | ideal per-row arrays]
size_t ws_dtab_off() { return align256(agg_ws_bytes()); }
size_t ws_ideal_off() { return ws_dtab_off() + align256((size_t)DTAB_MAX_WARPS * DTAB_SLAB_BYTES); }

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

int dstack_version(void) { return 1; }

int dstack_last_launch_count(void) { return g_launches; }

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
  size_t sz = ws_ideal_off();
  if (p->flags & DSTACK_FLAG_IDEAL) sz += align256(ideal_ws_bytes(pb->num_rows));
  return sz;
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
                         dstack_out_t *out, void *ws, size_t ws_bytes, cudaStream_t s) {
  CycArgs c;
  std::memset(&c, 0, sizeof(c));
  c.pb = *pb; c.p = *p; c.demand = demand; c.batch = batch; c.alloc = alloc_q16;
  if (hook) { c.hook_level = hook->level; c.hook_d = hook->d_slots; }
  c.level = out->level; c.runs = out->runs; c.served = out->served; c.scen_status = out->scen_status;
  c.T_us = out->T_us; c.u_static = out->u_static; c.u = out->u; c.thr = out->thr; c.misses = out->misses;
  c.dtab_slab = (uint16_t *)((char *)ws + ws_dtab_off());
  int rc = launch_cycle(c, s, &g_launches);
  if (rc) return rc;
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
    rc = launch_ideal(ia, (char *)ws + ws_ideal_off(), s, &g_launches);
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
                        out->u_ideal, out->thr_ideal, out->agg};
  for (const void *o : outs)
    if (!disjoint(pb, o)) return DSTACK_EINVAL;
  const size_t need = dstack_workspace_size(pb, p);
  if (ws_bytes < need || (need > 0 && !ws)) return DSTACK_EWORKSPACE;
  if (!have_device()) return DSTACK_ELAUNCH;
  cudaStream_t s = (cudaStream_t)stream;
  FusedArgs f;
  std::memset(&f, 0, sizeof(f));
  f.pb = *pb; f.p = *p; f.demand = out->demand; f.batch = out->batch; f.knee = out->knee; f.status = out->status;
  f.alloc = out->alloc_q16; f.level = out->level; f.runs = out->runs; f.served = out->served;
  f.scen_status = out->scen_status; f.T_us = out->T_us; f.u_static = out->u_static; f.u = out->u; f.thr = out->thr;
  f.misses = out->misses; f.dtab_slab = (uint16_t *)((char *)ws + ws_dtab_off());
  int rc = launch_fused(f, s, &g_launches);
  if (!rc) rc = ideal_impl(pb, p, out->demand, out->batch, nullptr, out, ws, s);
  if (!rc && out->agg) rc = aggregate_impl(pb, out, ws, s);
  return finish(rc);
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
