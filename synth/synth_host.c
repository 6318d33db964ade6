/* synth_host.c -- host build of the seeded workload generator (see include/dstack_synth.h). */
#include "../include/dstack_synth.h"
#include <stddef.h>

int synth_host_ndnn(const synth_spec_t *sp, int32_t *ndnn) {
  if (!sp || (!ndnn && sp->num_scen > 0) || sp->num_scen < 0) return -1;
#pragma omp parallel for schedule(static)
  for (int64_t s = 0; s < sp->num_scen; ++s) ndnn[s] = sy_ndnn(sp, s);
  return 0;
}

int synth_host_headers(const synth_spec_t *sp, const int32_t *off, int32_t *nrows, int32_t *t_p,
                       int32_t *t_np, int32_t *mem_bw, int32_t *slo_us, int32_t *asm_us, int32_t *bmax,
                       int32_t *shape, int32_t *lam_pct) {
  if (!sp || !off || sp->num_scen < 0) return -1;
#pragma omp parallel for schedule(static)
  for (int64_t s = 0; s < sp->num_scen; ++s) {
    for (int32_t k = off[s]; k < off[s + 1]; ++k) {
      sy_dnn_t h = sy_dnn(sp, s, k - off[s]);
      nrows[k] = h.nrows; t_p[k] = h.t_p; t_np[k] = h.t_np; mem_bw[k] = h.mem_bw;
      slo_us[k] = h.slo_us; asm_us[k] = h.asm_us; bmax[k] = h.bmax; shape[k] = h.shape; lam_pct[k] = h.lam_pct;
    }
  }
  return 0;
}

int synth_host_rows(const synth_spec_t *sp, const int32_t *off, const int64_t *roff, uint32_t *n,
                    uint16_t *r, uint32_t *d) {
  if (!sp || !off || !roff || sp->num_scen < 0) return -1;
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t s = 0; s < sp->num_scen; ++s) {
    for (int32_t k = off[s]; k < off[s + 1]; ++k) {
      sy_dnn_t h = sy_dnn(sp, s, k - off[s]);
      for (int32_t i = 0; i < h.nrows; ++i) {
        sy_row_t w = sy_row(sp, s, k - off[s], &h, i);
        int64_t at = roff[k] + i;
        n[at] = w.n; r[at] = w.r; d[at] = w.d;
      }
    }
  }
  return 0;
}

int synth_host_arrival_gaps(uint64_t seed, int32_t cfg_tag, int64_t gscen, uint32_t dnn, uint64_t mean_q32,
                            uint32_t k0, uint32_t count, uint64_t *gaps) {
  if (!gaps) return -1;
  for (uint32_t i = 0; i < count; ++i) gaps[i] = sy_arrival_gap(mean_q32, sy_arrival_word(seed, cfg_tag, gscen, dnn, k0 + i));
  return 0;
}
