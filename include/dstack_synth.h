/* dstack_synth.h -- C-ABI of the seeded synthetic-workload generator.
 *
 * The generator is the only code shared between the CPU oracle's tests and
 * the CUDA product path (it draws inputs; it holds none of the method's
 * arithmetic).  Two builds of the same header-only core (synth/synth_core.h):
 *   libdstack_synth_host.so  -- gcc, host pointers
 *   libdstack_synth_dev.so   -- nvcc sm_100a, device pointers, async on `stream`
 * Both produce byte-identical arrays for the same spec and global scenario index.
 *
 * Three phases (the caller does the exclusive prefix sums between them):
 *   1. ndnn[s]        -> scen_dnn_off = exclusive_cumsum(ndnn)          (int32, num_scen+1)
 *   2. headers[dnn]   -> dnn_row_off  = exclusive_cumsum(nrows)         (int64, num_dnn+1)
 *   3. rows[row]      -> n (u32), r (u16), d (u32)
 * Ownership: all buffers are caller-owned; nothing is allocated.  Errors:
 * return 0 on success, -1 on bad arguments (NULL pointer, num_scen < 0),
 * -2 on a CUDA launch error (device build only).
 */
#ifndef DSTACK_SYNTH_H
#define DSTACK_SYNTH_H
#include <stdint.h>
#include "../synth/synth_core.h"   /* synth_spec_t */

#ifdef __cplusplus
extern "C" {
#endif

int synth_host_ndnn(const synth_spec_t *spec, int32_t *ndnn /*[num_scen]*/);
int synth_host_headers(const synth_spec_t *spec, const int32_t *scen_dnn_off,
                       int32_t *nrows, int32_t *t_p, int32_t *t_np, int32_t *mem_bw, int32_t *slo_us,
                       int32_t *asm_us, int32_t *bmax, int32_t *shape, int32_t *lam_pct /*[num_dnn] each*/);
int synth_host_rows(const synth_spec_t *spec, const int32_t *scen_dnn_off, const int64_t *dnn_row_off,
                    uint32_t *n, uint16_t *r, uint32_t *d /*[num_rows] each*/);

/* Gaps (us) of arrivals k0 .. k0+count-1 of the (gscen, dnn) Poisson stream with mean gap mean_q32 (Q32 us). */
int synth_host_arrival_gaps(uint64_t seed, int32_t cfg_tag, int64_t gscen, uint32_t dnn, uint64_t mean_q32,
                            uint32_t k0, uint32_t count, uint64_t *gaps);

/* Device build: same semantics, device pointers, asynchronous on `stream` (a cudaStream_t). */
int synth_dev_ndnn(const synth_spec_t *spec, int32_t *ndnn, void *stream);
int synth_dev_headers(const synth_spec_t *spec, const int32_t *scen_dnn_off,
                      int32_t *nrows, int32_t *t_p, int32_t *t_np, int32_t *mem_bw, int32_t *slo_us,
                      int32_t *asm_us, int32_t *bmax, int32_t *shape, int32_t *lam_pct, void *stream);
int synth_dev_rows(const synth_spec_t *spec, const int32_t *scen_dnn_off, const int64_t *dnn_row_off,
                   uint32_t *n, uint16_t *r, uint32_t *d, void *stream);

#ifdef __cplusplus
}
#endif
#endif
