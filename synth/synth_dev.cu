// synth_dev.cu -- device build of the seeded workload generator (see include/dstack_synth.h).
// Same header-only core as synth_host.c, so outputs are byte-identical.
#include "../include/dstack_synth.h"
#include <cuda_runtime.h>

namespace {

__global__ void k_ndnn(synth_spec_t sp, int32_t *ndnn) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < sp.num_scen;
       s += (int64_t)gridDim.x * blockDim.x)
    ndnn[s] = sy_ndnn(&sp, s);
}

__global__ void k_headers(synth_spec_t sp, const int32_t *off, int32_t *nrows, int32_t *t_p, int32_t *t_np,
                          int32_t *mem_bw, int32_t *slo_us, int32_t *asm_us, int32_t *bmax, int32_t *shape,
                          int32_t *lam_pct) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < sp.num_scen;
       s += (int64_t)gridDim.x * blockDim.x) {
    for (int32_t k = off[s]; k < off[s + 1]; ++k) {
      sy_dnn_t h = sy_dnn(&sp, s, k - off[s]);
      nrows[k] = h.nrows; t_p[k] = h.t_p; t_np[k] = h.t_np; mem_bw[k] = h.mem_bw;
      slo_us[k] = h.slo_us; asm_us[k] = h.asm_us; bmax[k] = h.bmax; shape[k] = h.shape; lam_pct[k] = h.lam_pct;
    }
  }
}

// one warp per scenario; lanes stride over the rows of each DNN (coalesced stores)
__global__ void k_rows(synth_spec_t sp, const int32_t *off, const int64_t *roff, uint32_t *n, uint16_t *r,
                       uint32_t *d) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = warp; s < sp.num_scen; s += nwarps) {
    for (int32_t k = off[s]; k < off[s + 1]; ++k) {
      sy_dnn_t h = sy_dnn(&sp, s, k - off[s]);
      for (int32_t i = lane; i < h.nrows; i += 32) {
        sy_row_t w = sy_row(&sp, s, k - off[s], &h, i);
        int64_t at = roff[k] + i;
        n[at] = w.n; r[at] = w.r; d[at] = w.d;
      }
    }
  }
}

int grid_for(int64_t items, int per_block) {
  int64_t g = (items + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > 148 * 32) g = 148 * 32;
  return (int)g;
}

}  // namespace

extern "C" int synth_dev_ndnn(const synth_spec_t *sp, int32_t *ndnn, void *stream) {
  if (!sp || sp->num_scen < 0) return -1;
  if (sp->num_scen == 0) return 0;
  k_ndnn<<<grid_for(sp->num_scen, 256), 256, 0, (cudaStream_t)stream>>>(*sp, ndnn);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

extern "C" int synth_dev_headers(const synth_spec_t *sp, const int32_t *off, int32_t *nrows, int32_t *t_p,
                                 int32_t *t_np, int32_t *mem_bw, int32_t *slo_us, int32_t *asm_us,
                                 int32_t *bmax, int32_t *shape, int32_t *lam_pct, void *stream) {
  if (!sp || !off || sp->num_scen < 0) return -1;
  if (sp->num_scen == 0) return 0;
  k_headers<<<grid_for(sp->num_scen, 256), 256, 0, (cudaStream_t)stream>>>(*sp, off, nrows, t_p, t_np, mem_bw,
                                                                          slo_us, asm_us, bmax, shape, lam_pct);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

extern "C" int synth_dev_rows(const synth_spec_t *sp, const int32_t *off, const int64_t *roff, uint32_t *n,
                              uint16_t *r, uint32_t *d, void *stream) {
  if (!sp || !off || !roff || sp->num_scen < 0) return -1;
  if (sp->num_scen == 0) return 0;
  k_rows<<<grid_for(sp->num_scen * 32, 256), 256, 0, (cudaStream_t)stream>>>(*sp, off, roff, n, r, d);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}
