/* synth_core.h -- seeded synthetic D-STACK workload generator (header-only core).
 *
 * This is the ONE module shared by the CPU oracle's tests and the CUDA product
 * path: it only draws inputs, it holds none of the method's arithmetic (no
 * latency model, no knee, no scheduling).  Everything here is integer-only so
 * the host build (gcc) and the device build (nvcc) produce byte-identical
 * arrays from the same (seed, spec, global scenario index).
 *
 * Counter-based RNG: Philox4x32-10 (Salmon et al., SC'11), keyed by the 64-bit
 * seed; counter = (cfg_tag<<16 | field, global scenario, dnn, row).  So every
 * value depends only on its own coordinates: shard-invariant, order-free.
 *
 * Shape recipes follow SURVEY.md §8(d) "Synthetic inputs" (calibration targets
 * from PAPER.md Table 4; narrow/wide kernel mix from Fig. 6,
 * P:1696-1705; Eq. 1 decreasing-parallelism shape; SM-wave
 * conversion ceil(threads/2048)).  The recipe is restated in DESIGN.md.
 */
#ifndef DSTACK_SYNTH_CORE_H
#define DSTACK_SYNTH_CORE_H
#include <stdint.h>

#ifdef __CUDACC__
#define SY_FN __host__ __device__ __forceinline__
#else
#define SY_FN static inline
#endif

enum { SY_MOBILENET = 0, SY_RESNET50 = 1, SY_VGG19 = 2, SY_BERT = 3, SY_NSHAPES = 4 };

/* Field tags (counter word 0, low 16 bits). */
enum { SY_F_SCEN = 1, SY_F_DNN = 2, SY_F_DNN2 = 3, SY_F_ROW = 4, SY_F_ROW2 = 5, SY_F_ROWPAT = 6, SY_F_ARR = 7 };

typedef struct {
  uint64_t seed;
  int64_t  scen_base;       /* global index of local scenario 0 (sharding) */
  int32_t  num_scen;
  int32_t  cfg_tag;         /* domain separation between configs */
  int32_t  S_tot;           /* modelled SMs: kernel widths scale with it */
  int32_t  ndnn_min, ndnn_max;
  int32_t  shape_mask;      /* bit s set => shape s may be drawn */
  int32_t  paper_mix;       /* 1 => config-1 C-4 mix (ResNet-50, VGG-19, BERT, MobileNet) */
  int32_t  slot_us;         /* Delta */
  int32_t  slo_min_slots, slo_max_slots;  /* SLO = U{min..max} * slot_us */
  int32_t  asm_min_us, asm_max_us;        /* a_j (request assembly us / request) */
  int32_t  bmax;            /* per-DNN max batch */
  int32_t  mem_bw;          /* M, bytes/us/SM */
  int32_t  threads;         /* 1 => row field n holds per-sample thread count theta */
  int32_t  rows_pct;        /* row-count scale, 100 = nominal (small test instances) */
  int32_t  heavy;           /* 1 => config-4 heavy mix (ResNet/VGG/BERT only, wider kernels) */
} synth_spec_t;

typedef struct { uint32_t v[4]; } sy_u4;

/* Philox4x32-10 (Random123 round structure: round, then key bump, 10 rounds). */
SY_FN sy_u4 sy_philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  sy_u4 o; o.v[0] = c0; o.v[1] = c1; o.v[2] = c2; o.v[3] = c3;
  return o;
}

SY_FN sy_u4 sy_draw(const synth_spec_t *sp, uint32_t field, int64_t gscen, uint32_t dnn, uint32_t row) {
  return sy_philox(((uint32_t)sp->cfg_tag << 16) | (field & 0xFFFFu), (uint32_t)gscen,
                   dnn ^ ((uint32_t)((uint64_t)gscen >> 32) << 24), row,
                   (uint32_t)sp->seed, (uint32_t)(sp->seed >> 32));
}

/* Uniform integer in [lo, hi] (hi >= lo, hi-lo < 2^32) by multiply-shift. */
SY_FN int64_t sy_uni(uint32_t u, int64_t lo, int64_t hi) {
  uint64_t span = (uint64_t)(hi - lo) + 1u;
  return lo + (int64_t)(((uint64_t)u * span) >> 32);
}

/* P(u/2^32 < pct/100) */
SY_FN int sy_bern(uint32_t u, uint32_t pct) { return (uint64_t)u * 100u < (uint64_t)pct << 32; }

SY_FN int32_t sy_max32(int32_t a, int32_t b) { return a > b ? a : b; }

SY_FN int32_t sy_scale_rows(const synth_spec_t *sp, int32_t rows) {
  int64_t r = (int64_t)rows * sp->rows_pct / 100;
  return r < 1 ? 1 : (int32_t)r;
}

/* Number of DNNs in (local) scenario s. */
SY_FN int32_t sy_ndnn(const synth_spec_t *sp, int64_t s) {
  if (sp->paper_mix) return 4;
  sy_u4 w = sy_draw(sp, SY_F_SCEN, sp->scen_base + s, 0xFFFFu, 0u);
  return (int32_t)sy_uni(w.v[0], sp->ndnn_min, sp->ndnn_max);
}

typedef struct {
  int32_t shape, nrows, t_p, t_np, slo_us, asm_us, bmax, mem_bw;
  int32_t n0;      /* ResNet: first-kernel width; BERT: block length */
} sy_dnn_t;

SY_FN int32_t sy_pick_shape(const synth_spec_t *sp, uint32_t u) {
  int32_t allowed[SY_NSHAPES]; int32_t na = 0;
  int32_t mask = sp->heavy ? (sp->shape_mask & 0xE) : sp->shape_mask;
  if (mask == 0) mask = 0xF;
  for (int32_t s = 0; s < SY_NSHAPES; ++s) if (mask & (1 << s)) allowed[na++] = s;
  return allowed[sy_uni(u, 0, na - 1)];
}

/* Per-DNN header of DNN j of (local) scenario s. */
SY_FN sy_dnn_t sy_dnn(const synth_spec_t *sp, int64_t s, int32_t j) {
  const int64_t gs = sp->scen_base + s;
  sy_u4 w = sy_draw(sp, SY_F_DNN, gs, (uint32_t)j, 0xFFFFu);
  sy_u4 w2 = sy_draw(sp, SY_F_DNN2, gs, (uint32_t)j, 0xFFFFu);
  const int32_t S = sp->S_tot;
  sy_dnn_t h;
  if (sp->paper_mix) {
    /* PAPER.md P:2670 (C-4 caption: ResNet-50 + VGG-19 + BERT + Mobilenet), SLOs from Table 4:
       50 / 100 / 25 / 25 ms; a = 481 us per image. */
    const int32_t shp[4] = {SY_RESNET50, SY_VGG19, SY_BERT, SY_MOBILENET};
    const int32_t slo_ms[4] = {50, 100, 25, 25};
    h.shape = shp[j & 3];
    h.slo_us = slo_ms[j & 3] * 1000;
    h.asm_us = 481;
  } else {
    h.shape = sy_pick_shape(sp, w.v[0]);
    h.slo_us = (int32_t)sy_uni(w.v[1], sp->slo_min_slots, sp->slo_max_slots) * sp->slot_us;
    h.asm_us = (int32_t)sy_uni(w.v[2], sp->asm_min_us, sp->asm_max_us);
  }
  h.bmax = sp->bmax;
  h.mem_bw = sp->mem_bw;
  h.t_np = (int32_t)sy_uni(w2.v[1], 3, 8) * (sp->heavy ? 2 : 1);
  switch (h.shape) {
    case SY_MOBILENET:
      h.nrows = sy_scale_rows(sp, (int32_t)sy_uni(w.v[3], 50, 160));
      h.t_p = (int32_t)sy_uni(w2.v[0], 5, 15);
      h.n0 = 0;
      break;
    case SY_RESNET50:
      h.nrows = sy_scale_rows(sp, (int32_t)sy_uni(w.v[3], 100, 200));
      h.t_p = (int32_t)sy_uni(w2.v[0], 10, 30);
      /* first-kernel width U[0.5, 0.8] * S_tot (heavy: U[0.8, 1.6] * S_tot) */
      h.n0 = sp->heavy ? (int32_t)sy_uni(w2.v[2], (4 * S) / 5, (8 * S) / 5)
                       : (int32_t)sy_uni(w2.v[2], S / 2, (4 * S) / 5);
      h.n0 = sy_max32(h.n0, 1);
      break;
    case SY_VGG19:
      h.nrows = sy_scale_rows(sp, (int32_t)sy_uni(w.v[3], 50, 90));
      h.t_p = (int32_t)sy_uni(w2.v[0], 30, 80);
      h.n0 = 0;
      break;
    default: /* SY_BERT: 12 repeated blocks of B rows */ {
      int32_t B = (int32_t)sy_uni(w.v[3], 13, 25);
      B = sy_scale_rows(sp, B);
      h.nrows = 12 * B;
      h.n0 = B;
      h.t_p = (int32_t)sy_uni(w2.v[0], 5, 20);
      break;
    }
  }
  return h;
}

typedef struct { uint32_t n; uint16_t r; uint32_t d; } sy_row_t;

SY_FN uint16_t sy_repeat(uint32_t u) {
  /* R_i in {1,2,3}, P(1) = 0.8, P(2) = P(3) = 0.1 */
  if (sy_bern(u, 80)) return 1;
  return sy_bern(u << 8, 50) ? 2 : 3;
}

/* Row i of DNN j of (local) scenario s with header h. */
SY_FN sy_row_t sy_row(const synth_spec_t *sp, int64_t s, int32_t j, const sy_dnn_t *h, int32_t i) {
  const int64_t gs = sp->scen_base + s;
  const int32_t S = sp->S_tot;
  sy_row_t o;
  sy_u4 w;
  int64_t n;
  if (h->shape == SY_BERT) {
    /* same n/R/d pattern in each of the 12 blocks: draw by position within block */
    w = sy_draw(sp, SY_F_ROWPAT, gs, (uint32_t)j, (uint32_t)(i % h->n0));
  } else {
    w = sy_draw(sp, SY_F_ROW, gs, (uint32_t)j, (uint32_t)i);
  }
  switch (h->shape) {
    case SY_MOBILENET:
      /* ~10% wide rows n in [S, 4S], ~90% narrow rows n in [1, S/10] */
      if (sy_bern(w.v[0], 10)) n = sy_uni(w.v[1], S, 4 * (int64_t)S);
      else n = sy_uni(w.v[1], 1, sy_max32(1, S / 10));
      o.d = (uint32_t)sy_uni(w.v[3], 10000, 1000000);
      break;
    case SY_RESNET50: {
      /* linearly decreasing from n0 to ~1 with +-20% jitter (Eq. 1 shape) */
      int64_t base = (int64_t)h->n0 * (h->nrows - i) / h->nrows;
      int64_t jit = sy_uni(w.v[0], -20, 20);
      n = base + base * jit / 100;
      if (n < 1) n = 1;
      o.d = (uint32_t)sy_uni(w.v[3], 100000, 5000000);
      break;
    }
    case SY_VGG19:
      /* mostly n >= S/2, some > S */
      if (sy_bern(w.v[0], 80)) n = sy_uni(w.v[1], sy_max32(1, S / 2), S);
      else n = sy_uni(w.v[1], (int64_t)S + 1, 2 * (int64_t)S);
      o.d = (uint32_t)sy_uni(w.v[3], 1000000, 50000000);
      break;
    default: /* BERT: wide GEMM rows at 0.3-0.6 S, narrow softmax/layer-norm rows */
      if (sy_bern(w.v[0], 50)) n = sy_uni(w.v[1], sy_max32(1, (3 * S) / 10), sy_max32(1, (6 * S) / 10));
      else n = sy_uni(w.v[1], 1, sy_max32(1, S / 10));
      if (sp->heavy) n = 2 * n;
      o.d = (uint32_t)sy_uni(w.v[3], 1000000, 10000000);
      break;
  }
  o.r = sy_repeat(w.v[2]);
  if (sp->threads) {
    /* per-sample thread count theta in ((n-1)*2048, n*2048] so both modes describe the same DNN */
    sy_u4 w2 = sy_draw(sp, SY_F_ROW2, gs, (uint32_t)j, (uint32_t)i);
    int64_t th = sy_uni(w2.v[0], (n - 1) * 2048 + 1, n * 2048);
    o.n = (uint32_t)th;
  } else {
    o.n = (uint32_t)n;
  }
  return o;
}

#endif
