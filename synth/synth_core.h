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
  int32_t lam_pct; /* config 5: offered load as % of standalone capacity, U{30..120} */
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
  h.lam_pct = (int32_t)sy_uni(w2.v[3], 30, 120);
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


/* ---------------------------------------------------------------- arrivals ----
 * Poisson request arrivals for the long-horizon simulation (config 5): gap_k =
 * max(1, floor(mean * E_k)) us, E_k = -ln U_k, U_k = (u_k + 1) / 2^32, u_k the k-th Philox word of the
 * (scenario, dnn) stream.  -ln U is evaluated in Q31 fixed point (log2 by a 257-entry table with linear
 * interpolation) so host and device draw IDENTICAL integer gaps.  The mean gap (Q32 us) is an input:
 * the generator holds no method arithmetic. */
#define SY_LOG2_Q31_INIT { \
  0u, 12078627u, 24110347u, 36095523u, 48034513u, 59927671u, 71775349u, 83577893u, \
  95335645u, 107048945u, 118718126u, 130343521u, 141925456u, 153464255u, 164960239u, 176413723u, \
  187825021u, 199194443u, 210522295u, 221808880u, 233054496u, 244259442u, 255424009u, 266548488u, \
  277633165u, 288678325u, 299684247u, 310651211u, 321579490u, 332469358u, 343321082u, 354134928u, \
  364911162u, 375650043u, 386351829u, 397016776u, 407645136u, 418237160u, 428793095u, 439313187u, \
  449797678u, 460246807u, 470660814u, 481039932u, 491384396u, 501694436u, 511970279u, 522212153u, \
  532420281u, 542594885u, 552736183u, 562844395u, 572919734u, 582962413u, 592972645u, 602950638u, \
  612896598u, 622810731u, 632693241u, 642544327u, 652364189u, 662153025u, 671911030u, 681638398u, \
  691335320u, 701001986u, 710638585u, 720245302u, 729822324u, 739369832u, 748888009u, 758377033u, \
  767837083u, 777268336u, 786670965u, 796045145u, 805391046u, 814708840u, 823998694u, 833260775u, \
  842495250u, 851702282u, 860882034u, 870034667u, 879160341u, 888259214u, 897331443u, 906377184u, \
  915396590u, 924389816u, 933357012u, 942298328u, 951213914u, 960103918u, 968968484u, 977807760u, \
  986621888u, 995411012u, 1004175273u, 1012914810u, 1021629764u, 1030320272u, 1038986470u, 1047628495u, \
  1056246482u, 1064840562u, 1073410869u, 1081957534u, 1090480686u, 1098980456u, 1107456970u, 1115910356u, \
  1124340739u, 1132748245u, 1141132997u, 1149495118u, 1157834731u, 1166151954u, 1174446910u, 1182719716u, \
  1190970490u, 1199199350u, 1207406412u, 1215591791u, 1223755601u, 1231897955u, 1240018966u, 1248118746u, \
  1256197405u, 1264255053u, 1272291800u, 1280307752u, 1288303019u, 1296277705u, 1304231918u, 1312165761u, \
  1320079339u, 1327972754u, 1335846110u, 1343699509u, 1351533050u, 1359346835u, 1367140963u, 1374915531u, \
  1382670639u, 1390406384u, 1398122861u, 1405820167u, 1413498396u, 1421157644u, 1428798003u, 1436419566u, \
  1444022426u, 1451606675u, 1459172403u, 1466719700u, 1474248656u, 1481759361u, 1489251901u, 1496726366u, \
  1504182841u, 1511621414u, 1519042169u, 1526445193u, 1533830570u, 1541198383u, 1548548716u, 1555881652u, \
  1563197273u, 1570495661u, 1577776895u, 1585041058u, 1592288229u, 1599518487u, 1606731910u, 1613928578u, \
  1621108567u, 1628271955u, 1635418819u, 1642549234u, 1649663276u, 1656761020u, 1663842541u, 1670907913u, \
  1677957208u, 1684990500u, 1692007863u, 1699009366u, 1705995083u, 1712965083u, 1719919439u, 1726858219u, \
  1733781493u, 1740689331u, 1747581801u, 1754458972u, 1761320910u, 1768167684u, 1774999361u, 1781816006u, \
  1788617686u, 1795404466u, 1802176412u, 1808933588u, 1815676059u, 1822403888u, 1829117139u, 1835815874u, \
  1842500157u, 1849170050u, 1855825614u, 1862466912u, 1869094003u, 1875706949u, 1882305810u, 1888890646u, \
  1895461516u, 1902018479u, 1908561594u, 1915090920u, 1921606515u, 1928108435u, 1934596739u, 1941071483u, \
  1947532725u, 1953980519u, 1960414922u, 1966835990u, 1973243777u, 1979638338u, 1986019729u, 1992388003u, \
  1998743213u, 2005085414u, 2011414658u, 2017730999u, 2024034488u, 2030325179u, 2036603122u, 2042868370u, \
  2049120974u, 2055360984u, 2061588451u, 2067803426u, 2074005959u, 2080196099u, 2086373895u, 2092539398u, \
  2098692655u, 2104833716u, 2110962628u, 2117079439u, 2123184198u, 2129276951u, 2135357746u, 2141426629u, \
  2147483648u, \
}
static const uint32_t SY_LOG2_Q31_H[257] = SY_LOG2_Q31_INIT;
#ifdef __CUDACC__
static __constant__ uint32_t SY_LOG2_Q31_D[257] = SY_LOG2_Q31_INIT;
#endif
#if defined(__CUDA_ARCH__)
#define SY_LOG2_Q31 SY_LOG2_Q31_D
#else
#define SY_LOG2_Q31 SY_LOG2_Q31_H
#endif

SY_FN uint32_t sy_arrival_word(uint64_t seed, int32_t cfg_tag, int64_t gscen, uint32_t dnn, uint32_t k) {
  sy_u4 w = sy_philox(((uint32_t)cfg_tag << 16) | SY_F_ARR, (uint32_t)gscen,
                      dnn ^ ((uint32_t)((uint64_t)gscen >> 32) << 24), k >> 2, (uint32_t)seed, (uint32_t)(seed >> 32));
  return w.v[k & 3u];
}

/* -ln((u + 1) / 2^32) in Q31 (0 <= result < 22.2 * 2^31) */
SY_FN uint64_t sy_neglog_q31(uint32_t u) {
  const uint64_t v = (uint64_t)u + 1u;            /* 1 .. 2^32 */
  if (v >> 32) return 0;                          /* U = 1 */
  int e = 31;
  while (!((v >> e) & 1u)) --e;                   /* floor(log2 v) */
  const uint32_t mant = (uint32_t)(v << (31 - e)); /* 1.f in Q31, top bit set */
  const uint32_t frac = mant & 0x7FFFFFFFu;
  const uint32_t i = frac >> 23, rem = frac & 0x7FFFFFu;
  const uint64_t l2f = SY_LOG2_Q31[i] + (((uint64_t)(SY_LOG2_Q31[i + 1] - SY_LOG2_Q31[i]) * rem) >> 23);
  const uint64_t l2 = ((uint64_t)e << 31) + l2f;  /* log2 v in Q31 */
  const uint64_t d = ((uint64_t)32 << 31) - l2;   /* -log2 U in Q31, < 2^36 */
  return (uint64_t)(((unsigned __int128)d * 1488522236u) >> 31);   /* x ln 2 (Q31) */
}

/* gap in us for the mean gap mean_q32 (Q32 us, < 2^62): max(1, floor(mean * E)) */
SY_FN uint64_t sy_arrival_gap(uint64_t mean_q32, uint32_t u) {
  const uint64_t g = (uint64_t)(((unsigned __int128)mean_q32 * sy_neglog_q31(u)) >> 63);
  return g < 1 ? 1 : g;
}

#endif
