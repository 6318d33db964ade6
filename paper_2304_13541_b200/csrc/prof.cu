// prof.cu -- a1-a3 kernels (dstack_batch_opt, dstack_knee, first stage of dstack_eval_batch / _simulate):
// one warp per DNN, grid-stride.
//
//  k_prof<PAR>     generic path, every mode (prof.cuh: row pass, coefficient tables, exact branch-and-bound
//                  over all batches).
//  k_prof_fast<CB> the printed model's defaults (linear N_i(b) = b n_i, per-request W_se, b_lo = 1;
//                  SURVEY §8(c) O1/O3), register-resident: the width histogram is scanned into per-lane
//                  registers (CB consecutive widths per lane), the b = 1 row is evaluated from them, and
//                  one b-independent certificate proves that no b >= 2 can beat it ("batch
//                  certificate").  A DNN whose certificate fails is re-analysed by the generic path.
#include "kernels.cuh"
#include "prof.cuh"

namespace dstack {

__host__ __device__ inline size_t prof_warp_bytes(int S_tot) {
  return (((size_t)20 * (S_tot + 1)) + 15) & ~(size_t)15;   // cA, cU u64 + hist u32
}

#ifndef DSTACK_PROF_MINB
#define DSTACK_PROF_MINB 4
#endif
#ifndef DSTACK_PROF_FAST
#define DSTACK_PROF_FAST 1   // 0: every launch takes the generic kernel (A/B switch)
#endif

// generic per-DNN analysis and its outputs
template <int PAR>
__device__ __forceinline__ void prof_one(const ProfArgs &a, int64_t k, const uint16_t *Stab, uint32_t *hist,
                                         uint64_t *cA, uint64_t *cU, int lane) {
  const DnnRes r = analyze_dnn<PAR>(a.pb, a.p, k, Stab, hist, cA, cU, lane, a.knee_only, a.knee_b);
  if (a.dtab_rows && r.st == DSTACK_ST_OK) {   // eval path: d_j(b) at g = demand, b in [b_lo, b*]
    if (PAR == 0)
      dtab_from_tables(a.pb, a.p, k, cA, cU, r.RT, r.D, r.demand, a.p.b_min, r.b, a.dtab_rows + k * DTAB_ROW, lane);
    else
      dtab_from_rows(a.pb, a.p, k, r.RT, r.D, r.demand, a.p.b_min, r.b, a.dtab_rows + k * DTAB_ROW, lane);
  }
  if (lane == 0) {
    if (a.ws_RT) { a.ws_RT[k] = (uint32_t)r.RT; a.ws_D[k] = r.D; }
    const bool ok = r.st == DSTACK_ST_OK;
    if (a.knee) a.knee[k] = ok ? r.knee : 0;
    if (a.status) a.status[k] = r.st;
    if (!a.knee_only) {
      if (a.demand) a.demand[k] = ok ? r.demand : 0;
      if (a.batch) a.batch[k] = ok ? r.b : 0;
    }
  }
  __syncwarp();
}

template <int PAR>
__global__ void __launch_bounds__(256, DSTACK_PROF_MINB) k_prof(ProfArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int L = a.p.L, S_tot = a.p.S_tot;
  uint16_t *Stab = (uint16_t *)smem;
  const int tab_bytes = ((L + 1 + S_tot + 1) * 2 + 15) & ~15;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char *wreg = smem + tab_bytes + (size_t)warp * prof_warp_bytes(S_tot);
  uint64_t *cA = (uint64_t *)wreg;
  uint64_t *cU = cA + (S_tot + 1);
  uint32_t *hist = (uint32_t *)(cU + (S_tot + 1));
  fill_stab(Stab, L, S_tot);
  __syncthreads();
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t k = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; k < a.pb.num_dnn; k += nwarps)
    prof_one<PAR>(a, k, Stab, hist, cA, cU, lane);
}

// ------------------------------------------------------------------------------------------------------
// fast path
// ------------------------------------------------------------------------------------------------------

// cold: generic re-analysis of DNN k (certificate failed); leaves the histogram zeroed for the fast path
static __device__ __noinline__ void prof_one_cold(const ProfArgs *a, int64_t k, const uint16_t *Stab, uint32_t *hist,
                                                  uint64_t *cA, uint64_t *cU, int lane) {
  PSTAT(8, lane == 0);
  prof_one<0>(*a, k, Stab, hist, cA, cU, lane);
  for (int m = lane; m <= a->p.S_tot; m += 32) hist[m] = 0;
  __syncwarp();
}

// cold: exact argmax of S / X^2 (ties -> smaller S) over the band members scr[S] != 0, S in [1, S_tot]
static __device__ __noinline__ void band_exact(const uint64_t *scr, int S_tot, int lane, uint32_t *S_out,
                                               uint64_t *X_out) {
  Best v = best_none();
  for (int S = 1 + lane; S <= S_tot; S += 32) {
    const uint64_t X = scr[S];
    if (!X) continue;
    Best c; c.found = 1; c.l = (uint32_t)S; c.b = 1; c.S = (uint32_t)S; c.X = X; c.sc = score_f((uint32_t)S, X);
    if (better(c, v)) v = c;
  }
  v = warp_best_exact(v);
  *S_out = v.found ? v.S : 0u;
  *X_out = v.X;
}

// Warp argmax over the register-resident candidates (bins S = m0 + i with bit i of `mask`): the float
// maximum decides unless a second candidate lies within 2^-16 of it (float scores are within 2^-20 of the
// exact ones, so the exact winner is always in that band); then the band is resolved exactly.
template <int CB>
__device__ __forceinline__ void fast_argmax(float vmax, uint32_t mask, const float (&sc)[CB], const uint64_t (&xs)[CB],
                                            int m0, int S_tot, uint64_t *scr, int lane, uint32_t &Sw, uint64_t &Xw) {
  const uint32_t mx = __reduce_max_sync(FULL, __float_as_uint(vmax));   // scores > 0: u32 order = float order
  Sw = 0; Xw = 0;
  if (mx == 0) return;
  const float band = __uint_as_float(mx) * 0.9999847f;   // 1 - 2^-16
  uint32_t cnt = 0, sel = 0;
  uint64_t xsel = 0;
#pragma unroll
  for (int i = 0; i < CB; ++i)
    if (((mask >> i) & 1u) && sc[i] >= band) { ++cnt; sel = (uint32_t)(m0 + i); xsel = xs[i]; }
  if (__reduce_add_sync(FULL, cnt) == 1) {
    const int src = __ffs(__ballot_sync(FULL, cnt != 0)) - 1;
    Sw = __shfl_sync(FULL, sel, src);
    Xw = shfl_u64(xsel, src);
    return;
  }
  PSTAT(9, lane == 0);
#pragma unroll
  for (int i = 0; i < CB; ++i)
    if (m0 + i <= S_tot) scr[m0 + i] = (((mask >> i) & 1u) && sc[i] >= band) ? xs[i] : 0ull;
  __syncwarp();
  band_exact(scr, S_tot, lane, &Sw, &Xw);
  __syncwarp();
}

template <int CB>
__device__ __forceinline__ void fast_one(const ProfArgs &a, int64_t k, const uint16_t *Stab, const uint16_t *lmin,
                                         uint32_t *hist, uint64_t *cA, uint64_t *cU, int lane) {
  const dstack_problem_t &pb = a.pb;
  const dstack_params_t &p = a.p;
  const int L = p.L, S_tot = p.S_tot;
  const int64_t r0 = pb.dnn_row_off[k], K64 = pb.dnn_row_off[k + 1] - r0;
  const int32_t t_p = pb.t_p[k], t_np = pb.t_np[k], slo = pb.slo_us[k], asm_us = pb.asm_us[k];
  const int32_t bmax = pb.bmax[k], mbw = pb.mem_bw[k];
  const int mem_mode = p.mem_mode;
  const uint64_t M = mem_mode == 0 ? 1 : (uint64_t)mbw;
  const int32_t b_hi = bmax < p.b_max ? bmax : p.b_max;   // b_lo = 1 on this path
  uint8_t st = DSTACK_ST_OK;
  uint32_t RT = 0, knee = 0, demand = 0, dslots = 0;
  uint64_t D = 0;
  do {
    // ---- header validation (DSTACK_ST_INVALID conditions, dstack.h) ----
    if (K64 < 1 || K64 > DSTACK_MAX_ROWS_PER_DNN || t_p < 1 || t_np < 0 || slo < 1 || slo > (1 << 30) ||
        (slo % p.slot_us) != 0 || asm_us < 0 || asm_us > (1 << 24) || bmax < 1 ||
        (mem_mode != 0 && (mbw < 1 || mbw > (1 << 24)))) {
      st = DSTACK_ST_INVALID;
      break;
    }
    // ---- a1: one coalesced pass over the rows: RT, D, W = sum R n, width histogram (smem) ----
    const int32_t K = (int32_t)K64;
    const uint32_t *n = pb.n + r0;
    const uint16_t *r = pb.r + r0;
    const uint32_t *d = pb.d + r0;
    uint32_t anyR0 = 0;
    uint64_t Wn = 0;
    for (int i0 = lane; i0 < K; i0 += 64) {
      const int i1 = i0 + 32;
      const bool h1 = i1 < K;
      const uint32_t n0 = __ldg(n + i0), d0 = __ldg(d + i0), R0 = __ldg(r + i0);
      uint32_t n1 = 0, d1 = 0, R1 = 0;
      if (h1) { n1 = __ldg(n + i1); d1 = __ldg(d + i1); R1 = __ldg(r + i1); }
      RT += R0; D += (uint64_t)R0 * d0; Wn += (uint64_t)R0 * n0; anyR0 |= (R0 == 0);
      if (n0 <= (uint32_t)S_tot) atomicAdd(&hist[n0], R0);
      if (h1) {
        RT += R1; D += (uint64_t)R1 * d1; Wn += (uint64_t)R1 * n1; anyR0 |= (R1 == 0);
        if (n1 <= (uint32_t)S_tot) atomicAdd(&hist[n1], R1);
      }
    }
    RT = __reduce_add_sync(FULL, RT);
    D = warp_sum_u64(D);
    Wn = warp_sum_u64(Wn);
    anyR0 = __reduce_or_sync(FULL, anyR0);
    __syncwarp();
    // ---- scan of the histogram into registers: lane owns widths m0..m0+CB-1; re-zero the histogram ----
    //   pa[i] = PA[m] = sum_{1<=n<=m} R,   pw[i] = sum_{n<=m} n R   (Q[m] = W - pw[i])
    const int m0 = lane * CB;
    uint32_t pa[CB];
    uint64_t pw[CB];
    {
      uint32_t h[CB], sa = 0;
      uint64_t sw = 0;
#pragma unroll
      for (int i = 0; i < CB; ++i) {
        const int m = m0 + i;
        h[i] = 0;
        if (m <= S_tot) { h[i] = hist[m]; hist[m] = 0; }
        if (m == 0) h[i] = 0;   // n = 0 rows: in neither PA nor sum n R
        sa += h[i]; sw += (uint64_t)h[i] * (uint32_t)m;
      }
      uint32_t ia = sa;
      uint64_t iw = sw;
#pragma unroll
      for (int dd = 1; dd < 32; dd <<= 1) {
        const uint32_t ua = __shfl_up_sync(FULL, ia, dd);
        const uint64_t uw = shfl_up_u64(iw, dd);
        if (lane >= dd) { ia += ua; iw += uw; }
      }
      uint32_t ra = ia - sa;
      uint64_t rw = iw - sw;
#pragma unroll
      for (int i = 0; i < CB; ++i) {
        ra += h[i]; rw += (uint64_t)h[i] * (uint32_t)(m0 + i);
        pa[i] = ra; pw[i] = rw;
      }
    }
    __syncwarp();
    if (anyR0 || (t_np == 0 && Wn == 0 && (mem_mode == 0 || D == 0))) { st = DSTACK_ST_INVALID; break; }
    if (b_hi < 1) { st = DSTACK_ST_INFEASIBLE; break; }
    // ---- overflow: X(L, b_hi) = b_hi t_np RT S_tot M + M t_p (S_tot PA[mb] + b_hi Q[mb]) + mem < 2^56 ----
    {
      const int mb = S_tot / b_hi;
      uint32_t pam = 0;
      uint64_t pwm = 0;
#pragma unroll
      for (int i = 0; i < CB; ++i)
        if (m0 + i == mb) { pam = pa[i]; pwm = pw[i]; }
      pam = __shfl_sync(FULL, pam, mb / CB);
      pwm = shfl_u64(pwm, mb / CB);
      const u128 v = (u128)S_tot * pam + (u128)b_hi * (Wn - pwm);
      const uint64_t Vmax = v >= ((u128)1 << 63) ? (1ull << 63) : (uint64_t)v;
      double xe = (double)b_hi * (double)t_np * (double)RT * (double)S_tot * (double)M +
                  (double)M * (double)t_p * (double)Vmax;
      if (mem_mode == 1) xe += (double)b_hi * (double)D;
      else if (mem_mode == 2) xe += (double)b_hi * (double)D * (double)(S_tot * S_tot);
      bool over;
      if (Vmax >= (1ull << 63) || xe >= 72057594037927936.0 * 1.0001) over = true;
      else if (xe < 72057594037927936.0 * 0.9999) over = false;
      else over = xub_exact_over((uint32_t)b_hi, (uint64_t)t_np, (uint64_t)RT, (uint32_t)S_tot, M, (uint64_t)t_p, Vmax,
                                 mem_mode, (uint32_t)b_hi, D);
      if (over) { st = DSTACK_ST_OVERFLOW; break; }
    }
    // ---- a2/a3 at b = 1: X(S, 1) = S (C1 + Mtp PA[S]) + Mtp Q[S] + mem for every attained S; in the same
    //      pass the batch certificate G (below) over the segments m <= S_tot/2 ----
    const uint64_t Mtp = M * (uint64_t)t_p, C1 = (uint64_t)t_np * RT * M;
    const uint64_t SLOM = (uint64_t)slo * M, aM = (uint64_t)asm_us * M;
    const uint64_t memb = mem_mode == 1 ? D : 0ull;
    const float half = 0.5f * (float)S_tot;
    const int mh = S_tot >> 1;
    uint64_t xs[CB];
    float sc[CB];
    uint32_t va = 0, fe = 0;
    float kmax = 0.f, emax = 0.f, G = 0.f;
#pragma unroll
    for (int i = 0; i < CB; ++i) {
      const int S = m0 + i;
      const uint64_t cAi = Mtp * pa[i], cUi = Mtp * (Wn - pw[i]);
      uint64_t X = (uint64_t)S * (C1 + cAi) + cUi;
      if (mem_mode == 1) X += D;
      else if (mem_mode == 2) X += D * (uint64_t)(S * S);
      xs[i] = X;
      const float f = score_f((uint32_t)S, X);
      sc[i] = f;
      const bool valid = S >= 1 && S <= S_tot && lmin[S <= S_tot ? S : 0] != 0;
      const uint64_t cap = (uint64_t)S * SLOM;
      const bool feas = valid && X + (uint64_t)S * aM <= cap && 2 * X <= cap;   // Eq. 11, Eq. 12
      if (valid) { va |= 1u << i; kmax = fmaxf(kmax, f); }
      if (feas) { fe |= 1u << i; emax = fmaxf(emax, f); }
      // Batch certificate: for b >= 2 and s = S/b in segment m = floor(s),
      // X(S, b) >= b (alpha s + beta), alpha = 2 C1 + Mtp PA[m], beta = Mtp Q[m] + mem, hence
      // eta(S, b) <= s / (alpha s + beta)^2; G = max over m <= S_tot/2 of its supremum on [m, m+1).
      if (S <= mh) {
        const float af = (float)(2 * C1 + cAi), bf = (float)(cUi + memb);
        const float lo = (float)S, hi = fminf((float)(S + 1), half);
        float v;
        if (bf == 0.f) v = __int_as_float(0x7f800000);          // s/(alpha s)^2 is unbounded at s -> 0
        else if (bf <= af * lo) { const float x = af * lo + bf; v = lo * rcp_approx(x * x); }
        else if (bf >= af * hi) { const float x = af * hi + bf; v = hi * rcp_approx(x * x); }
        else v = rcp_approx(4.f * af * bf);                     // interior peak at s = beta / alpha
        G = fmaxf(G, v);
      }
    }
    uint32_t Sk, Se;
    uint64_t Xk, Xe;
    fast_argmax<CB>(kmax, va, sc, xs, m0, S_tot, cA, lane, Sk, Xk);
    fast_argmax<CB>(emax, fe, sc, xs, m0, S_tot, cA, lane, Se, Xe);
    if (Se == 0) { st = DSTACK_ST_INFEASIBLE; break; }   // b = 1 is feasible whenever any b is (O3)
    // b* = 1 is certified when the incumbent beats G with a 2^-12 margin (f32 rounding of both sides is
    // < 2^-19); otherwise the generic exact branch-and-bound decides this DNN.
    if (b_hi >= 2) {
      const float Gw = __uint_as_float(__reduce_max_sync(FULL, __float_as_uint(G)));
      if (!(score_f(Se, Xe) * 0.99975586f > Gw)) { prof_one_cold(&a, k, Stab, hist, cA, cU, lane); return; }
    }
    knee = lmin[Sk];
    const uint32_t le = lmin[Se];
    demand = le + (uint32_t)p.margin < (uint32_t)L ? le + (uint32_t)p.margin : (uint32_t)L;
    // d_j(1) = ceil(X(S(g), 1) / (S(g) M Delta)) at g = demand
    if (a.dtab_rows) {
      const uint32_t Sg = Stab[demand];
      uint64_t Xg = Xe;
      if (Sg != Se) {
        uint64_t xo = 0;
#pragma unroll
        for (int i = 0; i < CB; ++i)
          if ((uint32_t)(m0 + i) == Sg) xo = xs[i];
        Xg = shfl_u64(xo, Sg / CB);
      }
      dslots = ceil_div_clamp16(Xg, (uint64_t)Sg * M * (uint64_t)p.slot_us);
    }
  } while (0);
  if (lane == 0) {
    const bool ok = st == DSTACK_ST_OK;
    if (a.ws_RT) { a.ws_RT[k] = RT; a.ws_D[k] = D; }
    if (a.dtab_rows && ok) a.dtab_rows[k * DTAB_ROW] = (uint16_t)dslots;
    if (a.knee) a.knee[k] = ok ? (uint16_t)knee : 0;
    if (a.status) a.status[k] = st;
    if (a.demand) a.demand[k] = ok ? (uint16_t)demand : 0;
    if (a.batch) a.batch[k] = ok ? 1 : 0;
  }
  __syncwarp();
}

template <int CB>
__global__ void __launch_bounds__(256, DSTACK_PROF_MINB) k_prof_fast(const __grid_constant__ ProfArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int L = a.p.L, S_tot = a.p.S_tot;
  uint16_t *Stab = (uint16_t *)smem;
  uint16_t *lmin = Stab + (L + 1);
  const int tab_bytes = ((L + 1 + S_tot + 1) * 2 + 15) & ~15;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char *wreg = smem + tab_bytes + (size_t)warp * prof_warp_bytes(S_tot);
  uint64_t *cA = (uint64_t *)wreg;
  uint64_t *cU = cA + (S_tot + 1);
  uint32_t *hist = (uint32_t *)(cU + (S_tot + 1));
  fill_stab(Stab, L, S_tot);
  // lmin[S] = smallest level l with S(l) = S (0: S not attained); ties between levels -> smaller l
  for (int S = threadIdx.x; S <= S_tot; S += blockDim.x) {
    const int l = S == 0 ? 0 : ((S - 1) * L) / S_tot + 1;
    lmin[S] = (uint16_t)((S >= 1 && l <= L && s_of(l, S_tot, L) == S) ? l : 0);
  }
  for (int m = lane; m <= S_tot; m += 32) hist[m] = 0;
  __syncthreads();
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t k = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; k < a.pb.num_dnn; k += nwarps)
    fast_one<CB>(a, k, Stab, lmin, hist, cA, cU, lane);
}

size_t prof_smem_bytes(const dstack_params_t *p, int warps) {
  return (size_t)(((p->L + 1 + p->S_tot + 1) * 2 + 15) & ~15) + (size_t)warps * prof_warp_bytes(p->S_tot);
}

template <typename KernelT>
static void launch_k(KernelT kern, const ProfArgs &a, int64_t blocks, int threads, size_t smem, cudaStream_t s) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<(unsigned)blocks, threads, smem, s>>>(a);
}

int launch_prof(const ProfArgs &a, cudaStream_t s, int *launches) {
  if (a.pb.num_dnn <= 0) return 0;
  const int threads = 256, warps = threads / 32;
  const size_t smem = prof_smem_bytes(&a.p, warps);
  int64_t blocks = (a.pb.num_dnn + warps - 1) / warps;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  const bool fast = DSTACK_PROF_FAST && a.p.par_mode == 0 && a.p.wse_mode == 0 && a.p.b_min == 1 && !a.knee_only;
  if (fast && a.p.S_tot < 5 * 32) launch_k(k_prof_fast<5>, a, blocks, threads, smem, s);
  else if (fast) launch_k(k_prof_fast<9>, a, blocks, threads, smem, s);
  else if (a.p.par_mode == 0) launch_k(k_prof<0>, a, blocks, threads, smem, s);
  else launch_k(k_prof<1>, a, blocks, threads, smem, s);
  ++*launches;
  return cudaGetLastError() == cudaSuccess ? 0 : DSTACK_ELAUNCH;
}

}  // namespace dstack

#if DSTACK_PROF_STATS
extern "C" int dstack_debug_stats(unsigned long long *out16, int reset) {
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(out16, dstack::g_pstats, sizeof(unsigned long long) * 16) != cudaSuccess) return -1;
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(dstack::g_pstats, z, sizeof(z));
  }
  return 0;
}
#endif
