// prof.cu -- a1-a3: profile ingest, knee (Eq. 6) and batch/GPU% search (Eqs. 7-12).
//
// One warp per DNN, grid-stride.  The kernel-row SoA (n u32, R u16, d u32 = 10 B/row) is streamed
// once with coalesced loads; the per-DNN reduction builds, in a per-warp shared-memory slice,
// the histogram of R_i and R_i*n_i over the widths n_i <= S_tot and turns it with a warp scan
// into two coefficient tables (linear mode, b-independent):
//     cA[m] = M t_p sum_{1<=n_i<=m} R_i            (the "S * A(S,b)" term, A = rows that fit)
//     cU[m] = M t_p sum_{n_i>m}     R_i n_i        (the "U(S,b)" term, saturated rows)
// so that for every (level l, batch b), with S = S(l) and m = floor(S/b),
//     X(l,b) = E_t*S*M = S*(w_b*C1 + cA[m]) + b*cU[m] + mem,   C1 = t_np*RT*M
// costs O(1) (Eqs. 2-5 multiplied through by S*M; w_b = b per_request, 1 per_launch;
// mem = 0 | b*D | b*D*S^2 for Eq. 3 off | bw | verbatim).  In threads mode N_i(b) = ceil(b theta/2048)
// does not factor out b, so the tables are rebuilt per b (an O(K) pass each).
//
// The (l, b) search is exhaustive over the grid (lanes over l, loop over b); each comparison of
// eta = b S / X^2 is a float filter with an exact 128-bit fallback (common.cuh), so the argmax and
// its tie-breaks (smaller l, then smaller b) are exact.
#include "kernels.cuh"

namespace dstack {



struct Best {
  uint32_t found, P, l, b;   // P = b*S (eta numerator) or S (knee)
  uint64_t X;
};

__device__ __forceinline__ bool better(const Best &c, const Best &o) {
  if (!c.found) return false;
  if (!o.found) return true;
  int s = cmp_score(c.P, c.X, (float)c.X, o.P, o.X, (float)o.X);
  if (s != 0) return s > 0;
  return c.l < o.l || (c.l == o.l && c.b < o.b);
}

__device__ __forceinline__ Best warp_best(Best v) {
#pragma unroll
  for (int m = 16; m; m >>= 1) {
    Best o;
    o.found = __shfl_xor_sync(FULL, v.found, m);
    o.P = __shfl_xor_sync(FULL, v.P, m);
    o.l = __shfl_xor_sync(FULL, v.l, m);
    o.b = __shfl_xor_sync(FULL, v.b, m);
    o.X = shfl_xor_u64(v.X, m);
    if (better(o, v)) v = o;
  }
  return v;
}

// Histogram + scan into the coefficient tables.  PAR 0: bins of n (b-independent, b_eval unused);
// PAR 1: bins of N = ceil(b_eval * theta / 2048).  Returns W = sum R*N (threads) via *Wout.
template <int PAR>
__device__ __forceinline__ void build_tables(const uint32_t *__restrict__ n, const uint16_t *__restrict__ r,
                                             int32_t K, int32_t S_tot, uint64_t Mtp, uint64_t Wn, int32_t b_eval,
                                             uint64_t *cA, uint64_t *cU, int lane) {
  for (int m = lane; m <= S_tot; m += 32) { cA[m] = 0; cU[m] = 0; }
  __syncwarp();
  uint64_t W = Wn;
  if (PAR == 1) W = 0;
  for (int i = lane; i < K; i += 32) {
    uint64_t nn = n[i];
    uint32_t R = r[i];
    uint64_t N = PAR == 0 ? nn : ((uint64_t)b_eval * nn + 2047) >> 11;
    if (PAR == 1) W += (uint64_t)R * N;
    if (N >= 1 && N <= (uint64_t)S_tot) {
      atomicAdd((unsigned long long *)&cA[N], (unsigned long long)R);
      atomicAdd((unsigned long long *)&cU[N], (unsigned long long)(R * N));
    }
  }
  if (PAR == 1) W = warp_sum_u64(W);
  __syncwarp();
  uint64_t carryA = 0, carryW = 0;
  for (int base = 0; base <= S_tot; base += 32) {
    const int m = base + lane;
    uint64_t a = m <= S_tot ? cA[m] : 0, w = m <= S_tot ? cU[m] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      uint64_t ua = shfl_up_u64(a, d), uw = shfl_up_u64(w, d);
      if (lane >= d) { a += ua; w += uw; }
    }
    a += carryA; w += carryW;
    if (m <= S_tot) { cA[m] = Mtp * a; cU[m] = Mtp * (W - w); }
    carryA = shfl_u64(a, 31); carryW = shfl_u64(w, 31);
  }
  __syncwarp();
}

template <int PAR>
__device__ __forceinline__ uint64_t cell_X(int32_t S, int32_t b, uint32_t magic, uint64_t wC1, const uint64_t *cA,
                                           const uint64_t *cU, int mem_mode, uint64_t D) {
  int32_t m;
  uint64_t ub;
  if (PAR == 0) { m = (b == 1) ? S : (int32_t)__umulhi((uint32_t)S, magic); ub = (uint64_t)b; }
  else { m = S; ub = 1; }
  uint64_t X = (uint64_t)S * (wC1 + cA[m]) + ub * cU[m];
  if (mem_mode == 1) X += (uint64_t)b * D;
  else if (mem_mode == 2) X += (uint64_t)b * D * (uint64_t)S * (uint64_t)S;
  return X;
}

template <int PAR>
__global__ void __launch_bounds__(256) k_prof(ProfArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int L = a.p.L, S_tot = a.p.S_tot;
  uint16_t *Stab = (uint16_t *)smem;                                   // [L+1]
  const int stab_bytes = ((L + 1) * 2 + 15) & ~15;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t *cA = (uint64_t *)(smem + stab_bytes) + (size_t)warp * 2 * (S_tot + 1);
  uint64_t *cU = cA + (S_tot + 1);
  for (int l = threadIdx.x; l <= L; l += blockDim.x) Stab[l] = (uint16_t)s_of(l, S_tot, L);
  __syncthreads();

  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t k = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; k < a.pb.num_dnn; k += nwarps) {
    const int64_t r0 = a.pb.dnn_row_off[k], r1 = a.pb.dnn_row_off[k + 1];
    const int64_t K64 = r1 - r0;
    const int32_t t_p = a.pb.t_p[k], t_np = a.pb.t_np[k], slo = a.pb.slo_us[k], asm_us = a.pb.asm_us[k];
    const int32_t bmax = a.pb.bmax[k], mbw = a.pb.mem_bw[k];
    const int mem_mode = a.p.mem_mode;
    const uint64_t M = mem_mode == 0 ? 1 : (uint64_t)mbw;
    const int32_t b_lo = a.p.b_min, b_hi = bmax < a.p.b_max ? bmax : a.p.b_max;
    const int32_t b_eval = a.knee_only ? a.knee_b : b_hi;   // where the overflow bound is checked

    // ---- header validation (DSTACK_ST_INVALID conditions, dstack.h) ----
    bool invalid = K64 < 1 || K64 > DSTACK_MAX_ROWS_PER_DNN || t_p < 1 || t_np < 0 || slo < 1 ||
                   slo > (1 << 30) || (slo % a.p.slot_us) != 0 || asm_us < 0 || asm_us > (1 << 24) || bmax < 1 ||
                   (mem_mode != 0 && (mbw < 1 || mbw > (1 << 24)));
    uint8_t st = DSTACK_ST_OK;
    uint16_t o_dem = 0, o_knee = 0;
    uint8_t o_b = 0;
    if (!invalid) {
      const int32_t K = (int32_t)K64;
      const uint32_t *n = a.pb.n + r0;
      const uint16_t *r = a.pb.r + r0;
      const uint32_t *d = a.pb.d + r0;
      // ---- a1: one coalesced pass over the rows: totals, overflow bound, width histogram ----
      if (PAR == 0) { for (int m = lane; m <= S_tot; m += 32) { cA[m] = 0; cU[m] = 0; } __syncwarp(); }
      uint64_t RT = 0, D = 0, Wn = 0, Vmax = 0;
      uint32_t anyR0 = 0, anyN = 0;
      for (int i = lane; i < K; i += 32) {
        const uint64_t nn = n[i];
        const uint32_t R = r[i];
        const uint64_t dd = d[i];
        RT += R; D += (uint64_t)R * dd; Wn += (uint64_t)R * nn;
        anyR0 |= (R == 0); anyN |= (nn != 0);
        const uint64_t Nb = PAR == 0 ? (uint64_t)b_eval * nn : ((uint64_t)b_eval * nn + 2047) >> 11;
        if (Nb >= 1) Vmax = sat_add(Vmax, (uint64_t)R * (Nb > (uint64_t)S_tot ? Nb : (uint64_t)S_tot));
        if (PAR == 0 && nn >= 1 && nn <= (uint64_t)S_tot) {
          atomicAdd((unsigned long long *)&cA[nn], (unsigned long long)R);
          atomicAdd((unsigned long long *)&cU[nn], (unsigned long long)(R * nn));
        }
      }
      RT = warp_sum_u64(RT); D = warp_sum_u64(D); Wn = warp_sum_u64(Wn); Vmax = warp_sum_sat(Vmax);
      anyR0 = warp_or(anyR0); anyN = warp_or(anyN);
      if (anyR0 || (t_np == 0 && !anyN && (mem_mode == 0 || D == 0))) {
        st = DSTACK_ST_INVALID;
      } else if (!a.knee_only && b_hi < b_lo) {
        st = DSTACK_ST_INFEASIBLE;
      } else {
        // X(L, b_eval) = w t_np RT S_tot M + M t_p Vmax + mem  (the maximum of X over the grid)
        const u128 w = a.p.wse_mode == 0 ? (u128)b_eval : (u128)1;
        u128 Xub = w * (u128)t_np * (u128)RT * (u128)S_tot * (u128)M + (u128)M * (u128)t_p * (u128)Vmax;
        if (mem_mode == 1) Xub += (u128)b_eval * (u128)D;
        else if (mem_mode == 2) Xub += (u128)b_eval * (u128)D * (u128)(S_tot * S_tot);
        if (Vmax >= (1ull << 63) || Xub >= (u128)X_LIMIT) st = DSTACK_ST_OVERFLOW;
      }
      if (st == DSTACK_ST_OK) {
        const uint64_t Mtp = M * (uint64_t)t_p;
        const uint64_t C1 = (uint64_t)t_np * RT * M;
        if (PAR == 0) {
          // scan the histogram in place into cA / cU
          __syncwarp();
          uint64_t carryA = 0, carryW = 0;
          for (int base = 0; base <= S_tot; base += 32) {
            const int m = base + lane;
            uint64_t av = m <= S_tot ? cA[m] : 0, wv = m <= S_tot ? cU[m] : 0;
#pragma unroll
            for (int dd = 1; dd < 32; dd <<= 1) {
              uint64_t ua = shfl_up_u64(av, dd), uw = shfl_up_u64(wv, dd);
              if (lane >= dd) { av += ua; wv += uw; }
            }
            av += carryA; wv += carryW;
            if (m <= S_tot) { cA[m] = Mtp * av; cU[m] = Mtp * (Wn - wv); }
            carryA = shfl_u64(av, 31); carryW = shfl_u64(wv, 31);
          }
          __syncwarp();
        }
        int32_t kb = a.knee_b;
        if (!a.knee_only) {
          // ---- a3: exhaustive feasible argmax of eta = b S / X^2 (Eqs. 9-12) ----
          const uint64_t SLOM = (uint64_t)slo * M;
          Best best; best.found = 0; best.P = 0; best.l = 0; best.b = 0; best.X = 0;
          for (int32_t b = b_lo; b <= b_hi; ++b) {
            if (PAR == 1) build_tables<1>(n, r, K, S_tot, Mtp, 0, b, cA, cU, lane);
            const uint32_t magic = b == 1 ? 0u : (uint32_t)(0xFFFFFFFFu / (uint32_t)b) + 1u;
            const uint64_t wC1 = (a.p.wse_mode == 0 ? (uint64_t)b : 1ull) * C1;
            const uint64_t baM = (uint64_t)b * (uint64_t)asm_us * M;
            for (int32_t l = 1 + lane; l <= L; l += 32) {
              const int32_t S = Stab[l];
              const uint64_t X = cell_X<PAR>(S, b, magic, wC1, cA, cU, mem_mode, D);
              const uint64_t cap = (uint64_t)S * SLOM;
              if (X + (uint64_t)S * baM > cap || 2 * X > cap) continue;   // Eq. 11, Eq. 12
              Best c; c.found = 1; c.P = (uint32_t)(b * S); c.l = l; c.b = b; c.X = X;
              if (better(c, best)) best = c;
            }
          }
          best = warp_best(best);
          if (!best.found) {
            st = DSTACK_ST_INFEASIBLE;
          } else {
            int32_t dm = (int32_t)best.l + a.p.margin;
            o_dem = (uint16_t)(dm < L ? dm : L);
            o_b = (uint8_t)best.b;
            kb = (int32_t)best.b;
          }
        }
        if (st == DSTACK_ST_OK) {
          // ---- a2: knee(kb) = argmax_l S / X^2 (Eq. 6), ties -> smaller l ----
          if (PAR == 1) build_tables<1>(n, r, K, S_tot, Mtp, 0, kb, cA, cU, lane);
          const uint32_t magic = kb == 1 ? 0u : (uint32_t)(0xFFFFFFFFu / (uint32_t)kb) + 1u;
          const uint64_t wC1 = (a.p.wse_mode == 0 ? (uint64_t)kb : 1ull) * C1;
          Best kn; kn.found = 0; kn.P = 0; kn.l = 0; kn.b = 0; kn.X = 0;
          for (int32_t l = 1 + lane; l <= L; l += 32) {
            const int32_t S = Stab[l];
            Best c; c.found = 1; c.P = (uint32_t)S; c.l = l; c.b = 0;
            c.X = cell_X<PAR>(S, kb, magic, wC1, cA, cU, mem_mode, D);
            if (better(c, kn)) kn = c;
          }
          kn = warp_best(kn);
          o_knee = (uint16_t)kn.l;
        }
      }
    } else {
      st = DSTACK_ST_INVALID;
    }
    if (lane == 0) {
      if (a.knee) a.knee[k] = st == DSTACK_ST_OK ? o_knee : 0;
      if (a.status) a.status[k] = st;
      if (!a.knee_only) {
        if (a.demand) a.demand[k] = st == DSTACK_ST_OK ? o_dem : 0;
        if (a.batch) a.batch[k] = st == DSTACK_ST_OK ? o_b : 0;
      }
    }
    __syncwarp();
  }
}

size_t prof_smem_bytes(const dstack_params_t *p, int warps) {
  return (size_t)(((p->L + 1) * 2 + 15) & ~15) + (size_t)warps * 2 * 8 * (p->S_tot + 1);
}

int launch_prof(const ProfArgs &a, cudaStream_t s, int *launches) {
  if (a.pb.num_dnn <= 0) return 0;
  const int threads = 256, warps = threads / 32;
  size_t smem = prof_smem_bytes(&a.p, warps);
  int64_t blocks = (a.pb.num_dnn + warps - 1) / warps;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
  if (a.p.par_mode == 0) {
    cudaFuncSetAttribute(k_prof<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_prof<0><<<(unsigned)blocks, threads, smem, s>>>(a);
  } else {
    cudaFuncSetAttribute(k_prof<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_prof<1><<<(unsigned)blocks, threads, smem, s>>>(a);
  }
  ++*launches;
  return cudaGetLastError() == cudaSuccess ? 0 : DSTACK_ELAUNCH;
}

}  // namespace dstack
