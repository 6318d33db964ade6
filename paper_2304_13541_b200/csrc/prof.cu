// prof.cu -- standalone a1-a3 kernel (dstack_batch_opt, dstack_knee): one warp per DNN, grid-stride.
// The per-DNN analysis (row pass, coefficient tables, exact branch-and-bound) is in prof.cuh.
#include "kernels.cuh"
#include "prof.cuh"

namespace dstack {

__host__ __device__ inline size_t prof_warp_bytes(int S_tot) {
  return (((size_t)20 * (S_tot + 1)) + 15) & ~(size_t)15;   // cA, cU u64 + hist u32
}

template <int PAR>
#ifndef DSTACK_PROF_PF
#define DSTACK_PROF_PF 0   // L2 bulk prefetch of the next DNN's rows: measured slower (r01), off
#endif
#ifndef DSTACK_PROF_MINB
#define DSTACK_PROF_MINB 4
#endif
__global__ void __launch_bounds__(256, DSTACK_PROF_MINB) k_prof(ProfArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int L = a.p.L, S_tot = a.p.S_tot;
  uint16_t *Stab = (uint16_t *)smem;
  const int stab_bytes = ((L + 1) * 2 + 15) & ~15;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char *wreg = smem + stab_bytes + (size_t)warp * prof_warp_bytes(S_tot);
  uint64_t *cA = (uint64_t *)wreg;
  uint64_t *cU = cA + (S_tot + 1);
  uint32_t *hist = (uint32_t *)(cU + (S_tot + 1));
  fill_stab(Stab, L, S_tot);
  __syncthreads();
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t k_first = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  // software-pipelined L2 staging: while DNN k is analysed, the rows of this warp's next DNN are bulk-
  // prefetched into L2 (offsets loaded one iteration ahead so the prefetch never waits on them)
  int64_t pf0 = 0, pf1 = 0;
  if (DSTACK_PROF_PF && lane == 0 && k_first + nwarps < a.pb.num_dnn) { pf0 = a.pb.dnn_row_off[k_first + nwarps]; pf1 = a.pb.dnn_row_off[k_first + nwarps + 1]; }
  for (int64_t k = k_first; k < a.pb.num_dnn; k += nwarps) {
    if (DSTACK_PROF_PF && lane == 0) {
      if (pf1 > pf0) {
        prefetch_l2(a.pb.n + pf0, (pf1 - pf0) * 4);
        prefetch_l2(a.pb.r + pf0, (pf1 - pf0) * 2);
        prefetch_l2(a.pb.d + pf0, (pf1 - pf0) * 4);
      }
      const int64_t kn = k + 2 * nwarps;
      if (kn < a.pb.num_dnn) { pf0 = a.pb.dnn_row_off[kn]; pf1 = a.pb.dnn_row_off[kn + 1]; } else { pf0 = pf1 = 0; }
    }
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
}

size_t prof_smem_bytes(const dstack_params_t *p, int warps) {
  return (size_t)(((p->L + 1) * 2 + 15) & ~15) + (size_t)warps * prof_warp_bytes(p->S_tot);
}

int launch_prof(const ProfArgs &a, cudaStream_t s, int *launches) {
  if (a.pb.num_dnn <= 0) return 0;
  const int threads = 256, warps = threads / 32;
  const size_t smem = prof_smem_bytes(&a.p, warps);
  int64_t blocks = (a.pb.num_dnn + warps - 1) / warps;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
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
