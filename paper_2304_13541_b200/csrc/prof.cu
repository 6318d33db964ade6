// prof.cu -- standalone a1-a3 kernel (dstack_batch_opt, dstack_knee): one warp per DNN, grid-stride.
// The per-DNN analysis (row pass, coefficient tables, exact branch-and-bound) is in prof.cuh.
#include "kernels.cuh"
#include "prof.cuh"

namespace dstack {

template <int PAR>
__global__ void __launch_bounds__(256) k_prof(ProfArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int L = a.p.L, S_tot = a.p.S_tot;
  uint16_t *Stab = (uint16_t *)smem;
  const int stab_bytes = ((L + 1) * 2 + 15) & ~15;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t *cA = (uint64_t *)(smem + stab_bytes) + (size_t)warp * 2 * (S_tot + 1);
  uint64_t *cU = cA + (S_tot + 1);
  fill_stab(Stab, L, S_tot);
  __syncthreads();
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t k = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; k < a.pb.num_dnn; k += nwarps) {
    const DnnRes r = analyze_dnn<PAR>(a.pb, a.p, k, Stab, cA, cU, lane, a.knee_only, a.knee_b);
    if (lane == 0) {
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
  return (size_t)(((p->L + 1) * 2 + 15) & ~15) + (size_t)warps * 2 * 8 * (p->S_tot + 1);
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
