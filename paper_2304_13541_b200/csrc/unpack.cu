// unpack.cu -- compact row transport (dstack_unpack_nr): rows cross PCIe as nr = n | R << 12 (u16) plus d (u32),
// 6 bytes instead of 10, and are expanded on the device into the problem's n (u32) and r (u16) arrays.  Pure data
// movement (no method arithmetic): 16-byte loads of 8 encoded rows per thread, HBM-bound.
#include "kernels.cuh"

namespace dstack {

__global__ void __launch_bounds__(256) k_unpack_nr(int64_t num_rows, const uint16_t *__restrict__ nr,
                                                   uint32_t *__restrict__ n, uint16_t *__restrict__ r) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t nvec = num_rows >> 3;   // groups of 8 rows
  const uint4 *nr8 = reinterpret_cast<const uint4 *>(nr);
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += stride) {
    const uint4 w = nr8[v];
    const uint32_t x[4] = {w.x, w.y, w.z, w.w};
    uint32_t nn[8];
    uint32_t rr[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t lo = x[i] & 0xFFFFu, hi = x[i] >> 16;
      nn[2 * i] = lo & 0x0FFFu;
      nn[2 * i + 1] = hi & 0x0FFFu;
      rr[i] = (lo >> 12) | ((hi >> 12) << 16);
    }
    reinterpret_cast<uint4 *>(n)[2 * v] = make_uint4(nn[0], nn[1], nn[2], nn[3]);
    reinterpret_cast<uint4 *>(n)[2 * v + 1] = make_uint4(nn[4], nn[5], nn[6], nn[7]);
    reinterpret_cast<uint4 *>(r)[v] = make_uint4(rr[0], rr[1], rr[2], rr[3]);
  }
  // tail rows
  for (int64_t i = (nvec << 3) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < num_rows; i += stride) {
    const uint32_t e = nr[i];
    n[i] = e & 0x0FFFu;
    r[i] = (uint16_t)(e >> 12);
  }
}

int launch_unpack_nr(int64_t num_rows, const uint16_t *nr, uint32_t *n, uint16_t *r, cudaStream_t s, int *launches) {
  if (num_rows <= 0) return 0;
  int64_t blocks = ((num_rows >> 3) + 255) / 256;
  if (blocks < 1) blocks = 1;
  const int64_t cap = (int64_t)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  k_unpack_nr<<<(unsigned)blocks, 256, 0, s>>>(num_rows, nr, n, r);
  ++*launches;
  return cudaGetLastError() == cudaSuccess ? 0 : DSTACK_ELAUNCH;
}

}  // namespace dstack

namespace dstack {

// 5-byte rows: w (u32) = d | (R - 1) << 26 | (n >> 8) << 28 and lo (u8) = n & 255 (d < 2^26, 1 <= R <= 4,
// n < 4096); four rows per thread: one 16-byte load of w and one 4-byte load of lo.
__global__ void __launch_bounds__(256) k_unpack_w5(int64_t num_rows, const uint32_t *__restrict__ w,
                                                   const uint8_t *__restrict__ lo, uint32_t *__restrict__ n,
                                                   uint16_t *__restrict__ r, uint32_t *__restrict__ d) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t nvec = num_rows >> 2;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += stride) {
    const uint4 ww = reinterpret_cast<const uint4 *>(w)[v];
    const uint32_t ll = reinterpret_cast<const uint32_t *>(lo)[v];
    const uint32_t x[4] = {ww.x, ww.y, ww.z, ww.w};
    uint32_t nn[4], dd[4], rr[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      dd[i] = x[i] & 0x03FFFFFFu;
      rr[i] = ((x[i] >> 26) & 3u) + 1u;
      nn[i] = ((x[i] >> 28) << 8) | ((ll >> (8 * i)) & 0xFFu);
    }
    reinterpret_cast<uint4 *>(n)[v] = make_uint4(nn[0], nn[1], nn[2], nn[3]);
    reinterpret_cast<uint4 *>(d)[v] = make_uint4(dd[0], dd[1], dd[2], dd[3]);
    reinterpret_cast<uint2 *>(r)[v] = make_uint2(rr[0] | (rr[1] << 16), rr[2] | (rr[3] << 16));
  }
  for (int64_t i = (nvec << 2) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < num_rows; i += stride) {
    const uint32_t x = w[i];
    d[i] = x & 0x03FFFFFFu;
    r[i] = (uint16_t)(((x >> 26) & 3u) + 1u);
    n[i] = ((x >> 28) << 8) | lo[i];
  }
}

int launch_unpack_w5(int64_t num_rows, const uint32_t *w, const uint8_t *lo, uint32_t *n, uint16_t *r, uint32_t *d,
                     cudaStream_t s, int *launches) {
  if (num_rows <= 0) return 0;
  int64_t blocks = ((num_rows >> 2) + 255) / 256;
  if (blocks < 1) blocks = 1;
  const int64_t cap = (int64_t)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  k_unpack_w5<<<(unsigned)blocks, 256, 0, s>>>(num_rows, w, lo, n, r, d);
  ++*launches;
  return cudaGetLastError() == cudaSuccess ? 0 : DSTACK_ELAUNCH;
}

}  // namespace dstack
