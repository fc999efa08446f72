// Pure HBM read bandwidth on this B200 (the ceiling of the A^T r streaming pass):
// a 4 GiB buffer read with 128-bit non-allocating loads, grid = 148 x blocks_per_sm,
// each warp streaming a contiguous range with 8 loads in flight per lane.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__global__ void read_kernel(const double2* __restrict__ a, int64_t n2, double* out) {
  const int64_t nw = (int64_t)gridDim.x * blockDim.x / 32, gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int l = threadIdx.x & 31;
  const int64_t per = (n2 + nw - 1) / nw, lo = gw * per, hi = lo + per < n2 ? lo + per : n2;
  double s = 0.0;
  for (int64_t e = lo + l; e < hi; e += 32 * 8) {
    double2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t i = e + 32 * u;
      if (i < hi) asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v[u].x), "=d"(v[u].y) : "l"(a + i));
      else v[u] = make_double2(0, 0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) s += v[u].x + v[u].y;
  }
  if (s == 12345.0) out[0] = s;
}

int main() {
  const int64_t bytes = 4LL << 30, n2 = bytes / 16;
  double2* a; double* out;
  cudaMalloc(&a, bytes); cudaMalloc(&out, 8);
  cudaMemset(a, 0, bytes);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int bps : {1, 2, 4}) for (int thr : {256, 512}) {
    float best = 1e9;
    for (int it = 0; it < 6; ++it) {
      cudaEventRecord(e0);
      read_kernel<<<148 * bps, thr>>>(a, n2, out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (it > 0 && ms < best) best = ms;
    }
    printf("blocks/SM %d threads %d: %.1f GB/s\n", bps, thr, bytes / (best * 1e-3) / 1e9);
  }
  return 0;
}
