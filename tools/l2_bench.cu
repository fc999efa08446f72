// Microbenchmark: repeated read passes over a working set of W MB (148 CTAs x 256 threads,
// 128-bit loads, each CTA a contiguous slice) -- effective bandwidth vs W, i.e. how much of
// a working set the 126 MB L2 keeps between passes.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256, 1) pass(const double2* __restrict__ a, long n2, int reps, double* out, bool serp) {
  long per = (n2 + gridDim.x - 1) / gridDim.x;
  long lo = blockIdx.x * per, hi = min(n2, lo + per);
  double s = 0.0;
  for (int r = 0; r < reps; ++r) {
    const bool rev = serp && (r & 1);
    for (long i0 = lo + threadIdx.x; i0 < hi; i0 += 256 * 8) {
      const long i = rev ? (hi - 1 - i0 + lo) - 7 * 256 : i0;  // serpentine: odd passes run backwards
      double2 v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = (i + 256 * q < hi && i + 256 * q >= lo) ? __ldcg(a + i + 256 * q) : make_double2(0, 0);
#pragma unroll
      for (int q = 0; q < 8; ++q) s += v[q].x + v[q].y;
    }
  }
  if (s == 123.456) out[0] = s;
}
int main() {
  double2* a; double* o;
  const long maxb = 512L << 20;
  cudaMalloc(&a, maxb); cudaMalloc(&o, 8); cudaMemset(a, 0, maxb);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int serp = 0; serp < 2; ++serp)
  for (int mb : {8, 16, 32, 48, 64, 80, 96, 112, 128, 160, 200, 256, 512}) {
    long n2 = (long(mb) << 20) / 16;
    int reps = 20;
    pass<<<148, 256>>>(a, n2, 2, o, serp);
    cudaEventRecord(e0);
    pass<<<148, 256>>>(a, n2, reps, o, serp);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%s W=%4d MB: %.2f us/pass, %.0f GB/s\n", serp ? "serpentine" : "forward   ", mb, ms * 1e3 / reps,
           double(mb << 20) * reps / (ms * 1e-3) / 1e9);
  }
  return 0;
}
