// fp64 tensor-core (DMMA m8n8k4) and DFMA peak on this GPU: register-only loops,
// all SMs, CUDA-event timing. Prints TFLOP/s.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dmma_loop(double* out, int iters) {
  double c[16][2];
  for (int i = 0; i < 16; ++i) c[i][0] = c[i][1] = 0.0;
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0.0;
  for (int i = 0; i < 16; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}
__global__ void dfma_loop(double* out, int iters) {
  double c[16];
  for (int i = 0; i < 16; ++i) c[i] = threadIdx.x;
  const double a = 1.0000001, b = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0.0;
  for (int i = 0; i < 16; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}
int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {4, 8, 16}) {
    const int iters = 20000;
    dmma_loop<<<sms, warps * 32>>>(out, 100);
    cudaEventRecord(e0);
    dmma_loop<<<sms, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = double(sms) * warps * iters * 16 * 512.0;
    printf("DMMA m8n8k4: %2d warps/SM  %.2f TFLOP/s\n", warps, flops / (ms * 1e-3) / 1e12);
  }
  for (int warps : {8, 16, 32}) {
    const int iters = 20000;
    dfma_loop<<<sms, warps * 32>>>(out, 100);
    cudaEventRecord(e0);
    dfma_loop<<<sms, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = double(sms) * warps * 32 * iters * 16 * 2.0;
    printf("DFMA:        %2d warps/SM  %.2f TFLOP/s\n", warps, flops / (ms * 1e-3) / 1e12);
  }
  return 0;
}
