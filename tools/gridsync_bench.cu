// Microbenchmark: cost of cooperative grid.sync() on this GPU vs grid size.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int iters, unsigned long long* out) {
  cg::grid_group g = cg::this_grid();
  unsigned long long t0;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  for (int i = 0; i < iters; ++i) g.sync();
  unsigned long long t1;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = t1 - t0;
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int grids[] = {8, 16, 32, 64, 74, 148, 296};
  for (int threads : {256, 512, 1024}) for (int gsz : grids) {
    int per = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, threads, 0);
    if (gsz > per * sms) continue;
    int iters = 2000; void* args[] = {&iters, &d};
    cudaLaunchCooperativeKernel((void*)k, gsz, threads, args, 0, 0);
    cudaDeviceSynchronize();
    cudaLaunchCooperativeKernel((void*)k, gsz, threads, args, 0, 0);
    cudaDeviceSynchronize();
    unsigned long long ns; cudaMemcpy(&ns, d, 8, cudaMemcpyDeviceToHost);
    printf("threads %4d grid %4d : %.3f us per grid.sync\n", threads, gsz, ns / 1000.0 / iters);
  }
  // launch overhead of an empty cooperative kernel
  int iters = 0; void* args[] = {&iters, &d};
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < 100; ++r) cudaLaunchCooperativeKernel((void*)k, 148, 512, args, 0, 0);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("empty cooperative launch (148x512): %.2f us each\n", ms * 1000 / 100);
  return 0;
}
