// Do cooperative launches on different streams overlap?
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void spin(long long ns, int syncs) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < syncs; ++i) {
    long long t0 = clock64();
    while (clock64() - t0 < ns) {}
    g.sync();
  }
}
int main() {
  cudaStream_t s[8];
  for (int i = 0; i < 8; ++i) cudaStreamCreateWithFlags(&s[i], cudaStreamNonBlocking);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int M : {1, 2, 4, 8}) {
    int grid = 148 / M;
    long long ns = 200000; int syncs = 10;
    void* args[] = {&ns, &syncs};
    cudaEventRecord(a);
    for (int r = 0; r < 8; ++r) cudaLaunchCooperativeKernel((void*)spin, grid, 256, args, 0, s[r % M]);
    for (int i = 0; i < M; ++i) cudaStreamSynchronize(s[i]);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("M=%d streams, grid=%d: 8 launches in %.2f ms (serial would be ~%.2f ms)\n", M, grid, ms, 8 * syncs * 0.105);
    cudaError_t e = cudaGetLastError(); if (e) printf("err %s\n", cudaGetErrorString(e));
  }
}
