// Microbenchmark of the phase-E column-split apply pattern at c4's shape: 148 CTAs x 256
// threads, CTA c streams E/148 whole columns (8192 doubles, 64 KiB each) of a 4 GiB
// column-major matrix into a partial u of 8192 rows (8 rows per thread per row tile,
// kB columns' loads in flight), then writes it. Prints us per launch.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>

template <int kB, int kRows>
__global__ void colsplit(const double* __restrict__ A, int64_t ld, const int* __restrict__ cols, const double* __restrict__ xs,
                         int E, double* __restrict__ out) {
  const int c = blockIdx.x, G = gridDim.x;
  const int e0 = (int)((int64_t)E * c / G), e1 = (int)((int64_t)E * (c + 1) / G);
  for (int64_t r0 = 0; r0 < ld; r0 += kRows * blockDim.x) {
    double acc[kRows];
#pragma unroll
    for (int r = 0; r < kRows; ++r) acc[r] = 0.0;
    for (int q = e0; q < e1; q += kB) {
      double av[kB][kRows];
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const bool on = q + u < e1;
        const double* col = A + (int64_t)(on ? cols[q + u] : 0) * ld + r0 + threadIdx.x;
#pragma unroll
        for (int r = 0; r < kRows; ++r) av[u][r] = on ? __ldcs(col + r * blockDim.x) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const double x = q + u < e1 ? xs[q + u] : 0.0;
#pragma unroll
        for (int r = 0; r < kRows; ++r) acc[r] = fma(x, av[u][r], acc[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < kRows; ++r) __stcg(out + (int64_t)c * ld + r0 + threadIdx.x + r * blockDim.x, acc[r]);
  }
}

int main() {
  const int64_t n = 8192, k = 65536;
  double* A; cudaMalloc(&A, sizeof(double) * n * k); cudaMemset(A, 0, sizeof(double) * n * k);
  double* out; cudaMalloc(&out, sizeof(double) * n * 148);
  std::mt19937 rng(1);
  for (int E : {150, 900, 1500}) {
    std::vector<int> cols(E); std::vector<double> xs(E, 1.0);
    std::vector<int> all(k); for (int i = 0; i < k; ++i) all[i] = i;
    std::shuffle(all.begin(), all.end(), rng);
    std::copy(all.begin(), all.begin() + E, cols.begin()); std::sort(cols.begin(), cols.end());
    int* dc; double* dx; cudaMalloc(&dc, 4 * E); cudaMalloc(&dx, 8 * E);
    cudaMemcpy(dc, cols.data(), 4 * E, cudaMemcpyHostToDevice); cudaMemcpy(dx, xs.data(), 8 * E, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](auto kern, const char* name) {
      float best = 1e9;
      for (int it = 0; it < 20; ++it) {
        cudaEventRecord(e0); kern<<<148, 256>>>(A, n, dc, dx, E, out); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (it > 2) best = std::min(best, ms);
      }
      printf("E %5d %-10s %7.1f us  %6.2f TB/s\n", E, name, best * 1e3, E * n * 8.0 / (best * 1e-3) / 1e12);
    };
    run(colsplit<4, 8>, "kB4 r8");
    run(colsplit<8, 8>, "kB8 r8");
    run(colsplit<4, 4>, "kB4 r4");
    run(colsplit<8, 4>, "kB8 r4");
    run(colsplit<16, 2>, "kB16 r2");
  }
  return 0;
}
