// Does an L2 persisting window speed up repeated full passes over a 200 MB matrix (c2's
// size, > 126 MB L2)? Streams the buffer with the A^T r pass's load shape (256 threads per
// SM, 16 x 128-bit loads in flight per lane), 20 passes back to back, with and without a
// cudaAccessPolicyWindow (persisting) over the first `win` bytes.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <algorithm>

__global__ void pass(const double2* __restrict__ a, int64_t n2, double* out, int persist_hint, int64_t win2) {
  const int64_t nw = (int64_t)gridDim.x * blockDim.x / 32, gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int l = threadIdx.x & 31;
  const int64_t per = (n2 + nw - 1) / nw, lo = gw * per, hi = lo + per < n2 ? lo + per : n2;
  double s = 0.0;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  for (int64_t e = lo + l; e < hi; e += 32 * 16) {
    double2 v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int64_t i = e + 32 * u;
      if (i < hi) {
        if (persist_hint && i < win2)
          asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;" : "=d"(v[u].x), "=d"(v[u].y) : "l"(a + i), "l"(pol));
        else
          asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v[u].x), "=d"(v[u].y) : "l"(a + i));
      } else v[u] = make_double2(0, 0);
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) s += v[u].x + v[u].y;
  }
  if (s == 12345.0) out[0] = s;
}

int main() {
  int dev = 0; cudaDeviceProp pr; cudaGetDeviceProperties(&pr, dev);
  printf("L2 %d MB, persisting max %d MB, window max %d MB\n", pr.l2CacheSize >> 20, pr.persistingL2CacheMaxSize >> 20, pr.accessPolicyMaxWindowSize >> 20);
  const int64_t bytes = 200LL << 20, n2 = bytes / 16;
  double2* a; double* out; cudaMalloc(&a, bytes); cudaMalloc(&out, 8); cudaMemset(a, 0, bytes);
  cudaStream_t st; cudaStreamCreate(&st);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, int hint, int64_t win) {
    for (int w = 0; w < 3; ++w) pass<<<148, 256, 0, st>>>(a, n2, out, hint, win / 16);
    cudaEventRecord(e0, st);
    for (int it = 0; it < 20; ++it) pass<<<148, 256, 0, st>>>(a, n2, out, hint, win / 16);
    cudaEventRecord(e1, st); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-44s %7.1f us/pass  %6.2f TB/s effective\n", name, ms * 1e3 / 20, bytes / (ms * 1e-3 / 20) / 1e12);
  };
  run("no window", 0, 0);
  for (int64_t winmb : {64, 96, 110}) {
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min<int64_t>(winmb << 20, pr.persistingL2CacheMaxSize));
    cudaStreamAttrValue at = {};
    at.accessPolicyWindow.base_ptr = a;
    at.accessPolicyWindow.num_bytes = std::min<int64_t>(winmb << 20, pr.accessPolicyMaxWindowSize);
    at.accessPolicyWindow.hitRatio = 1.0f;
    at.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    at.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &at);
    char nm[64]; snprintf(nm, 64, "persisting window %lld MB", (long long)winmb); run(nm, 0, 0);
    snprintf(nm, 64, "window %lld MB + evict_last hint", (long long)winmb); run(nm, 1, winmb << 20);
    at.accessPolicyWindow.num_bytes = 0; cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &at);
    cudaCtxResetPersistingL2Cache();
  }
  for (int64_t winmb : {64, 96, 110}) {
    char nm[64]; snprintf(nm, 64, "evict_last hint only, first %lld MB", (long long)winmb); run(nm, 1, winmb << 20);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
