// Lockstep contraction microbenchmark (c5 shapes): Corr = A^T R with A 1024 x 4096
// (column-major, ld 1024) and R 1024 x 512, 128 x 64 DMMA tiles over 32-deep chunks,
// one 512-thread CTA per SM, each CTA streaming `units` chunks of its own tiles.
// Modes isolate where a unit's time goes:
//   0  compute only (operands already in shared memory)
//   1  warp-0 producer: TMA box of the A tile + cp.async R pieces, 3-stage mbarrier ring
//   2  as 1, A tile only (TMA)
//   3  as 1, R pieces only (cp.async)
//   4  all threads issue cp.async for both tiles, 2 stages, one CTA barrier per chunk
//   5  as 1 with 4 producer warps (one per SM sub-partition) for the R pieces
//   6  TMA A + one 2D TMA box per R column (box {36, 1}), lane 0
//   7  TMA A + R columns by tile::gather4 (four columns per copy), lane 0
//   8  TMA A + one 1D bulk copy per R column, spread over warp 0's lanes
//   9  TMA A + one 2D TMA box of 64 consecutive R columns (slot-ordered R: no gather)
//  10  latency: one A box (36 x 128) at a time, issue -> full barrier, no compute
//  11  latency: one W-layout A box (132 x 32) at a time
//  12  latency: the A tile by all threads' cp.async (wait_group 0 + CTA barrier), one at a time
//  13  as 9 with a dedicated producer warp (17 warps: the 16 DMMA warps never issue copies)
//  15  as 9 the way the lockstep issues: thread 0 alone (expect_tx + two boxes), full
//      barrier count 1, no cp.async arrivals
//  14  as 9 with a lookahead of kRing - 2 units: warp 0 refills the stage released two
//      units ago (no wait on the slowest warp's previous unit)
// R columns are gathered through a permutation (signal = 37 c mod 512), as the lockstep
// gathers its unfinished signals.
// Prints us per unit and the DMMA rate. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 sk_bench.cu -o sk_bench
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <algorithm>
#include <cmath>
#include <vector>

constexpr int kPT = 512, kPW = 16;
constexpr int kTM = 128, kTN = 64, kTK = 32, kSS = 36;
constexpr int kWR = 8, kWC = 2, kRT = 2, kCT = 4;
constexpr int kStage = (kTM + kTN) * kSS;
constexpr int kRing = 3;
constexpr unsigned kAll = 0xffffffffu;

__shared__ __align__(8) uint64_t s_full[kRing];
__shared__ __align__(8) uint64_t s_empty[kRing];

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp16(double* dst, const double* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(su32(dst)), "l"(src));
}
__device__ __forceinline__ void mb_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok)
                 : "r"(su32(bar)), "r"(parity)
                 : "memory");
}

template <int CT = kCT>
__device__ __forceinline__ void mma_unit(const double* Xs, double (&acc)[kRT][kCT][2]) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, g = l >> 2, tg = l & 3;
  const int wr = w % kWR, wc = w / kWR;
  const double* Ys = Xs + kTM * kSS;
#pragma unroll
  for (int ks = 0; ks < kTK / 4; ++ks) {
    double av[kRT], bv[CT];
#pragma unroll
    for (int h = 0; h < kRT; ++h) av[h] = Xs[((h * kWR + wr) * 8 + g) * kSS + ks * 4 + tg];
#pragma unroll
    for (int c = 0; c < CT; ++c) bv[c] = Ys[((wc * CT + c) * 8 + g) * kSS + ks * 4 + tg];
#pragma unroll
    for (int h = 0; h < kRT; ++h)
#pragma unroll
      for (int c = 0; c < CT; ++c) dmma(acc[h][c], av[h], bv[c]);
  }
}

struct Args {
  CUtensorMap tm;
  CUtensorMap tmr;  // R, box {36, 1}
  CUtensorMap tmr64;  // R, box {36, 64}
  CUtensorMap tmw;    // A, box {132, 32}
  int validate;
  int stagger;
  int ct;  // DMMA width of the ring modes' units (4: 64 signals, 2: 32)  // 1: each CTA starts its chunk walk at a different depth (no CTAs on the same R lines at once)
  const double* a;
  const double* r;
  int64_t ld, k, b;
  int units;
  int mode;
  double* out;
};

// unit u of CTA g: tile (g * 7 + u / 32) mod 256, chunk u mod 32
__device__ __forceinline__ void unit_coords(const Args& p, int u, int& j0, int& a0, int& k0) {
  const int tile = (blockIdx.x * 7 + u / 32) % 256;
  j0 = (tile % 32) * kTM;
  a0 = (tile / 32) * kTN;
  k0 = ((u + p.stagger * blockIdx.x) % 32) * kTK;
}

__device__ __forceinline__ int sig_of(int c) { return (37 * c) % 512; }
__device__ __forceinline__ void issue_y(const Args& p, int u, double* Ys, int lane_base, int nlanes_total, int lane) {
  int j0, a0, k0;
  unit_coords(p, u, j0, a0, k0);
  // lanes [0, nlanes_total): piece (lane & 15) of columns lane >> 4, + nlanes_total / 16, ...
  const int gl = lane_base + lane;
  const int kk = (gl & 15) * 2;
  for (int c = gl >> 4; c < kTN; c += nlanes_total / 16)
    cp16(Ys + c * kSS + kk, p.r + sig_of(a0 + c) * p.ld + k0 + kk);
}

__global__ void __launch_bounds__(kPT, 1) bench_kernel(const __grid_constant__ Args p) {
  extern __shared__ __align__(128) double dsm[];
  double* stage = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(dsm) + 127) & ~uintptr_t(127));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  double acc[kRT][kCT][2] = {};
  const int nprod = p.mode == 5 ? 4 : 1;  // producer warps: w % 4 == 0 && w < 4 * nprod ... (warps 0,4,8,12)
  const bool producer = p.mode == 5 ? (w % 4 == 0) : (w == 0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kRing; ++s) {
      const int cnt = (p.mode >= 10 && p.mode != 14) ? 1 : 1 + 32 * nprod;  // 15: the issuing thread alone  // latency modes: the expect_tx arrival alone
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&s_full[s])), "r"(cnt));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&s_empty[s])), "r"(kPW));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < kRing * kStage; i += kPT) stage[i] = 1e-3 * (i % 97);
  __syncthreads();
  if (p.mode == 0) {
    for (int u = 0; u < p.units; ++u) mma_unit(stage + (u % kRing) * kStage, acc);
  } else if (p.mode == 10 || p.mode == 11) {
    for (int u = 0; u < p.units; ++u) {
      int j0, a0, k0;
      unit_coords(p, u, j0, a0, k0);
      if (threadIdx.x == 0) {
        const bool w = p.mode == 11;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&s_full[0])),
                     "r"(w ? 32 * 132 * 8 : kTM * kSS * 8)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
            "[%4];" ::"r"(su32(stage)),
            "l"(reinterpret_cast<uint64_t>(w ? &p.tmw : &p.tm)), "r"(w ? j0 % 1024 : k0), "r"(w ? (u * 32) % 4096 : j0),
            "r"(su32(&s_full[0]))
            : "memory");
        mb_wait(&s_full[0], u & 1u);
      }
      __syncthreads();
    }
    acc[0][0][0] = stage[threadIdx.x];
  } else if (p.mode == 12) {
    for (int u = 0; u < p.units; ++u) {
      int j0, a0, k0;
      unit_coords(p, u, j0, a0, k0);
      for (int e = threadIdx.x; e < kTM * 16; e += kPT) {
        const int r = e / 16, kk = (e % 16) * 2;
        cp16(stage + r * kSS + kk, p.a + (j0 + r) * p.ld + k0 + kk);
      }
      asm volatile("cp.async.commit_group;\n" ::);
      asm volatile("cp.async.wait_group 0;\n" ::);
      __syncthreads();
    }
    acc[0][0][0] = stage[threadIdx.x];
  } else if (p.mode == 4) {
    auto issue = [&](int s, int u) {
      int j0, a0, k0;
      unit_coords(p, u, j0, a0, k0);
      double* As = stage + s * kStage;
      double* Rs = As + kTM * kSS;
      for (int e = threadIdx.x; e < kTM * 16; e += kPT) {
        const int r = e / 16, kk = (e % 16) * 2;
        cp16(As + r * kSS + kk, p.a + (j0 + r) * p.ld + k0 + kk);
      }
      for (int e = threadIdx.x; e < kTN * 16; e += kPT) {
        const int c = e / 16, kk = (e % 16) * 2;
        cp16(Rs + c * kSS + kk, p.r + (a0 + c) * p.ld + k0 + kk);
      }
      asm volatile("cp.async.commit_group;\n" ::);
    };
    issue(0, 0);
    for (int u = 0; u < p.units; ++u) {
      asm volatile("cp.async.wait_group 0;\n" ::);
      __syncthreads();
      if (u + 1 < p.units) issue((u + 1) % 2, u + 1);
      mma_unit(stage + (u % 2) * kStage, acc);
    }
  } else {
    const bool do_x = p.mode != 3, do_y = p.mode != 2;
    auto issue = [&](int u, int st) {
      double* Xs = stage + st * kStage;
      uint64_t* full = &s_full[st];
      const int pw = p.mode == 5 ? w / 4 : 0;
      const bool tma_y = p.mode >= 6;
      const bool box_y = p.mode == 9 || p.mode == 14 || p.mode == 15;
      if (pw == 0 && l == 0) {
        const uint32_t xb = (do_x ? kTM * kSS * 8 : 0) + (tma_y ? (p.mode == 8 ? kTN * kTK * 8 : kTN * kSS * 8) : 0);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(full)), "r"(xb) : "memory");
        if (do_x) {
          int j0, a0, k0;
          unit_coords(p, u, j0, a0, k0);
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
              "[%4];" ::"r"(su32(Xs)),
              "l"(reinterpret_cast<uint64_t>(&p.tm)), "r"(k0), "r"(j0), "r"(su32(full))
              : "memory");
        }
      }
      if (tma_y) {
        int j0, a0, k0;
        unit_coords(p, u, j0, a0, k0);
        double* Ys = Xs + kTM * kSS;
        __syncwarp();
        if (box_y && l == 0) {
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
              "[%4];" ::"r"(su32(Ys)),
              "l"(reinterpret_cast<uint64_t>(&p.tmr64)), "r"(k0), "r"(a0), "r"(su32(full))
              : "memory");
        } else if (p.mode == 6 && l == 0) {
          for (int c = 0; c < kTN; ++c)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
                "[%4];" ::"r"(su32(Ys + c * kSS)),
                "l"(reinterpret_cast<uint64_t>(&p.tmr)), "r"(k0), "r"(sig_of(a0 + c)), "r"(su32(full))
                : "memory");
        } else if (p.mode == 7 && l == 0) {
          for (int c = 0; c < kTN; c += 4)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
                "%3, %4, %5, %6}], [%7];" ::"r"(su32(Ys + c * kSS)),
                "l"(reinterpret_cast<uint64_t>(&p.tmr)), "r"(k0), "r"(sig_of(a0 + c)), "r"(sig_of(a0 + c + 1)),
                "r"(sig_of(a0 + c + 2)), "r"(sig_of(a0 + c + 3)), "r"(su32(full))
                : "memory");
        } else if (p.mode == 8) {
          for (int c = l; c < kTN; c += 32)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             su32(Ys + c * kSS)),
                         "l"(p.r + sig_of(a0 + c) * p.ld + k0), "r"(kTK * 8), "r"(su32(full))
                         : "memory");
        }
      } else if (do_y) {
        issue_y(p, u, Xs + kTM * kSS, pw * 32, 32 * nprod, l);
      }
      if (p.mode != 15) asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(full)) : "memory");
    };
    const int ahead = p.mode == 14 ? kRing - 2 : kRing - 1;
    if (producer)
      for (int i = 0; i < ahead && i < p.units; ++i) issue(i, i % kRing);
    for (int u = 0; u < p.units; ++u) {
      if (producer && u + ahead < p.units) {
        const uint32_t qn = u + ahead;
        if (l == 0) mb_wait(&s_empty[qn % kRing], ((qn / kRing) & 1u) ^ 1u);
        __syncwarp();
        issue(qn, qn % kRing);
      }
      mb_wait(&s_full[u % kRing], (u / kRing) & 1u);
      if (p.ct == 2) mma_unit<2>(stage + (u % kRing) * kStage, acc);
      else mma_unit(stage + (u % kRing) * kStage, acc);
      __syncwarp();
      if (l == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&s_empty[u % kRing])) : "memory");
    }
  }
  if (p.validate && blockIdx.x == 0) {
    __syncthreads();
    const double* Ys = stage + ((p.units - 1) % (p.mode == 4 ? 2 : kRing)) * kStage + kTM * kSS;
    for (int i = threadIdx.x; i < kTN * kTK; i += kPT) p.out[i] = Ys[(i / kTK) * kSS + i % kTK];
    return;
  }
  double s = 0;
  for (int h = 0; h < kRT; ++h)
    for (int c = 0; c < kCT; ++c) s += acc[h][c][0] + acc[h][c][1];
  if (s == 123.456) p.out[threadIdx.x] = s;
}

// mode 13: warp 16 only issues (TMA A + TMA box of 64 R columns), warps 0-15 only compute
__global__ void __launch_bounds__(kPT + 32, 1) bench_kernel_ws(const __grid_constant__ Args p) {
  extern __shared__ __align__(128) double dsm[];
  double* stage = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(dsm) + 127) & ~uintptr_t(127));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kRing; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&s_full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&s_empty[s])), "r"(kPW));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (w == kPW) {  // producer
    if (l == 0) {
      for (int u = 0; u < p.units; ++u) {
        const int st = u % kRing;
        mb_wait(&s_empty[st], ((u / kRing) & 1u) ^ 1u);
        int j0, a0, k0;
        unit_coords(p, u, j0, a0, k0);
        double* Xs = stage + st * kStage;
        uint64_t* full = &s_full[st];
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(full)),
                     "r"(kTM * kSS * 8 + kTN * kSS * 8)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
            "[%4];" ::"r"(su32(Xs)),
            "l"(reinterpret_cast<uint64_t>(&p.tm)), "r"(k0), "r"(j0), "r"(su32(full))
            : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
            "[%4];" ::"r"(su32(Xs + kTM * kSS)),
            "l"(reinterpret_cast<uint64_t>(&p.tmr64)), "r"(k0), "r"(a0), "r"(su32(full))
            : "memory");
      }
    }
    return;
  }
  double acc[kRT][kCT][2] = {};
  for (int u = 0; u < p.units; ++u) {
    mb_wait(&s_full[u % kRing], (u / kRing) & 1u);
    if (p.ct == 2) mma_unit<2>(stage + (u % kRing) * kStage, acc);
    else mma_unit(stage + (u % kRing) * kStage, acc);
    __syncwarp();
    if (l == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&s_empty[u % kRing])) : "memory");
  }
  double s = 0;
  for (int h = 0; h < kRT; ++h)
    for (int c = 0; c < kCT; ++c) s += acc[h][c][0] + acc[h][c][1];
  if (s == 123.456) p.out[threadIdx.x] = s;
}

int main() {
  const int64_t ld = 1024, k = 4096, b = 512;
  double *a, *r, *out;
  cudaMalloc(&a, ld * k * 8);
  cudaMalloc(&r, ld * b * 8);
  cudaMalloc(&out, 4096 * 8);
  std::vector<double> hr(ld * b);
  std::vector<double> h(ld * k);
  for (size_t i = 0; i < h.size(); ++i) h[i] = 1e-3 * (i % 1013);
  cudaMemcpy(a, h.data(), ld * k * 8, cudaMemcpyHostToDevice);
  for (size_t i = 0; i < hr.size(); ++i) hr[i] = 1e-3 * ((i * 7) % 1009) + 1.0;
  cudaMemcpy(r, hr.data(), ld * b * 8, cudaMemcpyHostToDevice);
  using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q{};
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  Args p{};
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(ld), static_cast<cuuint64_t>(k)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 8)};
  const cuuint32_t box[2] = {36, 128}, es[2] = {1, 1};
  CUresult cr = reinterpret_cast<Encode>(f)(&p.tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, a, dims, strides, box, es,
                                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) {
    printf("encode failed %d\n", cr);
    return 1;
  }
  {
    const cuuint64_t rd[2] = {static_cast<cuuint64_t>(ld), static_cast<cuuint64_t>(b)};
    const cuuint32_t rbox[2] = {36, 1};
    cr = reinterpret_cast<Encode>(f)(&p.tmr, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, r, rd, strides, rbox, es,
                                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) printf("encode R failed %d\n", cr);
    const cuuint32_t wbox[2] = {132, 32};
    cr = reinterpret_cast<Encode>(f)(&p.tmw, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, a, dims, strides, wbox, es,
                                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const cuuint32_t rbox64[2] = {36, 64};
    cr = reinterpret_cast<Encode>(f)(&p.tmr64, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, r, rd, strides, rbox64, es,
                                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  p.a = a;
  p.r = r;
  p.ld = ld;
  p.k = k;
  p.b = b;
  p.out = out;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = kRing * kStage * 8 + 128;
  cudaFuncSetAttribute(bench_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  cudaFuncSetAttribute(bench_kernel_ws, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[] = {"compute only", "TMA A + warp-0 cp.async R (3-stage ring)", "TMA A only",
                         "warp-0 cp.async R only", "all-thread cp.async, 2 stages + CTA barrier",
                         "TMA A + 4 producer warps for R", "TMA A + per-column 2D TMA R", "TMA A + gather4 R",
                         "TMA A + per-column 1D bulk R", "TMA A + 2D TMA box of 64 R columns",
                         "latency: Corr A box alone", "latency: W A box alone", "latency: A tile by cp.async",
                         "as 9, dedicated producer warp", "as 9, lookahead kRing - 2", "as 9, thread 0 alone"};
  // mode 6 is listed for the record: a tile-mode tensor copy needs a 128-byte aligned
  // destination, which a 288-byte padded column stride cannot give (misaligned address)
  for (int stg = 0; stg < 1; ++stg)
  for (int mode : {0, 9, 13, 14, 15, 109, 113, 114, 115, 1, 2, 3, 4, 5, 8, 7, 10, 11, 12}) {
    p.ct = mode >= 100 ? 2 : 4;
    if (mode >= 100) mode -= 100;
    p.stagger = stg;
    p.mode = mode;
    p.units = 448;
    if (mode == 13) bench_kernel_ws<<<sms, kPT + 32, smem>>>(p);
    else bench_kernel<<<sms, kPT, smem>>>(p);
    cudaEventRecord(e0);
    if (mode == 13) bench_kernel_ws<<<sms, kPT + 32, smem>>>(p);
    else bench_kernel<<<sms, kPT, smem>>>(p);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const cudaError_t err = cudaGetLastError();
    const double flops = double(sms) * p.units * 2.0 * kTM * (kTN * p.ct / 4) * kTK;
    // validation: CTA 0's last unit's R tile against the host gather
    double bad = -1;
    if (mode >= 1 && mode != 2 && mode < 10) {  // (mode 13 loads what mode 9 loads)
      p.validate = 1;
      bench_kernel<<<sms, kPT, smem>>>(p);
      std::vector<double> got(kTN * kTK);
      cudaMemcpy(got.data(), out, kTN * kTK * 8, cudaMemcpyDeviceToHost);
      const int u = p.units - 1, tile = (0 * 7 + u / 32) % 256, a0 = (tile / 32) * kTN, k0 = (u % 32) * kTK;  // CTA 0
      bad = 0;
      for (int c = 0; c < kTN; ++c)
        for (int d = 0; d < kTK; ++d) {
          const double e = hr[(mode == 9 ? a0 + c : (37 * (a0 + c)) % 512) * ld + k0 + d];
          bad = std::max(bad, std::abs(e - got[c * kTK + d]));
        }
      p.validate = 0;
    }
    printf("ct %d mode %d %-45s %7.3f us/unit  %6.2f TFLOP/s  %s  max|R tile err| %g\n", p.ct, mode, names[mode],
           ms * 1e3 / p.units, flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()), bad);
  }
  return 0;
}
