// Lockstep batched engine (BASELINE configs[4]: many signals, one dictionary).
//
// B independent run_lasso calls share one dense exact dictionary. Every global
// step, each unfinished signal performs its own next unit of Engine::run
// (fastl1.cpp:459-645): one FISTA iteration, or one step of its restricted power
// iteration (solver.cpp:72-104). The dictionary products of all signals are then
// two dense contractions on the fp64 tensor cores (DMMA m8n8k4 over shared-memory
// tiles; by default stream-K over a TMA / mbarrier ring, `sk_contract`; the earlier
// split-K cp.async double buffer stays behind FL1_LOCKSTEP_TMA=0):
//     W    = A  V            for the signals in a power step   (N x K times K x P)
//     Corr = A^T [rho | w]   for every signal                  (K x N times N x B)
// reading each A tile once per 64 signals instead of once per signal. Preserved
// sets are per-signal masks over the atoms (the reference's compacted order is
// ascending atom order, so positions = ranks among unmasked atoms); a masked atom
// has x = x_prev = lead = 0 and its Corr row is ignored. The per-signal rest of an
// iteration (dual scaling, gaps, stop and screening tests, prox, FISTA
// bookkeeping, restriction with the v fix, sparse apply u = A x, ledger, trace)
// runs in one CTA per signal. A signal finishes here; only the exact-fit branch
// (rho_g == 0, fastl1.cpp:428-449) is handed to the per-signal engine (engine.cu).
// Every reduction has a fixed order, so results are reproducible run to run.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <math_constants.h>

#include <algorithm>
#include <cfloat>
#include <cstdint>

#include "engine.cuh"

namespace cg = cooperative_groups;

namespace fl1 {
cudaError_t gemm_tn_launch(const double* X, int64_t ldx, int64_t nx, const double* Y, int64_t ldy, int64_t ny,
                           int64_t kdim, double* C, int64_t ldc, double* work, size_t work_elems, int device,
                           cudaStream_t stream);
namespace {

#ifndef FL1_PREFIX_THREADS
#define FL1_PREFIX_THREADS 512
#endif
constexpr int kPT = FL1_PREFIX_THREADS;  // threads per CTA
constexpr int kPW = kPT / 32;
constexpr int kIt = 9;  // atoms per lane of a warp range: K <= prefix_max_atoms() = 4608 -> 288 per warp
#ifndef FL1_ITB
#define FL1_ITB 3
#endif
constexpr int kItB = FL1_ITB;  // atoms per lane loaded together in the prox pass
constexpr int kTM = 128, kTN = 64;  // output tile: 128 rows (atoms / samples) x 64 signals
// warp grid over a 128 x 64 output tile: kWR x kWC warps, each kRT x kCT 8x8 DMMA tiles
constexpr int kWR = 8, kWC = (kPT / 32) / kWR;
constexpr int kRT = kTM / 8 / kWR, kCT = kTN / 8 / kWC;
constexpr int kTK = 32;             // K chunk (rows of A / rho)
constexpr int kSS = kTK + 4;        // padded smem row stride (doubles)
constexpr int kStage = (kTM + kTN) * kSS;  // doubles per pipeline stage
#ifndef FL1_PREFIX_STAGES
#define FL1_PREFIX_STAGES 2
#endif
constexpr int kStages = FL1_PREFIX_STAGES;  // cp.async pipeline depth (3 measured no faster)
constexpr unsigned kAll = 0xffffffffu;
constexpr int kSplitMax = 16;      // split-K parts of the contractions (load balance)

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp16(double* dst, const double* src, bool valid) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  const int n = valid ? 16 : 0;  // zero-fill out of range
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(n));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }
__device__ __forceinline__ void cp_wait_pipe() { asm volatile("cp.async.wait_group %0;\n" ::"n"(kStages - 2)); }
__device__ __forceinline__ void cp_wait0() { asm volatile("cp.async.wait_group 0;\n" ::); }

#ifdef FL1_SIGPROF  // diagnostics build: per-phase time of CTA 0's per-signal FISTA steps
#define SIGPROF(k)                                                            \
  do {                                                                        \
    if (p.sigprof && blockIdx.x == 0 && threadIdx.x == 0) {                   \
      const double t_ = gtimer();                                             \
      p.sigprof[k] += t_ - p.sigprof[15];                                     \
      p.sigprof[15] = t_;                                                     \
    }                                                                         \
  } while (0)
#else
#define SIGPROF(k) \
  do {             \
  } while (0)
#endif
__device__ __forceinline__ double gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return static_cast<double>(t);
}

struct PSh {
  double red[kPW * 4];
  double res[4];
  int32_t wcnt[kPW];
  // per-signal step decisions (thread 0 -> block)
  double m, t_next, sp, radius, gap_tilde, primal;
  int release, screen;
  int64_t n_act, off;
  int32_t nzc[kPW], fxc[kPW];
  int32_t qnext;
};

// deterministic block reductions (fixed tree)
__device__ double block_sum(double v, PSh& sh) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(kAll, v, o);
  if (l == 0) sh.red[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kPW; ++i) t += sh.red[i];
    sh.res[0] = t;
  }
  __syncthreads();
  t = sh.res[0];
  __syncthreads();
  return t;
}
__device__ double block_max(double v, PSh& sh) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(kAll, v, o));
  if (l == 0) sh.red[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kPW; ++i) t = fmax(t, sh.red[i]);
    sh.res[0] = t;
  }
  __syncthreads();
  t = sh.res[0];
  __syncthreads();
  return t;
}
// block sum of three values
__device__ void block_sum3(double (&v)[3], PSh& sh) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < 3; ++j) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[j] += __shfl_down_sync(kAll, v[j], o);
    if (l == 0) sh.red[w * 4 + j] = v[j];
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double t = 0.0;
    for (int i = 0; i < kPW; ++i) t += sh.red[i * 4 + threadIdx.x];
    sh.res[threadIdx.x] = t;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 3; ++j) v[j] = sh.res[j];
  __syncthreads();
}

// Corr tile (atoms j0..j0+127) x (slots a0..a0+TN-1), TN = 8 kWC CT, over K-part kp of
// sk (rows of A / rho), DMMA, into the split-K partial buffer kp. CT (column 8x8 tiles
// per warp) is 4 for full 64-signal tiles and 2 / 1 for narrow steps (<= 32 / 16
// signals), so every warp's DMMA work shrinks with the width instead of computing
// empty columns (the slowest warp sets the tile's time).
template <int CT>
__device__ __noinline__ void gemm_tile(const PrefixParams& p, int rt, int64_t a0, int kp, int sk, int64_t n_act,
                                       const int32_t* act, double* stage) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, g = l >> 2, tg = l & 3;
  const int64_t j0 = static_cast<int64_t>(rt) * kTM;
  const int64_t K = p.k, ld = p.ld;
  const int nch = static_cast<int>((ld + kTK - 1) / kTK);
  const int c_lo = nch * kp / sk, c_hi = nch * (kp + 1) / sk;
  const int wr = w % kWR, wc = w / kWR;
  double acc[kRT][CT][2];
#pragma unroll
  for (int h = 0; h < kRT; ++h)
#pragma unroll
    for (int c = 0; c < CT; ++c) acc[h][c][0] = acc[h][c][1] = 0.0;
  auto issue = [&](int s, int kc) {
    double* As = stage + s * kStage;
    double* Rs = As + kTM * kSS;
    const int64_t k0 = static_cast<int64_t>(kc) * kTK;
#pragma unroll
    for (int e0 = 0; e0 < kTM * (kTK / 2); e0 += kPT) {  // 16-byte copies, A rows (atoms)
      const int e = e0 + threadIdx.x;
      const int r = e / (kTK / 2), kk = (e % (kTK / 2)) * 2;
      const int64_t j = j0 + r, kg = k0 + kk;
      const bool ok = j < K && kg < ld;
      cp16(As + r * kSS + kk, ok ? p.a + j * ld + kg : p.a, ok);
    }
#pragma unroll
    for (int e0 = 0; e0 < 8 * kWC * CT * (kTK / 2); e0 += kPT) {  // R columns (slots)
      const int e = e0 + threadIdx.x;
      const int c = e / (kTK / 2), kk = (e % (kTK / 2)) * 2;
      const int64_t a = a0 + c, kg = k0 + kk;
      const bool ok = a < n_act && kg < ld;
      const int64_t b = ok ? act[a] : 0;  // R columns are per signal
      cp16(Rs + c * kSS + kk, ok ? p.R + b * ld + kg : p.R, ok);
    }
  };
  for (int st = 0; st < kStages - 1; ++st) {
    if (c_lo + st < c_hi) issue(st, c_lo + st);
    cp_commit();
  }
  for (int kc = c_lo; kc < c_hi; ++kc) {
    cp_wait_pipe();
    __syncthreads();  // chunk kc landed; every thread is done with chunk kc-1's stage
    if (kc + kStages - 1 < c_hi) issue((kc + kStages - 1 - c_lo) % kStages, kc + kStages - 1);
    cp_commit();
    const double* As = stage + ((kc - c_lo) % kStages) * kStage;
    const double* Rs = As + kTM * kSS;
#pragma unroll
    for (int ks = 0; ks < kTK / 4; ++ks) {
      double av[kRT], bv[CT];
#pragma unroll
      for (int h = 0; h < kRT; ++h) av[h] = As[((h * kWR + wr) * 8 + g) * kSS + ks * 4 + tg];
#pragma unroll
      for (int c = 0; c < CT; ++c) bv[c] = Rs[((wc * CT + c) * 8 + g) * kSS + ks * 4 + tg];
#pragma unroll
      for (int h = 0; h < kRT; ++h)
#pragma unroll
        for (int c = 0; c < CT; ++c) dmma(acc[h][c], av[h], bv[c]);
    }
  }
  cp_wait0();
  __syncthreads();  // the staging area is reused by the next tile / the per-signal steps
  double* __restrict__ out = p.corr + static_cast<int64_t>(kp) * K * p.bcap;
#pragma unroll
  for (int h = 0; h < kRT; ++h) {
    const int64_t j = j0 + (h * kWR + wr) * 8 + g;
#pragma unroll
    for (int c = 0; c < CT; ++c) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int64_t a = a0 + (wc * CT + c) * 8 + 2 * tg + i;
        if (j < K && a < n_act) __stcg(out + a * K + j, acc[h][c][i]);
      }
    }
  }
}

// column 8x8 tiles per warp for a column tile holding n (of up to 64) columns: the
// narrowest of 16 / 32 / 48 / 64 that holds them when width tiles are on
// (FL1_LOCKSTEP_WIDTH), else the full 64-column tile
__device__ __forceinline__ int tile_ct(int n, int width_tiles) {
  if (!width_tiles) return kCT;
  return n <= 8 * kWC ? 1 : (n <= 16 * kWC ? 2 : (n <= 24 * kWC ? 3 : kCT));
}

// split-K factor for T output tiles of nch K-chunks on G CTAs: the fewest-waves choice,
// cost ceil(T s / G) / s (tile waves in units of a whole tile) plus ~2% per extra part
// (partial write + read, per-item prologue), each part at least 4 chunks deep
__device__ __forceinline__ int split_for(int T, int G, int nch, int smax = kSplitMax) {
  int best = 1;
  float best_cost = static_cast<float>((T + G - 1) / G) * 1.02f;
  for (int s = 2; s <= smax && s <= kSplitMax && nch / s >= 4; ++s) {
    const float cost = static_cast<float>((T * s + G - 1) / G) / static_cast<float>(s) * (1.0f + 0.02f * s);
    if (cost < best_cost) {
      best = s;
      best_cost = cost;
    }
  }
  return best;
}

// split parts allowed by the partial-buffer budget (FL1_SPLIT_BUDGET_MB: partials that
// stay L2-resident instead of round-tripping DRAM); out = output elements of the product
__device__ __forceinline__ int split_cap(const PrefixParams& p, int64_t out) {
  if (p.split_budget <= 0 || out <= 0) return kSplitMax;
  const int64_t c = p.split_budget / (out * 8);
  return static_cast<int>(c < 1 ? 1 : (c > kSplitMax ? kSplitMax : c));
}

__device__ __forceinline__ int split_old(int T, int G) {
  int s = 1;
  while (s < kSplitMax && 3 * T * s < 2 * G) s *= 2;
  return s;
}

// ---------------------------------------------------------------------------
// W = A V tile: rows i0..i0+63 of ld, power slots c0..c0+63 (index into pact),
// atoms of K-part kp of sk; partial into np[kp][pslot][ld].
template <int CT>
__device__ __noinline__ void gemm_n_tile(const PrefixParams& p, int rt, int64_t c0, int kp, int sk, int n_pow,
                                         const int32_t* pact, const int32_t* act, double* stage) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, g = l >> 2, tg = l & 3;
  const int64_t i0 = static_cast<int64_t>(rt) * kTM;
  const int64_t K = p.k, ld = p.ld;
  constexpr int kAS = kTM + 4;  // As[kk][i] row stride
  const int nch = static_cast<int>((K + kTK - 1) / kTK);
  const int c_lo = nch * kp / sk, c_hi = nch * (kp + 1) / sk;
  const int wr = w % kWR, wc = w / kWR;
  double acc[kRT][CT][2];
#pragma unroll
  for (int h = 0; h < kRT; ++h)
#pragma unroll
    for (int c = 0; c < CT; ++c) acc[h][c][0] = acc[h][c][1] = 0.0;
  auto issue = [&](int s, int kc) {
    double* As = stage + s * kStage;
    double* Bs = As + kTK * kAS;
    const int64_t k0 = static_cast<int64_t>(kc) * kTK;
#pragma unroll
    for (int e0 = 0; e0 < kTK * (kTM / 2); e0 += kPT) {  // A(i, k): k-major, i contiguous
      const int e = e0 + threadIdx.x;
      const int kk = e / (kTM / 2), ii = (e % (kTM / 2)) * 2;
      const int64_t kg = k0 + kk, ig = i0 + ii;
      const bool ok = kg < K && ig < ld;
      cp16(As + kk * kAS + ii, ok ? p.a + kg * ld + ig : p.a, ok);
    }
#pragma unroll
    for (int e0 = 0; e0 < 8 * kWC * CT * (kTK / 2); e0 += kPT) {  // V(k, slot): slot-major, k contiguous
      const int e = e0 + threadIdx.x;
      const int c = e / (kTK / 2), kk = (e % (kTK / 2)) * 2;
      const int64_t pc = c0 + c, kg = k0 + kk;
      const bool ok = pc < n_pow && kg < K;
      const int64_t b = ok ? act[pact[pc]] : 0;
      cp16(Bs + c * kSS + kk, ok ? p.vp + b * K + kg : p.vp, ok);
    }
  };
  for (int st = 0; st < kStages - 1; ++st) {
    if (c_lo + st < c_hi) issue(st, c_lo + st);
    cp_commit();
  }
  for (int kc = c_lo; kc < c_hi; ++kc) {
    cp_wait_pipe();
    __syncthreads();
    if (kc + kStages - 1 < c_hi) issue((kc + kStages - 1 - c_lo) % kStages, kc + kStages - 1);
    cp_commit();
    const double* As = stage + ((kc - c_lo) % kStages) * kStage;
    const double* Bs = As + kTK * kAS;
#pragma unroll
    for (int ks = 0; ks < kTK / 4; ++ks) {
      double av[kRT], bv[CT];
#pragma unroll
      for (int h = 0; h < kRT; ++h) av[h] = As[(ks * 4 + tg) * kAS + (h * kWR + wr) * 8 + g];
#pragma unroll
      for (int c = 0; c < CT; ++c) bv[c] = Bs[((wc * CT + c) * 8 + g) * kSS + ks * 4 + tg];
#pragma unroll
      for (int h = 0; h < kRT; ++h)
#pragma unroll
        for (int c = 0; c < CT; ++c) dmma(acc[h][c], av[h], bv[c]);
    }
  }
  cp_wait0();
  __syncthreads();
#pragma unroll
  for (int h = 0; h < kRT; ++h) {
    const int64_t i = i0 + (h * kWR + wr) * 8 + g;
#pragma unroll
    for (int c = 0; c < CT; ++c) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int64_t pc = c0 + (wc * CT + c) * 8 + 2 * tg + q;
        if (i < ld && pc < n_pow) __stcg(p.np + (static_cast<int64_t>(kp) * p.bcap + pc) * ld + i, acc[h][c][q]);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Stream-K contractions on a TMA / mbarrier ring (FL1_LOCKSTEP_TMA, default).
//
// One product (Corr = A^T R or W = A V) is a list of (tile, 32-deep chunk) units,
// tiles in (column tile, row tile) order; a unit costs its tile's DMMA width CT, and
// CTA g takes the contiguous unit range covering costs [W g / G, W (g+1) / G). A tile
// the range covers whole is written from registers; a range shares at most two tiles
// with other CTAs (its first and its last), whose segment partials go to the CTA's two
// slots of p.part, flagged with the product's epoch. Each shared tile is then reduced
// by its own contributors, every one a slice of the elements, adding the partials in
// chunk (= CTA) order -- a narrow W tile spans ~20 CTAs, so a single reducer would
// chain ~20 L2 round trips. Corr goes to p.corr (one part: no split-K sum in the
// per-signal steps), W straight into the power slots' Rc columns (no combine pass and
// grid barrier). The reduction order is fixed by (tile count, grid), so results are
// reproducible run to run.
//
// Loads: thread 0 keeps kRing - 1 units ahead of the CTA's consumption. Per unit it arms
// the stage's full barrier with the unit's bytes and issues two 2D tensor copies: the A
// tile and the 64 slot-ordered R / V columns (p.rc / p.vc, staged in slot order at the
// start of the step: gathering the columns by signal instead -- per-thread cp.async,
// bulk copies or tile::gather4 -- measured 1.2-1.9x slower per unit, tools/sk_bench.cu).
// The boxes over-fetch rows / atoms so that each dense box lands in the padded,
// bank-conflict-free layout the DMMA fragments read (Corr [atom][36], W [atom][132],
// R / V [slot][36]). Every warp releases a stage through its empty barrier: no CTA-wide
// barrier per chunk, and the ring runs on across tile boundaries.
constexpr int kRing = 3;
constexpr int kLogW = 10;  // step-log fields per step (FL1_STEP_LOG diagnostics)
constexpr int kPartTile = kTM * kTN;  // doubles per partial slot (two per CTA)
constexpr int kStageBufs = kStages > kRing ? kStages : kRing;  // staging area, in kStage units
__shared__ __align__(8) uint64_t s_full[kRing];
__shared__ __align__(8) uint64_t s_empty[kRing];
constexpr int kMaxGrid = 256;             // stream-K route: CTAs (one per SM) at most
__shared__ int32_t s_contrib[2 * kMaxGrid];  // the shared tiles' contributor slots, chunk order
__shared__ int32_t sh_scal[2];
__shared__ int64_t s_begin[kMaxGrid + 1];  // the product's unit-range starts of every CTA

__device__ __forceinline__ uint32_t su32(const void* ptr) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(ptr));
}
__device__ __forceinline__ void mb_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(su32(bar)), "r"(parity)
        : "memory");
  }
}
__device__ void sk_init_barriers() {
  if (threadIdx.x == 0) {
    for (int s = 0; s < kRing; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&s_full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&s_empty[s])), "r"(kPW));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
}

struct SkShape {
  int which;       // 0: W = A V (rows of ld, depth K), 1: Corr = A^T R (atoms, depth ld)
  int64_t M, D;    // output rows, contraction depth
  int nch, n_rt, n_ct, ct_last;
  int64_t n_cols;  // output columns (signals)
  int64_t F, W;    // cost of the full-width column tiles; total cost
  __device__ SkShape(const PrefixParams& p, int wh, int64_t ncols) {
    which = wh;
    M = wh ? p.k : p.ld;
    D = wh ? p.ld : p.k;
    nch = static_cast<int>((D + kTK - 1) / kTK);
    n_rt = static_cast<int>((M + kTM - 1) / kTM);
    n_cols = ncols;
    n_ct = static_cast<int>((ncols + kTN - 1) / kTN);
    ct_last = tile_ct(static_cast<int>(ncols - static_cast<int64_t>(n_ct - 1) * kTN), p.width_tiles);
    F = static_cast<int64_t>(n_ct - 1) * n_rt * nch * kCT;
    W = F + static_cast<int64_t>(n_rt) * nch * ct_last;
  }
  // first unit whose starting cost is >= c
  __device__ int64_t pos(int64_t c) const {
    if (c <= F) return (c + kCT - 1) / kCT;
    return F / kCT + (c - F + ct_last - 1) / ct_last;
  }
  __device__ int64_t begin(int g, int G) const { return pos(W * g / G); }
  __device__ int ct_of(int64_t tile) const { return tile / n_rt == n_ct - 1 ? ct_last : kCT; }
};

// issue unit u's loads into stage st (one thread): a 2D tensor copy of the A tile and one
// of the 64 slot-ordered R / V columns, both on the stage's full barrier
// The issue cursor: unit -> (row tile, column offset, chunk) advanced incrementally (the
// issuing thread is a DMMA warp's lane: 64-bit divisions per unit cost ~10% of the unit)
struct SkCursor {
  int kc, rt, c0;
  __device__ SkCursor(const SkShape& sh, int64_t u) {
    const int64_t tile = u / sh.nch;
    kc = static_cast<int>(u - tile * sh.nch);
    rt = static_cast<int>(tile % sh.n_rt);
    c0 = static_cast<int>((tile / sh.n_rt) * kTN);
  }
  __device__ __forceinline__ void advance(const SkShape& sh) {
    if (++kc == sh.nch) {
      kc = 0;
      if (++rt == sh.n_rt) {
        rt = 0;
        c0 += kTN;
      }
    }
  }
};

__device__ __forceinline__ void sk_issue(const PrefixParams& p, const SkShape& sh, const SkCursor& cu, int st,
                                         double* stage) {
  const int rt = cu.rt, c0 = cu.c0;
  const int d0 = cu.kc * kTK;
  double* Xs = stage + st * kStage;
  const uint32_t xbytes = sh.which ? kTM * kSS * 8 : kTK * (kTM + 4) * 8;
  double* Ys = Xs + (sh.which ? kTM * kSS : kTK * (kTM + 4));
  uint64_t* full = &s_full[st];
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(full)),
               "r"(xbytes + static_cast<uint32_t>(kTN * kSS * 8))
               : "memory");
  const int x_in = sh.which ? d0 : rt * kTM;    // coordinate along ld
  const int x_out = sh.which ? rt * kTM : d0;  // coordinate along the atoms
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(su32(Xs)),
      "l"(reinterpret_cast<uint64_t>(sh.which ? &p.tm_corr : &p.tm_w)), "r"(x_in), "r"(x_out), "r"(su32(full))
      : "memory");
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(su32(Ys)),
      "l"(reinterpret_cast<uint64_t>(sh.which ? &p.tm_rc : &p.tm_vc)), "r"(d0), "r"(c0), "r"(su32(full))
      : "memory");
}

// DMMA over one landed unit (layouts as sk_issue)
__device__ __forceinline__ double lds64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
// (the operands are read through 32-bit shared-window addresses: from the staging pointer
// the compiler would emit generic loads, measurably slower than LDS in the DMMA loop)
template <int WHICH, int CT>
__device__ __forceinline__ void sk_mma(const double* Xs, double (&acc)[kRT][kCT][2]) {
  constexpr int which = WHICH;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, g = l >> 2, tg = l & 3;
  const int wr = w % kWR, wc = w / kWR;
  const uint32_t xa = su32(Xs) +
                      8u * static_cast<uint32_t>(which ? (wr * 8 + g) * kSS + tg : tg * (kTM + 4) + wr * 8 + g);
  const uint32_t ya = su32(Xs) + 8u * static_cast<uint32_t>((which ? kTM * kSS : kTK * (kTM + 4)) +
                                                            (wc * CT * 8 + g) * kSS + tg);
#pragma unroll
  for (int ks = 0; ks < kTK / 4; ++ks) {
    double av[kRT], bv[CT];
#pragma unroll
    for (int h = 0; h < kRT; ++h)
      av[h] = lds64(xa + 8u * (which ? h * kWR * 8 * kSS + ks * 4 : ks * 4 * (kTM + 4) + h * kWR * 8));
#pragma unroll
    for (int c = 0; c < CT; ++c) bv[c] = lds64(ya + 8u * (c * 8 * kSS + ks * 4));
#pragma unroll
    for (int h = 0; h < kRT; ++h)
#pragma unroll
      for (int c = 0; c < CT; ++c) dmma(acc[h][c], av[h], bv[c]);
  }
}

// the CTAs whose ranges hold units of the tile [ta, tb): gA .. gB (consecutive), n_ne of
// them non-empty, j of those before this CTA (s_begin of the current product)
struct SkContrib {
  int gA, gB, n_ne, j;
};
__device__ __forceinline__ SkContrib sk_contrib(int64_t ta, int64_t tb, int gi, int G) {
  SkContrib t{gi, gi, 0, 0};
  while (s_begin[t.gA] > ta) --t.gA;  // the range holding the tile's first unit
  while (t.gA + 1 < G && s_begin[t.gA + 1] <= ta) ++t.gA;
  while (t.gB + 1 < G && s_begin[t.gB + 1] < tb) ++t.gB;  // ... and its last unit
  for (int g2 = t.gA; g2 <= t.gB; ++g2)
    if (s_begin[g2 + 1] > s_begin[g2]) {
      if (g2 < gi) ++t.j;
      ++t.n_ne;
    }
  return t;
}

// output element (h, c, e) of thread tid's fragments of `tile`: Corr into p.corr (slot
// columns), W into the power slots' Rc columns (zero past row n)
__device__ __forceinline__ void sk_store(const PrefixParams& p, const SkShape& sh, const int32_t* pact, int64_t tile,
                                         int CT, int h, int c, int e, int tid, double v) {
  const int w = tid >> 5, l = tid & 31;
  const int64_t r = (tile % sh.n_rt) * kTM + (h * kWR + w % kWR) * 8 + (l >> 2);
  const int64_t col = (tile / sh.n_rt) * kTN + ((w / kWR) * CT + c) * 8 + 2 * (l & 3) + e;
  if (r >= sh.M || col >= sh.n_cols) return;
  if (sh.which) __stcg(p.corr + col * p.k + r, v);
  else __stcg(p.rc + static_cast<int64_t>(pact[col]) * p.ld + r, r < p.n ? v : 0.0);
}

// The units [ub, ue) of one segment (a single tile: DMMA width CT): thread 0 refills the
// stage released at the previous unit, every warp waits for its unit's stage, computes and
// releases it. utr (diagnostics): per unit, the times around the full-barrier wait.
template <int WHICH, int CT>
__device__ __forceinline__ void sk_units(const PrefixParams& p, const SkShape& sh, double* stage, SkCursor& cur,
                                         uint32_t ring, int64_t u0, int64_t nu, int64_t ub, int64_t ue,
                                         double (&acc)[kRT][kCT][2], double* utr) {
  const int l = threadIdx.x & 31;
  for (int64_t u = ub; u < ue; ++u) {
    const int64_t i = u - u0;
    if (threadIdx.x == 0 && i + kRing - 1 < nu) {  // refill the stage released at unit i - 1
      const uint32_t qn = ring + static_cast<uint32_t>(i + kRing - 1);
      mb_wait(&s_empty[qn % kRing], ((qn / kRing) & 1u) ^ 1u);
      sk_issue(p, sh, cur, static_cast<int>(qn % kRing), stage);
      cur.advance(sh);
    }
    const uint32_t q = ring + static_cast<uint32_t>(i);
    if (utr && i < 128) utr[2 * i] = gtimer();
    mb_wait(&s_full[q % kRing], (q / kRing) & 1u);
    if (utr && i < 128) utr[2 * i + 1] = gtimer();
    sk_mma<WHICH, CT>(stage + (q % kRing) * kStage, acc);
    __syncwarp();
    if (l == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&s_empty[q % kRing])) : "memory");
  }
}

// Stage the step's contraction inputs in slot order: Rc[a] = R[act[a]] and Vc[c] = the
// power vector of power slot c (32-bit index arithmetic: one pass is far below 2^31
// elements; four elements per thread and round, their loads in flight together; out of
// line, so that its registers do not weigh on the kernel body's allocation).
__device__ __noinline__ void sk_stage(const PrefixParams& p, int n_act, int n_pow, const int32_t* act,
                                      const int32_t* pact) {
  const int64_t ld = p.ld, K = p.k;
  const uint32_t hl = static_cast<uint32_t>(ld / 2), hk = static_cast<uint32_t>(K / 2);
  const uint32_t nr = static_cast<uint32_t>(n_act) * hl, nv = static_cast<uint32_t>(n_pow) * hk;
  const uint32_t stride = gridDim.x * kPT;
  for (uint32_t e0 = blockIdx.x * kPT + threadIdx.x; e0 < nr + nv; e0 += 4 * stride) {
    double2 v[4];
    double2* d[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t e = e0 + q * stride;
      d[q] = nullptr;
      if (e >= nr + nv) continue;
      if (e < nr) {
        const uint32_t a = e / hl, i = e - a * hl;
        d[q] = reinterpret_cast<double2*>(p.rc + static_cast<int64_t>(a) * ld) + i;
        v[q] = __ldcg(reinterpret_cast<const double2*>(p.R + static_cast<int64_t>(act[a]) * ld) + i);
      } else {
        const uint32_t f = e - nr, c = f / hk, j = f - c * hk;
        d[q] = reinterpret_cast<double2*>(p.vc + static_cast<int64_t>(c) * K) + j;
        v[q] = __ldcg(reinterpret_cast<const double2*>(p.vp + static_cast<int64_t>(act[pact[c]]) * K) + j);
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (d[q]) __stcg(d[q], v[q]);
  }
}

// One stream-K product over this CTA's unit range. ring: the CTA's running unit count
// (stage and phase of the ring; identical in every thread). epoch: unique per product
// within the launch (the flags are zeroed at the launch's start).
__device__ __noinline__ void sk_contract(const PrefixParams& p, int which, int64_t ncols, const int32_t* pact,
                                         double* stage, uint32_t& ring, int32_t epoch) {
  const SkShape sh(p, which, ncols);
  const int G = gridDim.x, gi = blockIdx.x;
  for (int g2 = threadIdx.x; g2 <= G; g2 += kPT) s_begin[g2] = sh.begin(g2, G);
  // the per-signal phases' generic-proxy writes into the staging area precede the
  // async-proxy copies below
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const int64_t u0 = s_begin[gi], u1 = s_begin[gi + 1];
  double* trc = (p.sk_trace && (epoch - 1 - which) / 2 == p.sk_trace_step && threadIdx.x == 0)
                    ? p.sk_trace + (which * kMaxGrid + gi) * 4 : nullptr;
  if (trc) trc[0] = gtimer();
  if (u0 >= u1) return;
  const int64_t nu = u1 - u0;
  SkCursor cur(sh, u0);  // next unit to issue (thread 0)
  if (threadIdx.x == 0)
    for (int64_t i = 0; i < kRing - 1 && i < nu; ++i) {
      sk_issue(p, sh, cur, static_cast<int>((ring + i) % kRing), stage);
      cur.advance(sh);
    }
  double acc[kRT][kCT][2];
  int64_t u = u0;
  while (u < u1) {
    const int64_t tile = u / sh.nch;
    const int kc0 = static_cast<int>(u - tile * sh.nch);
    const int64_t useg = min(u1, (tile + 1) * sh.nch);
    const int CT = sh.ct_of(tile);
#pragma unroll
    for (int h = 0; h < kRT; ++h)
#pragma unroll
      for (int c = 0; c < kCT; ++c) acc[h][c][0] = acc[h][c][1] = 0.0;
    double* utr = (trc && gi < 4) ? p.sk_trace + 2 * kMaxGrid * 4 + (which * 4 + gi) * 128 * 2 : nullptr;
    switch (CT + 8 * which) {  // one instantiation of the unit loop per segment
      case 1: sk_units<0, 1>(p, sh, stage, cur, ring, u0, nu, u, useg, acc, utr); break;
      case 2: sk_units<0, 2>(p, sh, stage, cur, ring, u0, nu, u, useg, acc, utr); break;
      case 3: sk_units<0, 3>(p, sh, stage, cur, ring, u0, nu, u, useg, acc, utr); break;
      case 4: sk_units<0, 4>(p, sh, stage, cur, ring, u0, nu, u, useg, acc, utr); break;
      case 9: sk_units<1, 1>(p, sh, stage, cur, ring, u0, nu, u, useg, acc, utr); break;
      case 10: sk_units<1, 2>(p, sh, stage, cur, ring, u0, nu, u, useg, acc, utr); break;
      case 11: sk_units<1, 3>(p, sh, stage, cur, ring, u0, nu, u, useg, acc, utr); break;
      default: sk_units<1, 4>(p, sh, stage, cur, ring, u0, nu, u, useg, acc, utr);
    }
    u = useg;
    // ---- segment epilogue
    if (kc0 == 0 && useg == (tile + 1) * sh.nch) {  // the whole tile: write it
#pragma unroll
      for (int h = 0; h < kRT; ++h)
#pragma unroll
        for (int c = 0; c < kCT; ++c)
          if (c < CT)
#pragma unroll
            for (int e = 0; e < 2; ++e) sk_store(p, sh, pact, tile, CT, h, c, e, threadIdx.x, acc[h][c][e]);
      continue;
    }
    // a segment of a shared tile. The range's last segment holding the tile's chunk 0 of
    // a tile with few contributors: this CTA reduces the tile alone after the loop, from
    // these registers. Otherwise: partial into this CTA's slot (0: its first segment, 1:
    // its last), flagged with the product's epoch.
    if (useg == u1 && kc0 == 0 && sk_contrib(tile * sh.nch, (tile + 1) * sh.nch, gi, G).n_ne <= p.sk_fanin) break;
    const int slot = u0 >= tile * sh.nch ? 0 : 1;
    double* dst = p.part + (2 * static_cast<int64_t>(gi) + slot) * kPartTile;
#pragma unroll
    for (int h = 0; h < kRT; ++h)
#pragma unroll
      for (int c = 0; c < kCT; ++c)
        if (c < CT)
#pragma unroll
          for (int e = 0; e < 2; ++e) __stcg(dst + ((h * kCT + c) * 2 + e) * kPT + threadIdx.x, acc[h][c][e]);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0)
      asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p.flags + 2 * gi + slot), "r"(epoch) : "memory");
  }
  ring += static_cast<uint32_t>(nu);
  if (trc) trc[1] = gtimer();
  // ---- shared tiles (at most the first and the last of this CTA's range). A tile with at
  // most p.sk_fanin contributors is reduced by its chunk-0 holder alone (it reaches the
  // tile last, at the end of its range, so the others' partials are there: no wait),
  // starting from its registers; one with more contributors (narrow products: ~20) by
  // all of them, each a slice of the elements. Partials are added in chunk (= CTA) order.
  const int64_t tiles[2] = {u0 / sh.nch, (u1 - 1) / sh.nch};
  int nt = 0, solo_k = -1;  // shared tiles this CTA reduces (solo: the holder's, from registers)
  int64_t rtile[2];
  SkContrib rtc[2];
  for (int s2 = 0; s2 < 2; ++s2) {
    const int64_t tile = tiles[s2];
    if (s2 == 1 && tile == tiles[0]) break;
    const int64_t ta = tile * sh.nch, tb = ta + sh.nch;
    if (u0 <= ta && u1 >= tb) continue;  // whole tile here (written above)
    const SkContrib tc = sk_contrib(ta, tb, gi, G);
    const bool solo = tc.n_ne <= p.sk_fanin;
    if (solo && gi != tc.gA) continue;
    if (solo) solo_k = nt;
    rtile[nt] = tile;
    rtc[nt++] = tc;
  }
  if (nt > 0) {
    // contributor slots of both tiles (chunk order), then every flag waited at once
    __syncthreads();  // s_contrib of the previous product is no longer read
    if (threadIdx.x == 0)
      for (int k = 0; k < nt; ++k) {
        int n = 0;
        const int64_t ta = rtile[k] * sh.nch;
        for (int g2 = rtc[k].gA; g2 <= rtc[k].gB; ++g2)
          if (s_begin[g2 + 1] > s_begin[g2]) s_contrib[k * kMaxGrid + n++] = 2 * g2 + (s_begin[g2] >= ta ? 0 : 1);
      }
    __syncthreads();
    for (int k = 0; k < nt; ++k) {
      const int first = k == solo_k ? 1 : 0;  // the holder's own segment is in registers
      const int t = static_cast<int>(threadIdx.x) - (k == 0 ? 0 : rtc[0].n_ne);
      if (t >= first && t < rtc[k].n_ne) {
        int32_t f = 0;
        do {
          asm volatile("ld.acquire.gpu.global.b32 %0, [%1];"
                       : "=r"(f)
                       : "l"(p.flags + s_contrib[k * kMaxGrid + t])
                       : "memory");
        } while (f != epoch);
      }
    }
    __syncthreads();
  }
  if (trc) trc[3] = gtimer();
  for (int k = 0; k < nt; ++k) {
    const int64_t tile = rtile[k];
    const int CT = sh.ct_of(tile);
    const int32_t* con = s_contrib + k * kMaxGrid;
    const int n_ne = rtc[k].n_ne;
    if (k == solo_k) {
      for (int k2 = 1; k2 < n_ne; ++k2) {
        const double* s2p = p.part + static_cast<int64_t>(con[k2]) * kPartTile;
#pragma unroll
        for (int h = 0; h < kRT; ++h)
#pragma unroll
          for (int c = 0; c < kCT; ++c)
            if (c < CT)
#pragma unroll
              for (int e = 0; e < 2; ++e) acc[h][c][e] += __ldcg(s2p + ((h * kCT + c) * 2 + e) * kPT + threadIdx.x);
      }
#pragma unroll
      for (int h = 0; h < kRT; ++h)
#pragma unroll
        for (int c = 0; c < kCT; ++c)
          if (c < CT)
#pragma unroll
            for (int e = 0; e < 2; ++e) sk_store(p, sh, pact, tile, CT, h, c, e, threadIdx.x, acc[h][c][e]);
      continue;
    }
    const int j = rtc[k].j;
    const int E = kRT * CT * 2 * kPT;  // valid elements of the tile
    const int q0 = E * j / n_ne, q1 = E * (j + 1) / n_ne;
    for (int q = q0 + threadIdx.x; q < q1; q += kPT) {
      const int h = q / (CT * 2 * kPT);
      const int rem = q - h * CT * 2 * kPT;
      const int c = rem / (2 * kPT), e = (rem / kPT) & 1, tid = rem % kPT;
      const int off = ((h * kCT + c) * 2 + e) * kPT + tid;
      double v = 0.0;
      for (int k0 = 0; k0 < n_ne; k0 += 16) {  // up to 16 partials' loads in flight, added in order
        double t[16];
#pragma unroll
        for (int z = 0; z < 16; ++z)
          t[z] = k0 + z < n_ne ? __ldcg(p.part + static_cast<int64_t>(con[k0 + z]) * kPartTile + off) : 0.0;
#pragma unroll
        for (int z = 0; z < 16; ++z)
          if (k0 + z < n_ne) v += t[z];
      }
      sk_store(p, sh, pact, tile, CT, h, c, e, tid, v);
    }
  }
  // W's Rc columns are read by the next product's tensor copies (async proxy) after the
  // caller's grid barrier (Corr is read by generic loads only)
  if (!which) asm volatile("fence.proxy.async.global;" ::: "memory");
  if (trc) trc[2] = gtimer();
}


// ordered compaction of one 256-wide batch: returns the running total; writes the
// flagged items at base offset `tot` (position order)
__device__ __forceinline__ int block_compact(PSh& sh, bool flag, int tot, int* at) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const unsigned bal = __ballot_sync(kAll, flag);
  if (l == 0) sh.wcnt[w] = __popc(bal);
  __syncthreads();
  int off = 0, add = 0;
  for (int ww = 0; ww < kPW; ++ww) {
    if (ww < w) off += sh.wcnt[ww];
    add += sh.wcnt[ww];
  }
  *at = tot + off + __popc(bal & ((1u << l) - 1u));
  __syncthreads();
  return tot + add;
}

__device__ __forceinline__ uint64_t row_flops_dense(const PrefixParams& p, int64_t active, int64_t nnz) {
  const uint64_t un = static_cast<uint64_t>(p.n), uk = static_cast<uint64_t>(p.k);
  const uint64_t ua = static_cast<uint64_t>(active), uz = static_cast<uint64_t>(nnz);
  if (p.variant == FL1_PLAIN) return (uk + uz) * un + 4 * uk + un;  // fastl1.cpp:647-665
  return (ua + uz) * un + 6 * ua + 5 * un;
}

// Signal b finished in the lockstep: final state + packed (final_active, x) outputs
// in the cluster engine's format (finish, fastl1.cpp:741-748).
__device__ void finish_signal(const PrefixParams& p, PSh& sh, int64_t b, bool converged, double gap, double t0) {
  PrefixSig& sg = p.sig[b];
  const int64_t K = p.k;
  const int8_t* mk = p.mask + b * K;
  const double* xc = p.X3[sg.rot % 3] + b * K;
  if (threadIdx.x == 0)
    sh.off = static_cast<int64_t>(atomicAdd(reinterpret_cast<unsigned long long*>(p.out_used),
                                            static_cast<unsigned long long>(sg.S)));
  __syncthreads();
  const int64_t off = sh.off;
  int tot = 0;
  for (int64_t base = 0; base < K; base += kPT) {
    const int64_t j = base + threadIdx.x;
    const bool on = j < K && mk[j] != 0;
    int at;
    tot = block_compact(sh, on, tot, &at);
    if (on) {
      p.out_idx[off + at] = static_cast<int32_t>(j);
      p.out_x[off + at] = xc[j];
    }
  }
  if (threadIdx.x == 0) {
    EngineState st{};
    st.t = converged ? sg.t + 1 : sg.t;
    st.ledger = sg.ledger;
    st.S = sg.S;
    st.active_at_last_l = sg.active_at_last_l;
    st.n_trace = sg.n_trace;
    st.power_steps = sg.power_steps;
    st.t_k = sg.t_k;
    st.lipschitz = sg.lipschitz;
    st.inv_l = sg.inv_l;
    st.y_sq = sg.y_sq;
    st.final_gap = gap;
    st.start_ns = t0;
    st.t0_ns = t0;
    st.end_ns = gtimer();
    st.momentum_ready = sg.ready;
    st.warning = sg.warning;
    st.converged = converged ? 1 : 0;
    st.done = 1;
    st.event = kEvDone;
    p.states[b] = st;
    p.out_off[b] = off;
    Handoff h{};
    h.state = 2;
    p.hand[b] = h;
    sg.mode = 2;
  }
  __syncthreads();
}

// Exact fit (rho_g == 0): hand the signal to the per-signal engine at the start of
// iteration t with its preserved set compacted (ActiveOp layout).
__device__ void handoff_signal(const PrefixParams& p, PSh& sh, int64_t b, double t0) {
  PrefixSig& sg = p.sig[b];
  const int64_t K = p.k;
  const int8_t* mk = p.mask + b * K;
  const int rot = sg.rot;
  const double* xc = p.X3[rot % 3] + b * K;
  const double* xpc = p.X3[(rot + 1) % 3] + b * K;
  double* gx = p.X3[(rot + 2) % 3] + b * K;  // x_next role: free between iterations
  double* gxp = p.psrc + b * K;               // free outside power steps
  double* gl = p.vp + b * K;
  int32_t* gi = p.hidx + b * K;
  const double* ld_ = p.lead + b * K;
  int tot = 0;
  for (int64_t base = 0; base < K; base += kPT) {
    const int64_t j = base + threadIdx.x;
    const bool on = j < K && mk[j] != 0;
    const double xv = on ? xc[j] : 0.0, xpv = on ? xpc[j] : 0.0, lv = on ? ld_[j] : 0.0;
    int at;
    tot = block_compact(sh, on, tot, &at);
    if (on) {
      gi[at] = static_cast<int32_t>(j);
      gx[at] = xv;
      gxp[at] = xpv;
      gl[at] = lv;
    }
  }
  if (threadIdx.x == 0) {
    Handoff h{};
    h.idx = gi;
    h.x = gx;
    h.xp = gxp;
    h.lead = gl;
    h.u = p.U2[sg.uswap] + b * p.ld;
    h.v = p.U2[1 - sg.uswap] + b * p.ld;
    h.t = sg.t;
    h.ledger = sg.ledger;
    h.n_trace = sg.n_trace;
    h.S = sg.S;
    h.active_at_last_l = sg.active_at_last_l;
    h.power_steps = sg.power_steps;
    h.t_k = sg.t_k;
    h.lipschitz = sg.lipschitz;
    h.elapsed_ns = gtimer() - t0;
    h.ready = sg.ready;
    h.warning = sg.warning;
    h.lead_valid = sg.lead_valid;
    h.state = 1;
    p.hand[b] = h;
    sg.mode = 3;
  }
  __syncthreads();
}

// compute_products (fastl1.cpp:359-369) for signal b's NEXT iteration: rho_g =
// y - ((1+m)u - m v) into its R column, with ||rho_g||^2, rho_g.y, ||y - u||^2.
__device__ void compute_rho(const PrefixParams& p, PSh& sh, int64_t b) {
  PrefixSig& sg = p.sig[b];
  const int64_t N = p.n, ld = p.ld;
  double m = 0.0;
  if (p.solver == FL1_FISTA && sg.ready) m = (sg.t_k - 1.0) / (0.5 * (1.0 + sqrt(1.0 + 4.0 * sg.t_k * sg.t_k)));
  const bool mom = m != 0.0;
  const double* uc = p.U2[sg.uswap] + b * ld;
  const double* vc = p.U2[1 - sg.uswap] + b * ld;
  double v[3] = {0.0, 0.0, 0.0};
  for (int64_t i = threadIdx.x; i < ld; i += kPT) {
    double r = 0.0;
    if (i < N) {
      const double u = uc[i];
      const double uw = mom ? (1.0 + m) * u - m * vc[i] : u;
      const double yi = p.y[b * p.ldy + i];
      r = yi - uw;
      v[0] = fma(r, r, v[0]);
      v[1] = fma(yi, r, v[1]);
      if (mom) {
        const double e = yi - u;
        v[2] = fma(e, e, v[2]);
      }
    }
    __stcg(p.R + b * ld + i, r);
  }
  block_sum3(v, sh);
  if (threadIdx.x == 0) {
    sg.rsq = v[0];
    sg.rdy = v[1];
    sg.ree = v[2];
  }
  __syncthreads();
}

// Per-signal passes over the K atoms: warp w owns the contiguous atom range
// [w Kw, (w+1) Kw), so lists built by per-warp ballots are in atom order when read
// warp by warp -- no block barrier per 256 atoms.
struct WarpRange {
  int64_t lo, hi;
  __device__ WarpRange(int64_t K) {
    const int64_t kw = (K + kPW - 1) / kPW;
    const int w = threadIdx.x >> 5;
    lo = min(K, kw * w);
    hi = min(K, lo + kw);
  }
};

// append (v, j) to this warp's list segment when flag; returns the new count
__device__ __forceinline__ int warp_append(bool flag, double v, int32_t j, double* ev, int32_t* ej, int cnt) {
  const int l = threadIdx.x & 31;
  const unsigned bal = __ballot_sync(kAll, flag);
  if (flag) {
    const int at = cnt + __popc(bal & ((1u << l) - 1u));
    ev[at] = v;
    ej[at] = j;
  }
  return cnt + __popc(bal);
}

// rows over threads: acc_i += sum over the warp segments (in warp = atom order).
// The entries are walked as one list across the segments (a uniform cursor), eight
// per round, two rows per thread: 16 loads in flight and ~nnz/8 L2 round trips
// instead of one per entry at every segment's tail.
#ifndef FL1_APE
#define FL1_APE 8
#endif
constexpr int kApE = FL1_APE, kApR = 2;
__device__ __forceinline__ void apply_segments(const PrefixParams& p, double* us, const double* ev, const int32_t* ej,
                                               int64_t seg, const int32_t* cnt, double sign) {
  const int64_t ld = p.ld;
  const double* __restrict__ A = p.a;
  for (int64_t i0 = threadIdx.x; i0 < ld; i0 += kApR * kPT) {
    double acc[kApR];
    bool ok[kApR];
#pragma unroll
    for (int r = 0; r < kApR; ++r) {
      ok[r] = i0 + r * kPT < ld;
      acc[r] = ok[r] ? us[i0 + r * kPT] : 0.0;
    }
    int cw = 0, ce = 0;  // cursor: segment, entry
    while (true) {
      int32_t jq[kApE];
      double vq[kApE];
      int got = 0;
#pragma unroll
      for (int q = 0; q < kApE; ++q) {
        while (cw < kPW && ce >= cnt[cw]) {
          ++cw;
          ce = 0;
        }
        jq[q] = -1;
        vq[q] = 0.0;
        if (cw < kPW) {
          jq[q] = ej[cw * seg + ce];
          vq[q] = sign * ev[cw * seg + ce];
          ++ce;
          ++got;
        }
      }
      if (got == 0) break;
      double a[kApE][kApR];
#pragma unroll
      for (int q = 0; q < kApE; ++q) {
        const double* col = A + static_cast<int64_t>(jq[q] < 0 ? 0 : jq[q]) * ld + i0;
#pragma unroll
        for (int r = 0; r < kApR; ++r) a[q][r] = (ok[r] && jq[q] >= 0) ? __ldg(col + r * kPT) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < kApE; ++q) {
        if (jq[q] < 0) continue;
#pragma unroll
        for (int r = 0; r < kApR; ++r) acc[r] = fma(vq[q], a[q][r], acc[r]);
      }
      if (got < kApE) break;
    }
#pragma unroll
    for (int r = 0; r < kApR; ++r)
      if (ok[r]) us[i0 + r * kPT] = acc[r];
  }
  __syncthreads();
}

// Enter the restricted power iteration (power_iteration_sq_norm, solver.cpp:72-104):
// warm from the gathered leading vector when it is nonzero, else the fixed Gaussian
// start by preserved position (rank among unmasked atoms).
__device__ void enter_power(const PrefixParams& p, PSh& sh, int64_t b) {
  PrefixSig& sg = p.sig[b];
  const int64_t K = p.k;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int8_t* mk = p.mask + b * K;
  const double* ldv = p.lead + b * K;
  double* vp = p.vp + b * K;
  const WarpRange wr(K);
  // pass 1: |lead|^2 over the set and the warp's active count (rank offsets)
  double a_lead = 0.0;
  int cnt = 0;
  for (int64_t base = wr.lo; base < wr.hi; base += 32) {
    const int64_t j = base + l;
    const bool on = j < wr.hi && mk[j] != 0;
    if (on && sg.lead_valid) a_lead = fma(ldv[j], ldv[j], a_lead);
    cnt += __popc(__ballot_sync(kAll, on));
  }
  if (l == 0) sh.wcnt[w] = cnt;
  a_lead = block_sum(a_lead, sh);
  const bool warm = sg.lead_valid && a_lead > 0.0;
  int off = 0;
  for (int ww = 0; ww < w; ++ww) off += sh.wcnt[ww];
  // pass 2: the start vector (this lane's atoms wr.lo + l + 32 i, in registers)
  double acc = 0.0, sv[kIt];
#pragma unroll
  for (int i = 0; i < kIt; ++i) {
    const int64_t j = wr.lo + l + 32 * i;
    sv[i] = 0.0;
    if (wr.lo + 32 * i >= wr.hi) continue;  // warp-uniform
    const bool on = j < wr.hi && mk[j] != 0;
    const unsigned bal = __ballot_sync(kAll, on);
    if (on) sv[i] = warm ? ldv[j] : p.gauss0[off + __popc(bal & ((1u << l) - 1u))];
    acc = fma(sv[i], sv[i], acc);
    off += __popc(bal);
  }
  const double nrm2 = warm ? a_lead : block_sum(acc, sh);
  const double div = sqrt(nrm2);
#pragma unroll
  for (int i = 0; i < kIt; ++i) {
    const int64_t j = wr.lo + l + 32 * i;
    if (j < wr.hi) vp[j] = sv[i] / div;
  }
  if (threadIdx.x == 0) {
    sg.mode = 1;
    sg.p_div = div;
    sg.p_est = 0.0;
    sg.p_it = 0;
    sg.p_have_w = 0;
    sg.p_max = warm ? 12 : 200;
    sg.p_min = warm ? 2 : 4;
    sg.p_tol = warm ? 1e-5 : 1e-9;
  }
  __syncthreads();
}

// corr of this lane's atoms (wr.lo + l + 32 i) summed over the split-K parts in part
// order, two parts' loads in flight together
__device__ __forceinline__ void sum_parts(const double* __restrict__ cr, int64_t part, int sk, const WarpRange& wr,
                                          double (&cv)[kIt]) {
  const int l = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < kIt; ++i) {
    const int64_t j = wr.lo + l + 32 * i;
    cv[i] = j < wr.hi ? __ldcg(cr + j) : 0.0;
  }
  for (int kp0 = 1; kp0 < sk; kp0 += 2) {
    double pv[2][kIt];
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int i = 0; i < kIt; ++i) {
        const int64_t j = wr.lo + l + 32 * i;
        pv[q][i] = (kp0 + q < sk && j < wr.hi) ? __ldcg(cr + (kp0 + q) * part + j) : 0.0;
      }
#pragma unroll
    for (int q = 0; q < 2; ++q)
      if (kp0 + q < sk)
#pragma unroll
        for (int i = 0; i < kIt; ++i) cv[i] += pv[q][i];
  }
}

// One power step's update after v_new = A_S^T A_S v (slot a's corr column parts).
__device__ __noinline__ void power_step(const PrefixParams& p, PSh& sh, int64_t a, int64_t b, int sk, double t0) {
  PrefixSig& sg = p.sig[b];
  const int64_t K = p.k, part = K * p.bcap;
  const double* cr = p.corr + a * K;
  const int8_t* mk = p.mask + b * K;
  double* vp = p.vp + b * K;
  const WarpRange wr(K);
  const int l = threadIdx.x & 31;
  double v[3] = {0.0, 0.0, 0.0};  // |v_new|^2, v.v_new
  // v_new (unnormalised, the reference's cur_src) stays in registers: every load of the
  // pass (corr, mask, v) is issued before the first is used
  double cv[kIt], vv[kIt];
  bool on[kIt];
  sum_parts(cr, part, sk, wr, cv);
#pragma unroll
  for (int i = 0; i < kIt; ++i) {
    const int64_t j = wr.lo + l + 32 * i;
    on[i] = j < wr.hi && mk[j] != 0;
    vv[i] = j < wr.hi ? vp[j] : 0.0;
  }
#pragma unroll
  for (int i = 0; i < kIt; ++i)
    if (on[i]) {
      v[0] = fma(cv[i], cv[i], v[0]);
      v[1] = fma(vv[i], cv[i], v[1]);
    }
  block_sum3(v, sh);
  if (threadIdx.x == 0) {
    sg.power_steps += 1;
    const double nrm = sqrt(v[0]);
    int stop = 0;
    double est = sg.p_est;
    if (nrm == 0.0) {
      est = 0.0;
      stop = 2;  // lead = have_w ? w / div : v  (w = 0 here)
    } else {
      const double prev = est;
      est = v[1];
      sg.p_div = nrm;
      sg.p_have_w = 1;
      if (sg.p_it > sg.p_min && fabs(est - prev) <= sg.p_tol * est) stop = 1;
      else if (sg.p_it + 1 >= sg.p_max) stop = 1;
    }
    sg.p_est = est;
    sg.p_it += 1;
    sh.release = stop;
    sh.m = sg.p_div;
  }
  __syncthreads();
  const int stop = sh.release;
  const double div = sh.m;
  const bool have_w = stop == 2 && sg.p_have_w;
#pragma unroll
  for (int i = 0; i < kIt; ++i) {  // same thread mapping as above
    const int64_t j = wr.lo + l + 32 * i;
    if (j >= wr.hi) break;
    if (stop == 2) {
      p.lead[b * K + j] = have_w ? 0.0 : vv[i];
    } else {
      const double v1 = on[i] ? cv[i] / div : 0.0;
      if (stop) p.lead[b * K + j] = v1;
      else vp[j] = v1;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && stop) {
    sg.lipschitz = fmax(sg.p_est, 1e-300) * 1.05;  // restricted_lipschitz (fastl1.cpp:326-333)
    sg.inv_l = 1.0 / sg.lipschitz;
    sg.lead_valid = 1;
    sg.active_at_last_l = sg.S;
    sg.mode = 0;
  }
  __syncthreads();
  if (stop && p.policy == 2) {
    handoff_signal(p, sh, b, t0);
  } else if (stop) {
    compute_rho(p, sh, b);
  }
}

// One FISTA / ISTA iteration of signal b (slot a): fastl1.cpp:459-645 with the
// exact dictionary, GAP rule, preserved set = mask.
__device__ __noinline__ void fista_step(const PrefixParams& p, PSh& sh, int64_t a, int64_t b, double t0, int sk,
                                        double* us, double* stage) {
  PrefixSig& sg = p.sig[b];
  if (p.policy == 3 && sg.lead_valid && sg.S <= p.handoff_s) {  // leave at the start of this iteration
    handoff_signal(p, sh, b, t0);
    return;
  }
  const int64_t K = p.k, ld = p.ld, part = K * p.bcap;
  const double lambda = p.lambdas[b];
  const uint64_t t = sg.t;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const WarpRange wr(K);
  double* cr = p.corr + a * K;
  int8_t* mk = p.mask + b * K;
  SIGPROF(14);
  // corr = sum of the split-K parts, written back to part 0; max |corr| over the set
  // (all kIt atoms of a lane loaded together: one L2 round trip per split part)
  double dp = 0.0;
  // thread 0's scalars, loaded before the reduction so that their L2 round trip overlaps it
  double q_tk = 0.0, q_rsq = 0.0, q_rdy = 0.0, q_ree = 0.0, q_xl1 = 0.0, q_ysq = 0.0;
  int q_ready = 0;
  int64_t q_S = 0;
  if (threadIdx.x == 0) {
    q_tk = sg.t_k;
    q_rsq = sg.rsq;
    q_rdy = sg.rdy;
    q_ree = sg.ree;
    q_xl1 = sg.x_l1;
    q_ysq = sg.y_sq;
    q_ready = sg.ready;
    q_S = sg.S;
  }
  {
    double cv[kIt];
    sum_parts(cr, part, sk, wr, cv);
#pragma unroll
    for (int i = 0; i < kIt; ++i) {
      const int64_t j = wr.lo + l + 32 * i;
      if (j < wr.hi) {
        if (sk > 1) __stcg(cr + j, cv[i]);
        if (mk[j]) dp = fmax(dp, fabs(cv[i]));
      }
    }
  }
  dp = block_max(dp, sh);
  SIGPROF(0);
  if (threadIdx.x == 0) {
    double m = 0.0, t_next = q_tk;  // 465-470
    if (p.solver == FL1_FISTA && q_ready) {
      t_next = 0.5 * (1.0 + sqrt(1.0 + 4.0 * q_tk * q_tk));
      m = (q_tk - 1.0) / t_next;
    }
    const double rsq = q_rsq, rdy = q_rdy;
    const double rho_x_sq = m != 0.0 ? q_ree : rsq;
    const double primal = 0.5 * rho_x_sq + lambda * q_xl1;
    int rel = 0, screen = 0;
    double sp = 0.0, radius = 0.0, gt = 0.0;
    if (!(rsq > 0.0)) {
      rel = 3;  // exact fit: the per-signal engine takes the y-ray branch (428-449)
    } else {
      const double projection = rdy / (lambda * rsq);  // dual_scalars (406-450), eps = 0
      const double ap = (q_S > 0 && dp > 0) ? 1.0 / dp : CUDART_INF;
      sp = fmin(fmax(projection, -ap), ap);
      const double dist_sq = sp * sp * rsq - 2.0 * sp * rdy / lambda + q_ysq / (lambda * lambda);
      const double dual = 0.5 * q_ysq - 0.5 * lambda * lambda * dist_sq;  // 453-457
      double gp = primal - dual;  // scale' == scale~ on the exact dictionary
      if (gp < -1e-10) sg.warning = 1;
      gp = fmax(gp, 0.0);
      gt = gp;
      const double stop_tol = p.rel_tol > 0 ? p.rel_tol * primal : p.tol;
      if (gt <= stop_tol) rel = 2;
      screen = !rel && p.variant != FL1_PLAIN && (t % static_cast<uint64_t>(p.interval) == 0);
      radius = sqrt(2.0 * gp) / lambda;
    }
    sh.m = m;
    sh.t_next = t_next;
    sh.sp = sp;
    sh.radius = radius;
    sh.gap_tilde = gt;
    sh.release = rel;
    sh.screen = screen;
  }
  __syncthreads();
  SIGPROF(1);
  if (sh.release == 3) {
    handoff_signal(p, sh, b, t0);
    return;
  }
  const int rot = sg.rot;
  double* __restrict__ xc = p.X3[rot % 3] + b * K;
  double* __restrict__ xpc = p.X3[(rot + 1) % 3] + b * K;
  double* __restrict__ xn = p.X3[(rot + 2) % 3] + b * K;
  const int64_t S_old = sg.S;
  if (sh.release == 2) {  // stop (fastl1.cpp:568-571, 625-633)
    double nnz = 0.0;
    for (int64_t j = threadIdx.x; j < K; j += kPT) nnz += (mk[j] && xc[j] != 0.0) ? 1.0 : 0.0;
    nnz = block_sum(nnz, sh);
    if (threadIdx.x == 0) {
      sg.ledger += row_flops_dense(p, S_old, static_cast<int64_t>(nnz));
      if (p.collect_trace && sg.n_trace < p.trace_cap) {
        fl1_trace_row row{};
        row.iter = t;
        row.active_size = static_cast<int32_t>(S_old);
        row.gap = sh.gap_tilde;
        row.gamma = -1.0;
        row.flops_cum = sg.ledger;
        row.wall_ms = (gtimer() - t0) * 1e-6;
        row.x_nnz = static_cast<int32_t>(nnz);
        p.traces[b * p.trace_cap + sg.n_trace] = row;
        sg.n_trace += 1;
      }
    }
    __syncthreads();
    finish_signal(p, sh, b, true, sh.gap_tilde, t0);
    return;
  }
  if (p.policy == 1 && sh.screen) {  // policy 1: leave at the start of an iteration that would shrink
    double drops = 0.0;
    for (int64_t j = threadIdx.x; j < K; j += kPT)
      if (mk[j] && !(__fma_rn(sh.radius, p.en[j], fabs(__dmul_rn(sh.sp, __ldcg(cr + j)))) >= 1.0)) drops += 1.0;
    drops = block_sum(drops, sh);
    if (drops > 0.0) {
      handoff_signal(p, sh, b, t0);
      return;
    }
  }
  // One pass: screening (494-566; stable test with eps = 0), prox (572-579), and the
  // restriction (667-702) folded in: a dropped atom's x_next is discarded, its
  // x_prev (the old x) feeds the v fix, and it leaves x, x_prev, lead and the mask.
  // Lists per warp segment: nonzeros of the new x (u = A x) and the v-fix entries.
  const double m = sh.m, inv_l = sg.inv_l, thresh = lambda * sg.inv_l;
  const bool screen = sh.screen != 0, fista = p.solver == FL1_FISTA;
  const double spv = sh.sp, rad = sh.radius;
  const int64_t seg = (K + kPW - 1) / kPW;
  double* nz_v = stage;                                   // K values
  double* fx_v = stage + seg * kPW;                       // K values
  int32_t* nz_j = reinterpret_cast<int32_t*>(stage + 2 * seg * kPW);
  int32_t* fx_j = nz_j + seg * kPW;
  int nz_c = 0, fx_c = 0;
  double red3[3] = {0.0, 0.0, 0.0};  // kept, nnz(x_new), |x_new|_1
  for (int64_t b0 = wr.lo; b0 < wr.hi; b0 += 32 * kItB) {
    // the next kItB groups of 32 atoms: every load issued before the first is used
    bool onv[kItB];
    double cq[kItB], xq[kItB], xpq[kItB], eq[kItB];
#pragma unroll
    for (int i = 0; i < kItB; ++i) {
      const int64_t j = b0 + 32 * i + l;
      onv[i] = j < wr.hi && mk[j];
      cq[i] = onv[i] ? __ldcg(cr + j) : 0.0;
      xq[i] = onv[i] ? xc[j] : 0.0;
      xpq[i] = (onv[i] && m != 0.0) ? xpc[j] : 0.0;
      eq[i] = (onv[i] && screen) ? p.en[j] : 0.0;
    }
#pragma unroll
  for (int i = 0; i < kItB; ++i) {
    const int64_t base = b0 + 32 * i;
    if (base >= wr.hi) break;  // warp-uniform
    const int64_t j = base + l;
    double v = 0.0, fixv = 0.0;
    if (onv[i]) {
      const double c = cq[i];
      const double xo = xq[i];
      const double xpv = xpq[i];
      const double gg = m != 0.0 ? __fma_rn(1.0 + m, xo, -__dmul_rn(m, xpv)) : xo;
      const double z = __fma_rn(inv_l, c, gg);
      const double mag = fabs(z) - thresh;
      v = mag <= 0.0 ? 0.0 : (z > 0.0 ? mag : -mag);
      const bool keep = !screen || __fma_rn(rad, eq[i], fabs(__dmul_rn(spv, c))) >= 1.0;
      if (keep) {
        red3[0] += 1.0;
      } else {  // dropped: x_prev of the shifted history is the old x
        if (fista && xo != 0.0) fixv = -xo;
        v = 0.0;
        mk[j] = 0;
        xc[j] = 0.0;  // becomes x_prev after the role rotation
        p.lead[b * K + j] = 0.0;
      }
      red3[1] += v != 0.0 ? 1.0 : 0.0;
      red3[2] += fabs(v);
    }
    if (j < wr.hi) xn[j] = v;
    nz_c = warp_append(v != 0.0, v, static_cast<int32_t>(j), nz_v + w * seg, nz_j + w * seg, nz_c);
    fx_c = warp_append(fixv != 0.0, fixv, static_cast<int32_t>(j), fx_v + w * seg, fx_j + w * seg, fx_c);
  }
  }
  if (l == 0) {
    sh.nzc[w] = nz_c;
    sh.fxc[w] = fx_c;
  }
  block_sum3(red3, sh);  // (syncs: the warp counts are visible after it)
  SIGPROF(2);
  const int64_t S_new = static_cast<int64_t>(red3[0]);
  const double nnz = red3[1], l1n = red3[2];
  // FISTA bookkeeping (581-590): x_prev = x, v = u (the old u buffer, minus the fix), x = x_next
  const double* __restrict__ uo = p.U2[sg.uswap] + b * ld;
  double* __restrict__ un = p.U2[1 - sg.uswap] + b * ld;
  int any_fix = 0;
  for (int ww = 0; ww < kPW; ++ww) any_fix += sh.fxc[ww];
  if (fista && any_fix) {
    for (int64_t i = threadIdx.x; i < ld; i += kPT) us[i] = uo[i];
    __syncthreads();
    apply_segments(p, us, fx_v, fx_j, seg, sh.fxc, 1.0);
    for (int64_t i = threadIdx.x; i < ld; i += kPT) const_cast<double*>(uo)[i] = us[i];
  }
  SIGPROF(3);
  for (int64_t i = threadIdx.x; i < ld; i += kPT) us[i] = 0.0;
  __syncthreads();
  apply_segments(p, us, nz_v, nz_j, seg, sh.nzc, 1.0);  // u = A x (ActiveOp::apply 131-146)
  for (int64_t i = threadIdx.x; i < ld; i += kPT) un[i] = us[i];
  SIGPROF(4);
  if (threadIdx.x == 0) {
    if (fista) {
      if (sg.ready) sg.t_k = sh.t_next;
      sg.ready = 1;
    }
    sg.rot = (rot + 2) % 3;
    sg.uswap = 1 - sg.uswap;
    sg.x_l1 = l1n;
    sg.S = S_new;
    sg.ledger += row_flops_dense(p, S_old, static_cast<int64_t>(nnz));
    if (p.collect_trace && sg.n_trace < p.trace_cap) {
      fl1_trace_row row{};
      row.iter = t;
      row.active_size = static_cast<int32_t>(S_old);
      row.gap = sh.gap_tilde;
      row.gamma = -1.0;
      row.flops_cum = sg.ledger;
      row.wall_ms = (gtimer() - t0) * 1e-6;
      row.x_nnz = static_cast<int32_t>(nnz);
      p.traces[b * p.trace_cap + sg.n_trace] = row;
      sg.n_trace += 1;
    }
    sg.t = t + 1;
    // restricted Lipschitz refresh when the set halved (603-608); the cap ends the run (640-644)
    sh.screen = (S_new * 2 <= sg.active_at_last_l && S_new > 0) ? 1 : 0;
    sh.release = sg.t >= p.max_it ? 1 : 0;
  }
  __syncthreads();
  if (sh.release) {
    finish_signal(p, sh, b, false, 0.0, t0);
  } else if (sh.screen) {
    enter_power(p, sh, b);
  } else {
    compute_rho(p, sh, b);
  }
  SIGPROF(5);
  if (p.sigprof && blockIdx.x == 0 && threadIdx.x == 0) p.sigprof[13] += 1.0;
}

// ---------------------------------------------------------------------------
// Narrow steps (few unfinished signals: the lockstep's tail, where most signals have
// left and the rest are in their cold power iterations). A 128 x 64 DMMA tile would be
// 1-12 signals wide and the contraction latency-bound (~30 us each at any width), so
// the two products run on the CUDA cores instead, each reading A once from L2:
//   Corr = A^T R: one warp per atom, the n residual columns staged in shared memory,
//                 n warp-shuffle dot products per atom (written as split part 0);
//   W = A V:      CTA (g, r) sums the atoms of column group g (kNarrowParts groups) for
//                 the rows of slice r (128 rows), four column subsets per row combined in
//                 shared memory in fixed order; the group partials are summed in group
//                 order by the combine (deterministic).
constexpr int kNarrow = 12;        // widest narrow step (R columns staged in shared memory)
constexpr int kNarrowParts = 16;   // column groups of W = A V
constexpr int kNarrowRows = 128;   // rows per CTA of W = A V (kPT / 4 threads per subset)

__device__ __forceinline__ bool narrow_fits(int n, int64_t ld) {
  return n <= kNarrow && static_cast<int64_t>(n) * ld <= static_cast<int64_t>(kStages) * kStage;
}

__device__ __noinline__ void narrow_corr(const PrefixParams& p, int n_act, const int32_t* act, double* stage) {
  const int64_t K = p.k, ld = p.ld;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int64_t e = threadIdx.x; e < static_cast<int64_t>(n_act) * ld; e += kPT) {
    const int64_t a = e / ld, i = e - a * ld;
    stage[e] = __ldcg(p.R + static_cast<int64_t>(act[a]) * ld + i);
  }
  __syncthreads();
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * kPW + w, nw = static_cast<int64_t>(gridDim.x) * kPW;
  for (int64_t j = gw; j < K; j += nw) {
    double acc[kNarrow];
#pragma unroll
    for (int a = 0; a < kNarrow; ++a) acc[a] = 0.0;
    const double2* col = reinterpret_cast<const double2*>(p.a + j * ld);
    const int64_t n2 = ld >> 1;
    for (int64_t e0 = l; e0 < n2; e0 += 128) {
      double2 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = e0 + 32 * u < n2 ? __ldg(col + e0 + 32 * u) : make_double2(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t i = 2 * (e0 + 32 * u);
        if (i < ld) {
#pragma unroll
          for (int a = 0; a < kNarrow; ++a)
            if (a < n_act) {
              const double2 r = *reinterpret_cast<const double2*>(stage + a * ld + i);
              acc[a] = fma(v[u].x, r.x, fma(v[u].y, r.y, acc[a]));
            }
        }
      }
    }
#pragma unroll
    for (int a = 0; a < kNarrow; ++a) {
      if (a < n_act) {
        double t = acc[a];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(kAll, t, o);
        if (l == 0) __stcg(p.corr + static_cast<int64_t>(a) * K + j, t);
      }
    }
  }
  __syncthreads();  // the staging area is reused by the per-signal steps
}

// W partial of column group g = item % kNarrowParts, row slice r = item / kNarrowParts,
// into np[(g * n_pow + c) * ld + i]
__device__ __noinline__ void narrow_w(const PrefixParams& p, int n_pow, const int32_t* pact, const int32_t* act,
                                      double* stage) {
  const int64_t K = p.k, ld = p.ld;
  const int n_slices = static_cast<int>((ld + kNarrowRows - 1) / kNarrowRows);
  const int64_t gk = (K + kNarrowParts - 1) / kNarrowParts;
  double* Vs = stage;                                              // [gk][n_pow]
  double* Red = stage + gk * kNarrow;                              // [4][kNarrowRows][n_pow]
  const int row = threadIdx.x % kNarrowRows, sub = threadIdx.x / kNarrowRows;
  for (int item = blockIdx.x; item < kNarrowParts * n_slices; item += gridDim.x) {
    const int g = item % kNarrowParts, r = item / kNarrowParts;
    const int64_t j0 = g * gk, j1 = min(K, j0 + gk), i = static_cast<int64_t>(r) * kNarrowRows + row;
    __syncthreads();
    for (int64_t e = threadIdx.x; e < (j1 - j0) * n_pow; e += kPT) {
      const int64_t jj = e / n_pow, c = e - jj * n_pow;
      Vs[e] = __ldcg(p.vp + static_cast<int64_t>(act[pact[c]]) * K + j0 + jj);
    }
    __syncthreads();
    double acc[kNarrow];
#pragma unroll
    for (int c = 0; c < kNarrow; ++c) acc[c] = 0.0;
    if (i < ld) {
      for (int64_t j = j0 + sub; j < j1; j += 4) {
        const double av = __ldg(p.a + j * ld + i);
        const double* vr = Vs + (j - j0) * n_pow;
#pragma unroll
        for (int c = 0; c < kNarrow; ++c)
          if (c < n_pow) acc[c] = fma(av, vr[c], acc[c]);
      }
    }
#pragma unroll
    for (int c = 0; c < kNarrow; ++c)
      if (c < n_pow) Red[(sub * kNarrowRows + row) * n_pow + c] = acc[c];
    __syncthreads();
    if (sub == 0 && i < ld) {
      for (int c = 0; c < n_pow; ++c) {
        double t = Red[row * n_pow + c];
        for (int s2 = 1; s2 < 4; ++s2) t += Red[(s2 * kNarrowRows + row) * n_pow + c];
        __stcg(p.np + (static_cast<int64_t>(g) * n_pow + c) * ld + i, t);
      }
    }
  }
}

}  // namespace

// The split-K route's products (FL1_LOCKSTEP_TMA=0) and the narrow W combine, out of the
// kernel body (its register allocation is shared by every step's control flow).
constexpr int kNarrowTag = -1;  // legacy_w_combine: the narrow W partials' layout
__device__ __noinline__ int legacy_w_tiles(const PrefixParams& p, int n_pow, const int32_t* pact, const int32_t* act,
                                           double* stage) {
  const int64_t ld = p.ld, K = p.k;
  const int n_rt = static_cast<int>((ld + kTM - 1) / kTM);
  const int n_ct = (n_pow + kTN - 1) / kTN;
  const int sk = p.split_mode ? split_for(n_rt * n_ct, gridDim.x, static_cast<int>((K + kTK - 1) / kTK),
                                          split_cap(p, ld * n_pow))
                              : split_old(n_rt * n_ct, gridDim.x);
  for (int item = blockIdx.x; item < n_rt * n_ct * sk; item += gridDim.x) {
    const int tile = item % (n_rt * n_ct), kp = item / (n_rt * n_ct);
    const int64_t c0 = static_cast<int64_t>(tile / n_rt) * kTN;
    switch (tile_ct(static_cast<int>(n_pow - c0), p.width_tiles)) {  // the last column tile may be narrow
      case 1: gemm_n_tile<1>(p, tile % n_rt, c0, kp, sk, n_pow, pact, act, stage); break;
      case 2: gemm_n_tile<2>(p, tile % n_rt, c0, kp, sk, n_pow, pact, act, stage); break;
      case 3: gemm_n_tile<3>(p, tile % n_rt, c0, kp, sk, n_pow, pact, act, stage); break;
      default: gemm_n_tile<kCT>(p, tile % n_rt, c0, kp, sk, n_pow, pact, act, stage);
    }
  }
  return sk;
}
// w of power slot pc = the partials in part order into R (split-K: parts of bcap columns;
// narrow: kNarrowParts groups of n_pow columns)
__device__ __noinline__ void legacy_w_combine(const PrefixParams& p, int n_pow, const int32_t* pact,
                                              const int32_t* act, int layout, int parts) {
  const int64_t ld = p.ld, N = p.n;
  const int64_t pstride = layout == kNarrowTag ? static_cast<int64_t>(n_pow) : static_cast<int64_t>(p.bcap);
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * kPT + threadIdx.x; e < static_cast<int64_t>(n_pow) * ld;
       e += static_cast<int64_t>(gridDim.x) * kPT) {
    const int64_t pc = e / ld, i = e - pc * ld;
    double w = 0.0;
    for (int kp = 0; kp < parts; ++kp) w += __ldcg(p.np + (static_cast<int64_t>(kp) * pstride + pc) * ld + i);
    __stcg(p.R + static_cast<int64_t>(act[pact[pc]]) * ld + i, i < N ? w : 0.0);
  }
}
__device__ __noinline__ int legacy_corr_tiles(const PrefixParams& p, int n_act, const int32_t* act, double* stage) {
  const int64_t ld = p.ld, K = p.k;
  const int n_rt = static_cast<int>((K + kTM - 1) / kTM);
  const int n_ct = (n_act + kTN - 1) / kTN;
  const int sk = p.split_mode ? split_for(n_rt * n_ct, gridDim.x, static_cast<int>((ld + kTK - 1) / kTK),
                                          split_cap(p, K * n_act))
                              : split_old(n_rt * n_ct, gridDim.x);
  for (int item = blockIdx.x; item < n_rt * n_ct * sk; item += gridDim.x) {
    const int tile = item % (n_rt * n_ct), kp = item / (n_rt * n_ct);
    const int64_t a0 = static_cast<int64_t>(tile / n_rt) * kTN;
    switch (tile_ct(static_cast<int>(n_act - a0), p.width_tiles)) {  // the last column tile may be narrow
      case 1: gemm_tile<1>(p, tile % n_rt, a0, kp, sk, n_act, act, stage); break;
      case 2: gemm_tile<2>(p, tile % n_rt, a0, kp, sk, n_act, act, stage); break;
      case 3: gemm_tile<3>(p, tile % n_rt, a0, kp, sk, n_act, act, stage); break;
      default: gemm_tile<kCT>(p, tile % n_rt, a0, kp, sk, n_act, act, stage);
    }
  }
  return sk;
}

__global__ void __launch_bounds__(kPT, 1) prefix_kernel(const __grid_constant__ PrefixParams p) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(128) double dsm[];
  __shared__ PSh sh;
  const int64_t B = p.batch, K = p.k, N = p.n, ld = p.ld;
  const double t0 = gtimer();
  // dynamic smem: [staging (contraction tiles; lists in the per-signal steps) | u | act | pact],
  // the staging area 128-byte aligned (tensor-copy destinations)
  double* stage = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(dsm) + 127) & ~static_cast<uintptr_t>(127));
  double* us = stage + kStageBufs * kStage;
  uint32_t ring = 0;  // stream-K ring: units consumed by this CTA (identical in every thread)
  if (p.tma) {
    sk_init_barriers();
    for (int g = blockIdx.x * kPT + threadIdx.x; g < 2 * static_cast<int>(gridDim.x); g += gridDim.x * kPT) p.flags[g] = 0;
  }
  int32_t* act = reinterpret_cast<int32_t*>(us + ld);
  int32_t* pact = act + B;
  int32_t* qord = pact + B;  // per-signal queue order: the FISTA slots first, then the power steps
  // ---- Engine ctor (254-276) with x = 0, S = K, cached full L: u = 0, momentum off
  for (int64_t b = blockIdx.x; b < B; b += gridDim.x) {
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < N; i += kPT) {
      const double yi = p.y[b * p.ldy + i];
      acc = fma(yi, yi, acc);
    }
    acc = block_sum(acc, sh);
    for (int64_t j = threadIdx.x; j < K; j += kPT) {
      p.X3[0][b * K + j] = 0.0;
      p.X3[1][b * K + j] = 0.0;
      p.mask[b * K + j] = 1;
      p.lead[b * K + j] = 0.0;
    }
    for (int64_t i = threadIdx.x; i < ld; i += kPT) {
      p.U2[0][b * ld + i] = 0.0;
      p.U2[1][b * ld + i] = 0.0;
    }
    if (threadIdx.x == 0) {
      PrefixSig s{};
      s.t_k = 1.0;
      s.y_sq = acc;
      s.S = K;
      s.active_at_last_l = K;
      s.lipschitz = p.lipschitz;
      s.inv_l = 1.0 / p.lipschitz;
      p.sig[b] = s;
    }
    __syncthreads();
    if (p.max_it == 0) finish_signal(p, sh, b, false, 0.0, t0);
    else compute_rho(p, sh, b);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    p.queue[0] = 0;
    p.queue[1] = 0;
  }
  grid.sync();
  int32_t steps = 0;
  int64_t work_act = 0, work_pow = 0;  // contraction widths summed over the steps (roofline accounting)
  for (;; ++steps) {
    // unfinished signals in signal order, and the ones in a power step (identical in every CTA)
    int n_act = 0, n_pow = 0, n_fista = 0;
    for (int64_t base = 0; base < B; base += kPT) {
      const int64_t b = base + threadIdx.x;
      const int mode = b < B ? __ldcg(&p.sig[b].mode) : 2;
      const bool on = mode == 0 || mode == 1;
      int at;
      const int na = block_compact(sh, on, n_act, &at);
      if (on) act[at] = static_cast<int32_t>(b);
      int atp;
      const int np = block_compact(sh, mode == 1, n_pow, &atp);
      if (mode == 1) pact[atp] = at;
      int atf;
      const int nf = block_compact(sh, mode == 0, n_fista, &atf);
      if (mode == 0) qord[atf] = at;
      n_act = na;
      n_pow = np;
      n_fista = nf;
    }
    // the power steps (~12 us on one CTA) queue behind the FISTA steps (~25-30 us at the full
    // set): longest first, so that the step's last CTA is not one that took a FISTA step late
    for (int i = threadIdx.x; i < n_pow; i += kPT) qord[n_fista + i] = pact[i];
    __syncthreads();
    if (n_act == 0) break;
    work_act += n_act;
    work_pow += n_pow;
    const bool logit = p.step_log && blockIdx.x == 0 && threadIdx.x == 0 && steps < p.max_log;
    if (logit) {
      p.step_log[kLogW * steps] = n_act;
      p.step_log[kLogW * steps + 1] = n_pow;
      p.step_log[kLogW * steps + 2] = gtimer() - t0;
    }
    const bool narrow = p.narrow && narrow_fits(n_act, ld);
    if (p.tma && !narrow) {
      // stage the contraction inputs in slot order (2D tensor boxes, no per-column gather):
      // Rc[a] = R[act[a]] (the power slots' columns are overwritten by W below) and
      // Vc[c] = v of power slot c
      sk_stage(p, n_act, n_pow, act, pact);
      // the staged columns are read by tensor copies (async proxy) after the barrier
      asm volatile("fence.proxy.async.global;" ::: "memory");
      grid.sync();
      if (logit) p.step_log[kLogW * steps + 5] = gtimer() - t0;
    }
    // ---- power-step signals: w = A_S v (one contraction), then summed into R
    if (n_pow > 0 && narrow) {
      narrow_w(p, n_pow, pact, act, stage);
      grid.sync();
      legacy_w_combine(p, n_pow, pact, act, kNarrowTag, kNarrowParts);
      grid.sync();
    } else if (n_pow > 0 && p.tma) {
      sk_contract(p, 0, n_pow, pact, stage, ring, 2 * steps + 1);  // writes the power slots' Rc columns
      if (logit) p.step_log[kLogW * steps + 6] = gtimer() - t0;
      grid.sync();
    } else if (n_pow > 0) {
      const int sk = legacy_w_tiles(p, n_pow, pact, act, stage);
      grid.sync();
      legacy_w_combine(p, n_pow, pact, act, sk, sk == kNarrowTag ? kNarrowParts : sk);
      grid.sync();
    }
    if (logit) p.step_log[kLogW * steps + 3] = gtimer() - t0;
    // ---- Corr = A^T [rho | w] for every unfinished signal (fp64 tensor cores; CUDA
    // cores when narrow)
    int sk = 1;
    if (narrow) {
      narrow_corr(p, n_act, act, stage);
    } else if (p.tma) {
      sk_contract(p, 1, n_act, pact, stage, ring, 2 * steps + 2);  // one part in p.corr
      if (logit) p.step_log[kLogW * steps + 7] = gtimer() - t0;
    } else {
      sk = legacy_corr_tiles(p, n_act, act, stage);
    }
    grid.sync();
    if (logit) p.step_log[kLogW * steps + 4] = gtimer() - t0;
    // ---- the rest of each signal's unit of work, one signal per CTA; CTAs take the
    // next signal from a counter (FISTA and power steps differ in cost), which the
    // result does not depend on. The other step's counter is reset for the next step
    // (its last users finished before this step's barriers).
    if (blockIdx.x == 0 && threadIdx.x == 0) p.queue[(steps + 1) & 1] = 0;
    for (;;) {
      if (threadIdx.x == 0) sh.qnext = atomicAdd(p.queue + (steps & 1), 1);
      __syncthreads();
      const int64_t qi = sh.qnext;
      __syncthreads();
      if (qi >= n_act) break;
      const int64_t a = qord[qi];
      const int64_t b = act[a];
      const int mode = __ldcg(&p.sig[b].mode);
      if (mode == 0) fista_step(p, sh, a, b, t0, sk, us, stage);
      else if (mode == 1) power_step(p, sh, a, b, sk, t0);
    }
    if (logit) p.step_log[kLogW * steps + 8] = gtimer() - t0;
    grid.sync();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && p.steps_out) *p.steps_out = steps;
  if (blockIdx.x == 0 && threadIdx.x == 0 && p.work_out) {
    p.work_out[0] = work_act;
    p.work_out[1] = work_pow;
  }
}


// ---------------------------------------------------------------------------
// C = X^T Y on the fp64 tensor cores: X is kdim x nx (leading dimension ldx), Y is
// kdim x ny (ldy), both column-major along the contraction with ldx, ldy even and zero
// padding past kdim (16-byte cp.async pairs); C is nx x ny (ldc). The same DMMA tiles
// as the lockstep contraction (128 x 64 outputs, 32-deep K chunks, cp.async double
// buffer). parts > 1 splits the contraction: part kp covers chunks [kp nch / parts,
// (kp + 1) nch / parts) and writes its partial tile to C + kp * pstride (summed in part
// order by parts_sum_kernel: deterministic).
// Users: the Gram matrix G = A^T A (RunOptions::exact_gram, bench.cpp:190-197; X = Y = A)
// and the randomized range finder of build_sukro_sequence (dictionary.cpp:253-279).
__global__ void __launch_bounds__(kPT, 1) gemm_tn_kernel(const double* __restrict__ X, int64_t ldx, int64_t nx,
                                                         const double* __restrict__ Y, int64_t ldy, int64_t ny,
                                                         int64_t kdim, int parts, double* __restrict__ C, int64_t ldc,
                                                         int64_t pstride) {
  extern __shared__ __align__(128) double dsm[];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, gi = l >> 2, tg = l & 3;
  const int wr = w % kWR, wc = w / kWR;
  const int n_rt = static_cast<int>((nx + kTM - 1) / kTM), n_ct = static_cast<int>((ny + kTN - 1) / kTN);
  const int nch = static_cast<int>((kdim + kTK - 1) / kTK);
  for (int item = blockIdx.x; item < n_rt * n_ct * parts; item += gridDim.x) {
    const int tile = item % (n_rt * n_ct), kp = item / (n_rt * n_ct);
    const int kc0 = static_cast<int>(static_cast<int64_t>(kp) * nch / parts);
    const int kc1 = static_cast<int>(static_cast<int64_t>(kp + 1) * nch / parts);
    const int64_t j0 = static_cast<int64_t>(tile % n_rt) * kTM, c0 = static_cast<int64_t>(tile / n_rt) * kTN;
    double acc[kRT][kCT][2];
#pragma unroll
    for (int h = 0; h < kRT; ++h)
#pragma unroll
      for (int c = 0; c < kCT; ++c) acc[h][c][0] = acc[h][c][1] = 0.0;
    auto issue = [&](int s, int kc) {
      double* As = dsm + s * kStage;
      double* Bs = As + kTM * kSS;
      const int64_t k0 = static_cast<int64_t>(kc) * kTK;
      for (int e = threadIdx.x; e < kTM * (kTK / 2); e += kPT) {
        const int r = e / (kTK / 2), kk = (e % (kTK / 2)) * 2;
        const bool ok = j0 + r < nx && k0 + kk < kdim;
        cp16(As + r * kSS + kk, ok ? X + (j0 + r) * ldx + k0 + kk : X, ok);
      }
      for (int e = threadIdx.x; e < kTN * (kTK / 2); e += kPT) {
        const int c = e / (kTK / 2), kk = (e % (kTK / 2)) * 2;
        const bool ok = c0 + c < ny && k0 + kk < kdim;
        cp16(Bs + c * kSS + kk, ok ? Y + (c0 + c) * ldy + k0 + kk : Y, ok);
      }
    };
    __syncthreads();
    if (kc0 < kc1) issue(0, kc0);
    cp_commit();
    for (int kc = kc0; kc < kc1; ++kc) {
      if (kc + 1 < kc1) issue((kc + 1 - kc0) & 1, kc + 1);
      cp_commit();
      cp_wait1();
      __syncthreads();
      const double* As = dsm + ((kc - kc0) & 1) * kStage;
      const double* Bs = As + kTM * kSS;
#pragma unroll
      for (int ks = 0; ks < kTK / 4; ++ks) {
        double av[kRT], bv[kCT];
#pragma unroll
        for (int h = 0; h < kRT; ++h) av[h] = As[((h * kWR + wr) * 8 + gi) * kSS + ks * 4 + tg];
#pragma unroll
        for (int c = 0; c < kCT; ++c) bv[c] = Bs[((wc * kCT + c) * 8 + gi) * kSS + ks * 4 + tg];
#pragma unroll
        for (int h = 0; h < kRT; ++h)
#pragma unroll
          for (int c = 0; c < kCT; ++c) dmma(acc[h][c], av[h], bv[c]);
      }
      __syncthreads();
    }
    cp_wait0();
    double* out = C + static_cast<int64_t>(kp) * pstride;
#pragma unroll
    for (int h = 0; h < kRT; ++h) {
      const int64_t i = j0 + (h * kWR + wr) * 8 + gi;
#pragma unroll
      for (int c = 0; c < kCT; ++c)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int64_t j = c0 + (wc * kCT + c) * 8 + 2 * tg + q;
          if (i < nx && j < ny) out[j * ldc + i] = acc[h][c][q];
        }
    }
  }
}

// C(i, j) = sum over parts kp (in order) of P[kp * pstride + j * ldc + i]
__global__ void parts_sum_kernel(const double* __restrict__ P, int parts, int64_t pstride, int64_t rows, int64_t cols,
                                 int64_t ldc, double* __restrict__ C) {
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < rows * cols;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = e / rows, i = e - j * rows;
    double s = 0.0;
    for (int kp = 0; kp < parts; ++kp) s += P[kp * pstride + j * ldc + i];
    C[j * ldc + i] = s;
  }
}

// column 2-norms of a column-major k x k matrix (one warp per column, fixed order)
__global__ void colnorm_kernel(const double* __restrict__ g, int64_t k, int64_t ldg, double* __restrict__ out) {
  const int64_t col = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int l = threadIdx.x & 31;
  if (col >= k) return;
  double s = 0.0;
  for (int64_t i = l; i < k; i += 32) {
    const double v = g[col * ldg + i];
    s = fma(v, v, s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(kAll, s, o);
  if (l == 0) out[col] = sqrt(s);
}

cudaError_t colnorm_launch(const double* g, int64_t k, int64_t ldg, double* out, cudaStream_t stream) {
  const int64_t threads = k * 32;
  colnorm_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, stream>>>(g, k, ldg, out);
  return cudaGetLastError();
}

cudaError_t gram_launch(const double* a, int64_t ld, int64_t k, double* g, int64_t ldg, int device,
                        cudaStream_t stream) {
  return gemm_tn_launch(a, ld, k, a, ld, k, ld, g, ldg, nullptr, 0, device, stream);
}

// C = X^T Y (see gemm_tn_kernel). The contraction is split when the output has fewer
// tiles than the device has SMs (tall-skinny products): parts from the fewest-waves rule,
// each at least 4 chunks deep, partials in `work` (parts * ldc * ny doubles; without
// enough work space the product is not split).
cudaError_t gemm_tn_launch(const double* X, int64_t ldx, int64_t nx, const double* Y, int64_t ldy, int64_t ny,
                           int64_t kdim, double* C, int64_t ldc, double* work, size_t work_elems, int device,
                           cudaStream_t stream) {
  const size_t smem = static_cast<size_t>(2 * kStage) * sizeof(double);
  cudaError_t e =
      cudaFuncSetAttribute(gemm_tn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int sms = 0;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) return e;
  const int64_t tiles = ((nx + kTM - 1) / kTM) * ((ny + kTN - 1) / kTN);
  const int64_t nch = (kdim + kTK - 1) / kTK;
  int parts = 1;
  if (work && tiles < sms) {
    parts = static_cast<int>(std::min<int64_t>({static_cast<int64_t>(kSplitMax), (sms + tiles - 1) / tiles,
                                                std::max<int64_t>(1, nch / 4)}));
    if (static_cast<size_t>(parts) * static_cast<size_t>(ldc) * static_cast<size_t>(ny) > work_elems) parts = 1;
  }
  const int64_t items = tiles * parts;
  const unsigned grid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(items, 4 * sms)));
  if (parts == 1) {
    gemm_tn_kernel<<<grid, kPT, smem, stream>>>(X, ldx, nx, Y, ldy, ny, kdim, 1, C, ldc, 0);
    return cudaGetLastError();
  }
  const int64_t pstride = ldc * ny;
  gemm_tn_kernel<<<grid, kPT, smem, stream>>>(X, ldx, nx, Y, ldy, ny, kdim, parts, work, ldc, pstride);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int64_t n = nx * ny;
  parts_sum_kernel<<<static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 4 * sms)), 256, 0, stream>>>(
      work, parts, pstride, nx, ny, ldc, C);
  return cudaGetLastError();
}

size_t prefix_smem_bytes(int64_t ld, int64_t batch) {
  return 128 + static_cast<size_t>(kStageBufs * kStage + ld) * sizeof(double) +
         static_cast<size_t>(3 * batch) * sizeof(int32_t);
}
int64_t prefix_part_elems(int grid) { return 2 * static_cast<int64_t>(grid) * kPartTile; }
int prefix_stream_k_max_grid() { return kMaxGrid; }
int prefix_split_max() { return kSplitMax; }
// the per-signal lists live in the staging area: two atom lists (12 bytes per entry each)
// and the flattened copy the apply walks (12 more): 36 bytes per atom
int64_t prefix_max_atoms() { return (static_cast<int64_t>(kStageBufs) * kStage * 8) / 36 / kPW * kPW; }

// the lockstep's shared memory (staging, u, three per-signal index lists) fits one CTA
bool prefix_fits(int64_t ld, int64_t batch, int device) {
  int optin = 0;
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device) != cudaSuccess) return false;
  cudaFuncAttributes fa{};
  if (cudaFuncGetAttributes(&fa, prefix_kernel) != cudaSuccess) return false;
  return prefix_smem_bytes(ld, batch) + fa.sharedSizeBytes <= static_cast<size_t>(optin);
}

cudaError_t prefix_launch(const PrefixParams& p, int device, cudaStream_t stream) {
  const size_t smem = prefix_smem_bytes(p.ld, p.batch);
  int optin = 0;
  cudaError_t e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  if (e != cudaSuccess) return e;
  cudaFuncAttributes fa{};
  e = cudaFuncGetAttributes(&fa, prefix_kernel);
  if (e != cudaSuccess) return e;
  if (smem + fa.sharedSizeBytes > static_cast<size_t>(optin)) return cudaErrorInvalidConfiguration;
  e = cudaFuncSetAttribute(prefix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int per_sm = 0, sms = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, prefix_kernel, kPT, smem);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  PrefixParams local = p;
  void* args[] = {&local};
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(prefix_kernel), dim3(sms), dim3(kPT), args, smem,
                                     stream);
}

// Batched traces: signal b's rows [b * cap, b * cap + n_b) packed to [off[b], off[b+1]).
__global__ void trace_pack_kernel(const fl1_trace_row* __restrict__ src, int64_t cap, const int64_t* __restrict__ off,
                                  int32_t batch, fl1_trace_row* __restrict__ dst) {
  for (int32_t b = blockIdx.x; b < batch; b += gridDim.x) {
    const int64_t o = off[b], n = off[b + 1] - o;
    const fl1_trace_row* s = src + static_cast<int64_t>(b) * cap;
    for (int64_t r = threadIdx.x; r < n; r += blockDim.x) dst[o + r] = s[r];
  }
}

cudaError_t trace_pack_launch(const fl1_trace_row* src, int64_t cap, const int64_t* off, int32_t batch,
                              fl1_trace_row* dst, cudaStream_t stream) {
  if (batch <= 0) return cudaSuccess;
  trace_pack_kernel<<<std::min<int32_t>(batch, 1024), 128, 0, stream>>>(src, cap, off, batch, dst);
  return cudaGetLastError();
}

}  // namespace fl1
