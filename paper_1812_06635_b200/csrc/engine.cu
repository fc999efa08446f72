// engine.cu — the FastL1 iteration loop as ONE persistent cooperative kernel.
//
// Reference path replaced: Engine::run and everything it calls per iteration
// (fastl1.cpp:459-645): compute_products (359-394), dual_scalars/dual_of
// (406-457), the GAP / Dynamic sphere tests (494-566, screening.cpp:103-106,
// 136-150), the switching rule (26-38, 556-565), the prox / FISTA update
// (572-591, solver.cpp:9-13), apply_restriction + ActiveOp compaction
// (667-702, 115-129, 176-201), ActiveOp::apply / apply_adjoint for dense and
// SuKro operators (131-161, dictionary.cpp:150-164), the restricted power
// iteration (326-333, solver.cpp:72-104) and the ledger / trace (611-623).
//
// Layout: one CTA of 512 threads per SM, launched cooperatively. One
// iteration is four grid-wide phases separated by grid.sync():
//   A  rho_g = y - ((1+m)u - m v) built redundantly in every CTA's shared
//      memory; A_S^T rho_g streams every preserved column ONCE: each CTA owns
//      a contiguous column range, each warp a contiguous range of 4 KiB units
//      inside it, loads are 128-bit and software-pipelined one unit ahead, the
//      dot is a warp-shuffle reduction, and columns split between warps are
//      merged in shared memory in warp order. The pass also emits the per-CTA
//      maxima of |corr_j| and |corr_j| + eps_j ||rho_g|| (dual scaling).
//   B  every CTA reduces the per-CTA partials in the same fixed order, so all
//      CTAs hold bit-identical scales, gaps, stop / screen / switch decisions;
//      per-atom sphere test, soft-threshold and FISTA update on a CTA slice.
//   D  stream compaction of the preserved set into the other bank; the
//      sparse apply u = A_S x as (row tile x position chunk) partials plus the
//      v-history fix for dropped atoms; ledger + trace row.
//   E  partials combined by row slices into u (and v <- u_old - fix).
// Restricted power iterations (halvings) and dictionary switches run in the
// same kernel. No reduction uses floating-point atomics: every sum has a
// fixed order, so a solve is bit-reproducible on a given device.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <math_constants.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "engine.cuh"

namespace cg = cooperative_groups;

// The engine is compiled twice (build.py). FL1_FUSED_VARIANT=1 adds the single-read power
// steps (dense_fused_power_pass) and exports every entry point with an _fp suffix; api.cpp
// launches that instance only for dictionaries the pass applies to (4096 < N <= 8192, beyond
// L2). The default instance does not contain the pass: its register allocation, and with it
// the latency-bound phases of every other configuration, is unchanged by it.
#ifndef FL1_FUSED_VARIANT
#define FL1_FUSED_VARIANT 0
#endif
#if FL1_FUSED_VARIANT
#define FL1_ANON fpv
#define engine_kernel engine_kernel_fp
#define engine_body engine_body_fp
#define engine_smem_bytes engine_smem_bytes_fp
#define engine_scratch_len engine_scratch_len_fp
#define engine_bulk_stages engine_bulk_stages_fp
#define engine_configure engine_configure_fp
#define engine_launch engine_launch_fp
#define engine_cluster_capacity engine_cluster_capacity_fp
#define engine_launch_clusters engine_launch_clusters_fp
#define screen_kernel screen_kernel_fp
#define screen_kernel_launch screen_kernel_launch_fp
namespace fl1 {
namespace fpv {}
using namespace fpv;
}  // namespace fl1
#else
#define FL1_ANON
#endif

namespace fl1 {
namespace FL1_ANON {

constexpr unsigned kFull = 0xffffffffu;

// FL1_TIMELINE builds record, per iteration (< 4096) and per CTA, %globaltimer at
// 8 points (phase boundaries before / after each grid sync) into p.timeline.
#ifndef FL1_TIMELINE
#define FL1_TIMELINE 0
#endif
#if FL1_TIMELINE
#define FL1_MARK(pt)                                                                                      \
  do {                                                                                                    \
    if (threadIdx.x == 0 && s.t < 4096 && p.timeline) {                                                   \
      uint64_t t_;                                                                                        \
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_));                                              \
      p.timeline[(static_cast<int64_t>(s.t) * vsize() + vrank()) * 8 + (pt)] = t_;                  \
    }                                                                                                     \
  } while (0)
#else
#define FL1_MARK(pt) \
  do {               \
  } while (0)
#endif
constexpr int64_t kRedundantCombine = 8192;  // doubles of partials each CTA may re-sum instead of a sync

// per-CTA partial slots (bred[cta * kBred + slot])
enum Slot {
  kSlMaxPlain = 0,
  kSlMaxStable = 1,
  kSlL1 = 2,
  kSlKept = 3,
  kSlLook = 4,
  kSlNnz = 5,
  kSlMaxEps = 6,
  kSlPw2 = 7,
  kSlPvw = 8,
  kSlSum = 9,
  kSlMaxPlainY = 10,
  kSlMaxStableY = 11,
  kSlLead2 = 12,
  kSlRhoSq = 13,   // ||rho_g||^2 partials (written by the combine phase)
  kSlRhoY = 14,    // rho_g . y
  kSlRhoE = 15,    // ||y - u||^2 (momentum != 0)
};
// ||x||_1 partials for iteration t live in kSlL1 (t even) / kSlL1b (t odd); written
// by phase B of iteration t-1 (over the kept new iterate) or by the constructor.
constexpr int kSlL1b = 16;
constexpr int kSlGwa = 17;   // Gram mode: w . A^T y   (w = extrapolated x)
constexpr int kSlGwg = 18;   //            w . G w
constexpr int kSlGxa = 19;   //            x . A^T y
constexpr int kSlGxg = 20;   //            x . G x
constexpr int kSlNnzX = 21;  // early prox: nnz of the current x (the ledger row if the iteration stops)

// Virtual grid: the engine runs either on the whole GPU (one cooperative launch,
// grid-wide barrier) or inside one thread-block cluster per solve (batched mode,
// cluster barrier). Every slice / work partition / barrier below goes through these.
__shared__ int s_vsize;     // CTAs of the virtual grid
__shared__ int s_vrank;     // this CTA's rank in it
__shared__ int s_vcluster;  // 1: cluster mode

// Bulk-copy (TMA 1D) streaming ring of the dense adjoint pass: per warp up to
// kMaxBulk 4 KiB stages in shared memory, one mbarrier each; phase bits persist
// across passes (and across solves of a cluster).
constexpr int kMaxBulk = 6;
__shared__ __align__(8) uint64_t s_bar[FL1_THREADS / 32 * kMaxBulk];
__shared__ uint32_t s_bphase[FL1_THREADS / 32];
__device__ __forceinline__ uint32_t smem_u32(const void* ptr) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(ptr));
}
__device__ __forceinline__ void bulk_init_barriers() {
  if ((threadIdx.x & 31) == 0) {
    const int w = threadIdx.x >> 5;
    for (int s = 0; s < kMaxBulk; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&s_bar[w * kMaxBulk + s])));
    s_bphase[w] = 0u;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
// Per-CTA column results of a dense adjoint pass (merge + statistics stay on chip
// when the CTA's slice has at most kColBuf columns).
constexpr int kColBuf = 512;  // 4 KiB: keeps c2's shared memory under the 100 KiB carve-out (more L1)
__shared__ double s_colsum[kColBuf];
// early prox: each thread's first atom of the slice, staged during the pass
__shared__ double s_ex[FL1_THREADS];
__shared__ double s_exp[FL1_THREADS];
__shared__ int32_t s_eidx[FL1_THREADS];
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ int vsize() { return s_vsize; }
__device__ __forceinline__ int vrank() { return s_vrank; }
__device__ __forceinline__ void vsync() {
  if (s_vcluster)
    cg::this_cluster().sync();
  else
    cg::this_grid().sync();
}

struct Frag {
  int64_t pos;
  double sum;
};

struct Sh {
  EngineState s;
  double red[kWarps * 8];
  double res[kBred];
  // per-iteration scalars (identical in every CTA)
  double t_next;
  double rho_sq, rho_dot_y, rho_x_sq, rho_norm;
  double scale_prime, scale_tilde, ray_sq, ray_dot_y;
  double gap_prime, gap_tilde, primal, x_l1;
  double radius, center_norm, gamma;
  int ray_is_y, stop_now, screen_now, stable_test, next_dict, speed;
  int64_t S_new, look, nnz;
  int64_t scan_base;
  int32_t wscan[kWarps];
  int32_t wcount[2][kWarps];
  Frag frag[kWarps][2];
  int32_t nfrag[kWarps];
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(kFull, v, o);
  return v;  // valid in lane 0
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(kFull, v, o));
  return v;
}

// Deterministic block reduction of up to 4 values (sum or max per value).
template <int NV>
__device__ void block_reduce(double (&v)[NV], const bool (&is_max)[NV], Sh& sh) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < NV; ++q) v[q] = is_max[q] ? warp_max(v[q]) : warp_sum(v[q]);
  __syncthreads();
  if (l == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) sh.red[q * kWarps + w] = v[q];
  }
  __syncthreads();
  if (w == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double r = l < kWarps ? sh.red[q * kWarps + l] : (is_max[q] ? -DBL_MAX : 0.0);
      r = is_max[q] ? warp_max(r) : warp_sum(r);
      if (l == 0) sh.red[q * kWarps] = r;
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NV; ++q) v[q] = sh.red[q * kWarps];
  __syncthreads();
}

// Reduce per-CTA partial slots in a fixed order; warp `slot` handles one slot.
__device__ void grid_reduce(const EngineParams& p, Sh& sh, unsigned mask_sum, unsigned mask_max) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int slot = w; slot < kBred; slot += kWarps) {
    if (!(((mask_sum | mask_max) >> slot) & 1u)) continue;
    const bool mx = (mask_max >> slot) & 1u;
    double acc = mx ? -DBL_MAX : 0.0;
    if (p.grid <= 32) {  // one partial per lane (cluster mode)
      if (l < p.grid) acc = __ldcg(p.bred + static_cast<int64_t>(l) * kBred + slot);
    } else
    for (int b0 = l; b0 < p.grid; b0 += 256) {  // 8 loads in flight per lane, added in b order
      double e[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int b = b0 + 32 * q;
        e[q] = b < p.grid ? __ldcg(p.bred + static_cast<int64_t>(b) * kBred + slot) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (b0 + 32 * q < p.grid) acc = mx ? fmax(acc, e[q]) : acc + e[q];
    }
    acc = mx ? warp_max(acc) : warp_sum(acc);
    if (l == 0) sh.res[slot] = acc;
  }
  __syncthreads();
}

__device__ __forceinline__ void put_slot(const EngineParams& p, int slot, double v) {
  __stcg(p.bred + static_cast<int64_t>(vrank()) * kBred + slot, v);
}

__device__ __forceinline__ double2 ldg_stream2(const double2* ptr) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(ptr));
  return r;
}

// CTA slice [lo, hi) of n items (balanced, contiguous).
__device__ __forceinline__ void slice(int64_t n, int64_t& lo, int64_t& hi) {
  lo = n * vrank() / vsize();
  hi = n * (vrank() + 1) / vsize();
}

__device__ __forceinline__ double globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return static_cast<double>(t);
}

// Fixed-order sums of apply partials: sum_{c < C} part[c * ld + i].
// Few chunks: one thread per row, all C loads in flight, added in c order.
// Many chunks: one warp per row, lane l adds chunks l, l+32, ..., then a fixed
// shuffle tree. Either way the order depends only on C.
constexpr int kThreadCombineMax = 16;

__device__ __forceinline__ double thread_sum_partials(const double* __restrict__ part, int C, int64_t ld, int64_t i) {
  double v[kThreadCombineMax];
#pragma unroll
  for (int c = 0; c < kThreadCombineMax; ++c) v[c] = c < C ? __ldcg(part + static_cast<int64_t>(c) * ld + i) : 0.0;
  double acc = 0.0;
#pragma unroll
  for (int c = 0; c < kThreadCombineMax; ++c)
    if (c < C) acc += v[c];
  return acc;
}

// Lane g of an 8-lane row group: sum of part[c * ld + i] over c = g, g + 8, ... < C
// in that order, with up to 8 loads in flight (not one L2 round trip per chunk).
__device__ __forceinline__ double lane_sum_partials(const double* __restrict__ part, int C, int64_t ld, int64_t i,
                                                    int g) {
  double acc = 0.0;
  for (int c0 = g; c0 < C; c0 += 64) {
    double v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int c = c0 + 8 * q;
      v[q] = c < C ? __ldcg(part + static_cast<int64_t>(c) * ld + i) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (c0 + 8 * q < C) acc += v[q];
  }
  return acc;
}

// Calls f(i, value) for rows i in [lo, hi) (by one thread per row).
// Few chunks: one thread per row with every load in flight. More: 8 lanes per
// row (lane g adds chunks g, g+8, ...; a fixed 3-step shuffle tree), so 32 rows
// are combined per 256-thread pass with ~C/8 loads in flight per lane.
template <class Fn>
__device__ __forceinline__ void combine_rows(const double* __restrict__ part, int C, int64_t ld, int64_t lo, int64_t hi,
                                             Fn&& f) {
  if (C <= kThreadCombineMax) {
    for (int64_t i = lo + threadIdx.x; i < hi; i += kThreads) f(i, thread_sum_partials(part, C, ld, i));
  } else {
    const int g = threadIdx.x & 7;
    for (int64_t i0 = lo; i0 < hi; i0 += kThreads / 8) {  // uniform trip count (shuffles below)
      const int64_t i = i0 + (threadIdx.x >> 3);
      double acc = 0.0;
      if (i < hi) acc = lane_sum_partials(part, C, ld, i, g);
      acc += __shfl_xor_sync(kFull, acc, 4);
      acc += __shfl_xor_sync(kFull, acc, 2);
      acc += __shfl_xor_sync(kFull, acc, 1);
      if (g == 0 && i < hi) f(i, acc);
    }
  }
}

// dst[0:ld) = src[0:ld) with 128-bit loads, 4 in flight per thread (ld is even).
__device__ __forceinline__ void load_vec_smem(const EngineParams& p, const double* src, double* dst) {
  const int64_t n2 = p.ld >> 1;
  const double2* __restrict__ s2 = reinterpret_cast<const double2*>(src);
  double2* d2 = reinterpret_cast<double2*>(dst);
  for (int64_t i0 = threadIdx.x; i0 < n2; i0 += 4 * kThreads) {
    double2 v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t i = i0 + q * kThreads;
      v[q] = i < n2 ? __ldcg(s2 + i) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t i = i0 + q * kThreads;
      if (i < n2) d2[i] = v[q];
    }
  }
  __syncthreads();
}

// What an adjoint pass emits besides out[pos].
struct PassOut {
  double* out;
  int track;             // per-CTA maxima of |out| and |out| + eps*eps_scale
  double eps_scale;
  bool div_lambda;       // maxima of |out|/lambda (exact-fit branch, fastl1.cpp:440-446)
  int slot_plain, slot_stable;
  const double* vdot;    // non-null: per-CTA sums of out^2 and vdot*out (power iteration)
  int bulk;              // stream through the bulk-copy ring (p.bulk_stages > 0; power iterations)
};

struct PassAcc {
  double mp = 0.0, ms = 0.0, w2 = 0.0, vw = 0.0;
  __device__ __forceinline__ void add(const EngineParams& p, const PassOut& po, const double* eps, int64_t pos,
                                      double total, bool store = false) {
    if (store) __stcg(po.out + pos, total);
    if (po.track) {
      const double ac = po.div_lambda ? fabs(total) / p.lambda : fabs(total);
      mp = fmax(mp, ac);
      ms = fmax(ms, ac + eps[pos] * po.eps_scale);
    }
    if (po.vdot) {
      w2 = fma(total, total, w2);
      vw = fma(po.vdot[pos], total, vw);
    }
  }
};

__device__ void finish_pass(const EngineParams& p, Sh& sh, const PassOut& po, PassAcc& acc) {
  if (po.track) {
    double v[2] = {acc.mp, acc.ms};
    const bool mx[2] = {true, true};
    block_reduce<2>(v, mx, sh);
    if (threadIdx.x == 0) {
      put_slot(p, po.slot_plain, v[0]);
      put_slot(p, po.slot_stable, v[1]);
    }
  }
  if (po.vdot) {
    double v[2] = {acc.w2, acc.vw};
    const bool mx[2] = {false, false};
    block_reduce<2>(v, mx, sh);
    if (threadIdx.x == 0) {
      put_slot(p, kSlPw2, v[0]);
      put_slot(p, kSlPvw, v[1]);
    }
  }
}

// ----------------------------------------------------------------------------
// Dense adjoint over the preserved columns: out[pos] = a_{idx[pos]} . r, with
// r (length ld, zero padded) in shared memory (ActiveOp::apply_adjoint 148-161).
// ----------------------------------------------------------------------------
__device__ __noinline__ void dense_adjoint(const EngineParams& p, Sh& sh, const DevLevel& lv,
                                           const int32_t* __restrict__ idx, const double* __restrict__ eps, int64_t S,
                                           const double* __restrict__ r, double* __restrict__ ring,
                                           const PassOut& po) {
  const int64_t n = p.n;
  const int U = static_cast<int>((n + kUnit - 1) / kUnit);
  const int last_nd2 = static_cast<int>(((n - static_cast<int64_t>(U - 1) * kUnit) + 1) >> 1);
  const int64_t ld2 = p.ld >> 1;
  int64_t c0, c1;
  slice(S, c0, c1);
  const int Ub = static_cast<int>((c1 - c0) * U);  // units of this CTA (< 2^31 by construction)
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int u_lo = static_cast<int>(static_cast<int64_t>(Ub) * w / kWarps);
  const int u_hi = static_cast<int>(static_cast<int64_t>(Ub) * (w + 1) / kWarps);
  const double2* __restrict__ A2 = reinterpret_cast<const double2*>(lv.a) + l;
  const double2* __restrict__ r2 = reinterpret_cast<const double2*>(r) + l;
  double* __restrict__ out = po.out;
  const bool on_chip = c1 - c0 <= kColBuf;
  double* __restrict__ dst = on_chip ? s_colsum : out + c0;  // column results, relative to c0
  PassAcc acc;
  int nf = 0;
  // Units are visited in order; three register buffers form a ring so two
  // units' 128-bit loads are in flight while the current unit is reduced.
  // (ic, ih) is the column / unit of the next unit to issue, (cc, ch) of the
  // next unit to consume: incremented, never divided.
  constexpr int kV = kUnit / 64;  // double2 loads per lane per unit
  double s = 0.0;
  bool began_here = (u_lo % U) == 0;
  int ic = (U == 0) ? 0 : u_lo / U, ih = u_lo - ic * U;
  int cc = ic, ch = ih;
  const double2* colp = nullptr;
  int colp_c = -1;
#define FL1_ISSUE(B)                                                                                  \
  do {                                                                                                \
    if (ic != colp_c) {                                                                               \
      colp = A2 + static_cast<int64_t>(__ldg(idx + c0 + ic)) * ld2;                                   \
      colp_c = ic;                                                                                    \
    }                                                                                                 \
    const double2* src_ = colp + ih * (kUnit / 2);                                                    \
    const int lim_ = (ih == U - 1 ? last_nd2 : kUnit / 2) - l; /* branch-free: predicated loads */    \
    _Pragma("unroll") for (int q = 0; q < kV; ++q) B[q] =                                             \
        (32 * q < lim_) ? ldg_stream2(src_ + 32 * q) : make_double2(0.0, 0.0);                       \
    if (++ih == U) {                                                                                  \
      ih = 0;                                                                                         \
      ++ic;                                                                                           \
    }                                                                                                 \
  } while (0)
#define FL1_RV(q) rr_[32 * q]
#define FL1_CONSUME(B, U_)                                                                            \
  do {                                                                                                \
    const double2* rr_ = r2 + ch * (kUnit / 2);                                                       \
    _Pragma("unroll") for (int q = 0; q < kV; ++q) {                                                  \
      const double2 rv_ = FL1_RV(q);                                                                  \
      s = fma(B[q].x, rv_.x, s);                                                                      \
      s = fma(B[q].y, rv_.y, s);                                                                      \
    }                                                                                                 \
    const bool col_end_ = ch == U - 1;                                                                \
    if (col_end_ || (U_) + 1 == u_hi) {                                                               \
      const double t_ = warp_sum(s);                                                                  \
      const bool whole_ = col_end_ && began_here;                                                     \
      if (l == 0) {                                                                                   \
        if (whole_) {                                                                                 \
          dst[cc] = t_;                                                                               \
        } else {                                                                                      \
          sh.frag[w][nf].pos = c0 + cc;                                                               \
          sh.frag[w][nf].sum = t_;                                                                    \
        }                                                                                             \
      }                                                                                               \
      if (!whole_) ++nf;                                                                              \
      s = 0.0;                                                                                        \
      began_here = true;                                                                              \
    }                                                                                                 \
    if (++ch == U) {                                                                                  \
      ch = 0;                                                                                         \
      ++cc;                                                                                           \
    }                                                                                                 \
  } while (0)
  if (u_lo < u_hi && po.bulk && !s_vcluster && p.bulk_stages >= 2) {
    // bulk-copy ring: lane 0 streams whole units into shared memory (one mbarrier per
    // stage), so R units per warp are in flight instead of two register units
    const int R = p.bulk_stages;
    double2* wring = reinterpret_cast<double2*>(ring) + static_cast<int64_t>(w) * R * (kUnit / 2);
    uint64_t* bars = &s_bar[w * kMaxBulk];
    uint32_t ph = s_bphase[w];
    const double* __restrict__ A = lv.a;
    auto bulk_issue = [&](int st) {
      if (l == 0) {
        const double* src = A + static_cast<int64_t>(__ldg(idx + c0 + ic)) * p.ld + static_cast<int64_t>(ih) * kUnit;
        const uint32_t bytes =
            static_cast<uint32_t>(((ih == U - 1) ? (p.ld - static_cast<int64_t>(ih) * kUnit) : kUnit) * 8);
        bulk_load(wring + st * (kUnit / 2), src, bytes, bars + st);
      }
      if (++ih == U) {
        ih = 0;
        ++ic;
      }
    };
    int iu = u_lo;
    for (int st = 0; st < R && iu < u_hi; ++st, ++iu) bulk_issue(st);
    int st = 0;
    for (int u = u_lo; u < u_hi; ++u) {
      bulk_wait(bars + st, (ph >> st) & 1u);
      ph ^= 1u << st;
      double2 b0[kV];
      const double2* sp = wring + st * (kUnit / 2) + l;
      const int lim = (ch == U - 1 ? last_nd2 : kUnit / 2) - l;
#pragma unroll
      for (int q = 0; q < kV; ++q) b0[q] = (32 * q < lim) ? sp[32 * q] : make_double2(0.0, 0.0);
      __syncwarp();
      if (iu < u_hi) {
        bulk_issue(st);
        ++iu;
      }
      FL1_CONSUME(b0, u);
      if (++st == R) st = 0;
    }
    if (l == 0) s_bphase[w] = ph;
  } else if (u_lo < u_hi) {
#if FL1_RING == 3
    double2 b0[kV], b1[kV], b2[kV];
    FL1_ISSUE(b0);
    if (u_lo + 1 < u_hi) FL1_ISSUE(b1);
    int u = u_lo;
    while (true) {
      if (u + 2 < u_hi) FL1_ISSUE(b2);
      FL1_CONSUME(b0, u);
      if (++u >= u_hi) break;
      if (u + 2 < u_hi) FL1_ISSUE(b0);
      FL1_CONSUME(b1, u);
      if (++u >= u_hi) break;
      if (u + 2 < u_hi) FL1_ISSUE(b1);
      FL1_CONSUME(b2, u);
      if (++u >= u_hi) break;
    }
#else
    double2 b0[kV], b1[kV];
    FL1_ISSUE(b0);
    int u = u_lo;
    while (true) {
      if (u + 1 < u_hi) FL1_ISSUE(b1);
      FL1_CONSUME(b0, u);
      if (++u >= u_hi) break;
      if (u + 1 < u_hi) FL1_ISSUE(b0);
      FL1_CONSUME(b1, u);
      if (++u >= u_hi) break;
    }
#endif
  }
#undef FL1_ISSUE
#undef FL1_CONSUME
#undef FL1_RV
  if (l == 0) sh.nfrag[w] = nf;
  __syncthreads();
  // merge columns split between warps, in warp (= unit) order: the fragments, in
  // (warp, slot) order, are sorted by column; the first fragment of each column sums
  // its run left to right (the order of a serial merge), one thread per fragment
  if (threadIdx.x < 2 * kWarps) {
    const int ww = threadIdx.x >> 1, f = threadIdx.x & 1;
    if (f < sh.nfrag[ww]) {
      const Frag fr = sh.frag[ww][f];
      bool head = true;
      for (int k = 2 * ww + f - 1; k >= 0; --k)
        if ((k & 1) < sh.nfrag[k >> 1]) {
          head = sh.frag[k >> 1][k & 1].pos != fr.pos;
          break;
        }
      if (head) {
        double cs = fr.sum;
        for (int k = 2 * ww + f + 1; k < 2 * kWarps; ++k) {
          if ((k & 1) >= sh.nfrag[k >> 1]) continue;
          const Frag nx = sh.frag[k >> 1][k & 1];
          if (nx.pos != fr.pos) break;
          cs += nx.sum;
        }
        dst[fr.pos - c0] = cs;
      }
    }
  }
  __syncthreads();
  // per-CTA statistics over this CTA's columns (fixed thread -> position map); a
  // separate short pass is cheaper than statistics inside the streaming loop
  if (on_chip) {
    for (int64_t pos = c0 + threadIdx.x; pos < c1; pos += kThreads) {
      const double v = s_colsum[pos - c0];
      out[pos] = v;
      if (po.track || po.vdot) acc.add(p, po, eps, pos, v);
    }
  } else if (po.track || po.vdot) {
    for (int64_t pos = c0 + threadIdx.x; pos < c1; pos += kThreads) acc.add(p, po, eps, pos, out[pos]);
  }
  finish_pass(p, sh, po, acc);
  __syncthreads();  // sh.frag is reused by the next pass
}

// ----------------------------------------------------------------------------
// fp64 tensor-core MMA (DMMA): D(8x8) += A(8x4, row) B(4x8, col). Fragments:
// a = A[g][t], b = B[t][g], c[i] = D[g][2t+i] with g = lane/4, t = lane%4.
// ----------------------------------------------------------------------------
__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// ----------------------------------------------------------------------------
// SuKro adjoint (SukroDictionary::apply_adjoint, dictionary.cpp:158-164, then the
// ActiveOp gather 157-160): out[pos] = d_j * Z(s, jj), j = idx[pos] = jj*q + s,
// Z = sum_t C_t^T R B_t (q x q), R = reshape(r, m, m) resident in shared memory.
// Each CTA owns (8 columns jj) x (SB rows s) tiles of Z and needs no other CTA:
//   V_t = R B_t(:, jj-block)          (m x 8, DMMA, K = m)
//   Z  += C_t(:, s-block)^T V_t       (SB x 8, DMMA, K = m; split-K over warps)
// Z goes to HBM/L2, one virtual-grid barrier, then every CTA gathers its own
// slice of preserved positions with the pass statistics.
// ----------------------------------------------------------------------------
__device__ __noinline__ void sukro_adjoint(const EngineParams& p, Sh& sh, const DevLevel& lv, const int32_t* __restrict__ idx,
                              const double* __restrict__ eps, int64_t S, const double* __restrict__ r,
                              double* __restrict__ scratch, const PassOut& po) {
  const int m = static_cast<int>(lv.m), q = static_cast<int>(lv.q);
  const int nt = lv.nterms;
  const int64_t mq = static_cast<int64_t>(m) * q;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, g = l >> 2, tg = l & 3;
  const int m4 = (m + 3) & ~3, mt = (m + 7) >> 3, ks_n = m4 >> 2;
  const int q8 = (q + 7) >> 3, n_jb = q8;
  int n_sb = vsize() / n_jb;
  n_sb = max(n_sb, (q8 + 3) / 4);
  n_sb = min(n_sb, q8);
  int sb8 = (q8 + n_sb - 1) / n_sb;  // 8-row tiles per s-block: 1, 2 or 4
  if (sb8 == 3) sb8 = 4;
  n_sb = (q8 + sb8 - 1) / sb8;
  const int SB = sb8 * 8, ksplit = 8 / sb8;
  const int my_mt = w % sb8, kpart = w / sb8;
  const int k_lo = ks_n * kpart / ksplit, k_hi = ks_n * (kpart + 1) / ksplit;
  // per term: B block (m4 x 8), V (m4 x 8), C block (SB x (m4+1)); as many terms
  // per staging round as the scratch holds (one load latency per round)
  const int per_term = 16 * m4 + SB * (m4 + 1);
  const int G = max(1, min(nt, static_cast<int>((p.scratch_len - kWarps * 64) / per_term)));
  double* Red = scratch;                // split-K partials: kWarps x 64
  double* Z = p.sk_z;
  const int tiles = n_jb * n_sb;
  for (int tile = vrank(); tile < tiles; tile += vsize()) {
    const int jj0 = (tile % n_jb) * 8, s0 = (tile / n_jb) * SB;
    double acc[2] = {0.0, 0.0};
    for (int t0 = 0; t0 < nt; t0 += G) {
      const int gn = min(G, nt - t0);
      __syncthreads();  // previous users of the staging area are done
      for (int e = threadIdx.x; e < gn * 8 * m4; e += kThreads) {
        const int tt = e / (8 * m4), e2 = e - tt * 8 * m4;
        const int n = e2 / m4, k = e2 - n * m4;
        double* Bs = scratch + kWarps * 64 + tt * per_term;
        Bs[k * 8 + n] = (k < m && jj0 + n < q)
                            ? __ldg(lv.left + (t0 + tt) * mq + static_cast<int64_t>(jj0 + n) * m + k) : 0.0;
      }
      for (int e = threadIdx.x; e < gn * SB * m4; e += kThreads) {
        const int tt = e / (SB * m4), e2 = e - tt * SB * m4;
        const int i = e2 / m4, rc = e2 - i * m4;
        double* Cs = scratch + kWarps * 64 + tt * per_term + 16 * m4;
        Cs[i * (m4 + 1) + rc] = (rc < m && s0 + i < q)
                                    ? __ldg(lv.right + (t0 + tt) * mq + static_cast<int64_t>(s0 + i) * m + rc) : 0.0;
      }
      __syncthreads();
      // V_t = R B_t(:, jj-block): warp w owns (row tile, term) items w, w + 8, ...
      for (int it = w; it < mt * gn; it += kWarps) {
        const int rt = it % mt, tt = it / mt;
        const double* Bs = scratch + kWarps * 64 + tt * per_term;
        double* Vs = scratch + kWarps * 64 + tt * per_term + 8 * m4;
        double c[2] = {0.0, 0.0};
        const int rc = rt * 8 + g;
        for (int ks = 0; ks < ks_n; ++ks) {
          const int k = ks * 4 + tg;
          const double a = (rc < m && k < m) ? r[rc + k * m] : 0.0;
          dmma884(c, a, Bs[k * 8 + g]);
        }
        if (rc < m4) {
          Vs[rc * 8 + 2 * tg] = c[0];
          Vs[rc * 8 + 2 * tg + 1] = c[1];
        }
      }
      __syncthreads();
      // Z(s-block, jj-block) += C_t(:, s-block)^T V_t: warp = (row tile, K part)
      for (int tt = 0; tt < gn; ++tt) {
        const double* Vs = scratch + kWarps * 64 + tt * per_term + 8 * m4;
        const double* Cs = scratch + kWarps * 64 + tt * per_term + 16 * m4;
        for (int ks = k_lo; ks < k_hi; ++ks) {
          const int k = ks * 4 + tg;
          dmma884(acc, Cs[(my_mt * 8 + g) * (m4 + 1) + k], Vs[k * 8 + g]);
        }
      }
    }
    // fixed-order sum of the K parts, then Z tile to memory (Z[j], j = jj*q + s)
    __syncthreads();
    Red[w * 64 + g * 8 + 2 * tg] = acc[0];
    Red[w * 64 + g * 8 + 2 * tg + 1] = acc[1];
    __syncthreads();
    for (int e = threadIdx.x; e < SB * 8; e += kThreads) {
      const int i = e >> 3, n = e & 7;  // tile row i (s), column n (jj)
      const int rt = i >> 3, gi = i & 7;
      double z = 0.0;
      for (int kp = 0; kp < ksplit; ++kp) z += Red[(kp * sb8 + rt) * 64 + gi * 8 + n];
      if (s0 + i < q && jj0 + n < q) __stcg(Z + static_cast<int64_t>(jj0 + n) * q + s0 + i, z);
    }
  }
  vsync();
  int64_t lo, hi;
  slice(S, lo, hi);
  PassAcc acc;
  for (int64_t pos = lo + threadIdx.x; pos < hi; pos += kThreads) {
    const int64_t j = idx[pos];
    const double z = __ldcg(Z + j);
    acc.add(p, po, eps, pos, lv.col_scale ? lv.col_scale[j] * z : z, true);
  }
  finish_pass(p, sh, po, acc);
}

__device__ void op_adjoint(const EngineParams& p, Sh& sh, const DevLevel& lv, const int32_t* idx, const double* eps,
                           int64_t S, const double* r, double* scratch, const PassOut& po) {
  if (lv.kind == kDense)
    dense_adjoint(p, sh, lv, idx, eps, S, r, scratch, po);
  else
    sukro_adjoint(p, sh, lv, idx, eps, S, r, scratch, po);
}

// ----------------------------------------------------------------------------
// Apply: partial sums of u = sum_pos coef(pos) a_{idx[pos]}.
// ----------------------------------------------------------------------------
// Per-atom screening test + prox step of one iteration (fastl1.cpp:519-548, 572-579,
// screening.cpp:136-150, solver.cpp:9-13), written with explicit rounding
// intrinsics so every caller (the slice owner in phase B and the apply work items
// that re-derive coefficients on the fly) gets bit-identical results.
struct ProxCtx {
  const double* corr;
  const double* corr_y;
  const double* x;
  const double* xp;
  const double* eps;
  const double* en;
  const double* an;
  const double* aty;
  const double* atye;
  double m, inv_l, thresh, sp, cn, R, lambda;
  int screen_now, stable_test, rule_gap, ray_is_y, use_atye;
  // per-atom inputs, loaded once (prefetchable)
  struct Atom {
    double c, cy, xo, xpv, eps, en, an, aty;
  };
  __device__ __forceinline__ Atom load(int64_t q) const {
    Atom a;
    a.c = corr[q];
    a.xo = x[q];
    a.xpv = m != 0.0 ? xp[q] : 0.0;
    a.cy = (screen_now && rule_gap && ray_is_y) ? corr_y[q] : 0.0;
    a.eps = (screen_now && stable_test) ? eps[q] : 0.0;
    a.en = screen_now ? en[q] : 0.0;
    a.an = (screen_now && stable_test) ? an[q] : 0.0;
    a.aty = (screen_now && !rule_gap) ? (use_atye ? atye[q] : aty[q]) : 0.0;
    return a;
  }
  __device__ __forceinline__ double dot(const Atom& a) const {
    if (rule_gap) return fabs(__dmul_rn(sp, ray_is_y ? a.cy : a.c));
    return fabs(__ddiv_rn(a.aty, lambda));
  }
  __device__ __forceinline__ bool keep(const Atom& a, double d) const {
    if (!screen_now) return true;
    if (stable_test) return __fma_rn(R, a.en, __fma_rn(a.eps, cn, d)) >= 1.0;  // stable_zone_test
    return __fma_rn(R, a.en, d) >= 1.0;                                          // sphere_test
  }
  __device__ __forceinline__ bool look(const Atom& a, double d, bool kp) const {
    if (!screen_now) return false;
    if (stable_test) return __fma_rn(R, a.an, d) >= 1.0;  // lookahead on approx norms
    return kp;
  }
  __device__ __forceinline__ double xnew(const Atom& a) const {
    const double g = m != 0.0 ? __fma_rn(1.0 + m, a.xo, -__dmul_rn(m, a.xpv)) : a.xo;
    const double z = __fma_rn(inv_l, a.c, g);
    const double mag = fabs(z) - thresh;
    if (mag <= 0.0) return 0.0;
    return z > 0.0 ? mag : -mag;
  }
  __device__ __forceinline__ bool keep_at(int64_t q, const Atom& a) const {
    return keep(a, screen_now ? dot(a) : 0.0);
  }
};

struct ApplySrc {
  const int32_t* idx;
  const double* coef;      // values (x or power vector)
  const double* coef_div;  // if non-null: coef = coef_div[pos] / div
  double div;
  const int8_t* keep;      // nullable: only keep != 0 contribute
  const double* xp;        // nullable: keep == 0 && xp != 0 feed the v fix (apply_restriction 673-684)
  const ProxCtx* prox;     // non-null: coefficients re-derived on the fly (phase B)
  __device__ __forceinline__ double c(int64_t pos) const { return coef_div ? coef_div[pos] / div : coef[pos]; }
  __device__ __forceinline__ bool kept(int64_t pos) const { return keep == nullptr || keep[pos] != 0; }
  // coefficient of position pos for pass `fix` (0: kept atoms, 1: dropped atoms' history)
  __device__ __forceinline__ double coef_for(int64_t pos, bool fix) const {
    if (prox) {
      const ProxCtx::Atom a = prox->load(pos);
      const bool kp = prox->keep_at(pos, a);
      if (!fix) return kp ? prox->xnew(a) : 0.0;
      return kp ? 0.0 : a.xo;
    }
    if (!fix) return kept(pos) ? c(pos) : 0.0;
    return keep[pos] == 0 ? xp[pos] : 0.0;
  }
};

// Dense apply as streamed (column, 256-row unit) work, the transpose of the
// adjoint's traversal: work item (h, c) = row unit h x column chunk c; the 16
// warps of a CTA split the chunk's positions contiguously, read the
// coefficients 32 at a time, skip zeros by ballot, and stream the nonzero
// columns' units through the same three-stage register ring (kV x 128-bit
// loads per lane) into per-lane accumulators. Warp partials are added in warp
// order in shared memory; out[c*ld + row] holds chunk c's partial sum.
__device__ __forceinline__ int dense_apply_chunks(const EngineParams& p, const DevLevel& lv, int64_t S) {
  const int64_t U = ((lv.rows ? lv.rows : p.n) + kUnit - 1) / kUnit;
  int64_t c = p.grid / U;
  const int64_t by_work = (S + 31) / 32;  // at least ~2 positions per warp
  if (c > by_work) c = by_work;
  return static_cast<int>(c < 1 ? 1 : c);
}

__device__ __noinline__ void dense_apply_units(const EngineParams& p, const DevLevel& lv, const ApplySrc& src,
                                               int64_t S, bool fix, double* __restrict__ out, double* red) {
  constexpr int kV = kUnit / 64;
  const int64_t n = lv.rows ? lv.rows : p.n, ld = lv.rows ? lv.ld : p.ld, ld2 = ld >> 1;
  const int U = static_cast<int>((n + kUnit - 1) / kUnit);
  const int last_nd2 = static_cast<int>(((n - static_cast<int64_t>(U - 1) * kUnit) + 1) >> 1);
  const int C = dense_apply_chunks(p, lv, S);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const double2* __restrict__ A2 = reinterpret_cast<const double2*>(lv.a) + l;
  for (int64_t item = vrank(); item < static_cast<int64_t>(U) * C; item += vsize()) {
    const int h = static_cast<int>(item % U);
    const int64_t c = item / U;
    const int64_t clo = S * c / C, chi = S * (c + 1) / C;
    const int64_t p0 = clo + (chi - clo) * w / kWarps, p1 = clo + (chi - clo) * (w + 1) / kWarps;
    const int nd2 = h == U - 1 ? last_nd2 : kUnit / 2;
    const int64_t hoff = static_cast<int64_t>(h) * (kUnit / 2);
    double2 acc[kV];
#pragma unroll
    for (int q = 0; q < kV; ++q) acc[q] = make_double2(0.0, 0.0);
    auto issue = [&](double2 (&b)[kV], int32_t col) {
      const double2* srcp = A2 + static_cast<int64_t>(col) * ld2 + hoff;
      if (nd2 == kUnit / 2) {
#pragma unroll
        for (int q = 0; q < kV; ++q) b[q] = ldg_stream2(srcp + 32 * q);
      } else {
#pragma unroll
        for (int q = 0; q < kV; ++q) b[q] = (l + 32 * q < nd2) ? ldg_stream2(srcp + 32 * q) : make_double2(0.0, 0.0);
      }
    };
    auto consume = [&](const double2 (&b)[kV], double cf) {
#pragma unroll
      for (int q = 0; q < kV; ++q) {
        acc[q].x = fma(cf, b[q].x, acc[q].x);
        acc[q].y = fma(cf, b[q].y, acc[q].y);
      }
    };
    for (int64_t g0 = p0; g0 < p1; g0 += 32) {
      const int64_t pos = g0 + l;
      double cf = 0.0;
      int32_t col = 0;
      if (pos < p1) {
        cf = src.coef_for(pos, fix);
        if (cf != 0.0) col = src.idx[pos];
      }
      unsigned mask = __ballot_sync(kFull, cf != 0.0);
      // ring over the set bits, in position order
      double2 b0[kV], b1[kV], b2[kV];
      int l0 = -1, l1 = -1, l2 = -1;
      if (mask) {
        l0 = __ffs(mask) - 1;
        mask &= mask - 1;
        issue(b0, __shfl_sync(kFull, col, l0));
      }
      if (mask) {
        l1 = __ffs(mask) - 1;
        mask &= mask - 1;
        issue(b1, __shfl_sync(kFull, col, l1));
      }
      while (l0 >= 0) {
        if (mask) {
          l2 = __ffs(mask) - 1;
          mask &= mask - 1;
          issue(b2, __shfl_sync(kFull, col, l2));
        } else {
          l2 = -1;
        }
        consume(b0, __shfl_sync(kFull, cf, l0));
        if (l1 < 0) break;
        if (mask) {
          l0 = __ffs(mask) - 1;
          mask &= mask - 1;
          issue(b0, __shfl_sync(kFull, col, l0));
        } else {
          l0 = -1;
        }
        consume(b1, __shfl_sync(kFull, cf, l1));
        if (l2 < 0) break;
        if (mask) {
          l1 = __ffs(mask) - 1;
          mask &= mask - 1;
          issue(b1, __shfl_sync(kFull, col, l1));
        } else {
          l1 = -1;
        }
        consume(b2, __shfl_sync(kFull, cf, l2));
      }
    }
    // warp partials -> shared memory -> sum over warps in order
#pragma unroll
    for (int q = 0; q < kV; ++q) reinterpret_cast<double2*>(red)[w * (kUnit / 2) + l + 32 * q] = acc[q];
    __syncthreads();
    for (int e = threadIdx.x; e < kUnit; e += kThreads) {
      double t = 0.0;
      for (int ww = 0; ww < kWarps; ++ww) t += red[ww * kUnit + e];
      const int64_t row = static_cast<int64_t>(h) * kUnit + e;
      if (row < ld) __stcg(out + c * ld + row, t);
    }
    __syncthreads();
  }
}

// SuKro apply (SukroDictionary::apply, dictionary.cpp:150-156, on the ActiveOp
// zero-padded iterate 141-145): u = vec(sum_t C_t X B_t^T), X = reshape(d o x, q, q).
// Every nonzero x_j (j = jj*q + s) adds sum_t (d_j x_j C_t(:, s)) B_t(:, jj)^T, so
// each CTA forms the partial U of its own slice of positions as one DMMA rank-k
// update U_c = Cg Bg^T over the gathered columns (k = entry x term), staged through
// shared memory in chunks — no grid barrier. Partials go to chunk vrank of out
// (and of fix_out for the v-fix source: dropped atoms' previous iterate).
__device__ __noinline__ int sukro_apply_partials(const EngineParams& p, Sh& sh, const DevLevel& lv, const ApplySrc& src,
                                                 int64_t S, double* __restrict__ out, double* __restrict__ fix_out,
                                                 double* __restrict__ scratch) {
  const int m = static_cast<int>(lv.m), q = static_cast<int>(lv.q);
  const int nt = lv.nterms;
  const int64_t mq = static_cast<int64_t>(m) * q, nn = static_cast<int64_t>(m) * m, ld = p.ld;
  const int nsrc = fix_out ? 2 : 1;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, g = l >> 2, tg = l & 3;
  const int mt = (m + 7) >> 3, ntile = mt * mt, passes = (ntile + 63) / 64;
  const int m1 = m + 1;
  double* ent_v = scratch;                                   // kThreads entry values
  int32_t* ent_j = reinterpret_cast<int32_t*>(scratch + kThreads);  // kThreads atom indices
  double* stage = scratch + kThreads + kThreads / 2;
  const int64_t room = p.scratch_len - (kThreads + kThreads / 2);
  int kc = static_cast<int>(min(static_cast<int64_t>(128), room / (2 * m1))) & ~3;
  const int E = max(1, kc / nt);  // entries per chunk
  kc = (E * nt + 3) & ~3;
  double* Cg = stage;           // column k: Cg[k*m1 + row]
  double* Bg = stage + kc * m1;
  int64_t lo, hi;
  slice(S, lo, hi);
  for (int sr = 0; sr < nsrc; ++sr) {
    double* __restrict__ dst = (sr == 0 ? out : fix_out) + static_cast<int64_t>(vrank()) * ld;
    for (int pass = 0; pass < passes; ++pass) {
      double acc[8][2];
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
      for (int64_t base = lo; base < hi; base += kThreads) {
        // entries of this batch of positions, compacted in position order
        const int64_t pos = base + threadIdx.x;
        double v = 0.0;
        int32_t j = 0;
        if (pos < hi) {
          j = src.idx[pos];
          if (sr == 0) {
            if (src.kept(pos)) v = src.c(pos);
          } else if (!src.kept(pos)) {
            v = src.xp[pos];
          }
          if (v != 0.0 && lv.col_scale) v *= lv.col_scale[j];
        }
        const unsigned bal = __ballot_sync(kFull, v != 0.0);
        if (l == 0) sh.wscan[w] = __popc(bal);
        __syncthreads();
        int off = 0, tot = 0;
        for (int ww = 0; ww < kWarps; ++ww) {
          if (ww < w) off += sh.wscan[ww];
          tot += sh.wscan[ww];
        }
        if (v != 0.0) {
          const int at = off + __popc(bal & ((1u << l) - 1u));
          ent_v[at] = v;
          ent_j[at] = j;
        }
        __syncthreads();
        for (int e0 = 0; e0 < tot; e0 += E) {
          const int ne = min(E, tot - e0), ncol = ne * nt, ncol4 = (ncol + 3) & ~3;
          for (int e = threadIdx.x; e < ncol4 * m; e += kThreads) {
            const int col = e / m, row = e - col * m;
            double cv = 0.0, bv = 0.0;
            if (col < ncol) {
              const int en = e0 + col / nt, t = col - (col / nt) * nt;
              const int32_t jj = ent_j[en] / q, ss = ent_j[en] - jj * q;
              cv = ent_v[en] * __ldg(lv.right + t * mq + static_cast<int64_t>(ss) * m + row);
              bv = __ldg(lv.left + t * mq + static_cast<int64_t>(jj) * m + row);
            }
            Cg[col * m1 + row] = cv;
            Bg[col * m1 + row] = bv;
          }
          __syncthreads();
          for (int ks = 0; ks < (ncol4 >> 2); ++ks) {
            const int k = ks * 4 + tg;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int T = pass * 64 + w * 8 + i;
              if (T < ntile) {
                const int rc = (T / mt) * 8 + g, rb = (T % mt) * 8 + g;
                dmma884(acc[i], rc < m ? Cg[k * m1 + rc] : 0.0, rb < m ? Bg[k * m1 + rb] : 0.0);
              }
            }
          }
          __syncthreads();
        }
      }
      // U_c(rc, rb) at rc + rb*m
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int T = pass * 64 + w * 8 + i;
        if (T < ntile) {
          const int rc = (T / mt) * 8 + g;
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int rb = (T % mt) * 8 + 2 * tg + c;
            if (rc < m && rb < m) __stcg(dst + rc + static_cast<int64_t>(rb) * m, acc[i][c]);
          }
        }
      }
    }
    for (int64_t i = nn + threadIdx.x; i < ld; i += kThreads) __stcg(dst + i, 0.0);  // padding rows
  }
  return vsize();
}

// Returns the number of partial chunks written to out (and fix_out).
__device__ int op_apply_partials(const EngineParams& p, Sh& sh, const DevLevel& lv, const ApplySrc& src, int64_t S,
                                 double* out, double* fix_out, double* red) {
  if (lv.kind == kDense) {
    dense_apply_units(p, lv, src, S, false, out, red);
    if (fix_out) dense_apply_units(p, lv, src, S, true, fix_out, red);
    return dense_apply_chunks(p, lv, S);
  }
  return sukro_apply_partials(p, sh, lv, src, S, out, fix_out, red);
}

// ----------------------------------------------------------------------------
// Restricted power iteration (detail::power_iteration_sq_norm, solver.cpp:72-104)
// over the current bank. Returns the Rayleigh estimate and leaves the final
// normalised vector in bank.lead. Three grid syncs per step.
// ----------------------------------------------------------------------------
struct Scratch {
  double* vec;     // ld doubles (shared memory)
  double* rt;      // SuKro R^T (shared memory)
  double* red;     // kWarps * kUnit doubles: apply warp partials (aliases rt)
};

// Cluster mode, dense level, this CTA's preserved columns fit in shared memory: the
// whole restricted power iteration runs on chip. Each CTA keeps its slice's columns
// resident, writes its apply partial to shared memory, and every CTA reads all of
// them through distributed shared memory (and the step statistics likewise): two
// cluster barriers per step and no global-memory round trip. Same fixed-order sums
// on every CTA, so the estimate and the leading vector are identical everywhere.
__device__ __forceinline__ bool power_onchip_fits(const EngineParams& p, const DevLevel& lv, int64_t S) {
  if (!s_vcluster || vsize() > 16 || lv.kind != kDense || lv.rows != 0) return false;
  const int64_t nc = (S + vsize() - 1) / vsize();
  return nc * p.ld + p.ld + 4 + 2 * nc <= p.scratch_len;
}

__device__ __noinline__ double power_iteration_onchip(const EngineParams& p, Sh& sh, const DevLevel& lv, const Bank& bk,
                                                      int64_t S, const double* cur_src, double cur_div, int max_iter,
                                                      double rel_tol, int min_iter, const Scratch& sc) {
  cg::cluster_group cl = cg::this_cluster();
  const int G = vsize();
  const int64_t ld = p.ld;
  int64_t lo, hi;
  slice(S, lo, hi);
  const int nc = static_cast<int>(hi - lo), ncmax = static_cast<int>((S + G - 1) / G);
  double* cache = sc.red;                                 // [ncmax][ld] this CTA's columns
  double* P = cache + static_cast<int64_t>(ncmax) * ld;   // [ld] apply partial (read by the cluster)
  double* stats = P + ld;                                 // [4] step statistics (read by the cluster)
  double* vloc = stats + 4;                               // [ncmax] v on this CTA's positions
  double* zbuf = vloc + ncmax;                            // [ncmax] z on this CTA's positions
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int64_t n2 = ld >> 1;
  for (int c = 0; c < nc; ++c) {
    const double2* col = reinterpret_cast<const double2*>(lv.a + static_cast<int64_t>(bk.idx[lo + c]) * ld);
    double2* dst = reinterpret_cast<double2*>(cache + static_cast<int64_t>(c) * ld);
    for (int64_t e = threadIdx.x; e < n2; e += kThreads) dst[e] = ldg_stream2(col + e);
  }
  for (int c = threadIdx.x; c < nc; c += kThreads) vloc[c] = cur_src[lo + c] / cur_div;
  __syncthreads();
  double estimate = 0.0;
  bool have_w = false;
  for (int it = 0; it < max_iter; ++it) {
    double tq0 = 0.0;
    if (threadIdx.x == 0) {
      sh.s.power_steps += 1;
      sh.s.prof_power_bytes += 16.0 * static_cast<double>(p.n) * static_cast<double>(S);
      tq0 = globaltimer_ns();
    }
    for (int64_t i = threadIdx.x; i < ld; i += kThreads) {  // apply: this CTA's partial of A v
      double acc = 0.0;
      for (int c = 0; c < nc; ++c) acc = fma(vloc[c], cache[static_cast<int64_t>(c) * ld + i], acc);
      P[i] = acc;
    }
    cl.sync();
    for (int64_t i = threadIdx.x; i < ld; i += kThreads) {  // w = sum of the partials, rank order
      double acc = 0.0;
      for (int r = 0; r < G; ++r) acc += cl.map_shared_rank(P, r)[i];
      sc.vec[i] = acc;
    }
    __syncthreads();
    for (int c = w; c < nc; c += kWarps) {  // adjoint on this CTA's columns
      const double* col = cache + static_cast<int64_t>(c) * ld;
      double sd = 0.0;
      for (int64_t i = l; i < ld; i += 32) sd = fma(col[i], sc.vec[i], sd);
      sd = warp_sum(sd);
      if (l == 0) zbuf[c] = sd;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double s2 = 0.0, svw = 0.0;
      for (int c = 0; c < nc; ++c) {
        s2 = fma(zbuf[c], zbuf[c], s2);
        svw = fma(vloc[c], zbuf[c], svw);
      }
      stats[0] = s2;
      stats[1] = svw;
    }
    cl.sync();
    double tot2 = 0.0, totvw = 0.0;
    for (int r = 0; r < G; ++r) {
      const double* st = cl.map_shared_rank(stats, r);
      tot2 += st[0];
      totvw += st[1];
    }
    if (threadIdx.x == 0) sh.s.prof_pw[2] += globaltimer_ns() - tq0;
    const double nrm = sqrt(tot2);
    if (nrm == 0.0) {
      estimate = 0.0;
      break;
    }
    const double prev = estimate;
    estimate = totvw;
    __syncthreads();  // every thread has read vloc (statistics) before it changes
    for (int c = threadIdx.x; c < nc; c += kThreads) vloc[c] = zbuf[c] / nrm;
    have_w = true;
    __syncthreads();
    if (it > min_iter && fabs(estimate - prev) <= rel_tol * estimate) break;
  }
  (void)have_w;  // vloc is v after the last update either way (fastl1 lead_vector)
  for (int c = threadIdx.x; c < nc; c += kThreads) bk.lead[lo + c] = vloc[c];
  cl.sync();  // no CTA reuses its scratch while another may still read its partial / statistics
  return estimate;
}

#if FL1_FUSED_VARIANT
// ----------------------------------------------------------------------------
// Single-read power step for preserved sets beyond L2 (HBM-bound). With t = A v in
// shared memory, one pass over this CTA's columns gives z_j = a_j . t (= (A^T A v)_j,
// solver.cpp:92) and, in the same read, this CTA's partial of A z = sum_j z_j a_j --
// the next step's t after the division by ||z|| (v' = z / ||z||, solver.cpp:100) -- so a
// step streams the preserved columns once instead of twice. The CTA works on one
// column at a time; warp w owns the column's 4 KiB units w and w + 8 (8 < units <= 16:
// 4096 < n <= 8192), which land in its two bulk-ring stages; it keeps them in registers
// for the axpy that follows the column's block-wide dot, and refills its stages with
// the next column's units as soon as it has read them (16 units in flight per SM, as
// in the adjoint's bulk ring). One block barrier per column.
// ----------------------------------------------------------------------------
constexpr int kFuseMaxU = 16;
__shared__ double s_fred[2][FL1_THREADS / 32];

__device__ __forceinline__ bool fused_power_fits(const EngineParams& p, const DevLevel& lv, int64_t S) {
  const int64_t U = (p.n + kUnit - 1) / kUnit;
  return p.fused_power_bytes > 0 && !s_vcluster && lv.kind == kDense && lv.rows == 0 && p.bulk_stages == 2 &&
         kWarps == 8 && kUnit == 512 && U > kWarps && U <= kFuseMaxU && 8 * p.ld * S >= p.fused_power_bytes;
}

__device__ __noinline__ void dense_fused_power_pass(const EngineParams& p, Sh& sh, const DevLevel& lv,
                                                    const int32_t* __restrict__ idx, int64_t S,
                                                    const double* __restrict__ t, double* __restrict__ ring,
                                                    const PassOut& po, double* __restrict__ part) {
  constexpr int kV = kUnit / 64;  // double2 per lane per unit
  const int64_t ld = p.ld;
  const int U = static_cast<int>((p.n + kUnit - 1) / kUnit);
  const int last_nd2 = static_cast<int>((ld - static_cast<int64_t>(U - 1) * kUnit) >> 1);
  int64_t c0, c1;
  slice(S, c0, c1);
  const int nc = static_cast<int>(c1 - c0);
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  const bool on_chip = nc <= kColBuf;
  double* __restrict__ dst = on_chip ? s_colsum : po.out + c0;
  const double* __restrict__ A = lv.a;
  const int n_mine = 1 + (w + kWarps < U ? 1 : 0);  // this warp's units of every column: w (and w + 8)
  double2* wring = reinterpret_cast<double2*>(ring) + static_cast<int64_t>(w) * 2 * (kUnit / 2);
  uint64_t* bars = &s_bar[w * kMaxBulk];
  uint32_t ph = s_bphase[w];
  auto issue_col = [&](int c) {  // lane 0
    const double* colp = A + static_cast<int64_t>(__ldg(idx + c0 + c)) * ld;
    for (int st = 0; st < n_mine; ++st) {
      const int h = w + kWarps * st;
      const uint32_t bytes = static_cast<uint32_t>(((h == U - 1) ? (ld - static_cast<int64_t>(h) * kUnit) : kUnit) * 8);
      bulk_load(wring + st * (kUnit / 2), colp + static_cast<int64_t>(h) * kUnit, bytes, bars + st);
    }
  };
  // L2 prefetch kFusePf columns ahead: the stages refill only after a column's axpy, so the
  // refill's latency is on the column's critical path -- from L2 instead of HBM
  auto prefetch_col = [&](int c) {  // lane 0
    const double* colp = A + static_cast<int64_t>(__ldg(idx + c0 + c)) * ld;
    for (int st = 0; st < n_mine; ++st) {
      const int h = w + kWarps * st;
      const uint32_t bytes = static_cast<uint32_t>(((h == U - 1) ? (ld - static_cast<int64_t>(h) * kUnit) : kUnit) * 8);
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(colp + static_cast<int64_t>(h) * kUnit), "r"(bytes)
                   : "memory");
    }
  };
  const int pf = p.fused_prefetch;
  if (l == 0 && nc > 0) {
    issue_col(0);
    for (int c = 1; c <= pf && c < nc; ++c) prefetch_col(c);
  }
  double2 acc[2][kV];
#pragma unroll
  for (int st = 0; st < 2; ++st)
#pragma unroll
    for (int q = 0; q < kV; ++q) acc[st][q] = make_double2(0.0, 0.0);
  const double2* __restrict__ t2 = reinterpret_cast<const double2*>(t) + l;
  const int lim0 = (w == U - 1 ? last_nd2 : kUnit / 2) - l;
  const int lim1 = n_mine > 1 ? (w + kWarps == U - 1 ? last_nd2 : kUnit / 2) - l : 0;
  for (int c = 0; c < nc; ++c) {
    double d4[4] = {0.0, 0.0, 0.0, 0.0};  // four independent chains (a DFMA's latency is ~10 issue slots)
    if (l == 0 && pf > 0 && c + pf < nc) prefetch_col(c + pf);
#pragma unroll
    for (int st = 0; st < 2; ++st) {
      if (st < n_mine) {
        bulk_wait(bars + st, (ph >> st) & 1u);
        ph ^= 1u << st;
        const int lim = st ? lim1 : lim0;
        const double2* sp = wring + st * (kUnit / 2) + l;
        const double2* tp = t2 + (w + kWarps * st) * (kUnit / 2);
#pragma unroll
        for (int q = 0; q < kV; ++q) {
          if (32 * q < lim) {
            const double2 cv = sp[32 * q], tv = tp[32 * q];
            d4[(2 * q) & 3] = fma(cv.x, tv.x, d4[(2 * q) & 3]);
            d4[(2 * q + 1) & 3] = fma(cv.y, tv.y, d4[(2 * q + 1) & 3]);
          }
        }
      }
    }
    double dotp = warp_sum((d4[0] + d4[1]) + (d4[2] + d4[3]));
    if (l == 0) s_fred[c & 1][w] = dotp;
    __syncthreads();
    double z = 0.0;
#pragma unroll
    for (int ww = 0; ww < kWarps; ++ww) z += s_fred[c & 1][ww];
    if (tid == 0) dst[c] = z;
#pragma unroll
    for (int st = 0; st < 2; ++st) {
      const int lim = st ? lim1 : lim0;
      const double2* sp = wring + st * (kUnit / 2) + l;
#pragma unroll
      for (int q = 0; q < kV; ++q) {
        if (32 * q < lim) {
          const double2 cv = sp[32 * q];
          acc[st][q].x = fma(z, cv.x, acc[st][q].x);
          acc[st][q].y = fma(z, cv.y, acc[st][q].y);
        }
      }
    }
    __syncwarp();  // the stages have been read twice (dot, axpy): refill them with the next column's units
    if (l == 0 && c + 1 < nc) issue_col(c + 1);
  }
  if (l == 0) s_bphase[w] = ph;
  // this CTA's partial of A z
  double2* __restrict__ mine = reinterpret_cast<double2*>(part + static_cast<int64_t>(vrank()) * ld) + l;
#pragma unroll
  for (int st = 0; st < 2; ++st) {
    if (st < n_mine) {
      const int h = w + kWarps * st;
      const int lim = (h == U - 1 ? last_nd2 : kUnit / 2) - l;
#pragma unroll
      for (int q = 0; q < kV; ++q)
        if (32 * q < lim) __stcg(mine + h * (kUnit / 2) + 32 * q, acc[st][q]);
    }
  }
  __syncthreads();
  // z on this CTA's positions and the step statistics (as dense_adjoint)
  PassAcc sa;
  if (on_chip) {
    for (int64_t pos = c0 + tid; pos < c1; pos += kThreads) {
      const double v = s_colsum[pos - c0];
      po.out[pos] = v;
      sa.add(p, po, nullptr, pos, v);
    }
  } else {
    for (int64_t pos = c0 + tid; pos < c1; pos += kThreads) sa.add(p, po, nullptr, pos, po.out[pos]);
  }
  finish_pass(p, sh, po, sa);
  __syncthreads();
}

// The restricted power iteration with single-read steps (dense_fused_power_pass): the first
// step forms A v by the apply partials, every later step inherits it from the previous pass.
__device__ __noinline__ double power_iteration_fused(const EngineParams& p, Sh& sh, const DevLevel& lv, const Bank& bk,
                                                     int64_t S, const double* cur_src, double cur_div, int max_iter,
                                                     double rel_tol, int min_iter, const Scratch& sc) {
  int64_t lo, hi;
  slice(S, lo, hi);
  double estimate = 0.0;
  bool have_w = false, have_t = false;
  for (int it = 0; it < max_iter; ++it) {
    if (threadIdx.x == 0) {
      sh.s.power_steps += 1;
      sh.s.prof_power_bytes += 16.0 * static_cast<double>(p.n) * static_cast<double>(S);
    }
    for (int64_t q = lo + threadIdx.x; q < hi; q += kThreads) p.pv[q] = cur_src[q] / cur_div;
    {
      if (!have_t) {  // first step: A v by the apply partials (every later step inherits it from the pass)
        double ta0 = 0.0;
        if (threadIdx.x == 0) ta0 = globaltimer_ns();
        ApplySrc as0{bk.idx, nullptr, cur_src, cur_div, nullptr, nullptr, nullptr};
        const int C0 = op_apply_partials(p, sh, lv, as0, S, p.pup, nullptr, sc.red);
        vsync();
        int64_t ilo, ihi;
        slice(p.ld, ilo, ihi);
        combine_rows(p.pup, C0, p.ld, ilo, ihi, [&](int64_t i, double tt) { __stcg(p.PU + i, tt); });
        vsync();
        load_vec_smem(p, p.PU, sc.vec);
        if (threadIdx.x == 0) sh.s.prof_pw[0] += globaltimer_ns() - ta0;
      }
      double tf0 = 0.0;
      if (threadIdx.x == 0) tf0 = globaltimer_ns();
      __syncthreads();  // pv (this CTA's slice) before the pass's statistics read it
      PassOut pf{p.pw, 0, 0.0, false, 0, 0, p.pv, 1};
      dense_fused_power_pass(p, sh, lv, bk.idx, S, sc.vec, sc.rt, pf, p.pup);
      vsync();
      if (threadIdx.x == 0) sh.s.prof_pw[2] += globaltimer_ns() - tf0;
      grid_reduce(p, sh, (1u << kSlPw2) | (1u << kSlPvw), 0u);
      const double nrmf = sqrt(sh.res[kSlPw2]);
      if (nrmf == 0.0) {
        estimate = 0.0;
        break;
      }
      const double prevf = estimate;
      estimate = sh.res[kSlPvw];
      cur_src = p.pw;
      cur_div = nrmf;
      have_w = true;
      if (it > min_iter && fabs(estimate - prevf) <= rel_tol * estimate) break;
      if (it + 1 < max_iter) {  // the next step's A v = (sum of the partials of A z) / ||z||
        double tf1 = 0.0;
        if (threadIdx.x == 0) tf1 = globaltimer_ns();
        int64_t ilo, ihi;
        slice(p.ld, ilo, ihi);
        combine_rows(p.pup, vsize(), p.ld, ilo, ihi, [&](int64_t i, double tt) { __stcg(p.PU + i, tt / nrmf); });
        vsync();
        load_vec_smem(p, p.PU, sc.vec);
        have_t = true;
        if (threadIdx.x == 0) sh.s.prof_pw[1] += globaltimer_ns() - tf1;
      }
    }
  }
  for (int64_t q = lo + threadIdx.x; q < hi; q += kThreads) bk.lead[q] = have_w ? p.pw[q] / cur_div : p.pv[q];
  vsync();
  return estimate;
}

#endif  // FL1_FUSED_VARIANT

__device__ __noinline__ double power_iteration(const EngineParams& p, Sh& sh, const DevLevel& lv, const Bank& bk, int64_t S,
                                  bool try_warm, const Scratch& sc) {
  int64_t lo, hi;
  slice(S, lo, hi);
  {
    double a_lead = 0.0, a_g = 0.0;
    for (int64_t q = lo + threadIdx.x; q < hi; q += kThreads) {
      if (try_warm) a_lead = fma(bk.lead[q], bk.lead[q], a_lead);
      a_g = fma(p.gauss0[q], p.gauss0[q], a_g);
    }
    double v[2] = {a_lead, a_g};
    const bool mx[2] = {false, false};
    block_reduce<2>(v, mx, sh);
    if (threadIdx.x == 0) {
      put_slot(p, kSlLead2, v[0]);
      put_slot(p, kSlSum, v[1]);
    }
  }
  vsync();
  grid_reduce(p, sh, (1u << kSlLead2) | (1u << kSlSum), 0u);
  const bool warm = try_warm && sh.res[kSlLead2] > 0.0;
  const double* cur_src = warm ? bk.lead : p.gauss0;
  double cur_div = sqrt(warm ? sh.res[kSlLead2] : sh.res[kSlSum]);
  double estimate = 0.0;
  const int max_iter = warm ? 12 : 200;
  const double rel_tol = warm ? 1e-5 : 1e-9;
  const int min_iter = warm ? 2 : 4;
  if (p.power_onchip && power_onchip_fits(p, lv, S))
    return power_iteration_onchip(p, sh, lv, bk, S, cur_src, cur_div, max_iter, rel_tol, min_iter, sc);
#if FL1_FUSED_VARIANT
  if (fused_power_fits(p, lv, S))
    return power_iteration_fused(p, sh, lv, bk, S, cur_src, cur_div, max_iter, rel_tol, min_iter, sc);
#endif
  bool have_w = false;  // pw holds the last w (v = pw / cur_div)
  for (int it = 0; it < max_iter; ++it) {
    if (threadIdx.x == 0) {
      sh.s.power_steps += 1;
      if (lv.kind == kDense) sh.s.prof_power_bytes += 16.0 * static_cast<double>(p.n) * static_cast<double>(S);
    }
    // v for this step: materialise on this CTA's slice (Rayleigh quotient reads it)
    for (int64_t q = lo + threadIdx.x; q < hi; q += kThreads) p.pv[q] = cur_src[q] / cur_div;
    double tq0 = 0.0;
    if (threadIdx.x == 0) tq0 = globaltimer_ns();
    ApplySrc as{bk.idx, nullptr, cur_src, cur_div, nullptr, nullptr, nullptr};
    const int C = op_apply_partials(p, sh, lv, as, S, p.pup, nullptr, sc.red);
    vsync();
    double tq1 = 0.0;
    if (threadIdx.x == 0) {
      tq1 = globaltimer_ns();
      sh.s.prof_pw[0] += tq1 - tq0;
    }
    if (static_cast<int64_t>(C) * p.ld <= kRedundantCombine) {
      // few partials: every CTA sums them itself (same order) instead of a combine phase
      combine_rows(p.pup, C, p.ld, 0, p.ld, [&](int64_t i, double t) { sc.vec[i] = t; });
    } else {
      int64_t ilo, ihi;
      slice(p.ld, ilo, ihi);
      combine_rows(p.pup, C, p.ld, ilo, ihi, [&](int64_t i, double t) { __stcg(p.PU + i, t); });
      vsync();
        load_vec_smem(p, p.PU, sc.vec);
    }
    __syncthreads();
    double tq2 = 0.0;
    if (threadIdx.x == 0) {
      tq2 = globaltimer_ns();
      sh.s.prof_pw[1] += tq2 - tq1;
    }
    PassOut po{p.pw, 0, 0.0, false, 0, 0, p.pv, 1};
    op_adjoint(p, sh, lv, bk.idx, bk.eps, S, sc.vec, sc.rt, po);
    vsync();
    double tq3 = 0.0;
    if (threadIdx.x == 0) {
      tq3 = globaltimer_ns();
      sh.s.prof_pw[2] += tq3 - tq2;
    }
    grid_reduce(p, sh, (1u << kSlPw2) | (1u << kSlPvw), 0u);
    if (threadIdx.x == 0) sh.s.prof_pw[3] += globaltimer_ns() - tq3;
    const double nrm = sqrt(sh.res[kSlPw2]);
    if (nrm == 0.0) {
      estimate = 0.0;
      break;
    }
    const double prev = estimate;
    estimate = sh.res[kSlPvw];
    cur_src = p.pw;
    cur_div = nrm;
    have_w = true;
    if (it > min_iter && fabs(estimate - prev) <= rel_tol * estimate) break;
  }
  // leading vector (v after the last update)
  for (int64_t q = lo + threadIdx.x; q < hi; q += kThreads) bk.lead[q] = have_w ? p.pw[q] / cur_div : p.pv[q];
  vsync();
  return estimate;
}

// Physical compaction (FL1_COMPACT=1, the A/B alternative to the index gather): the
// column view the streaming passes (A_S^T r, power-iteration apply / adjoint) read --
// the level's matrix through the global index, or the compact copy through cix.
__device__ __forceinline__ DevLevel col_view(const EngineParams& p, const EngineState& s, const DevLevel& lv,
                                             Bank& bk) {
  DevLevel v = lv;
  if (s.csel != 0) {
    v.a = p.cbuf[s.csel - 1];
    bk.idx = p.bcix[s.cur];
  }
  return v;
}

// Copy the CTA's columns at new positions [o0, o1) into dst (column o at dst + o ld):
// the source slot of position o is slot[o] in src; slot[o] becomes o. One warp per
// column, four 16-byte loads in flight per lane.
__device__ void copy_columns(const double* __restrict__ src, int32_t* slot, double* __restrict__ dst, int64_t o0,
                             int64_t o1, int64_t ld) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int64_t n2 = ld >> 1;
  for (int64_t o = o0 + w; o < o1; o += kWarps) {
    const double2* s2 = reinterpret_cast<const double2*>(src + static_cast<int64_t>(slot[o]) * ld);
    double2* d2 = reinterpret_cast<double2*>(dst + o * ld);
    int64_t e = l;
    for (; e + 96 < n2; e += 128) {
      const double2 a = ldg_stream2(s2 + e), b = ldg_stream2(s2 + e + 32), c = ldg_stream2(s2 + e + 64),
                    d = ldg_stream2(s2 + e + 96);
      d2[e] = a;
      d2[e + 32] = b;
      d2[e + 64] = c;
      d2[e + 96] = d;
    }
    for (; e < n2; e += 32) d2[e] = ldg_stream2(s2 + e);
    __syncwarp();
    if (l == 0) slot[o] = static_cast<int32_t>(o);
  }
}

// ActiveOp::gather_metadata (189-201) for the CTA slice; per-CTA max eps to a slot.
__device__ void gather_metadata(const EngineParams& p, Sh& sh, const DevLevel& lv, const Bank& bk, int64_t S) {
  int64_t lo, hi;
  slice(S, lo, hi);
  double me = -DBL_MAX;
  for (int64_t q = lo + threadIdx.x; q < hi; q += kThreads) {
    const int64_t g = bk.idx[q];
    const double e = lv.eps[g];
    bk.eps[q] = e;
    bk.en[q] = lv.en[g];
    bk.an[q] = lv.an[g];
    me = fmax(me, e);
  }
  double v[1] = {me};
  const bool mx[1] = {true};
  block_reduce<1>(v, mx, sh);
  if (threadIdx.x == 0) put_slot(p, kSlMaxEps, v[0]);
}


// Phase E: combine the apply partials into U by row slices; shift: v <- u_old - fix
// (FISTA bookkeeping 581-590 + apply_restriction 673-684); then, for the same
// rows, the NEXT iteration's compute_products (359-369):
//   rho_g = y - ((1+m)u - m v)  into p.rho,
// with per-CTA partials of ||rho_g||^2, rho_g.y and ||y-u||^2 in slots, so phase A
// only loads rho_g and reduces three slots. m is the next iteration's momentum.
__device__ void combine_u(const EngineParams& p, Sh& sh, int C, bool shift, bool fix, double m) {
  int64_t lo, hi;
  slice(p.ld, lo, hi);
  // one pass per row: a group of G lanes sums the chunk partials (G = 1 for few
  // chunks, else 8 with a fixed shuffle tree); the group leader's loads of
  // u_old / v / y are issued together with the partials.
  const int G = C <= kThreadCombineMax ? 1 : 8;
  const int g = threadIdx.x % G;
  const bool mom = m != 0.0;
  double arr = 0.0, ary = 0.0, aee = 0.0;
  for (int64_t i0 = lo; i0 < hi; i0 += kThreads / G) {  // uniform trip count (shuffles)
    const int64_t i = i0 + threadIdx.x / G;
    const bool ok = i < hi;
    double u = 0.0, f = 0.0, u_old = 0.0, v_old = 0.0, yi = 0.0;
    if (ok) {
      if (g == 0) {
        if (shift) u_old = __ldcg(p.U + i);
        else if (mom) v_old = __ldcg(p.V + i);
        yi = p.y[i];  // zero on padded rows
      }
      if (G == 1) {
        u = thread_sum_partials(p.up, C, p.ld, i);
        if (fix) f = thread_sum_partials(p.dvp, C, p.ld, i);
      } else {
        u = lane_sum_partials(p.up, C, p.ld, i, g);
        if (fix) f = lane_sum_partials(p.dvp, C, p.ld, i, g);
      }
    }
    if (G == 8) {
      u += __shfl_xor_sync(kFull, u, 4);
      u += __shfl_xor_sync(kFull, u, 2);
      u += __shfl_xor_sync(kFull, u, 1);
      if (fix) {
        f += __shfl_xor_sync(kFull, f, 4);
        f += __shfl_xor_sync(kFull, f, 2);
        f += __shfl_xor_sync(kFull, f, 1);
      }
    }
    if (ok && g == 0) {
      double v = v_old;
      if (shift) {
        v = u_old - f;  // v = u_old with the history fix (581-590, 673-684)
        __stcg(p.V + i, v);
      }
      __stcg(p.U + i, u);
      const double uw = mom ? (1.0 + m) * u - m * v : u;
      const double r = i < p.n ? yi - uw : 0.0;
      __stcg(p.rho + i, r);
      arr = fma(r, r, arr);
      ary = fma(yi, r, ary);
      if (mom && i < p.n) {
        const double e = yi - u;
        aee = fma(e, e, aee);
      }
    }
  }
  double v[3] = {arr, ary, aee};
  const bool mx[3] = {false, false, false};
  block_reduce<3>(v, mx, sh);
  if (threadIdx.x == 0) {
    put_slot(p, kSlRhoSq, v[0]);
    put_slot(p, kSlRhoY, v[1]);
    put_slot(p, kSlRhoE, v[2]);
  }
}

// Phase E of dense levels with phase-B lists: u_i = sum over the kept nonzeros of
// x_next (the CTAs' lists in CTA = position order) of x_j A(i, j) for this CTA's rows,
// the v-fix sum over the dropped atoms' previous iterate likewise, then the same
// per-row epilogue as combine_u. Replaces the chunked apply partials (and their
// ProxCtx re-derivation) with one gather of the nonzero columns' row segments.
constexpr int kLRB = 64;  // rows per block (at most 2 per lane)

// This warp's share of one list for rows [rb, rb + 32 RL): lane l accumulates rows
// rb + l + 32 r in entry order; 32 / RL entries' column segments in flight per lane.
template <int RL>
__device__ __forceinline__ void list_rows(const double* __restrict__ A, int64_t ld, int64_t S, int G, const int32_t* pp,
                                          const double* lv_v, const int32_t* lv_j, int e0, int e1, int64_t rb,
                                          int64_t ihi, double (&acc)[2]) {
  constexpr int kE = 32 / RL;
  const int l = threadIdx.x & 31;
  for (int eb = e0; eb < e1; eb += 32) {
    // lane q fetches entry eb + q (its CTA by binary search over the prefix)
    int32_t cj = 0;
    double cv = 0.0;
    if (eb + l < e1) {
      const int e = eb + l;
      int a = 0, b = G;  // largest c with pp[c] <= e
      while (b - a > 1) {
        const int mid = (a + b) >> 1;
        if (pp[mid] <= e) a = mid;
        else b = mid;
      }
      const int64_t at = S * a / G + (e - pp[a]);
      cj = lv_j[at];
      cv = lv_v[at];
    }
    const int ne = min(32, e1 - eb);
    for (int q0 = 0; q0 < ne; q0 += kE) {
      double av[kE][RL];
#pragma unroll
      for (int q = 0; q < kE; ++q) {
        const int32_t j = __shfl_sync(kFull, cj, (q0 + q) & 31);
        const double* col = A + static_cast<int64_t>(j) * ld + rb + l;
#pragma unroll
        for (int r = 0; r < RL; ++r)
          av[q][r] = (q0 + q < ne && rb + l + 32 * r < ihi) ? __ldcg(col + 32 * r) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < kE; ++q) {
        const double v = __shfl_sync(kFull, cv, (q0 + q) & 31);
        if (q0 + q < ne) {
#pragma unroll
          for (int r = 0; r < RL; ++r) acc[r] = fma(v, av[q][r], acc[r]);
        }
      }
    }
  }
}

// Loads of combine_u_lists that depend on nothing decided in phase E (the list
// lengths, the first row block's u_old / v / y), issued at the start of the phase so
// they overlap its slot reduction.
struct ListPre {
  int32_t c[2];
  double u, v, y;
};
__device__ __forceinline__ ListPre lists_issue(const EngineParams& p, bool shift, bool mom) {
  ListPre lp{{0, 0}, 0.0, 0.0, 0.0};
  const int G = vsize();
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int t = threadIdx.x + q * kThreads;
    if (t < 2 * G) lp.c[q] = __ldcg(p.lcnt + t);
  }
  int64_t ilo, ihi;
  slice(p.ld, ilo, ihi);
  if (threadIdx.x < kLRB && ilo + threadIdx.x < ihi) {
    const int64_t i = ilo + threadIdx.x;
    lp.y = p.y[i];
    if (shift) lp.u = __ldcg(p.U + i);
    else if (mom) lp.v = __ldcg(p.V + i);
  }
  return lp;
}

__device__ __noinline__ void combine_u_lists(const EngineParams& p, Sh& sh, const DevLevel& lv, int64_t S, bool shift,
                                             bool fix, double m, double* scratch, const ListPre& lp) {
  const int G = vsize();
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  int64_t ilo, ihi;
  slice(p.ld, ilo, ihi);
  const bool mom = m != 0.0;
  const double pre_u = lp.u, pre_v = lp.v, pre_y = lp.y;
  int32_t* pre = reinterpret_cast<int32_t*>(scratch);  // [2][G + 1] exclusive prefix of the list lengths
  double* wpart = scratch + (G + 2);                    // [2][kWarps][kLRB]
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int t = threadIdx.x + q * kThreads;
    if (t < 2 * G) pre[(t / G) * (G + 1) + 1 + t % G] = lp.c[q];
  }
  if (threadIdx.x < 2) pre[threadIdx.x * (G + 1)] = 0;
  __syncthreads();
  if (w < 2) {  // warp 0: apply lists, warp 1: fix lists
    int32_t* pp = pre + w * (G + 1);
    int carry = 0;
    for (int c0 = 0; c0 < G; c0 += 32) {
      int v = c0 + l < G ? pp[1 + c0 + l] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(kFull, v, o);
        if (l >= o) v += t;
      }
      if (c0 + l < G) pp[1 + c0 + l] = v + carry;
      carry += __shfl_sync(kFull, v, 31);
    }
  }
  __syncthreads();
  const double* __restrict__ A = lv.a;
  const int64_t ld = p.ld;
  double arr = 0.0, ary = 0.0, aee = 0.0;
  for (int64_t rb = ilo; rb < ihi; rb += kLRB) {
    const bool one = ihi - rb <= 32;  // block-uniform
    for (int src = 0; src < (fix ? 2 : 1); ++src) {
      const int32_t* pp = pre + src * (G + 1);
      const int E = pp[G];
      const int e0 = static_cast<int>(static_cast<int64_t>(E) * w / kWarps);
      const int e1 = static_cast<int>(static_cast<int64_t>(E) * (w + 1) / kWarps);
      double acc[2] = {0.0, 0.0};
      if (one)
        list_rows<1>(A, ld, S, G, pp, src == 0 ? p.nzv : p.fxv, src == 0 ? p.nzj : p.fxj, e0, e1, rb, ihi, acc);
      else
        list_rows<2>(A, ld, S, G, pp, src == 0 ? p.nzv : p.fxv, src == 0 ? p.nzj : p.fxj, e0, e1, rb, ihi, acc);
#pragma unroll
      for (int r = 0; r < 2; ++r) wpart[(src * kWarps + w) * kLRB + l + 32 * r] = acc[r];
    }
    __syncthreads();
    for (int t = threadIdx.x; t < kLRB && rb + t < ihi; t += kThreads) {
      const int64_t i = rb + t;
      double u = 0.0, f = 0.0;
      for (int ww = 0; ww < kWarps; ++ww) u += wpart[ww * kLRB + t];
      if (fix)
        for (int ww = 0; ww < kWarps; ++ww) f += wpart[(kWarps + ww) * kLRB + t];
      const bool first = rb == ilo;
      const double yi = first ? pre_y : p.y[i];  // zero on padded rows
      double v = 0.0;
      if (shift) {
        v = (first ? pre_u : __ldcg(p.U + i)) - f;  // v = u_old with the history fix (581-590, 673-684)
        __stcg(p.V + i, v);
      } else if (mom) {
        v = first ? pre_v : __ldcg(p.V + i);
      }
      __stcg(p.U + i, u);
      const double uw = mom ? (1.0 + m) * u - m * v : u;
      const double r = i < p.n ? yi - uw : 0.0;
      __stcg(p.rho + i, r);
      arr = fma(r, r, arr);
      ary = fma(yi, r, ary);
      if (mom && i < p.n) {
        const double e = yi - u;
        aee = fma(e, e, aee);
      }
    }
    __syncthreads();  // wpart is reused by the next row block
  }
  double v[3] = {arr, ary, aee};
  const bool mx[3] = {false, false, false};
  block_reduce<3>(v, mx, sh);
  if (threadIdx.x == 0) {
    put_slot(p, kSlRhoSq, v[0]);
    put_slot(p, kSlRhoY, v[1]);
    put_slot(p, kSlRhoE, v[2]);
  }
}

// Column-split apply (large N x nnz): the same result as combine_u_lists (u = A x_next
// in list order, the v fix, the next rho and its statistics), organised for DRAM
// locality. The row-slice gather reads ld / G rows (~440 B at N = 8192) of every listed
// column per CTA, a latency-bound pattern (c4 lambda_9: 61 MB in 65 us per iteration);
// here CTA c takes the contiguous global list range [E c / G, E (c+1) / G) and streams
// whole columns (64 KiB contiguous at N = 8192) into a partial u of all ld rows (one
// partial per CTA, list order inside it), then after one virtual-grid barrier every CTA
// sums the non-empty partials in CTA order for its row slice (fixed order: reproducible).
constexpr int kCsRows = 8;     // rows per thread per row tile (row tile = 8 * kThreads rows)
constexpr int kCsStage = 512;  // list entries staged in shared memory per round
constexpr int64_t kCsMinLd = 8192;  // shorter columns: the row-slice gather is faster (c2 6.43 vs 6.48-7.67 ms, c3 8.64 vs 9.24)
constexpr int64_t kCsRowGroup = 2048;  // rows per row group of the 2D partition (16 KiB column pieces)
constexpr int kCsMaxRG = 8;

__device__ __forceinline__ int64_t cs_lo(int64_t E, int c, int G) { return E * c / G; }

// this CTA's partial of one list (entries [e0, e1) of the global list with prefix pp):
// the entries are staged in shared memory (once when they fit), then every row tile
// issues eight columns' loads (kCsRows rows each) before their FMAs
__device__ __forceinline__ void colsplit_stage(const int32_t* pp, int G, int64_t S, const double* lv_v,
                                               const int32_t* lv_j, int64_t eb, int ne, int32_t* ej, double* ev) {
  __syncthreads();
  for (int q = threadIdx.x; q < ne; q += kThreads) {  // list order
    const int64_t e = eb + q;
    int a = 0, b = G;  // largest CTA segment with pp[a] <= e
    while (b - a > 1) {
      const int mid = (a + b) >> 1;
      if (pp[mid] <= e) a = mid;
      else b = mid;
    }
    const int64_t at = S * a / G + (e - pp[a]);
    ej[q] = __ldcg(lv_j + at);
    ev[q] = __ldcg(lv_v + at);
  }
  __syncthreads();
}

__device__ void colsplit_partial(const EngineParams& p, const double* __restrict__ A, int64_t ld, int64_t S, int G,
                                 const int32_t* pp, const double* lv_v, const int32_t* lv_j, int64_t e0, int64_t e1,
                                 int64_t row_lo, int64_t row_hi, double* __restrict__ out, int32_t* ej, double* ev) {
  constexpr int kB = 4;  // columns per batch of loads
  const bool once = e1 - e0 <= kCsStage;
  if (once) colsplit_stage(pp, G, S, lv_v, lv_j, e0, static_cast<int>(e1 - e0), ej, ev);
  for (int64_t r0 = row_lo; r0 < row_hi; r0 += kCsRows * kThreads) {
    double acc[kCsRows];
#pragma unroll
    for (int r = 0; r < kCsRows; ++r) acc[r] = 0.0;
    for (int64_t eb = e0; eb < e1; eb += kCsStage) {
      const int ne = static_cast<int>(e1 - eb < kCsStage ? e1 - eb : kCsStage);
      if (!once) colsplit_stage(pp, G, S, lv_v, lv_j, eb, ne, ej, ev);
      for (int q = 0; q < ne; q += kB) {
        double av[kB][kCsRows];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          const bool on = q + u < ne;
          const double* col = A + static_cast<int64_t>(on ? ej[q + u] : 0) * ld + r0 + threadIdx.x;
#pragma unroll
          for (int r = 0; r < kCsRows; ++r)
            av[u][r] = (on && r0 + threadIdx.x + r * kThreads < row_hi) ? __ldcs(col + r * kThreads) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          const double x = q + u < ne ? ev[q + u] : 0.0;
#pragma unroll
          for (int r = 0; r < kCsRows; ++r) acc[r] = fma(x, av[u][r], acc[r]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < kCsRows; ++r) {
      const int64_t i = r0 + threadIdx.x + r * kThreads;
      if (i < row_hi) __stcg(out + i, acc[r]);
    }
  }
}

// Column split when the listed columns are long and many (identical decision in every
// CTA: the list lengths are read by all): ld >= kCsMinLd and E entries x ld rows >=
// p.colsplit_elems (FL1_COLSPLIT, default 2 Mi: c4 phase E 54 -> 37 ms over the path).
__device__ __forceinline__ bool colsplit_apply(const EngineParams& p, Sh& sh, const ListPre& lp, const DevLevel& lv) {
  if (p.colsplit_elems <= 0 || lv.kind != kDense || lv.rows != 0 || p.ld < kCsMinLd) return false;
  const int G = vsize();
  double v[1] = {0.0};
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int t = threadIdx.x + q * kThreads;
    if (t < G) v[0] += static_cast<double>(lp.c[q]);  // apply-list lengths of the CTAs this thread read
  }
  const bool mx[1] = {false};
  block_reduce<1>(v, mx, sh);  // exact: integers
  return static_cast<int64_t>(v[0]) * p.ld >= p.colsplit_elems;
}

__device__ __noinline__ void combine_u_colsplit(const EngineParams& p, Sh& sh, const DevLevel& lv, int64_t S,
                                                bool shift, bool fix, double m, double* scratch, const ListPre& lp) {
  const int G = vsize(), c = vrank();
  const bool mom = m != 0.0;
  int32_t* pre = reinterpret_cast<int32_t*>(scratch);  // [2][G + 1] exclusive prefix of the list lengths
  int32_t* ej = pre + 2 * (G + 1);                      // [kCsStage]
  double* ev = scratch + (2 * (G + 1) + kCsStage + 1) / 2 + 1;  // [kCsStage]
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int t = threadIdx.x + q * kThreads;
    if (t < 2 * G) pre[(t / G) * (G + 1) + 1 + t % G] = lp.c[q];
  }
  if (threadIdx.x < 2) pre[threadIdx.x * (G + 1)] = 0;
  __syncthreads();
  if (w < 2) {  // warp 0: apply lists, warp 1: fix lists
    int32_t* pp = pre + w * (G + 1);
    int carry = 0;
    for (int c0 = 0; c0 < G; c0 += 32) {
      int v = c0 + l < G ? pp[1 + c0 + l] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(kFull, v, o);
        if (l >= o) v += t;
      }
      if (c0 + l < G) pp[1 + c0 + l] = v + carry;
      carry += __shfl_sync(kFull, v, 31);
    }
  }
  __syncthreads();
  const int64_t ld = p.ld;
  const int64_t Ea = pre[G], Ef = fix ? pre[(G + 1) + G] : 0;
  // 2D partition: RG row groups x CG column groups; CTA c = rg + RG cg takes the rows of
  // group rg for the entries [E cg / CG, E (cg+1) / CG) (contiguous 16 KiB+ column pieces),
  // so a row sums CG partials instead of G. A CTA with an empty range writes nothing; the
  // combine skips it (the ranges are known to all).
  const int RG = static_cast<int>(ld / kCsRowGroup < 1 ? 1 : (ld / kCsRowGroup > kCsMaxRG ? kCsMaxRG : ld / kCsRowGroup));
  const int CG = G / RG;
  const int rg = c % RG, cg = c / RG;
  const int64_t row_lo = ld * rg / RG / 2 * 2, row_hi = rg + 1 == RG ? ld : ld * (rg + 1) / RG / 2 * 2;
  if (cg < CG) {
    if (cs_lo(Ea, cg, CG) < cs_lo(Ea, cg + 1, CG))
      colsplit_partial(p, lv.a, ld, S, G, pre, p.nzv, p.nzj, cs_lo(Ea, cg, CG), cs_lo(Ea, cg + 1, CG), row_lo, row_hi,
                       p.up + static_cast<int64_t>(c) * ld, ej, ev);
    if (cs_lo(Ef, cg, CG) < cs_lo(Ef, cg + 1, CG))
      colsplit_partial(p, lv.a, ld, S, G, pre + (G + 1), p.fxv, p.fxj, cs_lo(Ef, cg, CG), cs_lo(Ef, cg + 1, CG),
                       row_lo, row_hi, p.dvp + static_cast<int64_t>(c) * ld, ej, ev);
  }
  vsync();
  int64_t ilo, ihi;
  slice(ld, ilo, ihi);
  // partials summed by row slice: 4 groups of CTAs per row (contiguous CTA ranges, eight
  // loads in flight), the group sums added in group order (a fixed order: reproducible)
  constexpr int kGrp = 4, kRB = kThreads / kGrp;
  double* gsum = ev;  // [2][kGrp][kRB] (the entry staging is free after the barrier)
  double arr = 0.0, ary = 0.0, aee = 0.0;
  const int rr = threadIdx.x % kRB, gq = threadIdx.x / kRB;
  const int g0 = CG * gq / kGrp, g1 = CG * (gq + 1) / kGrp;
  auto group_sum = [&](const double* P, int64_t E, int64_t i) {
    int rgi = 0;  // the row group holding row i
    while (rgi + 1 < RG && i >= (rgi + 1 == RG ? ld : ld * (rgi + 1) / RG / 2 * 2)) ++rgi;
    double t = 0.0;
    int cc = g0;
    for (; cc + 8 <= g1; cc += 8) {
      double v8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        v8[u] = cs_lo(E, cc + u, CG) < cs_lo(E, cc + u + 1, CG)
                    ? __ldcg(P + static_cast<int64_t>(rgi + RG * (cc + u)) * ld + i)
                    : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u) t += v8[u];
    }
    for (; cc < g1; ++cc)
      if (cs_lo(E, cc, CG) < cs_lo(E, cc + 1, CG)) t += __ldcg(P + static_cast<int64_t>(rgi + RG * cc) * ld + i);
    return t;
  };
  for (int64_t rb = ilo; rb < ihi; rb += kRB) {
    const int64_t ir = rb + rr;
    __syncthreads();
    gsum[gq * kRB + rr] = ir < ihi ? group_sum(p.up, Ea, ir) : 0.0;
    if (fix) gsum[(kGrp + gq) * kRB + rr] = ir < ihi ? group_sum(p.dvp, Ef, ir) : 0.0;
    __syncthreads();
    if (threadIdx.x >= kRB || rb + threadIdx.x >= ihi) continue;
    const int64_t i = rb + threadIdx.x;
    double u = 0.0, f = 0.0;
#pragma unroll
    for (int q = 0; q < kGrp; ++q) u += gsum[q * kRB + threadIdx.x];
    if (fix)
#pragma unroll
      for (int q = 0; q < kGrp; ++q) f += gsum[(kGrp + q) * kRB + threadIdx.x];
    const bool first = rb == ilo && threadIdx.x < kLRB;  // prefetched by lists_issue
    const double yi = first ? lp.y : p.y[i];
    double v = 0.0;
    if (shift) {
      v = (first ? lp.u : __ldcg(p.U + i)) - f;  // v = u_old with the history fix (581-590, 673-684)
      __stcg(p.V + i, v);
    } else if (mom) {
      v = first ? lp.v : __ldcg(p.V + i);
    }
    __stcg(p.U + i, u);
    const double uw = mom ? (1.0 + m) * u - m * v : u;
    const double r = i < p.n ? yi - uw : 0.0;
    __stcg(p.rho + i, r);
    arr = fma(r, r, arr);
    ary = fma(yi, r, ary);
    if (mom && i < p.n) {
      const double e = yi - u;
      aee = fma(e, e, aee);
    }
  }
  double v[3] = {arr, ary, aee};
  const bool mx[3] = {false, false, false};
  block_reduce<3>(v, mx, sh);
  if (threadIdx.x == 0) {
    put_slot(p, kSlRhoSq, v[0]);
    put_slot(p, kSlRhoY, v[1]);
    put_slot(p, kSlRhoE, v[2]);
  }
}

// ||x||_1 partial of this CTA's slice into the slot of iteration t
__device__ __forceinline__ int l1_slot(uint64_t t) { return (t & 1) ? kSlL1b : kSlL1; }

// Per-atom sphere test + prox on the CTA slice [lo, hi) (results to xnew / keep), the
// CTA's ordered apply / v-fix lists, and its kept / look / nnz / ||x_next||_1 slots.
// `early`: called before the first barrier of a non-screening dense iteration, where
// the stop decision is not known yet; the nnz of the current x (the ledger row of a
// stopping iteration) goes to kSlNnzX.
__device__ __forceinline__ void slice_prox(const EngineParams& p, Sh& sh, const Bank& bk, const ProxCtx& px, int64_t lo,
                                        int64_t hi, bool stop_now, bool fix_pass, bool lists,
                                        const ProxCtx::Atom* pre, const int32_t* pre_idx, bool early,
                                        uint64_t t) {
  double kept = 0.0, look = 0.0, nnz = 0.0, l1n = 0.0, nnzx = 0.0;
  int32_t na = 0, nf = 0;  // list lengths (lists only)
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int64_t q0 = lo; q0 < hi; q0 += kThreads) {  // uniform trip count (list appends)
    const int64_t q = q0 + threadIdx.x;
    bool fa = false, ff = false;
    double va = 0.0, vf = 0.0;
    if (q < hi) {
      ProxCtx::Atom a;
      if (pre && q == lo + threadIdx.x) {
        a = *pre;
        if (px.m == 0.0) a.xpv = 0.0;
      } else {
        a = px.load(q);
      }
      if (early) nnzx += a.xo != 0.0 ? 1.0 : 0.0;
      if (stop_now) {
        nnz += a.xo != 0.0 ? 1.0 : 0.0;
      } else {
        const double d = px.screen_now ? px.dot(a) : 0.0;
        const bool kp = px.keep(a, d);
        look += px.look(a, d, kp) ? 1.0 : 0.0;
        const double xn = px.xnew(a);
        p.xnew[q] = xn;
        bk.keep[q] = static_cast<int8_t>(kp);
        if (kp) {
          kept += 1.0;
          nnz += xn != 0.0 ? 1.0 : 0.0;
          l1n += fabs(xn);  // ||x_{t+1}||_1 over the preserved set (next iteration's 473)
        }
        fa = kp && xn != 0.0;
        ff = fix_pass && !kp && a.xo != 0.0;
        va = xn;
        vf = a.xo;
      }
    }
    if (lists) {  // ordered appends (position order) at this CTA's slice offset
      const int32_t col = (fa || ff) ? ((pre_idx && q == lo + threadIdx.x) ? pre_idx[threadIdx.x] : bk.idx[q]) : 0;
      const unsigned ba = __ballot_sync(kFull, fa), bf = __ballot_sync(kFull, ff);
      if (l == 0) {
        sh.wcount[0][w] = __popc(ba);
        sh.wcount[1][w] = __popc(bf);
      }
      __syncthreads();
      int oa = na, of = nf, ta = 0, tf = 0;
      for (int ww = 0; ww < kWarps; ++ww) {
        if (ww < w) {
          oa += sh.wcount[0][ww];
          of += sh.wcount[1][ww];
        }
        ta += sh.wcount[0][ww];
        tf += sh.wcount[1][ww];
      }
      const unsigned below = (1u << l) - 1u;
      if (fa) {
        const int64_t at = lo + oa + __popc(ba & below);
        p.nzj[at] = col;
        p.nzv[at] = va;
      }
      if (ff) {
        const int64_t at = lo + of + __popc(bf & below);
        p.fxj[at] = col;
        p.fxv[at] = vf;
      }
      na += ta;
      nf += tf;
      __syncthreads();  // wcount is reused by the next round
    }
  }
  if (lists && threadIdx.x == 0) {
    p.lcnt[vrank()] = na;
    p.lcnt[vsize() + vrank()] = nf;
  }
  double v[5] = {kept, look, nnz, l1n, nnzx};
  const bool mx[5] = {false, false, false, false, false};
  block_reduce<5>(v, mx, sh);
  if (threadIdx.x == 0) {
    put_slot(p, kSlKept, v[0]);
    put_slot(p, kSlLook, v[1]);
    put_slot(p, kSlNnz, v[2]);
    if (!stop_now) put_slot(p, l1_slot(t + 1), v[3]);
    if (early) put_slot(p, kSlNnzX, v[4]);
  }
}

// momentum of the next iteration from the FISTA state (fastl1.cpp:465-470)
__device__ __forceinline__ double next_momentum(const EngineParams& p, double t_k, bool ready) {
  if (p.solver != FL1_FISTA || !ready) return 0.0;
  const double t_next = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t_k * t_k));
  return (t_k - 1.0) / t_next;
}


// Gram-mode compute_products (fastl1.cpp:373-393) on this CTA's slice: corr_j =
// aty_j - gw_j with gw = (1+m) gx - m gv, the y-ray correlations aty_j, both pairs of
// dual-scaling maxima (eps = 0 on the exact dictionary), and partials of w.aty, w.gw,
// x.aty, x.gx (w = (1+m) x - m x_prev) for ||rho_g||^2, rho_g.y and ||y - A x||^2.
__device__ __noinline__ void gram_products(const EngineParams& p, Sh& sh, const Bank& bk, int64_t S, double m) {
  int64_t lo, hi;
  slice(S, lo, hi);
  const bool mom = m != 0.0;
  double mp = 0.0, mpy = 0.0, wa = 0.0, wg = 0.0, xa = 0.0, xg = 0.0;
  for (int64_t q = lo + threadIdx.x; q < hi; q += kThreads) {
    const int64_t j = bk.idx[q];
    const double gx = __ldcg(p.GX + j), aty = __ldcg(p.ATYF + j);
    const double xo = bk.x[q];
    const double gw = mom ? (1.0 + m) * gx - m * __ldcg(p.GV + j) : gx;
    const double w = mom ? (1.0 + m) * xo - m * bk.xp[q] : xo;
    const double c = aty - gw;
    p.corr[q] = c;
    p.corr_y[q] = aty;
    mp = fmax(mp, fabs(c));
    mpy = fmax(mpy, fabs(aty) / p.lambda);
    wa = fma(w, aty, wa);
    wg = fma(w, gw, wg);
    if (mom) {
      xa = fma(xo, aty, xa);
      xg = fma(xo, gx, xg);
    }
  }
  double v[4] = {mp, mpy, wa, wg};
  const bool mx[4] = {true, true, false, false};
  block_reduce<4>(v, mx, sh);
  double v2[2] = {xa, xg};
  const bool mx2[2] = {false, false};
  block_reduce<2>(v2, mx2, sh);
  if (threadIdx.x == 0) {
    put_slot(p, kSlMaxPlain, v[0]);
    put_slot(p, kSlMaxStable, v[0]);  // + eps_j |rho| with eps = 0
    put_slot(p, kSlMaxPlainY, v[1]);
    put_slot(p, kSlMaxStableY, v[1]);
    put_slot(p, kSlGwa, v[2]);
    put_slot(p, kSlGwg, v[3]);
    put_slot(p, kSlGxa, v2[0]);
    put_slot(p, kSlGxg, v2[1]);
  }
}

// The Gram matrix as a dense K x K operator level (apply only).
__device__ __forceinline__ DevLevel gram_level(const EngineParams& p) {
  DevLevel g{};
  g.kind = kDense;
  g.a = p.gram;
  g.rows = p.k;
  g.ld = p.gram_ld;
  return g;
}

// Gram-mode phase E (fastl1.cpp:584-600, 678-679): GX = sum of the G x partials; with
// shift, GV = GX_old - fix (the history fix over dropped atoms, G columns).
__device__ void combine_g(const EngineParams& p, int C, bool shift, bool fix) {
  int64_t lo, hi;
  slice(p.k, lo, hi);
  const int64_t ldg = p.gram_ld;
  for (int64_t i = lo + threadIdx.x; i < hi; i += kThreads) {
    double u = 0.0, f = 0.0;
    for (int c = 0; c < C; ++c) u += __ldcg(p.up + static_cast<int64_t>(c) * ldg + i);
    if (fix)
      for (int c = 0; c < C; ++c) f += __ldcg(p.dvp + static_cast<int64_t>(c) * ldg + i);
    if (shift) __stcg(p.GV + i, __ldcg(p.GX + i) - f);
    __stcg(p.GX + i, u);
  }
}

// setup_dictionary (fastl1.cpp:283-324). first: constructor call.
// FL1_COMPACT paths, out of line so the default engine body keeps its register allocation.
__device__ __noinline__ void compact_adjoint(const EngineParams& p, Sh& sh, const DevLevel& lv, int64_t S,
                                             const Scratch& sc, const PassOut& po) {
  Bank cb = p.bank[sh.s.cur];
  const double* eps = cb.eps;
  const DevLevel cv = col_view(p, sh.s, lv, cb);
  op_adjoint(p, sh, cv, cb.idx, eps, S, sc.vec, sc.rt, po);
}

__device__ __noinline__ double compact_power_iteration(const EngineParams& p, Sh& sh, const DevLevel& lv,
                                                       const Scratch& sc) {
  Bank cb = p.bank[sh.s.cur];
  const DevLevel cv = col_view(p, sh.s, lv, cb);
  return power_iteration(p, sh, cv, cb, sh.s.S, sh.s.lead_valid != 0, sc);
}

// After the shrinking pass compacted bank cur into cur^1 (this CTA's kept atoms at new
// positions [sh.scan_base, ...) in position order): the compact-copy slots of the kept
// atoms, then the copy into the other buffer; the state flips to it.
__device__ __noinline__ void compact_shrink(const EngineParams& p, Sh& sh, const DevLevel& lv, int64_t lo, int64_t hi,
                                            int64_t S_new) {
  EngineState& s = sh.s;
  const Bank bk = p.bank[s.cur];
  const int32_t* src_slot = s.csel != 0 ? p.bcix[s.cur] : bk.idx;
  int32_t* dst_slot = p.bcix[s.cur ^ 1];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  int64_t out = sh.scan_base;
  for (int64_t q0 = lo; q0 < hi; q0 += kThreads) {  // the same ordered scan as the bank compaction
    const int64_t q = q0 + threadIdx.x;
    const int kp = q < hi ? bk.keep[q] : 0;
    const unsigned bal = __ballot_sync(kFull, kp);
    if (l == 0) sh.wscan[w] = __popc(bal);
    __syncthreads();
    int64_t off = out;
    int tot = 0;
    for (int ww = 0; ww < kWarps; ++ww) {
      if (ww < w) off += sh.wscan[ww];
      tot += sh.wscan[ww];
    }
    off += __popc(bal & ((1u << l) - 1u));
    if (kp) dst_slot[off] = src_slot[q];
    out += tot;
    __syncthreads();
  }
  copy_columns(s.csel != 0 ? p.cbuf[s.csel - 1] : lv.a, dst_slot, p.cbuf[s.csel == 1 ? 1 : 0], sh.scan_base, out,
               p.ld);
  __syncthreads();
  if (threadIdx.x == 0) {
    if (2 * S_new <= s.cwidth) s.cwidth = S_new;
    s.csel = s.csel == 1 ? 2 : 1;
  }
  __syncthreads();
}

__device__ __noinline__ void setup_dictionary(const EngineParams& p, Sh& sh, bool first, const Scratch& sc) {
  EngineState& s = sh.s;
  const DevLevel& lv = p.lv[s.dict_index];
  Bank bk = p.bank[s.cur];
  if (!first) {  // ActiveOp::rebase (105-112)
    gather_metadata(p, sh, lv, bk, s.S);
    // rebase drops the compact copy and re-runs maybe_compact on the new level (107-110)
    const bool cp = p.compact && lv.kind == kDense && lv.rows == 0 && 2 * s.S <= p.k;
    if (cp) {
      int64_t lo, hi;
      slice(s.S, lo, hi);
      int32_t* cix = p.bcix[s.cur];
      for (int64_t q = lo + threadIdx.x; q < hi; q += kThreads) cix[q] = bk.idx[q];
      __syncthreads();
      copy_columns(lv.a, cix, p.cbuf[0], lo, hi, p.ld);
    }
    if (threadIdx.x == 0) {
      s.csel = cp ? 1 : 0;
      s.cwidth = cp ? s.S : p.k;
    }
    vsync();
    grid_reduce(p, sh, 0u, 1u << kSlMaxEps);
    if (threadIdx.x == 0) s.max_eps = s.S > 0 ? sh.res[kSlMaxEps] : 0.0;
    __syncthreads();
  }
  if (p.rule == FL1_RULE_DYNAMIC) {
    load_vec_smem(p, p.y, sc.vec);
    PassOut po{bk.aty, 0, 0.0, false, 0, 0, nullptr};
    op_adjoint(p, sh, lv, bk.idx, bk.eps, s.S, sc.vec, sc.rt, po);
    if (p.precompute_aty && !s.atye_valid) {
      vsync();
      PassOut pe{bk.atye, 0, 0.0, false, 0, 0, nullptr};
      op_adjoint(p, sh, p.lv[p.n_levels - 1], bk.idx, bk.eps, s.S, sc.vec, sc.rt, pe);
      if (threadIdx.x == 0) s.atye_valid = 1;
    }
    vsync();
  }
  if (p.has_full_l && s.S == p.k) {
    if (threadIdx.x == 0) s.lipschitz = p.full_l[s.dict_index];
  } else {
    const double sq = s.csel == 0 ? power_iteration(p, sh, lv, bk, s.S, s.lead_valid != 0, sc)
                                  : compact_power_iteration(p, sh, lv, sc);
    if (threadIdx.x == 0) {
      s.lead_valid = 1;
      s.lipschitz = fmax(sq, 1e-300) * 1.05;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    s.inv_l = 1.0 / s.lipschitz;
    s.active_at_last_l = s.S;
  }
  // use_gram_now (278-281): exact level, a Gram matrix, no observer
  const bool gram = p.gram && !p.observe && s.dict_index == p.n_levels - 1;
  if (threadIdx.x == 0) s.gram_mode = gram ? 1 : 0;
  if (gram && !s.atyf_valid) {  // aty_full = A^T y over every atom (288-290)
    load_vec_smem(p, p.y, sc.vec);
    PassOut pa{p.ATYF, 0, 0.0, false, 0, 0, nullptr};
    op_adjoint(p, sh, lv, p.ident, lv.eps, p.k, sc.vec, sc.rt, pa);
    if (threadIdx.x == 0) s.atyf_valid = 1;
    vsync();
  }
  // u = op.apply(x), or gx = G x in Gram mode (315-321)
  ApplySrc as{bk.idx, bk.x, nullptr, 1.0, nullptr, nullptr, nullptr};
  const DevLevel glv = gram_level(p);
  const int C = op_apply_partials(p, sh, gram ? glv : lv, as, s.S, p.up, nullptr, sc.red);
  vsync();
  if (gram) combine_g(p, C, false, false);
  else combine_u(p, sh, C, false, false, 0.0);  // momentum restarts (fastl1.cpp:322-323)
  if (threadIdx.x == 0) {
    s.momentum_ready = 0;
    s.t_k = 1.0;
  }
  vsync();
}

__device__ uint64_t row_flops(const EngineParams& p, int dict, int64_t active, int64_t nnz) {  // 647-665
  const uint64_t un = static_cast<uint64_t>(p.n), uk = static_cast<uint64_t>(p.k);
  const uint64_t ua = static_cast<uint64_t>(active), uz = static_cast<uint64_t>(nnz);
  const int last = p.n_levels - 1;
  if (p.variant == FL1_PLAIN) return (uk + uz) * un + 4 * uk + un;
  if (p.variant == FL1_MULTI_DICT && dict < last) return p.lv[dict].matvec_flops + uz * un + 8 * ua + 7 * un;
  return (ua + uz) * un + 6 * ua + 5 * un;
}

}  // namespace

// ============================================================================
// The whole solve (Engine ctor + Engine::run) or a utility mode, on the virtual grid.
__device__ __noinline__ void engine_body(const EngineParams& p, Sh& sh, double* dyn) {
  EngineState& s = sh.s;
  Scratch sc;
  sc.vec = dyn;
  sc.rt = dyn + p.ld;  // SuKro R^T; aliases the apply scratch (never live together)
  sc.red = dyn + p.ld;

  if (threadIdx.x == 0) s = *p.st;
  __syncthreads();
  if (threadIdx.x == 0) s.launches += 1;

  const int64_t n = p.n, k = p.k, ld = p.ld;

  // --------------------------------------------------------------- utility modes
  if (p.mode == kModeAdjoint || p.mode == kModeApply || p.mode == kModePower) {
    const DevLevel& lv = p.lv[p.mode_level];
    Bank bk = p.bank[0];  // identity bank prepared by the host
    if (p.mode == kModeAdjoint) {
      load_vec_smem(p, p.x_init, sc.vec);
      PassOut po{p.vec_out, 0, 0.0, false, 0, 0, nullptr};
      op_adjoint(p, sh, lv, bk.idx, bk.eps, k, sc.vec, sc.rt, po);
    } else if (p.mode == kModeApply) {
      ApplySrc as{bk.idx, p.x_init, nullptr, 1.0, nullptr, nullptr, nullptr};
      const int C = op_apply_partials(p, sh, lv, as, k, p.up, nullptr, sc.red);
      vsync();
      int64_t lo, hi;
      slice(ld, lo, hi);
      combine_rows(p.up, C, ld, lo, hi, [&](int64_t i, double t) { p.vec_out[i] = t; });
    } else {
      const double sq = power_iteration(p, sh, lv, bk, k, false, sc);
      if (vrank() == 0 && threadIdx.x == 0) {
        s.power_est = sq;
        *p.st = s;
      }
    }
    return;
  }

  // --------------------------------------------------------------- Engine ctor
  if (p.mode == kModeSolve) {
    if (threadIdx.x == 0) s.start_ns = globaltimer_ns();
    {
      double acc = 0.0;
      for (int64_t i = threadIdx.x; i < n; i += kThreads) acc = fma(p.y[i], p.y[i], acc);
      double v[1] = {acc};
      const bool mx[1] = {false};
      block_reduce<1>(v, mx, sh);
      if (threadIdx.x == 0) {
        s.y_sq = v[0];
        s.y_norm = sqrt(v[0]);
      }
    }
    Bank bk = p.bank[0];
    const Handoff* hd = p.handoff;  // resume from the batched lockstep engine
    const int64_t S0 = hd ? hd->S : k;
    int64_t lo, hi;
    slice(k, lo, hi);
    for (int64_t q = lo + threadIdx.x; q < hi; q += kThreads) p.ident[q] = static_cast<int32_t>(q);
    slice(S0, lo, hi);
    for (int64_t q = lo + threadIdx.x; q < hi; q += kThreads) {
      bk.idx[q] = hd ? __ldcg(hd->idx + q) : static_cast<int32_t>(q);
      bk.x[q] = hd ? __ldcg(hd->x + q) : (p.has_x_init ? p.x_init[q] : 0.0);
      bk.xp[q] = hd ? __ldcg(hd->xp + q) : 0.0;
      if (hd && hd->lead_valid) bk.lead[q] = __ldcg(hd->lead + q);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      s.S = S0;
      s.cur = 0;
      s.csel = 0;
      s.cwidth = p.k;
    }
    __syncthreads();
    gather_metadata(p, sh, p.lv[s.dict_index], bk, S0);
    {  // ||x_0||_1 for iteration 0
      double acc = 0.0;
      for (int64_t q = lo + threadIdx.x; q < hi; q += kThreads) acc += fabs(bk.x[q]);
      double v[1] = {acc};
      const bool mx[1] = {false};
      block_reduce<1>(v, mx, sh);
      if (threadIdx.x == 0) put_slot(p, l1_slot(hd ? hd->t : 0), v[0]);
    }
    vsync();
    grid_reduce(p, sh, 0u, 1u << kSlMaxEps);
    if (threadIdx.x == 0) s.max_eps = sh.res[kSlMaxEps];
    __syncthreads();
    if (!hd) {
      setup_dictionary(p, sh, true, sc);
    } else {
      // the lockstep engine ran iterations 0..t-1 (setup_dictionary 311-323 there):
      // continue its FISTA state, Lipschitz estimate, leading vector, ledger and trace
      if (threadIdx.x == 0) {
        s.lipschitz = hd->lipschitz;
        s.inv_l = 1.0 / s.lipschitz;
        s.active_at_last_l = hd->active_at_last_l;
        s.lead_valid = hd->lead_valid;
        s.power_steps = hd->power_steps;
        s.t = hd->t;
        s.t_k = hd->t_k;
        s.momentum_ready = hd->ready;
        s.ledger = hd->ledger;
        s.warning = hd->warning;
        s.n_trace = hd->n_trace;
      }
      int64_t rlo, rhi;
      slice(ld, rlo, rhi);
      for (int64_t i = rlo + threadIdx.x; i < rhi; i += kThreads) {
        __stcg(p.up + i, __ldcg(hd->u + i));  // one partial chunk holding u
        __stcg(p.V + i, __ldcg(hd->v + i));
      }
      __syncthreads();
      vsync();
      combine_u(p, sh, 1, false, false, next_momentum(p, hd->t_k, hd->ready != 0));
      vsync();
    }
    if (threadIdx.x == 0) s.t0_ns = globaltimer_ns() - (hd ? hd->elapsed_ns : 0.0);
    __syncthreads();
  }

  // --------------------------------------------------------------- Engine::run
  const int last = p.n_levels - 1;
  const double lambda = p.lambda;
  while (true) {
    if (s.t >= p.max_it) {
      if (threadIdx.x == 0) {
        s.converged = 0;
        s.done = 1;
        s.event = kEvDone;
      }
      break;
    }
    if (p.collect_trace && s.n_trace >= p.trace_cap) {
      if (threadIdx.x == 0) s.event = kEvTraceFull;
      break;
    }
    const DevLevel& lv = p.lv[s.dict_index];
    const Bank bk = p.bank[s.cur];
    const int64_t S = s.S;
    int64_t lo, hi;
    slice(S, lo, hi);
    FL1_MARK(0);
    double tp0 = 0.0;
    if (threadIdx.x == 0) tp0 = globaltimer_ns();

    // ---------------------------------------------------------- phase A
    double momentum = 0.0, t_next = s.t_k;  // 465-470
    if (p.solver == FL1_FISTA && s.momentum_ready) {
      t_next = 0.5 * (1.0 + sqrt(1.0 + 4.0 * s.t_k * s.t_k));
      momentum = (s.t_k - 1.0) / t_next;
    }
    const bool gram = s.gram_mode != 0;
    if (!gram) {  // compute_products (359-369): rho_g was formed by the previous combine phase
      // the three slot sums are reduced by warps 0-2 while every thread's rho loads are in flight
      {
        const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
        double sacc = 0.0;
        if (w < 3) {
          const int slot = kSlRhoSq + w;
          if (p.grid <= 32) {
            if (l < p.grid) sacc = __ldcg(p.bred + static_cast<int64_t>(l) * kBred + slot);
          } else
          for (int b0 = l; b0 < p.grid; b0 += 256) {
            double e[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const int b = b0 + 32 * q;
              e[q] = b < p.grid ? __ldcg(p.bred + static_cast<int64_t>(b) * kBred + slot) : 0.0;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (b0 + 32 * q < p.grid) sacc += e[q];
          }
        }
        load_vec_smem(p, p.rho, sc.vec);  // ends with __syncthreads
        if (w < 3) {
          sacc = warp_sum(sacc);
          if (l == 0) sh.res[kSlRhoSq + w] = sacc;
        }
        __syncthreads();
      }
      if (p.observe && vrank() == 0)
        for (int64_t i = threadIdx.x; i < ld; i += kThreads) p.rho_obs[i] = sc.vec[i];
      if (threadIdx.x == 0) {
        sh.t_next = t_next;
        sh.rho_sq = sh.res[kSlRhoSq];
        sh.rho_dot_y = sh.res[kSlRhoY];
        sh.rho_x_sq = momentum != 0.0 ? sh.res[kSlRhoE] : sh.res[kSlRhoSq];
        sh.rho_norm = sqrt(sh.res[kSlRhoSq]);
      }
      __syncthreads();
    }
    bool exact_fit = !gram && !(sh.rho_sq > 0.0);  // Gram mode decides after the phase-B reduction
    // Non-screening dense iterations: the prox and the apply lists need only this CTA's
    // corr, so they run before the barrier, and the phase-B and phase-E reductions
    // become one (the stop decision, unknown here, only selects the ledger's nnz).
    // Each thread's first atom (x, x_prev, column) is staged into shared memory by
    // cp.async while the pass streams (no registers held across it).
    const bool early = p.early_prox && !gram && !exact_fit && lv.kind == kDense && p.list_apply && !p.observe &&
                       (ld + vsize() - 1) / vsize() <= kLRB &&
                       (p.variant == FL1_PLAIN || s.t % static_cast<uint64_t>(p.interval) != 0);
    if (early) {
      const int64_t q = lo + threadIdx.x;
      if (q < hi) {
        cp_async8(&s_ex[threadIdx.x], bk.x + q);
        if (momentum != 0.0) cp_async8(&s_exp[threadIdx.x], bk.xp + q);
        else s_exp[threadIdx.x] = 0.0;
        cp_async4(&s_eidx[threadIdx.x], bk.idx + q);
      }
      cp_async_commit();
    }
    if (gram) {
      gram_products(p, sh, bk, S, momentum);
    } else if (!exact_fit) {
      // corr = A_S^T rho_g fused with the dual-scaling maxima (414-418)
      PassOut po{p.corr, 1, sh.rho_norm, false, kSlMaxPlain, kSlMaxStable, nullptr};
      if (s.csel == 0) op_adjoint(p, sh, lv, bk.idx, bk.eps, S, sc.vec, sc.rt, po);
      else compact_adjoint(p, sh, lv, S, sc, po);  // FL1_COMPACT: the compact copy
    } else {
      // exact fit (428-449): corr = A^T 0 = 0, dual point along y
      for (int64_t q = lo + threadIdx.x; q < hi; q += kThreads) p.corr[q] = 0.0;
      if (p.rule == FL1_RULE_DYNAMIC) {
        double mp = 0.0, ms = 0.0;
        for (int64_t q = lo + threadIdx.x; q < hi; q += kThreads) {
          const double cy = bk.aty[q];
          p.corr_y[q] = cy;
          const double ac = fabs(cy) / lambda;
          mp = fmax(mp, ac);
          ms = fmax(ms, ac + bk.eps[q] * s.y_norm / lambda);
        }
        double v[2] = {mp, ms};
        const bool mx[2] = {true, true};
        block_reduce<2>(v, mx, sh);
        if (threadIdx.x == 0) {
          put_slot(p, kSlMaxPlainY, v[0]);
          put_slot(p, kSlMaxStableY, v[1]);
        }
      } else {
        load_vec_smem(p, p.y, sc.vec);
        PassOut po{p.corr_y, 1, s.y_norm / lambda, true, kSlMaxPlainY, kSlMaxStableY, nullptr};
        op_adjoint(p, sh, lv, bk.idx, bk.eps, S, sc.vec, sc.rt, po);
      }
    }
    double t_prox = 0.0;  // CTA 0's early-prox time (profile only)
    if (early) {  // the early prox (see above)
      cp_async_wait_all();
      __syncthreads();
      const int64_t q = lo + threadIdx.x;
      ProxCtx::Atom pre{};
      if (q < hi) {
        pre.c = hi - lo <= kColBuf ? s_colsum[threadIdx.x] : p.corr[q];  // the pass's column results
        pre.xo = s_ex[threadIdx.x];
        pre.xpv = s_exp[threadIdx.x];
      }
      ProxCtx px{};
      px.corr = p.corr;
      px.x = bk.x;
      px.xp = bk.xp;
      px.m = momentum;
      px.inv_l = s.inv_l;
      px.thresh = lambda * s.inv_l;
      px.lambda = lambda;
      px.rule_gap = p.rule == FL1_RULE_GAP;
      const double tx0 = threadIdx.x == 0 ? globaltimer_ns() : 0.0;
      slice_prox(p, sh, bk, px, lo, hi, false, false, true, &pre, s_eidx, true, s.t);
      if (threadIdx.x == 0) t_prox = globaltimer_ns() - tx0;
    }
    FL1_MARK(1);
    vsync();  // ------------------------------------------------ sync 1
    FL1_MARK(2);
    double tp1 = 0.0;
    if (threadIdx.x == 0) {
      tp1 = globaltimer_ns();
      // the early prox (phase-B work done before the barrier) is profiled as phase B
      s.prof_ns[0] += tp1 - tp0 - t_prox;
      s.prof_ns[1] += t_prox;
      if (lv.kind == kDense && !gram) {
        s.prof_bytes += 8.0 * static_cast<double>(p.n) * static_cast<double>(S);
        if (S == p.k) {
          s.prof_full_ns += tp1 - tp0 - t_prox;
          s.prof_full_bytes += 8.0 * static_cast<double>(p.n) * static_cast<double>(S);
        }
      }
    }

    // ---------------------------------------------------------- phase B
    const int l1s = l1_slot(s.t);
    if (gram) {
      grid_reduce(p, sh, (1u << l1s) | (1u << kSlGwa) | (1u << kSlGwg) | (1u << kSlGxa) | (1u << kSlGxg),
                  (1u << kSlMaxPlainY) | (1u << kSlMaxStableY) | (1u << kSlMaxPlain) | (1u << kSlMaxStable));
      // residual norms from the Gram dots (fastl1.cpp:385-393)
      const double ysq = s.y_sq;
      const double rgs = fmax(ysq - 2.0 * sh.res[kSlGwa] + sh.res[kSlGwg], 0.0);
      exact_fit = !(rgs > 0.0);
      if (threadIdx.x == 0) {
        sh.t_next = t_next;
        sh.rho_sq = rgs;
        sh.rho_dot_y = ysq - sh.res[kSlGwa];
        sh.rho_x_sq = momentum != 0.0 ? fmax(ysq - 2.0 * sh.res[kSlGxa] + sh.res[kSlGxg], 0.0) : rgs;
        sh.rho_norm = sqrt(rgs);
      }
      __syncthreads();
    } else {
      grid_reduce(p, sh,
                  (1u << l1s) | (early ? (1u << kSlKept) | (1u << kSlLook) | (1u << kSlNnz) | (1u << kSlNnzX) : 0u),
                  exact_fit ? ((1u << kSlMaxPlainY) | (1u << kSlMaxStableY))
                            : ((1u << kSlMaxPlain) | (1u << kSlMaxStable)));
    }
    // prefetch this thread's first atom (overlaps the scalar block below)
    ProxCtx::Atom pre{};
    if (!early) {
      const int64_t q = lo + threadIdx.x;
      if (q < hi) {
        pre.c = p.corr[q];
        pre.xo = bk.x[q];
        pre.xpv = bk.xp[q];
        pre.cy = (exact_fit || gram) ? p.corr_y[q] : 0.0;
        pre.eps = bk.eps[q];
        pre.en = bk.en[q];
        pre.an = bk.an[q];
        pre.aty = p.rule == FL1_RULE_DYNAMIC ? ((p.precompute_aty && s.atye_valid) ? bk.atye[q] : bk.aty[q]) : 0.0;
      }
    }
    if (threadIdx.x == 0) {
      const double x_l1 = sh.res[l1s];
      const double primal = 0.5 * sh.rho_x_sq + lambda * x_l1;
      double sp, st, ray_sq, ray_dot_y;  // dual_scalars (406-450)
      if (!exact_fit) {
        ray_sq = sh.rho_sq;
        ray_dot_y = sh.rho_dot_y;
        const double dp = S > 0 ? sh.res[kSlMaxPlain] : 0.0;
        const double ds = S > 0 ? sh.res[kSlMaxStable] : 0.0;
        const double projection = sh.rho_dot_y / (lambda * sh.rho_sq);
        const double ap = ds > 0 ? 1.0 / ds : CUDART_INF;
        const double at = dp > 0 ? 1.0 / dp : CUDART_INF;
        sp = fmin(fmax(projection, -ap), ap);
        st = fmin(fmax(projection, -at), at);
      } else {
        ray_sq = s.y_sq;
        ray_dot_y = s.y_sq;
        const double dp = S > 0 ? sh.res[kSlMaxPlainY] : 0.0;
        const double ds = S > 0 ? sh.res[kSlMaxStableY] : 0.0;
        sp = 1.0 / (lambda * fmax(1.0, ds));
        st = 1.0 / (lambda * fmax(1.0, dp));
      }
      auto dual_of = [&](double scale) {  // 453-457
        const double dist_sq =
            scale * scale * ray_sq - 2.0 * scale * ray_dot_y / lambda + s.y_sq / (lambda * lambda);
        return 0.5 * s.y_sq - 0.5 * lambda * lambda * dist_sq;
      };
      double gp = primal - dual_of(sp);
      double gt = primal - dual_of(st);
      if (gp < -1e-10 || gt < -1e-10) s.warning = 1;
      gp = fmax(gp, 0.0);
      gt = fmax(gt, 0.0);
      const bool exact_phase = s.dict_index == last;
      const double stop_tol = p.rel_tol > 0 ? p.rel_tol * primal : p.tol;
      const bool stop_now = exact_phase && gt <= stop_tol;
      const bool screen_now = !stop_now && p.variant != FL1_PLAIN && (s.t % static_cast<uint64_t>(p.interval) == 0);
      double radius = 0.0, center_norm = 0.0;
      int stable_test = 1;
      if (screen_now) {
        if (p.rule == FL1_RULE_GAP) {
          double delta = 0.0;
          if (!exact_phase) {  // stable_gap_delta (screening.cpp:103-106)
            const double rn = sqrt(sh.rho_x_sq), e = s.max_eps;
            delta = rn * e * x_l1 + 0.5 * e * e * x_l1 * x_l1;
          }
          radius = sqrt(2.0 * gp + 2.0 * delta) / lambda;
          center_norm = fabs(sp) * sqrt(ray_sq);
        } else {
          const double dist_sq = sp * sp * ray_sq - 2.0 * sp * ray_dot_y / lambda + s.y_sq / (lambda * lambda);
          radius = sqrt(fmax(dist_sq, 0.0));
          center_norm = s.y_norm / lambda;
          if (p.precompute_aty && s.atye_valid) stable_test = 0;
        }
      }
      sh.x_l1 = x_l1;
      sh.primal = primal;
      sh.scale_prime = sp;
      sh.scale_tilde = st;
      sh.ray_sq = ray_sq;
      sh.ray_dot_y = ray_dot_y;
      sh.ray_is_y = exact_fit ? 1 : 0;
      sh.gap_prime = gp;
      sh.gap_tilde = gt;
      sh.stop_now = stop_now ? 1 : 0;
      sh.screen_now = screen_now ? 1 : 0;
      sh.radius = radius;
      sh.center_norm = center_norm;
      sh.stable_test = stable_test;
    }
    __syncthreads();
    const bool stop_now = sh.stop_now;
    const bool fista = p.solver == FL1_FISTA;
    ProxCtx px;
    px.corr = p.corr;
    px.corr_y = p.corr_y;
    px.x = bk.x;
    px.xp = bk.xp;
    px.eps = bk.eps;
    px.en = bk.en;
    px.an = bk.an;
    px.aty = bk.aty;
    px.atye = bk.atye;
    px.m = momentum;
    px.inv_l = s.inv_l;
    px.thresh = lambda * s.inv_l;
    px.sp = sh.scale_prime;
    px.cn = sh.center_norm;
    px.R = sh.radius;
    px.lambda = lambda;
    px.screen_now = sh.screen_now;
    px.stable_test = sh.stable_test;
    px.rule_gap = p.rule == FL1_RULE_GAP;
    px.ray_is_y = sh.ray_is_y;
    px.use_atye = p.precompute_aty && s.atye_valid;
    const bool fix_pass = !stop_now && fista && sh.screen_now;
    // dense (not Gram): phase B lists this CTA's kept nonzeros and v-fix entries, and
    // phase E forms u (and the fix) by row slices straight from the lists
    const bool lists = p.list_apply && lv.kind == kDense && !gram && !stop_now &&
                       (ld + vsize() - 1) / vsize() <= kLRB;  // one row block per CTA
    if (!early) slice_prox(p, sh, bk, px, lo, hi, stop_now, fix_pass, lists, &pre, nullptr, false, s.t);
    // u = A_S x_next over the kept nonzeros (131-146) and the v history fix for atoms
    // dropped by this screening pass (FISTA, 673-684), in the same phase: dense work
    // items re-derive the coefficients with ProxCtx; the SuKro scatter is slice-owned.
    FL1_MARK(7);
    int C_apply = 0;
    if (!stop_now && !lists) {
      if (lv.kind == kDense) {
        ApplySrc as{bk.idx, nullptr, nullptr, 1.0, nullptr, nullptr, &px};
        const DevLevel glv = gram_level(p);  // Gram mode: gx = G x, gv fix over G columns (596-600, 678-679)
        C_apply = op_apply_partials(p, sh, gram ? glv : lv, as, S, p.up, fix_pass ? p.dvp : nullptr, sc.red);
      } else {
        __syncthreads();
        ApplySrc as{bk.idx, p.xnew, nullptr, 1.0, bk.keep, fix_pass ? bk.x : nullptr, nullptr};
        C_apply = op_apply_partials(p, sh, lv, as, S, p.up, fix_pass ? p.dvp : nullptr, sc.red);
      }
    }
    FL1_MARK(3);
    if (!early) vsync();  // -------------------------------------- sync 2
    FL1_MARK(4);
    double tp2 = 0.0;
    if (threadIdx.x == 0) {
      tp2 = globaltimer_ns();
      s.prof_ns[1] += tp2 - tp1;
    }

    // ---------------------------------------------------------- phase E
    const bool shift_u = fista;  // combine: v <- u_old - fix (FISTA history)
    const double tk_next = fista ? (s.momentum_ready ? sh.t_next : s.t_k) : s.t_k;
    const double m_next = next_momentum(p, tk_next, fista);
    ListPre lp{};
    double xo_pre = 0.0, xn_pre = 0.0;  // this thread's first slice position (x_prev <- x, x <- x_next)
    if (lists) {
      lp = lists_issue(p, shift_u, m_next != 0.0);
      if (lo + threadIdx.x < hi) {
        xo_pre = bk.x[lo + threadIdx.x];
        xn_pre = p.xnew[lo + threadIdx.x];
      }
    }
    if (!early) grid_reduce(p, sh, (1u << kSlKept) | (1u << kSlLook) | (1u << kSlNnz), 0u);  // (early: in phase B)
    if (threadIdx.x == 0) {
      sh.S_new = stop_now ? S : static_cast<int64_t>(sh.res[kSlKept]);
      sh.look = static_cast<int64_t>(sh.res[kSlLook]);
      sh.nnz = static_cast<int64_t>(sh.res[(early && stop_now) ? kSlNnzX : kSlNnz]);
      sh.gamma = -1.0;
      sh.next_dict = s.dict_index;
      sh.speed = 0;
      if (sh.screen_now && s.dict_index != last) {
        const double gp = sh.gap_prime, gt = sh.gap_tilde;  // gap_ratio (26-30)
        double gamma = 0.0;
        if (!(gp <= 1e-15)) gamma = fmin(fmax(gt / gp, 0.0), 1.0);
        sh.gamma = gamma;
        if (p.variant == FL1_MULTI_DICT) {  // switch_dictionary (32-38)
          const double rc = p.lv[s.dict_index].rc;
          const double la = static_cast<double>(sh.look);
          const bool speed = la <= rc * static_cast<double>(k);
          int nd = s.dict_index;
          if (speed)
            nd = last;
          else if (gamma <= p.gamma_threshold)
            nd = s.dict_index + 1;
          sh.next_dict = nd;
          sh.speed = speed ? 1 : 0;
        }
      }
      if (p.observe && sh.screen_now) {
        s.obs_pending = 1;
        s.obs_iter = s.t;
        s.obs_S = S;
        s.obs_radius = sh.radius;
        s.obs_scale_prime = sh.scale_prime;
        s.obs_scale_tilde = sh.scale_tilde;
        s.obs_center_scale = sh.scale_prime;
        s.obs_dict = s.dict_index;
        s.obs_bank = s.cur;
        s.obs_ray_is_y = sh.ray_is_y;
      }
      s.ledger += row_flops(p, s.dict_index, S, sh.nnz);  // ledger + trace (611-623)
      if (!stop_now && lv.kind == kDense)
        s.prof_apply_bytes += 8.0 * static_cast<double>(p.n) * static_cast<double>(sh.nnz);
      if (p.collect_trace && vrank() == 0) {
        fl1_trace_row row;
        row.iter = s.t;
        row.dict_index = s.dict_index;
        row.active_size = static_cast<int32_t>(S);
        row.gap = s.dict_index == last ? sh.gap_tilde : -1.0;
        row.gamma = sh.gamma;
        row.flops_cum = s.ledger;
        row.wall_ms = (globaltimer_ns() - s.t0_ns) * 1e-6;
        row.x_nnz = static_cast<int32_t>(sh.nnz);
        row.pad_ = 0;
        p.trace[s.n_trace] = row;
      }
      if (p.collect_trace) s.n_trace += 1;
    }
    __syncthreads();
    if (stop_now) {
      if (threadIdx.x == 0) {
        s.converged = 1;
        s.final_gap = sh.gap_tilde;
        s.t += 1;
        s.done = 1;
        s.event = kEvDone;
        s.prof_ns[2] += globaltimer_ns() - tp2;
      }
      __syncthreads();
      break;
    }
    const int64_t S_new = sh.S_new;
    const bool shrink = S_new < S;
    if (shrink) {  // apply_restriction: stream compaction into the other bank (686-701)
      const Bank nb = p.bank[s.cur ^ 1];
      if (threadIdx.x < 32) {
        double acc = 0.0;
        for (int b = threadIdx.x; b < vrank(); b += 32)
          acc += __ldcg(p.bred + static_cast<int64_t>(b) * kBred + kSlKept);
        acc = warp_sum(acc);
        if (threadIdx.x == 0) sh.scan_base = static_cast<int64_t>(acc);
      }
      __syncthreads();
      const bool lead_ok = s.lead_valid != 0;
      const bool dyn = p.rule == FL1_RULE_DYNAMIC;
      const bool atye = s.atye_valid != 0;
      int64_t out_base = sh.scan_base;
      double me = -DBL_MAX;
      const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
      for (int64_t q0 = lo; q0 < hi; q0 += kThreads) {
        const int64_t q = q0 + threadIdx.x;
        const int kp = q < hi ? bk.keep[q] : 0;
        const unsigned bal = __ballot_sync(kFull, kp);
        if (l == 0) sh.wscan[w] = __popc(bal);
        __syncthreads();
        int64_t off = out_base;
        int tot = 0;
        for (int ww = 0; ww < kWarps; ++ww) {
          if (ww < w) off += sh.wscan[ww];
          tot += sh.wscan[ww];
        }
        off += __popc(bal & ((1u << l) - 1u));
        if (kp) {
          nb.idx[off] = bk.idx[q];
          nb.x[off] = p.xnew[q];
          if (fista) nb.xp[off] = bk.x[q];  // x_prev = x (581-590)
          nb.eps[off] = bk.eps[q];
          nb.en[off] = bk.en[q];
          nb.an[off] = bk.an[q];
          if (dyn) nb.aty[off] = bk.aty[q];
          if (atye) nb.atye[off] = bk.atye[q];
          if (lead_ok) nb.lead[off] = bk.lead[q];
          me = fmax(me, bk.eps[q]);
        }
        out_base += tot;
        __syncthreads();
      }
      // restrict_to_local copies the kept columns once compacted; maybe_compact copies
      // them from the level's matrix at every halving of the compaction width (115-129, 176-187)
      if (p.compact && lv.kind == kDense && lv.rows == 0 && !gram && (s.csel != 0 || 2 * S_new <= s.cwidth))
        compact_shrink(p, sh, lv, lo, hi, S_new);
      double v[1] = {me};
      const bool mx[1] = {true};
      block_reduce<1>(v, mx, sh);
      if (threadIdx.x == 0) put_slot(p, kSlMaxEps, v[0]);
    } else {  // same positions: x_prev = x, x = x_next on this CTA's slice
      for (int64_t q = lo + threadIdx.x; q < hi; q += kThreads) {
        const bool first = lists && q == lo + threadIdx.x;
        const double xo = first ? xo_pre : bk.x[q];
        if (fista) bk.xp[q] = xo;
        bk.x[q] = first ? xn_pre : p.xnew[q];
      }
    }
    {  // combine u (and v <- u_old - fix), then the next iteration's rho_g
      if (gram) combine_g(p, C_apply, fista, fix_pass);
      else if (lists && colsplit_apply(p, sh, lp, lv)) combine_u_colsplit(p, sh, lv, S, shift_u, fix_pass, m_next, sc.red, lp);
      else if (lists) combine_u_lists(p, sh, lv, S, shift_u, fix_pass, m_next, sc.red, lp);
      else combine_u(p, sh, C_apply, shift_u, fix_pass, m_next);
    }
    if (threadIdx.x == 0) {
      if (fista) {  // 581-590
        if (s.momentum_ready) s.t_k = sh.t_next;
        s.momentum_ready = 1;
      }
      if (shrink) {
        s.cur ^= 1;
        s.S = S_new;
      }
    }
    FL1_MARK(5);
    vsync();  // ------------------------------------------------ sync 3
    FL1_MARK(6);
    if (shrink) {
      grid_reduce(p, sh, 0u, 1u << kSlMaxEps);
      if (threadIdx.x == 0) s.max_eps = S_new > 0 ? sh.res[kSlMaxEps] : 0.0;
      __syncthreads();
    }
    double tp3 = 0.0;
    if (threadIdx.x == 0) {
      tp3 = globaltimer_ns();
      s.prof_ns[2] += tp3 - tp2;
    }
    // Lipschitz refresh after a halving (603-608)
    if (s.S * 2 <= s.active_at_last_l && s.S > 0 && sh.next_dict == s.dict_index) {
      const double sq = s.csel == 0 ? power_iteration(p, sh, lv, p.bank[s.cur], s.S, s.lead_valid != 0, sc)
                                    : compact_power_iteration(p, sh, lv, sc);
      if (threadIdx.x == 0) {
        s.lead_valid = 1;
        s.lipschitz = fmax(sq, 1e-300) * 1.05;
        s.inv_l = 1.0 / s.lipschitz;
        s.active_at_last_l = s.S;
        s.prof_ns[3] += globaltimer_ns() - tp3;
      }
      __syncthreads();
    }
    const int next_dict = sh.next_dict;
    const int sw_speed = sh.speed;
    if (threadIdx.x == 0) s.t += 1;
    __syncthreads();
    if (next_dict != s.dict_index) {  // switch (633-637)
      if (threadIdx.x == 0) {
        if (vrank() == 0) {
          fl1_switch_event ev;
          ev.iter = s.t - 1;
          ev.from = s.dict_index;
          ev.to = next_dict;
          ev.speed = sw_speed;
          ev.pad_ = 0;
          p.sw[s.n_switches] = ev;
        }
        s.n_switches += 1;
        s.dict_index = next_dict;
      }
      __syncthreads();
      double tsw = 0.0;
      if (threadIdx.x == 0) tsw = globaltimer_ns();
      setup_dictionary(p, sh, false, sc);
      if (threadIdx.x == 0) s.prof_ns[4] += globaltimer_ns() - tsw;
    }
    if (s.obs_pending) {
      if (threadIdx.x == 0) s.event = kEvObserve;
      __syncthreads();
      break;
    }
  }
  __syncthreads();
  if (vrank() == 0 && threadIdx.x == 0) {
    s.end_ns = globaltimer_ns();
    *p.st = s;
  }
}

// ============================================================================
// Grid mode (p0.batch == nullptr): one cooperative launch over every SM runs one
// solve. Cluster mode: each thread-block cluster is a virtual grid with its own
// workspace and takes signals from a shared queue (BASELINE config 5: B
// independent run_lasso solves in one launch, cluster barriers instead of grid
// barriers).
__global__ void __launch_bounds__(kThreads, 1) engine_kernel(const __grid_constant__ EngineParams p0) {
  extern __shared__ __align__(16) double dyn[];
  __shared__ Sh sh;
  __shared__ __align__(16) EngineParams sp;
  auto copy_params = [&](const EngineParams* src) {
    const int4* a = reinterpret_cast<const int4*>(src);
    int4* b = reinterpret_cast<int4*>(&sp);
    for (int i = threadIdx.x; i < static_cast<int>(sizeof(EngineParams) / sizeof(int4)); i += kThreads) b[i] = a[i];
  };
  bulk_init_barriers();
  if (p0.batch == nullptr) {
    if (threadIdx.x == 0) {
      s_vsize = gridDim.x;
      s_vrank = blockIdx.x;
      s_vcluster = 0;
    }
    copy_params(&p0);
    __syncthreads();
    engine_body(sp, sh, dyn);
    return;
  }
  cg::cluster_group cl = cg::this_cluster();
  const int csize = static_cast<int>(cl.num_blocks());
  const int cid = blockIdx.x / csize;
  if (threadIdx.x == 0) {
    s_vsize = csize;
    s_vrank = static_cast<int>(cl.block_rank());
    s_vcluster = 1;
  }
  const BatchDesc& bd = *p0.batch;
  copy_params(bd.cluster_params + cid);
  __syncthreads();
  while (true) {
    if (s_vrank == 0 && threadIdx.x == 0) __stcg(bd.cluster_sig + cid, atomicAdd(bd.next, 1));
    cl.sync();
    const int b = __ldcg(bd.cluster_sig + cid);
    cl.sync();
    if (b >= bd.batch) break;
    if (bd.handoff && __ldcg(&bd.handoff[b].state) == 2) continue;  // finished in the lockstep engine
    if (threadIdx.x == 0) {
      sp.mode = kModeSolve;
      sp.lambda = bd.lambdas[b];
      sp.st = bd.states + b;
      sp.trace = bd.traces + static_cast<int64_t>(b) * bd.trace_cap;
      sp.sw = bd.sws + static_cast<int64_t>(b) * kMaxLevels;
      sp.handoff = (bd.handoff && bd.handoff[b].state == 1) ? bd.handoff + b : nullptr;
    }
    {  // y_b into the workspace (zero padded to ld), by CTA slices
      int64_t lo, hi;
      slice(sp.ld, lo, hi);
      double* yw = const_cast<double*>(sp.y);
      for (int64_t i = lo + threadIdx.x; i < hi; i += kThreads)
        yw[i] = i < sp.n ? bd.Y[static_cast<int64_t>(b) * bd.ldy + i] : 0.0;
    }
    __syncthreads();
    cl.sync();
    engine_body(sp, sh, dyn);
    cl.sync();
    {  // finish (fastl1.cpp:741-748): the preserved set and its iterate to the signal's outputs
      // packed: rank 0 reserves S slots and publishes the offset through the state
      const Bank fb = sp.bank[sh.s.cur];
      if (s_vrank == 0 && threadIdx.x == 0) {
        const unsigned long long off =
            atomicAdd(reinterpret_cast<unsigned long long*>(bd.out_used), static_cast<unsigned long long>(sh.s.S));
        bd.out_off[b] = static_cast<int64_t>(off);
      }
      cl.sync();
      const int64_t off = __ldcg(bd.out_off + b);
      int64_t lo, hi;
      slice(sh.s.S, lo, hi);
      for (int64_t q = lo + threadIdx.x; q < hi; q += kThreads) {
        bd.out_idx[off + q] = fb.idx[q];
        bd.out_x[off + q] = fb.x[q];
      }
    }
    __syncthreads();
    cl.sync();
  }
}

// screen_precomputed (screening.cpp:136-150) as a standalone device kernel.
__global__ void screen_kernel(int64_t n, const double* __restrict__ dots, const double* __restrict__ eps,
                              const double* __restrict__ en, const double* __restrict__ an, double cn, double r,
                              int8_t* keep, int8_t* look) {
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < n;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double d = dots[j];
    keep[j] = (d + eps[j] * cn + r * en[j]) >= 1.0 ? 1 : 0;
    look[j] = (d + r * an[j]) >= 1.0 ? 1 : 0;
  }
}

// ---------------------------------------------------------------- host helpers
cudaError_t screen_kernel_launch(int64_t n, const double* dots, const double* eps, const double* en,
                                 const double* an, double cn, double r, int8_t* keep, int8_t* look,
                                 cudaStream_t stream) {
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 4096);
  screen_kernel<<<static_cast<unsigned>(std::max<int64_t>(blocks, 1)), 256, 0, stream>>>(n, dots, eps, en, an, cn, r,
                                                                                         keep, look);
  return cudaGetLastError();
}

// Shared scratch after the resident residual: dense apply warp partials, or the
// SuKro staging (adjoint tiles; apply entry list + 64-column Cg / Bg chunks).
// The run-time tunables below are read ONCE per process (statics): the workspace that
// carves p.scratch_len is cached per context, so the launch's dynamic shared memory and
// the kernel's view of it must never disagree within a process.
namespace FL1_ANON {
int env_int_once(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}
}  // namespace

// Bulk-copy ring stages per warp for a residual of ld doubles (4 KiB each, 8 warps).
// Default 2: power-iteration adjoints stream through a 2-stage bulk-copy ring; the
// ring's shared memory is the engine's scratch, and the smaller carve-out leaves more
// L1 to the register-ring passes (c2 6.66 -> 6.57 ms, c4 897 -> 890 ms against 3
// stages). FL1_BULK_STAGES=R overrides it (0 = register ring everywhere).
int engine_bulk_stages(int64_t ld) {
  static const int stages = env_int_once("FL1_BULK_STAGES", 2);
  const int64_t room = 200 * 1024 / 8 - ld;  // doubles left beside the resident residual
  const int64_t fit = std::max<int64_t>(0, std::min<int64_t>(kMaxBulk, room / (kWarps * kUnit)));
  const int64_t r = std::min<int64_t>(fit, stages);
  return r >= 2 ? static_cast<int>(r) : 0;
}

int64_t engine_scratch_len(int64_t ld, int64_t sukro_m) {
  int64_t s = static_cast<int64_t>(kWarps) * kUnit;
  const int R = engine_bulk_stages(ld);
  if (R >= 2) s = std::max<int64_t>(s, static_cast<int64_t>(R) * kWarps * kUnit);
  if (sukro_m > 0) {
    const int64_t m4 = (sukro_m + 3) / 4 * 4;
    const int64_t term = 16 * m4 + 32 * (m4 + 1);
    s = std::max(s, term + kWarps * 64);                             // adjoint, one term per round
    s = std::max(s, kThreads + kThreads / 2 + 2 * (sukro_m + 1) * 64);  // apply
    const int64_t room = 200 * 1024 / 8 - ld;                        // bounded by the shared memory left
    // SuKro adjoint terms staged per round (default 2, FL1_SUKRO_TERMS overrides): 2 keeps
    // c3's engine in the 132 KiB shared-memory carve-out (more L1 for the exact phase):
    // c3 8.75 -> 8.65 ms against 4
    static const int64_t per_round = std::max(1, env_int_once("FL1_SUKRO_TERMS", 2));
    s = std::max(s, std::min(room, per_round * term + kWarps * 64));
  }
  return s;
}

size_t engine_smem_bytes(int64_t ld, int64_t sukro_m) {
  return static_cast<size_t>(ld + engine_scratch_len(ld, sukro_m)) * sizeof(double);
}

cudaError_t engine_configure(int64_t ld, int64_t sukro_m, int device, int* grid_out) {
  const size_t smem = engine_smem_bytes(ld, sukro_m);
  int optin = 0;
  cudaError_t e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  if (e != cudaSuccess) return e;
  cudaFuncAttributes fa{};
  e = cudaFuncGetAttributes(&fa, engine_kernel);
  if (e != cudaSuccess) return e;
  const int room = optin - static_cast<int>(fa.sharedSizeBytes);  // static: Sh, EngineParams, reduction scratch
  if (static_cast<int64_t>(smem) > room) return cudaErrorInvalidConfiguration;
  e = cudaFuncSetAttribute(engine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, room);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, engine_kernel, kThreads, smem);
  if (e != cudaSuccess) return e;
  int sms = 0;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  *grid_out = sms;  // one persistent CTA per SM
  return cudaSuccess;
}

namespace FL1_ANON {
cudaLaunchConfig_t cluster_config(int n_clusters, int csize, int64_t ld, int64_t sukro_m, cudaLaunchAttribute* at) {
  cudaLaunchConfig_t c{};
  c.gridDim = dim3(static_cast<unsigned>(n_clusters * csize));
  c.blockDim = dim3(kThreads);
  c.dynamicSmemBytes = engine_smem_bytes(ld, sukro_m);
  at->id = cudaLaunchAttributeClusterDimension;
  at->val.clusterDim.x = static_cast<unsigned>(csize);
  at->val.clusterDim.y = 1;
  at->val.clusterDim.z = 1;
  c.attrs = at;
  c.numAttrs = 1;
  return c;
}
}  // namespace

// How many clusters of csize CTAs can be co-resident (engine_configure first).
cudaError_t engine_cluster_capacity(int64_t ld, int64_t sukro_m, int csize, int* n_clusters) {
  if (csize > 8) {
    const cudaError_t e = cudaFuncSetAttribute(engine_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchAttribute at;
  cudaLaunchConfig_t c = cluster_config(1, csize, ld, sukro_m, &at);
  return cudaOccupancyMaxActiveClusters(n_clusters, engine_kernel, &c);
}

cudaError_t engine_launch_clusters(const EngineParams& p0, int n_clusters, int csize, int64_t sukro_m,
                                   cudaStream_t stream) {
  cudaLaunchAttribute at;
  cudaLaunchConfig_t c = cluster_config(n_clusters, csize, p0.ld, sukro_m, &at);
  c.stream = stream;
  return cudaLaunchKernelEx(&c, engine_kernel, p0);
}

cudaError_t engine_launch(const EngineParams& p, int64_t sukro_m, cudaStream_t stream) {
  EngineParams local = p;
  void* args[] = {&local};
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(engine_kernel), dim3(p.grid), dim3(kThreads), args,
                                     engine_smem_bytes(p.ld, sukro_m), stream);
}

}  // namespace fl1
