// Lockstep batched engine (BASELINE configs[4]: many signals, one dictionary).
//
// B independent run_lasso calls share one dense exact dictionary. Every global
// step, each unfinished signal performs its own next unit of Engine::run
// (fastl1.cpp:459-645): one FISTA iteration, or one step of its restricted power
// iteration (solver.cpp:72-104). The dictionary products of all signals are then
// two dense contractions on the fp64 tensor cores (DMMA m8n8k4, cp.async
// double-buffered shared-memory tiles, split-K for load balance):
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

#include <cfloat>
#include <cstdint>

#include "engine.cuh"

namespace cg = cooperative_groups;

namespace fl1 {
namespace {

constexpr int kPT = 256;            // threads per CTA
constexpr int kPW = kPT / 32;
constexpr int kTM = 128, kTN = 64;  // output tile: 128 rows (atoms / samples) x 64 signals
constexpr int kTK = 32;             // K chunk (rows of A / rho)
constexpr int kSS = kTK + 4;        // padded smem row stride (doubles)
constexpr int kStage = (kTM + kTN) * kSS;  // doubles per pipeline stage
constexpr unsigned kAll = 0xffffffffu;
constexpr int kSplitMax = 4;       // split-K parts of the contraction (load balance)

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
__device__ __forceinline__ void cp_wait0() { asm volatile("cp.async.wait_group 0;\n" ::); }

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

// Corr tile (atoms j0..j0+63) x (slots a0..a0+63) over K-part kp of sk (rows of A /
// rho), DMMA, into the split-K partial buffer kp.
__device__ __noinline__ void gemm_tile(const PrefixParams& p, int rt, int ct, int kp, int sk, int64_t n_act,
                                       double* stage) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, g = l >> 2, tg = l & 3;
  const int64_t j0 = static_cast<int64_t>(rt) * kTM, a0 = static_cast<int64_t>(ct) * kTN;
  const int64_t K = p.k, ld = p.ld;
  const int nch = static_cast<int>((ld + kTK - 1) / kTK);
  const int c_lo = nch * kp / sk, c_hi = nch * (kp + 1) / sk;
  double acc[2][8][2];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[h][c][0] = acc[h][c][1] = 0.0;
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
    for (int e0 = 0; e0 < kTN * (kTK / 2); e0 += kPT) {  // R columns (slots)
      const int e = e0 + threadIdx.x;
      const int c = e / (kTK / 2), kk = (e % (kTK / 2)) * 2;
      const int64_t a = a0 + c, kg = k0 + kk;
      const bool ok = a < n_act && kg < ld;
      cp16(Rs + c * kSS + kk, ok ? p.R + a * ld + kg : p.R, ok);
    }
  };
  if (c_lo < c_hi) issue(0, c_lo);
  cp_commit();
  for (int kc = c_lo; kc < c_hi; ++kc) {
    if (kc + 1 < c_hi) issue((kc + 1 - c_lo) & 1, kc + 1);
    cp_commit();
    cp_wait1();
    __syncthreads();
    const double* As = stage + ((kc - c_lo) & 1) * kStage;
    const double* Rs = As + kTM * kSS;
#pragma unroll
    for (int ks = 0; ks < kTK / 4; ++ks) {
      const double a0v = As[(w * 8 + g) * kSS + ks * 4 + tg];
      const double a1v = As[(64 + w * 8 + g) * kSS + ks * 4 + tg];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const double bv = Rs[(c * 8 + g) * kSS + ks * 4 + tg];
        dmma(acc[0][c], a0v, bv);
        dmma(acc[1][c], a1v, bv);
      }
    }
    __syncthreads();
  }
  cp_wait0();
  double* __restrict__ out = p.corr + static_cast<int64_t>(kp) * K * p.bcap;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t j = j0 + h * 64 + w * 8 + g;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int64_t a = a0 + c * 8 + 2 * tg + i;
        if (j < K && a < n_act) __stcg(out + a * K + j, acc[h][c][i]);
      }
    }
  }
}

// split-K factor for T output tiles on G CTAs: split only while the tiles alone
// leave more than a third of the CTAs idle (partials cost a write + read each)
__device__ __forceinline__ int split_for(int T, int G) {
  int s = 1;
  while (s < kSplitMax && 3 * T * s < 2 * G) s *= 2;
  return s;
}

// ---------------------------------------------------------------------------
// W = A V tile: rows i0..i0+63 of ld, power slots c0..c0+63 (index into pact),
// atoms of K-part kp of sk; partial into np[kp][pslot][ld].
__device__ __noinline__ void gemm_n_tile(const PrefixParams& p, int rt, int ct, int kp, int sk, int n_pow,
                                         const int32_t* pact, const int32_t* act, double* stage) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, g = l >> 2, tg = l & 3;
  const int64_t i0 = static_cast<int64_t>(rt) * kTM, c0 = static_cast<int64_t>(ct) * kTN;
  const int64_t K = p.k, ld = p.ld;
  constexpr int kAS = kTM + 4;  // As[kk][i] row stride
  const int nch = static_cast<int>((K + kTK - 1) / kTK);
  const int c_lo = nch * kp / sk, c_hi = nch * (kp + 1) / sk;
  double acc[2][8][2];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[h][c][0] = acc[h][c][1] = 0.0;
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
    for (int e0 = 0; e0 < kTN * (kTK / 2); e0 += kPT) {  // V(k, slot): slot-major, k contiguous
      const int e = e0 + threadIdx.x;
      const int c = e / (kTK / 2), kk = (e % (kTK / 2)) * 2;
      const int64_t pc = c0 + c, kg = k0 + kk;
      const bool ok = pc < n_pow && kg < K;
      const int64_t b = ok ? act[pact[pc]] : 0;
      cp16(Bs + c * kSS + kk, ok ? p.vp + b * K + kg : p.vp, ok);
    }
  };
  if (c_lo < c_hi) issue(0, c_lo);
  cp_commit();
  for (int kc = c_lo; kc < c_hi; ++kc) {
    if (kc + 1 < c_hi) issue((kc + 1 - c_lo) & 1, kc + 1);
    cp_commit();
    cp_wait1();
    __syncthreads();
    const double* As = stage + ((kc - c_lo) & 1) * kStage;
    const double* Bs = As + kTK * kAS;
#pragma unroll
    for (int ks = 0; ks < kTK / 4; ++ks) {
      const double a0v = As[(ks * 4 + tg) * kAS + w * 8 + g];
      const double a1v = As[(ks * 4 + tg) * kAS + 64 + w * 8 + g];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const double bv = Bs[(c * 8 + g) * kSS + ks * 4 + tg];
        dmma(acc[0][c], a0v, bv);
        dmma(acc[1][c], a1v, bv);
      }
    }
    __syncthreads();
  }
  cp_wait0();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t i = i0 + h * 64 + w * 8 + g;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int64_t pc = c0 + c * 8 + 2 * tg + q;
        if (i < ld && pc < n_pow) __stcg(p.np + (static_cast<int64_t>(kp) * p.bcap + pc) * ld + i, acc[h][c][q]);
      }
    }
  }
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

// u (or v) += sum over listed atoms of coef * a_j, rows over threads, list order
__device__ __forceinline__ void apply_list(const PrefixParams& p, double* us, const double* ent_v,
                                           const int32_t* ent_j, int n) {
  for (int64_t i = threadIdx.x; i < p.ld; i += kPT) {
    double acc = us[i];
#pragma unroll 4
    for (int e = 0; e < n; ++e) acc = fma(ent_v[e], __ldg(p.a + static_cast<int64_t>(ent_j[e]) * p.ld + i), acc);
    us[i] = acc;
  }
  __syncthreads();
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

// corr column of slot a: sum of the split-K parts (fixed order) written back to part
// 0; returns the block max of |corr| over the preserved atoms
__device__ double combine_corr(const PrefixParams& p, PSh& sh, int64_t a, int64_t b, int sk) {
  const int64_t K = p.k, part = K * p.bcap;
  double* cr = p.corr + a * K;
  const int8_t* mk = p.mask + b * K;
  double dp = 0.0;
  for (int64_t j = threadIdx.x; j < K; j += kPT) {
    double c = __ldcg(cr + j);
    for (int kp = 1; kp < sk; ++kp) c += __ldcg(cr + kp * part + j);
    if (sk > 1) __stcg(cr + j, c);
    if (mk[j]) dp = fmax(dp, fabs(c));
  }
  return block_max(dp, sh);
}

// Enter the restricted power iteration (power_iteration_sq_norm, solver.cpp:72-104):
// warm from the gathered leading vector when it is nonzero, else the fixed Gaussian
// start by preserved position.
__device__ void enter_power(const PrefixParams& p, PSh& sh, int64_t b) {
  PrefixSig& sg = p.sig[b];
  const int64_t K = p.k;
  const int8_t* mk = p.mask + b * K;
  const double* ldv = p.lead + b * K;
  double* src = p.psrc + b * K;
  double* vp = p.vp + b * K;
  double a_lead = 0.0;
  if (sg.lead_valid)
    for (int64_t j = threadIdx.x; j < K; j += kPT)
      if (mk[j]) a_lead = fma(ldv[j], ldv[j], a_lead);
  a_lead = block_sum(a_lead, sh);
  const bool warm = sg.lead_valid && a_lead > 0.0;
  double nrm2 = 0.0;
  if (warm) {
    for (int64_t j = threadIdx.x; j < K; j += kPT) src[j] = mk[j] ? ldv[j] : 0.0;
    nrm2 = a_lead;
  } else {
    int tot = 0;
    double acc = 0.0;
    for (int64_t base = 0; base < K; base += kPT) {
      const int64_t j = base + threadIdx.x;
      const bool on = j < K && mk[j] != 0;
      int at;
      tot = block_compact(sh, on, tot, &at);
      if (j < K) {
        const double gv = on ? p.gauss0[at] : 0.0;
        src[j] = gv;
        acc = fma(gv, gv, acc);
      }
    }
    nrm2 = block_sum(acc, sh);
  }
  const double div = sqrt(nrm2);
  __syncthreads();
  for (int64_t j = threadIdx.x; j < K; j += kPT) vp[j] = src[j] / div;
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

// One power step's update after v_new = A_S^T A_S v (slot a's corr column).
__device__ __noinline__ void power_step(const PrefixParams& p, PSh& sh, int64_t a, int64_t b, int sk, double t0) {
  PrefixSig& sg = p.sig[b];
  const int64_t K = p.k;
  (void)combine_corr(p, sh, a, b, sk);
  const double* cr = p.corr + a * K;
  const int8_t* mk = p.mask + b * K;
  double* src = p.psrc + b * K;
  double* vp = p.vp + b * K;
  double w2 = 0.0, vw = 0.0;
  for (int64_t j = threadIdx.x; j < K; j += kPT) {
    if (!mk[j]) continue;
    const double vn = __ldcg(cr + j);
    w2 = fma(vn, vn, w2);
    vw = fma(vp[j], vn, vw);
  }
  w2 = block_sum(w2, sh);
  vw = block_sum(vw, sh);
  if (threadIdx.x == 0) {
    sg.power_steps += 1;
    const double nrm = sqrt(w2);
    int stop = 0;
    double est = sg.p_est;
    if (nrm == 0.0) {
      est = 0.0;
      stop = 2;  // lead = have_w ? w / div : v  (w = 0 here)
    } else {
      const double prev = est;
      est = vw;
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
  if (stop == 2) {  // |w| == 0
    for (int64_t j = threadIdx.x; j < K; j += kPT) p.lead[b * K + j] = sg.p_have_w ? 0.0 : vp[j];
  } else {
    for (int64_t j = threadIdx.x; j < K; j += kPT) {
      const double vn = mk[j] ? __ldcg(cr + j) : 0.0;
      src[j] = vn;
      const double v1 = vn / div;
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
  if (stop && p.policy == 2) handoff_signal(p, sh, b, t0);
}

// One FISTA / ISTA iteration of signal b (slot a): fastl1.cpp:459-645 with the
// exact dictionary, GAP rule, preserved set = mask.
__device__ __noinline__ void fista_step(const PrefixParams& p, PSh& sh, int64_t a, int64_t b, double t0, int sk,
                                        double* us, double* stage) {
  PrefixSig& sg = p.sig[b];
  const int64_t K = p.k, ld = p.ld;
  const double lambda = p.lambdas[b];
  const uint64_t t = sg.t;
  const double dp = combine_corr(p, sh, a, b, sk);
  const double* cr = p.corr + a * K;
  int8_t* mk = p.mask + b * K;
  if (threadIdx.x == 0) {
    double m = 0.0, t_next = sg.t_k;  // 465-470
    if (p.solver == FL1_FISTA && sg.ready) {
      t_next = 0.5 * (1.0 + sqrt(1.0 + 4.0 * sg.t_k * sg.t_k));
      m = (sg.t_k - 1.0) / t_next;
    }
    const double rsq = sg.rsq, rdy = sg.rdy;
    const double rho_x_sq = m != 0.0 ? sg.ree : rsq;
    const double primal = 0.5 * rho_x_sq + lambda * sg.x_l1;
    int rel = 0, screen = 0;
    double sp = 0.0, radius = 0.0, gt = 0.0;
    if (!(rsq > 0.0)) {
      rel = 3;  // exact fit: the per-signal engine takes the y-ray branch (428-449)
    } else {
      const double projection = rdy / (lambda * rsq);  // dual_scalars (406-450), eps = 0
      const double ap = (sg.S > 0 && dp > 0) ? 1.0 / dp : CUDART_INF;
      sp = fmin(fmax(projection, -ap), ap);
      const double dist_sq = sp * sp * rsq - 2.0 * sp * rdy / lambda + sg.y_sq / (lambda * lambda);
      const double dual = 0.5 * sg.y_sq - 0.5 * lambda * lambda * dist_sq;  // 453-457
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
  if (sh.release == 3) {
    handoff_signal(p, sh, b, t0);
    return;
  }
  const int rot = sg.rot;
  double* __restrict__ xc = p.X3[rot % 3] + b * K;
  double* __restrict__ xpc = p.X3[(rot + 1) % 3] + b * K;
  double* __restrict__ xn = p.X3[(rot + 2) % 3] + b * K;
  const int64_t S_old = sg.S;
  const int cap = 2 * kStage / 3 - kPT;  // list entries (value + index) in the staging area
  double* ent_v = stage;
  int32_t* ent_j = reinterpret_cast<int32_t*>(stage + 2 * kStage / 3);
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
  // screening (494-566; stable test with eps = 0) and prox (572-579) over the set
  const double m = sh.m, inv_l = sg.inv_l, thresh = lambda * sg.inv_l;
  const bool screen = sh.screen != 0;
  const double spv = sh.sp, rad = sh.radius;
  double kept = 0.0;
  for (int64_t j = threadIdx.x; j < K; j += kPT) {
    double v = 0.0;
    if (mk[j]) {
      const double c = __ldcg(cr + j);
      const double xo = xc[j];
      const double xpv = m != 0.0 ? xpc[j] : 0.0;
      const double gg = m != 0.0 ? __fma_rn(1.0 + m, xo, -__dmul_rn(m, xpv)) : xo;
      const double z = __fma_rn(inv_l, c, gg);
      const double mag = fabs(z) - thresh;
      v = mag <= 0.0 ? 0.0 : (z > 0.0 ? mag : -mag);
      if (screen) {
        const double d = fabs(__dmul_rn(spv, c));
        if (__fma_rn(rad, p.en[j], d) >= 1.0) kept += 1.0;
        else mk[j] = 2;  // dropped at this instant
      } else {
        kept += 1.0;
      }
    }
    xn[j] = v;
  }
  kept = block_sum(kept, sh);
  const int64_t S_new = static_cast<int64_t>(kept);
  if (p.policy == 1 && S_new < S_old) {  // leave at the start of this iteration
    for (int64_t j = threadIdx.x; j < K; j += kPT)
      if (mk[j] == 2) mk[j] = 1;
    __syncthreads();
    handoff_signal(p, sh, b, t0);
    return;
  }
  const bool fista = p.solver == FL1_FISTA;
  // FISTA bookkeeping (581-590): x_prev = x, v = u; x = x_next. Roles rotate: the
  // new x_prev is the old x buffer, the new x the x_next buffer; v takes u's buffer.
  double* __restrict__ xnew = xn;
  double* __restrict__ xprev = xc;
  const double* __restrict__ uo = p.U2[sg.uswap] + b * ld;   // u = old u  -> becomes v
  double* __restrict__ un = p.U2[1 - sg.uswap] + b * ld;      // new u
  // apply_restriction (667-702): v -= x_prev_j a_j over dropped atoms (FISTA, momentum
  // ready after the shift above), then the dropped atoms leave x, x_prev, lead
  for (int64_t i = threadIdx.x; i < ld; i += kPT) us[i] = fista ? uo[i] : 0.0;
  __syncthreads();
  if (S_new < S_old) {
    int tot = 0;
    for (int64_t base = 0; base < K; base += kPT) {
      const int64_t j = base + threadIdx.x;
      double v = 0.0;
      if (j < K && mk[j] == 2) {
        if (fista && xprev[j] != 0.0) v = -xprev[j];
        mk[j] = 0;
        xnew[j] = 0.0;
        xprev[j] = 0.0;
        p.lead[b * K + j] = 0.0;
      }
      int at;
      const int ntot = block_compact(sh, v != 0.0, tot, &at);
      if (v != 0.0) {
        ent_v[at] = v;
        ent_j[at] = static_cast<int32_t>(j);
      }
      tot = ntot;
      if (tot > cap - kPT) {
        apply_list(p, us, ent_v, ent_j, tot);
        tot = 0;
      }
    }
    apply_list(p, us, ent_v, ent_j, tot);
  }
  // the v buffer (old u, fixed) is final; u = A x over the nonzeros of the new x
  if (fista)
    for (int64_t i = threadIdx.x; i < ld; i += kPT) const_cast<double*>(uo)[i] = us[i];
  for (int64_t i = threadIdx.x; i < ld; i += kPT) us[i] = 0.0;
  __syncthreads();
  double nnz = 0.0, l1n = 0.0;
  {
    int tot = 0;
    for (int64_t base = 0; base < K; base += kPT) {
      const int64_t j = base + threadIdx.x;
      const double v = j < K ? xnew[j] : 0.0;
      nnz += v != 0.0 ? 1.0 : 0.0;
      l1n += fabs(v);
      int at;
      const int ntot = block_compact(sh, v != 0.0, tot, &at);
      if (v != 0.0) {
        ent_v[at] = v;
        ent_j[at] = static_cast<int32_t>(j);
      }
      tot = ntot;
      if (tot > cap - kPT) {
        apply_list(p, us, ent_v, ent_j, tot);
        tot = 0;
      }
    }
    apply_list(p, us, ent_v, ent_j, tot);
  }
  nnz = block_sum(nnz, sh);
  l1n = block_sum(l1n, sh);
  for (int64_t i = threadIdx.x; i < ld; i += kPT) un[i] = us[i];
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
    // restricted Lipschitz refresh when the set halved (603-608)
    sh.screen = (S_new * 2 <= sg.active_at_last_l && S_new > 0) ? 1 : 0;
  }
  __syncthreads();
  if (sh.screen) enter_power(p, sh, b);
}

}  // namespace

__global__ void __launch_bounds__(kPT, 1) prefix_kernel(const __grid_constant__ PrefixParams p) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double dsm[];
  __shared__ PSh sh;
  const int64_t B = p.batch, K = p.k, N = p.n, ld = p.ld;
  const double t0 = gtimer();
  // dynamic smem: [staging x2 (contraction tiles; lists in the per-signal steps) | u | act | pact]
  double* stage = dsm;
  double* us = stage + 2 * kStage;
  int32_t* act = reinterpret_cast<int32_t*>(us + ld);
  int32_t* pact = act + B;
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
  }
  grid.sync();
  int32_t steps = 0;
  for (;; ++steps) {
    // unfinished signals in signal order, and the ones in a power step (identical in every CTA)
    int n_act = 0, n_pow = 0;
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
      n_act = na;
      n_pow = np;
    }
    if (n_act == 0) break;
    if (p.step_log && blockIdx.x == 0 && threadIdx.x == 0 && steps < p.max_log) {
      p.step_log[3 * steps] = n_act;
      p.step_log[3 * steps + 1] = n_pow;
      p.step_log[3 * steps + 2] = gtimer() - t0;
    }
    // ---- FISTA signals: compute_products (359-369) rho_g with its norms; max_iterations
    for (int64_t a = blockIdx.x; a < n_act; a += gridDim.x) {
      const int64_t b = act[a];
      PrefixSig& sg = p.sig[b];
      if (__ldcg(&sg.mode) != 0) continue;
      if (sg.t >= p.max_it) {  // fastl1.cpp:640-644
        finish_signal(p, sh, b, false, 0.0, t0);
        for (int64_t i = threadIdx.x; i < ld; i += kPT) __stcg(p.R + a * ld + i, 0.0);
        continue;
      }
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
        __stcg(p.R + a * ld + i, r);
      }
      block_sum3(v, sh);
      if (threadIdx.x == 0) {
        sg.rsq = v[0];
        sg.rdy = v[1];
        sg.ree = v[2];
      }
    }
    // ---- power-step signals: w = A_S v (one contraction), then summed into R
    if (n_pow > 0) {
      grid.sync();
      const int n_rt = static_cast<int>((ld + kTM - 1) / kTM);
      const int n_ct = (n_pow + kTN - 1) / kTN;
      const int sk = split_for(n_rt * n_ct, gridDim.x);
      for (int item = blockIdx.x; item < n_rt * n_ct * sk; item += gridDim.x) {
        const int tile = item % (n_rt * n_ct), kp = item / (n_rt * n_ct);
        gemm_n_tile(p, tile % n_rt, tile / n_rt, kp, sk, n_pow, pact, act, stage);
      }
      grid.sync();
      for (int64_t e = static_cast<int64_t>(blockIdx.x) * kPT + threadIdx.x; e < static_cast<int64_t>(n_pow) * ld;
           e += static_cast<int64_t>(gridDim.x) * kPT) {
        const int64_t pc = e / ld, i = e - pc * ld;
        double w = 0.0;
        for (int kp = 0; kp < sk; ++kp) w += __ldcg(p.np + (static_cast<int64_t>(kp) * p.bcap + pc) * ld + i);
        __stcg(p.R + static_cast<int64_t>(pact[pc]) * ld + i, i < N ? w : 0.0);
      }
    }
    grid.sync();
    // ---- Corr = A^T [rho | w] for every unfinished signal (fp64 tensor cores)
    const int n_rt = static_cast<int>((K + kTM - 1) / kTM);
    const int n_ct = (n_act + kTN - 1) / kTN;
    const int sk = split_for(n_rt * n_ct, gridDim.x);
    for (int item = blockIdx.x; item < n_rt * n_ct * sk; item += gridDim.x) {
      const int tile = item % (n_rt * n_ct), kp = item / (n_rt * n_ct);
      gemm_tile(p, tile % n_rt, tile / n_rt, kp, sk, n_act, stage);
    }
    grid.sync();
    // ---- the rest of each signal's unit of work, one signal per CTA
    for (int64_t a = blockIdx.x; a < n_act; a += gridDim.x) {
      const int64_t b = act[a];
      const int mode = __ldcg(&p.sig[b].mode);
      if (mode == 0) fista_step(p, sh, a, b, t0, sk, us, stage);
      else if (mode == 1) power_step(p, sh, a, b, sk, t0);
    }
    grid.sync();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && p.steps_out) *p.steps_out = steps;
}

size_t prefix_smem_bytes(int64_t ld, int64_t batch) {
  return static_cast<size_t>(2 * kStage + ld) * sizeof(double) + static_cast<size_t>(2 * batch) * sizeof(int32_t);
}
int prefix_split_max() { return kSplitMax; }

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

}  // namespace fl1
