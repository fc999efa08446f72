// engine.cuh — data layout shared by the host side (api.cpp) and the persistent
// engine kernel (engine.cu). Everything here lives in HBM; the kernel keeps a
// per-CTA copy of the scalar state (EngineState) in shared memory, and every
// CTA evolves it identically from identical, fixed-order reductions, so no
// scalar ever needs a host round trip.
#pragma once

#include <cuda.h>  // CUtensorMap (the lockstep contraction's TMA descriptors)

#include <cstdint>

#include "../../include/fl1cuda.h"

namespace fl1 {

constexpr int kMaxLevels = 8;
#ifndef FL1_THREADS
#define FL1_THREADS 256
#endif
#ifndef FL1_RING
#define FL1_RING 2  // register ring depth of the streaming passes (2: no spills at 255 regs)
#endif
#ifndef FL1_UNIT
#define FL1_UNIT 512
#endif
constexpr int kThreads = FL1_THREADS;  // one persistent CTA of 8 warps per SM (255 registers/thread)
constexpr int kWarps = kThreads / 32;
constexpr int kUnit = FL1_UNIT;  // doubles per A^T r work unit (one column segment)

enum OpKind : int32_t { kDense = 0, kSukro = 1 };

// One level of the ApproxSequence as the device sees it (dictionary.hpp:111-120).
struct DevLevel {
  int32_t kind;
  int32_t nterms;
  int64_t m, q;             // SuKro side lengths (N = m^2, K = q^2)
  const double* a;          // dense: column-major, leading dimension ld
  const double* left;       // SuKro: nterms blocks of m x q (B_t), column-major
  const double* right;      // SuKro: nterms blocks of m x q (C_t)
  const double* col_scale;  // SuKro column scale (extension), nullable
  const double* eps;        // K: atom_error_bounds
  const double* an;         // K: approx_atom_norms2
  const double* en;         // K: exact_atom_norms2
  double op_err;
  double rc;
  uint64_t matvec_flops;
  int64_t rows, ld;         // dense operator shape when not the dictionary's (Gram: K, ldG); 0 = p.n, p.ld
};

// Per-atom arrays over the preserved set, in position order (ActiveOp state,
// fastl1.cpp:203-210, plus the Engine's compact vectors, 226-247). Two banks:
// a shrinking screening pass compacts bank[cur] into bank[cur^1].
struct Bank {
  int32_t* idx;   // global column index
  double* x;      // iterate
  double* xp;     // FISTA history
  double* eps;    // gathered atom_error_bounds
  double* en;     // gathered exact norms
  double* an;     // gathered approx norms
  double* aty;    // Atilde^T y (dynamic rule)
  double* atye;   // A^T y (precompute_aty variant)
  double* lead;   // power-iteration leading vector
  int8_t* keep;   // screening decision of the last pass
};

enum Mode : int32_t { kModeSolve = 0, kModeResume = 1, kModePower = 2, kModeApply = 3, kModeAdjoint = 4 };
enum Event : int32_t { kEvNone = 0, kEvDone = 1, kEvTraceFull = 2, kEvObserve = 3 };

// Scalar engine state (Engine members, fastl1.cpp:213-252), persisted in HBM
// between launches (trace flush / observer) and mirrored in every CTA.
struct EngineState {
  uint64_t t;
  uint64_t ledger;
  uint64_t trace_base;   // iteration index of trace row 0 in the device buffer
  int64_t S;             // preserved-set size
  int64_t active_at_last_l;
  int64_t n_trace;       // rows in the device trace buffer
  int64_t power_steps;
  int64_t launches;
  double t_k;
  double lipschitz;
  double inv_l;
  double max_eps;
  double y_sq;
  double y_norm;
  double final_gap;
  double t0_ns;          // %globaltimer at run() start
  double start_ns;       // %globaltimer at kernel start (solve mode)
  double end_ns;         // %globaltimer at the final state write
  int32_t dict_index;
  int32_t cur;           // current bank
  int32_t momentum_ready;
  int32_t warning;
  int32_t u_chunks;      // partial chunks holding u = A x
  int32_t fix_pending;   // dvp holds a v correction to apply
  int32_t lead_valid;    // bank lead holds S entries
  int32_t atye_valid;
  int32_t gram_mode;     // exact phase on the Gram matrix (fastl1.cpp:278-281)
  int32_t atyf_valid;    // aty_full holds A^T y over all K atoms
  int32_t n_switches;
  int32_t converged;
  int32_t event;
  int32_t done;
  // observer snapshot of the last screening instant
  uint64_t obs_iter;
  int64_t obs_S;
  double obs_radius;
  double obs_scale_prime;
  double obs_scale_tilde;
  double obs_center_scale;  // center = obs_center_scale * ray (ray = rho or y)
  int32_t obs_dict;
  int32_t obs_bank;
  int32_t obs_ray_is_y;
  int32_t obs_pending;
  // mode results
  double power_est;
  // device-side phase profile (block 0, %globaltimer ns): A+sync1, B+sync2,
  // D+sync3, power iteration, switch setup; bytes of A^T r streamed
  double prof_ns[6];
  double prof_bytes;
  double prof_apply_bytes;
  double prof_power_bytes;
  double prof_full_ns;     // A-phase time of full-dictionary passes (|S| = K)
  double prof_full_bytes;
  double prof_pw[4];  // power-iteration sub-phases: apply, combine, adjoint+norms, reduce
  // physical compaction (FL1_COMPACT, ActiveOp::maybe_compact / restrict_to_local,
  // fastl1.cpp:115-129, 176-187): 0 = the streaming passes gather columns of the level's
  // matrix by index; 1 / 2 = they read the compact copy in EngineParams::cbuf[csel - 1]
  int64_t cwidth;  // compaction_width_
  int32_t csel;
  int32_t cpad_;
};

struct EngineParams;

// Batched lockstep engine -> per-signal engine hand-off (batched solves): the state
// of one signal at the START of iteration t, preserved set compacted in atom order.
struct Handoff {
  const int32_t* idx;   // S preserved atoms, ascending
  const double* x;      // S
  const double* xp;     // S
  const double* lead;   // S (valid if lead_valid)
  const double* u;      // ld
  const double* v;      // ld
  uint64_t t;
  uint64_t ledger;
  int64_t n_trace;
  int64_t S;
  int64_t active_at_last_l;
  int64_t power_steps;
  double t_k;
  double lipschitz;
  double elapsed_ns;    // device time the lockstep spent on this signal
  int32_t ready;
  int32_t warning;
  int32_t lead_valid;
  int32_t state;        // 0: not handled, 1: resume from this state, 2: finished in the lockstep
};

// Per-signal state of the lockstep engine.
struct PrefixSig {
  double t_k, x_l1, y_sq, rsq, rdy, ree;
  double lipschitz, inv_l;
  double p_est, p_div, p_tol;   // power iteration: estimate, |cur_src|, tolerance
  uint64_t t, ledger;
  int64_t n_trace, S, active_at_last_l, power_steps;
  int32_t ready, warning, lead_valid;
  int32_t mode;                 // 0: FISTA iteration, 1: power step, 2: finished, 3: handed off
  int32_t rot;                  // roles of X3: x = X3[rot], x_prev = X3[rot+1], x_next = X3[rot+2] (mod 3)
  int32_t uswap;                // u = U2[uswap], v = U2[1 - uswap]
  int32_t p_it, p_max, p_min, p_have_w;
};

// Lockstep batched engine: B independent solves on one dense exact dictionary (GAP
// rule, cached full Lipschitz constant). Every global step, each unfinished signal
// performs its own next unit of Engine::run — one FISTA iteration, or one step of
// its restricted power iteration — and the dictionary products of all of them are
// two dense contractions on the fp64 tensor cores: W = A V for the signals in a
// power step, Corr = A^T [rho | w] for all. Preserved sets are per-signal masks
// (atom order = the reference's compacted order).
struct PrefixParams {
  // TMA descriptors of A for the stream-K contractions (FL1_LOCKSTEP_TMA): dims (ld, k),
  // boxes over-fetched into the padded shared-memory layouts of the DMMA tiles
  CUtensorMap tm_corr;        // box {36 rows, 128 atoms}: Corr tile [atom][36]
  CUtensorMap tm_w;           // box {132 rows, 32 atoms}: W tile [atom][132]
  CUtensorMap tm_rc;          // Rc (ld x bcap), box {36 rows, 64 slots}: Corr R tile [slot][36]
  CUtensorMap tm_vc;          // Vc (k x bcap), box {36 atoms, 64 power slots}: W V tile [slot][36]
  double* rc;                 // ld x bcap: the step's contraction input columns in slot order
  double* vc;                 // k x bcap: the step's power-iteration vectors in power-slot order
  int32_t tma;                // 1: stream-K TMA contractions; 0: split-K cp.async tiles
  int32_t sk_fanin;           // shared tiles with <= this many contributors: one reducer (FL1_SK_FANIN)
  double* sk_trace;           // diagnostics (FL1_SK_TRACE=step): per product, per CTA: start, units done, end
  int32_t sk_trace_step;
  double* part;               // grid x 8192: stream-K partial tiles (one per CTA)
  int32_t* flags;             // grid: stream-K partial-ready epochs (zeroed by the kernel)
  int64_t n, k, ld;
  int32_t batch, bcap;        // signals; column capacity of R / corr (multiple of 64)
  const double* a;            // ld x k, zero-padded rows
  const double* en;           // exact atom norms
  const double* gauss0;       // cold power-iteration start (by preserved position)
  const double* y;            // N x B, leading dimension ldy
  int64_t ldy;
  const double* lambdas;
  double lipschitz;           // cached full-dictionary L
  double tol, rel_tol;
  uint64_t max_it;
  int32_t interval, solver, variant, collect_trace;
  int32_t policy;             // hand-off: 0 never, 1 at the first shrink, 2 after the first power iteration,
                              // 3 at the first iteration after it with |S| <= handoff_s
  int64_t handoff_s;
  int32_t split_mode;         // split-K choice of the contractions: 1 fewest waves, 0 fill-only (FL1_SPLIT_MODE)
  int32_t narrow;             // 1: steps with <= 12 unfinished signals use the CUDA-core products (FL1_LOCKSTEP_NARROW)
  double* sigprof;            // diagnostics builds (FL1_SIGPROF): 16 accumulators, CTA 0's per-signal phases
  int64_t split_budget;       // bytes of split-K partials per contraction (FL1_SPLIT_BUDGET_MB; 0 = unlimited)
  int32_t width_tiles;        // 1: contraction tiles 16 / 32 / 64 signals wide by step width (FL1_LOCKSTEP_WIDTH)
  int64_t* work_out;          // [2]: sum over steps of the unfinished / power-step signal counts
  double* X3[3];              // three k x B iterate buffers (roles rotate, PrefixSig::rot)
  double* U2[2];              // two ld x B buffers for u and v (PrefixSig::uswap)
  int8_t* mask;               // k x B preserved-set masks
  double* lead;               // k x B leading vectors (masked)
  double* psrc;               // k x B power iteration: cur_src
  double* vp;                 // k x B power iteration: v = cur_src / |cur_src| (contraction input)
  int32_t* hidx;              // k x B hand-off: compacted preserved atoms
  double* R;                  // ld x bcap: contraction input columns (rho or w)
  double* np;                 // kSplitMax x bcap x ld: W = A V split-K partials
  double* corr;               // kSplitMax x k x bcap: A^T R split-K partials
  PrefixSig* sig;             // B
  Handoff* hand;              // B (out)
  EngineState* states;        // B final states of signals finished here (host reads them)
  fl1_switch_event* sws;      // unused (single level)
  int64_t* out_used;          // packed final sets (shared with the cluster engine)
  int64_t* out_off;
  int32_t* out_idx;
  double* out_x;
  fl1_trace_row* traces;      // B x trace_cap
  int64_t trace_cap;
  int32_t* steps_out;         // global steps executed
  int32_t* queue;             // two per-step signal-queue counters (per-signal phase)
  double* step_log;           // nullable: per step (n_act, n_pow, %globaltimer) x max_log
  int32_t max_log;
};

// Batched (cluster) mode: B independent solves of one sequence, one per signal,
// taken from a queue by thread-block clusters (each cluster = one workspace).
struct BatchDesc {
  int32_t batch;
  int32_t* next;                        // work counter (starts at 0)
  int32_t* cluster_sig;                 // per cluster: signal being solved
  const EngineParams* cluster_params;   // per cluster: workspace + problem (grid = cluster size)
  const double* Y;                      // N x B, leading dimension ldy
  int64_t ldy;
  const double* lambdas;                // B
  EngineState* states;                  // B: initial state in, final state out
  fl1_trace_row* traces;                // B x trace_cap
  int64_t trace_cap;
  fl1_switch_event* sws;                // B x kMaxLevels
  int64_t* out_used;                    // packed-output counter (starts at 0)
  const Handoff* handoff;               // nullable: B lockstep-prefix states to resume from
  int64_t* out_off;                     // B: offset of each signal's final set
  int32_t* out_idx;                     // packed final preserved sets (capacity B x K)
  double* out_x;                        // iterate on them
};

struct alignas(16) EngineParams {
  int32_t mode;
  int32_t grid;
  int64_t n, k, ld;
  int32_t n_levels;
  DevLevel lv[kMaxLevels];
  double lambda;
  // SwitchConfig
  double gamma_threshold;
  int32_t interval;
  int32_t precompute_aty;
  double tol;
  double rel_tol;
  uint64_t max_it;
  // RunOptions
  int32_t solver, rule, variant;
  int32_t has_full_l;
  double full_l[kMaxLevels];
  int32_t collect_trace;
  int32_t observe;
  int32_t has_x_init;
  int32_t mode_level;  // level used by Power / Apply / Adjoint modes
  // vectors (length ld, zero padded)
  const double* y;
  const double* x_init;  // length K (solve) or K (apply mode input)
  double* U;    // u = A x (combined)
  double* V;    // v = A x_prev (before a pending fix)
  double* rho;  // rho_g of the next iteration (written by the combine phase)
  double* rho_obs;  // rho_g snapshot of the last screening instant (observer)
  double* up;   // apply partials: chunk-major, ld each
  double* dvp;  // v-fix partials
  double* pup;  // power-iteration apply partials
  double* vec_out;  // Apply/Adjoint mode output (length ld or K)
  double* corr;     // K
  double* xnew;     // K: prox output of the current bank positions (phase B -> E)
  double* corr_y;   // K (exact-fit fallback)
  double* part;     // K * units-per-column
  int32_t* cnt;     // K column-completion counters
  // dense phase B -> E: each CTA's kept nonzeros of x_next and the v-fix entries of its
  // dropped atoms, in position order at the CTA's slice offset, counts per CTA
  double* nzv;
  int32_t* nzj;
  double* fxv;
  int32_t* fxj;
  int32_t* lcnt;    // [grid] apply counts, [grid] fix counts
  int32_t list_apply;  // 1: dense u = A x from the lists in phase E (FL1_LIST_APPLY)
  int32_t power_onchip;  // 1: cluster-mode power iterations on chip when they fit (FL1_POWER_ONCHIP)
  int32_t early_prox;    // 1: non-screening dense iterations run the prox before the first barrier (FL1_EARLY_PROX)
  int64_t colsplit_elems;  // phase-E apply by column split when nnz x ld >= this (FL1_COLSPLIT; 0 = never)
  int32_t compact;       // 1: preserved columns physically compacted into cbuf (FL1_COMPACT, A/B switch)
  double* cbuf[2];       // ping-pong compact copies, ld x ceil(K/2) each
  int32_t* bcix[2];      // per bank: column slot of each position in the compact copy (csel != 0)
  double* pv;       // K
  double* pw;       // K
  double* PU;       // ld: power-iteration A v (combined)
  const double* gauss0;  // K: mt19937_64(0x11b5c417) normals (solver.cpp:80-82)
  double* sk_z;     // SuKro adjoint: Z = sum_t C_t^T R B_t (K doubles)
  int64_t scratch_len;  // doubles of shared scratch after the residual (engine_scratch_len)
  int32_t bulk_stages;  // dense adjoint bulk-copy ring depth per warp (0: register ring)
  double* bred;     // per-CTA partials: grid * kBred doubles
  Bank bank[2];
  fl1_trace_row* trace;
  int64_t trace_cap;
  fl1_switch_event* sw;
  EngineState* st;
  uint64_t* timeline;  // FL1_TIMELINE builds only: [iter][cta][8] %globaltimer marks
  const double* gram;      // nullable: K x K Gram of the exact dictionary (RunOptions::exact_gram)
  int64_t gram_ld;
  double* GX;              // K: G x (Gram mode's u)
  double* GV;              // K: G x_prev history (Gram mode's v)
  double* ATYF;            // K: A^T y over all atoms (Gram mode)
  int32_t* ident;          // K: 0..K-1 (full-dictionary passes)
  const BatchDesc* batch;  // non-null: cluster (batched) mode
  const Handoff* handoff;  // non-null: solve resumes from a lockstep-prefix state
  // (last, so that the default engine instance's parameter offsets are what they were without it)
  int64_t fused_power_bytes;  // single-read power steps when 8 ld |S| >= this (FL1_FUSED_POWER_MB; 0 = never)
  int32_t fused_prefetch;     // columns prefetched into L2 ahead of the single-read pass (FL1_FUSED_PREFETCH)
};

constexpr int kBred = 24;  // doubles of per-CTA partials (slots, see engine.cu)
constexpr int kApplyCap = 1024;  // positions compacted per apply sub-chunk
constexpr int kSukroMaxM = 128;
constexpr int kSukroMaxQ = 256;

}  // namespace fl1
