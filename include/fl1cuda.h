/*
 * fl1cuda.h — C-ABI of the B200-native FastL1 hot path (libfl1cuda.so).
 *
 * The reference (fastl1, C++20 + Eigen) exposes only a C++ API; this header is
 * the flat boundary a foreign caller (ctypes, cgo, JNI, or the C++ shim in
 * include/fl1/fastl1.hpp) binds. Every entry point names the reference symbol
 * it replaces (paths relative to /root/reference/proj).
 *
 * Conventions
 *   - All dense arrays are column-major float64 (Eigen::MatrixXd layout,
 *     core/include/fastl1/dictionary.hpp:13-15). Vectors are contiguous f64.
 *   - Every function returns an int status (FL1_OK == 0). On failure a
 *     thread-local message is available from fl1_last_error(). FL1_EINVAL is
 *     the C image of std::invalid_argument (the reference's only error type on
 *     this path: fastl1.cpp:268-273, dictionary.cpp:67,72,151,159,227-251).
 *   - Non-convergence is NOT an error (fastl1.cpp:640-644): the result carries
 *     converged = 0 and final_gap = NaN.
 *   - Handles are opaque. Dictionaries / approximations / sequences are
 *     immutable after creation and may be shared by concurrent solves
 *     (bench.cpp:283-301); each solve runs on its own stream.
 *   - Host pointers everywhere unless the function name ends in _device.
 */
#ifndef FL1CUDA_H
#define FL1CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FL1_OK 0
#define FL1_EINVAL 1      /* std::invalid_argument */
#define FL1_ECUDA 2       /* CUDA runtime / launch failure */
#define FL1_ENOMEM 3      /* allocation failure */
#define FL1_EUNSUPPORTED 4
#define FL1_ERUNTIME 5    /* std::runtime_error */

/* SolverKind / RuleKind / Variant — fastl1.hpp:14-18 */
#define FL1_ISTA 0
#define FL1_FISTA 1
#define FL1_RULE_DYNAMIC 0
#define FL1_RULE_GAP 1
#define FL1_PLAIN 0
#define FL1_SCREENED 1
#define FL1_MULTI_DICT 2

typedef struct fl1_ctx fl1_ctx;       /* device + stream pool + workspace cache */
typedef struct fl1_dict fl1_dict;     /* LinearOp (dictionary.hpp:86-104) resident in HBM */
typedef struct fl1_approx fl1_approx; /* ApproxDictionary (dictionary.hpp:111-120) */
typedef struct fl1_seq fl1_seq;       /* ApproxSequence (dictionary.hpp:128-134) */
typedef struct fl1_result fl1_result; /* SolveResult (fastl1.hpp:61-71) */

/* SwitchConfig (fastl1.hpp:25-31) + one documented extension. */
typedef struct fl1_switch_config {
  double gamma_threshold;     /* Γ in (0,1); default 0.5 */
  int32_t screening_interval; /* >= 1; default 1 */
  double tolerance;           /* absolute gap~ target (fastl1.cpp:483); default 1e-6 */
  uint64_t max_iterations;    /* default 1e6 */
  int32_t precompute_aty;     /* Table variant of the stable dynamic test */
  /* EXTENSION (BASELINE configs): when > 0 the exact-phase stop test becomes
   * gap~ <= rel_tolerance * P(x) instead of gap~ <= tolerance. 0 = reference. */
  double rel_tolerance;
} fl1_switch_config;

/* ScreeningEvent (fastl1.hpp:74-83) flattened. Pointers are valid only for the
 * duration of the callback. center/theta vectors have length n. */
typedef struct fl1_screen_event {
  uint64_t iter;
  int32_t dict_index;
  int64_t n;
  const double* center;
  double radius;
  const double* theta_prime;
  const double* theta_tilde;
  double scale_prime;
  double scale_tilde;
  int64_t n_active_before;
  const int32_t* active_before; /* global column indices */
  int64_t n_kept;
  const int32_t* kept;          /* global column indices */
} fl1_screen_event;
typedef void (*fl1_observer_fn)(const fl1_screen_event* ev, void* user);

/* RunOptions (fastl1.hpp:85-96) plus warm start. */
typedef struct fl1_run_options {
  int32_t solver;  /* FL1_FISTA */
  int32_t rule;    /* FL1_RULE_GAP */
  int32_t variant; /* FL1_MULTI_DICT */
  const double* full_lipschitz; /* per-level cache, nullable */
  int32_t n_full_lipschitz;
  int32_t collect_trace;        /* default 1 */
  fl1_observer_fn observer;     /* nullable; forces a host stop at each screening instant */
  void* observer_user;
  /* EXTENSION (BASELINE config 4): warm start, length K, nullable (reference: x = 0,
   * fastl1.cpp:274). */
  const double* x_init;
  /* exact_gram (fastl1.hpp:89-91): the K x K Gram matrix of the exact dictionary as a
   * dense dictionary handle (fl1_gram_create, or fl1_dict_dense of a host G); nullable.
   * The exact phase then runs on G (fastl1.cpp:283-324, 335-394); ignored while an
   * observer is attached (fastl1.cpp:278-281). */
  const struct fl1_dict* exact_gram;
} fl1_run_options;

/* TraceRow (fastl1.hpp:43-52) */
typedef struct fl1_trace_row {
  uint64_t iter;
  int32_t dict_index;
  int32_t active_size;
  double gap;
  double gamma;
  uint64_t flops_cum;
  double wall_ms;
  int32_t x_nnz;
  int32_t pad_;
} fl1_trace_row;

/* SwitchEvent (fastl1.hpp:54-59) */
typedef struct fl1_switch_event {
  uint64_t iter;
  int32_t from;
  int32_t to;
  int32_t speed;
  int32_t pad_;
} fl1_switch_event;

typedef struct fl1_result_info {
  int64_t k;
  int32_t converged;
  int32_t gap_warning;
  double final_gap;
  uint64_t iterations;
  uint64_t total_flops;
  int64_t n_trace;
  int64_t n_switches;
  int64_t n_final_active;
  double device_ms;    /* engine time on the solve stream (CUDA events), excl. H2D/D2H */
  double setup_ms;     /* constructor part (initial L, u = A x) on device */
  int64_t kernel_launches; /* launches of this library's kernels during the solve */
  int64_t power_iterations; /* total power-iteration steps (all L estimates) */
  int64_t h2d_bytes;        /* host->device bytes moved by this solve */
  int64_t d2h_bytes;        /* device->host bytes moved by this solve */
  double batch_device_ms;   /* batched solves: device time of the whole batch (every launch,
                               CUDA events on the batch stream); single solves: device_ms */
} fl1_result_info;

/* ---- errors ---- */
const char* fl1_last_error(void);
const char* fl1_version(void);

/* ---- context ---- */
int fl1_ctx_create(int device, fl1_ctx** out);
int fl1_ctx_destroy(fl1_ctx* ctx);
/* SM count, L2 bytes, etc. of the bound device. */
int fl1_ctx_info(fl1_ctx* ctx, int32_t* sm_count, int64_t* l2_bytes, int64_t* hbm_bytes);

/* ---- dictionaries: DenseDictionary (dictionary.hpp:19-48; dictionary.cpp:59-74) ---- */
int fl1_dict_dense(fl1_ctx* ctx, const double* colmajor, int64_t n, int64_t k, fl1_dict** out);
/* Same, from a device pointer (copied into the handle's own HBM buffer). */
int fl1_dict_dense_device(fl1_ctx* ctx, const double* colmajor_dev, int64_t n, int64_t k,
                          fl1_dict** out);
/* SukroDictionary (dictionary.hpp:53-81; dictionary.cpp:137-195). left[t], right[t] are
 * m x q column-major. col_scale (length q*q, nullable) is the EXTENSION for column-
 * normalised Kronecker sums (BASELINE config 3): A = Kron(.) diag(col_scale). */
int fl1_dict_sukro(fl1_ctx* ctx, int32_t n_terms, int64_t m, int64_t q,
                   const double* const* left, const double* const* right,
                   const double* col_scale, fl1_dict** out);
int fl1_dict_destroy(fl1_dict* d);
int fl1_dict_shape(const fl1_dict* d, int64_t* rows, int64_t* cols);
int fl1_dict_is_dense(const fl1_dict* d);
uint64_t fl1_dict_matvec_flops(const fl1_dict* d);          /* dictionary.hpp:36, cpp:179-185 */
int fl1_dict_atom_norms(const fl1_dict* d, double* out);    /* DenseDictionary::atom_norms2 */
/* LinearOp::apply / apply_adjoint / column (dictionary.cpp:197-214), computed on the GPU. */
int fl1_dict_apply(fl1_dict* d, const double* x, double* out);
int fl1_dict_apply_adjoint(fl1_dict* d, const double* r, double* out);
int fl1_dict_column(fl1_dict* d, int64_t j, double* out);

/* ---- approximations / sequences ---- */
/* ApproxDictionary aggregate (dictionary.hpp:111-120). Vectors have length K. */
int fl1_approx_create(fl1_dict* d, const double* atom_error_bounds, double operator_error_bound,
                      double relative_complexity, const double* approx_atom_norms2,
                      const double* exact_atom_norms2, fl1_approx** out);
/* make_exact_approx (dictionary.cpp:216-225); d must be dense. */
int fl1_approx_exact(fl1_dict* d, fl1_approx** out);
int fl1_approx_destroy(fl1_approx* a);
/* ApproxSequence{levels}; runs ApproxSequence::validate (dictionary.cpp:227-251). */
int fl1_seq_create(fl1_approx* const* levels, int32_t n_levels, fl1_seq** out);
int fl1_seq_destroy(fl1_seq* s);

/* ---- solve: run_lasso (fastl1.cpp:753-758) / fastl1_solve (fastl1.hpp:104-111) ---- */
int fl1_solve(fl1_seq* s, const double* y, double lambda, const fl1_switch_config* cfg,
              const fl1_run_options* opts, fl1_result** out);
/* Same with y (length N) already in HBM; no host copies of inputs. */
int fl1_solve_device(fl1_seq* s, const double* y_dev, double lambda,
                     const fl1_switch_config* cfg, const fl1_run_options* opts,
                     fl1_result** out);
/* Batched many-signal solve (BASELINE config 5): B independent run_lasso calls on one
 * sequence — per-signal FISTA state, preserved set, Lipschitz refreshes and stop —
 * on one device. concurrency <= 0: ONE launch in which every thread-block cluster
 * of -concurrency CTAs (0 = default 2; at most 16) is an engine with its own
 * workspace that takes signals from a device-side queue. concurrency > 0: that
 * many concurrent sub-grid engine launches (own stream and workspace each).
 * Both give the same per-signal results as fl1_solve. Y is N x B column-major with leading dimension
 * ldy (host), lambdas has B entries, out receives B results. Observers and x_init
 * are per-signal features of fl1_solve and are rejected here. */
int fl1_solve_batched(fl1_seq* s, const double* Y, int64_t ldy, const double* lambdas, int32_t batch,
                      const fl1_switch_config* cfg, const fl1_run_options* opts, int32_t concurrency,
                      fl1_result** out);
/* Same with Y (N x B, leading dimension ldy) resident in HBM. */
int fl1_solve_batched_device(fl1_seq* s, const double* Y_dev, int64_t ldy, const double* lambdas, int32_t batch,
                             const fl1_switch_config* cfg, const fl1_run_options* opts, int32_t concurrency,
                             fl1_result** out);
int fl1_result_info_get(const fl1_result* r, fl1_result_info* out);
int fl1_result_x(const fl1_result* r, double* out);  /* length K, zero over screened atoms */
int fl1_result_trace(const fl1_result* r, fl1_trace_row* out);
int fl1_result_switches(const fl1_result* r, fl1_switch_event* out);
int fl1_result_final_active(const fl1_result* r, int32_t* out);
/* Device-side phase profile of the solve (ns, %globaltimer, CTA 0):
 * [0] products + A^T r pass, [1] dual scalars / screening / prox, [2] compaction +
 * sparse apply + ledger, [3] restricted power iterations, [4] switch setups,
 * [5] bytes streamed by the A^T r passes, [6] bytes streamed by the sparse applies
 * (8 N nnz), [7] bytes streamed by power iterations (16 N |S| per step), [8..11] power-iteration
 * sub-phases (apply, combine, adjoint + norms, reduce; ns), [12] ns and [13] bytes of the
 * A^T r passes over the full dictionary (|S| = K). out has 14 entries. Signal 0 of a
 * batched call that ran the lockstep engine: [0] device ms from the batch start to the end
 * of the lockstep launch, [1] sum over lockstep steps of the unfinished signals (A^T R
 * widths), [2] the same for the power-step signals (A V widths), [3] lockstep steps. */
int fl1_result_profile(const fl1_result* r, double* out);
/* Bulk accessors for batched results (one call instead of one per result): infos
 * (count), x (count x K), profiles (count x 14), and the traces / switch events /
 * final active sets of all results concatenated in result order (sizes from infos). */
int fl1_results_collect(fl1_result* const* rs, int32_t count, fl1_result_info* infos, double* x, double* profiles);
int fl1_results_tables(fl1_result* const* rs, int32_t count, fl1_trace_row* traces, fl1_switch_event* switches,
                       int32_t* final_active);
void fl1_result_free(fl1_result* r);

/* ---- setup-side primitives on the path ---- */
/* lambda_max (screening.cpp:9-11): ||A^T y||_inf on the GPU. */
int fl1_lambda_max(fl1_dict* d, const double* y, double* out);
/* lipschitz_bound (solver.cpp:108-114): cold power iteration x 1.05 on the GPU. */
int fl1_lipschitz_bound(fl1_dict* d, double* out);

/* G = A^T A of a dense dictionary, computed on the GPU (one fp64 GEMM), as a dense
 * K x K dictionary handle for fl1_run_options.exact_gram (bench.cpp:180-200). */
int fl1_gram_create(fl1_dict* a, fl1_dict** out);

/* ---- harness generators (host; the reference's own <random> streams) ---- */
/* count draws of std::normal_distribution<double>(0, 1) on std::mt19937_64(seed): the
 * stream behind synthesize_scenario (dictionary.cpp:396-409, seed ^ 0xd1c7) and
 * truncated_svd (dictionary.cpp:258-262, seed 0x5eedf00d). */
int fl1_rng_normals(uint64_t seed, int64_t count, double* out);
/* draw_signal (bench.cpp:141-166): Bernoulli(p)-Gaussian x over K atoms from
 * mt19937_64(mix_seed(seed, trial)), y = A x on the GPU, both scaled so |y| = 1;
 * draws with an empty support or |y| <= 1e-12 are redrawn. y: N, x: K. */
int fl1_draw_signal(fl1_dict* d, double bernoulli_p, uint64_t seed, int32_t trial, double* y, double* x);

/* build_sukro_sequence (dictionary.cpp:281-357, truncated_svd 253-279) on the device for a
 * dense N x K dictionary (N = m^2, K = q^2): the SuKro levels of the given strictly
 * increasing ranks. Outputs (host): left / right = the T = ranks[n_ranks-1] factor pairs,
 * term t at t*m*q (m x q column-major each, sqrt(s_t) folded into both, as the reference);
 * eps / approx_norms = n_ranks x K (level l at l*K: atom_error_bounds after the running
 * max, approx_atom_norms2); rc / op_err = n_ranks (relative_complexity,
 * operator_error_bound). Errors (FL1_EINVAL) carry the reference's messages. Device limit:
 * rank + 8 <= 64 probes, <= 16 ranks. */
int fl1_build_sukro_sequence(fl1_dict* dense, const int32_t* ranks, int32_t n_ranks, double* left, double* right,
                             double* eps, double* approx_norms, double* rc, double* op_err);
/* screen_precomputed (screening.cpp:136-150) as a device kernel; kept gets positions. */
int fl1_screen_precomputed(fl1_ctx* ctx, int64_t n, const double* abs_dots, const double* eps,
                           const double* exact_norms, const double* approx_norms,
                           double center_norm, double radius, int32_t* kept, int64_t* n_kept,
                           int64_t* lookahead);

/* ---- scalar formulas of the path (host; no device needed) ---- */
double fl1_soft_threshold(double z, double u);                               /* solver.cpp:9-13 */
double fl1_gap_ratio(double gap_tilde, double gap_prime);                    /* fastl1.cpp:26-30 */
int fl1_switch_dictionary(int i, int last, double gamma, double gamma_threshold,
                          int64_t lookahead, double rc_i, int64_t total_atoms); /* fastl1.cpp:32-38 */
uint64_t fl1_flops_plain(uint64_t k, uint64_t n, uint64_t nnz);              /* fastl1.cpp:40-42 */
uint64_t fl1_flops_screened(uint64_t active, uint64_t n, uint64_t nnz);      /* fastl1.cpp:43-45 */
uint64_t fl1_flops_stable(uint64_t matvec, uint64_t n, uint64_t active, uint64_t nnz); /* 46-49 */
/* recompute_flops (fastl1.cpp:51-81); rows_match nullable. */
uint64_t fl1_recompute_flops(const fl1_trace_row* trace, int64_t n_rows, const fl1_seq* s,
                             int32_t variant, int64_t n, int64_t k, int32_t* rows_match);
double fl1_stable_gap_delta(double residual_norm, double operator_error_bound, double x_l1); /* screening.cpp:103-106 */
double fl1_sphere_test(double abs_atom_dot_center, double atom_norm, double radius);  /* screening.hpp:30-33 */
double fl1_stable_zone_test(double abs_approx_dot_center, double eps, double center_norm,
                            double exact_atom_norm, double radius);                  /* screening.hpp:36-41 */
double fl1_stable_ball_test(double abs_approx_dot_center, double eps, double center_norm,
                            double approx_atom_norm, double radius);                 /* screening.hpp:45-50 */

#ifdef __cplusplus
}
#endif

#endif /* FL1CUDA_H */
