/*
 * fl1_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * C-ABI of the CPU oracle: an Eigen-free restatement of the reference engine
 * (fastl1::run_lasso and the primitives it calls). It exports the SAME entry
 * points and structs as the product boundary include/fl1cuda.h, with the
 * prefix orc_ instead of fl1_, so the Python wrapper can drive either library
 * and the parity tests compare like with like.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this library. The product never links it.
 *
 * Parity status: the reference itself cannot be built here (Eigen3, doctest
 * absent — SURVEY.md §8c), so the oracle is pinned against every known-answer
 * test and structural oracle the reference's own tests hold for this path
 * (tests/test_oracle_kats.py; list in DESIGN.md §Oracle).
 */
#ifndef FL1_ORACLE_H
#define FL1_ORACLE_H

#include "../include/fl1cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_dict orc_dict;
typedef struct orc_approx orc_approx;
typedef struct orc_seq orc_seq;
typedef struct orc_result orc_result;
typedef struct orc_ctx orc_ctx;

const char* orc_last_error(void);
const char* orc_version(void);
/* threads used by the column-parallel products (results are bit-identical for
 * any thread count: per-column dots and per-row sums keep their order). */
void orc_set_threads(int n);
int orc_get_threads(void);

int orc_ctx_create(int device, orc_ctx** out);
int orc_ctx_destroy(orc_ctx* ctx);

int orc_gram_create(orc_dict* d, orc_dict** out);
int orc_dict_dense(orc_ctx* ctx, const double* colmajor, int64_t n, int64_t k, orc_dict** out);
int orc_dict_sukro(orc_ctx* ctx, int32_t n_terms, int64_t m, int64_t q,
                   const double* const* left, const double* const* right,
                   const double* col_scale, orc_dict** out);
int orc_dict_destroy(orc_dict* d);
int orc_dict_shape(const orc_dict* d, int64_t* rows, int64_t* cols);
int orc_dict_is_dense(const orc_dict* d);
uint64_t orc_dict_matvec_flops(const orc_dict* d);
int orc_dict_atom_norms(const orc_dict* d, double* out);
int orc_dict_apply(orc_dict* d, const double* x, double* out);
int orc_dict_apply_adjoint(orc_dict* d, const double* r, double* out);
int orc_dict_column(orc_dict* d, int64_t j, double* out);
int orc_dict_to_dense(orc_dict* d, double* out); /* SukroDictionary::to_dense */

int orc_approx_create(orc_dict* d, const double* atom_error_bounds, double operator_error_bound,
                      double relative_complexity, const double* approx_atom_norms2,
                      const double* exact_atom_norms2, orc_approx** out);
int orc_approx_exact(orc_dict* d, orc_approx** out);
int orc_approx_destroy(orc_approx* a);
int orc_seq_create(orc_approx* const* levels, int32_t n_levels, orc_seq** out);
int orc_seq_destroy(orc_seq* s);

int orc_solve(orc_seq* s, const double* y, double lambda, const fl1_switch_config* cfg,
              const fl1_run_options* opts, orc_result** out);
int orc_result_info_get(const orc_result* r, fl1_result_info* out);
int orc_result_x(const orc_result* r, double* out);
int orc_result_trace(const orc_result* r, fl1_trace_row* out);
int orc_result_switches(const orc_result* r, fl1_switch_event* out);
int orc_result_final_active(const orc_result* r, int32_t* out);
void orc_result_free(orc_result* r);

int orc_lambda_max(orc_dict* d, const double* y, double* out);
int orc_lipschitz_bound(orc_dict* d, double* out);
int orc_screen_precomputed(orc_ctx* ctx, int64_t n, const double* abs_dots, const double* eps,
                           const double* exact_norms, const double* approx_norms,
                           double center_norm, double radius, int32_t* kept, int64_t* n_kept,
                           int64_t* lookahead);

double orc_soft_threshold(double z, double u);
double orc_gap_ratio(double gap_tilde, double gap_prime);
int orc_switch_dictionary(int i, int last, double gamma, double gamma_threshold,
                          int64_t lookahead, double rc_i, int64_t total_atoms);
uint64_t orc_flops_plain(uint64_t k, uint64_t n, uint64_t nnz);
uint64_t orc_flops_screened(uint64_t active, uint64_t n, uint64_t nnz);
uint64_t orc_flops_stable(uint64_t matvec, uint64_t n, uint64_t active, uint64_t nnz);
uint64_t orc_recompute_flops(const fl1_trace_row* trace, int64_t n_rows, const orc_seq* s,
                             int32_t variant, int64_t n, int64_t k, int32_t* rows_match);
double orc_stable_gap_delta(double residual_norm, double operator_error_bound, double x_l1);
double orc_sphere_test(double abs_atom_dot_center, double atom_norm, double radius);
double orc_stable_zone_test(double abs_approx_dot_center, double eps, double center_norm,
                            double exact_atom_norm, double radius);
double orc_stable_ball_test(double abs_approx_dot_center, double eps, double center_norm,
                            double approx_atom_norm, double radius);

/* ---- oracle-only primitives (the reference's test oracles / steppers) ---- */
/* ista_step / fista_step (solver.cpp:21-50). aux_* is the SolverAux state:
 * x_prev (length K), t_k, momentum_ready; updated in place by fista. */
int orc_ista_step(orc_dict* d, const double* y, double lambda, double step_size,
                  const double* x, double* x_next, double* residual, double* correlations);
int orc_fista_step(orc_dict* d, const double* y, double lambda, double step_size,
                   const double* x, double* x_prev, double* t_k, int32_t* momentum_ready,
                   double* x_next, double* residual, double* correlations);
double orc_primal_value(orc_dict* d, const double* y, double lambda, const double* x);
double orc_dual_value(int64_t n, const double* y, double lambda, const double* theta);
double orc_duality_gap(orc_dict* d, const double* y, double lambda, const double* x,
                       const double* theta, int32_t* warn);
int orc_stable_lambda_max(orc_approx* a, const double* y, double* out);
int orc_dual_scale(orc_dict* d, const double* z, double* out);
int orc_stable_dual_scale(orc_approx* a, const double* z, double* out);
/* dual_point_dynamic (screening.cpp:56-101); dict nullable. */
int orc_dual_point_dynamic(int64_t n, int64_t m, const double* residual,
                           const double* correlations, const double* eps, const double* y,
                           double lambda, orc_dict* dict_for_degenerate, double* theta_prime,
                           double* theta_tilde, double* scale_prime, double* scale_tilde);
/* build_sphere (screening.cpp:108-134). rule: 0 static,1 stable_static,2 dynamic,
 * 3 stable_dynamic,4 gap,5 stable_gap. theta nullable for static rules. */
int orc_build_sphere(int32_t rule, int64_t n, const double* y, double lambda, double lambda_max,
                     double stable_lambda_max, const double* theta, double gap, double delta,
                     double* center, double* radius);
/* screen (screening.cpp:152-167): returns kept global indices. */
int orc_screen(const int32_t* active, int64_t n_active, const double* center, double radius,
               orc_approx* a, int32_t use_stable, int32_t* kept, int64_t* n_kept);

/* The first `count` draws of std::mt19937_64(seed) through libstdc++'s
 * std::normal_distribution<double>(0,1) — the RNG the reference uses for its
 * seeded matrices (tests/helpers.hpp:35-50, dictionary.cpp:258-262, 391-405). */
void orc_gen_normals(uint64_t seed, int64_t count, double* out);
/* std::uniform_int_distribution<int64_t>(0, hi) draws interleaved with normals, as
 * in testkit::random_instance / square_instance (helpers.hpp:76-89,
 * test_fastl1.cpp:18-31): for each of `support` draws, pos = pick(rng),
 * val = gauss(rng). */
void orc_gen_support(uint64_t seed, int64_t hi, int32_t support, int64_t* pos, double* val);

#ifdef __cplusplus
}
#endif
#endif
