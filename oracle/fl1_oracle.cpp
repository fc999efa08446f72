// fl1_oracle.cpp — TEST INFRASTRUCTURE ONLY (see fl1_oracle.h).
//
// Eigen-free C++ restatement of the reference FastL1 engine for the parity
// tests and the CPU baseline. It follows, statement by statement:
//   fastl1.cpp:26-49   gap_ratio, switch_dictionary, flop formulas
//   fastl1.cpp:51-81   recompute_flops
//   fastl1.cpp:85-211  count_nonzeros, ActiveOp
//   fastl1.cpp:213-749 Engine (ctor, setup_dictionary, restricted_lipschitz,
//                      compute_products, dual_scalars, dual_of, run,
//                      row_flops, apply_restriction, fire_observer, finish)
//   solver.cpp:9-104   soft_threshold, steppers, objectives, power iteration
//   screening.cpp      lambda_max, stable_lambda_max, tests, dual scalings,
//                      dual_point_dynamic, stable_gap_delta, build_sphere,
//                      screen_precomputed, screen
//   dictionary.cpp     dense/SuKro apply, adjoint, column, matvec_flops,
//                      to_dense, make_exact_approx, ApproxSequence::validate
// Eigen's exact summation order is not reproduced (it is unspecified); every
// reduction here is a plain sequential loop. Two documented extensions
// (rel_tolerance, x_init) and the SuKro column scale default to reference
// behaviour when unused. The Gram-backed exact phase (fastl1.cpp:335-394) is restated
// too (Engine::compute_products' gram_mode branch and apply_restriction's G-column fix).
#include "fl1_oracle.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <functional>
#include <limits>
#include <memory>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

thread_local std::string g_err;
int g_threads = 1;

using Vec = std::vector<double>;

double sqnorm(const Vec& v) {
  double s = 0.0;
  for (double e : v) s += e * e;
  return s;
}
double norm2(const Vec& v) { return std::sqrt(sqnorm(v)); }
double dot(const Vec& a, const Vec& b) {
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}
double l1(const Vec& v) {
  double s = 0.0;
  for (double e : v) s += std::abs(e);
  return s;
}

// ---------------------------------------------------------------- operators
struct Op {
  bool dense = true;
  int64_t n = 0, k = 0;
  // dense (dictionary.cpp:59-74)
  Vec a;      // column-major n x k
  Vec norms;  // atom_norms2
  // SuKro (dictionary.cpp:137-195) + column scale extension
  int64_t m = 0, q = 0;
  std::vector<Vec> left, right;  // m x q column-major
  Vec col_scale;                 // empty: none

  const double* col(int64_t j) const { return a.data() + j * n; }

  // DenseDictionary::apply (68): out = A x. Zero x_j contribute exact zeros, so
  // skipping them is the same sum (also the ActiveOp sparse form, 131-139).
  Vec apply(const Vec& x) const {
    if (static_cast<int64_t>(x.size()) != k) throw std::invalid_argument("matvec: x has wrong length");
    if (dense) {
      Vec out(static_cast<size_t>(n), 0.0);
#pragma omp parallel for num_threads(g_threads) schedule(static) if (g_threads > 1)
      for (int64_t i0 = 0; i0 < n; i0 += 256) {
        const int64_t i1 = std::min<int64_t>(n, i0 + 256);
        for (int64_t j = 0; j < k; ++j) {
          const double xj = x[static_cast<size_t>(j)];
          if (xj == 0.0) continue;
          const double* c = col(j);
          for (int64_t i = i0; i < i1; ++i) out[static_cast<size_t>(i)] += xj * c[i];
        }
      }
      return out;
    }
    return sukro_apply(x);
  }

  // DenseDictionary::apply_adjoint (73): out_j = a_j . r
  Vec adjoint(const Vec& r) const {
    if (static_cast<int64_t>(r.size()) != n) throw std::invalid_argument("adjoint matvec: r has wrong length");
    if (dense) {
      Vec out(static_cast<size_t>(k));
#pragma omp parallel for num_threads(g_threads) schedule(static) if (g_threads > 1)
      for (int64_t j = 0; j < k; ++j) {
        const double* c = col(j);
        double s = 0.0;
        for (int64_t i = 0; i < n; ++i) s += c[i] * r[static_cast<size_t>(i)];
        out[static_cast<size_t>(j)] = s;
      }
      return out;
    }
    return sukro_adjoint(r);
  }

  // restricted adjoint over a list of columns (ActiveOp::apply_adjoint 150-155)
  Vec adjoint_cols(const std::vector<int>& cols, const Vec& r) const {
    Vec out(cols.size());
#pragma omp parallel for num_threads(g_threads) schedule(static) if (g_threads > 1)
    for (int64_t p = 0; p < static_cast<int64_t>(cols.size()); ++p) {
      const double* c = col(cols[static_cast<size_t>(p)]);
      double s = 0.0;
      for (int64_t i = 0; i < n; ++i) s += c[i] * r[static_cast<size_t>(i)];
      out[static_cast<size_t>(p)] = s;
    }
    return out;
  }

  // restricted sparse apply (ActiveOp::apply 133-139)
  Vec apply_cols(const std::vector<int>& cols, const Vec& xc) const {
    Vec out(static_cast<size_t>(n), 0.0);
#pragma omp parallel for num_threads(g_threads) schedule(static) if (g_threads > 1)
    for (int64_t i0 = 0; i0 < n; i0 += 256) {
      const int64_t i1 = std::min<int64_t>(n, i0 + 256);
      for (size_t p = 0; p < cols.size(); ++p) {
        const double xj = xc[p];
        if (xj == 0.0) continue;
        const double* c = col(cols[p]);
        for (int64_t i = i0; i < i1; ++i) out[static_cast<size_t>(i)] += xj * c[i];
      }
    }
    return out;
  }

  // SukroDictionary::apply (150-156): vec(sum_t C_t X B_t^T), X = reshape(d∘x, q, q)
  Vec sukro_apply(const Vec& x) const {
    Vec xs = x;
    if (!col_scale.empty())
      for (int64_t j = 0; j < k; ++j) xs[static_cast<size_t>(j)] *= col_scale[static_cast<size_t>(j)];
    Vec acc(static_cast<size_t>(m * m), 0.0);
    Vec t(static_cast<size_t>(m * q));
    for (size_t term = 0; term < left.size(); ++term) {
      const Vec& b = left[term];
      const Vec& c = right[term];
      // T = C X  (m x q): T(rc, jj) = sum_s C(rc, s) X(s, jj)
      std::fill(t.begin(), t.end(), 0.0);
      for (int64_t jj = 0; jj < q; ++jj)
        for (int64_t s = 0; s < q; ++s) {
          const double xv = xs[static_cast<size_t>(jj * q + s)];
          if (xv == 0.0) continue;
          for (int64_t rc = 0; rc < m; ++rc) t[static_cast<size_t>(jj * m + rc)] += c[static_cast<size_t>(s * m + rc)] * xv;
        }
      // acc(rc, rb) += sum_jj T(rc, jj) B(rb, jj)
      for (int64_t rb = 0; rb < m; ++rb)
        for (int64_t jj = 0; jj < q; ++jj) {
          const double bv = b[static_cast<size_t>(jj * m + rb)];
          for (int64_t rc = 0; rc < m; ++rc) acc[static_cast<size_t>(rb * m + rc)] += t[static_cast<size_t>(jj * m + rc)] * bv;
        }
    }
    return acc;
  }

  // SukroDictionary::apply_adjoint (158-164): vec(sum_t C_t^T R B_t), then d∘
  Vec sukro_adjoint(const Vec& r) const {
    Vec acc(static_cast<size_t>(q * q), 0.0);
    Vec t(static_cast<size_t>(q * m));
    for (size_t term = 0; term < left.size(); ++term) {
      const Vec& b = left[term];
      const Vec& c = right[term];
      // T = C^T R (q x m): T(s, rb) = sum_rc C(rc, s) R(rc, rb)
      for (int64_t rb = 0; rb < m; ++rb)
        for (int64_t s = 0; s < q; ++s) {
          double acc_s = 0.0;
          for (int64_t rc = 0; rc < m; ++rc) acc_s += c[static_cast<size_t>(s * m + rc)] * r[static_cast<size_t>(rb * m + rc)];
          t[static_cast<size_t>(rb * q + s)] = acc_s;
        }
      // acc(s, jj) += sum_rb T(s, rb) B(rb, jj)
      for (int64_t jj = 0; jj < q; ++jj)
        for (int64_t s = 0; s < q; ++s) {
          double acc_s = 0.0;
          for (int64_t rb = 0; rb < m; ++rb) acc_s += t[static_cast<size_t>(rb * q + s)] * b[static_cast<size_t>(jj * m + rb)];
          acc[static_cast<size_t>(jj * q + s)] += acc_s;
        }
    }
    if (!col_scale.empty())
      for (int64_t j = 0; j < k; ++j) acc[static_cast<size_t>(j)] *= col_scale[static_cast<size_t>(j)];
    return acc;
  }

  // LinearOp::column (dictionary.cpp:166-177)
  Vec column(int64_t j) const {
    if (j < 0 || j >= k) throw std::invalid_argument("column index out of range");
    if (dense) return Vec(col(j), col(j) + n);
    const int64_t jb = j / q, jc = j % q;
    Vec out(static_cast<size_t>(n), 0.0);
    for (size_t term = 0; term < left.size(); ++term)
      for (int64_t rb = 0; rb < m; ++rb) {
        const double bv = left[term][static_cast<size_t>(jb * m + rb)];
        for (int64_t rc = 0; rc < m; ++rc)
          out[static_cast<size_t>(rb * m + rc)] += bv * right[term][static_cast<size_t>(jc * m + rc)];
      }
    if (!col_scale.empty())
      for (auto& e : out) e *= col_scale[static_cast<size_t>(j)];
    return out;
  }

  uint64_t matvec_flops() const {
    if (dense) return static_cast<uint64_t>(n) * static_cast<uint64_t>(k);
    return static_cast<uint64_t>(left.size()) *
           (static_cast<uint64_t>(m) * static_cast<uint64_t>(k) +
            static_cast<uint64_t>(q) * static_cast<uint64_t>(n));
  }
};

struct Approx {
  std::shared_ptr<const Op> op;
  Vec eps;
  double op_err = 0.0;
  double rc = 1.0;
  Vec approx_norms, exact_norms;
  bool is_exact() const { return op_err == 0.0; }
};

struct Seq {
  std::vector<std::shared_ptr<const Approx>> d;
  int levels() const { return static_cast<int>(d.size()); }
  const Approx& at(int i) const { return *d[static_cast<size_t>(i)]; }
  const Approx& exact() const { return *d.back(); }

  // ApproxSequence::validate (dictionary.cpp:227-251)
  void validate() const {
    if (d.empty()) throw std::invalid_argument("empty approximation sequence");
    const int64_t k = d.front()->op->k;
    for (size_t i = 0; i < d.size(); ++i) {
      const Approx& a = *d[i];
      if (a.op->k != k) throw std::invalid_argument("sequence has mismatched atom counts");
      bool bad = static_cast<int64_t>(a.eps.size()) != k;
      if (!bad)
        for (double e : a.eps) bad = bad || e < 0;
      if (bad) throw std::invalid_argument("invalid atom error bounds");
      if (a.rc <= 0.0 || a.rc > 1.0) throw std::invalid_argument("relative complexity out of (0, 1]");
      if (i > 0) {
        const Approx& p = *d[i - 1];
        if (a.rc <= p.rc) throw std::invalid_argument("relative complexity must strictly increase");
        for (int64_t j = 0; j < k; ++j)
          if (a.eps[static_cast<size_t>(j)] > p.eps[static_cast<size_t>(j)] + 1e-15)
            throw std::invalid_argument("error bounds must be non-increasing along the sequence");
      }
    }
    if (!d.back()->is_exact() || d.back()->rc != 1.0)
      throw std::invalid_argument("sequence must end with the exact dictionary");
  }
};

// ---------------------------------------------------------------- primitives
double soft_threshold(double z, double u) {  // solver.cpp:9-13
  const double mag = std::abs(z) - u;
  if (mag <= 0.0) return 0.0;
  return z > 0.0 ? mag : -mag;
}

constexpr double kGapRoundoffFloor = -1e-10;  // solver.hpp:53
constexpr double kLipschitzSafety = 1.05;     // solver.hpp:54

// detail::power_iteration_sq_norm (solver.cpp:72-104)
double power_iteration_sq_norm(const std::function<Vec(const Vec&)>& apply,
                               const std::function<Vec(const Vec&)>& apply_adjoint, int64_t cols,
                               const Vec* warm_start, Vec* leading_vector, int64_t* steps) {
  Vec v(static_cast<size_t>(cols));
  const bool warm = warm_start && static_cast<int64_t>(warm_start->size()) == cols && norm2(*warm_start) > 0;
  if (warm) {
    v = *warm_start;
  } else {
    std::mt19937_64 rng(0x11b5c417ULL);
    std::normal_distribution<double> gauss(0.0, 1.0);
    for (int64_t i = 0; i < cols; ++i) v[static_cast<size_t>(i)] = gauss(rng);
  }
  {
    const double nv = norm2(v);
    for (auto& e : v) e /= nv;
  }
  double estimate = 0.0;
  const int max_iter = warm ? 12 : 200;
  const double rel_tol = warm ? 1e-5 : 1e-9;
  const int min_iter = warm ? 2 : 4;
  for (int it = 0; it < max_iter; ++it) {
    if (steps) ++*steps;
    Vec w = apply_adjoint(apply(v));
    const double nrm = norm2(w);
    if (nrm == 0.0) {
      estimate = 0.0;
      break;
    }
    const double prev = estimate;
    estimate = dot(v, w);
    for (size_t i = 0; i < v.size(); ++i) v[i] = w[i] / nrm;
    if (it > min_iter && std::abs(estimate - prev) <= rel_tol * estimate) break;
  }
  if (leading_vector) *leading_vector = v;
  return estimate;
}

double gap_ratio(double gap_tilde, double gap_prime) {  // fastl1.cpp:26-30
  if (gap_prime <= 1e-15) return 0.0;
  const double ratio = gap_tilde / gap_prime;
  return std::min(std::max(ratio, 0.0), 1.0);
}

int switch_dictionary(int i, int last, double gamma, double gamma_threshold, int64_t lookahead,
                      double rc_i, int64_t total_atoms) {  // fastl1.cpp:32-38
  if (i >= last) return last;
  if (static_cast<double>(lookahead) <= rc_i * static_cast<double>(total_atoms)) return last;
  if (gamma <= gamma_threshold) return i + 1;
  return i;
}

uint64_t flops_plain(uint64_t k, uint64_t n, uint64_t nnz) { return (k + nnz) * n + 4 * k + n; }
uint64_t flops_screened(uint64_t a, uint64_t n, uint64_t nnz) { return (a + nnz) * n + 6 * a + 5 * n; }
uint64_t flops_stable(uint64_t mv, uint64_t n, uint64_t a, uint64_t nnz) { return mv + nnz * n + 8 * a + 7 * n; }

double stable_gap_delta(double rn, double e, double x1) {  // screening.cpp:103-106
  return rn * e * x1 + 0.5 * e * e * x1 * x1;
}
double sphere_test(double d, double an, double r) { return d + r * an; }  // screening.hpp:30-33
double stable_zone_test(double d, double eps, double cn, double en, double r) {  // :36-41
  return d + eps * cn + r * en;
}
double stable_ball_test(double d, double eps, double cn, double an, double r) {  // :45-50
  return d + eps * cn + r * an + r * eps;
}

struct ScreenResult {
  std::vector<int> kept;
  int lookahead_count = 0;
};
// screen_precomputed (screening.cpp:136-150)
ScreenResult screen_precomputed(const Vec& dots, const Vec& eps, const Vec& en, const Vec& an,
                                double cn, double r) {
  ScreenResult out;
  out.kept.reserve(dots.size());
  for (size_t j = 0; j < dots.size(); ++j) {
    const double d = dots[j];
    if (stable_zone_test(d, eps[j], cn, en[j], r) >= 1.0) out.kept.push_back(static_cast<int>(j));
    if (sphere_test(d, an[j], r) >= 1.0) ++out.lookahead_count;
  }
  return out;
}

int count_nonzeros(const Vec& v) {  // fastl1.cpp:85-91
  int c = 0;
  for (double e : v)
    if (e != 0.0) ++c;
  return c;
}

// ---------------------------------------------------------------- ActiveOp (fastl1.cpp:95-211)
// The reference's physical compaction (maybe_compact 176-187) only changes
// which Eigen kernel sums the products; here every product is the same
// sequential sum with or without it, so only the index list is kept.
class ActiveOp {
 public:
  explicit ActiveOp(const Approx* base) : base_(base) {
    active_.resize(static_cast<size_t>(base->op->k));
    std::iota(active_.begin(), active_.end(), 0);
    gather_metadata();
  }
  void rebase(const Approx* base) {  // 105-112
    base_ = base;
    gather_metadata();
  }
  void restrict_to_local(const std::vector<int>& kept) {  // 115-129
    std::vector<int> next;
    next.reserve(kept.size());
    for (int pos : kept) next.push_back(active_[static_cast<size_t>(pos)]);
    active_ = std::move(next);
    gather_metadata();
  }
  Vec apply(const Vec& xc) const {  // 131-146
    const Op& op = *base_->op;
    if (op.dense) return op.apply_cols(active_, xc);
    Vec padded(static_cast<size_t>(op.k), 0.0);
    for (size_t j = 0; j < active_.size(); ++j) padded[static_cast<size_t>(active_[j])] = xc[j];
    return op.apply(padded);
  }
  Vec apply_adjoint(const Vec& r) const {  // 148-161
    const Op& op = *base_->op;
    if (op.dense) return op.adjoint_cols(active_, r);
    const Vec full = op.adjoint(r);
    Vec out(active_.size());
    for (size_t j = 0; j < active_.size(); ++j) out[j] = full[static_cast<size_t>(active_[j])];
    return out;
  }
  Vec column_global(int j) const { return base_->op->column(j); }
  int64_t rows() const { return base_->op->n; }
  int64_t size() const { return static_cast<int64_t>(active_.size()); }
  const std::vector<int>& active() const { return active_; }
  const Approx& base() const { return *base_; }
  const Vec& eps() const { return eps_; }
  const Vec& exact_norms() const { return en_; }
  const Vec& approx_norms() const { return an_; }
  double max_eps() const { return max_eps_; }

 private:
  void gather_metadata() {  // 189-201
    const size_t n = active_.size();
    eps_.resize(n);
    en_.resize(n);
    an_.resize(n);
    for (size_t j = 0; j < n; ++j) {
      const size_t g = static_cast<size_t>(active_[j]);
      eps_[j] = base_->eps[g];
      en_[j] = base_->exact_norms[g];
      an_[j] = base_->approx_norms[g];
    }
    max_eps_ = 0.0;
    if (n > 0) {
      max_eps_ = eps_[0];
      for (double e : eps_) max_eps_ = std::max(max_eps_, e);
    }
  }
  const Approx* base_;
  std::vector<int> active_;
  Vec eps_, en_, an_;
  double max_eps_ = 0.0;
};

struct Result {
  Vec x;
  bool converged = false;
  double final_gap = std::numeric_limits<double>::quiet_NaN();
  uint64_t iterations = 0;
  uint64_t total_flops = 0;
  std::vector<fl1_trace_row> trace;
  std::vector<fl1_switch_event> switches;
  std::vector<int> final_active;
  bool gap_warning = false;
  double setup_ms = 0.0, run_ms = 0.0;
  int64_t power_steps = 0;
  double power_bytes = 0.0;  // 16 N |S| per power step (bench.py's byte accounting)
};

const Op* gram_of(const fl1_dict* d);  // exact_gram handle -> its dense K x K operator

// ---------------------------------------------------------------- Engine (fastl1.cpp:213-749)
struct Engine {
  const Seq& seq;
  const Vec& y;
  const double lambda;
  const fl1_switch_config& cfg;
  const fl1_run_options& opts;
  const int64_t n, k;
  const int last;
  int dict_index;
  ActiveOp op;
  Vec x, x_prev;
  double t_k = 1.0;
  bool momentum_ready = false;
  Vec u, v;
  Vec aty_active, aty_exact_active;
  const double y_sqnorm, y_norm;
  double lipschitz = 0.0, inv_l = 0.0;
  Vec lead_vector;
  int64_t active_at_last_l = 0;
  // Gram-backed exact phase (fastl1.cpp:232-237): tracked G x / G v and A^T y, full K
  const Op* gram = nullptr;
  bool gram_mode = false;
  Vec gx, gv, aty_full;
  Result result;
  uint64_t ledger = 0;
  std::chrono::steady_clock::time_point t_start;

  static int initial_index(const Seq& s, const fl1_run_options& o) {
    return o.variant == FL1_MULTI_DICT ? 0 : s.levels() - 1;
  }

  Engine(const Seq& s, const Vec& yy, double lam, const fl1_switch_config& c, const fl1_run_options& o)
      : seq(s),
        y(yy),
        lambda(lam),
        cfg(c),
        opts(o),
        n(s.exact().op->n),
        k(s.exact().op->k),
        last(s.levels() - 1),
        dict_index(initial_index(s, o)),
        op(s.d[static_cast<size_t>(initial_index(s, o))].get()),
        y_sqnorm(sqnorm(yy)),
        y_norm(std::sqrt(sqnorm(yy))) {
    if (lambda <= 0) throw std::invalid_argument("lambda must be positive");
    if (static_cast<int64_t>(y.size()) != n) throw std::invalid_argument("y has wrong length");
    if (cfg.gamma_threshold <= 0.0 || cfg.gamma_threshold >= 1.0)
      throw std::invalid_argument("gamma threshold must lie in (0, 1)");
    if (cfg.screening_interval < 1) throw std::invalid_argument("screening interval must be >= 1");
    x.assign(static_cast<size_t>(k), 0.0);
    if (opts.x_init) x.assign(opts.x_init, opts.x_init + k);  // extension
    if (opts.exact_gram) {
      gram = gram_of(opts.exact_gram);
      if (!gram->dense || gram->n != k || gram->k != k) throw std::invalid_argument("exact_gram must be K x K");
    }
    const auto t0 = std::chrono::steady_clock::now();
    setup_dictionary(true);
    result.setup_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }

  // use_gram_now (fastl1.cpp:278-281)
  bool use_gram_now() const {
    return gram != nullptr && !opts.observer && dict_index == last && seq.at(dict_index).op->dense;
  }

  void gather_from_full(const Vec& full, Vec& out) const {  // 343-346
    out.resize(static_cast<size_t>(op.size()));
    for (int64_t j = 0; j < op.size(); ++j) out[static_cast<size_t>(j)] = full[static_cast<size_t>(op.active()[static_cast<size_t>(j)])];
  }

  Vec gram_product(const Vec& compact) const {  // 335-341: sum over nonzeros of x_j G(:, active_j)
    Vec out(static_cast<size_t>(k), 0.0);
    for (int64_t j = 0; j < static_cast<int64_t>(compact.size()); ++j) {
      const double xj = compact[static_cast<size_t>(j)];
      if (xj == 0.0) continue;
      const double* col = gram->a.data() + static_cast<size_t>(op.active()[static_cast<size_t>(j)]) * static_cast<size_t>(k);
      for (int64_t i = 0; i < k; ++i) out[static_cast<size_t>(i)] += xj * col[i];
    }
    return out;
  }

  void setup_dictionary(bool first) {  // 283-324
    const Approx& d = seq.at(dict_index);
    if (!first) op.rebase(&d);
    gram_mode = use_gram_now();
    if (gram_mode && aty_full.empty()) aty_full = d.op->adjoint(y);
    if (opts.rule == FL1_RULE_DYNAMIC) {
      if (gram_mode) gather_from_full(aty_full, aty_active);
      else aty_active = op.apply_adjoint(y);
      if (cfg.precompute_aty && aty_exact_active.empty()) {
        const Vec full = seq.exact().op->adjoint(y);
        aty_exact_active.resize(static_cast<size_t>(op.size()));
        for (int64_t j = 0; j < op.size(); ++j)
          aty_exact_active[static_cast<size_t>(j)] = full[static_cast<size_t>(op.active()[static_cast<size_t>(j)])];
      }
    }
    if (opts.full_lipschitz && op.size() == k) {
      if (dict_index >= opts.n_full_lipschitz) throw std::invalid_argument("full_lipschitz too short");
      lipschitz = opts.full_lipschitz[dict_index];
    } else {
      lipschitz = restricted_lipschitz();
    }
    inv_l = 1.0 / lipschitz;
    active_at_last_l = op.size();
    if (gram_mode) {  // tracked products restart with the new operator
      gx = gram_product(x);
      gv.clear();
    } else {
      u = op.apply(x);
      v.clear();
    }
    momentum_ready = false;
    t_k = 1.0;
  }

  double restricted_lipschitz() {  // 326-333
    const Vec* warm = static_cast<int64_t>(lead_vector.size()) == op.size() && norm2(lead_vector) > 0
                          ? &lead_vector
                          : nullptr;
    Vec lead_out;
    const int64_t steps0 = result.power_steps;
    const double sq = power_iteration_sq_norm([&](const Vec& xv) { return op.apply(xv); },
                                              [&](const Vec& rv) { return op.apply_adjoint(rv); },
                                              op.size(), warm, &lead_out, &result.power_steps);
    result.power_bytes += 16.0 * static_cast<double>(op.rows()) * static_cast<double>(op.size()) *
                          static_cast<double>(result.power_steps - steps0);
    lead_vector = std::move(lead_out);
    return std::max(sq, 1e-300) * kLipschitzSafety;
  }

  struct Products {
    Vec corr;
    double rho_g_sq = 0, rho_g_dot_y = 0, rho_x_sq = 0;
    Vec rho_g;
  };

  Products compute_products(double momentum) {  // 359-394
    Products p;
    if (gram_mode) {  // 373-393: corr = A^T y - G w, residual norms from the dots
      Vec gw = gx;
      if (momentum != 0.0)
        for (int64_t i = 0; i < k; ++i)
          gw[static_cast<size_t>(i)] = (1.0 + momentum) * gx[static_cast<size_t>(i)] - momentum * gv[static_cast<size_t>(i)];
      Vec corr_full(static_cast<size_t>(k));
      for (int64_t i = 0; i < k; ++i) corr_full[static_cast<size_t>(i)] = aty_full[static_cast<size_t>(i)] - gw[static_cast<size_t>(i)];
      gather_from_full(corr_full, p.corr);
      Vec gw_active, aty_act;
      gather_from_full(gw, gw_active);
      gather_from_full(aty_full, aty_act);
      Vec w = x;
      if (momentum != 0.0)
        for (size_t j = 0; j < w.size(); ++j) w[j] = (1.0 + momentum) * x[j] - momentum * x_prev[j];
      const double w_aty = dot(w, aty_act), w_gw = dot(w, gw_active);
      p.rho_g_sq = std::max(y_sqnorm - 2.0 * w_aty + w_gw, 0.0);
      p.rho_g_dot_y = y_sqnorm - w_aty;
      if (momentum != 0.0) {
        Vec gx_active;
        gather_from_full(gx, gx_active);
        const double x_aty = dot(x, aty_act), x_gx = dot(x, gx_active);
        p.rho_x_sq = std::max(y_sqnorm - 2.0 * x_aty + x_gx, 0.0);
      } else {
        p.rho_x_sq = p.rho_g_sq;
      }
      return p;
    }
    Vec uw = u;
    if (momentum != 0.0)
      for (int64_t i = 0; i < n; ++i)
        uw[static_cast<size_t>(i)] = (1.0 + momentum) * u[static_cast<size_t>(i)] - momentum * v[static_cast<size_t>(i)];
    p.rho_g.resize(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) p.rho_g[static_cast<size_t>(i)] = y[static_cast<size_t>(i)] - uw[static_cast<size_t>(i)];
    p.corr = op.apply_adjoint(p.rho_g);
    p.rho_g_sq = sqnorm(p.rho_g);
    p.rho_g_dot_y = dot(y, p.rho_g);
    if (momentum != 0.0) {
      double s = 0.0;
      for (int64_t i = 0; i < n; ++i) {
        const double e = y[static_cast<size_t>(i)] - u[static_cast<size_t>(i)];
        s += e * e;
      }
      p.rho_x_sq = s;
    } else {
      p.rho_x_sq = p.rho_g_sq;
    }
    return p;
  }

  struct DualScalars {
    double scale_prime = 0, scale_tilde = 0;
    bool ray_is_y = false;
    double ray_sq = 0, ray_dot_y = 0;
  };

  Vec corr_of_y() const {  // 433-439
    if (opts.rule == FL1_RULE_DYNAMIC && static_cast<int64_t>(aty_active.size()) == op.size()) return aty_active;
    if (gram_mode) {
      Vec out;
      gather_from_full(aty_full, out);
      return out;
    }
    return op.apply_adjoint(y);
  }

  DualScalars dual_scalars(const Products& p) {  // 406-450
    DualScalars d;
    if (p.rho_g_sq > 0.0) {
      d.ray_sq = p.rho_g_sq;
      d.ray_dot_y = p.rho_g_dot_y;
      const double rho_norm = std::sqrt(p.rho_g_sq);
      double dp = 0.0, ds = 0.0;
      const Vec& eps = op.eps();
      for (size_t j = 0; j < p.corr.size(); ++j) {
        const double ac = std::abs(p.corr[j]);
        dp = std::max(dp, ac);
        ds = std::max(ds, ac + eps[j] * rho_norm);
      }
      const double projection = p.rho_g_dot_y / (lambda * p.rho_g_sq);
      const double ap = ds > 0 ? 1.0 / ds : std::numeric_limits<double>::infinity();
      const double at = dp > 0 ? 1.0 / dp : std::numeric_limits<double>::infinity();
      d.scale_prime = std::min(std::max(projection, -ap), ap);
      d.scale_tilde = std::min(std::max(projection, -at), at);
      return d;
    }
    d.ray_is_y = true;
    d.ray_sq = y_sqnorm;
    d.ray_dot_y = y_sqnorm;
    const Vec corr_y = corr_of_y();
    double dp = 0.0, ds = 0.0;
    const Vec& eps = op.eps();
    for (size_t j = 0; j < corr_y.size(); ++j) {
      const double ac = std::abs(corr_y[j]) / lambda;
      dp = std::max(dp, ac);
      ds = std::max(ds, ac + eps[j] * y_norm / lambda);
    }
    d.scale_prime = 1.0 / (lambda * std::max(1.0, ds));
    d.scale_tilde = 1.0 / (lambda * std::max(1.0, dp));
    return d;
  }

  double dual_of(double scale, const DualScalars& d) const {  // 453-457
    const double dist_sq =
        scale * scale * d.ray_sq - 2.0 * scale * d.ray_dot_y / lambda + y_sqnorm / (lambda * lambda);
    return 0.5 * y_sqnorm - 0.5 * lambda * lambda * dist_sq;
  }

  double elapsed_ms() const {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
  }

  uint64_t row_flops(int dict, int64_t active, int nnz) const {  // 647-665
    const auto un = static_cast<uint64_t>(n);
    const auto uk = static_cast<uint64_t>(k);
    const auto ua = static_cast<uint64_t>(active);
    const auto uz = static_cast<uint64_t>(nnz);
    switch (opts.variant) {
      case FL1_PLAIN:
        return flops_plain(uk, un, uz);
      case FL1_SCREENED:
        return flops_screened(ua, un, uz);
      default:
        if (dict < last) return flops_stable(seq.at(dict).op->matvec_flops(), un, ua, uz);
        return flops_screened(ua, un, uz);
    }
  }

  void apply_restriction(const std::vector<int>& kept_local) {  // 667-702
    std::vector<char> keep(static_cast<size_t>(op.size()), 0);
    for (int pos : kept_local) keep[static_cast<size_t>(pos)] = 1;
    const bool fix_history = opts.solver == FL1_FISTA && momentum_ready;
    for (int64_t j = 0; j < op.size(); ++j) {
      if (keep[static_cast<size_t>(j)]) continue;
      const int g = op.active()[static_cast<size_t>(j)];
      if (fix_history && static_cast<int64_t>(x_prev.size()) == op.size() && x_prev[static_cast<size_t>(j)] != 0.0) {
        const double xp = x_prev[static_cast<size_t>(j)];
        if (gram_mode) {  // 678-679: gv -= x_prev_j G(:, g)
          const double* col = gram->a.data() + static_cast<size_t>(g) * static_cast<size_t>(k);
          for (int64_t i = 0; i < k; ++i) gv[static_cast<size_t>(i)] -= xp * col[i];
        } else {
          const Vec col = op.column_global(g);
          for (int64_t i = 0; i < n; ++i) v[static_cast<size_t>(i)] -= xp * col[static_cast<size_t>(i)];
        }
      }
    }
    auto gather = [&](Vec& vec) {
      if (static_cast<int64_t>(vec.size()) != op.size()) return;
      Vec next(kept_local.size());
      for (size_t j = 0; j < kept_local.size(); ++j) next[j] = vec[static_cast<size_t>(kept_local[j])];
      vec = std::move(next);
    };
    gather(x);
    gather(x_prev);
    gather(aty_active);
    gather(aty_exact_active);
    if (static_cast<int64_t>(lead_vector.size()) == op.size())
      gather(lead_vector);
    else
      lead_vector.clear();
    op.restrict_to_local(kept_local);
  }

  void fire_observer(uint64_t t, const Products& p, const DualScalars& ds, double radius,
                     const std::vector<int>& kept_local) {  // 704-734
    const Vec& ray = ds.ray_is_y ? y : p.rho_g;
    Vec tp(static_cast<size_t>(n)), tt(static_cast<size_t>(n)), center(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
      tp[static_cast<size_t>(i)] = ds.scale_prime * ray[static_cast<size_t>(i)];
      tt[static_cast<size_t>(i)] = ds.scale_tilde * ray[static_cast<size_t>(i)];
      center[static_cast<size_t>(i)] = opts.rule == FL1_RULE_GAP ? tp[static_cast<size_t>(i)] : y[static_cast<size_t>(i)] / lambda;
    }
    std::vector<int32_t> active_global(op.active().begin(), op.active().end());
    std::vector<int32_t> kept_global;
    kept_global.reserve(kept_local.size());
    for (int pos : kept_local) kept_global.push_back(active_global[static_cast<size_t>(pos)]);
    fl1_screen_event ev{};
    ev.iter = t;
    ev.dict_index = dict_index;
    ev.n = n;
    ev.center = center.data();
    ev.radius = radius;
    ev.theta_prime = tp.data();
    ev.theta_tilde = tt.data();
    ev.scale_prime = ds.scale_prime;
    ev.scale_tilde = ds.scale_tilde;
    ev.n_active_before = static_cast<int64_t>(active_global.size());
    ev.active_before = active_global.data();
    ev.n_kept = static_cast<int64_t>(kept_global.size());
    ev.kept = kept_global.data();
    opts.observer(&ev, opts.observer_user);
  }

  void finish(bool warned) {  // 741-748
    result.gap_warning = warned;
    result.total_flops = ledger;
    result.final_active = op.active();
    Vec full(static_cast<size_t>(k), 0.0);
    for (int64_t j = 0; j < op.size(); ++j) full[static_cast<size_t>(op.active()[static_cast<size_t>(j)])] = x[static_cast<size_t>(j)];
    result.x = std::move(full);
    result.run_ms = elapsed_ms();
  }

  Result run() {  // 459-645
    t_start = std::chrono::steady_clock::now();
    const int64_t total_atoms = k;
    bool emitted_warning = false;
    const uint64_t interval = static_cast<uint64_t>(cfg.screening_interval);
    for (uint64_t t = 0; t < cfg.max_iterations; ++t) {
      double momentum = 0.0;
      double t_next = t_k;
      if (opts.solver == FL1_FISTA && momentum_ready) {
        t_next = 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * t_k * t_k));
        momentum = (t_k - 1.0) / t_next;
      }
      Products p = compute_products(momentum);
      const double x_l1 = l1(x);
      const double primal = 0.5 * p.rho_x_sq + lambda * x_l1;
      DualScalars ds = dual_scalars(p);
      double gap_prime = primal - dual_of(ds.scale_prime, ds);
      double gap_tilde = primal - dual_of(ds.scale_tilde, ds);
      if (gap_prime < kGapRoundoffFloor || gap_tilde < kGapRoundoffFloor) emitted_warning = true;
      gap_prime = std::max(gap_prime, 0.0);
      gap_tilde = std::max(gap_tilde, 0.0);

      const bool exact_phase = dict_index == last;
      const double stop_tol = cfg.rel_tolerance > 0 ? cfg.rel_tolerance * primal : cfg.tolerance;
      const bool stop_now = exact_phase && gap_tilde <= stop_tol;
      const bool screen_now = !stop_now && opts.variant != FL1_PLAIN && (t % interval == 0);

      const int64_t active_before = op.size();
      double gamma = -1.0;
      int next_dict = dict_index;
      bool speed_switch = false;
      std::vector<int> kept_local;
      bool kept_shrinks = false;

      if (screen_now) {  // 494-566
        double radius = 0.0, center_norm = 0.0;
        Vec dots(static_cast<size_t>(op.size()));
        bool stable_test = true;
        if (opts.rule == FL1_RULE_GAP) {
          const double delta = exact_phase ? 0.0 : stable_gap_delta(std::sqrt(p.rho_x_sq), op.max_eps(), x_l1);
          radius = std::sqrt(2.0 * gap_prime + 2.0 * delta) / lambda;
          const double s = std::abs(ds.scale_prime);
          center_norm = s * std::sqrt(ds.ray_sq);
          if (ds.ray_is_y) {
            Vec corr_y;
            if (static_cast<int64_t>(aty_active.size()) == op.size())
              corr_y = aty_active;
            else if (gram_mode)
              gather_from_full(aty_full, corr_y);
            else
              corr_y = op.apply_adjoint(y);
            for (size_t j = 0; j < dots.size(); ++j) dots[j] = std::abs(ds.scale_prime * corr_y[j]);
          } else {
            for (size_t j = 0; j < dots.size(); ++j) dots[j] = std::abs(ds.scale_prime * p.corr[j]);
          }
        } else {
          const double s = ds.scale_prime;
          const double dist_sq = s * s * ds.ray_sq - 2.0 * s * ds.ray_dot_y / lambda + y_sqnorm / (lambda * lambda);
          radius = std::sqrt(std::max(dist_sq, 0.0));
          center_norm = y_norm / lambda;
          if (cfg.precompute_aty && static_cast<int64_t>(aty_exact_active.size()) == op.size()) {
            for (size_t j = 0; j < dots.size(); ++j) dots[j] = std::abs(aty_exact_active[j] / lambda);
            stable_test = false;
          } else {
            for (size_t j = 0; j < dots.size(); ++j) dots[j] = std::abs(aty_active[j] / lambda);
          }
        }
        ScreenResult sr;
        if (stable_test) {
          sr = screen_precomputed(dots, op.eps(), op.exact_norms(), op.approx_norms(), center_norm, radius);
        } else {
          for (size_t j = 0; j < dots.size(); ++j)
            if (sphere_test(dots[j], op.exact_norms()[j], radius) >= 1.0) sr.kept.push_back(static_cast<int>(j));
          sr.lookahead_count = static_cast<int>(sr.kept.size());
        }
        kept_local = std::move(sr.kept);
        kept_shrinks = static_cast<int64_t>(kept_local.size()) < op.size();
        if (opts.observer) fire_observer(t, p, ds, radius, kept_local);
        if (!exact_phase) {
          gamma = gap_ratio(gap_tilde, gap_prime);
          if (opts.variant == FL1_MULTI_DICT) {
            const double rc = seq.at(dict_index).rc;
            next_dict = switch_dictionary(dict_index, last, gamma, cfg.gamma_threshold, sr.lookahead_count, rc, total_atoms);
            speed_switch = static_cast<double>(sr.lookahead_count) <= rc * static_cast<double>(total_atoms);
          }
        }
      }

      int x_nnz;
      if (stop_now) {
        x_nnz = count_nonzeros(x);
      } else {  // 572-609
        Vec g = x;
        if (momentum != 0.0)
          for (size_t j = 0; j < g.size(); ++j) g[j] = (1.0 + momentum) * x[j] - momentum * x_prev[j];
        Vec x_next(static_cast<size_t>(op.size()));
        const double thresh = lambda * inv_l;
        for (size_t j = 0; j < x_next.size(); ++j) x_next[j] = soft_threshold(g[j] + inv_l * p.corr[j], thresh);
        if (opts.solver == FL1_FISTA) {
          if (momentum_ready) t_k = t_next;
          x_prev = x;
          if (gram_mode) gv = gx;  // 584-588
          else v = u;
          momentum_ready = true;
        }
        x = std::move(x_next);
        if (kept_shrinks) apply_restriction(kept_local);
        if (gram_mode) gx = gram_product(x);  // 596-600
        else u = op.apply(x);
        x_nnz = count_nonzeros(x);
        if (op.size() * 2 <= active_at_last_l && op.size() > 0 && next_dict == dict_index) {
          lipschitz = restricted_lipschitz();
          inv_l = 1.0 / lipschitz;
          active_at_last_l = op.size();
        }
      }

      ledger += row_flops(dict_index, active_before, x_nnz);
      if (opts.collect_trace) {
        fl1_trace_row row{};
        row.iter = t;
        row.dict_index = dict_index;
        row.active_size = static_cast<int32_t>(active_before);
        row.gap = exact_phase ? gap_tilde : -1.0;
        row.gamma = gamma;
        row.flops_cum = ledger;
        row.wall_ms = elapsed_ms();
        row.x_nnz = x_nnz;
        result.trace.push_back(row);
      }
      if (stop_now) {
        result.converged = true;
        result.final_gap = gap_tilde;
        result.iterations = t + 1;
        finish(emitted_warning);
        return std::move(result);
      }
      if (next_dict != dict_index) {
        result.switches.push_back({t, dict_index, next_dict, speed_switch ? 1 : 0, 0});
        dict_index = next_dict;
        setup_dictionary(false);
      }
    }
    result.converged = false;
    result.iterations = cfg.max_iterations;
    result.final_gap = std::numeric_limits<double>::quiet_NaN();
    finish(emitted_warning);
    return std::move(result);
  }
};

template <class F>
int guard(F&& f) {
  try {
    f();
    return FL1_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return FL1_EINVAL;
  } catch (const std::bad_alloc&) {
    g_err = "out of memory";
    return FL1_ENOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return FL1_ERUNTIME;
  }
}

}  // namespace

struct orc_ctx {
  int device = 0;
};
struct orc_dict {
  std::shared_ptr<const Op> op;
};
namespace {
const Op* gram_of(const fl1_dict* d) { return reinterpret_cast<const orc_dict*>(d)->op.get(); }
}  // namespace
struct orc_approx {
  std::shared_ptr<const Approx> a;
};
struct orc_seq {
  Seq s;
};
struct orc_result {
  Result r;
  int64_t k = 0;
};

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
const char* orc_version(void) { return "fl1-oracle 1.0 (Eigen-free restatement of fastl1 run_lasso)"; }
void orc_set_threads(int n) { g_threads = n < 1 ? 1 : n; }
int orc_get_threads(void) { return g_threads; }

int orc_ctx_create(int device, orc_ctx** out) {
  return guard([&] { *out = new orc_ctx{device}; });
}
int orc_ctx_destroy(orc_ctx* ctx) {
  delete ctx;
  return FL1_OK;
}

int orc_gram_create(orc_dict* d, orc_dict** out) {  // G = A^T A (bench.cpp:190-197)
  return guard([&] {
    const Op& a = *d->op;
    if (!a.dense) throw std::invalid_argument("exact_gram needs a dense dictionary");
    const int64_t n = a.n, k = a.k;
    auto op = std::make_shared<Op>();
    op->dense = true;
    op->n = k;
    op->k = k;
    op->a.assign(static_cast<size_t>(k * k), 0.0);
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (int64_t j = 0; j < k; ++j)
      for (int64_t i = 0; i <= j; ++i) {
        double s = 0.0;
        for (int64_t r = 0; r < n; ++r) s += a.a[static_cast<size_t>(i * n + r)] * a.a[static_cast<size_t>(j * n + r)];
        op->a[static_cast<size_t>(j * k + i)] = s;
        op->a[static_cast<size_t>(i * k + j)] = s;
      }
    op->norms.resize(static_cast<size_t>(k));
    for (int64_t j = 0; j < k; ++j) {
      double s = 0.0;
      for (int64_t i = 0; i < k; ++i) s += op->a[static_cast<size_t>(j * k + i)] * op->a[static_cast<size_t>(j * k + i)];
      op->norms[static_cast<size_t>(j)] = std::sqrt(s);
    }
    *out = new orc_dict{op};
  });
}

int orc_dict_dense(orc_ctx*, const double* a, int64_t n, int64_t k, orc_dict** out) {
  return guard([&] {
    if (n < 1 || k < 1) throw std::invalid_argument("dictionary must have at least one row and one column");
    auto op = std::make_shared<Op>();
    op->dense = true;
    op->n = n;
    op->k = k;
    op->a.assign(a, a + n * k);
    op->norms.resize(static_cast<size_t>(k));
    for (int64_t j = 0; j < k; ++j) {
      double s = 0.0;
      for (int64_t i = 0; i < n; ++i) s += a[j * n + i] * a[j * n + i];
      op->norms[static_cast<size_t>(j)] = std::sqrt(s);
    }
    *out = new orc_dict{op};
  });
}

int orc_dict_sukro(orc_ctx*, int32_t n_terms, int64_t m, int64_t q, const double* const* left,
                   const double* const* right, const double* col_scale, orc_dict** out) {
  return guard([&] {
    if (n_terms < 1) throw std::invalid_argument("SuKro needs at least one term");
    if (m < 1 || q < 1) throw std::invalid_argument("empty SuKro factor");
    auto op = std::make_shared<Op>();
    op->dense = false;
    op->m = m;
    op->q = q;
    op->n = m * m;
    op->k = q * q;
    for (int t = 0; t < n_terms; ++t) {
      op->left.emplace_back(left[t], left[t] + m * q);
      op->right.emplace_back(right[t], right[t] + m * q);
    }
    if (col_scale) op->col_scale.assign(col_scale, col_scale + q * q);
    *out = new orc_dict{op};
  });
}

int orc_dict_destroy(orc_dict* d) {
  delete d;
  return FL1_OK;
}
int orc_dict_shape(const orc_dict* d, int64_t* rows, int64_t* cols) {
  *rows = d->op->n;
  *cols = d->op->k;
  return FL1_OK;
}
int orc_dict_is_dense(const orc_dict* d) { return d->op->dense ? 1 : 0; }
uint64_t orc_dict_matvec_flops(const orc_dict* d) { return d->op->matvec_flops(); }
int orc_dict_atom_norms(const orc_dict* d, double* out) {
  return guard([&] {
    if (d->op->dense) {
      std::copy(d->op->norms.begin(), d->op->norms.end(), out);
    } else {
      for (int64_t j = 0; j < d->op->k; ++j) out[j] = norm2(d->op->column(j));
    }
  });
}
int orc_dict_apply(orc_dict* d, const double* x, double* out) {
  return guard([&] {
    const Vec r = d->op->apply(Vec(x, x + d->op->k));
    std::copy(r.begin(), r.end(), out);
  });
}
int orc_dict_apply_adjoint(orc_dict* d, const double* r, double* out) {
  return guard([&] {
    const Vec o = d->op->adjoint(Vec(r, r + d->op->n));
    std::copy(o.begin(), o.end(), out);
  });
}
int orc_dict_column(orc_dict* d, int64_t j, double* out) {
  return guard([&] {
    const Vec c = d->op->column(j);
    std::copy(c.begin(), c.end(), out);
  });
}
int orc_dict_to_dense(orc_dict* d, double* out) {
  return guard([&] {
    for (int64_t j = 0; j < d->op->k; ++j) {
      const Vec c = d->op->column(j);
      std::copy(c.begin(), c.end(), out + j * d->op->n);
    }
  });
}

int orc_approx_create(orc_dict* d, const double* eps, double op_err, double rc, const double* an,
                      const double* en, orc_approx** out) {
  return guard([&] {
    auto a = std::make_shared<Approx>();
    const int64_t k = d->op->k;
    a->op = d->op;
    a->eps.assign(eps, eps + k);
    a->op_err = op_err;
    a->rc = rc;
    a->approx_norms.assign(an, an + k);
    a->exact_norms.assign(en, en + k);
    *out = new orc_approx{a};
  });
}
int orc_approx_exact(orc_dict* d, orc_approx** out) {  // make_exact_approx (dictionary.cpp:216-225)
  return guard([&] {
    if (!d->op->dense) throw std::invalid_argument("make_exact_approx needs a dense dictionary");
    auto a = std::make_shared<Approx>();
    a->op = d->op;
    a->eps.assign(static_cast<size_t>(d->op->k), 0.0);
    a->op_err = 0.0;
    a->rc = 1.0;
    a->approx_norms = d->op->norms;
    a->exact_norms = d->op->norms;
    *out = new orc_approx{a};
  });
}
int orc_approx_destroy(orc_approx* a) {
  delete a;
  return FL1_OK;
}
int orc_seq_create(orc_approx* const* levels, int32_t n_levels, orc_seq** out) {
  return guard([&] {
    auto s = std::make_unique<orc_seq>();
    for (int i = 0; i < n_levels; ++i) s->s.d.push_back(levels[i]->a);
    s->s.validate();
    *out = s.release();
  });
}
int orc_seq_destroy(orc_seq* s) {
  delete s;
  return FL1_OK;
}

int orc_solve(orc_seq* s, const double* y, double lambda, const fl1_switch_config* cfg,
              const fl1_run_options* opts, orc_result** out) {
  return guard([&] {
    s->s.validate();  // run_lasso (fastl1.cpp:755)
    const Vec yy(y, y + s->s.exact().op->n);
    Engine e(s->s, yy, lambda, *cfg, *opts);
    auto r = std::make_unique<orc_result>();
    r->r = e.run();
    r->k = s->s.exact().op->k;
    *out = r.release();
  });
}
int orc_result_info_get(const orc_result* r, fl1_result_info* o) {
  *o = fl1_result_info{};
  o->k = r->k;
  o->converged = r->r.converged;
  o->gap_warning = r->r.gap_warning;
  o->final_gap = r->r.final_gap;
  o->iterations = r->r.iterations;
  o->total_flops = r->r.total_flops;
  o->n_trace = static_cast<int64_t>(r->r.trace.size());
  o->n_switches = static_cast<int64_t>(r->r.switches.size());
  o->n_final_active = static_cast<int64_t>(r->r.final_active.size());
  o->device_ms = r->r.run_ms;
  o->batch_device_ms = r->r.run_ms;
  o->setup_ms = r->r.setup_ms;
  o->kernel_launches = 0;
  o->power_iterations = r->r.power_steps;
  return FL1_OK;
}
int orc_result_power_bytes(const orc_result* r, double* out) {
  *out = r->r.power_bytes;
  return FL1_OK;
}
int orc_result_x(const orc_result* r, double* out) {
  std::copy(r->r.x.begin(), r->r.x.end(), out);
  return FL1_OK;
}
int orc_result_trace(const orc_result* r, fl1_trace_row* out) {
  std::copy(r->r.trace.begin(), r->r.trace.end(), out);
  return FL1_OK;
}
int orc_result_switches(const orc_result* r, fl1_switch_event* out) {
  std::copy(r->r.switches.begin(), r->r.switches.end(), out);
  return FL1_OK;
}
int orc_result_final_active(const orc_result* r, int32_t* out) {
  std::copy(r->r.final_active.begin(), r->r.final_active.end(), out);
  return FL1_OK;
}
void orc_result_free(orc_result* r) { delete r; }

int orc_lambda_max(orc_dict* d, const double* y, double* out) {  // screening.cpp:9-11
  return guard([&] {
    const Vec c = d->op->adjoint(Vec(y, y + d->op->n));
    double m = 0.0;
    for (double e : c) m = std::max(m, std::abs(e));
    *out = m;
  });
}
int orc_lipschitz_bound(orc_dict* d, double* out) {  // solver.cpp:108-114
  return guard([&] {
    const Op& op = *d->op;
    const double sq = power_iteration_sq_norm([&](const Vec& x) { return op.apply(x); },
                                              [&](const Vec& r) { return op.adjoint(r); }, op.k,
                                              nullptr, nullptr, nullptr);
    *out = sq * kLipschitzSafety;
  });
}
int orc_screen_precomputed(orc_ctx*, int64_t n, const double* dots, const double* eps,
                           const double* en, const double* an, double cn, double r, int32_t* kept,
                           int64_t* n_kept, int64_t* lookahead) {
  return guard([&] {
    const ScreenResult sr = screen_precomputed(Vec(dots, dots + n), Vec(eps, eps + n), Vec(en, en + n),
                                               Vec(an, an + n), cn, r);
    std::copy(sr.kept.begin(), sr.kept.end(), kept);
    *n_kept = static_cast<int64_t>(sr.kept.size());
    *lookahead = sr.lookahead_count;
  });
}

double orc_soft_threshold(double z, double u) { return soft_threshold(z, u); }
double orc_gap_ratio(double a, double b) { return gap_ratio(a, b); }
int orc_switch_dictionary(int i, int last, double g, double gt, int64_t la, double rc, int64_t ta) {
  return switch_dictionary(i, last, g, gt, la, rc, ta);
}
uint64_t orc_flops_plain(uint64_t k, uint64_t n, uint64_t z) { return flops_plain(k, n, z); }
uint64_t orc_flops_screened(uint64_t a, uint64_t n, uint64_t z) { return flops_screened(a, n, z); }
uint64_t orc_flops_stable(uint64_t mv, uint64_t n, uint64_t a, uint64_t z) { return flops_stable(mv, n, a, z); }
uint64_t orc_recompute_flops(const fl1_trace_row* trace, int64_t n_rows, const orc_seq* s,
                             int32_t variant, int64_t n, int64_t k, int32_t* rows_match) {
  // fastl1.cpp:51-81
  const auto un = static_cast<uint64_t>(n), uk = static_cast<uint64_t>(k);
  const int last = s->s.levels() - 1;
  uint64_t total = 0;
  bool all = true;
  for (int64_t r = 0; r < n_rows; ++r) {
    const fl1_trace_row& row = trace[r];
    const auto a = static_cast<uint64_t>(row.active_size);
    const auto z = static_cast<uint64_t>(row.x_nnz);
    switch (variant) {
      case FL1_PLAIN:
        total += flops_plain(uk, un, z);
        break;
      case FL1_SCREENED:
        total += flops_screened(a, un, z);
        break;
      default:
        total += row.dict_index < last ? flops_stable(s->s.at(row.dict_index).op->matvec_flops(), un, a, z)
                                       : flops_screened(a, un, z);
    }
    all = all && total == row.flops_cum;
  }
  if (rows_match) *rows_match = all ? 1 : 0;
  return total;
}
double orc_stable_gap_delta(double rn, double e, double x1) { return stable_gap_delta(rn, e, x1); }
double orc_sphere_test(double d, double an, double r) { return sphere_test(d, an, r); }
double orc_stable_zone_test(double d, double eps, double cn, double en, double r) {
  return stable_zone_test(d, eps, cn, en, r);
}
double orc_stable_ball_test(double d, double eps, double cn, double an, double r) {
  return stable_ball_test(d, eps, cn, an, r);
}

// ---- steppers and objectives (solver.cpp:21-68)
int orc_ista_step(orc_dict* d, const double* y, double lambda, double step, const double* x,
                  double* x_next, double* residual, double* corr) {
  return guard([&] {
    const Op& op = *d->op;
    const Vec ax = op.apply(Vec(x, x + op.k));
    Vec res(static_cast<size_t>(op.n));
    for (int64_t i = 0; i < op.n; ++i) res[static_cast<size_t>(i)] = y[i] - ax[static_cast<size_t>(i)];
    const Vec c = op.adjoint(res);
    for (int64_t j = 0; j < op.k; ++j) x_next[j] = soft_threshold(x[j] + step * c[static_cast<size_t>(j)], lambda * step);
    if (residual) std::copy(res.begin(), res.end(), residual);
    if (corr) std::copy(c.begin(), c.end(), corr);
  });
}
int orc_fista_step(orc_dict* d, const double* y, double lambda, double step, const double* x,
                   double* x_prev, double* t_k, int32_t* momentum_ready, double* x_next,
                   double* residual, double* corr) {
  return guard([&] {
    const Op& op = *d->op;
    Vec g(x, x + op.k);
    if (*momentum_ready) {
      const double t_next = 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * *t_k * *t_k));
      const double mom = (*t_k - 1.0) / t_next;
      for (int64_t j = 0; j < op.k; ++j) g[static_cast<size_t>(j)] = x[j] + mom * (x[j] - x_prev[j]);
      *t_k = t_next;
    } else {
      *t_k = 1.0;
    }
    const Vec ag = op.apply(g);
    Vec res(static_cast<size_t>(op.n));
    for (int64_t i = 0; i < op.n; ++i) res[static_cast<size_t>(i)] = y[i] - ag[static_cast<size_t>(i)];
    const Vec c = op.adjoint(res);
    for (int64_t j = 0; j < op.k; ++j)
      x_next[j] = soft_threshold(g[static_cast<size_t>(j)] + step * c[static_cast<size_t>(j)], lambda * step);
    std::copy(x, x + op.k, x_prev);
    *momentum_ready = 1;
    if (residual) std::copy(res.begin(), res.end(), residual);
    if (corr) std::copy(c.begin(), c.end(), corr);
  });
}
double orc_primal_value(orc_dict* d, const double* y, double lambda, const double* x) {
  const Op& op = *d->op;
  const Vec ax = op.apply(Vec(x, x + op.k));
  double s = 0.0, a1 = 0.0;
  for (int64_t i = 0; i < op.n; ++i) {
    const double e = ax[static_cast<size_t>(i)] - y[i];
    s += e * e;
  }
  for (int64_t j = 0; j < op.k; ++j) a1 += std::abs(x[j]);
  return 0.5 * s + lambda * a1;
}
double orc_dual_value(int64_t n, const double* y, double lambda, const double* theta) {
  double ys = 0.0, ds = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    ys += y[i] * y[i];
    const double e = theta[i] - y[i] / lambda;
    ds += e * e;
  }
  return 0.5 * ys - 0.5 * lambda * lambda * ds;
}
double orc_duality_gap(orc_dict* d, const double* y, double lambda, const double* x,
                       const double* theta, int32_t* warn) {
  const double gap = orc_primal_value(d, y, lambda, x) - orc_dual_value(d->op->n, y, lambda, theta);
  if (warn) *warn = gap < kGapRoundoffFloor ? 1 : 0;
  return gap < 0.0 ? 0.0 : gap;
}
int orc_stable_lambda_max(orc_approx* a, const double* y, double* out) {  // screening.cpp:13-21
  return guard([&] {
    const Op& op = *a->a->op;
    const Vec c = op.adjoint(Vec(y, y + op.n));
    double yn = 0.0;
    for (int64_t i = 0; i < op.n; ++i) yn += y[i] * y[i];
    yn = std::sqrt(yn);
    double best = 0.0;
    for (int64_t j = 0; j < op.k; ++j) best = std::max(best, std::abs(c[static_cast<size_t>(j)]) + a->a->eps[static_cast<size_t>(j)] * yn);
    *out = best;
  });
}
int orc_dual_scale(orc_dict* d, const double* z, double* out) {  // screening.cpp:38-41
  return guard([&] {
    const Op& op = *d->op;
    const Vec c = op.adjoint(Vec(z, z + op.n));
    double m = 0.0;
    for (double e : c) m = std::max(m, std::abs(e));
    const double denom = std::max(1.0, m);
    for (int64_t i = 0; i < op.n; ++i) out[i] = z[i] / denom;
  });
}
int orc_stable_dual_scale(orc_approx* a, const double* z, double* out) {  // screening.cpp:43-51
  return guard([&] {
    const Op& op = *a->a->op;
    const Vec c = op.adjoint(Vec(z, z + op.n));
    double zn = 0.0;
    for (int64_t i = 0; i < op.n; ++i) zn += z[i] * z[i];
    zn = std::sqrt(zn);
    double worst = 0.0;
    for (int64_t j = 0; j < op.k; ++j) worst = std::max(worst, std::abs(c[static_cast<size_t>(j)]) + a->a->eps[static_cast<size_t>(j)] * zn);
    const double denom = std::max(1.0, worst);
    for (int64_t i = 0; i < op.n; ++i) out[i] = z[i] / denom;
  });
}
int orc_dual_point_dynamic(int64_t n, int64_t m, const double* residual, const double* corr,
                           const double* eps, const double* y, double lambda, orc_dict* dict,
                           double* theta_prime, double* theta_tilde, double* scale_prime,
                           double* scale_tilde) {  // screening.cpp:56-101
  return guard([&] {
    double rho_sq = 0.0;
    for (int64_t i = 0; i < n; ++i) rho_sq += residual[i] * residual[i];
    if (rho_sq <= 0.0) {
      if (!dict) throw std::invalid_argument("zero residual needs a dictionary");
      Vec z(static_cast<size_t>(n));
      for (int64_t i = 0; i < n; ++i) z[static_cast<size_t>(i)] = y[i] / lambda;
      const Vec cz = dict->op->adjoint(z);
      const double zn = norm2(z);
      double worst = 0.0, inf = 0.0;
      for (size_t j = 0; j < cz.size(); ++j) {
        const double e = static_cast<int64_t>(j) < m ? eps[j] : 0.0;
        worst = std::max(worst, std::abs(cz[j]) + e * zn);
        inf = std::max(inf, std::abs(cz[j]));
      }
      for (int64_t i = 0; i < n; ++i) {
        theta_prime[i] = z[static_cast<size_t>(i)] / std::max(1.0, worst);
        theta_tilde[i] = z[static_cast<size_t>(i)] / std::max(1.0, inf);
      }
      *scale_prime = *scale_tilde = 0.0;
      return;
    }
    const double rho_norm = std::sqrt(rho_sq);
    double ds = 0.0, dp = 0.0;
    for (int64_t j = 0; j < m; ++j) {
      const double ac = std::abs(corr[j]);
      dp = std::max(dp, ac);
      ds = std::max(ds, ac + eps[j] * rho_norm);
    }
    double ydr = 0.0;
    for (int64_t i = 0; i < n; ++i) ydr += y[i] * residual[i];
    const double projection = ydr / (lambda * rho_sq);
    const double ap = ds > 0 ? 1.0 / ds : std::numeric_limits<double>::infinity();
    const double at = dp > 0 ? 1.0 / dp : std::numeric_limits<double>::infinity();
    *scale_prime = std::min(std::max(projection, -ap), ap);
    *scale_tilde = std::min(std::max(projection, -at), at);
    for (int64_t i = 0; i < n; ++i) {
      theta_prime[i] = *scale_prime * residual[i];
      theta_tilde[i] = *scale_tilde * residual[i];
    }
  });
}
int orc_build_sphere(int32_t rule, int64_t n, const double* y, double lambda, double lmax,
                     double slmax, const double* theta, double gap, double delta, double* center,
                     double* radius) {  // screening.cpp:108-134
  return guard([&] {
    double yn = 0.0;
    for (int64_t i = 0; i < n; ++i) yn += y[i] * y[i];
    yn = std::sqrt(yn);
    switch (rule) {
      case 0:
      case 1:
        for (int64_t i = 0; i < n; ++i) center[i] = y[i] / lambda;
        *radius = std::abs(1.0 / (rule == 0 ? lmax : slmax) - 1.0 / lambda) * yn;
        break;
      case 2:
      case 3: {
        double s = 0.0;
        for (int64_t i = 0; i < n; ++i) {
          center[i] = y[i] / lambda;
          const double e = theta[i] - y[i] / lambda;
          s += e * e;
        }
        *radius = std::sqrt(s);
        break;
      }
      case 4:
        for (int64_t i = 0; i < n; ++i) center[i] = theta[i];
        *radius = std::sqrt(2.0 * std::max(gap, 0.0)) / lambda;
        break;
      case 5:
        for (int64_t i = 0; i < n; ++i) center[i] = theta[i];
        *radius = std::sqrt(2.0 * std::max(gap, 0.0) + 2.0 * delta) / lambda;
        break;
      default:
        throw std::invalid_argument("unknown rule");
    }
  });
}
int orc_screen(const int32_t* active, int64_t n_active, const double* center, double radius,
               orc_approx* a, int32_t use_stable, int32_t* kept, int64_t* n_kept) {  // 152-167
  return guard([&] {
    const Op& op = *a->a->op;
    const Vec c(center, center + op.n);
    const double cn = norm2(c);
    const Vec dots = op.adjoint(c);
    int64_t w = 0;
    for (int64_t p = 0; p < n_active; ++p) {
      const size_t j = static_cast<size_t>(active[p]);
      const double d = std::abs(dots[j]);
      const double val = use_stable ? stable_zone_test(d, a->a->eps[j], cn, a->a->exact_norms[j], radius)
                                    : sphere_test(d, a->a->approx_norms[j], radius);
      if (val >= 1.0) kept[w++] = active[p];
    }
    *n_kept = w;
  });
}

void orc_gen_normals(uint64_t seed, int64_t count, double* out) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> gauss(0.0, 1.0);
  for (int64_t i = 0; i < count; ++i) out[i] = gauss(rng);
}
void orc_gen_support(uint64_t seed, int64_t hi, int32_t support, int64_t* pos, double* val) {
  // Same expression as the reference, `x(pick(rng)) = gauss(rng);`, so the
  // compiler applies the same (C++17: right operand first) sequencing.
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> gauss(0.0, 1.0);
  std::uniform_int_distribution<int64_t> pick(0, hi);
  int64_t last = -1;
  auto slot = [&](int64_t i) -> double& {
    last = i;
    return *val;
  };
  for (int32_t s = 0; s < support; ++s) {
    slot(pick(rng)) = gauss(rng);
    pos[s] = last;
    ++val;
  }
}

}  // extern "C"
