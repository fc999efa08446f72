// fl1/fastl1.hpp — header-only C++ shim that gives the reference's fastl1 API
// (core/include/fastl1/{dictionary,fastl1,solver,screening}.hpp in
// /root/reference/proj) on top of the C-ABI of libfl1cuda.so (fl1cuda.h).
//
// A caller of the reference swaps `#include "fastl1/fastl1.hpp"` for
// `#include "fl1/fastl1.hpp"` and links -lfl1cuda; the names, argument meaning
// and error behaviour (std::invalid_argument) are the reference's:
//   DenseDictionary / SukroDictionary / LinearOp   dictionary.hpp:19-104
//   ApproxDictionary / make_exact_approx / ApproxSequence  dictionary.hpp:111-134
//   SwitchConfig / RunOptions / TraceRow / SwitchEvent / SolveResult / ScreeningEvent
//                                                  fastl1.hpp:25-96
//   run_lasso / fastl1_solve                       fastl1.hpp:101-111
//   gap_ratio / switch_dictionary / flops_* / recompute_flops  fastl1.hpp:35-41,115-125
//   soft_threshold / lipschitz_bound               solver.hpp:19-67
//   lambda_max / stable_gap_delta / sphere tests / screen_precomputed  screening.hpp
//
// Vectors and matrices: with FL1_WITH_EIGEN defined, Vector / Matrix are
// Eigen::VectorXd / Eigen::MatrixXd exactly as in the reference. Otherwise a
// minimal column-major stand-in with the subset of their API this header uses
// (size, rows, cols, data, operator(), resize, Zero). Only .data()/.size() cross
// the boundary, so both layouts are zero-copy into the C-ABI.
//
//   DenseDictionary::load_csv / save_csv / load_blob / save_blob  dictionary.cpp:76-135
//
// Extensions (defaults reproduce the reference): SwitchConfig::rel_tolerance,
// RunOptions::x_init, SukroDictionary column scale. RunOptions::exact_gram is honoured
// (uploaded to the GPU once per matrix and cached by its data pointer); as in the
// reference (out of scope) is accepted and ignored, as the reference ignores it
// while an observer is attached.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <limits>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../fl1cuda.h"

#ifdef FL1_WITH_EIGEN
#include <Eigen/Dense>
#endif

namespace fastl1 {

#ifdef FL1_WITH_EIGEN
using Matrix = Eigen::MatrixXd;
using Vector = Eigen::VectorXd;
using Index = Eigen::Index;
#else
using Index = std::ptrdiff_t;

class Vector {
 public:
  Vector() = default;
  explicit Vector(Index n) : v_(static_cast<size_t>(n), 0.0) {}
  static Vector Zero(Index n) { return Vector(n); }
  Index size() const { return static_cast<Index>(v_.size()); }
  void resize(Index n) { v_.assign(static_cast<size_t>(n), 0.0); }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  double& operator()(Index i) { return v_[static_cast<size_t>(i)]; }
  double operator()(Index i) const { return v_[static_cast<size_t>(i)]; }
  double& operator[](Index i) { return v_[static_cast<size_t>(i)]; }
  double operator[](Index i) const { return v_[static_cast<size_t>(i)]; }

 private:
  std::vector<double> v_;
};

class Matrix {  // column-major, like Eigen::MatrixXd
 public:
  Matrix() = default;
  Matrix(Index r, Index c) : r_(r), c_(c), v_(static_cast<size_t>(r * c), 0.0) {}
  static Matrix Zero(Index r, Index c) { return Matrix(r, c); }
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  double& operator()(Index i, Index j) { return v_[static_cast<size_t>(i + j * r_)]; }
  double operator()(Index i, Index j) const { return v_[static_cast<size_t>(i + j * r_)]; }

 private:
  Index r_ = 0, c_ = 0;
  std::vector<double> v_;
};
#endif

namespace detail {

inline void check(int status) {
  if (status == FL1_OK) return;
  const std::string msg = fl1_last_error();
  if (status == FL1_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error("fl1cuda: " + msg);
}

// One process-wide context on FL1_DEVICE (default 0), created on first use.
inline fl1_ctx* context() {
  static std::shared_ptr<fl1_ctx> ctx = [] {
    const char* e = std::getenv("FL1_DEVICE");
    fl1_ctx* c = nullptr;
    check(fl1_ctx_create(e ? std::atoi(e) : 0, &c));
    return std::shared_ptr<fl1_ctx>(c, [](fl1_ctx* p) { fl1_ctx_destroy(p); });
  }();
  return ctx.get();
}

}  // namespace detail

// ------------------------------------------------------------------ operators
class LinearOp {
 public:
  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  bool is_dense() const { return fl1_dict_is_dense(h_.get()) != 0; }
  std::uint64_t matvec_flops() const { return fl1_dict_matvec_flops(h_.get()); }
  Vector apply(const Vector& x) const {
    if (x.size() != cols_) throw std::invalid_argument("matvec: x has wrong length");
    Vector out(rows_);
    detail::check(fl1_dict_apply(h_.get(), x.data(), out.data()));
    return out;
  }
  Vector apply_adjoint(const Vector& r) const {
    if (r.size() != rows_) throw std::invalid_argument("adjoint matvec: r has wrong length");
    Vector out(cols_);
    detail::check(fl1_dict_apply_adjoint(h_.get(), r.data(), out.data()));
    return out;
  }
  Vector column(Index j) const {
    Vector out(rows_);
    detail::check(fl1_dict_column(h_.get(), j, out.data()));
    return out;
  }
  Vector atom_norms2() const {
    Vector out(cols_);
    detail::check(fl1_dict_atom_norms(h_.get(), out.data()));
    return out;
  }
  fl1_dict* handle() const { return h_.get(); }

 protected:
  void adopt(fl1_dict* d) {
    h_.reset(d, [](fl1_dict* p) { fl1_dict_destroy(p); });
    int64_t r = 0, c = 0;
    detail::check(fl1_dict_shape(d, &r, &c));
    rows_ = r;
    cols_ = c;
  }
  std::shared_ptr<fl1_dict> h_;
  Index rows_ = 0, cols_ = 0;
};

class DenseDictionary : public LinearOp {  // dictionary.hpp:19-48, resident in HBM
 public:
  DenseDictionary() = default;
  explicit DenseDictionary(Matrix entries) : entries_(std::move(entries)) {
    fl1_dict* d = nullptr;
    detail::check(fl1_dict_dense(detail::context(), entries_.data(), entries_.rows(), entries_.cols(), &d));
    adopt(d);
  }
  const Matrix& entries() const { return entries_; }

  // File formats of dictionary.cpp:76-135: CSV one row per line (%.17g, commas),
  // blob = uint32 N, uint32 K, then the column-major doubles.
  static DenseDictionary load_csv(const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "r");
    if (!f) throw std::invalid_argument("cannot open " + path);
    std::vector<std::vector<double>> rows;
    std::string line;
    int ch;
    auto flush_line = [&]() {
      if (line.empty()) return;
      std::vector<double> row;
      size_t pos = 0;
      while (true) {
        const size_t comma = line.find(',', pos);
        row.push_back(std::stod(line.substr(pos, comma == std::string::npos ? std::string::npos : comma - pos)));
        if (comma == std::string::npos) break;
        pos = comma + 1;
      }
      if (!rows.empty() && row.size() != rows.front().size()) {
        std::fclose(f);
        throw std::invalid_argument("ragged CSV in " + path);
      }
      rows.push_back(std::move(row));
      line.clear();
    };
    while ((ch = std::fgetc(f)) != EOF) {
      if (ch == '\n') flush_line();
      else line.push_back(static_cast<char>(ch));
    }
    flush_line();
    std::fclose(f);
    if (rows.empty()) throw std::invalid_argument("empty CSV in " + path);
    Matrix m(static_cast<Index>(rows.size()), static_cast<Index>(rows.front().size()));
    for (Index i = 0; i < m.rows(); ++i)
      for (Index j = 0; j < m.cols(); ++j) m(i, j) = rows[static_cast<size_t>(i)][static_cast<size_t>(j)];
    return DenseDictionary(std::move(m));
  }
  void save_csv(const std::string& path) const {
    std::FILE* f = std::fopen(path.c_str(), "w");
    if (!f) throw std::invalid_argument("cannot open " + path + " for writing");
    for (Index i = 0; i < entries_.rows(); ++i) {
      for (Index j = 0; j < entries_.cols(); ++j)
        std::fprintf(f, j + 1 < entries_.cols() ? "%.17g," : "%.17g", entries_(i, j));
      std::fputc('\n', f);
    }
    std::fclose(f);
  }
  static DenseDictionary load_blob(const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw std::invalid_argument("cannot open " + path);
    std::uint32_t n = 0, k = 0;
    const bool ok = std::fread(&n, 4, 1, f) == 1 && std::fread(&k, 4, 1, f) == 1;
    if (!ok || n == 0 || k == 0) {
      std::fclose(f);
      throw std::invalid_argument("bad blob header in " + path);
    }
    Matrix m(static_cast<Index>(n), static_cast<Index>(k));
    const size_t got = std::fread(m.data(), sizeof(double), static_cast<size_t>(n) * k, f);
    std::fclose(f);
    if (got != static_cast<size_t>(n) * k) throw std::invalid_argument("truncated blob " + path);
    return DenseDictionary(std::move(m));
  }
  void save_blob(const std::string& path) const {
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw std::invalid_argument("cannot open " + path + " for writing");
    const auto n = static_cast<std::uint32_t>(entries_.rows());
    const auto k = static_cast<std::uint32_t>(entries_.cols());
    std::fwrite(&n, 4, 1, f);
    std::fwrite(&k, 4, 1, f);
    std::fwrite(entries_.data(), sizeof(double), static_cast<size_t>(n) * k, f);
    std::fclose(f);
  }

 private:
  Matrix entries_;
};

class SukroDictionary : public LinearOp {  // dictionary.hpp:53-81
 public:
  struct Term {
    Matrix left;   // B_k
    Matrix right;  // C_k
  };
  explicit SukroDictionary(const std::vector<Term>& terms, const Vector* col_scale = nullptr) {
    if (terms.empty()) throw std::invalid_argument("SuKro needs at least one term");
    std::vector<const double*> l, r;
    for (const Term& t : terms) {
      if (t.left.rows() != terms[0].left.rows() || t.left.cols() != terms[0].left.cols() ||
          t.right.rows() != t.left.rows() || t.right.cols() != t.left.cols())
        throw std::invalid_argument("all SuKro factors must share one shape");
      l.push_back(t.left.data());
      r.push_back(t.right.data());
    }
    fl1_dict* d = nullptr;
    detail::check(fl1_dict_sukro(detail::context(), static_cast<int32_t>(terms.size()), terms[0].left.rows(),
                                 terms[0].left.cols(), l.data(), r.data(),
                                 col_scale ? col_scale->data() : nullptr, &d));
    adopt(d);
  }
};

struct ApproxDictionary {  // dictionary.hpp:111-120
  std::shared_ptr<const LinearOp> op;
  Vector atom_error_bounds;
  double operator_error_bound = 0.0;
  double relative_complexity = 1.0;
  Vector approx_atom_norms2;
  Vector exact_atom_norms2;
  bool is_exact() const { return operator_error_bound == 0.0; }
};

inline ApproxDictionary make_exact_approx(const DenseDictionary& dict) {  // dictionary.cpp:216-225
  ApproxDictionary d;
  d.atom_error_bounds = Vector::Zero(dict.cols());
  d.operator_error_bound = 0.0;
  d.relative_complexity = 1.0;
  d.approx_atom_norms2 = dict.atom_norms2();
  d.exact_atom_norms2 = d.approx_atom_norms2;
  d.op = std::make_shared<const DenseDictionary>(dict);
  return d;
}

struct ApproxSequence {  // dictionary.hpp:128-134
  std::vector<ApproxDictionary> dicts;
  int levels() const { return static_cast<int>(dicts.size()); }
  const ApproxDictionary& exact() const { return dicts.back(); }

  // Builds the device-side sequence (ApproxSequence::validate semantics).
  std::shared_ptr<fl1_seq> build() const {
    std::vector<std::shared_ptr<fl1_approx>> owned;
    std::vector<fl1_approx*> raw;
    for (const ApproxDictionary& d : dicts) {
      if (!d.op) throw std::invalid_argument("level without an operator");
      const Index k = d.op->cols();
      if (d.atom_error_bounds.size() != k || d.approx_atom_norms2.size() != k || d.exact_atom_norms2.size() != k)
        throw std::invalid_argument("invalid atom error bounds");
      fl1_approx* a = nullptr;
      detail::check(fl1_approx_create(d.op->handle(), d.atom_error_bounds.data(), d.operator_error_bound,
                                      d.relative_complexity, d.approx_atom_norms2.data(),
                                      d.exact_atom_norms2.data(), &a));
      owned.emplace_back(a, [](fl1_approx* p) { fl1_approx_destroy(p); });
      raw.push_back(a);
    }
    fl1_seq* s = nullptr;
    detail::check(fl1_seq_create(raw.data(), static_cast<int32_t>(raw.size()), &s));
    return std::shared_ptr<fl1_seq>(s, [](fl1_seq* p) { fl1_seq_destroy(p); });
  }
  void validate() const { build(); }  // throws std::invalid_argument on violation
};

// ------------------------------------------------------------------ engine API
enum class SolverKind { ista, fista };
enum class RuleKind { dynamic_safe, gap_safe };
enum class Variant { plain, screened, multi_dict };

struct SwitchConfig {  // fastl1.hpp:25-31
  double gamma_threshold = 0.5;
  int screening_interval = 1;
  double tolerance = 1e-6;
  std::uint64_t max_iterations = 1'000'000;
  bool precompute_aty = false;
  double rel_tolerance = 0.0;  // extension: stop at gap~ <= rel_tolerance * P(x) when > 0
};

struct TraceRow {  // fastl1.hpp:43-52
  std::uint64_t iter = 0;
  int dict_index = 0;
  int active_size = 0;
  double gap = -1.0;
  double gamma = -1.0;
  std::uint64_t flops_cum = 0;
  double wall_ms = 0.0;
  int x_nnz = 0;
};

struct SwitchEvent {  // fastl1.hpp:54-59
  std::uint64_t iter = 0;
  int from = 0;
  int to = 0;
  bool speed = false;
};

struct SolveResult {  // fastl1.hpp:61-71
  Vector x;
  bool converged = false;
  double final_gap = std::numeric_limits<double>::quiet_NaN();
  std::uint64_t iterations = 0;
  std::uint64_t total_flops = 0;
  std::vector<TraceRow> trace;
  std::vector<SwitchEvent> switches;
  std::vector<int> final_active;
  bool gap_warning = false;
};

struct SafeSphere {  // screening.hpp:14-18
  Vector center;
  double radius = 0.0;
  int norm_index = 2;
};
struct DualPoints {  // screening.hpp:60-66
  Vector theta_prime;
  Vector theta_tilde;
  double scale_prime = 0.0;
  double scale_tilde = 0.0;
};
struct ScreeningEvent {  // fastl1.hpp:74-83
  std::uint64_t iter = 0;
  int dict_index = 0;
  const SafeSphere* sphere = nullptr;
  const std::vector<int>* active_before = nullptr;
  const std::vector<int>* kept = nullptr;
  const DualPoints* duals = nullptr;
  const ApproxDictionary* dict = nullptr;
};
using ScreenObserver = std::function<void(const ScreeningEvent&)>;

struct RunOptions {  // fastl1.hpp:85-96
  SolverKind solver = SolverKind::fista;
  RuleKind rule = RuleKind::gap_safe;
  Variant variant = Variant::multi_dict;
  const Matrix* exact_gram = nullptr;  // K x K Gram of the exact dictionary: exact phase on G
  const std::vector<double>* full_lipschitz = nullptr;
  bool collect_trace = true;
  ScreenObserver observer;
  const Vector* x_init = nullptr;  // extension: warm start (length K)
};

namespace detail {
struct ObserverCtx {
  const ScreenObserver* fn;
  const ApproxSequence* seq;
};
inline void observer_trampoline(const fl1_screen_event* ev, void* user) {
  const ObserverCtx& c = *static_cast<const ObserverCtx*>(user);
  SafeSphere sphere;
  DualPoints duals;
  sphere.center.resize(ev->n);
  duals.theta_prime.resize(ev->n);
  duals.theta_tilde.resize(ev->n);
  for (Index i = 0; i < ev->n; ++i) {
    sphere.center(i) = ev->center[i];
    duals.theta_prime(i) = ev->theta_prime[i];
    duals.theta_tilde(i) = ev->theta_tilde[i];
  }
  sphere.radius = ev->radius;
  duals.scale_prime = ev->scale_prime;
  duals.scale_tilde = ev->scale_tilde;
  std::vector<int> before(ev->active_before, ev->active_before + ev->n_active_before);
  std::vector<int> kept(ev->kept, ev->kept + ev->n_kept);
  ScreeningEvent e;
  e.iter = ev->iter;
  e.dict_index = ev->dict_index;
  e.sphere = &sphere;
  e.active_before = &before;
  e.kept = &kept;
  e.duals = &duals;
  e.dict = &c.seq->dicts[static_cast<size_t>(ev->dict_index)];
  (*c.fn)(e);
}
// The Gram matrix uploaded once (sweeps pass the same matrix to every run_lasso).
inline std::shared_ptr<fl1_dict> gram_handle(const Matrix& g) {
  static std::mutex mu;
  static const double* key = nullptr;
  static Index key_rows = 0;
  static std::shared_ptr<fl1_dict> cached;
  std::lock_guard<std::mutex> lock(mu);
  if (key != g.data() || key_rows != g.rows() || !cached) {
    fl1_dict* d = nullptr;
    check(fl1_dict_dense(context(), g.data(), g.rows(), g.cols(), &d));
    cached.reset(d, [](fl1_dict* p) { fl1_dict_destroy(p); });
    key = g.data();
    key_rows = g.rows();
  }
  return cached;
}
}  // namespace detail

// run_lasso (fastl1.cpp:753-758): the whole solve runs on the GPU.
inline SolveResult run_lasso(const ApproxSequence& seq, const Vector& y, double lambda, const SwitchConfig& cfg,
                             const RunOptions& opts) {
  if (seq.dicts.empty()) throw std::invalid_argument("empty approximation sequence");
  if (y.size() != seq.exact().op->rows()) throw std::invalid_argument("y has wrong length");
  std::shared_ptr<fl1_seq> s = seq.build();
  fl1_switch_config c{cfg.gamma_threshold, cfg.screening_interval, cfg.tolerance,
                      cfg.max_iterations, cfg.precompute_aty ? 1 : 0, cfg.rel_tolerance};
  fl1_run_options o{};
  o.solver = opts.solver == SolverKind::fista ? FL1_FISTA : FL1_ISTA;
  o.rule = opts.rule == RuleKind::gap_safe ? FL1_RULE_GAP : FL1_RULE_DYNAMIC;
  o.variant = opts.variant == Variant::plain ? FL1_PLAIN
              : opts.variant == Variant::screened ? FL1_SCREENED
                                                  : FL1_MULTI_DICT;
  if (opts.full_lipschitz) {
    o.full_lipschitz = opts.full_lipschitz->data();
    o.n_full_lipschitz = static_cast<int32_t>(opts.full_lipschitz->size());
  }
  o.collect_trace = opts.collect_trace ? 1 : 0;
  detail::ObserverCtx octx{&opts.observer, &seq};
  if (opts.observer) {
    o.observer = &detail::observer_trampoline;
    o.observer_user = &octx;
  }
  if (opts.x_init) {
    if (opts.x_init->size() != seq.exact().op->cols()) throw std::invalid_argument("x_init has wrong length");
    o.x_init = opts.x_init->data();
  }
  std::shared_ptr<fl1_dict> gram;
  if (opts.exact_gram) {
    if (opts.exact_gram->rows() != seq.exact().op->cols() || opts.exact_gram->cols() != seq.exact().op->cols())
      throw std::invalid_argument("exact_gram must be K x K");
    gram = detail::gram_handle(*opts.exact_gram);
    o.exact_gram = gram.get();
  }
  fl1_result* r = nullptr;
  detail::check(fl1_solve(s.get(), y.data(), lambda, &c, &o, &r));
  std::unique_ptr<fl1_result, void (*)(fl1_result*)> guard(r, &fl1_result_free);
  fl1_result_info info{};
  detail::check(fl1_result_info_get(r, &info));
  SolveResult out;
  out.x.resize(info.k);
  detail::check(fl1_result_x(r, out.x.data()));
  out.converged = info.converged != 0;
  out.final_gap = info.final_gap;
  out.iterations = info.iterations;
  out.total_flops = info.total_flops;
  out.gap_warning = info.gap_warning != 0;
  std::vector<fl1_trace_row> rows(static_cast<size_t>(info.n_trace));
  if (!rows.empty()) detail::check(fl1_result_trace(r, rows.data()));
  for (const fl1_trace_row& t : rows)
    out.trace.push_back({t.iter, t.dict_index, t.active_size, t.gap, t.gamma, t.flops_cum, t.wall_ms, t.x_nnz});
  std::vector<fl1_switch_event> sw(static_cast<size_t>(info.n_switches));
  if (!sw.empty()) detail::check(fl1_result_switches(r, sw.data()));
  for (const fl1_switch_event& e : sw) out.switches.push_back({e.iter, e.from, e.to, e.speed != 0});
  std::vector<int32_t> fa(static_cast<size_t>(info.n_final_active));
  if (!fa.empty()) detail::check(fl1_result_final_active(r, fa.data()));
  out.final_active.assign(fa.begin(), fa.end());
  return out;
}

inline SolveResult fastl1_solve(const ApproxSequence& seq, const Vector& y, double lambda, const SwitchConfig& cfg,
                                SolverKind solver, RuleKind rule) {  // fastl1.hpp:104-111
  RunOptions opts;
  opts.solver = solver;
  opts.rule = rule;
  opts.variant = Variant::multi_dict;
  return run_lasso(seq, y, lambda, cfg, opts);
}

// ------------------------------------------------------------------ primitives
inline double soft_threshold(double z, double u) { return fl1_soft_threshold(z, u); }
inline double gap_ratio(double gt, double gp) { return fl1_gap_ratio(gt, gp); }
inline int switch_dictionary(int i, int last, double gamma, double thr, std::int64_t la, double rc,
                             std::int64_t total) {
  return fl1_switch_dictionary(i, last, gamma, thr, la, rc, total);
}
inline std::uint64_t flops_plain(std::uint64_t k, std::uint64_t n, std::uint64_t z) { return fl1_flops_plain(k, n, z); }
inline std::uint64_t flops_screened(std::uint64_t a, std::uint64_t n, std::uint64_t z) {
  return fl1_flops_screened(a, n, z);
}
inline std::uint64_t flops_stable(std::uint64_t mv, std::uint64_t n, std::uint64_t a, std::uint64_t z) {
  return fl1_flops_stable(mv, n, a, z);
}
inline double stable_gap_delta(double rn, double e, double x1) { return fl1_stable_gap_delta(rn, e, x1); }
inline double sphere_test(double d, double an, double r) { return fl1_sphere_test(d, an, r); }
inline double stable_zone_test(double d, double eps, double cn, double en, double r) {
  return fl1_stable_zone_test(d, eps, cn, en, r);
}
inline double stable_ball_test(double d, double eps, double cn, double an, double r) {
  return fl1_stable_ball_test(d, eps, cn, an, r);
}
inline double lambda_max(const LinearOp& dict, const Vector& y) {  // screening.cpp:9-11
  double out = 0.0;
  detail::check(fl1_lambda_max(dict.handle(), y.data(), &out));
  return out;
}
inline double lipschitz_bound(const LinearOp& op) {  // solver.cpp:108-114 (cold start)
  double out = 0.0;
  detail::check(fl1_lipschitz_bound(op.handle(), &out));
  return out;
}
inline std::uint64_t recompute_flops(const std::vector<TraceRow>& trace, const ApproxSequence& seq, Variant variant,
                                     Index n, Index k, bool* rows_match = nullptr) {
  std::vector<fl1_trace_row> rows;
  for (const TraceRow& t : trace) {
    fl1_trace_row r{};
    r.iter = t.iter;
    r.dict_index = t.dict_index;
    r.active_size = t.active_size;
    r.gap = t.gap;
    r.gamma = t.gamma;
    r.flops_cum = t.flops_cum;
    r.wall_ms = t.wall_ms;
    r.x_nnz = t.x_nnz;
    rows.push_back(r);
  }
  std::shared_ptr<fl1_seq> s = seq.build();
  int32_t m = 0;
  const int32_t v = variant == Variant::plain ? FL1_PLAIN : variant == Variant::screened ? FL1_SCREENED : FL1_MULTI_DICT;
  const std::uint64_t tot = fl1_recompute_flops(rows.data(), static_cast<int64_t>(rows.size()), s.get(), v, n, k, &m);
  if (rows_match) *rows_match = m != 0;
  return tot;
}

}  // namespace fastl1
