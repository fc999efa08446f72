// C++ drop-in check: the reference's own call pattern (tests/test_fastl1.cpp,
// bench.cpp:207-240) compiled against include/fl1/fastl1.hpp and run on the GPU.
#include <cmath>
#include <cstdio>
#include <random>
#include <stdexcept>

#include "fl1/fastl1.hpp"

using namespace fastl1;

#define CHECK(cond)                                                   \
  do {                                                                \
    if (!(cond)) {                                                    \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      return 1;                                                       \
    }                                                                 \
  } while (0)

int main() {
  // KATs (test_fastl1.cpp:41-58, test_solver.cpp:11-16)
  CHECK(soft_threshold(-2.0, 0.5) == -1.5);
  CHECK(gap_ratio(1e-9, 1e-16) == 0.0);
  CHECK(switch_dictionary(0, 4, 0.9, 0.2, 100, 0.15, 10000) == 4);
  CHECK(flops_screened(10000, 2500, 0) == 10000ull * 2500 + 6 * 10000 + 5 * 2500);

  // dense diagonal KAT (test_dictionary.cpp:25-37)
  Matrix diag = Matrix::Zero(2, 2);
  diag(0, 0) = 1.0;
  diag(1, 1) = 2.0;
  DenseDictionary dd(diag);
  Vector v(2);
  v(0) = 3.0;
  v(1) = 1.0;
  const Vector av = dd.apply(v);
  CHECK(av(0) == 3.0 && av(1) == 2.0);

  // a random column-normalised instance, solved like execute_run does
  const Index n = 200, k = 600;
  std::mt19937_64 rng(7);
  std::normal_distribution<double> g(0.0, 1.0);
  Matrix a(n, k);
  for (Index j = 0; j < k; ++j) {
    double s = 0.0;
    for (Index i = 0; i < n; ++i) {
      a(i, j) = g(rng);
      s += a(i, j) * a(i, j);
    }
    for (Index i = 0; i < n; ++i) a(i, j) /= std::sqrt(s);
  }
  Vector x0 = Vector::Zero(k);
  for (int s = 0; s < 8; ++s) x0(static_cast<Index>(rng() % k)) = g(rng);
  DenseDictionary dict(a);
  Vector y = dict.apply(x0);
  ApproxSequence seq;
  seq.dicts.push_back(make_exact_approx(dict));
  const double lmax = lambda_max(*seq.exact().op, y);
  const std::vector<double> full_l = {lipschitz_bound(*seq.exact().op)};
  SwitchConfig cfg;
  cfg.screening_interval = 10;
  cfg.tolerance = 1e-9;
  RunOptions opts;
  opts.variant = Variant::screened;
  opts.full_lipschitz = &full_l;
  int screens = 0;
  opts.observer = [&](const ScreeningEvent& ev) {
    ++screens;
    if (ev.kept->size() > ev.active_before->size()) throw std::runtime_error("kept grew");
  };
  SolveResult res = run_lasso(seq, y, 0.2 * lmax, cfg, opts);
  CHECK(res.converged);
  CHECK(res.final_gap <= 1e-9);
  CHECK(screens > 0);
  CHECK(!res.trace.empty() && res.trace.back().flops_cum == res.total_flops);
  bool rows_match = false;
  CHECK(recompute_flops(res.trace, seq, Variant::screened, n, k, &rows_match) == res.total_flops && rows_match);

  // Gram-backed exact phase (fastl1.cpp:278-394): same trajectory as the direct products
  Matrix gram(k, k);
  for (Index j = 0; j < k; ++j)
    for (Index i = 0; i < k; ++i) {
      double acc = 0.0;
      for (Index r = 0; r < n; ++r) acc += a(r, i) * a(r, j);
      gram(i, j) = acc;
    }
  RunOptions gopts = opts;
  gopts.observer = nullptr;  // the reference ignores the Gram while an observer is attached
  gopts.exact_gram = &gram;
  const SolveResult gres = run_lasso(seq, y, 0.2 * lmax, cfg, gopts);
  CHECK(gres.converged && gres.iterations == res.iterations && gres.total_flops == res.total_flops);
  double xdiff = 0.0;
  for (Index j = 0; j < k; ++j) xdiff = std::max(xdiff, std::abs(gres.x(j) - res.x(j)));
  CHECK(xdiff <= 1e-9);

  // invalid arguments surface as std::invalid_argument (fastl1.cpp:268-273)
  bool threw = false;
  try {
    run_lasso(seq, y, -1.0, cfg, opts);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);

  // DenseDictionary file formats (dictionary.cpp:76-135): exact round trips
  dict.save_blob("/tmp/fl1_shim_dict.blob");
  dict.save_csv("/tmp/fl1_shim_dict.csv");
  const DenseDictionary from_blob = DenseDictionary::load_blob("/tmp/fl1_shim_dict.blob");
  const DenseDictionary from_csv = DenseDictionary::load_csv("/tmp/fl1_shim_dict.csv");
  bool same = from_blob.rows() == n && from_blob.cols() == k && from_csv.rows() == n && from_csv.cols() == k;
  for (Index j = 0; same && j < k; ++j)
    for (Index i = 0; i < n; ++i)
      same = same && from_blob.entries()(i, j) == a(i, j) && from_csv.entries()(i, j) == a(i, j);
  CHECK(same);
  threw = false;
  try {
    DenseDictionary::load_blob("/tmp/fl1_shim_missing.blob");
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);
  std::printf("shim ok: %llu iterations, gap %.3e, %d screening events\n",
              static_cast<unsigned long long>(res.iterations), res.final_gap, screens);
  return 0;
}
