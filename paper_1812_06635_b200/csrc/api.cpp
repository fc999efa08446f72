// api.cpp — host side of libfl1cuda.so: the C-ABI declared in include/fl1cuda.h.
//
// Owns device memory for dictionaries (HBM-resident, immutable, shareable),
// per-solve workspaces (cached per context), the launch loop around the
// persistent engine kernel, and the marshalling of SolveResult
// (fastl1.hpp:61-71). There is no CPU compute path: every product with a
// dictionary runs on the GPU; the host only validates arguments (with the
// reference's messages) and moves bytes.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <atomic>
#include <map>
#include <mutex>
#include <tuple>
#include <thread>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "engine.cuh"

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda): a 2D
// fp64 tensor of dims (d0, d1), row pitch d0 doubles, box (b0, b1), no swizzle,
// out-of-bounds elements zero-filled.
static cudaError_t encode_tensor_map_2d(CUtensorMap* tm, const double* base, int64_t d0, int64_t d1, uint32_t b0,
                                        uint32_t b1) {
  using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Encode fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<Encode>(f);
  }();
  if (!fn) return cudaErrorNotSupported;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(d0), static_cast<cuuint64_t>(d1)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(d0) * sizeof(double)};
  const cuuint32_t box[2] = {b0, b1};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

namespace fl1 {
size_t engine_smem_bytes(int64_t ld, int64_t sukro_m);
int64_t engine_scratch_len(int64_t ld, int64_t sukro_m);
int engine_bulk_stages(int64_t ld);
cudaError_t engine_configure(int64_t ld, int64_t sukro_m, int device, int* grid_out);
cudaError_t engine_launch(const EngineParams& p, int64_t sukro_m, cudaStream_t stream);
// the engine instance with the single-read power steps (engine.cu, FL1_FUSED_VARIANT)
cudaError_t engine_configure_fp(int64_t ld, int64_t sukro_m, int device, int* grid_out);
cudaError_t engine_launch_fp(const EngineParams& p, int64_t sukro_m, cudaStream_t stream);
size_t prefix_smem_bytes(int64_t ld, int64_t batch);
cudaError_t prefix_launch(const PrefixParams& p, int device, cudaStream_t stream);
cudaError_t trace_pack_launch(const fl1_trace_row* src, int64_t cap, const int64_t* off, int32_t batch,
                              fl1_trace_row* dst, cudaStream_t stream);
int prefix_split_max();
cudaError_t gram_launch(const double* a, int64_t ld, int64_t k, double* g, int64_t ldg, int device,
                        cudaStream_t stream);
cudaError_t colnorm_launch(const double* g, int64_t k, int64_t ldg, double* out, cudaStream_t stream);
cudaError_t dense_norms_launch(const double* a, int64_t n, int64_t ld, int64_t k, double* out, cudaStream_t stream);
cudaError_t sukro_norms_launch(const double* left, const double* right, const double* scale, int nterms, int64_t m,
                               int64_t q, double* out, cudaStream_t stream);
int64_t prefix_max_atoms();
int64_t prefix_part_elems(int grid);
bool prefix_fits(int64_t ld, int64_t batch, int device);
int prefix_stream_k_max_grid();
constexpr int kStepLogW = 10;  // batched.cu kLogW
cudaError_t gemm_tn_launch(const double* X, int64_t ldx, int64_t nx, const double* Y, int64_t ldy, int64_t ny,
                           int64_t kdim, double* C, int64_t ldc, double* work, size_t work_elems, int device,
                           cudaStream_t stream);
cudaError_t rearrange_launch(const double* a, int64_t lda, int64_t m, int64_t q, double* R, double* Rt, int64_t ldr,
                             cudaStream_t stream);
cudaError_t householder_qr_launch(double* W, int64_t M, int p, int64_t ld, double* Q, int64_t ldq, double* Rf,
                                  cudaStream_t stream);
cudaError_t jacobi_svd_launch(const double* Rf, int p, double* S, double* W, double* V, cudaStream_t stream);
cudaError_t small_gemm_launch(const double* A, int64_t lda, int64_t M, int p, const double* B, const double* S, int r,
                              double* out, int64_t ldo, cudaStream_t stream);
cudaError_t residual_norms_launch(const double* a, int64_t lda, int64_t m, int64_t q, int T, const double* left,
                                  const double* right, int64_t ldt, const int* ranks, int n_ranks, double* eps,
                                  double* app, cudaStream_t stream);
int sukro_max_probe();
int sukro_max_snapshots();
cudaError_t engine_cluster_capacity(int64_t ld, int64_t sukro_m, int csize, int* n_clusters);
cudaError_t engine_launch_clusters(const EngineParams& p0, int n_clusters, int csize, int64_t sukro_m,
                                   cudaStream_t stream);
cudaError_t screen_kernel_launch(int64_t n, const double* dots, const double* eps, const double* en,
                                 const double* an, double cn, double r, int8_t* keep, int8_t* look,
                                 cudaStream_t stream);
}  // namespace fl1

using fl1::DevLevel;
using fl1::EngineParams;
using fl1::EngineState;

namespace {

thread_local std::string g_err;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return FL1_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return FL1_EINVAL;
  } catch (const CudaError& e) {
    g_err = e.what();
    return FL1_ECUDA;
  } catch (const std::bad_alloc&) {
    g_err = "out of memory";
    return FL1_ENOMEM;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return FL1_EUNSUPPORTED;
  } catch (const std::exception& e) {
    g_err = e.what();
    return FL1_ERUNTIME;
  }
}

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  explicit DevBuf(size_t b) : bytes(b) {
    if (b) ck(cudaMalloc(&p, b), "cudaMalloc");
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// batched solves: CTAs per signal engine. 1 measured best on c5 (the per-signal tails
// after the lockstep hand-off run on small preserved sets: 148 one-CTA engines beat 74
// two-CTA clusters, 56.6 vs 57.0 ms; 4 CTAs: 62.2 ms)
constexpr int kDefaultClusterSize = 1;

// leading dimension of dense columns / vectors: 128-byte aligned (FL1_LD_ALIGN doubles,
// default 16: every column starts on an L2 line; c1 -1.5%, no change where N % 16 == 0)
int64_t even_ld(int64_t n) {
  static const int64_t a = [] {
    const char* e = std::getenv("FL1_LD_ALIGN");
    const int64_t v = e ? std::atoll(e) : 16;
    // at most one bulk unit: the power-iteration ring's last-unit copy moves (ld - ih * kUnit)
    // doubles into a kUnit-double stage (engine.cu dense_adjoint)
    return v >= 2 && (v & (v - 1)) == 0 && v <= fl1::kUnit ? v : 16;
  }();
  return (n + a - 1) / a * a;
}

}  // namespace

// ---------------------------------------------------------------- handles
struct Workspace {
  int64_t n = 0, k = 0, ld = 0;
  int grid_cap = 0;  // 0: one CTA per SM; else the sub-grid of a concurrent batched solve
  bool fused_engine = false;  // launches go to the engine instance with the single-read power steps
  int64_t sk_elems = 0;  // SuKro scratch capacity (nterms * m * q)
  int64_t sk_m = 0;
  int grid = 0;
  int64_t units = 1;
  int64_t trace_cap = 0;
  std::unique_ptr<DevBuf> mem;
  std::unique_ptr<DevBuf> cbuf;  // FL1_COMPACT copies (allocated on first use)
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  EngineParams base{};  // pointers filled
  // pinned host staging: state, y, final (idx, x), switch events, trace rows
  void* pinned = nullptr;
  EngineState* h_st = nullptr;
  double* h_y = nullptr;
  int32_t* h_idx = nullptr;
  double* h_x = nullptr;
  fl1_switch_event* h_sw = nullptr;
  fl1_trace_row* h_trace = nullptr;
  int64_t h_trace_cap = 0;
  ~Workspace() {
    if (pinned) cudaFreeHost(pinned);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (stream) cudaStreamDestroy(stream);
  }
};

struct fl1_ctx {
  int device = 0;
  int sms = 0;
  int64_t l2 = 0, hbm = 0;
  std::mutex mu;
  std::vector<std::unique_ptr<Workspace>> pool;
  std::unique_ptr<DevBuf> gauss;  // cold-start vector (solver.cpp:80-82)
  int64_t gauss_len = 0;

  void bind() const { ck(cudaSetDevice(device), "cudaSetDevice"); }

  // first `len` draws of mt19937_64(0x11b5c417) / normal_distribution, resident in HBM
  const double* gauss0(int64_t len) {
    std::lock_guard<std::mutex> g(mu);
    if (gauss_len < len) {
      std::mt19937_64 rng(0x11b5c417ULL);
      std::normal_distribution<double> nd(0.0, 1.0);
      std::vector<double> h(static_cast<size_t>(len));
      for (auto& e : h) e = nd(rng);
      auto buf = std::make_unique<DevBuf>(h.size() * sizeof(double));
      ck(cudaMemcpy(buf->p, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice), "upload gauss0");
      gauss = std::move(buf);
      gauss_len = len;
    }
    return gauss->as<double>();
  }

  std::unique_ptr<Workspace> acquire(int64_t n, int64_t k, int64_t trace_cap, int64_t sk_elems, int64_t sk_m,
                                     int grid_cap = 0);
  // device scratch of the batched entry, kept between calls (one batched call at a time)
  std::mutex batch_mu;
  std::unique_ptr<DevBuf> batch_buf[3];
  cudaStream_t batch_stream = nullptr;
  cudaEvent_t batch_ev[3] = {nullptr, nullptr, nullptr};
  void* batch_pinned = nullptr;
  size_t batch_pinned_bytes = 0;
  void* trace_pinned = nullptr;  // packed trace rows of a batched call
  size_t trace_pinned_bytes = 0;
  char* pinned_traces(size_t bytes) {
    if (trace_pinned_bytes < bytes) {
      if (trace_pinned) cudaFreeHost(trace_pinned);
      trace_pinned = nullptr;
      trace_pinned_bytes = 0;
      ck(cudaHostAlloc(&trace_pinned, bytes + bytes / 8, cudaHostAllocDefault), "cudaHostAlloc");
      trace_pinned_bytes = bytes + bytes / 8;
    }
    return static_cast<char*>(trace_pinned);
  }
  std::map<std::tuple<int64_t, int64_t, int>, std::pair<int, int>> cluster_cfg;  // (ld, sk_m, csize) -> (grid, clusters)
  char* pinned_scratch(size_t bytes) {
    if (batch_pinned_bytes < bytes) {
      if (batch_pinned) cudaFreeHost(batch_pinned);
      batch_pinned = nullptr;
      batch_pinned_bytes = 0;
      ck(cudaHostAlloc(&batch_pinned, bytes + bytes / 8, cudaHostAllocDefault), "cudaHostAlloc");
      batch_pinned_bytes = bytes + bytes / 8;
    }
    return static_cast<char*>(batch_pinned);
  }
  void batch_objects() {
    if (!batch_stream) ck(cudaStreamCreateWithFlags(&batch_stream, cudaStreamNonBlocking), "stream");
    for (auto& e : batch_ev)
      if (!e) ck(cudaEventCreate(&e), "event");
  }
  ~fl1_ctx() {
    if (batch_pinned) cudaFreeHost(batch_pinned);
    if (trace_pinned) cudaFreeHost(trace_pinned);
    for (auto e : batch_ev)
      if (e) cudaEventDestroy(e);
    if (batch_stream) cudaStreamDestroy(batch_stream);
  }
  DevBuf& batch_scratch(int slot, size_t bytes) {
    auto& b = batch_buf[slot];
    if (!b || b->bytes < bytes) {
      b.reset();
      b = std::make_unique<DevBuf>(bytes + bytes / 8);
    }
    return *b;
  }
  void release(std::unique_ptr<Workspace> w) {
    std::lock_guard<std::mutex> g(mu);
    if (pool.size() < 64) pool.push_back(std::move(w));
  }
};

struct DictImpl {
  fl1_ctx* ctx = nullptr;
  int kind = fl1::kDense;
  int64_t n = 0, k = 0, ld = 0;
  int64_t m = 0, q = 0;
  int nterms = 0;
  std::unique_ptr<DevBuf> a, left, right, col_scale;
  std::vector<double> h_left, h_right, h_scale;  // SuKro factors (small) kept for column()
  std::vector<double> norms;                     // atom_norms2
  uint64_t matvec_flops() const {
    if (kind == fl1::kDense) return static_cast<uint64_t>(n) * static_cast<uint64_t>(k);
    return static_cast<uint64_t>(nterms) * (static_cast<uint64_t>(m) * static_cast<uint64_t>(k) +
                                            static_cast<uint64_t>(q) * static_cast<uint64_t>(n));
  }
};
struct fl1_dict {
  std::shared_ptr<DictImpl> d;
};

struct ApproxImpl {
  std::shared_ptr<DictImpl> dict;
  std::vector<double> eps, an, en;
  double op_err = 0.0, rc = 1.0;
  std::unique_ptr<DevBuf> d_eps, d_an, d_en;
  bool is_exact() const { return op_err == 0.0; }
};
struct fl1_approx {
  std::shared_ptr<ApproxImpl> a;
};

struct fl1_seq {
  std::vector<std::shared_ptr<ApproxImpl>> lv;
  void validate() const {  // ApproxSequence::validate (dictionary.cpp:227-251)
    if (lv.empty()) throw std::invalid_argument("empty approximation sequence");
    const int64_t k = lv.front()->dict->k;
    for (size_t i = 0; i < lv.size(); ++i) {
      const ApproxImpl& d = *lv[i];
      if (d.dict->k != k) throw std::invalid_argument("sequence has mismatched atom counts");
      bool bad = static_cast<int64_t>(d.eps.size()) != k;
      if (!bad)
        for (double e : d.eps) bad = bad || e < 0;
      if (bad) throw std::invalid_argument("invalid atom error bounds");
      if (d.rc <= 0.0 || d.rc > 1.0) throw std::invalid_argument("relative complexity out of (0, 1]");
      if (i > 0) {
        const ApproxImpl& p = *lv[i - 1];
        if (d.rc <= p.rc) throw std::invalid_argument("relative complexity must strictly increase");
        for (int64_t j = 0; j < k; ++j)
          if (d.eps[static_cast<size_t>(j)] > p.eps[static_cast<size_t>(j)] + 1e-15)
            throw std::invalid_argument("error bounds must be non-increasing along the sequence");
      }
    }
    if (!lv.back()->is_exact() || lv.back()->rc != 1.0)
      throw std::invalid_argument("sequence must end with the exact dictionary");
  }
};

struct fl1_result {
  int64_t k = 0;
  std::vector<double> xv;  // x at final_active (x is zero elsewhere; expanded by the accessors)
  bool converged = false;
  double final_gap = std::numeric_limits<double>::quiet_NaN();
  uint64_t iterations = 0;
  uint64_t total_flops = 0;
  std::vector<fl1_trace_row> trace;
  std::vector<fl1_switch_event> switches;
  std::vector<int32_t> final_active;
  bool gap_warning = false;
  double device_ms = 0.0, setup_ms = 0.0, batch_ms = -1.0;
  int64_t launches = 0, power_steps = 0;
  double prof[14] = {0};
  int64_t h2d = 0, d2h = 0;
};

// ---------------------------------------------------------------- workspace
namespace {

struct Carver {
  char* base;
  size_t off = 0;
  template <class T>
  T* take(int64_t count) {
    off = (off + 255) / 256 * 256;
    T* r = reinterpret_cast<T*>(base + off);
    off += static_cast<size_t>(count) * sizeof(T);
    return r;
  }
};

size_t carve(EngineParams& p, char* base, int64_t n, int64_t k, int64_t ld, int grid, int64_t units,
             int64_t trace_cap, int64_t sk_m) {
  (void)n;
  Carver c{base};
  const int64_t kk = std::max<int64_t>(k, 1);
  const int64_t vec = std::max(ld, kk);
  p.y = c.take<double>(ld);
  p.x_init = c.take<double>(vec);
  p.U = c.take<double>(ld);
  p.V = c.take<double>(ld);
  p.rho = c.take<double>(ld);
  p.rho_obs = c.take<double>(ld);
  // apply partials: at most one chunk per CTA, of length ld (u = A x) or, in the
  // Gram-backed exact phase, of the Gram's leading dimension (gx = G x)
  const int64_t chunks = std::max<int64_t>(grid, 8);
  const int64_t plen = std::max(ld, even_ld(kk));
  p.up = c.take<double>(chunks * plen);
  p.dvp = c.take<double>(chunks * plen);
  p.pup = c.take<double>(chunks * ld);
  p.GX = c.take<double>(kk);
  p.GV = c.take<double>(kk);
  p.ATYF = c.take<double>(kk);
  p.ident = c.take<int32_t>(kk);
  p.vec_out = c.take<double>(vec);
  p.corr = c.take<double>(kk);
  p.xnew = c.take<double>(kk);
  p.corr_y = c.take<double>(kk);
  p.part = c.take<double>(kk * units);
  p.cnt = c.take<int32_t>(kk);
  p.nzv = c.take<double>(kk);
  p.nzj = c.take<int32_t>(kk);
  p.fxv = c.take<double>(kk);
  p.fxj = c.take<int32_t>(kk);
  p.lcnt = c.take<int32_t>(2 * static_cast<int64_t>(grid));
  {
    const char* e = std::getenv("FL1_LIST_APPLY");
    p.list_apply = e ? std::atoi(e) : 1;
    const char* o = std::getenv("FL1_POWER_ONCHIP");
    p.power_onchip = o ? std::atoi(o) : 1;
    const char* ep = std::getenv("FL1_EARLY_PROX");
    p.early_prox = ep ? std::atoi(ep) : 1;
    const char* cs = std::getenv("FL1_COLSPLIT");
    p.colsplit_elems = cs ? std::atoll(cs) : (2ll << 20);
    // single-read power steps for preserved sets beyond L2 (HBM-bound: half the bytes per step)
    const char* fp = std::getenv("FL1_FUSED_POWER_MB");
    p.fused_power_bytes = (fp ? std::atoll(fp) : 192) << 20;
    const char* pf = std::getenv("FL1_FUSED_PREFETCH");
    p.fused_prefetch = pf ? std::atoi(pf) : 1;
  }
  p.pv = c.take<double>(kk);
  p.pw = c.take<double>(kk);
  p.PU = c.take<double>(ld);
  p.sk_z = sk_m > 0 ? c.take<double>(kk) : nullptr;
  p.scratch_len = fl1::engine_scratch_len(ld, sk_m);
  p.bulk_stages = fl1::engine_bulk_stages(ld);
  p.bred = c.take<double>(static_cast<int64_t>(grid) * fl1::kBred);
  for (int b = 0; b < 2; ++b) {
    fl1::Bank& bk = p.bank[b];
    bk.idx = c.take<int32_t>(kk);
    bk.x = c.take<double>(kk);
    bk.xp = c.take<double>(kk);
    bk.eps = c.take<double>(kk);
    bk.en = c.take<double>(kk);
    bk.an = c.take<double>(kk);
    bk.aty = c.take<double>(kk);
    bk.atye = c.take<double>(kk);
    bk.lead = c.take<double>(kk);
    bk.keep = c.take<int8_t>(kk);
    p.bcix[b] = c.take<int32_t>(kk);
  }
  p.trace = c.take<fl1_trace_row>(std::max<int64_t>(trace_cap, 1));
  p.sw = c.take<fl1_switch_event>(fl1::kMaxLevels);
  p.st = c.take<EngineState>(1);
  p.timeline = nullptr;
  return c.off + 256;
}

}  // namespace

std::unique_ptr<Workspace> fl1_ctx::acquire(int64_t n, int64_t k, int64_t trace_cap, int64_t sk_elems,
                                            int64_t sk_m, int grid_cap) {
  const int64_t ld = even_ld(n);
  {
    std::lock_guard<std::mutex> g(mu);
    for (size_t i = 0; i < pool.size(); ++i) {
      Workspace& w = *pool[i];
      if (w.n == n && w.k == k && w.trace_cap >= trace_cap && w.sk_elems >= sk_elems && w.sk_m >= sk_m &&
          w.grid_cap == grid_cap) {
        auto r = std::move(pool[i]);
        pool.erase(pool.begin() + static_cast<long>(i));
        return r;
      }
    }
  }
  auto w = std::make_unique<Workspace>();
  w->n = n;
  w->k = k;
  w->ld = ld;
  w->units = (n + fl1::kUnit - 1) / fl1::kUnit;
  w->trace_cap = trace_cap;
  w->sk_elems = sk_elems;
  w->sk_m = sk_m;
  {
    const cudaError_t e = fl1::engine_configure(ld, sk_m, device, &w->grid);
    if (e == cudaErrorInvalidConfiguration)
      throw std::logic_error("signal length too large for the shared-memory resident residual");
    ck(e, "engine_configure");
    if (grid_cap > 0 && grid_cap < w->grid) w->grid = grid_cap;  // sub-grid for concurrent solves
    w->grid_cap = grid_cap;
  }
  EngineParams p{};
  const size_t bytes = carve(p, nullptr, n, k, ld, w->grid, w->units, trace_cap, sk_m);
  w->mem = std::make_unique<DevBuf>(bytes);
  ck(cudaMemset(w->mem->p, 0, bytes), "workspace memset");
  carve(p, w->mem->as<char>(), n, k, ld, w->grid, w->units, trace_cap, sk_m);
  p.grid = w->grid;
  p.n = n;
  p.k = k;
  p.ld = ld;
  p.trace_cap = trace_cap;
  w->base = p;
  // dictionaries the single-read power steps apply to (tall columns, beyond L2) run on the engine
  // instance that contains them; every other workspace on the default instance
  if (p.fused_power_bytes > 0 && grid_cap == 0 && n > 8 * fl1::kUnit && n <= 16 * fl1::kUnit && p.bulk_stages == 2 &&
      8 * ld * k >= p.fused_power_bytes) {
    int g2 = 0;
    if (fl1::engine_configure_fp(ld, sk_m, device, &g2) == cudaSuccess && g2 >= w->grid) w->fused_engine = true;
  }
  ck(cudaStreamCreateWithFlags(&w->stream, cudaStreamNonBlocking), "stream");
  {
    w->h_trace_cap = std::min<int64_t>(trace_cap, 1 << 16);
    auto up = [](size_t x) { return (x + 255) / 256 * 256; };
    const size_t kk = static_cast<size_t>(std::max<int64_t>(k, 1));
    const size_t bytes = up(sizeof(EngineState)) + up(sizeof(double) * static_cast<size_t>(ld)) +
                         up(sizeof(int32_t) * kk) + up(sizeof(double) * kk) +
                         up(sizeof(fl1_switch_event) * fl1::kMaxLevels) +
                         up(sizeof(fl1_trace_row) * static_cast<size_t>(std::max<int64_t>(w->h_trace_cap, 1)));
    ck(cudaHostAlloc(&w->pinned, bytes, cudaHostAllocDefault), "cudaHostAlloc");
    char* c = static_cast<char*>(w->pinned);
    w->h_st = reinterpret_cast<EngineState*>(c);
    c += up(sizeof(EngineState));
    w->h_y = reinterpret_cast<double*>(c);
    c += up(sizeof(double) * static_cast<size_t>(ld));
    w->h_idx = reinterpret_cast<int32_t*>(c);
    c += up(sizeof(int32_t) * kk);
    w->h_x = reinterpret_cast<double*>(c);
    c += up(sizeof(double) * kk);
    w->h_sw = reinterpret_cast<fl1_switch_event*>(c);
    c += up(sizeof(fl1_switch_event) * fl1::kMaxLevels);
    w->h_trace = reinterpret_cast<fl1_trace_row*>(c);
  }
  ck(cudaEventCreate(&w->ev0), "event");
  ck(cudaEventCreate(&w->ev1), "event");
  return w;
}

namespace {

struct WsLease {
  fl1_ctx* ctx;
  std::unique_ptr<Workspace> w;
  WsLease(fl1_ctx* c, int64_t n, int64_t k, int64_t cap, int64_t sk_elems, int64_t sk_m, int grid_cap = 0)
      : ctx(c), w(c->acquire(n, k, cap, sk_elems, sk_m, grid_cap)) {}
  ~WsLease() {
    if (w) ctx->release(std::move(w));
  }
};

DevLevel make_level(const ApproxImpl* a) {
  DevLevel lv{};
  const DictImpl& d = *a->dict;
  lv.kind = d.kind;
  lv.nterms = d.nterms;
  lv.m = d.m;
  lv.q = d.q;
  lv.a = d.a ? d.a->as<double>() : nullptr;
  lv.left = d.left ? d.left->as<double>() : nullptr;
  lv.right = d.right ? d.right->as<double>() : nullptr;
  lv.col_scale = d.col_scale ? d.col_scale->as<double>() : nullptr;
  lv.eps = a->d_eps->as<double>();
  lv.an = a->d_an->as<double>();
  lv.en = a->d_en->as<double>();
  lv.op_err = a->op_err;
  lv.rc = a->rc;
  lv.matvec_flops = d.matvec_flops();
  return lv;
}

// A level over a bare dictionary (utility modes): eps = 0 metadata not needed.
DevLevel make_dict_level(const DictImpl& d) {
  DevLevel lv{};
  lv.kind = d.kind;
  lv.nterms = d.nterms;
  lv.m = d.m;
  lv.q = d.q;
  lv.a = d.a ? d.a->as<double>() : nullptr;
  lv.left = d.left ? d.left->as<double>() : nullptr;
  lv.right = d.right ? d.right->as<double>() : nullptr;
  lv.col_scale = d.col_scale ? d.col_scale->as<double>() : nullptr;
  lv.matvec_flops = d.matvec_flops();
  return lv;
}

int64_t sk_elems_of(const DictImpl& d) {
  return d.kind == fl1::kSukro ? static_cast<int64_t>(d.nterms) * d.m * d.q : 0;
}

EngineState run_utility(DictImpl& d, int mode, const double* in_host, double* out_host, size_t out_len) {
  d.ctx->bind();
  WsLease lease(d.ctx, d.n, d.k, 1, sk_elems_of(d), d.kind == fl1::kSukro ? d.m : 0);
  Workspace& w = *lease.w;
  EngineParams p = w.base;
  p.mode = mode;
  p.n_levels = 1;
  p.lv[0] = make_dict_level(d);
  p.mode_level = 0;
  p.gauss0 = d.ctx->gauss0(d.k);
  EngineState st{};
  ck(cudaMemcpyAsync(p.st, &st, sizeof(st), cudaMemcpyHostToDevice, w.stream), "state upload");
  // identity bank
  std::vector<int32_t> ident(static_cast<size_t>(d.k));
  for (int64_t j = 0; j < d.k; ++j) ident[static_cast<size_t>(j)] = static_cast<int32_t>(j);
  ck(cudaMemcpyAsync(p.bank[0].idx, ident.data(), ident.size() * sizeof(int32_t), cudaMemcpyHostToDevice,
                     w.stream),
     "ident upload");
  if (in_host) {
    const int64_t len = mode == fl1::kModeAdjoint ? d.n : d.k;
    double* dst = const_cast<double*>(p.x_init);
    if (mode == fl1::kModeAdjoint) ck(cudaMemsetAsync(dst, 0, static_cast<size_t>(w.ld) * sizeof(double), w.stream), "memset");
    ck(cudaMemcpyAsync(dst, in_host, static_cast<size_t>(len) * sizeof(double), cudaMemcpyHostToDevice, w.stream),
       "input upload");
  }
  ck((w.fused_engine ? fl1::engine_launch_fp : fl1::engine_launch)(p, w.sk_m, w.stream), "engine launch");
  if (out_host)
    ck(cudaMemcpyAsync(out_host, p.vec_out, out_len * sizeof(double), cudaMemcpyDeviceToHost, w.stream),
       "output download");
  ck(cudaMemcpyAsync(&st, p.st, sizeof(st), cudaMemcpyDeviceToHost, w.stream), "state download");
  ck(cudaStreamSynchronize(w.stream), "sync");
  if (std::getenv("FL1_UTIL_LOG"))  // diagnostics: power-step count and sub-phase times (ns)
    std::fprintf(stderr, "fl1 utility mode %d: %lld power steps, apply %.0f combine %.0f adjoint %.0f reduce %.0f ns\n",
                 mode, static_cast<long long>(st.power_steps), st.prof_pw[0], st.prof_pw[1], st.prof_pw[2],
                 st.prof_pw[3]);
  return st;
}

std::shared_ptr<DictImpl> new_dense(fl1_ctx* ctx, const double* a, int64_t n, int64_t k, bool device_src) {
  if (!ctx) throw std::invalid_argument("null context");
  if (n < 1 || k < 1) throw std::invalid_argument("dictionary must have at least one row and one column");
  if (k > std::numeric_limits<int32_t>::max()) throw std::invalid_argument("too many atoms");
  ctx->bind();
  auto d = std::make_shared<DictImpl>();
  d->ctx = ctx;
  d->kind = fl1::kDense;
  d->n = n;
  d->k = k;
  d->ld = even_ld(n);
  d->a = std::make_unique<DevBuf>(static_cast<size_t>(d->ld) * static_cast<size_t>(k) * sizeof(double));
  // host input: one H2D copy; device input: one D2D copy (the matrix never visits the host)
  const cudaMemcpyKind kind = device_src ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  if (d->ld == n) {
    ck(cudaMemcpy(d->a->p, a, static_cast<size_t>(n) * static_cast<size_t>(k) * sizeof(double), kind),
       "dictionary copy");
  } else {
    ck(cudaMemset(d->a->p, 0, d->a->bytes), "memset");
    ck(cudaMemcpy2D(d->a->p, static_cast<size_t>(d->ld) * sizeof(double), a, static_cast<size_t>(n) * sizeof(double),
                    static_cast<size_t>(n) * sizeof(double), static_cast<size_t>(k), kind),
       "dictionary copy");
  }
  // atom norms (DenseDictionary ctor, dictionary.cpp:63) on the device, sequential order per
  // column (bit-identical to the host restatement); only the K norms come back
  DevBuf nrm(static_cast<size_t>(k) * sizeof(double));
  ck(fl1::dense_norms_launch(d->a->as<double>(), n, d->ld, k, nrm.as<double>(), nullptr), "atom norms");
  d->norms.resize(static_cast<size_t>(k));
  ck(cudaMemcpy(d->norms.data(), nrm.p, nrm.bytes, cudaMemcpyDeviceToHost), "atom norms download");
  return d;
}

std::unique_ptr<DevBuf> upload(const std::vector<double>& v) {
  auto b = std::make_unique<DevBuf>(std::max<size_t>(v.size(), 1) * sizeof(double));
  if (!v.empty()) ck(cudaMemcpy(b->p, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice), "upload");
  return b;
}

// ---------------------------------------------------------------- solve
// run_lasso / Engine ctor validation shared by the single and batched entries.
struct SolvePlan {
  fl1_ctx* ctx = nullptr;
  int64_t n = 0, k = 0, sk_elems = 0, sk_m = 0;
  int levels = 0, start_level = 0;
};

SolvePlan plan_solve(fl1_seq* s, const fl1_switch_config* cfg, const fl1_run_options* opts) {
  if (!s || !cfg || !opts) throw std::invalid_argument("null argument");
  s->validate();  // run_lasso (fastl1.cpp:755)
  SolvePlan pl;
  const ApproxImpl& exact = *s->lv.back();
  const DictImpl& ed = *exact.dict;
  pl.ctx = ed.ctx;
  pl.n = ed.n;
  pl.k = ed.k;
  for (const auto& l : s->lv) {
    if (l->dict->ctx != pl.ctx) throw std::invalid_argument("levels live on different contexts");
    if (l->dict->n != pl.n) throw std::invalid_argument("sequence has mismatched signal lengths");
  }
  for (const auto& l : s->lv) {
    pl.sk_elems = std::max(pl.sk_elems, sk_elems_of(*l->dict));
    if (l->dict->kind == fl1::kSukro) pl.sk_m = std::max(pl.sk_m, l->dict->m);
  }
  if (s->lv.size() > static_cast<size_t>(fl1::kMaxLevels)) throw std::invalid_argument("too many levels");
  // Engine ctor validation (fastl1.cpp:268-273)
  if (cfg->gamma_threshold <= 0.0 || cfg->gamma_threshold >= 1.0)
    throw std::invalid_argument("gamma threshold must lie in (0, 1)");
  if (cfg->screening_interval < 1) throw std::invalid_argument("screening interval must be >= 1");
  if (opts->solver != FL1_ISTA && opts->solver != FL1_FISTA) throw std::invalid_argument("unknown solver");
  if (opts->rule != FL1_RULE_GAP && opts->rule != FL1_RULE_DYNAMIC) throw std::invalid_argument("unknown rule");
  if (opts->variant < FL1_PLAIN || opts->variant > FL1_MULTI_DICT) throw std::invalid_argument("unknown variant");
  pl.levels = static_cast<int>(s->lv.size());
  pl.start_level = opts->variant == FL1_MULTI_DICT ? 0 : pl.levels - 1;
  if (opts->full_lipschitz && opts->n_full_lipschitz < pl.levels)
    throw std::invalid_argument("full_lipschitz must list one value per level");
  return pl;
}

void fill_params(EngineParams& p, const SolvePlan& pl, fl1_seq* s, double lambda, const fl1_switch_config* cfg,
                 const fl1_run_options* opts) {
  p.mode = fl1::kModeSolve;
  p.n_levels = pl.levels;
  for (int i = 0; i < pl.levels; ++i) p.lv[i] = make_level(s->lv[static_cast<size_t>(i)].get());
  p.lambda = lambda;
  p.gamma_threshold = cfg->gamma_threshold;
  p.interval = cfg->screening_interval;
  p.precompute_aty = cfg->precompute_aty;
  p.tol = cfg->tolerance;
  p.rel_tol = cfg->rel_tolerance;
  p.max_it = cfg->max_iterations;
  p.solver = opts->solver;
  p.rule = opts->rule;
  p.variant = opts->variant;
  p.has_full_l = opts->full_lipschitz != nullptr;
  for (int i = 0; i < pl.levels && p.has_full_l; ++i) p.full_l[i] = opts->full_lipschitz[i];
  p.collect_trace = opts->collect_trace ? 1 : 0;
  p.observe = opts->observer ? 1 : 0;
  p.has_x_init = opts->x_init ? 1 : 0;
  p.gauss0 = pl.ctx->gauss0(pl.k);
  p.gram = nullptr;
  p.gram_ld = 0;
  if (opts->exact_gram) {  // RunOptions::exact_gram (fastl1.hpp:89-91)
    const DictImpl& g = *reinterpret_cast<const fl1_dict*>(opts->exact_gram)->d;
    if (g.kind != fl1::kDense || g.n != pl.k || g.k != pl.k) throw std::invalid_argument("exact_gram must be K x K");
    if (g.ctx != pl.ctx) throw std::invalid_argument("exact_gram lives on another context");
    p.gram = g.a->as<double>();
    p.gram_ld = g.ld;
  }
}

// finish (fastl1.cpp:741-748) and SolveResult fields from the final device state
void fill_result(fl1_result& r, const EngineState& st, const fl1_switch_config* cfg, int64_t k,
                 std::vector<int32_t> idx, const double* xs, std::vector<fl1_switch_event> sws) {
  r.k = k;
  r.xv.assign(xs, xs + idx.size());
  r.final_active = std::move(idx);
  r.converged = st.converged != 0;
  r.iterations = st.converged ? st.t : cfg->max_iterations;
  r.final_gap = st.converged ? st.final_gap : std::numeric_limits<double>::quiet_NaN();
  r.total_flops = st.ledger;
  r.gap_warning = st.warning != 0;
  r.switches = std::move(sws);
  r.setup_ms = (st.t0_ns - st.start_ns) * 1e-6;
  r.power_steps = st.power_steps;
  for (int i = 0; i < 5; ++i) r.prof[i] = st.prof_ns[i];
  r.prof[5] = st.prof_bytes;
  r.prof[6] = st.prof_apply_bytes;
  r.prof[7] = st.prof_power_bytes;
  for (int i = 0; i < 4; ++i) r.prof[8 + i] = st.prof_pw[i];
  r.prof[12] = st.prof_full_ns;
  r.prof[13] = st.prof_full_bytes;
}

void do_solve(fl1_seq* s, const double* y, bool y_device, double lambda, const fl1_switch_config* cfg,
              const fl1_run_options* opts, fl1_result** out, int grid_cap = 0) {
  if (!out) throw std::invalid_argument("null argument");
  const SolvePlan pl = plan_solve(s, cfg, opts);
  if (lambda <= 0) throw std::invalid_argument("lambda must be positive");
  fl1_ctx* ctx = pl.ctx;
  const int64_t n = pl.n, k = pl.k, sk_elems = pl.sk_elems, sk_m = pl.sk_m;
  const int start_level = pl.start_level;
  ctx->bind();
  const uint64_t want_rows = opts->collect_trace ? cfg->max_iterations : 1;
  uint64_t cap_limit = 1u << 20;  // device trace rows per launch; full buffers are flushed and the solve resumes
  if (const char* e = std::getenv("FL1_TRACE_CAP")) cap_limit = std::max<uint64_t>(1, std::strtoull(e, nullptr, 10));
  const int64_t cap = static_cast<int64_t>(std::min<uint64_t>(std::max<uint64_t>(want_rows, 1), cap_limit));
  WsLease lease(ctx, n, k, cap, sk_elems, sk_m, grid_cap);
  Workspace& w = *lease.w;
  EngineParams p = w.base;
  fill_params(p, pl, s, lambda, cfg, opts);
  p.trace_cap = cap;  // <= w.trace_cap (a cached workspace may be larger)
  // FL1_COMPACT=1: physically compacted preserved columns (the A/B alternative to the
  // index gather); two ping-pong copies of up to ceil(K/2) columns
  static const bool compact = [] {
    const char* e = std::getenv("FL1_COMPACT");
    return e && e[0] == '1';
  }();
  bool any_dense = false;
  for (const auto& l : s->lv) any_dense = any_dense || l->dict->kind == fl1::kDense;
  if (compact && any_dense) {
    const size_t half = static_cast<size_t>((k + 1) / 2) * static_cast<size_t>(w.ld);
    if (!w.cbuf || w.cbuf->bytes < 2 * half * sizeof(double)) w.cbuf = std::make_unique<DevBuf>(2 * half * sizeof(double));
    p.compact = 1;
    p.cbuf[0] = w.cbuf->as<double>();
    p.cbuf[1] = w.cbuf->as<double>() + half;
  }
  std::unique_ptr<DevBuf> timeline;
  const char* tl_path = std::getenv("FL1_TIMELINE_OUT");  // instrumented builds only
  if (tl_path) {
    timeline = std::make_unique<DevBuf>(static_cast<size_t>(4096) * w.grid * 8 * sizeof(uint64_t));
    ck(cudaMemset(timeline->p, 0, timeline->bytes), "timeline memset");
    p.timeline = timeline->as<uint64_t>();
  }

  auto res = std::make_unique<fl1_result>();
  res->k = k;
  EngineState st{};
  st.dict_index = start_level;
  st.t_k = 1.0;

  ck(cudaEventRecord(w.ev0, w.stream), "event");
  EngineState& hst = *w.h_st;  // pinned: every transfer below is asynchronous on the solve stream
  hst = st;
  ck(cudaMemcpyAsync(p.st, &hst, sizeof(st), cudaMemcpyHostToDevice, w.stream), "state upload");
  ck(cudaMemsetAsync(const_cast<double*>(p.y), 0, static_cast<size_t>(w.ld) * sizeof(double), w.stream), "memset");
  if (y_device) {
    ck(cudaMemcpyAsync(const_cast<double*>(p.y), y, static_cast<size_t>(n) * sizeof(double), cudaMemcpyDeviceToDevice,
                       w.stream),
       "y copy");
  } else {
    std::copy(y, y + n, w.h_y);
    ck(cudaMemcpyAsync(const_cast<double*>(p.y), w.h_y, static_cast<size_t>(n) * sizeof(double),
                       cudaMemcpyHostToDevice, w.stream),
       "y upload");
  }
  if (opts->x_init)
    ck(cudaMemcpyAsync(const_cast<double*>(p.x_init), opts->x_init, static_cast<size_t>(k) * sizeof(double),
                       cudaMemcpyHostToDevice, w.stream),
       "x_init upload");
  std::vector<fl1_trace_row> host_rows;
  int64_t launches = 0;
  int64_t h2d = static_cast<int64_t>(sizeof(st)) + (y_device ? 0 : 8 * n) + (opts->x_init ? 8 * k : 0);
  int64_t d2h = 0;
  std::vector<int32_t> h_idx;
  std::vector<int8_t> h_keep;
  std::vector<double> h_rho, h_y;
  while (true) {
    ck((w.fused_engine ? fl1::engine_launch_fp : fl1::engine_launch)(p, w.sk_m, w.stream), "engine launch");
    ++launches;
    ck(cudaMemcpyAsync(&hst, p.st, sizeof(st), cudaMemcpyDeviceToHost, w.stream), "state download");
    ck(cudaStreamSynchronize(w.stream), "engine sync");
    st = hst;
    d2h += static_cast<int64_t>(sizeof(st));
    if (st.event == fl1::kEvTraceFull || st.event == fl1::kEvDone) {
      if (p.collect_trace && st.n_trace > 0) {
        d2h += st.n_trace * static_cast<int64_t>(sizeof(fl1_trace_row));
        for (int64_t off = 0; off < st.n_trace; off += w.h_trace_cap) {
          const int64_t cnt = std::min(w.h_trace_cap, st.n_trace - off);
          ck(cudaMemcpyAsync(w.h_trace, p.trace + off, static_cast<size_t>(cnt) * sizeof(fl1_trace_row),
                             cudaMemcpyDeviceToHost, w.stream),
             "trace download");
          ck(cudaStreamSynchronize(w.stream), "trace sync");
          host_rows.insert(host_rows.end(), w.h_trace, w.h_trace + cnt);
        }
        st.trace_base += static_cast<uint64_t>(st.n_trace);
        st.n_trace = 0;
      }
    }
    if (st.event == fl1::kEvObserve) {
      // ScreeningEvent (fastl1.cpp:704-734) from the device snapshot
      const int64_t S0 = st.obs_S;
      const fl1::Bank& ob = p.bank[st.obs_bank];
      h_idx.resize(static_cast<size_t>(S0));
      h_keep.resize(static_cast<size_t>(S0));
      h_rho.resize(static_cast<size_t>(w.ld));
      if (S0 > 0) {
        ck(cudaMemcpy(h_idx.data(), ob.idx, static_cast<size_t>(S0) * sizeof(int32_t), cudaMemcpyDeviceToHost), "obs");
        ck(cudaMemcpy(h_keep.data(), ob.keep, static_cast<size_t>(S0), cudaMemcpyDeviceToHost), "obs");
      }
      ck(cudaMemcpy(h_rho.data(), p.rho_obs, static_cast<size_t>(w.ld) * sizeof(double), cudaMemcpyDeviceToHost), "obs");
      if (h_y.empty()) {
        h_y.resize(static_cast<size_t>(n));
        ck(cudaMemcpy(h_y.data(), p.y, static_cast<size_t>(n) * sizeof(double), cudaMemcpyDeviceToHost), "obs");
      }
      const std::vector<double>& ray = st.obs_ray_is_y ? h_y : h_rho;
      std::vector<double> tp(static_cast<size_t>(n)), tt(static_cast<size_t>(n)), center(static_cast<size_t>(n));
      for (int64_t i = 0; i < n; ++i) {
        tp[static_cast<size_t>(i)] = st.obs_scale_prime * ray[static_cast<size_t>(i)];
        tt[static_cast<size_t>(i)] = st.obs_scale_tilde * ray[static_cast<size_t>(i)];
        center[static_cast<size_t>(i)] =
            opts->rule == FL1_RULE_GAP ? tp[static_cast<size_t>(i)] : h_y[static_cast<size_t>(i)] / lambda;
      }
      std::vector<int32_t> kept;
      for (int64_t q = 0; q < S0; ++q)
        if (h_keep[static_cast<size_t>(q)]) kept.push_back(h_idx[static_cast<size_t>(q)]);
      fl1_screen_event ev{};
      ev.iter = st.obs_iter;
      ev.dict_index = st.obs_dict;
      ev.n = n;
      ev.center = center.data();
      ev.radius = st.obs_radius;
      ev.theta_prime = tp.data();
      ev.theta_tilde = tt.data();
      ev.scale_prime = st.obs_scale_prime;
      ev.scale_tilde = st.obs_scale_tilde;
      ev.n_active_before = S0;
      ev.active_before = h_idx.data();
      ev.n_kept = static_cast<int64_t>(kept.size());
      ev.kept = kept.data();
      opts->observer(&ev, opts->observer_user);
      st.obs_pending = 0;
    }
    if (st.done) break;
    // resume: push the edited state back
    st.event = fl1::kEvNone;
    p.mode = fl1::kModeResume;
    h2d += static_cast<int64_t>(sizeof(st));
    hst = st;
    ck(cudaMemcpyAsync(p.st, &hst, sizeof(st), cudaMemcpyHostToDevice, w.stream), "state upload");
  }
  // finish (fastl1.cpp:741-748)
  const fl1::Bank& fb = p.bank[st.cur];
  if (st.S > 0) {
    ck(cudaMemcpyAsync(w.h_idx, fb.idx, static_cast<size_t>(st.S) * sizeof(int32_t), cudaMemcpyDeviceToHost,
                       w.stream),
       "x");
    ck(cudaMemcpyAsync(w.h_x, fb.x, static_cast<size_t>(st.S) * sizeof(double), cudaMemcpyDeviceToHost, w.stream), "x");
  }
  if (st.n_switches > 0)
    ck(cudaMemcpyAsync(w.h_sw, p.sw, static_cast<size_t>(st.n_switches) * sizeof(fl1_switch_event),
                       cudaMemcpyDeviceToHost, w.stream),
       "switches");
  d2h += st.S * 12 + st.n_switches * static_cast<int64_t>(sizeof(fl1_switch_event));
  ck(cudaEventRecord(w.ev1, w.stream), "event");
  ck(cudaStreamSynchronize(w.stream), "finish sync");
  std::vector<int32_t> idx(w.h_idx, w.h_idx + st.S);
  std::vector<double> xs(w.h_x, w.h_x + st.S);
  std::vector<fl1_switch_event> sws(w.h_sw, w.h_sw + st.n_switches);
  float ms = 0.f;
  ck(cudaEventElapsedTime(&ms, w.ev0, w.ev1), "elapsed");
  if (timeline) {
    std::vector<uint64_t> h(timeline->bytes / sizeof(uint64_t));
    ck(cudaMemcpy(h.data(), timeline->p, timeline->bytes, cudaMemcpyDeviceToHost), "timeline");
    if (FILE* f = std::fopen(tl_path, "wb")) {
      std::fwrite(h.data(), sizeof(uint64_t), h.size(), f);
      std::fclose(f);
    }
  }
  fill_result(*res, st, cfg, k, std::move(idx), xs.data(), std::move(sws));
  res->trace = std::move(host_rows);
  res->device_ms = ms;
  res->launches = launches;
  res->h2d = h2d;
  res->d2h = d2h;
  *out = res.release();
}

}  // namespace

extern "C" {

const char* fl1_last_error(void) { return g_err.c_str(); }
const char* fl1_version(void) { return "fl1cuda 0.1 (sm_100a persistent engine)"; }

int fl1_ctx_create(int device, fl1_ctx** out) {
  return guard([&] {
    if (!out) throw std::invalid_argument("null out");
    int count = 0;
    ck(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
    if (device < 0 || device >= count) throw std::invalid_argument("no such CUDA device");
    auto c = std::make_unique<fl1_ctx>();
    c->device = device;
    c->bind();
    ck(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device), "attr");
    int l2 = 0;
    ck(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device), "attr");
    c->l2 = l2;
    size_t fr = 0, tot = 0;
    ck(cudaMemGetInfo(&fr, &tot), "meminfo");
    c->hbm = static_cast<int64_t>(tot);
    *out = c.release();
  });
}
int fl1_ctx_destroy(fl1_ctx* ctx) {
  return guard([&] {
    if (!ctx) return;
    ctx->bind();
    delete ctx;
  });
}
int fl1_ctx_info(fl1_ctx* ctx, int32_t* sm_count, int64_t* l2_bytes, int64_t* hbm_bytes) {
  return guard([&] {
    if (sm_count) *sm_count = ctx->sms;
    if (l2_bytes) *l2_bytes = ctx->l2;
    if (hbm_bytes) *hbm_bytes = ctx->hbm;
  });
}

int fl1_dict_dense(fl1_ctx* ctx, const double* a, int64_t n, int64_t k, fl1_dict** out) {
  return guard([&] { *out = new fl1_dict{new_dense(ctx, a, n, k, false)}; });
}
int fl1_dict_dense_device(fl1_ctx* ctx, const double* a, int64_t n, int64_t k, fl1_dict** out) {
  return guard([&] { *out = new fl1_dict{new_dense(ctx, a, n, k, true)}; });
}
int fl1_dict_sukro(fl1_ctx* ctx, int32_t n_terms, int64_t m, int64_t q, const double* const* left,
                   const double* const* right, const double* col_scale, fl1_dict** out) {
  return guard([&] {
    if (!ctx) throw std::invalid_argument("null context");
    if (n_terms < 1) throw std::invalid_argument("SuKro needs at least one term");
    if (m < 1 || q < 1) throw std::invalid_argument("empty SuKro factor");
    if (m > fl1::kSukroMaxM || q > fl1::kSukroMaxQ)
      throw std::logic_error("SuKro factors larger than 128 x 256 are not supported by this build");
    if (q * q > std::numeric_limits<int32_t>::max()) throw std::invalid_argument("too many atoms");
    ctx->bind();
    auto d = std::make_shared<DictImpl>();
    d->ctx = ctx;
    d->kind = fl1::kSukro;
    d->m = m;
    d->q = q;
    d->n = m * m;
    d->k = q * q;
    d->ld = even_ld(d->n);
    d->nterms = n_terms;
    const size_t blk = static_cast<size_t>(m * q);
    d->h_left.resize(blk * static_cast<size_t>(n_terms));
    d->h_right.resize(blk * static_cast<size_t>(n_terms));
    for (int t = 0; t < n_terms; ++t) {
      std::copy(left[t], left[t] + blk, d->h_left.begin() + static_cast<long>(blk) * t);
      std::copy(right[t], right[t] + blk, d->h_right.begin() + static_cast<long>(blk) * t);
    }
    if (col_scale) d->h_scale.assign(col_scale, col_scale + d->k);
    d->left = upload(d->h_left);
    d->right = upload(d->h_right);
    if (col_scale) d->col_scale = upload(d->h_scale);
    // exact atom norms of the explicit columns, expanded on the device (setup only)
    DevBuf nrm(static_cast<size_t>(d->k) * sizeof(double));
    ck(fl1::sukro_norms_launch(d->left->as<double>(), d->right->as<double>(),
                               col_scale ? d->col_scale->as<double>() : nullptr, n_terms, m, q, nrm.as<double>(),
                               nullptr),
       "sukro atom norms");
    d->norms.resize(static_cast<size_t>(d->k));
    ck(cudaMemcpy(d->norms.data(), nrm.p, nrm.bytes, cudaMemcpyDeviceToHost), "sukro atom norms download");
    *out = new fl1_dict{d};
  });
}
int fl1_dict_destroy(fl1_dict* d) {
  return guard([&] { delete d; });
}
int fl1_dict_shape(const fl1_dict* d, int64_t* rows, int64_t* cols) {
  return guard([&] {
    *rows = d->d->n;
    *cols = d->d->k;
  });
}
int fl1_dict_is_dense(const fl1_dict* d) { return d->d->kind == fl1::kDense ? 1 : 0; }
uint64_t fl1_dict_matvec_flops(const fl1_dict* d) { return d->d->matvec_flops(); }
int fl1_dict_atom_norms(const fl1_dict* d, double* out) {
  return guard([&] { std::copy(d->d->norms.begin(), d->d->norms.end(), out); });
}
int fl1_dict_apply(fl1_dict* d, const double* x, double* out) {
  return guard([&] { run_utility(*d->d, fl1::kModeApply, x, out, static_cast<size_t>(d->d->n)); });
}
int fl1_dict_apply_adjoint(fl1_dict* d, const double* r, double* out) {
  return guard([&] { run_utility(*d->d, fl1::kModeAdjoint, r, out, static_cast<size_t>(d->d->k)); });
}
int fl1_dict_column(fl1_dict* dh, int64_t j, double* out) {
  return guard([&] {
    const DictImpl& d = *dh->d;
    if (j < 0 || j >= d.k) throw std::invalid_argument("column index out of range");
    d.ctx->bind();
    if (d.kind == fl1::kDense) {
      ck(cudaMemcpy(out, d.a->as<double>() + j * d.ld, static_cast<size_t>(d.n) * sizeof(double),
                    cudaMemcpyDeviceToHost),
         "column download");
      return;
    }
    const size_t blk = static_cast<size_t>(d.m * d.q);
    const int64_t jb = j / d.q, jc = j % d.q;
    std::fill(out, out + d.n, 0.0);
    for (int t = 0; t < d.nterms; ++t)
      for (int64_t rb = 0; rb < d.m; ++rb) {
        const double bv = d.h_left[blk * static_cast<size_t>(t) + static_cast<size_t>(jb * d.m + rb)];
        for (int64_t rc = 0; rc < d.m; ++rc)
          out[rb * d.m + rc] += bv * d.h_right[blk * static_cast<size_t>(t) + static_cast<size_t>(jc * d.m + rc)];
      }
    if (!d.h_scale.empty())
      for (int64_t i = 0; i < d.n; ++i) out[i] *= d.h_scale[static_cast<size_t>(j)];
  });
}

int fl1_approx_create(fl1_dict* d, const double* eps, double op_err, double rc, const double* an,
                      const double* en, fl1_approx** out) {
  return guard([&] {
    if (!d || !eps || !an || !en) throw std::invalid_argument("null argument");
    auto a = std::make_shared<ApproxImpl>();
    const int64_t k = d->d->k;
    a->dict = d->d;
    a->eps.assign(eps, eps + k);
    a->an.assign(an, an + k);
    a->en.assign(en, en + k);
    a->op_err = op_err;
    a->rc = rc;
    d->d->ctx->bind();
    a->d_eps = upload(a->eps);
    a->d_an = upload(a->an);
    a->d_en = upload(a->en);
    *out = new fl1_approx{a};
  });
}
int fl1_approx_exact(fl1_dict* d, fl1_approx** out) {  // make_exact_approx (dictionary.cpp:216-225)
  return guard([&] {
    if (!d) throw std::invalid_argument("null argument");
    if (d->d->kind != fl1::kDense) throw std::invalid_argument("make_exact_approx needs a dense dictionary");
    auto a = std::make_shared<ApproxImpl>();
    a->dict = d->d;
    a->eps.assign(static_cast<size_t>(d->d->k), 0.0);
    a->an = d->d->norms;
    a->en = d->d->norms;
    a->op_err = 0.0;
    a->rc = 1.0;
    d->d->ctx->bind();
    a->d_eps = upload(a->eps);
    a->d_an = upload(a->an);
    a->d_en = upload(a->en);
    *out = new fl1_approx{a};
  });
}
int fl1_approx_destroy(fl1_approx* a) {
  return guard([&] { delete a; });
}
int fl1_seq_create(fl1_approx* const* levels, int32_t n_levels, fl1_seq** out) {
  return guard([&] {
    auto s = std::make_unique<fl1_seq>();
    for (int i = 0; i < n_levels; ++i) {
      if (!levels[i]) throw std::invalid_argument("null level");
      s->lv.push_back(levels[i]->a);
    }
    s->validate();
    *out = s.release();
  });
}
int fl1_seq_destroy(fl1_seq* s) {
  return guard([&] { delete s; });
}

namespace {
// A cluster launch cannot flush its device trace (the grid path of do_solve can), so it
// reserves max_iterations rows per signal up front. Reservations above this budget
// (e.g. the reference's default max_iterations = 1e6 with collect_trace over a large
// batch) take the grid path instead.
constexpr uint64_t kClusterTraceBudget = 2ull << 30;

bool cluster_trace_fits(const fl1_switch_config* cfg, const fl1_run_options* opts, int64_t batch) {
  if (!opts->collect_trace) return true;
  const uint64_t rows = std::max<uint64_t>(cfg->max_iterations, 1);
  const uint64_t per_signal = kClusterTraceBudget / sizeof(fl1_trace_row) / static_cast<uint64_t>(std::max<int64_t>(batch, 1));
  return rows <= per_signal;
}

// Batched solves in ONE launch: every thread-block cluster of `csize` CTAs is a
// virtual grid with its own workspace and pulls signals from a device queue
// (each signal runs the same Engine::run as fl1_solve, with cluster barriers).
void solve_clusters(fl1_seq* s, const double* Y, bool y_device, int64_t ldy, const double* lambdas, int32_t batch,
                    const fl1_switch_config* cfg, const fl1_run_options* opts, int csize, fl1_result** out,
                    bool allow_prefix = true) {
  const auto hl0 = std::chrono::steady_clock::now();
  const bool host_log = std::getenv("FL1_HOST_LOG") != nullptr;  // diagnostics: host-side stage times
  auto hlog = [&](const char* what) {
    if (host_log)
      std::fprintf(stderr, "fl1 batched host: %-12s %.3f ms\n", what,
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - hl0).count());
  };
  const SolvePlan pl = plan_solve(s, cfg, opts);
  for (int32_t b = 0; b < batch; ++b)
    if (!(lambdas[b] > 0)) throw std::invalid_argument("lambda must be positive");
  if (csize < 1 || csize > 16) throw std::invalid_argument("cluster size must lie in [1, 16]");
  fl1_ctx* ctx = pl.ctx;
  ctx->bind();
  const int64_t n = pl.n, k = pl.k, ld = even_ld(n), units = (n + fl1::kUnit - 1) / fl1::kUnit;
  std::lock_guard<std::mutex> batch_lock(ctx->batch_mu);
  int n_clusters = 0;
  {  // launch shape, cached per (ld, SuKro m, cluster size)
    const auto key = std::make_tuple(ld, pl.sk_m, csize);
    auto it = ctx->cluster_cfg.find(key);
    if (it == ctx->cluster_cfg.end()) {
      int grid = 0;
      const cudaError_t e = fl1::engine_configure(ld, pl.sk_m, ctx->device, &grid);
      if (e == cudaErrorInvalidConfiguration)
        throw std::logic_error("signal length too large for the shared-memory resident residual");
      ck(e, "engine_configure");
      int nc = 0;
      ck(fl1::engine_cluster_capacity(ld, pl.sk_m, csize, &nc), "cluster capacity");
      it = ctx->cluster_cfg.emplace(key, std::make_pair(grid, nc)).first;
    }
    n_clusters = it->second.second;
  }
  if (n_clusters < 1) throw std::runtime_error("no cluster of this size fits on the device");
  n_clusters = std::min<int>(n_clusters, std::max<int32_t>(batch, 1));
  if (!cluster_trace_fits(cfg, opts, batch)) throw std::logic_error("cluster trace reservation over budget");
  const int64_t cap = opts->collect_trace ? static_cast<int64_t>(std::max<uint64_t>(cfg->max_iterations, 1)) : 1;
  const int64_t B = std::max<int32_t>(batch, 1);

  EngineParams tmpl{};
  const size_t ws_bytes = (carve(tmpl, nullptr, n, k, ld, csize, units, 1, pl.sk_m) + 255) / 256 * 256;
  size_t top = ws_bytes * static_cast<size_t>(n_clusters);  // cluster workspaces first, then:
  auto region = [&](size_t bytes) {
    top = (top + 255) / 256 * 256;
    const size_t o = top;
    top += bytes;
    return o;
  };
  const size_t ub = static_cast<size_t>(B), kb = static_cast<size_t>(k);
  // upload block [params | desc | lambdas | states], download block [states | switches |
  // counters | offsets]: one pinned copy each way
  const size_t o_params = region(sizeof(EngineParams) * static_cast<size_t>(n_clusters));
  const size_t o_desc = region(sizeof(fl1::BatchDesc));
  const size_t o_lam = region(sizeof(double) * ub);
  const size_t o_st = region(sizeof(EngineState) * ub);
  const size_t o_sw = region(sizeof(fl1_switch_event) * fl1::kMaxLevels * ub);
  const size_t o_cnt = region(sizeof(int64_t) * static_cast<size_t>(2 + n_clusters));
  const size_t o_off = region(sizeof(int64_t) * ub);
  const size_t up_end = o_st + sizeof(EngineState) * ub, down_end = top;
  const size_t o_y = region(y_device ? 0 : sizeof(double) * static_cast<size_t>(ld) * ub);
  const size_t o_tr = region(sizeof(fl1_trace_row) * static_cast<size_t>(cap) * ub);
  const size_t o_idx = region(sizeof(int32_t) * kb * ub);
  const size_t o_x = region(sizeof(double) * kb * ub);
  char* base = ctx->batch_scratch(0, top + 256).as<char>();
  ctx->batch_objects();
  cudaStream_t stream = ctx->batch_stream;
  cudaEvent_t ev0 = ctx->batch_ev[0], ev1 = ctx->batch_ev[1], evp = ctx->batch_ev[2];
  // pinned host image of [params .. offsets] (+ y), then the final sets
  const size_t img = down_end - o_params;
  const size_t ybytes = y_device ? 0 : sizeof(double) * static_cast<size_t>(ld) * ub;
  char* pin = ctx->pinned_scratch(img + ybytes + 12 * kb * ub + 1024);
  auto at = [&](size_t off) { return pin + (off - o_params); };

  EngineParams* params = reinterpret_cast<EngineParams*>(at(o_params));
  // instrumented builds (FL1_TIMELINE): per-iteration phase marks of a one-signal call
  std::unique_ptr<DevBuf> timeline;
  const char* tl_path = batch == 1 ? std::getenv("FL1_TIMELINE_OUT") : nullptr;
  if (tl_path) {
    timeline = std::make_unique<DevBuf>(static_cast<size_t>(4096) * csize * 8 * sizeof(uint64_t));
    ck(cudaMemset(timeline->p, 0, timeline->bytes), "timeline memset");
  }
  for (int q = 0; q < n_clusters; ++q) {
    EngineParams& p = params[q];
    p = EngineParams{};
    carve(p, base + static_cast<size_t>(q) * ws_bytes, n, k, ld, csize, units, 1, pl.sk_m);
    fill_params(p, pl, s, 1.0, cfg, opts);
    p.grid = csize;
    p.n = n;
    p.k = k;
    p.ld = ld;
    p.trace_cap = cap;
    if (timeline) p.timeline = timeline->as<uint64_t>();
  }
  fl1::BatchDesc bd{};
  bd.batch = batch;
  int64_t* counters = reinterpret_cast<int64_t*>(base + o_cnt);
  bd.next = reinterpret_cast<int32_t*>(counters);
  bd.out_used = counters + 1;
  bd.cluster_sig = reinterpret_cast<int32_t*>(counters + 2);
  bd.cluster_params = reinterpret_cast<const EngineParams*>(base + o_params);
  bd.Y = y_device ? Y : reinterpret_cast<const double*>(base + o_y);
  bd.ldy = y_device ? ldy : ld;
  bd.lambdas = reinterpret_cast<const double*>(base + o_lam);
  bd.states = reinterpret_cast<EngineState*>(base + o_st);
  bd.traces = reinterpret_cast<fl1_trace_row*>(base + o_tr);
  bd.trace_cap = cap;
  bd.sws = reinterpret_cast<fl1_switch_event*>(base + o_sw);
  bd.out_off = reinterpret_cast<int64_t*>(base + o_off);
  bd.out_idx = reinterpret_cast<int32_t*>(base + o_idx);
  bd.out_x = reinterpret_cast<double*>(base + o_x);
  EngineParams p0{};
  p0.batch = reinterpret_cast<const fl1::BatchDesc*>(base + o_desc);
  p0.ld = ld;

  EngineState* hst = reinterpret_cast<EngineState*>(at(o_st));
  for (int64_t b = 0; b < B; ++b) {
    hst[b] = EngineState{};
    hst[b].dict_index = pl.start_level;
    hst[b].t_k = 1.0;
  }
  std::copy(lambdas, lambdas + batch, reinterpret_cast<double*>(at(o_lam)));
  hlog("prepared");
  ck(cudaEventRecord(ev0, stream), "event");
  ck(cudaMemsetAsync(base, 0, ws_bytes * static_cast<size_t>(n_clusters), stream), "workspace memset");
  ck(cudaMemsetAsync(counters, 0, sizeof(int64_t) * (2 + n_clusters), stream), "counter memset");
  int64_t h2d_sig = static_cast<int64_t>(sizeof(EngineState) + sizeof(double));
  if (!y_device && batch > 0) {
    double* yp = reinterpret_cast<double*>(pin + img);
    for (int32_t b = 0; b < batch; ++b) {
      std::copy(Y + static_cast<int64_t>(b) * ldy, Y + static_cast<int64_t>(b) * ldy + n, yp + b * ld);
      std::fill(yp + b * ld + n, yp + (b + 1) * ld, 0.0);
    }
    ck(cudaMemcpyAsync(base + o_y, yp, ybytes, cudaMemcpyHostToDevice, stream), "signal upload");
    h2d_sig += 8 * n;
  }
  // lockstep engine (batched.cu): dense exact dictionary, GAP rule, cached full L
  std::unique_ptr<DevBuf> step_log;
  int32_t* d_steps = nullptr;
  const ApproxImpl& ex = *s->lv.back();
  const char* pe = std::getenv("FL1_BATCH_PREFIX");
  const bool use_prefix = allow_prefix && batch > 0 && pl.levels == 1 && ex.dict->kind == fl1::kDense &&
                          opts->rule == FL1_RULE_GAP &&
                          (opts->variant == FL1_SCREENED || opts->variant == FL1_PLAIN) &&
                          opts->full_lipschitz != nullptr && k <= fl1::prefix_max_atoms() &&
                          fl1::prefix_fits(ld, batch, ctx->device) &&
                          k % 2 == 0 &&  // per-signal K-strided rows take 16-byte copies (V tiles, staging)
                          !(pe && pe[0] == '0');
  fl1::PrefixParams pp{};
  if (use_prefix) {
    const int64_t bcap = (B + 63) / 64 * 64, kt = (k + 63) / 64;
    size_t ptop = 0;
    auto preg = [&](size_t bytes) {
      ptop = (ptop + 255) / 256 * 256;
      const size_t o = ptop;
      ptop += bytes;
      return o;
    };
    const size_t kb8 = sizeof(double) * static_cast<size_t>(k) * ub, lb8 = sizeof(double) * static_cast<size_t>(ld) * ub;
    const size_t sm = static_cast<size_t>(fl1::prefix_split_max());
    const size_t q_x0 = preg(kb8), q_x1 = preg(kb8), q_x2 = preg(kb8), q_u0 = preg(lb8), q_u1 = preg(lb8);
    const size_t q_mk = preg(static_cast<size_t>(k) * ub), q_ld = preg(kb8), q_ps = preg(kb8), q_vp = preg(kb8);
    const size_t q_hi = preg(sizeof(int32_t) * static_cast<size_t>(k) * ub);
    const size_t q_r = preg(sizeof(double) * static_cast<size_t>(ld) * ub);  // per-signal R columns
    const size_t q_np = preg(sizeof(double) * static_cast<size_t>(ld * bcap) * sm);
    const size_t q_c = preg(sizeof(double) * static_cast<size_t>(k * bcap) * sm);
    const size_t q_s = preg(sizeof(fl1::PrefixSig) * ub), q_h = preg(sizeof(fl1::Handoff) * ub);
    const size_t q_n = preg(sizeof(int64_t) * 4);  // steps, two signal-queue counters | work: sum n_act, sum n_pow
    const size_t q_pt = preg(sizeof(double) * static_cast<size_t>(fl1::prefix_part_elems(ctx->sms)));  // stream-K
    const size_t q_fl = preg(sizeof(int32_t) * 2 * static_cast<size_t>(ctx->sms));
    (void)kt;
    char* pb = ctx->batch_scratch(1, ptop + 256).as<char>();
    pp.n = n;
    pp.k = k;
    pp.ld = ld;
    pp.batch = batch;
    pp.bcap = static_cast<int32_t>(bcap);
    pp.a = ex.dict->a->as<double>();
    pp.en = ex.d_en->as<double>();
    pp.gauss0 = ctx->gauss0(k);
    pp.y = bd.Y;
    pp.ldy = bd.ldy;
    pp.lambdas = bd.lambdas;
    pp.lipschitz = opts->full_lipschitz[pl.levels - 1];
    pp.tol = cfg->tolerance;
    pp.rel_tol = cfg->rel_tolerance;
    pp.max_it = cfg->max_iterations;
    pp.interval = cfg->screening_interval;
    pp.solver = opts->solver;
    pp.variant = opts->variant;
    pp.collect_trace = opts->collect_trace ? 1 : 0;
    // default: signals stay in the lockstep through their first (cold) restricted power
    // iteration -- the dense part of the solve -- and until their preserved set is at
    // most 512 atoms; the per-signal engine finishes the short, small-set tail (policy 3,
    // measured best on B200 with the stream-K contractions: c5 53.7 -> 53.0 ms against
    // policy 2, leaving right after the power iteration; 0 and 1 are the other policies)
    pp.policy = 3;
    if (const char* pol = std::getenv("FL1_LOCKSTEP_POLICY")) pp.policy = std::atoi(pol);
    const char* hs = std::getenv("FL1_HANDOFF_S");
    pp.handoff_s = hs ? std::atoll(hs) : 512;
    const char* smode = std::getenv("FL1_SPLIT_MODE");
    pp.split_mode = smode ? std::atoi(smode) : 1;
    const char* sb = std::getenv("FL1_SPLIT_BUDGET_MB");
    // split-K partials capped at 24 MiB per contraction: they stay L2-resident beside the
    // 33.5 MB dictionary instead of round-tripping DRAM (c5: lockstep DRAM 19.8 -> ~9 GB,
    // 55.7 -> 55.3 ms; 16 MiB costs waves, 32-48 MiB the same)
    pp.split_budget = sb ? (std::atoll(sb) << 20) : (24ll << 20);
    const char* nm = std::getenv("FL1_LOCKSTEP_NARROW");
    pp.narrow = nm ? std::atoi(nm) : 1;
    const char* wt = std::getenv("FL1_LOCKSTEP_WIDTH");
    pp.width_tiles = wt ? std::atoi(wt) : 1;
    pp.X3[0] = reinterpret_cast<double*>(pb + q_x0);
    pp.X3[1] = reinterpret_cast<double*>(pb + q_x1);
    pp.X3[2] = reinterpret_cast<double*>(pb + q_x2);
    pp.U2[0] = reinterpret_cast<double*>(pb + q_u0);
    pp.U2[1] = reinterpret_cast<double*>(pb + q_u1);
    pp.mask = reinterpret_cast<int8_t*>(pb + q_mk);
    pp.lead = reinterpret_cast<double*>(pb + q_ld);
    pp.psrc = reinterpret_cast<double*>(pb + q_ps);
    pp.vp = reinterpret_cast<double*>(pb + q_vp);
    pp.hidx = reinterpret_cast<int32_t*>(pb + q_hi);
    pp.R = reinterpret_cast<double*>(pb + q_r);
    pp.np = reinterpret_cast<double*>(pb + q_np);
    pp.corr = reinterpret_cast<double*>(pb + q_c);
    pp.sig = reinterpret_cast<fl1::PrefixSig*>(pb + q_s);
    pp.hand = reinterpret_cast<fl1::Handoff*>(pb + q_h);
    pp.states = bd.states;
    pp.out_used = bd.out_used;
    pp.out_off = bd.out_off;
    pp.out_idx = bd.out_idx;
    pp.out_x = bd.out_x;
    pp.traces = bd.traces;
    pp.trace_cap = cap;
    pp.steps_out = reinterpret_cast<int32_t*>(pb + q_n);
    pp.queue = pp.steps_out + 1;
    pp.work_out = reinterpret_cast<int64_t*>(pb + q_n) + 2;
    // stream-K contractions on the TMA ring (default); FL1_LOCKSTEP_TMA=0: split-K cp.async tiles
    const char* tma = std::getenv("FL1_LOCKSTEP_TMA");
    pp.tma = (tma ? std::atoi(tma) : 1) && ctx->sms <= fl1::prefix_stream_k_max_grid();
    const char* fi = std::getenv("FL1_SK_FANIN");
    pp.sk_fanin = fi ? std::atoi(fi) : 4;
    if (pp.tma) {
      pp.part = reinterpret_cast<double*>(pb + q_pt);
      pp.flags = reinterpret_cast<int32_t*>(pb + q_fl);
      // slot-ordered inputs reuse the split-K partial regions (unused on this route)
      pp.rc = pp.np;                                        // ld x bcap
      pp.vc = pp.corr + static_cast<size_t>(k) * bcap;      // k x bcap (corr part 1)
      // A is ld x k column-major; boxes over-fetch into the padded tile layouts (batched.cu)
      ck(encode_tensor_map_2d(&pp.tm_corr, pp.a, ld, k, 36, 128), "tensor map (Corr A)");
      ck(encode_tensor_map_2d(&pp.tm_w, pp.a, ld, k, 132, 32), "tensor map (W A)");
      ck(encode_tensor_map_2d(&pp.tm_rc, pp.rc, ld, bcap, 36, 64), "tensor map (Rc)");
      ck(encode_tensor_map_2d(&pp.tm_vc, pp.vc, k, bcap, 36, 64), "tensor map (Vc)");
    }
    static std::unique_ptr<DevBuf> sigprof;
    if (const char* sp = std::getenv("FL1_SIGPROF_OUT")) {  // diagnostics builds only (FL1_SIGPROF)
      if (!sigprof) sigprof = std::make_unique<DevBuf>(16 * sizeof(double));
      ck(cudaMemset(sigprof->p, 0, 16 * sizeof(double)), "sigprof");
      pp.sigprof = sigprof->as<double>();
      (void)sp;
    }
    static std::unique_ptr<DevBuf> sk_trace;
    if (const char* st = std::getenv("FL1_SK_TRACE")) {  // diagnostics: per-CTA times of one step's products
      // per product and CTA: 4 times | CTAs 0-3: per unit, the times before / after its full-barrier wait
      if (!sk_trace) sk_trace = std::make_unique<DevBuf>(sizeof(double) * (2 * 4 * 256 + 2 * 4 * 128 * 2));
      ck(cudaMemset(sk_trace->p, 0, sizeof(double) * (2 * 4 * 256 + 2 * 4 * 128 * 2)), "sk trace");
      pp.sk_trace = sk_trace->as<double>();
      pp.sk_trace_step = std::atoi(st);
    }
    if (std::getenv("FL1_STEP_LOG")) {  // diagnostics: per-step occupancy of the lockstep engine
      pp.max_log = 4096;
      step_log = std::make_unique<DevBuf>(sizeof(double) * fl1::kStepLogW * pp.max_log);
      ck(cudaMemset(step_log->p, 0, sizeof(double) * fl1::kStepLogW * pp.max_log), "step log");
      pp.step_log = step_log->as<double>();
    }
    bd.handoff = pp.hand;
    d_steps = pp.steps_out;
  }
  *reinterpret_cast<fl1::BatchDesc*>(at(o_desc)) = bd;
  ck(cudaMemcpyAsync(base + o_params, pin, up_end - o_params, cudaMemcpyHostToDevice, stream), "upload");
  if (use_prefix) ck(fl1::prefix_launch(pp, ctx->device, stream), "prefix launch");
  ck(cudaEventRecord(evp, stream), "event");
  if (batch > 0) ck(fl1::engine_launch_clusters(p0, n_clusters, csize, pl.sk_m, stream), "cluster launch");
  ck(cudaEventRecord(ev1, stream), "event");
  ck(cudaMemcpyAsync(at(o_st), base + o_st, down_end - o_st, cudaMemcpyDeviceToHost, stream), "state download");
  hlog("launched");
  ck(cudaStreamSynchronize(stream), "batched sync");
  hlog("synced");
  const int64_t used = reinterpret_cast<const int64_t*>(at(o_cnt))[1];
  const int64_t* offs = reinterpret_cast<const int64_t*>(at(o_off));
  const fl1_switch_event* all_sw = reinterpret_cast<const fl1_switch_event*>(at(o_sw));
  int32_t* all_idx = reinterpret_cast<int32_t*>(pin + img + ybytes);
  double* all_x = reinterpret_cast<double*>(pin + img + ybytes + ((4 * kb * ub + 15) / 16) * 16);
  if (host_log) std::fprintf(stderr, "fl1 batched host: packed outputs %lld\n", static_cast<long long>(used));
  if (used > 0) {
    ck(cudaMemcpyAsync(all_idx, base + o_idx, sizeof(int32_t) * used, cudaMemcpyDeviceToHost, stream), "idx");
    ck(cudaMemcpyAsync(all_x, base + o_x, sizeof(double) * used, cudaMemcpyDeviceToHost, stream), "x");
  }
  // traces: rows [b * cap, b * cap + n_trace_b) of every signal, packed on the device
  // and downloaded in one copy (not one pageable copy per signal)
  std::vector<int64_t> toff(static_cast<size_t>(B) + 1, 0);
  for (int32_t b = 0; b < batch; ++b)
    toff[static_cast<size_t>(b) + 1] = toff[static_cast<size_t>(b)] + (opts->collect_trace ? hst[b].n_trace : 0);
  const int64_t trows = toff[static_cast<size_t>(batch)];
  const fl1_trace_row* all_tr = nullptr;
  bool packed_launch = false;
  if (trows > 0) {
    const size_t off_bytes = (sizeof(int64_t) * (static_cast<size_t>(B) + 1) + 255) / 256 * 256;
    char* tp = ctx->pinned_traces(off_bytes + sizeof(fl1_trace_row) * static_cast<size_t>(trows));
    std::copy(toff.begin(), toff.end(), reinterpret_cast<int64_t*>(tp));
    if (batch <= 4) {  // few signals: one async copy each straight into pinned memory
      for (int32_t b = 0; b < batch; ++b) {
        const int64_t rows = toff[static_cast<size_t>(b) + 1] - toff[static_cast<size_t>(b)];
        if (rows > 0)
          ck(cudaMemcpyAsync(tp + off_bytes + sizeof(fl1_trace_row) * static_cast<size_t>(toff[static_cast<size_t>(b)]),
                             base + o_tr + sizeof(fl1_trace_row) * static_cast<size_t>(b * cap),
                             sizeof(fl1_trace_row) * static_cast<size_t>(rows), cudaMemcpyDeviceToHost, stream),
             "trace download");
      }
    } else {
      char* tb = ctx->batch_scratch(2, off_bytes + sizeof(fl1_trace_row) * static_cast<size_t>(trows)).as<char>();
      ck(cudaMemcpyAsync(tb, tp, sizeof(int64_t) * (static_cast<size_t>(B) + 1), cudaMemcpyHostToDevice, stream),
         "trace offsets");
      ck(fl1::trace_pack_launch(reinterpret_cast<const fl1_trace_row*>(base + o_tr), cap,
                                reinterpret_cast<const int64_t*>(tb), batch,
                                reinterpret_cast<fl1_trace_row*>(tb + off_bytes), stream),
         "trace pack");
      ck(cudaMemcpyAsync(tp + off_bytes, tb + off_bytes, sizeof(fl1_trace_row) * static_cast<size_t>(trows),
                         cudaMemcpyDeviceToHost, stream),
         "trace download");
      packed_launch = true;
    }
    all_tr = reinterpret_cast<const fl1_trace_row*>(tp + off_bytes);
  }
  ck(cudaStreamSynchronize(stream), "download sync");
  hlog("downloaded");
  if (timeline) {
    std::vector<uint64_t> h(timeline->bytes / sizeof(uint64_t));
    ck(cudaMemcpy(h.data(), timeline->p, timeline->bytes, cudaMemcpyDeviceToHost), "timeline");
    if (FILE* f = std::fopen(tl_path, "wb")) {
      std::fwrite(h.data(), sizeof(uint64_t), h.size(), f);
      std::fclose(f);
    }
  }
  float batch_ms = 0.f, lockstep_ms = 0.f;
  ck(cudaEventElapsedTime(&batch_ms, ev0, ev1), "elapsed");
  ck(cudaEventElapsedTime(&lockstep_ms, ev0, evp), "elapsed");
  int32_t lk_steps = 0;
  int64_t lk_work[2] = {0, 0};
  if (use_prefix) {  // lockstep accounting (signal 0's profile): steps and contraction widths
    ck(cudaMemcpy(&lk_steps, d_steps, sizeof(lk_steps), cudaMemcpyDeviceToHost), "steps");
    ck(cudaMemcpy(lk_work, pp.work_out, sizeof(lk_work), cudaMemcpyDeviceToHost), "work");
  }
  if (const char* sp = std::getenv("FL1_SIGPROF_OUT"); sp && pp.sigprof) {
    double h[16];
    ck(cudaMemcpy(h, pp.sigprof, sizeof(h), cudaMemcpyDeviceToHost), "sigprof");
    if (FILE* f = std::fopen(sp, "w")) {
      for (double v : h) std::fprintf(f, "%g\n", v);
      std::fclose(f);
    }
  }
  if (pp.sk_trace) {
    std::vector<double> h(2 * 4 * 256 + 2 * 4 * 128 * 2);
    ck(cudaMemcpy(h.data(), pp.sk_trace, h.size() * sizeof(double), cudaMemcpyDeviceToHost), "sk trace");
    if (FILE* f = std::fopen("fl1_sk_trace.txt", "w")) {
      for (size_t i = 0; i < h.size(); i += 4) std::fprintf(f, "%.17g %.17g %.17g %.17g\n", h[i], h[i + 1], h[i + 2], h[i + 3]);
      std::fclose(f);
    }
  }
  if (step_log && d_steps) {
    int32_t steps = 0;
    ck(cudaMemcpy(&steps, d_steps, sizeof(steps), cudaMemcpyDeviceToHost), "steps");
    std::vector<double> lg(fl1::kStepLogW * static_cast<size_t>(std::min(steps, 4096)));
    if (!lg.empty()) ck(cudaMemcpy(lg.data(), step_log->p, lg.size() * sizeof(double), cudaMemcpyDeviceToHost), "log");
    // per step: n_act n_pow | %globaltimer at the step start, after the W barrier, after the
    // Corr barrier | (stream-K route) after the staging barrier, CTA 0 done with W, with
    // Corr, with its per-signal work (0 when not reached)
    if (FILE* f = std::fopen(std::getenv("FL1_STEP_LOG"), "w")) {
      for (size_t i = 0; i + fl1::kStepLogW <= lg.size(); i += fl1::kStepLogW) {
        for (int c = 0; c < 9; ++c) std::fprintf(f, c ? " %g" : "%g", lg[i + c]);
        std::fprintf(f, "\n");
      }
      std::fclose(f);
    }
  }
  for (int32_t b = 0; b < batch; ++b) {
    const EngineState& st = hst[b];
    if (!st.done) throw std::runtime_error("batched solve did not finish");
    const int32_t* ib = all_idx + offs[b];
    const double* xb = all_x + offs[b];
    auto res = std::make_unique<fl1_result>();
    const fl1_switch_event* sb = all_sw + static_cast<size_t>(b) * fl1::kMaxLevels;
    fill_result(*res, st, cfg, k, std::vector<int32_t>(ib, ib + st.S), xb,
                std::vector<fl1_switch_event>(sb, sb + st.n_switches));
    if (all_tr)
      res->trace.assign(all_tr + toff[static_cast<size_t>(b)], all_tr + toff[static_cast<size_t>(b) + 1]);
    res->device_ms = (st.end_ns - st.start_ns) * 1e-6;
    if (res->setup_ms < 0.0) res->setup_ms = 0.0;  // hand-off signals ran their setup in the lockstep launch
    res->batch_ms = batch_ms;
    res->launches = 0;  // one launch for the whole batch (fl1_result_info.kernel_launches of signal 0 = 1)
    if (b == 0) res->launches = (use_prefix ? 2 : 1) + (packed_launch ? 1 : 0);  // + the trace packing kernel
    if (b == 0 && use_prefix) {  // fl1_result_profile of signal 0 of a batched call (include/fl1cuda.h)
      res->prof[0] = lockstep_ms;
      res->prof[1] = static_cast<double>(lk_work[0]);
      res->prof[2] = static_cast<double>(lk_work[1]);
      res->prof[3] = static_cast<double>(lk_steps);
    }
    res->h2d = h2d_sig;
    res->d2h = static_cast<int64_t>(sizeof(EngineState)) + 12 * st.S +
               st.n_switches * static_cast<int64_t>(sizeof(fl1_switch_event)) +
               st.n_trace * static_cast<int64_t>(sizeof(fl1_trace_row));
    out[b] = res.release();
  }
  hlog("results");
}

// A single solve on a small, L2-resident dictionary is latency-bound: one
// thread-block cluster of 16 CTAs (cluster barriers instead of grid barriers) beats
// the full cooperative grid (measured c1: 1.21 vs 1.58 ms). Larger dictionaries
// need every SM's bandwidth. Observers, x_init and forced trace flushes keep the
// grid path; FL1_SINGLE_CLUSTER=0 disables the route.
constexpr int64_t kSingleClusterBytes = 16ll << 20;
constexpr int kSingleClusterSize = 16;
constexpr int64_t kSmallClusterBytes = 8ll << 20;
constexpr int kSmallClusterSize = 12;

void solve_single(fl1_seq* s, const double* y, bool y_device, double lambda, const fl1_switch_config* cfg,
                  const fl1_run_options* opts, fl1_result** out) {
  if (s && cfg && opts && out && !opts->observer && !opts->x_init && !std::getenv("FL1_TRACE_CAP") &&
      cluster_trace_fits(cfg, opts, 1)) {
    const char* e = std::getenv("FL1_SINGLE_CLUSTER");
    int64_t bytes = 0;
    for (const auto& l : s->lv) {
      const DictImpl& d = *l->dict;
      bytes += d.kind == fl1::kDense ? 8 * d.ld * d.k : 8 * 2 * static_cast<int64_t>(d.nterms) * d.m * d.q;
    }
    if (opts->exact_gram) bytes += 8 * s->lv.back()->dict->k * s->lv.back()->dict->k;
    int64_t limit = kSingleClusterBytes;
    if (const char* mb = std::getenv("FL1_SINGLE_CLUSTER_MB")) limit = std::atoll(mb) << 20;
    if (!(e && e[0] == '0') && bytes <= limit) {
      // up to 8 MiB, 12 CTAs: the on-chip power iteration's distributed-shared-memory
      // sums get cheaper with fewer ranks faster than the passes slow down (c1: 16 CTAs
      // 1.070 ms, 12 CTAs 1.039 ms, 8 CTAs 1.066 ms)
      int csize = bytes <= kSmallClusterBytes ? kSmallClusterSize : kSingleClusterSize;
      if (const char* cs = std::getenv("FL1_SINGLE_CLUSTER_SIZE")) csize = std::atoi(cs);
      solve_clusters(s, y, y_device, s->lv.back()->dict->n, &lambda, 1, cfg, opts, csize, out, false);
      return;
    }
  }
  do_solve(s, y, y_device, lambda, cfg, opts, out);
}


constexpr int32_t kTraceFallbackConcurrency = 8;

int solve_batched_impl(fl1_seq* s, const double* Y, bool y_device, int64_t ldy, const double* lambdas, int32_t batch,
                       const fl1_switch_config* cfg, const fl1_run_options* opts, int32_t concurrency,
                       fl1_result** out) {
  return guard([&] {
    if (!s || !Y || !lambdas || !out || batch < 0) throw std::invalid_argument("null argument");
    if (opts && opts->observer) throw std::invalid_argument("observers are not supported in batched solves");
    if (opts && opts->x_init) throw std::invalid_argument("x_init is per signal: use fl1_solve");
    const int64_t n = s->lv.back()->dict->n;
    if (ldy < n) throw std::invalid_argument("ldy must be >= N");
    fl1_ctx* ctx = s->lv.back()->dict->ctx;
    ctx->bind();
    for (int32_t b = 0; b < batch; ++b) out[b] = nullptr;
    if (concurrency <= 0 && cfg && opts && !cluster_trace_fits(cfg, opts, batch))
      concurrency = kTraceFallbackConcurrency;  // trace too large to reserve: grid solves that flush
    if (concurrency <= 0) {  // one launch, thread-block clusters as virtual grids
      const int csize = concurrency == 0 ? kDefaultClusterSize : -concurrency;
      try {
        solve_clusters(s, Y, y_device, ldy, lambdas, batch, cfg, opts, csize, out);
      } catch (...) {
        for (int32_t b = 0; b < batch; ++b) {
          delete out[b];
          out[b] = nullptr;
        }
        throw;
      }
      return;
    }
    int M = concurrency;
    M = std::max(1, std::min({M, ctx->sms, std::max<int>(batch, 1)}));
    const int grid_cap = std::max(1, ctx->sms / M);
    for (int32_t b = 0; b < batch; ++b) out[b] = nullptr;
    std::vector<std::thread> pool;
    std::mutex mu;
    std::string first_err;
    int first_code = FL1_OK;
    std::atomic<int32_t> next{0};
    for (int wkr = 0; wkr < M; ++wkr) {
      pool.emplace_back([&] {
        const int dev = ctx->device;
        cudaSetDevice(dev);
        while (true) {
          const int32_t b = next.fetch_add(1);
          if (b >= batch) break;
          const int st = guard([&] { do_solve(s, Y + static_cast<int64_t>(b) * ldy, y_device, lambdas[b], cfg, opts,
                                              &out[b], grid_cap); });
          if (st != FL1_OK) {
            std::lock_guard<std::mutex> g(mu);
            if (first_code == FL1_OK) {
              first_code = st;
              first_err = g_err;
            }
          }
        }
      });
    }
    for (auto& t : pool) t.join();
    if (first_code != FL1_OK) {
      for (int32_t b = 0; b < batch; ++b) {
        delete out[b];
        out[b] = nullptr;
      }
      if (first_code == FL1_EINVAL) throw std::invalid_argument(first_err);
      throw std::runtime_error(first_err);
    }
  });
}
}  // namespace

int fl1_solve(fl1_seq* s, const double* y, double lambda, const fl1_switch_config* cfg,
              const fl1_run_options* opts, fl1_result** out) {
  return guard([&] { solve_single(s, y, false, lambda, cfg, opts, out); });
}
int fl1_solve_device(fl1_seq* s, const double* y, double lambda, const fl1_switch_config* cfg,
                     const fl1_run_options* opts, fl1_result** out) {
  return guard([&] { solve_single(s, y, true, lambda, cfg, opts, out); });
}
int fl1_solve_batched(fl1_seq* s, const double* Y, int64_t ldy, const double* lambdas, int32_t batch,
                      const fl1_switch_config* cfg, const fl1_run_options* opts, int32_t concurrency,
                      fl1_result** out) {
  return solve_batched_impl(s, Y, false, ldy, lambdas, batch, cfg, opts, concurrency, out);
}
int fl1_solve_batched_device(fl1_seq* s, const double* Y, int64_t ldy, const double* lambdas, int32_t batch,
                             const fl1_switch_config* cfg, const fl1_run_options* opts, int32_t concurrency,
                             fl1_result** out) {
  return solve_batched_impl(s, Y, true, ldy, lambdas, batch, cfg, opts, concurrency, out);
}
int fl1_result_info_get(const fl1_result* r, fl1_result_info* o) {
  return guard([&] {
    *o = fl1_result_info{};
    o->k = r->k;
    o->converged = r->converged;
    o->gap_warning = r->gap_warning;
    o->final_gap = r->final_gap;
    o->iterations = r->iterations;
    o->total_flops = r->total_flops;
    o->n_trace = static_cast<int64_t>(r->trace.size());
    o->n_switches = static_cast<int64_t>(r->switches.size());
    o->n_final_active = static_cast<int64_t>(r->final_active.size());
    o->device_ms = r->device_ms;
    o->setup_ms = r->setup_ms;
    o->kernel_launches = r->launches;
    o->power_iterations = r->power_steps;
    o->h2d_bytes = r->h2d;
    o->d2h_bytes = r->d2h;
    o->batch_device_ms = r->batch_ms >= 0.0 ? r->batch_ms : r->device_ms;
  });
}
namespace {
void expand_x(const fl1_result& r, double* out) {  // finish (741-748): scatter to length K
  std::fill(out, out + r.k, 0.0);
  for (size_t q = 0; q < r.xv.size(); ++q) out[r.final_active[q]] = r.xv[q];
}
}  // namespace
int fl1_result_x(const fl1_result* r, double* out) {
  return guard([&] { expand_x(*r, out); });
}
int fl1_result_trace(const fl1_result* r, fl1_trace_row* out) {
  return guard([&] { std::copy(r->trace.begin(), r->trace.end(), out); });
}
int fl1_result_switches(const fl1_result* r, fl1_switch_event* out) {
  return guard([&] { std::copy(r->switches.begin(), r->switches.end(), out); });
}
int fl1_result_final_active(const fl1_result* r, int32_t* out) {
  return guard([&] { std::copy(r->final_active.begin(), r->final_active.end(), out); });
}
int fl1_result_profile(const fl1_result* r, double* out) {
  return guard([&] { std::copy(r->prof, r->prof + 14, out); });
}
int fl1_results_collect(fl1_result* const* rs, int32_t count, fl1_result_info* infos, double* x, double* profiles) {
  for (int32_t i = 0; i < count; ++i) {
    const int st = fl1_result_info_get(rs[i], infos + i);
    if (st != FL1_OK) return st;
  }
  return guard([&] {
    for (int32_t i = 0; i < count; ++i) {
      const fl1_result& r = *rs[i];
      if (x) expand_x(r, x + static_cast<int64_t>(i) * r.k);
      if (profiles) std::copy(r.prof, r.prof + 14, profiles + static_cast<int64_t>(i) * 14);
    }
  });
}
int fl1_results_tables(fl1_result* const* rs, int32_t count, fl1_trace_row* traces, fl1_switch_event* switches,
                       int32_t* final_active) {
  return guard([&] {
    for (int32_t i = 0; i < count; ++i) {
      const fl1_result& r = *rs[i];
      if (traces) traces = std::copy(r.trace.begin(), r.trace.end(), traces);
      if (switches) switches = std::copy(r.switches.begin(), r.switches.end(), switches);
      if (final_active) final_active = std::copy(r.final_active.begin(), r.final_active.end(), final_active);
    }
  });
}
void fl1_result_free(fl1_result* r) { delete r; }

int fl1_lambda_max(fl1_dict* d, const double* y, double* out) {  // screening.cpp:9-11
  return guard([&] {
    std::vector<double> c(static_cast<size_t>(d->d->k));
    run_utility(*d->d, fl1::kModeAdjoint, y, c.data(), c.size());
    double m = 0.0;
    for (double e : c) m = std::max(m, std::abs(e));
    *out = m;
  });
}
int fl1_gram_create(fl1_dict* dh, fl1_dict** out) {  // bench.cpp:190-197
  return guard([&] {
    if (!dh || !out) throw std::invalid_argument("null argument");
    const DictImpl& d = *dh->d;
    if (d.kind != fl1::kDense) throw std::invalid_argument("exact_gram needs a dense dictionary");
    d.ctx->bind();
    auto g = std::make_shared<DictImpl>();
    g->ctx = d.ctx;
    g->kind = fl1::kDense;
    g->n = d.k;
    g->k = d.k;
    g->ld = even_ld(d.k);
    g->a = std::make_unique<DevBuf>(static_cast<size_t>(g->ld) * static_cast<size_t>(d.k) * sizeof(double));
    ck(cudaMemset(g->a->p, 0, g->a->bytes), "memset");
    ck(fl1::gram_launch(d.a->as<double>(), d.ld, d.k, g->a->as<double>(), g->ld, d.ctx->device, nullptr), "gram");
    ck(cudaDeviceSynchronize(), "gram sync");
    // column norms of G (LinearOp::atom_norms2 of the K x K operator), on the device
    DevBuf nrm(static_cast<size_t>(d.k) * sizeof(double));
    ck(fl1::colnorm_launch(g->a->as<double>(), d.k, g->ld, nrm.as<double>(), nullptr), "gram norms");
    g->norms.resize(static_cast<size_t>(d.k));
    ck(cudaMemcpy(g->norms.data(), nrm.p, nrm.bytes, cudaMemcpyDeviceToHost), "gram norms download");
    *out = new fl1_dict{g};
  });
}

int fl1_rng_normals(uint64_t seed, int64_t count, double* out) {
  return guard([&] {
    if (count < 0 || (count > 0 && !out)) throw std::invalid_argument("bad output");
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> gauss(0.0, 1.0);
    for (int64_t i = 0; i < count; ++i) out[i] = gauss(rng);
  });
}

namespace {
int64_t require_perfect_square(int64_t v, const char* what) {  // dictionary.cpp:19-33
  auto r = static_cast<int64_t>(std::llround(std::sqrt(static_cast<double>(v))));
  while (r * r > v) --r;
  while ((r + 1) * (r + 1) <= v) ++r;
  if (r * r != v) throw std::invalid_argument(std::string(what) + " must be a perfect square, got " + std::to_string(v));
  return r;
}
}  // namespace

// build_sukro_sequence (dictionary.cpp:281-357) with truncated_svd (253-279), on the
// device (csrc/sukro_build.cu + the DMMA gemm_tn of batched.cu). The dense dictionary
// never leaves HBM; only the Gaussian probes go up (the reference's mt19937_64 stream)
// and the factors / per-level vectors come down.
int fl1_build_sukro_sequence(fl1_dict* dh, const int32_t* ranks, int32_t n_ranks, double* left, double* right,
                             double* eps, double* approx_norms, double* rc, double* op_err) {
  return guard([&] {
    if (!dh || (n_ranks > 0 && !ranks)) throw std::invalid_argument("null argument");
    DictImpl& d = *dh->d;
    if (d.kind != fl1::kDense) throw std::invalid_argument("build_sukro_sequence needs a dense dictionary");
    const int64_t n = d.n, k = d.k;
    const int64_t m = require_perfect_square(n, "N");
    const int64_t q = require_perfect_square(k, "K");
    if (n_ranks < 1) throw std::invalid_argument("need at least one rank");
    for (int32_t i = 0; i < n_ranks; ++i)
      if (ranks[i] < 1 || (i > 0 && ranks[i] <= ranks[i - 1]))
        throw std::invalid_argument("ranks must be positive and strictly increasing");
    const int T = ranks[n_ranks - 1];
    const int64_t M = m * q;
    if (T > M) throw std::invalid_argument("rank exceeds rearranged dimension");
    if (!left || !right || !eps || !approx_norms || !rc || !op_err) throw std::invalid_argument("null argument");
    const uint64_t dense_flops = static_cast<uint64_t>(n) * static_cast<uint64_t>(k);  // matvec_flops
    for (int32_t i = 0; i < n_ranks; ++i) {
      const uint64_t mv = static_cast<uint64_t>(ranks[i]) * static_cast<uint64_t>(m * k + q * n);
      if (mv >= dense_flops)
        throw std::invalid_argument("rank " + std::to_string(ranks[i]) + " gives relative complexity >= 1");
      rc[i] = static_cast<double>(mv) / static_cast<double>(dense_flops);
    }
    const int p = static_cast<int>(std::min<int64_t>(T + 8, M));
    if (p > fl1::sukro_max_probe())
      throw std::invalid_argument("truncated_svd: rank + 8 probes exceed " + std::to_string(fl1::sukro_max_probe()) +
                                  " (device construction limit)");
    if (n_ranks > fl1::sukro_max_snapshots()) throw std::invalid_argument("too many ranks");
    d.ctx->bind();
    const int dev = d.ctx->device;
    const int64_t ldr = (M + 1) / 2 * 2;
    const size_t mat = static_cast<size_t>(ldr) * static_cast<size_t>(M), pan = static_cast<size_t>(ldr) * p;
    DevBuf R(mat * 8), Rt(mat * 8), Om(pan * 8), Y(pan * 8), Z(pan * 8), Wk(pan * 8), Qm(pan * 8), Q2(pan * 8);
    DevBuf Rf(64 * 64 * 8), R2(64 * 64 * 8), S(64 * 8), Wsv(64 * 64 * 8), Vsv(64 * 64 * 8);
    const size_t work_elems = 16 * pan;
    DevBuf work(work_elems * 8);
    DevBuf L(static_cast<size_t>(T) * M * 8), Rr(static_cast<size_t>(T) * M * 8);
    DevBuf E(static_cast<size_t>(n_ranks) * k * 8), Ap(static_cast<size_t>(n_ranks) * k * 8), rk(64 * 4);
    cudaStream_t st = nullptr;
    for (DevBuf* b : {&R, &Rt, &Om, &Y, &Z, &Wk, &Qm, &Q2}) ck(cudaMemsetAsync(b->p, 0, b->bytes, st), "memset");
    {  // Omega (cols x p, column-major): the reference's stream, omega(i, j) in j-major order
      std::vector<double> om(static_cast<size_t>(M) * p);
      std::mt19937_64 rng(0x5eedf00dULL);
      std::normal_distribution<double> gauss(0.0, 1.0);
      for (auto& v : om) v = gauss(rng);
      ck(cudaMemcpy2D(Om.p, ldr * 8, om.data(), M * 8, M * 8, p, cudaMemcpyHostToDevice), "probe upload");
    }
    ck(fl1::rearrange_launch(d.a->as<double>(), d.ld, m, q, R.as<double>(), Rt.as<double>(), ldr, st), "rearrange");
    auto gemm = [&](const DevBuf& X, const DevBuf& Yop, DevBuf& C) {  // C = X^T Yop, all mq x . with ld ldr
      ck(fl1::gemm_tn_launch(X.as<double>(), ldr, M, Yop.as<double>(), ldr, p, M, C.as<double>(), ldr,
                             work.as<double>(), work_elems, dev, st),
         "gemm_tn");
    };
    auto orth = [&](const DevBuf& Yin, DevBuf& Qout, DevBuf& Rout) {
      ck(cudaMemcpy2DAsync(Wk.p, ldr * 8, Yin.p, ldr * 8, M * 8, p, cudaMemcpyDeviceToDevice, st), "panel copy");
      ck(fl1::householder_qr_launch(Wk.as<double>(), M, p, ldr, Qout.as<double>(), ldr, Rout.as<double>(), st), "qr");
    };
    gemm(Rt, Om, Y);  // Y = R Omega
    for (int it = 0; it < 6; ++it) {
      orth(Y, Qm, Rf);
      gemm(R, Qm, Z);  // Z = R^T Q
      gemm(Rt, Z, Y);  // Y = R Z
    }
    orth(Y, Qm, Rf);
    gemm(R, Qm, Z);    // bt = R^T Q (cols x p)
    orth(Z, Q2, R2);   // bt = Q2 R2
    ck(fl1::jacobi_svd_launch(R2.as<double>(), p, S.as<double>(), Wsv.as<double>(), Vsv.as<double>(), st), "svd");
    // svd(bt): U = Q2 W, V = Vsv; u = Q V(:, :T), v = U(:, :T); terms scaled by sqrt(s_t)
    ck(fl1::small_gemm_launch(Qm.as<double>(), ldr, M, p, Vsv.as<double>(), S.as<double>(), T, L.as<double>(), M, st),
       "left factors");
    ck(fl1::small_gemm_launch(Q2.as<double>(), ldr, M, p, Wsv.as<double>(), S.as<double>(), T, Rr.as<double>(), M, st),
       "right factors");
    ck(cudaMemcpyAsync(rk.p, ranks, sizeof(int32_t) * n_ranks, cudaMemcpyHostToDevice, st), "ranks");
    ck(fl1::residual_norms_launch(d.a->as<double>(), d.ld, m, q, T, L.as<double>(), Rr.as<double>(), M,
                                  rk.as<int>(), n_ranks, E.as<double>(), Ap.as<double>(), st),
       "residual norms");
    ck(cudaMemcpyAsync(left, L.p, L.bytes, cudaMemcpyDeviceToHost, st), "left download");
    ck(cudaMemcpyAsync(right, Rr.p, Rr.bytes, cudaMemcpyDeviceToHost, st), "right download");
    ck(cudaMemcpyAsync(eps, E.p, E.bytes, cudaMemcpyDeviceToHost, st), "eps download");
    ck(cudaMemcpyAsync(approx_norms, Ap.p, Ap.bytes, cudaMemcpyDeviceToHost, st), "norms download");
    ck(cudaStreamSynchronize(st), "sukro build");
    // running max finer -> coarser (dictionary.cpp:344-349), operator_error_bound = max
    for (int32_t i = n_ranks - 1; i > 0; --i)
      for (int64_t j = 0; j < k; ++j) {
        double& c = eps[static_cast<int64_t>(i - 1) * k + j];
        c = std::max(c, eps[static_cast<int64_t>(i) * k + j]);
      }
    for (int32_t i = 0; i < n_ranks; ++i)
      op_err[i] = *std::max_element(eps + static_cast<int64_t>(i) * k, eps + static_cast<int64_t>(i + 1) * k);
  });
}

int fl1_draw_signal(fl1_dict* dh, double p, uint64_t seed, int32_t trial, double* y, double* x) {  // bench.cpp:141-166
  return guard([&] {
    if (!dh || !y || !x) throw std::invalid_argument("null argument");
    if (!(p > 0.0 && p <= 1.0)) throw std::invalid_argument("bernoulli-p must lie in (0, 1]");
    DictImpl& d = *dh->d;
    uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (static_cast<uint64_t>(trial) + 1);  // mix_seed (bench.cpp:45-50)
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    std::mt19937_64 rng(z ^ (z >> 31));
    std::bernoulli_distribution coin(p);
    std::normal_distribution<double> gauss(0.0, 1.0);
    std::vector<double> yy(static_cast<size_t>(d.n));
    for (int attempt = 0;; ++attempt) {
      if (attempt > 100000) throw std::runtime_error("signal draw kept failing");
      std::fill(x, x + d.k, 0.0);
      bool any = false;
      for (int64_t j = 0; j < d.k; ++j) {
        if (coin(rng)) {
          x[j] = gauss(rng);
          any = true;
        }
      }
      if (!any) continue;
      std::vector<double> out(static_cast<size_t>(even_ld(d.n)), 0.0);
      run_utility(d, fl1::kModeApply, x, out.data(), static_cast<size_t>(d.n));
      double nrm = 0.0;
      for (int64_t i = 0; i < d.n; ++i) nrm += out[static_cast<size_t>(i)] * out[static_cast<size_t>(i)];
      nrm = std::sqrt(nrm);
      if (nrm <= 1e-12) continue;
      for (int64_t j = 0; j < d.k; ++j) x[j] /= nrm;
      for (int64_t i = 0; i < d.n; ++i) y[i] = out[static_cast<size_t>(i)] / nrm;
      return;
    }
  });
}

int fl1_lipschitz_bound(fl1_dict* d, double* out) {  // solver.cpp:108-114
  return guard([&] {
    const EngineState st = run_utility(*d->d, fl1::kModePower, nullptr, nullptr, 0);
    *out = st.power_est * 1.05;
  });
}
int fl1_screen_precomputed(fl1_ctx* ctx, int64_t n, const double* dots, const double* eps, const double* en,
                           const double* an, double cn, double r, int32_t* kept, int64_t* n_kept,
                           int64_t* lookahead) {
  return guard([&] {
    ctx->bind();
    const size_t b = static_cast<size_t>(std::max<int64_t>(n, 1)) * sizeof(double);
    DevBuf dd(b), de(b), den(b), dan(b), keep(b), look(b);
    if (n > 0) {
      ck(cudaMemcpy(dd.p, dots, static_cast<size_t>(n) * 8, cudaMemcpyHostToDevice), "up");
      ck(cudaMemcpy(de.p, eps, static_cast<size_t>(n) * 8, cudaMemcpyHostToDevice), "up");
      ck(cudaMemcpy(den.p, en, static_cast<size_t>(n) * 8, cudaMemcpyHostToDevice), "up");
      ck(cudaMemcpy(dan.p, an, static_cast<size_t>(n) * 8, cudaMemcpyHostToDevice), "up");
      ck(fl1::screen_kernel_launch(n, dd.as<double>(), de.as<double>(), den.as<double>(), dan.as<double>(), cn, r,
                                   keep.as<int8_t>(), look.as<int8_t>(), nullptr),
         "screen kernel");
    }
    std::vector<int8_t> hk(static_cast<size_t>(n)), hl(static_cast<size_t>(n));
    if (n > 0) {
      ck(cudaMemcpy(hk.data(), keep.p, static_cast<size_t>(n), cudaMemcpyDeviceToHost), "down");
      ck(cudaMemcpy(hl.data(), look.p, static_cast<size_t>(n), cudaMemcpyDeviceToHost), "down");
    }
    int64_t w = 0, la = 0;
    for (int64_t j = 0; j < n; ++j) {
      if (hk[static_cast<size_t>(j)]) kept[w++] = static_cast<int32_t>(j);
      la += hl[static_cast<size_t>(j)];
    }
    *n_kept = w;
    *lookahead = la;
  });
}

// ---- scalar formulas (host)
double fl1_soft_threshold(double z, double u) {
  const double mag = std::abs(z) - u;
  if (mag <= 0.0) return 0.0;
  return z > 0.0 ? mag : -mag;
}
double fl1_gap_ratio(double gt, double gp) {
  if (gp <= 1e-15) return 0.0;
  return std::min(std::max(gt / gp, 0.0), 1.0);
}
int fl1_switch_dictionary(int i, int last, double gamma, double gthr, int64_t la, double rc, int64_t ta) {
  if (i >= last) return last;
  if (static_cast<double>(la) <= rc * static_cast<double>(ta)) return last;
  if (gamma <= gthr) return i + 1;
  return i;
}
uint64_t fl1_flops_plain(uint64_t k, uint64_t n, uint64_t z) { return (k + z) * n + 4 * k + n; }
uint64_t fl1_flops_screened(uint64_t a, uint64_t n, uint64_t z) { return (a + z) * n + 6 * a + 5 * n; }
uint64_t fl1_flops_stable(uint64_t mv, uint64_t n, uint64_t a, uint64_t z) { return mv + z * n + 8 * a + 7 * n; }
uint64_t fl1_recompute_flops(const fl1_trace_row* trace, int64_t n_rows, const fl1_seq* s, int32_t variant,
                             int64_t n, int64_t k, int32_t* rows_match) {
  const auto un = static_cast<uint64_t>(n), uk = static_cast<uint64_t>(k);
  const int last = static_cast<int>(s->lv.size()) - 1;
  uint64_t total = 0;
  bool all = true;
  for (int64_t r = 0; r < n_rows; ++r) {
    const fl1_trace_row& row = trace[r];
    const auto a = static_cast<uint64_t>(row.active_size), z = static_cast<uint64_t>(row.x_nnz);
    if (variant == FL1_PLAIN) total += fl1_flops_plain(uk, un, z);
    else if (variant == FL1_SCREENED) total += fl1_flops_screened(a, un, z);
    else if (row.dict_index < last)
      total += fl1_flops_stable(s->lv[static_cast<size_t>(row.dict_index)]->dict->matvec_flops(), un, a, z);
    else total += fl1_flops_screened(a, un, z);
    all = all && total == row.flops_cum;
  }
  if (rows_match) *rows_match = all ? 1 : 0;
  return total;
}
double fl1_stable_gap_delta(double rn, double e, double x1) { return rn * e * x1 + 0.5 * e * e * x1 * x1; }
double fl1_sphere_test(double d, double an, double r) { return d + r * an; }
double fl1_stable_zone_test(double d, double eps, double cn, double en, double r) { return d + eps * cn + r * en; }
double fl1_stable_ball_test(double d, double eps, double cn, double an, double r) {
  return d + eps * cn + r * an + r * eps;
}

}  // extern "C"
