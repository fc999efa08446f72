// sukro_build.cu — build_sukro_sequence (dictionary.cpp:281-357) on the device.
//
// The reference approximates a dense N x K dictionary (N = m^2, K = q^2) by sums of
// Kronecker products: the rearrangement R = rearrange(A) (dictionary.cpp:37-45) maps
// every Kronecker term B (x) C of A to the rank-one vec(B) vec(C)^T of R, so a rank-r
// truncated SVD of R gives the r-term approximations. truncated_svd
// (dictionary.cpp:253-279) is a randomized range finder: p = rank + 8 Gaussian probes
// (mt19937_64(0x5eedf00d), drawn on the host exactly as the reference does), six
// subspace iterations Y <- R (R^T orth(Y)) with Householder QR, then the SVD of the
// small projected matrix. Then the per-level residual norms eps_j = ||a_j - a~_j|| of
// the running truncation (running max finer -> coarser) and the approximate atom norms.
//
// Kernels (all fixed-order, run to run reproducible):
//   rearrange_kernel      A -> R and R^T (one HBM pass; both layouts feed the tensor-core
//                         products with the contraction dimension contiguous)
//   gemm_tn (batched.cu)  the tall-skinny products R^T Q, R Z, R Omega on DMMA tiles
//   householder_qr_kernel thin QR of an M x p panel (one CTA; Eigen::HouseholderQR's
//                         reflector convention, beta = -sign(alpha) ||x||), Q formed by
//                         backward accumulation
//   jacobi_svd_kernel     SVD of the p x p triangular factor (one-sided Jacobi, round-robin
//                         pair order, one warp per pair), singular values descending
//   small_gemm_kernel     u = Q V(:, :r) sqrt(s), v = Q2 W(:, :r) sqrt(s) (the terms)
//   residual_norms_kernel one streaming pass over A: per column, the residual after each
//                         term (residual -= left_t(i, j) right_t, dictionary.cpp:330-333)
//                         and its norm at every requested rank, plus ||a_j - residual_j||
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

namespace fl1 {

constexpr int kMaxProbe = 64;     // p = rank + 8 <= 64 (the small SVD lives in shared memory)
constexpr int kMaxSnapshots = 16; // requested ranks per call
constexpr unsigned kFull = 0xffffffffu;

// R(i + j m, rr + s m) = A(i m + rr, j q + s); R and R^T are mq x mq with leading
// dimension ldr (even, zero padded).
__global__ void rearrange_kernel(const double* __restrict__ a, int64_t lda, int64_t m, int64_t q,
                                 double* __restrict__ R, double* __restrict__ Rt, int64_t ldr) {
  const int64_t n = m * m, k = q * q;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n * k;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t col = e / n, row = e - col * n;
    const int64_t i = row / m, rr = row - i * m, j = col / q, s = col - j * q;
    const double v = a[col * lda + row];
    const int64_t ri = i + j * m, ci = rr + s * m;
    R[ci * ldr + ri] = v;
    Rt[ri * ldr + ci] = v;
  }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// Thin Householder QR of the M x p panel W (column-major, ld), in place: R in the upper
// triangle, the essential parts of the reflectors below the diagonal; Q (M x p, ldq)
// formed by accumulating the reflectors backwards on the first p identity columns.
// One CTA of 1024 threads: column norms by block reduction, the reflector's dot
// products and rank-one updates by one warp per column.
__global__ void __launch_bounds__(1024, 1) householder_qr_kernel(double* __restrict__ W, int64_t M, int p, int64_t ld,
                                                                 double* __restrict__ Q, int64_t ldq,
                                                                 double* __restrict__ Rf) {
  __shared__ double tau[kMaxProbe], wdot[kMaxProbe], red[32];
  __shared__ double s_scale;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int k = 0; k < p; ++k) {
    double* x = W + static_cast<int64_t>(k) * ld;
    double part = 0.0;
    for (int64_t i = k + 1 + tid; i < M; i += blockDim.x) part += x[i] * x[i];
    part = warp_sum(part);
    if (lane == 0) red[warp] = part;
    __syncthreads();
    if (tid == 0) {
      double tail = 0.0;
      for (int w = 0; w < nw; ++w) tail += red[w];
      const double alpha = x[k];
      if (tail <= 2.2250738585072014e-308) {  // makeHouseholder: tau = 0, beta = alpha
        tau[k] = 0.0;
        s_scale = 0.0;
      } else {
        double beta = sqrt(alpha * alpha + tail);
        if (alpha >= 0.0) beta = -beta;
        tau[k] = (beta - alpha) / beta;
        s_scale = 1.0 / (alpha - beta);
        x[k] = beta;
      }
    }
    __syncthreads();
    const double sc = s_scale;
    if (sc == 0.0) {
      for (int64_t i = k + 1 + tid; i < M; i += blockDim.x) x[i] = 0.0;
    } else {
      for (int64_t i = k + 1 + tid; i < M; i += blockDim.x) x[i] *= sc;  // essential part of v (v_k = 1)
    }
    __syncthreads();
    const double tk = tau[k];
    if (tk != 0.0) {
      // H = I - tau v v^T on the trailing columns c > k: w_c = y_kc + sum_{i>k} v_i y_ic
      for (int c = k + 1 + warp; c < p; c += nw) {
        const double* y = W + static_cast<int64_t>(c) * ld;
        double d = 0.0;
        for (int64_t i = k + 1 + lane; i < M; i += 32) d += x[i] * y[i];
        d = warp_sum(d);
        if (lane == 0) wdot[c] = y[k] + d;
      }
      __syncthreads();
      for (int c = k + 1 + warp; c < p; c += nw) {
        double* y = W + static_cast<int64_t>(c) * ld;
        const double f = tk * wdot[c];
        if (lane == 0) y[k] -= f;
        for (int64_t i = k + 1 + lane; i < M; i += 32) y[i] -= f * x[i];
      }
    }
    __syncthreads();
  }
  // R (p x p, column-major)
  for (int e = tid; e < p * p; e += blockDim.x) {
    const int c = e / p, r = e - c * p;
    Rf[e] = r <= c ? W[static_cast<int64_t>(c) * ld + r] : 0.0;
  }
  // Q = H_0 H_1 ... H_{p-1} [I_p; 0]
  for (int c = warp; c < p; c += nw) {
    double* qc = Q + static_cast<int64_t>(c) * ldq;
    for (int64_t i = lane; i < M; i += 32) qc[i] = i == c ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int k = p - 1; k >= 0; --k) {
    const double tk = tau[k];
    if (tk == 0.0) continue;
    const double* v = W + static_cast<int64_t>(k) * ld;
    for (int c = k + warp; c < p; c += nw) {
      double* qc = Q + static_cast<int64_t>(c) * ldq;
      double d = 0.0;
      for (int64_t i = k + 1 + lane; i < M; i += 32) d += v[i] * qc[i];
      d = warp_sum(d) + qc[k];
      const double f = tk * d;
      if (lane == 0) qc[k] -= f;
      for (int64_t i = k + 1 + lane; i < M; i += 32) qc[i] -= f * v[i];
    }
    __syncthreads();
  }
}

// SVD of the p x p matrix Rf (column-major): Rf V = W diag(S) by one-sided Jacobi
// rotations (Hestenes) on the columns; round-robin pair order, one warp per pair, sweeps
// until no pair needs a rotation. Outputs sorted by descending singular value: S (p),
// W (p x p left vectors), V (p x p right vectors).
__global__ void __launch_bounds__(1024, 1) jacobi_svd_kernel(const double* __restrict__ Rf, int p,
                                                             double* __restrict__ S, double* __restrict__ Wout,
                                                             double* __restrict__ Vout) {
  extern __shared__ double jsm[];
  double* A = jsm;      // p x p
  double* V = jsm + p * p;
  __shared__ int order[kMaxProbe + 1], perm[kMaxProbe];
  __shared__ double nrm[kMaxProbe];
  __shared__ int any_rot;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int e = tid; e < p * p; e += blockDim.x) {
    A[e] = Rf[e];
    V[e] = (e / p) == (e % p) ? 1.0 : 0.0;
  }
  const int pe = p + (p & 1);  // round-robin over an even number of slots (slot p = bye)
  if (tid < pe) order[tid] = tid;
  __syncthreads();
  for (int sweep = 0; sweep < 100; ++sweep) {
    if (tid == 0) any_rot = 0;
    __syncthreads();
    for (int round = 0; round < pe - 1; ++round) {
      for (int pr = warp; pr < pe / 2; pr += nw) {
        int a = order[pr], b = order[pe - 1 - pr];
        if (a >= p || b >= p) continue;
        if (a > b) {
          const int t = a;
          a = b;
          b = t;
        }
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int r = lane; r < p; r += 32) {
          const double x = A[a * p + r], y = A[b * p + r];
          al += x * x;
          be += y * y;
          ga += x * y;
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum(ga);
        if (ga != 0.0 && fabs(ga) > 1e-15 * sqrt(al * be)) {
          const double zeta = (be - al) / (2.0 * ga);
          const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
          for (int r = lane; r < p; r += 32) {
            const double x = A[a * p + r], y = A[b * p + r];
            A[a * p + r] = c * x - s * y;
            A[b * p + r] = s * x + c * y;
            const double vx = V[a * p + r], vy = V[b * p + r];
            V[a * p + r] = c * vx - s * vy;
            V[b * p + r] = s * vx + c * vy;
          }
          if (lane == 0) any_rot = 1;
        }
      }
      __syncthreads();
      if (tid == 0) {  // rotate the slots, slot 0 fixed
        const int last = order[pe - 1];
        for (int i = pe - 1; i > 1; --i) order[i] = order[i - 1];
        order[1] = last;
      }
      __syncthreads();
    }
    if (!any_rot) break;
    __syncthreads();
  }
  for (int c = warp; c < p; c += nw) {
    double s = 0.0;
    for (int r = lane; r < p; r += 32) s += A[c * p + r] * A[c * p + r];
    s = warp_sum(s);
    if (lane == 0) nrm[c] = sqrt(s);
  }
  __syncthreads();
  if (tid == 0) {  // stable sort by descending singular value
    for (int i = 0; i < p; ++i) perm[i] = i;
    for (int i = 1; i < p; ++i) {
      const int v = perm[i];
      int j = i - 1;
      while (j >= 0 && nrm[perm[j]] < nrm[v]) {
        perm[j + 1] = perm[j];
        --j;
      }
      perm[j + 1] = v;
    }
  }
  __syncthreads();
  for (int e = tid; e < p * p; e += blockDim.x) {
    const int c = e / p, r = e - c * p, src = perm[c];
    const double sv = nrm[src];
    Wout[e] = sv > 0.0 ? A[src * p + r] / sv : (r == c ? 1.0 : 0.0);
    Vout[e] = V[src * p + r];
  }
  if (tid < p) S[tid] = nrm[perm[tid]];
}

// out(i, t) = (sum_c A(i, c) B(c, t)) * sqrt(max(S[t], 0)), t < r; A is M x p (lda),
// B is p x p (column-major)
__global__ void small_gemm_kernel(const double* __restrict__ A, int64_t lda, int64_t M, int p,
                                  const double* __restrict__ B, const double* __restrict__ S, int r,
                                  double* __restrict__ out, int64_t ldo) {
  __shared__ double Bs[kMaxProbe * kMaxProbe];
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) Bs[e] = B[e];
  __syncthreads();
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < M;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    for (int t = 0; t < r; ++t) {
      double s = 0.0;
      for (int c = 0; c < p; ++c) s += A[c * lda + i] * Bs[t * p + c];
      out[t * ldo + i] = s * sqrt(fmax(S[t], 0.0));
    }
  }
}

// One warp per atom j = jj * q + s (A column-major, lda): left_t(i, jj) and right_t(rr, s)
// for every term t staged in shared memory; element (i m + rr) of the residual is
// a - sum_t left_t(i, jj) right_t(rr, s), subtracted term by term as the reference does.
// At every requested rank ranks[l] the residual's norm (eps) and ||a - residual|| (the
// approximate atom norm) are taken: eps[l * K + j], app[l * K + j].
__global__ void __launch_bounds__(256) residual_norms_kernel(const double* __restrict__ a, int64_t lda, int64_t m,
                                                              int64_t q, int T, const double* __restrict__ left,
                                                              const double* __restrict__ right, int64_t ldt,
                                                              const int* __restrict__ ranks, int n_ranks,
                                                              double* __restrict__ eps, double* __restrict__ app,
                                                              int smem_ok) {
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int64_t N = m * m, K = q * q;
  const bool staged = smem_ok != 0;  // else the factors are read from global memory (L1 / L2)
  double* lsh = smem + static_cast<int64_t>(warp) * 2 * T * m;  // [t][i] left column jj, then [t][rr] right col s
  double* rsh = lsh + static_cast<int64_t>(T) * m;
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * nw + warp; j < K; j += static_cast<int64_t>(gridDim.x) * nw) {
    const int64_t jj = j / q, s = j - jj * q;
    // left_t is m x q column-major: (i, jj); right_t (rr, s); stride between terms
    const double* lg = left + jj * m;
    const double* rg = right + s * m;
    const int64_t ls = staged ? m : ldt;
    if (staged) {
      for (int64_t e = lane; e < static_cast<int64_t>(T) * m; e += 32) {
        const int64_t t = e / m, i = e - t * m;
        lsh[e] = lg[t * ldt + i];
        rsh[e] = rg[t * ldt + i];
      }
      __syncwarp();
    }
    const double* lp = staged ? lsh : lg;
    const double* rp = staged ? rsh : rg;
    double e2[kMaxSnapshots], a2[kMaxSnapshots];
#pragma unroll
    for (int l = 0; l < kMaxSnapshots; ++l) e2[l] = a2[l] = 0.0;
    const double* col = a + j * lda;
    for (int64_t row = lane; row < N; row += 32) {
      const int64_t i = row / m, rr = row - i * m;
      const double av = col[row];
      double r = av;
      int l = 0;
      for (int t = 0; t < T && l < n_ranks; ++t) {
        r = __dsub_rn(r, __dmul_rn(lp[t * ls + i], rp[t * ls + rr]));
        if (t + 1 == ranks[l]) {
#pragma unroll
          for (int z = 0; z < kMaxSnapshots; ++z)
            if (z == l) {
              e2[z] += r * r;
              const double d = av - r;
              a2[z] += d * d;
            }
          ++l;
        }
      }
    }
#pragma unroll
    for (int l = 0; l < kMaxSnapshots; ++l) {
      if (l < n_ranks) {
        const double se = warp_sum(e2[l]), sa = warp_sum(a2[l]);
        if (lane == 0) {
          eps[l * K + j] = sqrt(se);
          app[l * K + j] = sqrt(sa);
        }
      }
    }
    __syncwarp();
  }
}

cudaError_t rearrange_launch(const double* a, int64_t lda, int64_t m, int64_t q, double* R, double* Rt, int64_t ldr,
                             cudaStream_t stream) {
  const int64_t n = m * m * q * q;
  rearrange_kernel<<<static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 8192)), 256, 0, stream>>>(a, lda, m, q,
                                                                                                       R, Rt, ldr);
  return cudaGetLastError();
}

cudaError_t householder_qr_launch(double* W, int64_t M, int p, int64_t ld, double* Q, int64_t ldq, double* Rf,
                                  cudaStream_t stream) {
  if (p > kMaxProbe) return cudaErrorInvalidValue;
  householder_qr_kernel<<<1, 1024, 0, stream>>>(W, M, p, ld, Q, ldq, Rf);
  return cudaGetLastError();
}

cudaError_t jacobi_svd_launch(const double* Rf, int p, double* S, double* W, double* V, cudaStream_t stream) {
  if (p > kMaxProbe) return cudaErrorInvalidValue;
  const size_t smem = static_cast<size_t>(2 * p * p) * sizeof(double);
  const cudaError_t e =
      cudaFuncSetAttribute(jacobi_svd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  jacobi_svd_kernel<<<1, 1024, smem, stream>>>(Rf, p, S, W, V);
  return cudaGetLastError();
}

cudaError_t small_gemm_launch(const double* A, int64_t lda, int64_t M, int p, const double* B, const double* S, int r,
                              double* out, int64_t ldo, cudaStream_t stream) {
  if (p > kMaxProbe) return cudaErrorInvalidValue;
  small_gemm_kernel<<<static_cast<unsigned>(std::min<int64_t>((M + 255) / 256, 1024)), 256, 0, stream>>>(
      A, lda, M, p, B, S, r, out, ldo);
  return cudaGetLastError();
}

cudaError_t residual_norms_launch(const double* a, int64_t lda, int64_t m, int64_t q, int T, const double* left,
                                  const double* right, int64_t ldt, const int* ranks, int n_ranks, double* eps,
                                  double* app, cudaStream_t stream) {
  if (n_ranks > kMaxSnapshots) return cudaErrorInvalidValue;
  const size_t per_warp = static_cast<size_t>(2) * T * m * sizeof(double);  // the warp's staged factor columns
  const int fit = static_cast<int>(std::min<size_t>(8, (200 * 1024) / per_warp));
  static const bool no_stage = [] {  // FL1_SUKRO_STAGE=0 forces the global-memory path (tests)
    const char* e = std::getenv("FL1_SUKRO_STAGE");
    return e && e[0] == '0';
  }();
  const bool staged = fit >= 1 && !no_stage;  // factor columns too long to stage: read them from global memory
  const int warps = staged ? fit : 8;
  const size_t smem = staged ? per_warp * warps : 0;
  cudaError_t e = cudaFuncSetAttribute(residual_norms_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const int64_t K = q * q;
  residual_norms_kernel<<<static_cast<unsigned>(std::min<int64_t>((K + warps - 1) / warps, 8192)), 32 * warps, smem,
                          stream>>>(a, lda, m, q, T, left, right, ldt, ranks, n_ranks, eps, app, staged ? 1 : 0);
  return cudaGetLastError();
}

int sukro_max_probe() { return kMaxProbe; }
int sukro_max_snapshots() { return kMaxSnapshots; }

}  // namespace fl1
