// kernels.cu -- the CUDA kernels of the hot path (sm_100a) and their launchers.
//
// Paper: "GPU-based parallel computation support for Stan" (arXiv:1907.01063),
// PAPER.md §3.3.  Step names follow SURVEY.md §8(a):
//   F0 se_cov_kernel           SE covariance of the GP example
//   F1 potrf_tile_kernel       chol of the diagonal b x b block, "classic sequential
//                              algorithm ... inner loop parallel"
//   F2 trsm_panel_kernel       L21 = A21 (L11^T)^-1 by substitution
//                              (R11: no explicit inverse in the forward)
//   F3 gemm_dmma (MODE_LOWER)  A22 -= L21 L21^T, gemm_dmma.cuh
//   R*  adjoint building blocks: tri_inverse_batched (D^-1 for all
//       diagonal blocks), gemm128 (128^3 products of the symbolic
//       diagonal step), phi_sym,
//       splitk_reduce_sub (the paper's large-k reduction)
#include <atomic>
#include <climits>
#include <vector>

#include "common.cuh"
#include "gemm_dmma.cuh"
#include "kernels.h"

namespace stancl {

static std::atomic<long long> g_launches{0};
void count_launch(int k) { g_launches.fetch_add(k, std::memory_order_relaxed); }
long long launches() { return g_launches.load(std::memory_order_relaxed); }

// ---- per-kernel-class CUDA-event timing (stan_cl_profile_*) ----
namespace {
struct ProfRec {
  int kind;
  double flops;
  cudaEvent_t e0, e1;
};
struct ProfState {
  bool on = false;
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> pool;
  double ms[PROF_KINDS] = {0};
  double flops[PROF_KINDS] = {0};
  long long count[PROF_KINDS] = {0};
};
ProfState g_prof;
cudaEvent_t prof_event() {
  if (!g_prof.pool.empty()) {
    cudaEvent_t e = g_prof.pool.back();
    g_prof.pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

Prof::Prof(int kind, double flops, cudaStream_t st) : kind_(kind), flops_(flops), st_(st) {
  count_launch();
  if (g_prof.on) {
    e0_ = prof_event();
    e1_ = prof_event();
    cudaEventRecord(e0_, st_);
  }
}
Prof::~Prof() {
  if (g_prof.on && e0_) {
    cudaEventRecord(e1_, st_);
    g_prof.recs.push_back({kind_, flops_, e0_, e1_});
  }
}
void prof_enable(bool on) { g_prof.on = on; }
void prof_collect() {
  for (auto& r : g_prof.recs) {
    cudaEventSynchronize(r.e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.e0, r.e1);
    g_prof.ms[r.kind] += ms;
    g_prof.flops[r.kind] += r.flops;
    g_prof.count[r.kind] += 1;
    g_prof.pool.push_back(r.e0);
    g_prof.pool.push_back(r.e1);
  }
  g_prof.recs.clear();
}
void prof_reset() {
  prof_collect();
  for (int k = 0; k < PROF_KINDS; ++k) g_prof.ms[k] = g_prof.flops[k] = 0, g_prof.count[k] = 0;
}
void prof_read(int kind, double* ms, double* flops, long long* count) {
  prof_collect();
  *ms = g_prof.ms[kind];
  *flops = g_prof.flops[kind];
  *count = g_prof.count[kind];
}

static inline int grid_for(long long work, int threads, int cap = 148 * 16) {
  long long b = (work + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return (int)b;
}

// ----------------------------------------------------------------------- F0
__global__ void se_cov_kernel(int64_t n, const double* __restrict__ x, double sq_alpha,
                              double neg_half_inv_rho2, double jitter, double* __restrict__ K) {
  const long long total = (long long)n * n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long i = idx / n, j = idx - i * n;
    const double d = x[i] - x[j];
    // same association as the definition: (d*d)*c, then alpha^2 * exp(.), + jitter on i == j
    const double e = __dmul_rn(__dmul_rn(d, d), neg_half_inv_rho2);
    double v = __dmul_rn(sq_alpha, exp(e));
    if (i == j) v = __dadd_rn(v, jitter);
    K[idx] = v;
  }
}

cudaError_t se_cov(int64_t n, const double* x, double alpha, double rho, double jitter, double* K,
                   cudaStream_t st) {
  Prof prof_(PROF_SE, 0.0, st);
  if (n == 0) return cudaSuccess;
  const double sq_alpha = alpha * alpha;
  const double c = -0.5 / (rho * rho);
  se_cov_kernel<<<grid_for((long long)n * n, 256), 256, 0, st>>>(n, x, sq_alpha, c, jitter, K);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------- K11
__global__ void copy_lower_pad_kernel(const double* __restrict__ src, int64_t n, int64_t lds,
                                      double* __restrict__ dst, int64_t N, int64_t ldd,
                                      double diag_pad) {
  const long long total = (long long)N * N;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long i = idx / N, j = idx - i * N;
    double v;
    if (i < n && j < n) v = (j <= i) ? src[i * lds + j] : 0.0;
    else v = (i == j) ? diag_pad : 0.0;
    dst[i * ldd + j] = v;
  }
}

cudaError_t copy_lower_pad(const double* src, int64_t n, int64_t lds, double* dst, int64_t N,
                           int64_t ldd, double diag_pad, cudaStream_t st) {
  Prof prof_(PROF_MISC, 0.0, st);
  if (N == 0) return cudaSuccess;
  copy_lower_pad_kernel<<<grid_for((long long)N * N, 256), 256, 0, st>>>(src, n, lds, dst, N, ldd,
                                                                          diag_pad);
  return cudaGetLastError();
}

__global__ void copy_lower_out_kernel(const double* __restrict__ src, int64_t lds,
                                      double* __restrict__ dst, int64_t n, int64_t ldd) {
  const long long total = (long long)n * n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long i = idx / n, j = idx - i * n;
    dst[i * ldd + j] = (j <= i) ? src[i * lds + j] : 0.0;
  }
}

cudaError_t copy_lower_out(const double* src, int64_t lds, double* dst, int64_t n, int64_t ldd,
                           cudaStream_t st) {
  Prof prof_(PROF_MISC, 0.0, st);
  if (n == 0) return cudaSuccess;
  copy_lower_out_kernel<<<grid_for((long long)n * n, 256), 256, 0, st>>>(src, lds, dst, n, ldd);
  return cudaGetLastError();
}

__global__ void zero_upper_kernel(double* A, int64_t n, int64_t ld) {
  const long long total = (long long)n * n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long i = idx / n, j = idx - i * n;
    if (j > i) A[i * ld + j] = 0.0;
  }
}

cudaError_t zero_upper(double* A, int64_t n, int64_t ld, cudaStream_t st) {
  Prof prof_(PROF_MISC, 0.0, st);
  if (n == 0) return cudaSuccess;
  zero_upper_kernel<<<grid_for((long long)n * n, 256), 256, 0, st>>>(A, n, ld);
  return cudaGetLastError();
}

// ----------------------------------------------------------------------- F1
// One CTA factors the 128 x 128 diagonal tile in shared memory, right-looking
// column by column: pivot sqrt (IEEE), column scale by IEEE division, rank-1
// update of the trailing lower part (one FMA per element, ascending j).
constexpr int TP = NB + 1;  // tile pitch (doubles): conflict-free column access
constexpr int POTRF_SMEM = (NB * TP + NB) * (int)sizeof(double);

__global__ void __launch_bounds__(256, 1) potrf_tile_kernel(double* W, int64_t ld, int64_t k0,
                                                            int* status) {
  if (*status != 0) return;
  extern __shared__ double sm[];
  double* T = sm;
  double* col = sm + NB * TP;
  __shared__ int fail_j;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* base = W + k0 * ld + k0;
  for (int idx = tid; idx < NB * NB; idx += 256) {
    const int i = idx >> 7, l = idx & (NB - 1);
    if (l <= i) T[i * TP + l] = base[(long long)i * ld + l];
  }
  if (tid == 0) fail_j = -1;
  __syncthreads();
  for (int j = 0; j < NB; ++j) {
    if (tid == 0) {
      const double d = T[j * TP + j];
      if (!(d > 0.0)) fail_j = j;
      else T[j * TP + j] = sqrt(d);
    }
    __syncthreads();
    if (fail_j >= 0) break;
    const double djj = T[j * TP + j];
    for (int i = j + 1 + tid; i < NB; i += 256) {
      const double v = T[i * TP + j] / djj;
      T[i * TP + j] = v;
      col[i] = v;
    }
    __syncthreads();
    for (int i = j + 1 + warp; i < NB; i += 8) {
      const double ci = col[i];
      for (int l = j + 1 + lane; l <= i; l += 32) T[i * TP + l] = fma(-ci, col[l], T[i * TP + l]);
    }
    __syncthreads();
  }
  __syncthreads();
  for (int idx = tid; idx < NB * NB; idx += 256) {
    const int i = idx >> 7, l = idx & (NB - 1);
    if (l <= i) base[(long long)i * ld + l] = T[i * TP + l];
  }
  if (tid == 0 && fail_j >= 0) atomicCAS(status, 0, (int)(k0 + fail_j + 1));
}

cudaError_t potrf_tile(double* W, int64_t ld, int64_t k0, int* status, cudaStream_t st) {
  Prof prof_(PROF_POTRF, (double)NB * NB * NB / 3.0, st);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(potrf_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         POTRF_SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  potrf_tile_kernel<<<1, 256, POTRF_SMEM, st>>>(W, ld, k0, status);
  return cudaGetLastError();
}

// ----------------------------------------------------------------------- F2
// X L11^T = A21 for a 64-row slab per CTA.  L11^T is staged in shared memory
// (LT[j][l] = L11[l][j]); four threads own a row (columns p, p+4, ...), and
// column j is finished by its owner with an IEEE division, then broadcast to
// the other three through shared memory (same warp: __syncwarp suffices).
constexpr int TRSM_ROWS = 64;
constexpr int RP = NB + 4;  // row pitch: 4 rows x 4 threads per half-warp hit distinct banks
constexpr int TRSM_SMEM = (NB * TP + TRSM_ROWS * RP + NB) * (int)sizeof(double);

__global__ void __launch_bounds__(256, 1) trsm_panel_kernel(double* W, int64_t ld, int64_t k0,
                                                            int64_t r0, const int* status) {
  if (*status != 0) return;
  extern __shared__ double sm[];
  double* LT = sm;
  double* R = sm + NB * TP;
  double* dg = R + TRSM_ROWS * RP;
  const int tid = threadIdx.x;
  const double* L11 = W + k0 * ld + k0;
  for (int idx = tid; idx < NB * NB; idx += 256) {
    const int l = idx >> 7, j = idx & (NB - 1);
    if (j <= l) LT[j * TP + l] = L11[(long long)l * ld + j];
    if (j == l) dg[j] = L11[(long long)l * ld + j];
  }
  const long long row0 = r0 + (long long)blockIdx.x * TRSM_ROWS;
  double* P = W + row0 * ld + k0;
  for (int idx = tid; idx < TRSM_ROWS * NB; idx += 256) {
    const int r = idx >> 7, c = idx & (NB - 1);
    R[r * RP + c] = P[(long long)r * ld + c];
  }
  __syncthreads();
  const int r = tid >> 2, p = tid & 3;
  double* row = R + r * RP;
  for (int j = 0; j < NB; ++j) {
    if ((j & 3) == p) row[j] = row[j] / dg[j];
    __syncwarp();
    const double x = row[j];
    const double* lt = LT + j * TP;
    for (int c = j + 1 + ((p - (j + 1)) & 3); c < NB; c += 4) row[c] = fma(-x, lt[c], row[c]);
    __syncwarp();
  }
  __syncthreads();
  for (int idx = tid; idx < TRSM_ROWS * NB; idx += 256) {
    const int rr = idx >> 7, c = idx & (NB - 1);
    P[(long long)rr * ld + c] = R[rr * RP + c];
  }
}

cudaError_t trsm_panel(double* W, int64_t ld, int64_t k0, int64_t r0, int64_t r1, const int* status,
                       cudaStream_t st) {
  Prof prof_(PROF_TRSM, (double)(r1 - r0) * NB * NB, st);
  if (r1 <= r0) return cudaSuccess;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(trsm_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         TRSM_SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int blocks = (int)((r1 - r0) / TRSM_ROWS);
  trsm_panel_kernel<<<blocks, 256, TRSM_SMEM, st>>>(W, ld, k0, r0, status);
  return cudaGetLastError();
}

// ------------------------------------------------------------ DMMA GEMM family
cudaError_t gemm_full(bool a_kmaj, bool b_kmaj, int M, int N, int K, double sign, int beta,
                      const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                      int64_t ldc, const int* status, cudaStream_t st) {
  Prof prof_(PROF_GEMM, 2.0 * M * N * K, st);
  if (M == 0 || N == 0) return cudaSuccess;
  GemmArgs p{A, lda, B, ldb, C, ldc, M, N, K, K, sign, beta, status};
  if (a_kmaj && b_kmaj) return launch_gemm<true, true, MODE_FULL>(p, 1, st);
  if (a_kmaj && !b_kmaj) return launch_gemm<true, false, MODE_FULL>(p, 1, st);
  if (!a_kmaj && b_kmaj) return launch_gemm<false, true, MODE_FULL>(p, 1, st);
  return launch_gemm<false, false, MODE_FULL>(p, 1, st);
}

cudaError_t gemm_lower_nt(int M, int K, const double* A, int64_t lda, const double* B, int64_t ldb,
                          double* C, int64_t ldc, const int* status, cudaStream_t st) {
  Prof prof_(PROF_SYRK, (double)K * M * (M + 1.0), st);
  if (M == 0) return cudaSuccess;
  GemmArgs p{A, lda, B, ldb, C, ldc, M, M, K, K, -1.0, 1, status};
  return launch_gemm<true, true, MODE_LOWER>(p, 1, st);
}

cudaError_t gemm_splitk_tn(int M, int N, int K, int splits, int kps, const double* A, int64_t lda,
                           const double* B, int64_t ldb, double* P, const int* status,
                           cudaStream_t st) {
  Prof prof_(PROF_SPLITK, 2.0 * M * N * K, st);
  if (M == 0 || N == 0) return cudaSuccess;
  GemmArgs p{A, lda, B, ldb, P, N, M, N, K, kps, 1.0, 0, status};
  return launch_gemm<false, false, MODE_SPLITK>(p, splits, st);
}

__global__ void splitk_reduce_sub_kernel(const double* __restrict__ P, int splits, int M, int N,
                                         double* __restrict__ dst, int64_t ldd, const int* status) {
  if (*status != 0) return;
  const long long half = (long long)M * N / 2;
  const long long plane = (long long)M * N;
  for (long long h = blockIdx.x * (long long)blockDim.x + threadIdx.x; h < half;
       h += (long long)gridDim.x * blockDim.x) {
    const long long e = 2 * h;
    const long long r = e / N, c = e - r * N;
    double2 s = *reinterpret_cast<const double2*>(P + e);
    for (int z = 1; z < splits; ++z) {
      const double2 v = *reinterpret_cast<const double2*>(P + z * plane + e);
      s.x += v.x;
      s.y += v.y;
    }
    double2* d = reinterpret_cast<double2*>(dst + r * ldd + c);
    double2 o = *d;
    o.x -= s.x;
    o.y -= s.y;
    *d = o;
  }
}

cudaError_t splitk_reduce_sub(const double* P, int splits, int M, int N, double* dst, int64_t ldd,
                              const int* status, cudaStream_t st) {
  Prof prof_(PROF_MISC, 0.0, st);
  if (M == 0 || N == 0) return cudaSuccess;
  splitk_reduce_sub_kernel<<<grid_for((long long)M * N / 2, 256), 256, 0, st>>>(P, splits, M, N, dst,
                                                                                ldd, status);
  return cudaGetLastError();
}

// ------------------------------------------------------------- R1/R4 helpers
// D^-1 of each 128 x 128 diagonal block of L, column c by thread c:
//   x_c = 1 / D[c][c];  x_i = -(sum_{k=c}^{i-1} D[i][k] x_k) / D[i][i],  i > c
// (lower_triangular_inverse of PAPER.md:207-225, by substitution per column)
constexpr int TRI_PACKED = NB * (NB + 1) / 2;  // D lower triangle, row i at i(i+1)/2
constexpr int TINV_SMEM = (TRI_PACKED + NB * TP) * (int)sizeof(double);

__global__ void __launch_bounds__(128, 1) tri_inverse_kernel(const double* L, int64_t ld,
                                                             double* Dinv, const int* status) {
  if (*status != 0) return;
  extern __shared__ double sm[];
  double* D = sm;               // packed lower: D[i][k] at i(i+1)/2 + k
  double* X = sm + TRI_PACKED;  // X[c][i] = (D^-1)[i][c]  (column c of the inverse, contiguous)
  const int b = blockIdx.x, c = threadIdx.x;
  const double* src = L + (long long)b * NB * ld + (long long)b * NB;
  for (int idx = c; idx < NB * NB; idx += NB) {
    const int i = idx >> 7, k = idx & (NB - 1);
    if (k <= i) D[i * (i + 1) / 2 + k] = src[(long long)i * ld + k];
  }
  __syncthreads();
  double* x = X + c * TP;
  for (int i = 0; i < c; ++i) x[i] = 0.0;
  x[c] = 1.0 / D[c * (c + 1) / 2 + c];
  for (int i = c + 1; i < NB; ++i) {
    double s = 0.0;
    const double* di = D + i * (i + 1) / 2;
    for (int k = c; k < i; ++k) s = fma(di[k], x[k], s);
    x[i] = -s / di[i];
  }
  __syncthreads();
  double* dst = Dinv + (long long)b * NB * NB;
  for (int idx = c; idx < NB * NB; idx += NB) {
    const int i = idx >> 7, k = idx & (NB - 1);
    dst[idx] = X[k * TP + i];
  }
}

cudaError_t tri_inverse_batched(const double* L, int64_t ld, int nblk, double* Dinv,
                                const int* status, cudaStream_t st) {
  Prof prof_(PROF_TRINV, (double)nblk * NB * NB * NB / 3.0, st);
  if (nblk == 0) return cudaSuccess;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tri_inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         TINV_SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  tri_inverse_kernel<<<nblk, NB, TINV_SMEM, st>>>(L, ld, Dinv, status);
  return cudaGetLastError();
}

// 128^3 product on 16 CTAs (32 x 32 output tiles, 4 warps of 16 x 16, DMMA)
constexpr int G128_AP = NB + 4, G128_BP = 32 + 4;
constexpr int G128_SMEM = (32 * G128_AP + NB * G128_BP) * (int)sizeof(double);

__global__ void __launch_bounds__(128) gemm128_kernel(bool a_t, bool a_tril, bool b_t, bool b_sym,
                                                      const double* __restrict__ A, int64_t lda,
                                                      const double* __restrict__ B, int64_t ldb,
                                                      double* __restrict__ C, int64_t ldc,
                                                      const int* status) {
  if (*status != 0) return;
  extern __shared__ double sm[];
  double* As = sm;                 // [32][G128_AP]   As[m][k]
  double* Bs = sm + 32 * G128_AP;  // [128][G128_BP]  Bs[k][n]
  const int m0 = blockIdx.y * 32, n0 = blockIdx.x * 32;
  const int tid = threadIdx.x;
  for (int idx = tid; idx < 32 * NB; idx += 128) {
    int m, k;
    double v;
    if (a_t) {
      k = idx >> 5;
      m = idx & 31;
      v = (a_tril && m0 + m > k) ? 0.0 : A[(long long)k * lda + m0 + m];
    } else {
      m = idx >> 7;
      k = idx & (NB - 1);
      v = (a_tril && k > m0 + m) ? 0.0 : A[(long long)(m0 + m) * lda + k];
    }
    As[m * G128_AP + k] = v;
  }
  for (int idx = tid; idx < 32 * NB; idx += 128) {
    int k, n;
    double v;
    if (b_sym) {
      k = idx >> 5;
      n = idx & 31;
      const int gn = n0 + n;
      v = (k >= gn) ? B[(long long)k * ldb + gn] : B[(long long)gn * ldb + k];
    } else if (b_t) {
      n = idx >> 7;
      k = idx & (NB - 1);
      v = B[(long long)(n0 + n) * ldb + k];
    } else {
      k = idx >> 5;
      n = idx & 31;
      v = B[(long long)k * ldb + n0 + n];
    }
    Bs[k * G128_BP + n] = v;
  }
  __syncthreads();
  const int lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1, g = lane >> 2, t = lane & 3;
  double acc[2][2][2] = {};
#pragma unroll 8
  for (int k4 = 0; k4 < NB; k4 += 4) {
    double af[2], bf[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) af[i] = As[(wm * 16 + i * 8 + g) * G128_AP + k4 + t];
#pragma unroll
    for (int j = 0; j < 2; ++j) bf[j] = Bs[(k4 + t) * G128_BP + wn * 16 + j * 8 + g];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int r = m0 + wm * 16 + i * 8 + g, c = n0 + wn * 16 + j * 8 + 2 * t;
      C[(long long)r * ldc + c] = acc[i][j][0];
      C[(long long)r * ldc + c + 1] = acc[i][j][1];
    }
}

cudaError_t gemm128(bool a_t, bool a_tril, bool b_t, bool b_sym, const double* A, int64_t lda,
                    const double* B, int64_t ldb, double* C, int64_t ldc, const int* status,
                    cudaStream_t st) {
  Prof prof_(PROF_SMALL, 2.0 * NB * NB * NB, st);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gemm128_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         G128_SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  gemm128_kernel<<<dim3(4, 4), 128, G128_SMEM, st>>>(a_t, a_tril, b_t, b_sym, A, lda, B, ldb, C, ldc, status);
  return cudaGetLastError();
}

// S -> Ssym = mirror(tril S) and D_bar = Phi(S)
__global__ void phi_sym_kernel(const double* __restrict__ S, double* __restrict__ Ssym,
                               double* __restrict__ Dbar, int64_t ldd, const int* status) {
  if (*status != 0) return;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < NB * NB; idx += gridDim.x * blockDim.x) {
    const int a = idx >> 7, b = idx & (NB - 1);
    const double low = (a >= b) ? S[a * NB + b] : S[b * NB + a];
    Ssym[idx] = low;
    Dbar[(long long)a * ldd + b] = (a > b) ? low : (a == b ? 0.5 * low : 0.0);
  }
}

cudaError_t phi_sym(const double* S, double* Ssym, double* Dbar, int64_t ldd, const int* status,
                    cudaStream_t st) {
  Prof prof_(PROF_MISC, 0.0, st);
  phi_sym_kernel<<<64, 256, 0, st>>>(S, Ssym, Dbar, ldd, status);
  return cudaGetLastError();
}

__global__ void check_diag_kernel(const double* L, int64_t n, int64_t ld, int* status) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
       k += (long long)gridDim.x * blockDim.x) {
    const double d = L[k * ld + k];
    if (!(d > 0.0) || !isfinite(d)) {
      const int v = (int)(k + 1);
      int old = *(volatile int*)status;
      while (old == 0 || v < old) {
        const int prev = atomicCAS(status, old, v);
        if (prev == old) break;
        old = prev;
      }
    }
  }
}

cudaError_t check_diag(const double* L, int64_t n, int64_t ld, int* status, cudaStream_t st) {
  Prof prof_(PROF_MISC, 0.0, st);
  if (n == 0) return cudaSuccess;
  check_diag_kernel<<<grid_for(n, 256, 148), 256, 0, st>>>(L, n, ld, status);
  return cudaGetLastError();
}

}  // namespace stancl
