// batched.cu -- NEXT-4: many independent small matrices
// (n <= 128) per call, e.g. one covariance per MCMC chain --
// "batched linear algebra".  The forward is one CTA per matrix
// running the diagonal-tile POTRF (kernels.cu, identity-padded to 128); the
// adjoint is the paper's symbolic diagonal step on every
// matrix at once: P = D^T D_bar (lower tiles, mirrored), S = D^-T sym(P) D^-1,
// A_bar = Phi(sym S), with D^-1 from the batched triangular inverse and the
// products from the batched 128^3 DMMA kernel, on 128 x 128 zero/identity
// padded copies (exact: the padding decouples).
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace stancl {

constexpr int64_t T2 = (int64_t)NB * NB;  // padded tile, doubles

// Lp[b] = [[L_b, 0], [0, I]] (lower; upper 0), Wp[b] = [[tril(L_bar_b), 0], [0, 0]]
__global__ void batched_pad_kernel(const double* L, const double* Lbar, int n, int64_t batch, double* Lp,
                                   double* Wp) {
  const int64_t total = batch * T2;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = idx / T2;
    const int e = (int)(idx - b * T2), r = e >> 7, c = e & (NB - 1);
    double l = 0.0, w = 0.0;
    if (r < n && c < n) {
      if (c <= r) {
        l = L[b * n * n + (int64_t)r * n + c];
        w = Lbar[b * n * n + (int64_t)r * n + c];
      }
    } else if (r == c) {
      l = 1.0;
    }
    Lp[idx] = l;
    Wp[idx] = w;
  }
}

// info[b] = first k with L_b[k][k] not finite and > 0, plus 1
__global__ void batched_check_diag_kernel(const double* L, int n, int64_t batch, int* info) {
  for (int64_t b = blockIdx.x; b < batch; b += gridDim.x) {
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
      const double d = L[b * n * n + (int64_t)k * n + k];
      if (!(d > 0.0) || !isfinite(d)) atomicMin(info + b, k + 1);
    }
  }
}
__global__ void batched_info_init_kernel(int* info, int64_t batch) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < batch; b += (int64_t)gridDim.x * blockDim.x)
    info[b] = 0x7fffffff;
}
__global__ void batched_info_fin_kernel(int* info, int64_t batch) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < batch; b += (int64_t)gridDim.x * blockDim.x)
    if (info[b] == 0x7fffffff) info[b] = 0;
}

// Abar[b] (n x n) = Phi(sym(S_b)) restricted to the leading n x n block
__global__ void batched_phi_out_kernel(const double* S, int n, int64_t batch, double* Abar) {
  const int64_t total = batch * n * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = idx / ((int64_t)n * n);
    const int e = (int)(idx - b * n * n), r = e / n, c = e - r * n;
    const double* Sb = S + b * T2;
    double v = 0.0;
    if (r > c) v = Sb[(int64_t)r * NB + c];
    else if (r == c) v = 0.5 * Sb[(int64_t)r * NB + r];
    Abar[idx] = v;
  }
}

__global__ void batched_first_fail_kernel(const int* info, int64_t batch, int* status) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < batch; b += (int64_t)gridDim.x * blockDim.x)
    if (info[b] != 0) atomicMin(status, (int)(b + 1));
}
__global__ void status_init_kernel(int* status, int v) { *status = v; }
__global__ void status_fin_kernel(int* status) {
  if (*status == 0x7fffffff) *status = 0;
}

static inline int gcap(int64_t work, int threads) {
  int64_t b = (work + threads - 1) / threads;
  return (int)(b < 1 ? 1 : (b > 148 * 16 ? 148 * 16 : b));
}

cudaError_t batched_pad(const double* L, const double* Lbar, int n, int64_t batch, double* Lp, double* Wp,
                        cudaStream_t st) {
  Prof prof_(PROF_MISC, 0.0, st, 8.0 * batch * (double)n * n + 16.0 * batch * (double)T2);
  batched_pad_kernel<<<gcap(batch * T2, 256), 256, 0, st>>>(L, Lbar, n, batch, Lp, Wp);
  return cudaGetLastError();
}

cudaError_t batched_check_diag(const double* L, int n, int64_t batch, int* info, cudaStream_t st) {
  Prof prof_(PROF_MISC, 0.0, st, 8.0 * batch * n);
  batched_info_init_kernel<<<gcap(batch, 256), 256, 0, st>>>(info, batch);
  batched_check_diag_kernel<<<(int)(batch < 148 * 16 ? batch : 148 * 16), 128, 0, st>>>(L, n, batch, info);
  batched_info_fin_kernel<<<gcap(batch, 256), 256, 0, st>>>(info, batch);
  return cudaGetLastError();
}

cudaError_t batched_phi_out(const double* S, int n, int64_t batch, double* Abar, cudaStream_t st) {
  Prof prof_(PROF_MISC, 0.0, st, 12.0 * batch * (double)n * n);
  batched_phi_out_kernel<<<gcap(batch * n * n, 256), 256, 0, st>>>(S, n, batch, Abar);
  return cudaGetLastError();
}

cudaError_t batched_first_fail(const int* info, int64_t batch, int* status, cudaStream_t st) {
  Prof prof_(PROF_MISC, 0.0, st, 4.0 * batch);
  status_init_kernel<<<1, 1, 0, st>>>(status, 0x7fffffff);
  batched_first_fail_kernel<<<gcap(batch, 256), 256, 0, st>>>(info, batch, status);
  status_fin_kernel<<<1, 1, 0, st>>>(status);
  return cudaGetLastError();
}

}  // namespace stancl
