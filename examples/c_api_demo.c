/*
 * c_api_demo.c -- the C ABI (include/stan_cl.h) from plain C: no Python, no
 * torch.  Builds the SE covariance of the paper's GP example on the device,
 * factors it, runs the adjoint with L_bar = diag(2 / L_ii) (the gradient of
 * log det A, so A_bar = Phi(2 A^-1)) and checks the identity
 * sum_{i >= j} A_bar_ij A_ij = tr(A^-1 A) = n; exercises the status codes and
 * the caller-owned workspace.
 *
 *   gcc -O2 -std=c99 examples/c_api_demo.c -Iinclude -I/usr/local/cuda/include \
 *       -Lpaper_1907_01063_b200 -lstancl -L/usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_1907_01063_b200 -lm -o c_api_demo && ./c_api_demo 2000
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "stan_cl.h"

#define CHECK_CUDA(x)                                                   \
  do {                                                                  \
    cudaError_t e_ = (x);                                               \
    if (e_ != cudaSuccess) {                                            \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));          \
      return 2;                                                         \
    }                                                                   \
  } while (0)
#define CHECK_SC(x)                                                     \
  do {                                                                  \
    int s_ = (x);                                                       \
    if (s_ != 0) {                                                      \
      fprintf(stderr, "%s -> %d (%s)\n", #x, s_, stan_cl_status_string(s_)); \
      return 3;                                                         \
    }                                                                   \
  } while (0)

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 2000;
  const size_t bytes = (size_t)n * (size_t)n * sizeof(double);
  double* x_h = (double*)malloc(n * sizeof(double));
  unsigned long long s = 42;
  for (int64_t i = 0; i < n; ++i) {  /* x ~ U(-10, 10), a simple LCG here */
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    x_h[i] = -10.0 + 20.0 * (double)(s >> 11) * 0x1.0p-53;
  }
  double *x, *K, *L, *W;
  CHECK_CUDA(cudaMalloc((void**)&x, n * sizeof(double)));
  CHECK_CUDA(cudaMalloc((void**)&K, bytes));
  CHECK_CUDA(cudaMalloc((void**)&L, bytes));
  CHECK_CUDA(cudaMalloc((void**)&W, bytes));
  CHECK_CUDA(cudaMemcpy(x, x_h, n * sizeof(double), cudaMemcpyHostToDevice));

  /* caller-owned workspace: the library allocates nothing of its own */
  void* ws = NULL;
  const size_t wsb = stan_cl_workspace_bytes(n);
  CHECK_CUDA(cudaMalloc(&ws, wsb));
  CHECK_SC(stan_cl_set_workspace(ws, wsb));

  CHECK_SC(stan_cl_gp_exp_quad_cov(n, x, 1.0, 1.0, 1e-2, K));
  CHECK_SC(stan_cl_check_matrix(n, K, 7, 0.0));          /* no NaN, symmetric, no zero diagonal */
  CHECK_SC(stan_cl_cholesky(n, K, L));

  double* L_h = (double*)malloc(bytes);
  double* A_h = (double*)malloc(bytes);
  CHECK_CUDA(cudaMemcpy(L_h, L, bytes, cudaMemcpyDeviceToHost));
  /* L_bar = diag(2 / L_ii): d log det A / d L */
  double* Wb_h = (double*)calloc((size_t)n * n, sizeof(double));
  double logdet = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    Wb_h[i * n + i] = 2.0 / L_h[i * n + i];
    logdet += 2.0 * log(L_h[i * n + i]);
  }
  CHECK_CUDA(cudaMemcpy(W, Wb_h, bytes, cudaMemcpyHostToDevice));
  CHECK_SC(stan_cl_cholesky_adjoint(n, L, W, W));        /* in place */
  CHECK_CUDA(cudaMemcpy(Wb_h, W, bytes, cudaMemcpyDeviceToHost));
  CHECK_CUDA(cudaMemcpy(A_h, K, bytes, cudaMemcpyDeviceToHost));
  /* A_bar = Phi(2 A^-1) (diagonal A^-1_ii, strictly lower 2 A^-1_ij), so
     sum_{i >= j} A_bar_ij A_ij = sum_{i,j} A^-1_ij A_ij = tr(A^-1 A) = n */
  double tr = 0.0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j <= i; ++j) tr += Wb_h[i * n + j] * A_h[i * n + j];
  const double rel = fabs(tr - (double)n) / (double)n;

  /* error paths: not positive definite, bad arguments */
  CHECK_CUDA(cudaMemset(K, 0, bytes));
  const int info = stan_cl_cholesky(n, K, L);           /* zero matrix: pivot 0 fails -> 1 */
  const int einval = stan_cl_cholesky(-1, K, L);
  CHECK_SC(stan_cl_set_workspace(NULL, 0));
  printf("c_api_demo n=%lld: log det = %.6f, trace identity rel err = %.2e, not-PD info = %d, EINVAL = %d, "
         "workspace %zu bytes\n", (long long)n, logdet, rel, info, einval, wsb);
  cudaFree(ws);
  cudaFree(x);
  cudaFree(K);
  cudaFree(L);
  cudaFree(W);
  stan_cl_finalize();
  return (rel < 1e-8 && info == 1 && einval == STAN_CL_EINVAL) ? 0 : 1;
}
