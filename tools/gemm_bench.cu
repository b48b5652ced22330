// Standalone timing + cross-check of the DMMA GEMM kernels on the hot path's
// shapes: SYRK lower (M x M, K), rank-K update (k-major A, n-major B),
// split-K long-K contraction (both m/n-major).  Links the library's host
// helpers by including kernels.cu directly.
#include <cstdio>
#include <vector>
#include "../paper_1907_01063_b200/csrc/kernels.cu"
using namespace stancl;

__global__ void fill(double* p, size_t n, double s) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = s * ((double)((i * 2654435761u) % 1000) * 1e-3 - 0.5);
}
__global__ void maxdiff(const double* a, const double* b, size_t n, double* out) {
  double m = 0, s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    m = fmax(m, fabs(a[i] - b[i]));
    s = fmax(s, fabs(b[i]));
  }
  atomicMax((unsigned long long*)&out[0], __double_as_longlong(m));
  atomicMax((unsigned long long*)&out[1], __double_as_longlong(s));
}

int g_impl = 0;  // 0 = w8 (one tile per CTA), 1 = tma, 2 = tma 2 CTAs/SM, 3 = tma 2 CTAs + C prefetch
template <bool AK, bool BK, int MODE>
cudaError_t launch(GemmArgs p, int splits) {
  if (g_impl == 1) return launch_tma<tg::CfgT, AK, BK, MODE>(p, splits, 0);
  if (g_impl == 2) return launch_tma<tg::CfgT2, AK, BK, MODE>(p, splits, 0);
  if (g_impl == 3) return launch_tma<tg::CfgT2P, AK, BK, MODE>(p, splits, 0);
  if (g_impl == 4) return launch_tma<tg::CfgT32, AK, BK, MODE>(p, splits, 0);
  if (g_impl == 5) return launch_tma<tg::CfgT128, AK, BK, MODE>(p, splits, 0);
  return launch_gemm<gemm::CfgW8, AK, BK, MODE>(p, splits, 0);
}
template <bool AK, bool BK, int MODE>
double timeit(GemmArgs p, int splits, int reps = 5) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  launch<AK, BK, MODE>(p, splits);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    launch<AK, BK, MODE>(p, splits);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("ERR %s\n", cudaGetErrorString(e));
  return best;
}
const char* NAMES[] = {"w8", "tma", "tma2", "tma2p", "tma32", "tma128"};

// run once with impl 0 and impl 1 from the same C0 and compare
template <bool AK, bool BK, int MODE>
void check(GemmArgs p, int splits, double* C0, double* C1, double* C2, size_t nC, double* d, const char* what) {
  double h[2] = {0, 0};
  cudaMemcpy(C1, C0, nC * 8, cudaMemcpyDeviceToDevice);
  cudaMemcpy(C2, C0, nC * 8, cudaMemcpyDeviceToDevice);
  GemmArgs q = p; q.C = C1; g_impl = 0; launch<AK, BK, MODE>(q, splits);
  q.C = C2; g_impl = 4; launch<AK, BK, MODE>(q, splits);
  cudaMemset(d, 0, 16);
  maxdiff<<<256, 256>>>(C2, C1, nC, d);
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("{\"check\": \"%s\", \"maxdiff\": %.3e, \"maxabs\": %.3e, \"rel\": %.3e, \"err\": \"%s\"}\n", what, h[0], h[1],
         h[0] / (h[1] > 0 ? h[1] : 1), cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int M = 8192;
  double *A, *B, *C, *P, *C1, *C2, *d;
  cudaMalloc(&A, (size_t)M * 1024 * 8);
  cudaMalloc(&B, (size_t)M * M * 8);
  cudaMalloc(&C, (size_t)M * M * 8);
  cudaMalloc(&C1, (size_t)M * M * 8);
  cudaMalloc(&C2, (size_t)M * M * 8);
  cudaMalloc(&P, (size_t)16 * 128 * M * 8);
  cudaMalloc(&d, 16);
  fill<<<1024, 256>>>(A, (size_t)M * 1024, 1.0);
  fill<<<1024, 256>>>(B, (size_t)M * M, 1.0);
  fill<<<1024, 256>>>(C, (size_t)M * M, 1.0);
  cudaDeviceSynchronize();
  {  // correctness cross-checks (small shapes)
    const int m = 1024;
    GemmArgs s{A, 128, A, 128, nullptr, m, m, m, 128, 128, -1.0, 1, 1, nullptr, 0};
    check<true, true, MODE_LOWER>(s, 1, C, C1, C2, (size_t)m * m, d, "syrk_lower_m1024_k128");
    GemmArgs g{A, 128, B, 2048, nullptr, 2048, m, 2048, 128, 128, -1.0, 1, 0, nullptr, 0};
    check<true, false, MODE_FULL>(g, 1, C, C1, C2, (size_t)m * 2048, d, "gemm_kn_m1024_n2048");
    GemmArgs g2{A, 128, A + 128 * 128, 128, nullptr, 128, m, 128, 128, 128, 1.0, 0, 0, nullptr, 0};
    check<true, true, MODE_FULL>(g2, 1, C, C1, C2, (size_t)m * 128, d, "gemm_kk_beta0");
    GemmArgs s2{A, 256, A, 256, nullptr, m, m, m, 256, 256, -1.0, 1, 1, nullptr, 0};
    check<true, true, MODE_LOWER>(s2, 1, C, C1, C2, (size_t)m * m, d, "syrk_lower_m1024_k256");
    GemmArgs g3{A, 256, A + 4096 * 256, 256, nullptr, 256, 4096, 256, 256, 256, -1.0, 1, 1, nullptr, 0};
    check<true, true, MODE_FULL>(g3, 1, C, C1, C2, (size_t)4096 * 256, d, "lookahead_m4096_n256_k256");
    GemmArgs g4{A, 256, B, 2048, nullptr, 2048, m, 2048, 256, 256, -1.0, 1, 0, nullptr, 0};
    check<true, false, MODE_FULL>(g4, 1, C, C1, C2, (size_t)m * 2048, d, "gemm_kn_k256");
    GemmArgs sk{B, 128, B, 2048, nullptr, 2048, 128, 2048, 4096, 1024, 1.0, 0, 0, nullptr, 0};
    check<false, false, MODE_SPLITK>(sk, 4, C, C1, C2, (size_t)4 * 128 * 2048, d, "splitk_n2048_k4096");
  }
  for (int impl : {0, 4}) {
    g_impl = impl;
    for (int K : {128, 256}) {
      GemmArgs s{A, K, A, K, C, M, M, M, K, K, -1.0, 1, 1, nullptr, 0};
      double ms = timeit<true, true, MODE_LOWER>(s, 1);
      printf("{\"op\": \"syrk\", \"impl\": \"%s\", \"M\": %d, \"K\": %d, \"ms\": %.4f, \"tflops\": %.2f}\n", NAMES[impl], M, K, ms, (double)K * M * (M + 1.0) / ms / 1e9);
      GemmArgs g{A, K, B, M / 2, C, M / 2, M, M / 2, K, K, -1.0, 1, 0, nullptr, 0};
      ms = timeit<true, false, MODE_FULL>(g, 1);
      printf("{\"op\": \"gemm_kn\", \"impl\": \"%s\", \"M\": %d, \"N\": %d, \"K\": %d, \"ms\": %.4f, \"tflops\": %.2f}\n", NAMES[impl], M, M / 2, K, ms, 2.0 * M * (M / 2) * K / ms / 1e9);
    }
    for (int sp : {2, 4, 8}) {
      int kps = ((M + sp - 1) / sp + 15) / 16 * 16;
      GemmArgs sk{B, 128, B, M, P, M, 128, M, M, kps, 1.0, 0, 0, nullptr, 0};
      double ms = timeit<false, false, MODE_SPLITK>(sk, sp);
      printf("{\"op\": \"splitk\", \"impl\": \"%s\", \"N\": %d, \"K\": %d, \"splits\": %d, \"ms\": %.4f, \"tflops\": %.2f}\n", NAMES[impl], M, M, sp, ms, 2.0 * 128 * M * M / ms / 1e9);
    }
  }
  return 0;
}
