// PCIe copy-engine rates for the host-transfer shapes of the *_host entry points.
#include <cstdio>
#include <cuda_runtime.h>
int main() {
  const size_t n = 16384;
  double *h, *d;
  cudaHostAlloc(&h, n * n * 8, cudaHostAllocDefault);
  cudaMalloc(&d, n * n * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto rep = [&](const char* name, double bytes, float ms) { printf("{\"copy\": \"%s\", \"GB\": %.3f, \"ms\": %.2f, \"GBps\": %.1f}\n", name, bytes / 1e9, ms, bytes / ms / 1e6); };
  float ms;
  for (int dir = 0; dir < 2; ++dir) {
    cudaMemcpyKind k = dir ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice;
    void* dst = dir ? (void*)h : (void*)d; const void* src = dir ? (const void*)d : (const void*)h;
    cudaMemcpyAsync(dst, src, n * n * 8, k); cudaDeviceSynchronize();
    cudaEventRecord(a); cudaMemcpyAsync(dst, src, n * n * 8, k); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); rep(dir ? "d2h_contig_2GiB" : "h2d_contig_2GiB", n * n * 8.0, ms);
    // lower rectangles per 128-row block
    double bytes = 0;
    cudaEventRecord(a);
    for (size_t r0 = 0; r0 < n; r0 += 128) {
      size_t r1 = r0 + 128;
      cudaMemcpy2DAsync((char*)dst + r0 * n * 8, n * 8, (const char*)src + r0 * n * 8, n * 8, r1 * 8, 128, k);
      bytes += r1 * 8.0 * 128;
    }
    cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    rep(dir ? "d2h_rowblock_rects" : "h2d_rowblock_rects", bytes, ms);
    // column blocks (1 KB wide)
    bytes = 0;
    cudaEventRecord(a);
    for (size_t j = 0; j < n; j += 128) {
      cudaMemcpy2DAsync((char*)dst + (j * n + j) * 8, n * 8, (const char*)src + (j * n + j) * 8, n * 8, 128 * 8, n - j, k);
      bytes += 128 * 8.0 * (n - j);
    }
    cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    rep(dir ? "d2h_colblock_1KB" : "h2d_colblock_1KB", bytes, ms);
  }
  // both directions at once (two streams)
  cudaStream_t s1, s2; cudaStreamCreate(&s1); cudaStreamCreate(&s2);
  double* h2; cudaHostAlloc(&h2, n * n * 8 / 2, cudaHostAllocDefault);
  cudaEventRecord(a);
  cudaMemcpyAsync(d, h, n * n * 4, cudaMemcpyHostToDevice, s1);
  cudaMemcpyAsync(h2, d + n * n / 2, n * n * 4, cudaMemcpyDeviceToHost, s2);
  cudaStreamSynchronize(s1); cudaStreamSynchronize(s2);
  cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
  rep("duplex_1GiB_each", n * n * 8.0, ms);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
