// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync .f64) vs DFMA.
// Register-resident loops; reports TFLOP/s (2 flops per FMA) per variant.
// Used to fix the FP64 roofline denominator.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int NACC>
__global__ void dmma_m8n8k4(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void dmma_m16n8k16(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + (threadIdx.x + i) * 1e-9;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - (threadIdx.x + i) * 1e-9;
  double c[NACC][4];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <typename K>
static double run(K kern, int blocks, int threads, int iters, double fma_per_thread_iter, const char* name, double* out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(out, iters / 10);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  double flops = 2.0 * fma_per_thread_iter * (double)blocks * threads * iters;
  double tf = flops / (best * 1e-3) / 1e12;
  printf("{\"kernel\": \"%s\", \"blocks\": %d, \"threads\": %d, \"ms\": %.3f, \"tflops\": %.3f}\n", name, blocks, threads, best, tf);
  return tf;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_per_block_optin\": %zu, \"clock_khz\": %d}\n",
         p.name, p.multiProcessorCount, p.l2CacheSize, p.sharedMemPerBlockOptin, clk);
  double* out; CK(cudaMalloc(&out, 1 << 20));
  int sms = p.multiProcessorCount;
  // m8n8k4: 256 FMAs per warp-instruction = 8 per thread
  for (int w : {4, 8, 16}) {
    run(dmma_m8n8k4<8>, sms, 32 * w, 20000, 8.0 * 8, w == 4 ? "dmma_m8n8k4_acc8_w4" : w == 8 ? "dmma_m8n8k4_acc8_w8" : "dmma_m8n8k4_acc8_w16", out);
  }
  run(dmma_m8n8k4<4>, sms * 2, 256, 20000, 8.0 * 4, "dmma_m8n8k4_acc4_2cta_w8", out);
  // m16n8k16: 2048 FMAs per warp-instruction = 64 per thread
  run(dmma_m16n8k16<4>, sms, 256, 4000, 64.0 * 4, "dmma_m16n8k16_acc4_w8", out);
  run(dmma_m16n8k16<2>, sms, 512, 4000, 64.0 * 2, "dmma_m16n8k16_acc2_w16", out);
  // DFMA
  run(dfma_loop<8>, sms, 256, 40000, 8.0, "dfma_acc8_w8", out);
  run(dfma_loop<8>, sms * 4, 256, 40000, 8.0, "dfma_acc8_4cta_w8", out);
  run(dfma_loop<16>, sms * 2, 512, 40000, 16.0, "dfma_acc16_2cta_w16", out);
  // sustained DMMA ~3 s for clock/power behaviour
  run(dmma_m8n8k4<8>, sms, 256, 400000, 8.0 * 8, "dmma_m8n8k4_sustained", out);
  return 0;
}
