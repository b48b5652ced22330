// Dependent-latency probe (cycles per op, one warp): DFMA, DMUL, MUFU.RSQ64H,
// double shfl, the call-free sqrt_rcp_pos chain and div_pos (common.cuh).
#include <cstdio>
#include "../paper_1907_01063_b200/csrc/common.cuh"
using namespace stancl;
__global__ void probe(double seed, long long* out, double* sink) {
  double x = seed + threadIdx.x * 1e-3;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) x = fma(x, 0.999999, 1e-9);
  t1 = clock64(); out[0] = (t1 - t0) / 1024;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) x = x * 1.0000001;
  t1 = clock64(); out[1] = (t1 - t0) / 1024;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) { double r; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r + 1.0; }
  t1 = clock64(); out[2] = (t1 - t0) / 1024;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + 1e-9;
  t1 = clock64(); out[3] = (t1 - t0) / 1024;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { double sq, y; sqrt_rcp_pos(x + 2.0, sq, y); x = sq * 0.5 + y; }
  t1 = clock64(); out[4] = (t1 - t0) / 256;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { double sq, y; scaled_sqrt_rcp(x + 2.0, sq, y); x = sq * 0.5 + y; }
  t1 = clock64(); out[5] = (t1 - t0) / 256;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) x = div_pos(x, 1.37, 0.7299270072992701) + 1.0;
  t1 = clock64(); out[6] = (t1 - t0) / 1024;
  __shared__ double sm[64];
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) { sm[threadIdx.x] = x; __syncwarp(); x = sm[(threadIdx.x + 1) & 31] + 1e-9; __syncwarp(); }
  t1 = clock64(); out[7] = (t1 - t0) / 1024;
  sink[threadIdx.x] = x;
}
int main() {
  long long* d; double* s; cudaMalloc(&d, 64); cudaMalloc(&s, 256);
  probe<<<1, 32>>>(1.5, d, s);
  long long h[8]; cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
  const char* nm[] = {"dfma", "dmul", "mufu.rsq64h(+dadd)", "shfl.f64(+dadd)", "sqrt_rcp_pos chain(+2 ops)", "scaled_sqrt_rcp(+2 ops)", "div_pos(+dadd)", "sts+syncwarp+lds(+dadd)"};
  for (int i = 0; i < 8; ++i) printf("%-30s %lld cycles/iter\n", nm[i], h[i]);
  return 0;
}
