// Dependent-latency probe (cycles per op, one warp): DFMA, DMUL, MUFU.RSQ64H,
// double shfl, the call-free sqrt_rcp_pos chain and div_pos (common.cuh), DMMA.8x8x4
// dependent / independent, DFMA issue, dependent LDS.
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
  // DMMA.8x8x4: dependent chain on one accumulator, then 4 independent accumulators (one warp)
  double c0 = x, c1 = x, d0 = x, d1 = x, e0 = x, e1 = x, f0 = x, f1 = x;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) dmma_8x8x4(c0, c1, 1e-9, 1e-9);
  t1 = clock64(); out[8] = (t1 - t0) / 1024;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
    dmma_8x8x4(c0, c1, 1e-9, 1e-9); dmma_8x8x4(d0, d1, 1e-9, 1e-9);
    dmma_8x8x4(e0, e1, 1e-9, 1e-9); dmma_8x8x4(f0, f1, 1e-9, 1e-9);
  }
  t1 = clock64(); out[9] = (t1 - t0) / 1024;
  // independent DFMAs (8 chains), cycles per instruction
  double y0 = x, y1 = x + 1, y2 = x + 2, y3 = x + 3, y4 = x + 4, y5 = x + 5, y6 = x + 6, y7 = x + 7;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
    y0 = fma(y0, 0.999, 1e-9); y1 = fma(y1, 0.999, 1e-9); y2 = fma(y2, 0.999, 1e-9); y3 = fma(y3, 0.999, 1e-9);
    y4 = fma(y4, 0.999, 1e-9); y5 = fma(y5, 0.999, 1e-9); y6 = fma(y6, 0.999, 1e-9); y7 = fma(y7, 0.999, 1e-9);
  }
  t1 = clock64(); out[10] = (t1 - t0) / 2048;
  // LDS.64 broadcast, dependent (address from the loaded value)
  sm[threadIdx.x] = 0.0;
  __syncwarp();
  int idx = 0;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) idx = (int)sm[idx];
  t1 = clock64(); out[11] = (t1 - t0) / 1024;
  sink[threadIdx.x] = x + c0 + c1 + d0 + d1 + e0 + e1 + f0 + f1 + y0 + y1 + y2 + y3 + y4 + y5 + y6 + y7 + idx;
}
int main() {
  long long* d; double* s; cudaMalloc(&d, 128); cudaMalloc(&s, 256);
  probe<<<1, 32>>>(1.5, d, s);
  long long h[12]; cudaMemcpy(h, d, 96, cudaMemcpyDeviceToHost);
  const char* nm[] = {"dfma", "dmul", "mufu.rsq64h(+dadd)", "shfl.f64(+dadd)", "sqrt_rcp_pos chain(+2 ops)", "scaled_sqrt_rcp(+2 ops)", "div_pos(+dadd)", "sts+syncwarp+lds(+dadd)", "dmma dependent", "dmma 4 independent (per instr)", "dfma 8 independent (per instr)", "lds.64 dependent (+cvt)"};
  for (int i = 0; i < 12; ++i) printf("%-30s %lld cycles/iter\n", nm[i], h[i]);
  return 0;
}
