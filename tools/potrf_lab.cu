// Diagonal-tile POTRF lab: per-launch time of candidate 128 x 128 tile
// factorizations (isolated, tile restored before each launch), bitwise
// agreement with the production kernel, and clock64 phase timers.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I ../include -I <nccl include> -o potrf_lab potrf_lab.cu -lcuda -ldl
#include <cstdio>
#include <cmath>
#include <vector>
#define STANCL_POTRF_TIMERS 1
namespace stancl { __device__ long long g_ptimer[8]; }
#include "../paper_1907_01063_b200/csrc/kernels.cu"
using namespace stancl;

__device__ long long g_phase[8];
namespace stancl {
constexpr int TP0 = NB + 1;
__global__ void __launch_bounds__(256, 1) potrf_v0_kernel(double* W, int64_t ld, int64_t k0,
                                                            int* status) {
  if (*status != 0) return;
  __shared__ double colbuf[NB];
  __shared__ double diag_s;
  __shared__ int fail_j;
  const int tid = threadIdx.x;
  const int ti = tid >> 4, tj = tid & 15;
  double* base = W + k0 * ld + k0;
  double T[8][8];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const int r = ti + 16 * a, c = tj + 16 * b;
      T[a][b] = (c <= r) ? base[(long long)r * ld + c] : 0.0;
    }
  if (tid == 0) fail_j = -1;
  bool failed = false;  // uniform across the CTA (every thread tests the same pivot)
#pragma unroll
  for (int jb = 0; jb < 8; ++jb) {
    for (int jt = 0; jt < 16; ++jt) {
      const int j = 16 * jb + jt;
      // diagonal owner (ti == jt, tj == jt) publishes the updated pivot
      if (ti == jt && tj == jt) diag_s = T[jb][jb];
      __syncthreads();
      const double s = diag_s;
      if (!(s > 0.0)) {
        if (tid == 0) fail_j = j;
        failed = true;
        break;
      }
      if (tj == jt) {  // owners of column j (register column jb)
        const double d = sqrt(s);
#pragma unroll
        for (int a = 0; a < 8; ++a) {
          const int r = ti + 16 * a;
          if (r > j) {
            const double l = T[a][jb] / d;
            T[a][jb] = l;
            colbuf[r] = l;
          } else if (r == j) {
            T[a][jb] = d;
          }
        }
      }
      __syncthreads();
      double cr[8], cc[8];
#pragma unroll
      for (int a = 0; a < 8; ++a) cr[a] = colbuf[ti + 16 * a];
#pragma unroll
      for (int b = 0; b < 8; ++b) cc[b] = colbuf[tj + 16 * b];
      // trailing update of columns c > j (rows r <= j of those columns are the
      // strict upper triangle: never read or stored, so left unpredicated)
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        if (tj + 16 * b > j) {
#pragma unroll
          for (int a = 0; a < 8; ++a) T[a][b] = fma(-cr[a], cc[b], T[a][b]);
        }
      }
    }
    if (failed) break;
  }
  __syncthreads();
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const int r = ti + 16 * a, c = tj + 16 * b;
      base[(long long)r * ld + c] = (c <= r) ? T[a][b] : 0.0;  // strict upper of the tile: +0.0
    }
  if (tid == 0 && fail_j >= 0) atomicCAS(status, 0, (int)(k0 + fail_j + 1));
}

}


// ---- call-free correctly rounded helpers for positive normal operands -------
__device__ __forceinline__ double sqrt_pos(double a) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
  const double h = 0.5 * a;
  double e = fma(-h * r, r, 0.5); r = fma(r, e, r);
  e = fma(-h * r, r, 0.5); r = fma(r, e, r);
  const double s = a * r;
  return fma(fma(-s, s, a), 0.5 * r, s);
}
// sq = RN(sqrt(a)) and y = RN(1/sq) from one rsqrt iteration chain
__device__ unsigned long long g_bad[4];
__device__ __forceinline__ unsigned long long mix(unsigned long long z) {
  z += 0x9e3779b97f4a7c15ull; z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull; return z ^ (z >> 31);
}
__global__ void validate(unsigned long long n, int emin, int espan) {
  unsigned long long bad0 = 0, bad1 = 0, bad2 = 0, bad3 = 0;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long u = mix(i), v = mix(i ^ 0xabcdef12345ull);
    // random significands, exponents in [emin, emin + espan)
    const double a = __longlong_as_double((long long)(((unsigned long long)(1023 + emin + (int)(u % espan)) << 52) | (v & 0xfffffffffffffull)));
    const double b = __longlong_as_double((long long)(((unsigned long long)(1023 + emin + (int)((u >> 20) % espan)) << 52) | (mix(v) & 0xfffffffffffffull)));
    const double x = (u >> 63) ? -a : a;
    bad0 += sqrt_pos(b) != sqrt(b);
    const double y = rcp_pos(b);
    bad1 += y != 1.0 / b;
    bad2 += div_pos(x, b, y) != x / b;
    double sq, yy;
    sqrt_rcp_pos(b, sq, yy);
    bad3 += (sq != sqrt(b)) || (yy != 1.0 / sq) || (div_pos(x, sq, yy) != x / sq);
  }
  atomicAdd(&g_bad[0], bad0); atomicAdd(&g_bad[1], bad1); atomicAdd(&g_bad[2], bad2); atomicAdd(&g_bad[3], bad3);
}



// one column of the 32 x 32 warp factorization; templated on the column so
// every register index is a compile-time constant (a runtime-bounded inner loop
// sends row[] to local memory)
template <int J, bool FAST>
__device__ __forceinline__ void wchol_step(double (&row)[32], int lane, double* rc) {
  const double d = __shfl_sync(0xffffffffu, row[J], J);
  const double sq = FAST ? sqrt_pos(d) : sqrt(d);
  const double y = FAST ? rcp_pos(sq) : 1.0 / sq;
  if (lane == J) { row[J] = sq; rc[J] = y; }
  else row[J] = div_pos(row[J], sq, y);
#pragma unroll
  for (int c = J + 1; c < 32; ++c) {
    const double lc = __shfl_sync(0xffffffffu, row[J], c);
    if (lane >= c) row[c] = fma(-row[J], lc, row[c]);
  }
  if constexpr (J + 1 < 32) wchol_step<J + 1, FAST>(row, lane, rc);
}


template <int J>
__device__ __forceinline__ void wchol_step_c(double (&row)[32], int lane, double* rc, double* col) {
  const double d = __shfl_sync(0xffffffffu, row[J], J);
  double sq, y;
  sqrt_rcp_pos(d, sq, y);
  if (lane == J) { row[J] = sq; rc[J] = y; }
  else row[J] = div_pos(row[J], sq, y);
  col[lane] = row[J];
  __syncwarp();
#pragma unroll
  for (int c = J + 1; c < 32; ++c) {
    const double lc = col[c];
    if (lane >= c) row[c] = fma(-row[J], lc, row[c]);
  }
  __syncwarp();
  if constexpr (J + 1 < 32) wchol_step_c<J + 1>(row, lane, rc, col);
}

// ---- B: blocked by 32; warp-shuffle diagonal block; phases timed ----------
template <bool TIMED, bool FAST, bool CV = false>
__global__ void __launch_bounds__(256, 1) potrf_b(double* W, int64_t ld, int* status) {
  extern __shared__ double S[];
  __shared__ int fail_j;
  __shared__ double rc[NB];
  __shared__ double colb[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  long long t0 = clock64(), ta = 0, tb = 0, tc = 0;
  for (int idx = tid; idx < NB * NB; idx += 256) {
    const int r = idx >> 7, c = idx & (NB - 1);
    if (c <= r) S[r * TP + c] = W[(long long)r * ld + c];
  }
  if (tid == 0) fail_j = -1;
  __syncthreads();
  long long tl = clock64();
  for (int c0 = 0; c0 < NB; c0 += 32) {
    long long p0 = clock64();
    if (warp == 0) {
      double row[32];
      double* Sr = S + (c0 + lane) * TP + c0;
#pragma unroll
      for (int c = 0; c < 32; ++c) row[c] = (c <= lane) ? Sr[c] : 0.0;
      if constexpr (CV) wchol_step_c<0>(row, lane, rc + c0, colb);
      else wchol_step<0, FAST>(row, lane, rc + c0);
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (c <= lane) Sr[c] = row[c];
    }
    __syncthreads();
    long long p1 = clock64();
    const int r0 = c0 + 32, R = NB - r0;
    if (R == 0) { ta += p1 - p0; break; }
    if (tid < R) {
      double* Sx = S + (r0 + tid) * TP + c0;
      double x[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) x[c] = Sx[c];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const double l = S[(c0 + j) * TP + c0 + j];
        x[j] = FAST ? div_pos(x[j], l, rc[c0 + j]) : x[j] / l;
#pragma unroll
        for (int c = j + 1; c < 32; ++c) x[c] = fma(-x[j], S[(c0 + c) * TP + c0 + j], x[c]);
      }
#pragma unroll
      for (int c = 0; c < 32; ++c) Sx[c] = x[c];
    }
    __syncthreads();
    long long p2 = clock64();
    {
      const int ti = tid >> 4, tj = tid & 15;
      double acc[6][6];
#pragma unroll
      for (int a = 0; a < 6; ++a)
#pragma unroll
        for (int b = 0; b < 6; ++b) {
          const int i = ti + 16 * a, k = tj + 16 * b;
          acc[a][b] = (i < R && k <= i) ? S[(r0 + i) * TP + r0 + k] : 0.0;
        }
#pragma unroll 4
      for (int j = 0; j < 32; ++j) {
        double xi[6], xk[6];
#pragma unroll
        for (int a = 0; a < 6; ++a) {
          xi[a] = (16 * a < R) ? S[(r0 + ti + 16 * a) * TP + c0 + j] : 0.0;
          xk[a] = (16 * a < R) ? S[(r0 + tj + 16 * a) * TP + c0 + j] : 0.0;
        }
#pragma unroll
        for (int a = 0; a < 6; ++a)
#pragma unroll
          for (int b = 0; b <= a; ++b)
            if (16 * a < R) acc[a][b] = fma(-xi[a], xk[b], acc[a][b]);
      }
#pragma unroll
      for (int a = 0; a < 6; ++a)
#pragma unroll
        for (int b = 0; b <= a; ++b) {
          const int i = ti + 16 * a, k = tj + 16 * b;
          if (i < R && k <= i) S[(r0 + i) * TP + r0 + k] = acc[a][b];
        }
    }
    __syncthreads();
    long long p3 = clock64();
    ta += p1 - p0; tb += p2 - p1; tc += p3 - p2;
  }
  long long te = clock64();
  for (int idx = tid; idx < NB * NB; idx += 256) {
    const int r = idx >> 7, c = idx & (NB - 1);
    W[(long long)r * ld + c] = (c <= r) ? S[r * TP + c] : 0.0;
  }
  if (TIMED && tid == 0) {
    g_phase[0] = tl - t0; g_phase[1] = ta; g_phase[2] = tb; g_phase[3] = tc; g_phase[4] = clock64() - te;
  }
}

__global__ void restore(double* dst, const double* src, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[i] = src[i];
}

int main() {
  const int n = 128;
  std::vector<double> h(n * n);
  std::vector<double> x(n);
  unsigned s = 12345;
  for (int i = 0; i < n; ++i) { s = s * 1664525u + 1013904223u; x[i] = 20.0 * (s >> 8) / 16777216.0 - 10.0; }
  for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) {
    double d = x[i] - x[j]; h[i * n + j] = exp(-0.5 * d * d) + (i == j ? 1e-6 : 0.0); }
  double *orig, *work, *ref; int* status;
  cudaMalloc(&orig, n * n * 8); cudaMalloc(&work, n * n * 8); cudaMalloc(&ref, n * n * 8); cudaMalloc(&status, 4);
  cudaMemcpy(orig, h.data(), n * n * 8, cudaMemcpyHostToDevice);
  const int SM_B = NB * TP * 8;
  cudaFuncSetAttribute(potrf_b<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM_B);
  cudaFuncSetAttribute(potrf_b<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM_B);
  cudaFuncSetAttribute(potrf_b<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM_B);
  cudaFuncSetAttribute(potrf_b<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM_B);
  cudaFuncSetAttribute(potrf_b<false, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM_B);
  cudaFuncSetAttribute(potrf_b<true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM_B);
  auto run = [&](int v) {
    if (v == 0) potrf_v0_kernel<<<1, 256>>>(work, n, 0, status);
    if (v == 7) potrf_tile_kernel<<<1, 256, POTRF_SMEM>>>(work, n, 0, status);
    if (v == 1) potrf_b<false, false><<<1, 256, SM_B>>>(work, n, status);
    if (v == 2) potrf_b<true, false><<<1, 256, SM_B>>>(work, n, status);
    if (v == 3) potrf_b<false, true><<<1, 256, SM_B>>>(work, n, status);
    if (v == 4) potrf_b<true, true><<<1, 256, SM_B>>>(work, n, status);
    if (v == 5) potrf_b<false, true, true><<<1, 256, SM_B>>>(work, n, status);
    if (v == 6) potrf_b<true, true, true><<<1, 256, SM_B>>>(work, n, status);
  };
  const char* names[] = {"v0 register rank-1 (round-1 kernel)", "B blocked32 ieee-calls", "B timed", "B blocked32 call-free", "B call-free timed", "C sqrt_rcp + smem column", "C timed", "production potrf_tile_kernel"};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int R = 200;
  float tc;
  cudaEventRecord(e0); for (int r = 0; r < R; ++r) restore<<<16, 256>>>(work, orig, n * n);
  cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&tc, e0, e1);
  std::vector<double> a(n * n), b(n * n);
  long long ph[8];
  cudaFuncSetAttribute(potrf_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, POTRF_SMEM);
  for (int v = 0; v < 8; ++v) {
    cudaMemset(status, 0, 4);
    restore<<<16, 256>>>(work, orig, n * n); run(v);
    cudaMemcpy(v == 0 ? a.data() : b.data(), work, n * n * 8, cudaMemcpyDeviceToHost);
    float ms;
    cudaEventRecord(e0);
    for (int r = 0; r < R; ++r) { restore<<<16, 256>>>(work, orig, n * n); run(v); }
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    long long ndiff = 0;
    if (v) for (int i = 0; i < n * n; ++i) ndiff += a[i] != b[i];
    printf("%-34s %8.2f us/launch  differ from v0: %lld  err %s\n", names[v], (ms - tc) * 1000.0 / R, ndiff,
           cudaGetErrorString(cudaGetLastError()));
    if (v == 7) {
      long long pt[8] = {0};
      cudaMemcpyToSymbol(g_ptimer, pt, sizeof(pt));
      cudaMemset(status, 0, 4);
      restore<<<16, 256>>>(work, orig, n * n); run(7); cudaDeviceSynchronize();
      cudaMemcpyFromSymbol(pt, g_ptimer, sizeof(pt));
      printf("   production phases (cycles): load %lld  warp-diag %lld  trsm %lld  syrk %lld  store %lld\n", pt[0], pt[1], pt[2], pt[3], pt[4]);
    }
    if (v == 2 || v == 4 || v == 6) {
      cudaMemcpyFromSymbol(ph, g_phase, sizeof(ph));
      printf("   phases (cycles): load %lld  warp-diag %lld  trsm %lld  syrk %lld  store %lld\n", ph[0], ph[1], ph[2], ph[3], ph[4]);
    }
  }
  for (int rng = 0; rng < 3; ++rng) {
    const int emin[3] = {-30, -200, -1000}, espan[3] = {60, 400, 2000};
    unsigned long long z[4] = {0, 0, 0, 0};
    cudaMemcpyToSymbol(g_bad, z, sizeof(z));
    const unsigned long long N = 1ull << 32;
    cudaEventRecord(e0);
    validate<<<148 * 8, 256>>>(N, emin[rng], espan[rng]);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpyFromSymbol(z, g_bad, sizeof(z));
    printf("validate 2^32 samples, exponents [%d, %d): sqrt mismatches %llu, rcp %llu, div %llu, sqrt_rcp+div %llu (%.0f ms) %s\n",
           emin[rng], emin[rng] + espan[rng], z[0], z[1], z[2], z[3], ms, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
