// gp.cu -- NEXT-1/NEXT-2 kernels around the hot path:
// the single right-hand-side triangular solve (the paper's triangular_solve,
// PAPER.md:231-238) and the O(n^2) pieces of the GP marginal log density and
// its gradient (the per-gradient work of the paper's GP example, PAPER.md:
// 470-479 §4.2).  The O(n^3) work -- Cholesky and its adjoint -- is the hot
// path (api.cu); everything here is memory- or latency-bound.
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace stancl {

static inline int grid_cap(long long work, int threads, int cap = 148 * 8) {
  long long b = (work + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return (int)b;
}

// ------------------------------------------------------------ triangular solve
// L x = b (TRANS = false) or L^T x = b (TRANS = true), L lower with positive
// diagonal, one right-hand side.  Sync-free blocked substitution: one CTA per
// 64-row block, blocks taken in dependency order from an atomic ticket (so a
// CTA only ever waits on blocks whose CTAs are already resident); a CTA
// streams the off-diagonal tiles it needs as their x blocks are published
// (per-block ready flags), then solves its 64 x 64 diagonal tile by
// substitution (ascending j for L, descending for L^T) and publishes its x.
// Reads each entry of L's lower triangle once: n^2/2 * 8 bytes per solve.
constexpr int TV = 64;

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <bool TRANS>
__global__ void __launch_bounds__(256) trsv_kernel(const double* __restrict__ L, int64_t ld, int64_t n,
                                                   const double* b, double* x, int* flags, int* ticket,
                                                   const int* status) {
  // no early exit on a set status: the CTAs wait on each other's ready flags, so a
  // per-CTA decision could strand a waiter (the result is unspecified on failure)
  (void)status;
  __shared__ double Ld[TV][TV + 1];
  __shared__ double rc[TV];
  __shared__ double part[8][TV];
  __shared__ int s_t;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_t = atomicAdd(ticket, 1);
  __syncthreads();
  const int nblk = (int)((n + TV - 1) / TV);
  const int ib = TRANS ? nblk - 1 - s_t : s_t;
  const int64_t r0 = (int64_t)ib * TV;
  const int rows = (int)(n - r0 < TV ? n - r0 : TV);
  for (int idx = tid; idx < TV * TV; idx += 256) {
    const int r = idx / TV, c = idx % TV;
    Ld[r][c] = (r < rows && c <= r) ? L[(r0 + r) * ld + r0 + c] : 0.0;
  }
  if (tid < rows) rc[tid] = rcp_pos(L[(r0 + tid) * ld + r0 + tid]);
  // off-diagonal contributions; every warp streams its share of each tile
  double acc[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q] = 0.0;
  if (!TRANS) {
    // row r0 + 8 warp + q, columns of block jb: lanes over columns (coalesced)
    // the tile's L entries are loaded BEFORE waiting for its x block, so their
    // latency overlaps the wait on the dependency chain
    for (int jb = 0; jb < ib; ++jb) {
      const int64_t c0 = (int64_t)jb * TV;
      double l0[8], l1[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int r = warp * 8 + q;
        const double* Lr = L + (r0 + (r < rows ? r : 0)) * ld + c0;
        l0[q] = __ldcs(Lr + lane);
        l1[q] = __ldcs(Lr + 32 + lane);
      }
      if (lane == 0)
        while (ld_acquire(flags + jb) == 0) {
        }
      __syncwarp();
      const double x0 = __ldcg(x + c0 + lane), x1 = __ldcg(x + c0 + 32 + lane);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        acc[q] = fma(l0[q], x0, acc[q]);
        acc[q] = fma(l1[q], x1, acc[q]);
      }
    }
    // fixed-order butterfly over the lanes: part[warp][row]
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      double v = acc[q];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) part[0][warp * 8 + q] = v;
    }
  } else {
    // column r0 + lane (+32) of L, rows of block jb: warp w takes rows 8w..8w+7
    for (int jb = nblk - 1; jb > ib; --jb) {
      const int64_t j0 = (int64_t)jb * TV;
      const int jrows = (int)(n - j0 < TV ? n - j0 : TV);
      double l0[8], l1[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int j = warp * 8 + q;
        const double* Lj = L + (j0 + (j < jrows ? j : 0)) * ld + r0;
        l0[q] = (j < jrows && lane < rows) ? __ldcs(Lj + lane) : 0.0;
        l1[q] = (j < jrows && lane + 32 < rows) ? __ldcs(Lj + 32 + lane) : 0.0;
      }
      if (lane == 0)
        while (ld_acquire(flags + jb) == 0) {
        }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int j = warp * 8 + q;
        const double xj = (j < jrows) ? __ldcg(x + j0 + j) : 0.0;
        acc[0] = fma(l0[q], xj, acc[0]);
        acc[1] = fma(l1[q], xj, acc[1]);
      }
    }
    part[warp][lane] = acc[0];
    part[warp][32 + lane] = acc[1];
  }
  __syncthreads();
  if (warp == 0) {
    // right-hand sides of rows lane, lane + 32
    double h[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int r = lane + 32 * s;
      double off = 0.0;
      if (!TRANS) {
        off = part[0][r];
      } else {
#pragma unroll
        for (int w = 0; w < 8; ++w) off += part[w][r];
      }
      h[s] = (r < rows) ? (b[r0 + r] - off) : 0.0;
    }
    // substitution over the tile; row j's right-hand side lives in lane j%32,
    // slot j/32; its quotient is broadcast and applied to the later rows
    if (!TRANS) {
      for (int j = 0; j < rows; ++j) {
        const bool hi = j >= 32;
        const double own = div_pos(hi ? h[1] : h[0], Ld[j][j], rc[j]);
        const double xj = __shfl_sync(0xffffffffu, own, j & 31);
        if (lane == (j & 31)) {
          if (hi) h[1] = xj;
          else h[0] = xj;
        }
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const int r = lane + 32 * t;
          if (r > j && r < rows) h[t] = fma(-Ld[r][j], xj, h[t]);
        }
      }
    } else {
      for (int j = rows - 1; j >= 0; --j) {
        const bool hi = j >= 32;
        const double own = div_pos(hi ? h[1] : h[0], Ld[j][j], rc[j]);
        const double xj = __shfl_sync(0xffffffffu, own, j & 31);
        if (lane == (j & 31)) {
          if (hi) h[1] = xj;
          else h[0] = xj;
        }
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const int r = lane + 32 * t;
          if (r < j) h[t] = fma(-Ld[j][r], xj, h[t]);
        }
      }
    }
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int r = lane + 32 * s;
      if (r < rows) x[r0 + r] = h[s];
    }
    __threadfence();
    __syncwarp();
    if (lane == 0) st_release(flags + ib, 1);
  }
}

cudaError_t trsv(const double* L, int64_t ld, int64_t n, const double* b, double* x, bool trans, int* flags,
                 const int* status, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  Prof prof_(PROF_GP, (double)n * n, st, 4.0 * (double)n * (n + 1) + 24.0 * n);
  const int nblk = (int)((n + TV - 1) / TV);
  // flags[0..nblk) ready words, flags[nblk] the ticket
  cudaError_t e = cudaMemsetAsync(flags, 0, sizeof(int) * (nblk + 1), st);
  if (e != cudaSuccess) return e;
  if (trans)
    trsv_kernel<true><<<nblk, 256, 0, st>>>(L, ld, n, b, x, flags, flags + nblk, status);
  else
    trsv_kernel<false><<<nblk, 256, 0, st>>>(L, ld, n, b, x, flags, flags + nblk, status);
  return cudaGetLastError();
}

// ------------------------------------------------------------ GP log density
// lp = -1/2 z.z - sum log L_ii - n/2 log(2 pi), one CTA, fixed-order tree
__global__ void __launch_bounds__(256) gp_lp_kernel(const double* L, int64_t ld, int64_t n, const double* z,
                                                    double* out, const int* status) {
  if (cta_status_set(status)) return;
  __shared__ double s_zz[256], s_ld[256];
  double zz = 0.0, lg = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += 256) {
    zz = fma(z[i], z[i], zz);
    lg += log(L[i * ld + i]);
  }
  s_zz[threadIdx.x] = zz;
  s_ld[threadIdx.x] = lg;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      s_zz[threadIdx.x] += s_zz[threadIdx.x + o];
      s_ld[threadIdx.x] += s_ld[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = -0.5 * s_zz[0] - s_ld[0] - 0.5 * (double)n * 1.8378770664093454835606594728112;
}

// L_bar = tril(a z^T) - diag(1 / L_ii), lower triangle only (d lp / d L)
__global__ void gp_lbar_kernel(const double* L, int64_t ld, int64_t n, const double* a, const double* z, double* W,
                               int64_t ldw, const int* status) {
  if (cta_status_set(status)) return;
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const double ai = a[i];
    double* Wi = W + i * ldw;
    for (int64_t j = threadIdx.x; j <= i; j += blockDim.x) {
      double v = ai * z[j];
      if (j == i) v -= 1.0 / L[i * ld + i];
      Wi[j] = v;
    }
  }
}

// per-CTA partial sums of A_bar_ij dK_ij/dtheta over i >= j (theta = alpha, rho, sigma)
constexpr int GP_RED_CTAS = 148 * 4;
__global__ void __launch_bounds__(256) gp_hyper_partial_kernel(const double* A, int64_t lda, int64_t n,
                                                               const double* x, double alpha, double rho,
                                                               double sigma, double* partial,
                                                               const int* status) {
  if (cta_status_set(status)) return;
  __shared__ double s[3][256];
  const double c = -0.5 / (rho * rho), ra = 2.0 * alpha, rr = alpha * alpha / (rho * rho * rho);
  double g0 = 0.0, g1 = 0.0, g2 = 0.0;
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const double xi = x[i];
    const double* Ai = A + i * lda;
    for (int64_t j = threadIdx.x; j <= i; j += 256) {
      const double d = xi - x[j];
      const double e = exp(d * d * c);
      const double ab = Ai[j];
      g0 = fma(ab, ra * e, g0);
      g1 = fma(ab, rr * e * (d * d), g1);
      if (j == i) g2 = fma(ab, 2.0 * sigma, g2);
    }
  }
  s[0][threadIdx.x] = g0;
  s[1][threadIdx.x] = g1;
  s[2][threadIdx.x] = g2;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o)
#pragma unroll
      for (int k = 0; k < 3; ++k) s[k][threadIdx.x] += s[k][threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x < 3) partial[blockIdx.x * 3 + threadIdx.x] = s[threadIdx.x][0];
}

__global__ void gp_hyper_final_kernel(const double* partial, int nparts, double* out, const int* status) {
  if (cta_status_set(status)) return;
  if (threadIdx.x < 3) {
    double v = 0.0;
    for (int p = 0; p < nparts; ++p) v += partial[p * 3 + threadIdx.x];
    out[threadIdx.x] = v;
  }
}

__global__ void negate_kernel(const double* a, double* y, int64_t n, const int* status) {
  if (cta_status_set(status)) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = -a[i];
}

cudaError_t gp_lp(const double* L, int64_t ld, int64_t n, const double* z, double* out, const int* status,
                  cudaStream_t st) {
  Prof prof_(PROF_GP, 3.0 * n, st, 16.0 * n);
  gp_lp_kernel<<<1, 256, 0, st>>>(L, ld, n, z, out, status);
  return cudaGetLastError();
}

cudaError_t gp_lbar(const double* L, int64_t ld, int64_t n, const double* a, const double* z, double* W,
                    int64_t ldw, const int* status, cudaStream_t st) {
  Prof prof_(PROF_GP, (double)n * (n + 1) / 2.0, st, 4.0 * (double)n * (n + 1));
  gp_lbar_kernel<<<grid_cap(n, 1, 148 * 16), 256, 0, st>>>(L, ld, n, a, z, W, ldw, status);
  return cudaGetLastError();
}

size_t gp_hyper_scratch_doubles() { return (size_t)GP_RED_CTAS * 3; }

cudaError_t gp_hyper(const double* A, int64_t lda, int64_t n, const double* x, double alpha, double rho,
                     double sigma, double* partial, double* out, const int* status, cudaStream_t st) {
  Prof prof_(PROF_GP, 8.0 * (double)n * (n + 1) / 2.0, st, 4.0 * (double)n * (n + 1));
  const int ctas = (int)(n < GP_RED_CTAS ? (n > 0 ? n : 1) : GP_RED_CTAS);
  gp_hyper_partial_kernel<<<ctas, 256, 0, st>>>(A, lda, n, x, alpha, rho, sigma, partial, status);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  gp_hyper_final_kernel<<<1, 32, 0, st>>>(partial, ctas, out, status);
  return cudaGetLastError();
}

cudaError_t negate(const double* a, double* y, int64_t n, const int* status, cudaStream_t st) {
  Prof prof_(PROF_GP, 0.0, st, 16.0 * n);
  negate_kernel<<<grid_cap(n, 256), 256, 0, st>>>(a, y, n, status);
  return cudaGetLastError();
}

}  // namespace stancl
