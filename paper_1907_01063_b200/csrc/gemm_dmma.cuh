// gemm_dmma.cuh -- FP64 tensor-core (DMMA) tile GEMM used by every O(n^3)
// step of the path:
//   F3  SYRK trailing update   A22 -= L21 L21^T
//   R3  rank-nb update         B_bar -= C_bar R
//   R2  long-K contraction     W = C_bar^T [B C]         (split-K as in
//                                                          the paper's large-k GEMM)
//   R1/R4/R5 small products     C_bar D^-1, D^T D_bar, D^-T M D^-1, S R
//
// C[M x N] (row-major, ldc) (+)= sign * op(A) op(B), all row-major storage:
//   A_KMAJ: A is M x K (A[m*lda + k])      else K x M (A[k*lda + m])
//   B_KMAJ: B is N x K (B[n*ldb + k])      else K x N (B[k*ldb + n])
// MODE_FULL    every 128x128 tile of C; C = beta*C + sign*AB (beta in {0,1}); A may alias C
//              when N == 128 (each CTA reads all of its own rows before its epilogue)
// MODE_LOWER   square C, tiles with ti >= tj only; diagonal tiles store i >= j only
// MODE_SPLITK  acc starts at 0; blockIdx.z takes K range [z*kps, (z+1)*kps) and writes
//              P[z][M][N] (row-major, ld N); a separate kernel reduces in fixed order
// Requirements (the driver guarantees them by padding to multiples of NB):
//   M, N multiples of 128; K (and kps) multiples of 16; pointers 16-B aligned; ld even.
//
// Design: 256 threads = 8 warps as 2 (M) x 4 (N), warp tile 64 x 32 -> 32 DMMA.8x8x4
// per k4 step against 12 LDS.64; cp.async 16-B chunks into a STAGES-deep ring of
// padded shared tiles (row pitch = 4 mod 16 doubles, so the 16 lanes of each
// LDS.64 phase hit 16 distinct 8-byte bank pairs).  Accumulators are initialised
// from C, and A fragments are negated for sign = -1, so each C element sees one
// FMA chain c <- c - a*b in ascending k (the oracle's order, R12).
#pragma once
#include "common.cuh"

namespace stancl {

enum GemmMode { MODE_FULL = 0, MODE_LOWER = 1, MODE_SPLITK = 2 };

struct GemmArgs {
  const double* A;
  long long lda;
  const double* B;
  long long ldb;
  double* C;        // output (MODE_SPLITK: partial buffer base)
  long long ldc;
  int M, N, K;
  int kps;          // K per split (MODE_SPLITK)
  double sign;      // +1 or -1
  int beta;         // MODE_FULL/LOWER: 1 = accumulate onto C, 0 = overwrite C with the product
  const int* status;  // optional: skip work if *status != 0
};

namespace gemm {
constexpr int BM = 128, BN = 128, BK = 16, STAGES = 4, THREADS = 256;
constexpr int KPITCH = BK + 4;     // k-major tile row pitch (doubles)
constexpr int MPITCH = BM + 4;     // m/n-major tile row pitch (doubles)
template <bool KMAJ>
struct Tile {
  static constexpr int ELEMS = KMAJ ? (BM * KPITCH) : (BK * MPITCH);
};
template <bool AK, bool BK_>
constexpr int smem_bytes() {
  return STAGES * (Tile<AK>::ELEMS + Tile<BK_>::ELEMS) * (int)sizeof(double);
}
}  // namespace gemm

// load one BK-slab of a 128-row/col operand tile into shared memory
template <bool KMAJ>
__device__ __forceinline__ void load_tile(double* s, const double* g, long long ld, int row0, int k0,
                                          int tid) {
  using namespace gemm;
  if constexpr (KMAJ) {
    // 128 rows x 16 doubles = 128 x 8 chunks of 16 B
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int c = tid + i * THREADS;  // 0..1023
      int r = c >> 3, ch = c & 7;
      cp_async16(s + r * KPITCH + ch * 2, g + (long long)(row0 + r) * ld + k0 + ch * 2);
    }
  } else {
    // 16 k-rows x 128 doubles = 16 x 64 chunks
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int c = tid + i * THREADS;
      int r = c >> 6, ch = c & 63;
      cp_async16(s + r * MPITCH + ch * 2, g + (long long)(k0 + r) * ld + row0 + ch * 2);
    }
  }
}

template <bool KMAJ>
__device__ __forceinline__ double frag(const double* s, int rc, int k) {
  using namespace gemm;
  if constexpr (KMAJ) return s[rc * KPITCH + k];
  else return s[k * MPITCH + rc];
}

__device__ __forceinline__ void tri_index(int b, int& ti, int& tj) {
  // b -> (ti, tj), ti >= tj, row-major over the lower triangle of tiles
  int t = (int)((sqrt(8.0 * (double)b + 1.0) - 1.0) * 0.5);
  while ((t + 1) * (t + 2) / 2 <= b) ++t;
  while (t * (t + 1) / 2 > b) --t;
  ti = t;
  tj = b - t * (t + 1) / 2;
}

template <bool A_KMAJ, bool B_KMAJ, int MODE>
__global__ void __launch_bounds__(gemm::THREADS, 1) gemm_dmma_kernel(GemmArgs p) {
  using namespace gemm;
  if (p.status && *p.status != 0) return;
  extern __shared__ __align__(16) double smem[];
  double* sA = smem;
  double* sB = smem + STAGES * Tile<A_KMAJ>::ELEMS;

  int tm, tn, kbeg, kend;
  if constexpr (MODE == MODE_LOWER) {
    tri_index(blockIdx.x, tm, tn);
  } else {
    tn = blockIdx.x;
    tm = blockIdx.y;
  }
  if constexpr (MODE == MODE_SPLITK) {
    kbeg = blockIdx.z * p.kps;
    kend = min(p.K, kbeg + p.kps);
  } else {
    kbeg = 0;
    kend = p.K;
  }
  const int m0 = tm * BM, n0 = tn * BN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;  // 2 x 4 warps
  const int g = lane >> 2, t = lane & 3;
  const int ktiles = (kend - kbeg) / BK;

  // prologue: start the first STAGES-1 slabs
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) {
      load_tile<A_KMAJ>(sA + s * Tile<A_KMAJ>::ELEMS, p.A, p.lda, m0, kbeg + s * BK, tid);
      load_tile<B_KMAJ>(sB + s * Tile<B_KMAJ>::ELEMS, p.B, p.ldb, n0, kbeg + s * BK, tid);
    }
    cp_async_commit();
  }

  double acc[8][4][2];
  double* Cout;
  long long ldo;
  if constexpr (MODE == MODE_SPLITK) {
    Cout = p.C + (long long)blockIdx.z * p.M * p.N;
    ldo = p.N;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  } else {
    Cout = p.C;
    ldo = p.ldc;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (!p.beta) {
          acc[i][j][0] = acc[i][j][1] = 0.0;
          continue;
        }
        const int r = m0 + wm * 64 + i * 8 + g, c = n0 + wn * 32 + j * 8 + 2 * t;
        double2 v = *reinterpret_cast<const double2*>(Cout + (long long)r * ldo + c);
        acc[i][j][0] = v.x;
        acc[i][j][1] = v.y;
      }
  }
  const double sgn = p.sign;

  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      int nk = kt + STAGES - 1;
      if (nk < ktiles) {
        int slot = nk % STAGES;
        load_tile<A_KMAJ>(sA + slot * Tile<A_KMAJ>::ELEMS, p.A, p.lda, m0, kbeg + nk * BK, tid);
        load_tile<B_KMAJ>(sB + slot * Tile<B_KMAJ>::ELEMS, p.B, p.ldb, n0, kbeg + nk * BK, tid);
      }
      cp_async_commit();
    }
    const double* a_s = sA + (kt % STAGES) * Tile<A_KMAJ>::ELEMS;
    const double* b_s = sB + (kt % STAGES) * Tile<B_KMAJ>::ELEMS;
#pragma unroll
    for (int s = 0; s < BK / 4; ++s) {
      const int k = 4 * s + t;
      double af[8], bf[4];
#pragma unroll
      for (int i = 0; i < 8; ++i) af[i] = sgn * frag<A_KMAJ>(a_s, wm * 64 + i * 8 + g, k);
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = frag<B_KMAJ>(b_s, wn * 32 + j * 8 + g, k);
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  // epilogue
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = wm * 64 + i * 8 + g, c = wn * 32 + j * 8 + 2 * t;
      double* dst = Cout + (long long)(m0 + r) * ldo + (n0 + c);
      if (MODE == MODE_LOWER && tm == tn) {
        if (r >= c) dst[0] = acc[i][j][0];
        if (r >= c + 1) dst[1] = acc[i][j][1];
      } else {
        *reinterpret_cast<double2*>(dst) = make_double2(acc[i][j][0], acc[i][j][1]);
      }
    }
}

// host-side launcher
template <bool A_KMAJ, bool B_KMAJ, int MODE>
cudaError_t launch_gemm(const GemmArgs& p, int splits, cudaStream_t st) {
  using namespace gemm;
  constexpr int smem = smem_bytes<A_KMAJ, B_KMAJ>();
  auto kern = gemm_dmma_kernel<A_KMAJ, B_KMAJ, MODE>;
  static bool attr_set = false;  // per template instantiation
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  dim3 grid;
  if (MODE == MODE_LOWER) {
    int T = p.M / BM;
    grid = dim3(T * (T + 1) / 2, 1, 1);
  } else {
    grid = dim3(p.N / BN, p.M / BM, MODE == MODE_SPLITK ? splits : 1);
  }
  if (grid.x == 0 || grid.y == 0) return cudaSuccess;
  kern<<<grid, THREADS, smem, st>>>(p);
  return cudaGetLastError();
}

}  // namespace stancl
