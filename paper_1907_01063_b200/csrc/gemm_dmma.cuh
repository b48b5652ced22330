// gemm_dmma.cuh -- FP64 tensor-core (DMMA) tile GEMM used by every O(n^3)
// step of the path:
//   F3  SYRK trailing update   A22 -= L21 L21^T
//   R3  rank-nb update         B_bar -= C_bar R
//   R2  long-K contraction     W = C_bar^T [B C]         (split-K as in
//                                                          the paper's large-k GEMM)
//   R1/R5 products             C_bar D^-1, S R
//
// C[M x N] (row-major, ldc) = beta*C + sign * op(A) op(B), all row-major storage:
//   A_KMAJ: A is M x K (A[m*lda + k])      else K x M (A[k*lda + m])
//   B_KMAJ: B is N x K (B[n*ldb + k])      else K x N (B[k*ldb + n])
// MODE_FULL    every BM x BN tile of C.  A may alias C when N == BN-multiple covering
//              all of K's columns of the same rows (each CTA reads its rows before its
//              epilogue).  lower_only: store only r >= c (relative to C's origin).
// MODE_LOWER   square C (M x M): only tiles that touch the lower triangle are launched
//              (triangular grid), stores masked to r >= c.
// MODE_SPLITK  acc starts at 0; blockIdx.z takes K range [z*kps, (z+1)*kps) and writes
//              P[z][M][N] (row-major, ld N); a separate kernel reduces in fixed order.
// Requirements (the driver guarantees them by padding to multiples of 128):
//   M % BM == 0, N % BN == 0, K % 16 == 0 (kps too); 16-B aligned pointers; even ld.
//
// Design (SURVEY.md §7 hard part 1): warp tile 64 x 32 (or 32 x 32) -> 32 (16)
// DMMA.8x8x4 per k4 step against 12 (8) LDS.64; cp.async 16-B chunks into a
// STAGES-deep ring of padded shared tiles (row pitch = 4 mod 16 doubles, so the 16
// lanes of an LDS.64 phase hit 16 distinct 8-byte bank pairs).  A fragments are
// negated with a sign-bit XOR (integer pipe, not the shared FP64 pipe).  With
// beta = 1 the accumulators start from C, so every C element sees one FMA chain
// c <- c - a*b in ascending k (the oracle's order, R12).
#pragma once
#include "common.cuh"

namespace stancl {

// MODE_CYC: MODE_FULL restricted to the lower tiles of a 2-D block-cyclic
// local array (persistent TMA GEMM only; its item map carries the per-block-
// column prefix table, so plain MODE_FULL launches do not)
enum GemmMode { MODE_FULL = 0, MODE_LOWER = 1, MODE_SPLITK = 2, MODE_CYC = 3 };

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
  int lower_only;   // MODE_FULL: mask stores to r >= c
  const int* status;  // optional: skip work if *status != 0
  int pingpong;     // serialise the MMA main loops of co-resident CTAs (per-SM token)
  // TMA kernel, MODE_FULL, BM = 128, BN = 64: block-cyclic lower mask (the
  // distributed forward's trailing update, rank (cy_p, cy_q) of a cy_P x cy_Q grid).
  // C is a rectangle of 256 x 256 blocks whose local block (i, j) is global tile
  // (I, J) = ((cy_li + i) cy_P + cy_p, (cy_lj + j) cy_Q + cy_q): tiles with I < J are
  // skipped (no loads, no stores), I == J blocks keep their lower part only.
  int cyc = 0, cy_P = 1, cy_p = 0, cy_Q = 1, cy_q = 0, cy_li = 0, cy_lj = 0;
  // TMA kernel, MODE_FULL: triangular operands (TRI_* bits of op(A) M x K,
  // op(B) K x N): each output tile contracts only the k-slabs that can be
  // nonzero -- the skipped terms are exact zeros
  int tri = 0;
};


// Per-SM MMA token ("ping-pong" between the CTAs resident on one SM): a CTA
// issues its prologue loads, then waits for the token, runs its DMMA main loop
// and releases the token before its epilogue, so one CTA's prologue/epilogue
// (HBM latency) overlaps the other's tensor work instead of both CTAs running
// in lockstep.  One warp per SMSP already saturates the FP64 pipe
// (tools/dmma_inner.cu), so serialising the main loops costs nothing.
__device__ int g_sm_mma_token[1024];

namespace gemm {

// tile configurations
template <int BM_, int BN_, int WARPS_M_, int WARPS_N_, int STAGES_, int MIN_CTAS_, int BK_ = 16>
struct Cfg {
  static constexpr int BM = BM_, BN = BN_, WARPS_M = WARPS_M_, WARPS_N = WARPS_N_;
  static constexpr int STAGES = STAGES_, MIN_CTAS = MIN_CTAS_, BK = BK_;
  static constexpr int THREADS = 32 * WARPS_M * WARPS_N;
  static constexpr int WTM = BM / WARPS_M, WTN = BN / WARPS_N;  // warp tile
  static constexpr int MI = WTM / 8, NI = WTN / 8;               // DMMA blocks per warp
};
using CfgBig = Cfg<128, 128, 2, 4, 4, 1>;   // 8 warps of 64x32, 1 CTA/SM
using CfgMid = Cfg<128, 64, 2, 2, 3, 2>;    // 4 warps of 64x32, 2 CTAs/SM
using CfgW8 = Cfg<128, 64, 4, 2, 3, 2>;     // 8 warps of 32x32, 2 CTAs/SM
using CfgW16 = Cfg<128, 128, 4, 4, 4, 1>;   // 16 warps of 32x32, 1 CTA/SM
using CfgW8K32 = Cfg<128, 64, 4, 2, 3, 1, 32>;  // w8 with 32-deep slabs, 1 CTA/SM
using CfgW8K32S2 = Cfg<128, 64, 4, 2, 2, 2, 32>;  // w8, 32-deep double buffer, 2 CTAs/SM
using CfgMidK32 = Cfg<128, 64, 2, 2, 2, 2, 32>;   // mid, 32-deep double buffer, 2 CTAs/SM

// padded shared tile of one BK-slab: k-major rows of BK+4 doubles, or BK rows of
// ROWS+4 doubles (both pitches are 4 mod 16)
template <int ROWS, bool KMAJ, int BK>
struct Tile {
  static constexpr int PITCH = KMAJ ? (BK + 4) : (ROWS + 4);
  static constexpr int ELEMS = KMAJ ? (ROWS * (BK + 4)) : (BK * (ROWS + 4));
  static constexpr int CHUNKS = ROWS * BK / 2;  // 16-B chunks per slab
};

template <class C, bool AK, bool BKM>
constexpr int smem_bytes() {
  return C::STAGES * (Tile<C::BM, AK, C::BK>::ELEMS + Tile<C::BN, BKM, C::BK>::ELEMS) * (int)sizeof(double);
}
}  // namespace gemm

// load one BK-slab of a ROWS-row/col operand tile into shared memory
template <int ROWS, bool KMAJ, int BK, int THREADS>
__device__ __forceinline__ void load_tile(double* s, const double* g, long long ld, int row0, int k0,
                                          int tid) {
  using T = gemm::Tile<ROWS, KMAJ, BK>;
#pragma unroll
  for (int c = tid; c < T::CHUNKS; c += THREADS) {
    if constexpr (KMAJ) {
      constexpr int CPR = BK / 2;  // chunks per row
      const int r = c / CPR, ch = c % CPR;
      cp_async16(s + r * T::PITCH + ch * 2, g + (long long)(row0 + r) * ld + k0 + ch * 2);
    } else {
      constexpr int CPR = ROWS / 2;  // chunks per k-row
      const int r = c / CPR, ch = c % CPR;
      cp_async16(s + r * T::PITCH + ch * 2, g + (long long)(k0 + r) * ld + row0 + ch * 2);
    }
  }
}

template <int ROWS, bool KMAJ, int BK>
__device__ __forceinline__ double frag(const double* s, int rc, int k) {
  using T = gemm::Tile<ROWS, KMAJ, BK>;
  if constexpr (KMAJ) return s[rc * T::PITCH + k];
  else return s[k * T::PITCH + rc];
}

__device__ __forceinline__ double xor_sign(double v, unsigned long long m) {
  return __longlong_as_double(__double_as_longlong(v) ^ (long long)m);
}

// triangular tile enumeration for MODE_LOWER with BM = R * BN: tile-row tm holds
// column tiles tn = 0 .. R*tm + R - 1; b -> (tm, tn)
template <int R>
__device__ __forceinline__ void tri_index(int b, int& tm, int& tn) {
  // cumulative count before row t: R * t (t + 1) / 2
  // single-precision estimate (MUFU, keeps the FP64 pipe free), fixed up exactly
  int t = (int)((sqrtf(8.0f * (float)b / R + 1.0f) - 1.0f) * 0.5f);
  while (R * (t + 1) * (t + 2) / 2 <= b) ++t;
  while (R * t * (t + 1) / 2 > b) --t;
  tm = t;
  tn = b - R * t * (t + 1) / 2;
}

template <class CF, bool A_KMAJ, bool B_KMAJ, int MODE>
__global__ void __launch_bounds__(CF::THREADS, CF::MIN_CTAS) gemm_dmma_kernel(GemmArgs p) {
  using namespace gemm;
  constexpr int BM = CF::BM, BN = CF::BN, STAGES = CF::STAGES, THREADS = CF::THREADS;
  constexpr int MI = CF::MI, NI = CF::NI, BK = CF::BK;
  using TA = Tile<BM, A_KMAJ, BK>;
  using TB = Tile<BN, B_KMAJ, BK>;
  pdl_enter();
  if (cta_status_set(p.status)) return;
  extern __shared__ __align__(16) double smem[];
  double* sA = smem;
  double* sB = smem + STAGES * TA::ELEMS;

  int tm, tn, kbeg, kend;
  if constexpr (MODE == MODE_LOWER) {
    tri_index<BM / BN>(blockIdx.x, tm, tn);
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
  const int wm = warp / CF::WARPS_N, wn = warp % CF::WARPS_N;
  const int g = lane >> 2, t = lane & 3;
  const int ktiles = (kend - kbeg) / BK;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) {
      load_tile<BM, A_KMAJ, BK, THREADS>(sA + s * TA::ELEMS, p.A, p.lda, m0, kbeg + s * BK, tid);
      load_tile<BN, B_KMAJ, BK, THREADS>(sB + s * TB::ELEMS, p.B, p.ldb, n0, kbeg + s * BK, tid);
    }
    cp_async_commit();
  }

  // sign = -1 is applied by negating the accumulator on the way in and out
  // (acc = -C; acc += a b; C = -acc), which is exact and keeps the DMMA
  // operands straight from shared memory
  const unsigned long long smask = (p.sign < 0) ? 0x8000000000000000ull : 0ull;
  double acc[MI][NI][2];
  double* Cout;
  long long ldo;
  bool load_c = false;
  if constexpr (MODE == MODE_SPLITK) {
    Cout = p.C + (long long)blockIdx.z * p.M * p.N;
    ldo = p.N;
  } else {
    Cout = p.C;
    ldo = p.ldc;
    load_c = p.beta != 0;
  }
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) {
      if (load_c) {
        const int r = m0 + wm * CF::WTM + i * 8 + g, c = n0 + wn * CF::WTN + j * 8 + 2 * t;
        const double2 v = *reinterpret_cast<const double2*>(Cout + (long long)r * ldo + c);
        acc[i][j][0] = xor_sign(v.x, smask);
        acc[i][j][1] = xor_sign(v.y, smask);
      } else {
        acc[i][j][0] = acc[i][j][1] = 0.0;
      }
    }
  unsigned smid = 0;
  if (p.pingpong) {
    // make the C loads and the first slab land before taking the token
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NI; ++j) asm volatile("" : "+d"(acc[i][j][0]), "+d"(acc[i][j][1]));
    cp_async_wait<STAGES - 2>();
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if (tid == 0) {
      while (atomicCAS(&g_sm_mma_token[smid], 0, 1) != 0) __nanosleep(64);
    }
    __syncthreads();
  }

  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nk = kt + STAGES - 1;
      if (nk < ktiles) {
        const int slot = nk % STAGES;
        load_tile<BM, A_KMAJ, BK, THREADS>(sA + slot * TA::ELEMS, p.A, p.lda, m0, kbeg + nk * BK, tid);
        load_tile<BN, B_KMAJ, BK, THREADS>(sB + slot * TB::ELEMS, p.B, p.ldb, n0, kbeg + nk * BK, tid);
      }
      cp_async_commit();
    }
    const double* a_s = sA + (kt % STAGES) * TA::ELEMS;
    const double* b_s = sB + (kt % STAGES) * TB::ELEMS;
#pragma unroll
    for (int s = 0; s < BK / 4; ++s) {
      const int k = 4 * s + t;
      double af[MI], bf[NI];
#pragma unroll
      for (int i = 0; i < MI; ++i) af[i] = frag<BM, A_KMAJ, BK>(a_s, wm * CF::WTM + i * 8 + g, k);
#pragma unroll
      for (int j = 0; j < NI; ++j) bf[j] = frag<BN, B_KMAJ, BK>(b_s, wn * CF::WTN + j * 8 + g, k);
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();
  if (p.pingpong) {
    __syncthreads();
    if (tid == 0) atomicExch(&g_sm_mma_token[smid], 0);
  }

  const bool mask = (MODE == MODE_LOWER) || (MODE == MODE_FULL && p.lower_only);
  const bool crosses = mask && (n0 + BN - 1 > m0);  // tile has elements with c > r
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) {
      const int r = m0 + wm * CF::WTM + i * 8 + g, c = n0 + wn * CF::WTN + j * 8 + 2 * t;
      double* dst = Cout + (long long)r * ldo + c;
      if (crosses) {
        if (r >= c) dst[0] = xor_sign(acc[i][j][0], smask);
        if (r >= c + 1) dst[1] = xor_sign(acc[i][j][1], smask);
      } else {
        *reinterpret_cast<double2*>(dst) = make_double2(xor_sign(acc[i][j][0], smask), xor_sign(acc[i][j][1], smask));
      }
    }
}

// host-side launcher
template <class CF, bool A_KMAJ, bool B_KMAJ, int MODE>
cudaError_t launch_gemm(const GemmArgs& p, int splits, cudaStream_t st) {
  constexpr int smem = gemm::smem_bytes<CF, A_KMAJ, B_KMAJ>();
  auto kern = gemm_dmma_kernel<CF, A_KMAJ, B_KMAJ, MODE>;
  static bool attr_set = false;  // per template instantiation
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  dim3 grid;
  if (MODE == MODE_LOWER) {
    constexpr int R = CF::BM / CF::BN;
    const int T = p.M / CF::BM;
    grid = dim3(R * T * (T + 1) / 2, 1, 1);
  } else {
    grid = dim3(p.N / CF::BN, p.M / CF::BM, MODE == MODE_SPLITK ? splits : 1);
  }
  if (grid.x == 0 || grid.y == 0) return cudaSuccess;
  return launch_pdl(kern, grid, CF::THREADS, smem, st, p);
  return cudaGetLastError();
}

}  // namespace stancl
