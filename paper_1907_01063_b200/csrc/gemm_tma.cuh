// gemm_tma.cuh -- the production FP64 tensor-core GEMM: persistent,
// warp-specialised, TMA-fed DMMA tiles.
//
// Used by every O(n^3) step of the path:
//   F3  SYRK trailing update   A22 -= L21 L21^T
//   R3  rank-nb update         B_bar -= C_bar R
//   R2  long-K contraction     W = C_bar^T [B C]        (split-K as the
//                                                        paper's large-k GEMM)
//   R5  R_bar -= S R
// Semantics: C[M x N] = beta*C + sign * op(A) op(B), row-major storage with the
// layout flags and modes of gemm_dmma.cuh (A_KMAJ: A is M x K, else K x M;
// B_KMAJ: B is N x K, else K x N; MODE_FULL / MODE_LOWER / MODE_SPLITK).
//
// Why this shape (measurements in profiles/r01_gemm_notes.md):
//  * FP64 MMA on sm_100a is warp-level mma.sync (DMMA.8x8x4, 16 cycles per
//    instruction per SM sub-partition); there is no tcgen05 .kind::f64.  Fed
//    from shared memory the DMMA loop reaches 35-37 TFLOP/s, but every
//    thread-issued staging scheme (cp.async + __syncthreads, 1 or 2 CTAs/SM,
//    persistent or not) stalled at 26-31 TFLOP/s.
//  * So one PRODUCER warp moves all operand slabs with the TMA engine:
//    k-contiguous operands as one 2-D tensor copy per slab (box 16 x rows,
//    SWIZZLE_128B), m/n-contiguous operands as one 1-D bulk copy per k-row
//    (cp.async.bulk, rows of 512 B-1 KB).  Completion is byte-counted on a
//    per-slot "full" mbarrier; the 8 CONSUMER warps wait on it, run LDS + DMMA
//    and release the slot on an "empty" mbarrier.  No CTA-wide barrier in the
//    main loop; one CTA per SM walks a list of work items (persistent).
//  * Bank conflicts: within a k4 step lane (g, t) uses k = kappa(s, t) =
//    4 * ((((s & 1) ^ (t >> 1)) << 1) | (s >> 1)) + t, a permutation of the 16
//    k of a slab that is conflict-free for BOTH the 128B-swizzled k-major
//    tiles and the padded (pitch = 4 mod 16) m/n-major tiles.  A and B use the
//    same permutation, so the contraction is unchanged.
//  * C (beta = 1) is prefetched per lane into private shared slots one item
//    ahead; sign = -1 is applied by negating the accumulator on the way in and
//    out (exact), so the DMMA operands come straight from shared memory.
#pragma once
#include <cuda.h>

#include "gemm_dmma.cuh"

namespace stancl {

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// 1-D bulk copy global -> shared (SASS UBLKCP)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// 2-D tensor copy global -> shared (SASS UTMALDG)
__device__ __forceinline__ void tma_g2s_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

namespace tg {
constexpr int BK = 16;
template <int BM_, int BN_, int WARPS_M_, int WARPS_N_, int STAGES_, int MINB_ = 1, bool CPREF_ = true,
          int BKS_ = 16>
struct Cfg {
  static constexpr int BM = BM_, BN = BN_, WARPS_M = WARPS_M_, WARPS_N = WARPS_N_, STAGES = STAGES_;
  static constexpr int BKS = BKS_;       // slab depth (k per pipeline stage): 16 or 32
  static constexpr int MINB = MINB_;     // CTAs per SM (launch bound)
  static constexpr bool CPREF = CPREF_;  // prefetch C through shared memory
  static constexpr int NCONS = 32 * WARPS_M * WARPS_N;  // consumer threads
  static constexpr int WTM = BM / WARPS_M, WTN = BN / WARPS_N;
  static constexpr int MI = WTM / 8, NI = WTN / 8;
};
using CfgT = Cfg<128, 64, 4, 2, 4>;  // 8 consumer warps of 32 x 32 + 1 producer warp
using CfgT2 = Cfg<128, 64, 4, 2, 3, 2, false>;  // same, 2 CTAs/SM, C straight from global
using CfgT2P = Cfg<128, 64, 4, 2, 2, 2, true>;  // 2 CTAs/SM, double-buffered ring, C prefetch
using CfgT32 = Cfg<128, 64, 4, 2, 3, 1, true, 32>;  // 32-deep slabs (two TMA boxes per operand)
using CfgT128 = Cfg<128, 128, 2, 4, 3, 1, true, 16>;  // 128x128 tiles, 8 consumer warps of 64x32

constexpr int align1k(int b) { return (b + 1023) / 1024 * 1024; }
// shared slab of ROWS rows/cols and depth BKS: k-major = BKS/16 dense sub-tiles of
// ROWS x 128-B rows (one TMA box each, 128B swizzle); m/n-major = BKS rows of
// ROWS + 4 doubles (bulk row copies, padded)
template <int ROWS, bool KMAJ, int BKS = 16>
struct Slab {
  static constexpr int PITCH = KMAJ ? BK : ROWS + 4;
  static constexpr int BYTES = align1k((KMAJ ? ROWS * BKS : BKS * (ROWS + 4)) * 8);
  static constexpr unsigned TX = ROWS * BKS * 8;  // bytes landed per slab
};
template <class CF, bool AK, bool BKM>
struct Smem {
  static constexpr int A = 0;
  static constexpr int B = CF::STAGES * Slab<CF::BM, AK, CF::BKS>::BYTES;
  static constexpr int C = B + CF::STAGES * Slab<CF::BN, BKM, CF::BKS>::BYTES;
  static constexpr int BAR = C + (CF::CPREF ? CF::BM * CF::BN * 8 : 0);
  static constexpr int TOTAL = BAR + 2 * CF::STAGES * 8 + 1024;  // + alignment slack
};

__device__ __forceinline__ int kappa(int s, int t) {
  return 4 * (((((s & 1) ^ (t >> 1)) << 1)) | (s >> 1)) + t;
}
// element (row/col rc, k) of a slab; k in [0, BKS)
template <int ROWS, bool KMAJ>
__device__ __forceinline__ double frag(const double* s, int rc, int k) {
  if constexpr (KMAJ) {
    const int kk = k & 15;
    return s[(k >> 4) * ROWS * BK + rc * BK + ((((kk >> 1) ^ (rc & 7)) << 1) | (kk & 1))];
  } else {
    return s[k * (ROWS + 4) + rc];
  }
}
}  // namespace tg

template <class CF, int MODE, bool EXT = false>
struct TItemMap {
  int ntn, ntm, ntiles, ktiles_full;
  // MODE_FULL: enumerate the last first_cols tile columns first (a fused
  // launch's dependency tiles, TFuse), then the rest row-major
  int first_cols = 0;
  // block-cyclic mode (MODE_CYC): items enumerate, per 256-wide
  // block column j, only its tile rows from the first block row that reaches
  // the diagonal (RB f_j) down; cyc_pref[j] = first item of block column j
  static constexpr int kCycMax = (MODE == MODE_CYC) ? 512 : 1;  // only MODE_CYC launches carry the table
  int cyc_nb = 0;
  int cyc_pref[kCycMax + 1];
  // item -> tile (tm, tn) in the rectangle (cyc) or row-major (otherwise)
  __device__ __forceinline__ void tile_of(const GemmArgs& p, int tile, int& tm, int& tn) const {
    if constexpr (MODE == MODE_CYC) {
      {
        int lo = 0, hi = cyc_nb;  // largest j with cyc_pref[j] <= tile
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (cyc_pref[mid] <= tile) lo = mid;
          else hi = mid;
        }
        // a 256 x 256 block holds RB x CB tiles of BM x BN
        constexpr int RB = 256 / CF::BM, CB = 256 / CF::BN;
        static_assert(RB * CF::BM == 256 && CB * CF::BN == 256, "cyclic tiles must divide the 256-wide blocks");
        const int rows = (cyc_pref[lo + 1] - cyc_pref[lo]) / CB;  // tile rows of block column lo
        const int first = RB * (p.M / 256) - rows;                  // = RB f_j
        const int local = tile - cyc_pref[lo];
        tm = first + local / CB;
        tn = CB * lo + local % CB;
        return;
      }
    }
    if constexpr (MODE == MODE_SPLITK) {
      // column-major over tiles: the M tiles that share one B slab (the long
      // m x k operand, streamed once per split) are adjacent items, so they run
      // at the same time on neighbouring CTAs and the second read hits L2
      tn = tile / ntm;
      tm = tile - tn * ntm;
      return;
    }
    if constexpr (EXT && MODE == MODE_FULL) {  // the fused kernel's orderings only
      if (first_cols > 0) {
        const int d = ntm * first_cols;
        if (tile < d) {
          tm = tile / first_cols;
          tn = ntn - first_cols + (tile - tm * first_cols);
        } else {
          const int t2 = tile - d, w = ntn - first_cols;
          tm = t2 / w;
          tn = t2 - tm * w;
        }
        return;
      }
      // a triangular operand makes the items' K extents unequal: enumerate
      // longest first (tiles are dealt to the CTAs round-robin, so the long
      // items land in the first round and the short ones fill the second)
      if (p.tri & (TRI_B_LOWER | TRI_B_UPPER)) {
        tn = tile / ntm;
        tm = tile - tn * ntm;
        if (p.tri & TRI_B_UPPER) tn = ntn - 1 - tn;  // K = n0 + BN: longest at the right
        return;
      }
      if (p.tri & TRI_A_LOWER) {  // K = m0 + BM: longest at the bottom
        tm = ntm - 1 - tile / ntn;
        tn = tile - (ntm - 1 - tm) * ntn;
        return;
      }
    }
    tm = tile / ntn;
    tn = tile - tm * ntn;
  }
  // block-cyclic lower mask (GemmArgs::cyc): is the item computed, and the
  // diagonal offset d of its block (elements kept iff r >= c + d) if masked
  __device__ __forceinline__ bool valid(const GemmArgs& p, int item, bool& masked, int& d) const {
    masked = false;
    d = 0;
    if constexpr (MODE != MODE_CYC) {
      return true;
    } else {
      int tm, tn;
      tile_of(p, item, tm, tn);
      const int bi = tm / (256 / CF::BM), bj = tn / (256 / CF::BN);
      const long long I = (long long)(p.cy_li + bi) * p.cy_P + p.cy_p, J = (long long)(p.cy_lj + bj) * p.cy_Q + p.cy_q;
      if (I < J) return false;
      if (I > J) return true;
      d = (bi - bj) * 256;
      const int rr0 = (tm % (256 / CF::BM)) * CF::BM, cc0 = (tn % (256 / CF::BN)) * CF::BN;
      if (rr0 + CF::BM - 1 < cc0) return false;  // wholly above the block diagonal
      masked = true;
      return true;
    }
  }
  __device__ __forceinline__ int next_valid(const GemmArgs& p, int item, int stride, int nitems) const {
    bool m;
    int d;
    while (item < nitems && !valid(p, item, m, d)) item += stride;
    return item;
  }
  __device__ __forceinline__ void get(const GemmArgs& p, int item, int& m0, int& n0, int& kbeg, int& ns,
                                      int& z) const {
    int tm, tn, tile = item;
    z = 0;
    if constexpr (MODE == MODE_SPLITK) {
      z = item / ntiles;
      tile = item - z * ntiles;
    }
    if constexpr (MODE == MODE_LOWER) {
      tri_index<CF::BM / CF::BN>(tile, tm, tn);
    } else {
      tile_of(p, tile, tm, tn);
    }
    m0 = tm * CF::BM;
    n0 = tn * CF::BN;
    if constexpr (MODE == MODE_SPLITK) {
      kbeg = z * p.kps;
      ns = (min(p.K, kbeg + p.kps) - kbeg) / CF::BKS;
    } else {
      kbeg = 0;
      ns = ktiles_full;
      if constexpr (MODE == MODE_FULL) {
        if (p.tri) {
          int kend = p.K;
          if (p.tri & TRI_A_LOWER) kend = min(kend, m0 + CF::BM);  // op(A)(m, k) = 0 for k > m
          if (p.tri & TRI_A_UPPER) kbeg = max(kbeg, m0);           // op(A)(m, k) = 0 for k < m
          if (p.tri & TRI_B_LOWER) kbeg = max(kbeg, n0);           // op(B)(k, n) = 0 for k < n
          if (p.tri & TRI_B_UPPER) kend = min(kend, n0 + CF::BN);  // op(B)(k, n) = 0 for k > n
          kbeg = kbeg / CF::BKS * CF::BKS;
          kend = (kend + CF::BKS - 1) / CF::BKS * CF::BKS;
          ns = kend > kbeg ? (kend - kbeg) / CF::BKS : 0;
        }
      }
    }
  }
};

// Two GEMM problems in one persistent launch (MODE_FULL, same layouts, B not
// k-major): items [0, n1) are problem 1 (p, map), [n1, nitems) problem 2
// (p2, map2, A through the second tensor map).  Problem 2 may read what
// problem 1 writes: the first `dep` items of problem 1 each add 1 to *cnt when
// their tile is stored (release), and problem 2's producer waits until *cnt >=
// target (acquire, then a generic -> async proxy fence) before its first TMA
// load.  Problem-2 items come last in every CTA's list and all CTAs of the
// persistent grid are resident, so the wait always ends.
template <class CF>
struct TFuse {
  GemmArgs p2;
  TItemMap<CF, MODE_FULL, true> map2;
  int n1 = 0x7fffffff;
  int* cnt = nullptr;
  int dep = 0;
  int target = 0;
};

__device__ __forceinline__ int ld_acquire_gpu(const int* a) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(a) : "memory");
  return v;
}

template <int ROWS, bool KMAJ, int BKS>
__device__ __forceinline__ void produce_slab(double* dst, const CUtensorMap* map, const double* g, long long ld,
                                             int row0, int k0, int lane, uint64_t* bar) {
  if constexpr (KMAJ) {
#pragma unroll
    for (int h = 0; h < BKS / 16; ++h)
      if (lane == h) tma_g2s_2d(dst + h * ROWS * tg::BK, map, k0 + 16 * h, row0, bar);
  } else {
    constexpr int P = ROWS + 4;
    if (lane < BKS) bulk_g2s(dst + lane * P, g + (long long)(k0 + lane) * ld + row0, ROWS * 8, bar);
  }
}

template <class CF, bool A_KMAJ, bool B_KMAJ, int MODE>
__global__ void __launch_bounds__(CF::NCONS + 32, CF::MINB)
    gemm_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    GemmArgs p, int nitems, TItemMap<CF, MODE> map) {
  using namespace tg;
  constexpr int BM = CF::BM, BN = CF::BN, STAGES = CF::STAGES, NCONS = CF::NCONS;
  constexpr int MI = CF::MI, NI = CF::NI;
  constexpr int BKS = CF::BKS;
  using SA = Slab<BM, A_KMAJ, BKS>;
  using SB = Slab<BN, B_KMAJ, BKS>;
  using SM = Smem<CF, A_KMAJ, B_KMAJ>;
  pdl_enter();
  if (cta_status_set(p.status)) return;
  if ((int)blockIdx.x >= nitems) return;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-B aligned slab base (128B-swizzle atoms) as an OFFSET from the shared
  // array: integer round-tripping the pointer would drop its address space and
  // turn every fragment read into a generic 64-bit LD instead of an LDS
  const unsigned sraw = (unsigned)__cvta_generic_to_shared(smem_raw);
  unsigned char* base = smem_raw + ((1024u - (sraw & 1023u)) & 1023u);
  double* sA = reinterpret_cast<double*>(base + SM::A);
  double* sB = reinterpret_cast<double*>(base + SM::B);
  double* sC = reinterpret_cast<double*>(base + SM::C);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + SM::BAR);
  uint64_t* empty = full + STAGES;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);            // the producer's arrive.expect_tx
      mbar_init(&empty[s], NCONS / 32);  // one arrive per consumer warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  __syncthreads();

  if (warp == NCONS / 32) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      if (A_KMAJ) prefetch_tmap(&tmA);
      if (B_KMAJ) prefetch_tmap(&tmB);
    }
    int it = 0;
    for (int item = map.next_valid(p, blockIdx.x, gridDim.x, nitems); item < nitems;
         item = map.next_valid(p, item + gridDim.x, gridDim.x, nitems)) {
      int m0, n0, kbeg, ns, z;
      map.get(p, item, m0, n0, kbeg, ns, z);
      for (int s = 0; s < ns; ++s, ++it) {
        const int slot = it % STAGES, round = it / STAGES;
        if (round > 0) mbar_wait(&empty[slot], (round - 1) & 1);
        if (lane == 0) mbar_arrive_expect_tx(&full[slot], SA::TX + SB::TX);
        __syncwarp();
        const int k0 = kbeg + s * BKS;
        produce_slab<BM, A_KMAJ, BKS>(sA + slot * (SA::BYTES / 8), &tmA, p.A, p.lda, m0, k0, lane, &full[slot]);
        produce_slab<BN, B_KMAJ, BKS>(sB + slot * (SB::BYTES / 8), &tmB, p.B, p.ldb, n0, k0, lane, &full[slot]);
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int wm = warp / CF::WARPS_N, wn = warp % CF::WARPS_N;
  const int g = lane >> 2, t = lane & 3;
  const bool need_c = (MODE != MODE_SPLITK) && p.beta != 0;
  const unsigned long long smask = (p.sign < 0) ? 0x8000000000000000ull : 0ull;
  double2* myC = reinterpret_cast<double2*>(sC) + (size_t)warp * MI * NI * 32 + lane;
  auto load_c = [&](int m0, int n0) {
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NI; ++j) {
        const int r = m0 + wm * CF::WTM + i * 8 + g, c = n0 + wn * CF::WTN + j * 8 + 2 * t;
        cp_async16(myC + (i * NI + j) * 32, p.C + (long long)r * p.ldc + c);
      }
    cp_async_commit();
  };
  int m0, n0, kbeg, ns, z;
  const int first = map.next_valid(p, blockIdx.x, gridDim.x, nitems);
  if (first >= nitems) return;
  map.get(p, first, m0, n0, kbeg, ns, z);
  if (CF::CPREF && need_c) load_c(m0, n0);
  int kap[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) kap[s] = kappa(s, t);
  int it = 0;
  double acc[MI][NI][2];
  for (int item = first; item < nitems;) {
    const int nxt_item = map.next_valid(p, item + gridDim.x, gridDim.x, nitems);
    if (need_c && CF::CPREF) {
      cp_async_wait<0>();
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) {
          const double2 v = myC[(i * NI + j) * 32];
          acc[i][j][0] = xor_sign(v.x, smask);
          acc[i][j][1] = xor_sign(v.y, smask);
        }
    } else if (need_c) {
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) {
          const int r = m0 + wm * CF::WTM + i * 8 + g, c = n0 + wn * CF::WTN + j * 8 + 2 * t;
          const double2 v = *reinterpret_cast<const double2*>(p.C + (long long)r * p.ldc + c);
          acc[i][j][0] = xor_sign(v.x, smask);
          acc[i][j][1] = xor_sign(v.y, smask);
        }
    } else {
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    }
    // lower-triangular outputs: a warp whose whole 32 x 32 sub-tile lies above the
    // diagonal (the upper half of a diagonal block's tiles) only keeps the slab
    // protocol; its sub-partition's DMMA pipe then serves the other warp alone
    const bool idle = MODE == MODE_LOWER && (m0 + wm * CF::WTM + CF::WTM - 1 < n0 + wn * CF::WTN);
    for (int s = 0; s < ns; ++s, ++it) {
      const int slot = it % STAGES, round = it / STAGES;
      mbar_wait(&full[slot], round & 1);
      const double* a_s = sA + slot * (SA::BYTES / 8);
      const double* b_s = sB + slot * (SB::BYTES / 8);
      if (!idle) {
#pragma unroll
        for (int kk = 0; kk < BKS / 4; ++kk) {
          const int k = ((kk >> 2) << 4) + kap[kk & 3];
          double af[MI], bf[NI];
#pragma unroll
          for (int i = 0; i < MI; ++i) af[i] = tg::frag<BM, A_KMAJ>(a_s, wm * CF::WTM + i * 8 + g, k);
#pragma unroll
          for (int j = 0; j < NI; ++j) bf[j] = tg::frag<BN, B_KMAJ>(b_s, wn * CF::WTN + j * 8 + g, k);
#pragma unroll
          for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < NI; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      if (CF::CPREF && need_c && s == 0) {
        // prefetch the next item's C into the private slots only now: the DMMAs
        // above consumed acc (loaded from these slots), and asm-volatile order
        // keeps this cp.async behind them, so the refill cannot overtake the read
        const int nxt = nxt_item;
        if (nxt < nitems) {
          int m1, n1, kb1, ns1, z1;
          map.get(p, nxt, m1, n1, kb1, ns1, z1);
          load_c(m1, n1);
        }
      }
    }
    // epilogue: registers -> global
    double* Cout;
    long long ldo;
    if constexpr (MODE == MODE_SPLITK) {
      Cout = p.C + (long long)z * p.M * p.N;
      ldo = p.N;
    } else {
      Cout = p.C;
      ldo = p.ldc;
    }
    bool cmask;
    int dd;
    map.valid(p, item, cmask, dd);  // block-cyclic diagonal block: keep r >= c + dd
    const bool mask = (MODE == MODE_LOWER) || ((MODE == MODE_FULL || MODE == MODE_CYC) && (p.lower_only || cmask));
    const bool crosses = mask && (n0 + BN - 1 + dd > m0);
#pragma unroll
    for (int i = 0; i < (idle ? 0 : MI); ++i)
#pragma unroll
      for (int j = 0; j < NI; ++j) {
        const int r = m0 + wm * CF::WTM + i * 8 + g, c = n0 + wn * CF::WTN + j * 8 + 2 * t;
        double* dst = Cout + (long long)r * ldo + c;
        const double v0 = xor_sign(acc[i][j][0], smask), v1 = xor_sign(acc[i][j][1], smask);
        if (crosses) {
          if (r >= c + dd) dst[0] = v0;
          if (r >= c + 1 + dd) dst[1] = v1;
        } else {
          *reinterpret_cast<double2*>(dst) = make_double2(v0, v1);
        }
      }
    if (nxt_item < nitems) map.get(p, nxt_item, m0, n0, kbeg, ns, z);
    item = nxt_item;
  }
}

// The two-problem (fused) variant of gemm_tma_kernel (TFuse): same pipeline and
// main loop; per item it resolves which problem the tile belongs to.  Kept as a
// separate kernel so the single-problem launches compile exactly as before.
template <class CF, bool A_KMAJ, bool B_KMAJ>
__global__ void __launch_bounds__(CF::NCONS + 32, CF::MINB)
    gemm_tma_fused_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ GemmArgs p, int nitems, TItemMap<CF, MODE_FULL, true> map,
                    const __grid_constant__ CUtensorMap tmA2,
                    const __grid_constant__ TFuse<CF> fz) {
  using namespace tg;
  constexpr int MODE = MODE_FULL;
  constexpr bool FUSE = true;
  constexpr int BM = CF::BM, BN = CF::BN, STAGES = CF::STAGES, NCONS = CF::NCONS;
  constexpr int MI = CF::MI, NI = CF::NI;
  constexpr int BKS = CF::BKS;
  using SA = Slab<BM, A_KMAJ, BKS>;
  using SB = Slab<BN, B_KMAJ, BKS>;
  using SM = Smem<CF, A_KMAJ, B_KMAJ>;
  pdl_enter();
  if (cta_status_set(p.status)) return;
  if ((int)blockIdx.x >= nitems) return;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-B aligned slab base (128B-swizzle atoms) as an OFFSET from the shared
  // array: integer round-tripping the pointer would drop its address space and
  // turn every fragment read into a generic 64-bit LD instead of an LDS
  const unsigned sraw = (unsigned)__cvta_generic_to_shared(smem_raw);
  unsigned char* base = smem_raw + ((1024u - (sraw & 1023u)) & 1023u);
  double* sA = reinterpret_cast<double*>(base + SM::A);
  double* sB = reinterpret_cast<double*>(base + SM::B);
  double* sC = reinterpret_cast<double*>(base + SM::C);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + SM::BAR);
  uint64_t* empty = full + STAGES;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);            // the producer's arrive.expect_tx
      mbar_init(&empty[s], NCONS / 32);  // one arrive per consumer warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  __syncthreads();

  if (warp == NCONS / 32) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      if (A_KMAJ) prefetch_tmap(&tmA);
      if (B_KMAJ) prefetch_tmap(&tmB);
    }
    int it = 0;
    bool waited = false;
    for (int item = map.next_valid(p, blockIdx.x, gridDim.x, nitems); item < nitems;
         item = map.next_valid(p, item + gridDim.x, gridDim.x, nitems)) {
      int m0, n0, kbeg, ns, z;
      const bool two = FUSE && item >= fz.n1;
      const GemmArgs& q = two ? fz.p2 : p;
      if (two) {
        fz.map2.get(q, item - fz.n1, m0, n0, kbeg, ns, z);
        if (!waited && fz.cnt) {
          if (lane == 0) {
            while (ld_acquire_gpu(fz.cnt) < fz.target) __nanosleep(100);
            asm volatile("fence.proxy.async.global;\n" ::: "memory");
          }
          __syncwarp();
          waited = true;
        }
      } else {
        map.get(p, item, m0, n0, kbeg, ns, z);
      }
      const CUtensorMap* ta = two ? &tmA2 : &tmA;
      for (int s = 0; s < ns; ++s, ++it) {
        const int slot = it % STAGES, round = it / STAGES;
        if (round > 0) mbar_wait(&empty[slot], (round - 1) & 1);
        if (lane == 0) mbar_arrive_expect_tx(&full[slot], SA::TX + SB::TX);
        __syncwarp();
        const int k0 = kbeg + s * BKS;
        produce_slab<BM, A_KMAJ, BKS>(sA + slot * (SA::BYTES / 8), ta, q.A, q.lda, m0, k0, lane, &full[slot]);
        produce_slab<BN, B_KMAJ, BKS>(sB + slot * (SB::BYTES / 8), &tmB, q.B, q.ldb, n0, k0, lane, &full[slot]);
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int wm = warp / CF::WARPS_N, wn = warp % CF::WARPS_N;
  const int g = lane >> 2, t = lane & 3;
  double2* myC = reinterpret_cast<double2*>(sC) + (size_t)warp * MI * NI * 32 + lane;
  auto load_c = [&](const GemmArgs& q, int m0, int n0) {
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NI; ++j) {
        const int r = m0 + wm * CF::WTM + i * 8 + g, c = n0 + wn * CF::WTN + j * 8 + 2 * t;
        cp_async16(myC + (i * NI + j) * 32, q.C + (long long)r * q.ldc + c);
      }
    cp_async_commit();
  };
  const GemmArgs* const P1 = &p;  // __grid_constant__: addresses of the parameters themselves
  const GemmArgs* const P2 = &fz.p2;
  auto resolve = [&](int item, int& m0, int& n0, int& kbeg, int& ns, int& z) -> const GemmArgs* {
    if (FUSE && item >= fz.n1) {
      fz.map2.get(fz.p2, item - fz.n1, m0, n0, kbeg, ns, z);
      return P2;
    }
    map.get(p, item, m0, n0, kbeg, ns, z);
    return P1;
  };
  auto needs_c = [&](const GemmArgs& q) { return (MODE != MODE_SPLITK) && q.beta != 0; };
  int m0, n0, kbeg, ns, z;
  const int first = map.next_valid(p, blockIdx.x, gridDim.x, nitems);
  if (first >= nitems) return;
  const GemmArgs* q = resolve(first, m0, n0, kbeg, ns, z);
  if (CF::CPREF && needs_c((FUSE ? *q : p))) load_c((FUSE ? *q : p), m0, n0);
  int kap[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) kap[s] = kappa(s, t);
  int it = 0;
  double acc[MI][NI][2];
  for (int item = first; item < nitems;) {
    const int nxt_item = map.next_valid(p, item + gridDim.x, gridDim.x, nitems);
    const bool need_c = needs_c((FUSE ? *q : p));
    const unsigned long long smask = ((FUSE ? *q : p).sign < 0) ? 0x8000000000000000ull : 0ull;
    if (need_c && CF::CPREF) {
      cp_async_wait<0>();
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) {
          const double2 v = myC[(i * NI + j) * 32];
          acc[i][j][0] = xor_sign(v.x, smask);
          acc[i][j][1] = xor_sign(v.y, smask);
        }
    } else if (need_c) {
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) {
          const int r = m0 + wm * CF::WTM + i * 8 + g, c = n0 + wn * CF::WTN + j * 8 + 2 * t;
          const double2 v = *reinterpret_cast<const double2*>((FUSE ? *q : p).C + (long long)r * (FUSE ? *q : p).ldc + c);
          acc[i][j][0] = xor_sign(v.x, smask);
          acc[i][j][1] = xor_sign(v.y, smask);
        }
    } else {
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    }
    for (int s = 0; s < ns; ++s, ++it) {
      const int slot = it % STAGES, round = it / STAGES;
      mbar_wait(&full[slot], round & 1);
      const double* a_s = sA + slot * (SA::BYTES / 8);
      const double* b_s = sB + slot * (SB::BYTES / 8);
#pragma unroll
      for (int kk = 0; kk < BKS / 4; ++kk) {
        const int k = ((kk >> 2) << 4) + kap[kk & 3];
        double af[MI], bf[NI];
#pragma unroll
        for (int i = 0; i < MI; ++i) af[i] = tg::frag<BM, A_KMAJ>(a_s, wm * CF::WTM + i * 8 + g, k);
#pragma unroll
        for (int j = 0; j < NI; ++j) bf[j] = tg::frag<BN, B_KMAJ>(b_s, wn * CF::WTN + j * 8 + g, k);
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int j = 0; j < NI; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      if (CF::CPREF && s == 0 && nxt_item < nitems) {
        // prefetch the next item's C into the private slots only now: the DMMAs
        // above consumed acc (loaded from these slots), and asm-volatile order
        // keeps this cp.async behind them, so the refill cannot overtake the read
        int m1, n1, kb1, ns1, z1;
        const GemmArgs* q1 = resolve(nxt_item, m1, n1, kb1, ns1, z1);
        if (needs_c(FUSE ? *q1 : p)) load_c(FUSE ? *q1 : p, m1, n1);
      }
    }
    // epilogue: registers -> global
    double* Cout;
    long long ldo;
    if constexpr (MODE == MODE_SPLITK) {
      Cout = (FUSE ? *q : p).C + (long long)z * (FUSE ? *q : p).M * (FUSE ? *q : p).N;
      ldo = (FUSE ? *q : p).N;
    } else {
      Cout = (FUSE ? *q : p).C;
      ldo = (FUSE ? *q : p).ldc;
    }
    bool cmask = false;
    int dd = 0;
    if (!FUSE || item < fz.n1) map.valid(p, item, cmask, dd);  // block-cyclic diagonal block: keep r >= c + dd
    const bool mask = (MODE == MODE_LOWER) || ((MODE == MODE_FULL || MODE == MODE_CYC) && ((FUSE ? *q : p).lower_only || cmask));
    const bool crosses = mask && (n0 + BN - 1 + dd > m0);
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NI; ++j) {
        const int r = m0 + wm * CF::WTM + i * 8 + g, c = n0 + wn * CF::WTN + j * 8 + 2 * t;
        double* dst = Cout + (long long)r * ldo + c;
        const double v0 = xor_sign(acc[i][j][0], smask), v1 = xor_sign(acc[i][j][1], smask);
        if (crosses) {
          if (r >= c + dd) dst[0] = v0;
          if (r >= c + 1 + dd) dst[1] = v1;
        } else {
          *reinterpret_cast<double2*>(dst) = make_double2(v0, v1);
        }
      }
    if (FUSE && item < fz.dep && fz.cnt) {
      // a dependency tile of the fused problem 2: every consumer's stores, then
      // one release increment
      asm volatile("bar.sync 1, %0;\n" ::"n"(NCONS) : "memory");
      if (tid == 0) {
        __threadfence();
        atomicAdd(fz.cnt, 1);
      }
    }
    if (nxt_item < nitems) q = resolve(nxt_item, m0, n0, kbeg, ns, z);
    item = nxt_item;
  }
}

// ------------------------------------------------------------------ host side
int tma_num_sms();
// k-contiguous operand X[rows][K] (ld doubles): 2-D map, box {16, box_rows}, 128B swizzle
bool make_kmajor_map(CUtensorMap* map, const double* X, long long rows, long long K, long long ld,
                     int box_rows);

template <class CF, bool A_KMAJ, bool B_KMAJ, int MODE>
cudaError_t launch_tma(const GemmArgs& p, int splits, cudaStream_t st, int reserve_sms = 0) {
  using SM = tg::Smem<CF, A_KMAJ, B_KMAJ>;
  auto kern = gemm_tma_kernel<CF, A_KMAJ, B_KMAJ, MODE>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SM::TOTAL);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  CUtensorMap ma, mb;
  memset(&ma, 0, sizeof(ma));
  memset(&mb, 0, sizeof(mb));
  if (A_KMAJ && !make_kmajor_map(&ma, p.A, p.M, p.K, p.lda, CF::BM)) return cudaErrorInvalidValue;
  if (B_KMAJ && !make_kmajor_map(&mb, p.B, p.N, p.K, p.ldb, CF::BN)) return cudaErrorInvalidValue;
  TItemMap<CF, MODE> map;
  map.ntn = p.N / CF::BN;
  map.ntm = p.M / CF::BM;
  map.ktiles_full = p.K / CF::BKS;
  int ntiles;
  if (MODE == MODE_LOWER) {
    constexpr int R = CF::BM / CF::BN;
    const int T = p.M / CF::BM;
    ntiles = R * T * (T + 1) / 2;
  } else {
    ntiles = (p.M / CF::BM) * map.ntn;
  }
  if constexpr (MODE == MODE_CYC) {
    {  // valid tile rows per 256-wide block column
      const int nbc = p.N / 256, nbr = p.M / 256;
      if (nbc > TItemMap<CF, MODE>::kCycMax) return cudaErrorInvalidValue;
      map.cyc_nb = nbc;
      map.cyc_pref[0] = 0;
      for (int j = 0; j < nbc; ++j) {
        const long long J = (long long)(p.cy_lj + j) * p.cy_Q + p.cy_q;
        // first local block row with global I >= J, relative to the rectangle's first row
        long long f = (J > p.cy_p ? (J - p.cy_p + p.cy_P - 1) / p.cy_P : 0) - p.cy_li;
        f = f < 0 ? 0 : (f > nbr ? nbr : f);
        map.cyc_pref[j + 1] = map.cyc_pref[j] + (256 / CF::BM) * (256 / CF::BN) * (int)(nbr - f);
      }
      ntiles = map.cyc_pref[nbc];
    }
  }
  map.ntiles = ntiles;
  const int nitems = ntiles * (MODE == MODE_SPLITK ? splits : 1);
  if (nitems == 0) return cudaSuccess;
  // reserve_sms: SMs left free for kernels on other streams
  const int nsm = (tma_num_sms() - (reserve_sms > 0 && reserve_sms < tma_num_sms() ? reserve_sms : 0)) * CF::MINB;
  const int grid = nitems < nsm ? nitems : nsm;
  return launch_pdl(kern, grid, CF::NCONS + 32, SM::TOTAL, st, ma, mb, p, nitems, map);
}


// Problem 1 (its last first_cols tile columns first, each counted on *cnt when
// stored) and problem 2 (waiting for *cnt >= cnt_base + those tiles) in one
// persistent launch of gemm_tma_fused_kernel: MODE_FULL, B not k-major.
template <class CF, bool A_KMAJ>
cudaError_t launch_tma_fused(const GemmArgs& p, const GemmArgs& p2, int first_cols, int* cnt, int cnt_base,
                             cudaStream_t st, int reserve_sms = 0) {
  using SM = tg::Smem<CF, A_KMAJ, false>;
  auto kern = gemm_tma_fused_kernel<CF, A_KMAJ, false>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SM::TOTAL);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  CUtensorMap ma, mb, ma2;
  memset(&ma, 0, sizeof(ma));
  memset(&mb, 0, sizeof(mb));
  memset(&ma2, 0, sizeof(ma2));
  if (A_KMAJ && !make_kmajor_map(&ma, p.A, p.M, p.K, p.lda, CF::BM)) return cudaErrorInvalidValue;
  if (A_KMAJ && !make_kmajor_map(&ma2, p2.A, p2.M, p2.K, p2.lda, CF::BM)) return cudaErrorInvalidValue;
  auto fill = [](const GemmArgs& q, TItemMap<CF, MODE_FULL, true>& m) {
    m.ntn = q.N / CF::BN;
    m.ntm = q.M / CF::BM;
    m.ktiles_full = q.K / CF::BKS;
    m.ntiles = m.ntm * m.ntn;
    return m.ntiles;
  };
  TItemMap<CF, MODE_FULL, true> map;
  const int n1 = fill(p, map);
  if (first_cols <= 0 || first_cols > map.ntn) return cudaErrorInvalidValue;
  map.first_cols = first_cols;
  TFuse<CF> fz;
  fz.p2 = p2;
  const int n2 = fill(p2, fz.map2);
  fz.n1 = n1;
  fz.cnt = cnt;
  fz.dep = map.ntm * first_cols;
  fz.target = cnt_base + fz.dep;  // *cnt counts monotonically across launches
  const int nitems = n1 + n2;
  if (nitems == 0) return cudaSuccess;
  const int nsm = (tma_num_sms() - (reserve_sms > 0 && reserve_sms < tma_num_sms() ? reserve_sms : 0)) * CF::MINB;
  const int grid = nitems < nsm ? nitems : nsm;
  return launch_pdl(kern, grid, CF::NCONS + 32, SM::TOTAL, st, ma, mb, p, nitems, map, ma2, fz);
}

}  // namespace stancl
