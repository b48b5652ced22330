// common.cuh -- shared device helpers for libstancl (sm_100a only).
//
// FP64 tensor-core math on Blackwell is warp-level mma.sync .f64 (SASS
// DMMA.8x8x4); tcgen05.mma has no .kind::f64 (SURVEY.md §0 finding 2, measured
// 37.1 TFLOP/s peak for DMMA vs 34.2 for DFMA on this pool's B200s,
// profiles/fp64_peak_r01.jsonl).  Operands are staged global -> shared with
// cp.async (LDGSTS) multi-stage pipelines.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "libstancl is written for sm_100a only"
#endif

namespace stancl {

constexpr int NB = 128;  // block size of the blocked algorithms (tile edge)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// D(8x8) += A(8x4, row) * B(4x8, col).  Lane (g = lane>>2, t = lane&3):
//   a = A[g][t], b = B[t][g], c0 = C[g][2t], c1 = C[g][2t+1].
__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Device-side status word shared by the kernels of one call: 0 = fine,
// k > 0 = first failing pivot row + 1 (LAPACK info).  Kernels that see a
// nonzero word exit early (the result is unspecified on failure).
struct Status {
  int info;
};

}  // namespace stancl
