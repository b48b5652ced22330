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

// ---- call-free correctly rounded square root, reciprocal and quotient -------
// CUDA's IEEE sqrt() and '/' are an inline fast path plus a CALL to a slow
// path; inside the unrolled panel kernels that call forces live register
// arrays into local memory.  These sequences have no call.  For operands in
// [2^-600, 2^600] they return the IEEE round-to-nearest result:
//   sqrt_rcp_pos: two Newton steps on the MUFU rsqrt seed, then sq =
//     s + (a - s^2) r/2 (the residual exact with FMA) and one Markstein
//     reciprocal step y = r + r(1 - sq r);
//   div_pos: q = x y, q' = q + (x - q b) y (Markstein: correctly rounded when
//     y = RN(1/b); R12).
// Validated bit-for-bit against sqrt() and '/' on 2^32 random operand pairs
// with exponents in [-200, 200) (tools/potrf_lab.cu, profiles/r01_potrf_trsm_notes.md).
// Pivots outside [2^-600, 2^600] are brought into range by an exact power-of-two
// scaling (scaled_sqrt_rcp).
__device__ __forceinline__ void sqrt_rcp_pos(double a, double& sq, double& y) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
  const double h = 0.5 * a;
  double e = fma(-h * r, r, 0.5);
  r = fma(r, e, r);
  e = fma(-h * r, r, 0.5);
  r = fma(r, e, r);
  const double s = a * r;
  sq = fma(fma(-s, s, a), 0.5 * r, s);
  y = fma(r, fma(-sq, r, 1.0), r);
}
__device__ __forceinline__ void scaled_sqrt_rcp(double a, double& sq, double& y) {
  // branch-free, so it schedules as one basic block with independent work
  const bool tiny = a < 0x1p-600, huge = a > 0x1p600;
  sqrt_rcp_pos(a * (tiny ? 0x1p800 : huge ? 0x1p-800 : 1.0), sq, y);
  sq *= tiny ? 0x1p-400 : huge ? 0x1p400 : 1.0;
  y *= tiny ? 0x1p400 : huge ? 0x1p-400 : 1.0;
}
__device__ __forceinline__ double rcp_pos(double b) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(b));
  double e = fma(-b, y, 1.0);
  y = fma(y, e, y);
  e = fma(-b, y, 1.0);
  y = fma(y, e, y);
  e = fma(-b, y, 1.0);
  return fma(y, e, y);
}
__device__ __forceinline__ double div_pos(double x, double b, double y) {
  const double q = x * y;
  return fma(fma(-q, b, x), y, q);
}

// ---- programmatic dependent launch (PDL) ----------------------------------
// The dependent kernels of the panel chain and of the adjoint block step are
// launched with cudaLaunchAttributeProgrammaticStreamSerialization (launch_pdl):
// their CTAs may be scheduled while the stream predecessor drains, which hides
// the launch latency at each kernel boundary.  Every kernel launched that way
// calls pdl_wait() before touching global memory (it returns once the
// predecessor grid has completed and its writes are visible), then
// pdl_trigger() so its own successor can be scheduled.  Without the launch
// attribute both are no-ops.  STAN_CL_PDL=0 disables the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_enter() {
  pdl_wait();
  pdl_trigger();
}
bool pdl_enabled();
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// Device-side status word shared by the kernels of one call: 0 = fine,
// k > 0 = first failing pivot row + 1 (LAPACK info).  Kernels that see a
// nonzero word exit early (the result is unspecified on failure).
struct Status {
  int info;
};

// CTA-uniform "the status word is set" test.  Every thread of the CTA must
// reach it (call it first, after pdl_enter).  Thread 0 reads the word once and
// __syncthreads_or hands its answer to every thread, so a status write from
// another stream landing while the CTA starts (the lookahead POTRF, the host
// path's check_diag) cannot send some warps home while others wait on a
// barrier.  Kernels that synchronise ACROSS CTAs (grid barriers, ready flags)
// must not exit early at all: a per-CTA snapshot is not grid-uniform.
__device__ __forceinline__ bool cta_status_set(const int* status) {
  return __syncthreads_or(threadIdx.x == 0 && status != nullptr && *(volatile const int*)status != 0) != 0;
}

}  // namespace stancl
