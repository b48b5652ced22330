// kernels.h -- host-side launchers for the libstancl CUDA kernels (internal).
// Every launcher enqueues on `st` and returns the launch error (no sync).
// All matrices are row-major with an explicit leading dimension (doubles).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace stancl {

// ---- launch accounting (gpu_launches in bench.py) and per-class event timing ----
void count_launch(int k = 1);
long long launches();
enum ProfKind {
  PROF_SYRK = 0,       // F3 trailing update outside the lookahead column (DMMA, lower tiles)
  PROF_GEMM = 1,       // R3/R5 DMMA GEMMs (B_bar -= C_bar R, R_bar -= S R)
  PROF_SPLITK = 2,     // R2 long-K contraction C_bar^T [B C] (DMMA, split-K)
  PROF_POTRF = 3,      // F1 diagonal tile
  PROF_TRSM = 4,       // F2 panel solve
  PROF_TRINV = 5,      // R1 batched diagonal-block inverses
  PROF_SMALL = 6,      // R4 128^3 products of the symbolic diagonal step
  PROF_SE = 7,         // F0 covariance build
  PROF_MISC = 8,       // copies, reductions, Phi, checks
  PROF_LOOKAHEAD = 9,  // F3 lookahead column + in-panel update (DMMA)
  PROF_TRMM = 10,      // R1 C_bar <- C_bar D^-1 (DMMA)
  PROF_GP = 11,        // NEXT-1/2: triangular solves, GP log density / gradient reductions
  PROF_KINDS = 12
};
// RAII launch scope: counts the launch and, when profiling is on, brackets it
// with CUDA events on its stream
struct Prof {
  Prof(int kind, double flops, cudaStream_t st, double bytes = 0.0);  // bytes: algorithmic HBM bytes
  ~Prof();
  int kind_;
  double flops_, bytes_;
  cudaStream_t st_;
  cudaEvent_t e0_ = nullptr, e1_ = nullptr;
};
// programmatic dependent launch on/off for the calls that follow (common.cuh;
// the host-streamed entry points turn it off: early-resident dependent CTAs
// would hold SMs the copy-stream kernels of the streamed transfers need)
void pdl_allow(bool on);
void prof_enable(unsigned mask);  // bit k enables class k
bool prof_active();
void prof_reset();
void prof_read(int kind, double* ms, double* flops, long long* count, double* bytes = nullptr);
// timeline of every launch from trace_start (base event on st) to trace_stop
void trace_start(cudaStream_t st);
void trace_stop();
int trace_read(double* out, int max_records);  // 4 doubles per launch: kind, stream id, start, end (ms)

// ---- F0: SE covariance (K1) ----
cudaError_t se_cov(int64_t n, const double* x, double alpha, double rho, double jitter, double* K,
                   cudaStream_t st);

// owned 256-wide block columns of K for rank q of G (block-column-cyclic layout)
cudaError_t se_cov_cols(int64_t n, const double* x, double alpha, double rho, double jitter, double* K,
                        int64_t ld, int G, int q, cudaStream_t st);

// tiles (I, J), I % P == p, J % Q == q, of K for rank (p, q) of a P x Q grid
// (2-D block-cyclic, 256 x 256 tiles; local tile (I / P, J / Q))
cudaError_t se_cov_tiles(int64_t n, const double* x, double alpha, double rho, double jitter, double* K,
                         int64_t ld, int P, int Q, int p, int q, cudaStream_t st);

// ---- layout helpers (K11) ----
// dst tile (d0 + ds*t) <- src tile (s0 + ss*t) for t < cnt (contiguous tiles of `elems` doubles)
cudaError_t copy_tiles(const double* src, int64_t s0, int64_t ss, double* dst, int64_t d0, int64_t ds, int64_t cnt,
                       int64_t elems, cudaStream_t st);
// dst[rows x cols] (ldd) += src (lds); cols even, 16-B aligned rows
cudaError_t add_block(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows, int64_t cols,
                      cudaStream_t st);
// dst[N x N] (ldd) <- lower(src[n x n], lds) with +0.0 strict upper; rows/cols >= n
// become diag_pad * I (diag_pad = 1 for L/A, 0 for adjoints).  N >= n.
cudaError_t copy_lower_pad(const double* src, int64_t n, int64_t lds, double* dst, int64_t N,
                           int64_t ldd, double diag_pad, cudaStream_t st);
// dst[n x n] (ldd) <- lower(src) (lds), strict upper written +0.0
cudaError_t copy_lower_out(const double* src, int64_t lds, double* dst, int64_t n, int64_t ldd,
                           cudaStream_t st);
// dst[rows x cols] (ldd) <- src[rows x cols] (lds); cols even, 16-B aligned rows
cudaError_t copy_block(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows, int64_t cols,
                       cudaStream_t st);
// zero the strict upper triangle in place
cudaError_t zero_upper(double* A, int64_t n, int64_t ld, cudaStream_t st);
// zero the strict upper of the rows x rows diagonal tile at (r0, r0)
cudaError_t zero_tile_upper(double* A, int64_t ld, int64_t r0, int rows, cudaStream_t st);
// rows >= n and columns >= n of the N x N matrix W become diag_pad * I
cudaError_t init_pad(double* W, int64_t n, int64_t N, double diag_pad, cudaStream_t st);

// ---- F1/F2: diagonal tile POTRF (K2) and panel TRSM (K3), NB = 128 ----
// factor W[k0:k0+128, k0:k0+128] in place (lower); on failure status = k0 + j + 1
cudaError_t potrf_tile(double* W, int64_t ld, int64_t k0, int* status, cudaStream_t st);
// C[128 x 128, lower] -= A A^T (A 128 x K, K a multiple of 64 up to 512): the
// lookahead update of the next diagonal tile alone, on ten CTAs (kernels.cu)
cudaError_t diag_tile_update(const double* A, int64_t lda, double* C, int64_t ldc, int K, const int* status,
                             cudaStream_t st);
// rows [r0, r1) of columns [k0, k0+128): X <- X L11^-T (L11 = W[k0.., k0..]), substitution
cudaError_t trsm_panel(double* W, int64_t ld, int64_t k0, int64_t r0, int64_t r1, const int* status,
                       cudaStream_t st);

// ---- DMMA GEMM family (F3, R1, R2, R3, R5) ----
// triangular operands of gemm_full (tri bits; op(A) is M x K, op(B) is K x N):
// each output tile contracts only the k-slabs that can be nonzero
enum TriBits { TRI_A_LOWER = 1, TRI_A_UPPER = 2, TRI_B_LOWER = 4, TRI_B_UPPER = 8 };
// C[M x N] = beta*C + sign * op(A) op(B)   (see gemm_dmma.cuh)
//   a_kmaj: A is M x K row-major (else K x M);  b_kmaj: B is N x K (else K x N)
// lower_only: store only r >= c (relative to C); prof_kind: profiling class;
// allow_persistent = false keeps the one-tile-per-CTA kernel (for work issued on
// the lookahead side stream, which must not hold SMs the trailing update needs);
// reserve_sms: the persistent kernel leaves that many SMs free for other streams
// [R_bar; B_bar] -= [S; C_bar D^-1] R of step s with C_bar' D'^-1 of step s+1 in
// one persistent launch (kernels.cu; gemm_tma.cuh TFuse)
cudaError_t adj_update_fused_trmm(int M1, int N1, int K, const double* A1, int64_t lda1, const double* B1,
                                  int64_t ldb1, double* C1, int64_t ldc1, int M2, const double* A2, int64_t lda2,
                                  const double* B2, int64_t ldb2, double* C2, int64_t ldc2, int first_cols, int* cnt,
                                  int cnt_base, int* dep_out, const int* status, cudaStream_t st);
cudaError_t gemm_full(bool a_kmaj, bool b_kmaj, int M, int N, int K, double sign, int beta,
                      const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                      int64_t ldc, const int* status, cudaStream_t st, int lower_only = 0,
                      int prof_kind = 1, bool allow_persistent = true, int reserve_sms = 0, int tri = 0);
// C[M x N] -= A B^T (A M x K, B N x K, both k-major) on the block-cyclic lower
// tiles of rank (p, q) of a P x Q grid: C's 256 x 256 block (i, j) is global tile
// ((li0 + i) P + p, (lj0 + j) Q + q); blocks above the diagonal are skipped and
// diagonal blocks keep their lower part (the distributed trailing update)
cudaError_t gemm_cyclic_lower(int M, int N, int K, const double* A, int64_t lda, const double* B, int64_t ldb,
                              double* C, int64_t ldc, int P, int p, int Q, int q, int li0, int lj0, const int* status,
                              cudaStream_t st, int reserve_sms = 0);
// lower tiles of square C[M x M] -= A A'^T style: C -= A B^T, A, B both k-major (SYRK)
cudaError_t gemm_lower_nt(int M, int K, const double* A, int64_t lda, const double* B, int64_t ldb,
                          double* C, int64_t ldc, const int* status, cudaStream_t st);
// split-K: P[z][M][N] = op(A) op(B) over K range z*kps..; a_kmaj=false, b_kmaj=false only
cudaError_t gemm_splitk_tn(int M, int N, int K, int splits, int kps, const double* A, int64_t lda,
                           const double* B, int64_t ldb, double* P, const int* status,
                           cudaStream_t st, int reserve_sms = 0);
// dst[r][c] -= sum_{z=0}^{splits-1} P[z][r][c]  (fixed order), r < M, c < N
cudaError_t splitk_reduce_sub(const double* P, int splits, int M, int N, double* dst, int64_t ldd,
                              const int* status, cudaStream_t st);

// R0 + the split-K reduction of rows [j, j+B) (first write to them in the sweep):
// dst[j+r][c] = [c <= j+r] src[j+r][c] - [c < kc] sum_z P[z][r][c] for c < N
// (P: splits planes of B x kc; src may equal dst; 16-B aligned rows, N, kc even)
// (optional, fused) copy csrc[crows x B] (ld cld) -> cdst (ld cldd): the step's C_bar write-back
cudaError_t adj_rows_init(const double* P, int splits, int B, int64_t kc, const double* src, int64_t lds, double* dst,
                          int64_t ldd, int64_t j, int64_t N, const int* status, cudaStream_t st,
                          const double* csrc = nullptr, int64_t cld = 0, double* cdst = nullptr, int64_t cldd = 0,
                          int64_t crows = 0);
// +0.0 into the strict upper triangle outside the 128 x 128 diagonal tiles
cudaError_t zero_upper_offdiag(double* A, int64_t n, int64_t ld, cudaStream_t st);

// ---- adjoint diagonal-block helpers (R4, R5) ----
// (L[b*128.., b*128..])^-1 for b in [0, nblk), lower, by substitution; block b is
// written with leading dimension ldo at Dinv + (b/per)*ostride + (b%per)*(128*ldo+128)
// (defaults: contiguous 128 x 128 blocks; per = 2 fills the diagonal halves of
// 256 x 256 blocks)
cudaError_t tri_inverse_batched(const double* L, int64_t ld, int nblk, double* Dinv,
                                const int* status, cudaStream_t st, int64_t ldo = 0, int64_t ostride = 0,
                                int per = 1, int64_t istride = 0);
// C[S x S] (ldc) = sign * op(A) op(B) over K = S, S in {128, 256}, batched over
// `batch` problems with element strides sA/sB/sC.  a_t: A given as K x M;
// a_tril: only the lower triangle of A's storage is read (upper taken as 0);
// b_sym: B read as sym(tril(B)) i.e. B[max][min]; B is otherwise K x N.
// c_sym: only the lower tiles are computed and C = sym(tril(product)) is stored
// (both triangles), so a consumer reads it as a plain matrix.
cudaError_t gemm_small(int S, bool a_t, bool a_tril, bool b_sym, const double* A, int64_t lda, const double* B,
                       int64_t ldb, double* C, int64_t ldc, const int* status, cudaStream_t st,
                       double sign = 1.0, int batch = 1, int64_t sA = 0, int64_t sB = 0, int64_t sC = 0,
                       bool c_sym = false);
// S (n x n, ld n): Ssym = mirror(tril(S)) -> ws; Dbar = Phi(S) = tril(S) with halved diagonal
cudaError_t phi_sym(const double* S, double* Ssym, double* Dbar, int64_t ldd, const int* status,
                    cudaStream_t st, int n = 128);
// the symbolic diagonal step fused (S = 128 or 256):
// T1 = sym(tril(D^T D_bar)), T2 = D^-T T1, T3 = T2 D^-1 (S x S scratch each,
// ld S), Ssym = mirror(tril T3), D_bar = Phi(T3); one launch with grid-wide
// barriers on ctr[0..1] (device scratch that must be zero before the first
// call; every launch leaves it zero)
cudaError_t adj_diag_fused(int S, const double* D, int64_t ldl, double* Dbar, int64_t ldw, const double* Di,
                           double* T1, double* T2, double* T3, double* Ssym, unsigned* ctr, const int* status,
                           cudaStream_t st);
// *flags |= 1 (NaN), 2 (|A_ij - A_ji| > tol), 4 (zero diagonal) over the n x n
// matrix; checks selects the bits
cudaError_t check_matrix(const double* A, int64_t n, int checks, double tol, int* flags, cudaStream_t st);
// status = first base+k+1 with !(L[k][k] > 0 && finite), k < n
cudaError_t check_diag(const double* L, int64_t n, int64_t ld, int* status, cudaStream_t st, int64_t base = 0);

// ---- NEXT-4: batched small matrices (n <= 128) ----
// L_b = chol(A_b) for b < batch, n x n contiguous each (A may equal L); info[b]
// (zeroed by the caller) = LAPACK info of matrix b
cudaError_t potrf_batched(const double* A, double* L, int n, int64_t batch, int* info, cudaStream_t st);
// n <= 32: one warp per matrix (info written, no zeroing needed)
cudaError_t potrf_batched_w32(const double* A, double* L, int n, int64_t batch, int* info, cudaStream_t st);
cudaError_t adjoint_batched_w32(const double* L, const double* Lbar, double* Abar, int n, int64_t batch, int* info,
                                cudaStream_t st);
// 32 < n <= 64: two warps per matrix (forward: bit-identical to the tile kernel)
cudaError_t potrf_batched_w64(const double* A, double* L, int n, int64_t batch, int* info, cudaStream_t st);
cudaError_t adjoint_batched_w64(const double* L, const double* Lbar, double* Abar, int n, int64_t batch, int* info,
                                cudaStream_t st);
// batched.cu: the adjoint of the batched factorization and helpers
cudaError_t batched_pad(const double* L, const double* Lbar, int n, int64_t batch, double* Lp, double* Wp,
                        cudaStream_t st);
cudaError_t batched_check_diag(const double* L, int n, int64_t batch, int* info, cudaStream_t st);
cudaError_t batched_phi_out(const double* S, int n, int64_t batch, double* Abar, cudaStream_t st);
// status <- (first b with info[b] != 0) + 1, or 0
cudaError_t batched_first_fail(const int* info, int64_t batch, int* status, cudaStream_t st);

// ---- NEXT-1/NEXT-2 (gp.cu) ----
// x = L^-1 b (trans = false) or L^-T b (trans = true); L lower, positive normal
// diagonal.  flags: (ceil(n/64) + 1) ints of scratch (zeroed here).  x may alias b.
cudaError_t trsv(const double* L, int64_t ld, int64_t n, const double* b, double* x, bool trans, int* flags,
                 const int* status, cudaStream_t st);
// out[0] = -1/2 z.z - sum log L_ii - n/2 log(2 pi)
cudaError_t gp_lp(const double* L, int64_t ld, int64_t n, const double* z, double* out, const int* status,
                  cudaStream_t st);
// lower triangle of W <- tril(a z^T) - diag(1 / L_ii)
cudaError_t gp_lbar(const double* L, int64_t ld, int64_t n, const double* a, const double* z, double* W,
                    int64_t ldw, const int* status, cudaStream_t st);
// out[0..2] = sum_{i>=j} A_bar_ij dK_ij/d(alpha, rho, sigma); partial: gp_hyper_scratch_doubles()
size_t gp_hyper_scratch_doubles();
cudaError_t gp_hyper(const double* A, int64_t lda, int64_t n, const double* x, double alpha, double rho,
                     double sigma, double* partial, double* out, const int* status, cudaStream_t st);
cudaError_t negate(const double* a, double* y, int64_t n, const int* status, cudaStream_t st);

}  // namespace stancl
