/*
 * stan_cl.h -- C ABI of libstancl: FP64 Cholesky factorisation and its
 * reverse-mode adjoint on NVIDIA B200 (sm_100a), the computation Stan's GPU
 * backend accelerates for Gaussian-process models
 * ("GPU-based parallel computation support for Stan", arXiv:1907.01063,
 * /root/reference/PAPER.md; citations are PAPER.md line numbers).
 *
 * Conventions for every matrix argument unless stated otherwise
 *   - n x n, row-major, leading dimension n, IEEE binary64;
 *   - CUDA device pointers on the current device (the *_host entry points take
 *     host pointers instead);
 *   - only the lower triangle (i >= j) of A, L and L_bar is read
 *     (reading R1); the strict upper triangle of every output
 *     matrix is written as +0.0 ("filled with zeros", PAPER.md:321
 *     set_zeros_in_upper_tri);
 *   - work is enqueued on the library stream (stan_cl_set_stream; default:
 *     the legacy default stream).  The plain entry points return after the
 *     stream has drained (they read back the status word); the *_async entry
 *     points return immediately and leave the status in device memory.
 *
 * Ownership: the caller owns every buffer passed in.  The library owns only
 * its internal workspace (allocated lazily, released by stan_cl_finalize), or
 * uses a caller-provided one instead (stan_cl_set_workspace).  No pointer is
 * dereferenced after a call returns; the CUDA-graph cache of the n <= 4096
 * device calls remembers the buffer addresses of a call only as a lookup key
 * (a replay happens only for a call with the same addresses, and a cached
 * graph is discarded whenever a workspace buffer it wrote through moved).
 * Calls are not thread-safe with respect to each other (one library stream
 * and workspace per process).
 *
 * Return values: 0 = success; k > 0 = numerical failure (see each call);
 * negative = STAN_CL_E* error codes below.
 */
#ifndef STAN_CL_H
#define STAN_CL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STAN_CL_OK 0
#define STAN_CL_EINVAL (-1) /* bad argument: n < 0, NULL with n > 0, forbidden overlap, bad nb */
#define STAN_CL_ENOMEM (-2) /* device workspace allocation failed */
#define STAN_CL_ECUDA (-3)  /* a CUDA runtime error (launch, copy, sync) */
#define STAN_CL_ENCCL (-4)  /* reserved for the multi-GPU layer */

/*
 * L = chol(A): lower-triangular L with positive diagonal and L L^T = A.
 * Method: PAPER.md:244-291 (§3.3.1) -- blocked right-looking factorisation
 * (L11 = chol(A11); L21 = A21 L11^-T; A22 -= L21 L21^T), diagonal tiles by the
 * "classic sequential algorithm", L21 by substitution (R11).
 *   n   order (n == 0: returns 0, touches nothing)
 *   A   device, n x n, lower triangle read
 *   L   device, n x n, written in full; L == A (in place) allowed, any other
 *       overlap of the two n x n ranges -> STAN_CL_EINVAL
 * Returns k > 0 (LAPACK-style info) when A is not positive definite: the
 * first failing pivot (s <= 0 or NaN) is row k-1 (R4); L is then
 * unspecified.
 */
int stan_cl_cholesky(int64_t n, const double* A, double* L);

/*
 * A_bar = reverse-mode adjoint of L = chol(A) given L and L_bar = df/dL:
 *   A_bar = Phi(G + G^T),  G = L^-T Phi(L^T tril(L_bar)) L^-1,
 * Phi(X) = tril(X) with the diagonal halved (Stan's convention: strictly-lower
 * A_bar[i][j] is df/da_ij of the symmetric pair, the diagonal is df/da_ii;
 * DESIGN.md R5).  Method: the blocked gradient of PAPER.md:297-323 (§3.3.2),
 * reverse block order, with reading R6 of the garbled line PAPER.md:320.
 *   L      device, n x n, lower triangle read (diagonal must be finite and > 0)
 *   L_bar  device, n x n, lower triangle read
 *   A_bar  device, n x n, written in full (strict upper +0.0).  A_bar == L_bar
 *          allowed (in place); A_bar overlapping L, or partially overlapping
 *          L_bar -> STAN_CL_EINVAL.
 * Overwrites A_bar (Stan's A.adj += accumulation is the caller's job).
 * Returns k > 0 when L[k-1][k-1] is not finite and > 0.
 */
int stan_cl_cholesky_adjoint(int64_t n, const double* L, const double* L_bar, double* A_bar);

/*
 * Squared-exponential GP covariance of the paper's GP example (inputs
 * PAPER.md:475; kernel form DESIGN.md R14):
 *   K[i][j] = alpha^2 * exp((x_i - x_j)^2 * (-0.5 / rho^2)) + jitter * [i == j]
 *   x  device, n doubles;  K  device, n x n, written in full (symmetric).
 * rho must be finite and nonzero, else STAN_CL_EINVAL.
 */
int stan_cl_gp_exp_quad_cov(int64_t n, const double* x, double alpha, double rho, double jitter,
                            double* K);

/*
 * Asynchronous variants: same arguments and semantics, but the call returns
 * once the work is enqueued.  d_info (device int, caller-owned, may be NULL
 * when the caller does not need it) receives the status word the synchronous
 * call would return for a numerical failure (0 or k > 0) when the stream
 * reaches it.  Argument errors are still returned directly.
 */
int stan_cl_cholesky_async(int64_t n, const double* A, double* L, int* d_info);
int stan_cl_cholesky_adjoint_async(int64_t n, const double* L, const double* L_bar, double* A_bar,
                                   int* d_info);

/*
 * Host-buffer variants (end-to-end, the quantity PAPER.md:295, 332 measures):
 * all matrix pointers are HOST pointers (row-major, leading dimension n; pinned
 * memory is fastest).  Only the lower triangles cross PCIe -- the paper's
 * packed transfers -- as one rectangle per 128-row block
 * (rows r0..r1-1, columns 0..r1-1), streamed against the compute: the forward
 * ships each factored panel while the trailing update continues; the adjoint
 * uploads row blocks bottom-up (the order its reverse sweep consumes them) and
 * ships each column block of A_bar as soon as it is final.  The call returns
 * after the last copy-back.  Output contract as the device calls: the whole
 * n x n host output is written, strict upper triangle +0.0 (the diagonal
 * tiles' upper part comes over PCIe with them; the rest is zero-filled by host
 * threads while the device computes, so it costs no PCIe traffic).  A == L
 * (forward) and L_bar == A_bar (adjoint) are allowed; other overlaps ->
 * STAN_CL_EINVAL.  Same return values as the device calls.
 */
int stan_cl_cholesky_host(int64_t n, const double* A, double* L);
int stan_cl_cholesky_adjoint_host(int64_t n, const double* L, const double* L_bar, double* A_bar);

/*
 * ---- multi-GPU (one process per GPU) ----
 * Layout: 2-D block-cyclic by 256 x 256 tiles over a P x Q process grid
 * (nranks = P * Q; rank r is grid position (p, q) = (r / Q, r % Q)).  Tile
 * (I, J) (rows I*256.., columns J*256..) lives on rank (I % P, J % Q) as local
 * tile (I / P, J / Q) of a row-major (R_p * 256) x ld_local array, where R_p
 * (C_q) is the number of block indices I < n/256 with I % P == p (J % Q == q)
 * and ld_local >= 256 * C_q.  P = 1 is block-column cyclic (whole columns per
 * rank).  n must be a multiple of 256.  Only the lower tiles (I >= J) are read
 * or written; +0.0 is written above the diagonal inside the diagonal tiles.
 * Per forward step k: the diagonal owner factors L_kk
 * (column broadcast), process column k % Q solves its panel tiles, each
 * process row receives its panel rows (row broadcast), each process column
 * receives the panel tiles of its block columns (column broadcasts, P > 1),
 * every rank updates its lower trailing tiles.  Per adjoint step
 * (PAPER.md:298-322): broadcasts of D^-1 (column), C_bar D^-1 (row), L's row
 * block (column), sym(S) (row), and a column REDUCE (ncclReduce, sum) of the
 * partial products C_bar^T [B C] to the owners of the block row (P > 1).
 *   stan_cl_dist_get_unique_id  rank 0; the 128-byte NCCL id is shipped to the
 *                               other ranks by the caller (torch.distributed)
 *   stan_cl_dist_init           P, Q >= 1, P * Q == nranks; builds the world,
 *                               row (ncclCommSplit color p) and column (color q)
 *                               communicators; the CUDA device of the calling
 *                               thread is the rank's device
 *   stan_cl_dist_cholesky       in place on A_local (nb: 0 or 256)
 *   stan_cl_dist_cholesky_adjoint  L_local read-only; Lbar_to_Abar_local in
 *                               place; both with leading dimension ld_local
 * Every rank must make the same sequence of calls (collectives inside).
 * Return values as the single-GPU calls (numerical status all-reduced with max);
 * STAN_CL_ENCCL when NCCL cannot be loaded or fails -- including an
 * asynchronous communicator error or the stream not draining within
 * STAN_CL_NCCL_TIMEOUT_S seconds (environment; default 1800, 0 = no limit):
 * the call then aborts every communicator (ncclCommAbort) and returns instead
 * of hanging, and the grid must be re-initialised; STAN_CL_EINVAL for a bad
 * grid, n % 256 != 0, or ld_local too small.  Library-owned scratch: about
 * (R_p + 1) * 256^2 doubles (+ C_q * 256^2 * (P + 3) for P > 1 / the adjoint).
 */
int stan_cl_dist_get_unique_id(void* out128);
int stan_cl_dist_init(int nranks, int rank, const void* id128, int P, int Q);
int stan_cl_dist_cholesky(int64_t n, int nb, double* A_local, int64_t ld_local);
int stan_cl_dist_cholesky_adjoint(int64_t n, int nb, const double* L_local, double* Lbar_to_Abar_local,
                                  int64_t ld_local);
int stan_cl_dist_finalize(void);
/* the SE covariance's tiles for rank (p, q) of a P x Q grid (the layout above;
 * every local element is written, including tiles above the diagonal) */
int stan_cl_gp_exp_quad_cov_tiles(int64_t n, const double* x, double alpha, double rho, double jitter,
                                  double* K_local, int64_t ld_local, int P, int Q, int p, int q);
/* the 1 x G special case (block columns of rank q) */
int stan_cl_gp_exp_quad_cov_cols(int64_t n, const double* x, double alpha, double rho, double jitter,
                                 double* K_local, int64_t ld_local, int G, int q);
/* The same distributed algorithms with all P * Q ranks simulated in this
 * process on the current device (broadcasts become device copies, the column
 * reduce fixed-order additions): one local array per rank, locals[p * Q + q],
 * all with leading dimension ld_local.  For testing the multi-GPU path on one
 * GPU.  The *_sim_* forms are the 1 x G grid. */
int stan_cl_dist_sim2_cholesky(int64_t n, int P, int Q, double* const* A_locals, int64_t ld_local);
int stan_cl_dist_sim2_cholesky_adjoint(int64_t n, int P, int Q, const double* const* L_locals,
                                       double* const* W_locals, int64_t ld_local);
int stan_cl_dist_sim_cholesky(int64_t n, int G, double* const* A_locals, int64_t ld_local);
/* Collective trace of rank (p, q) of a P x Q grid, for checking the multi-GPU
 * schedule on one device: runs the real per-rank path of stan_cl_dist_cholesky
 * (adjoint == 0; A_local in place) or stan_cl_dist_cholesky_adjoint
 * (adjoint != 0; L_local, A_local = L_bar in place) with every NCCL call
 * replaced by a record of what it would issue, in host issue order (no data
 * moves, so the numbers are meaningless).  Each record is 6 int64 in out:
 * communicator kind (0 row, 1 column, 2 world), its index (p, q or 0), op
 * (0 broadcast, 1 sum-reduce, 2 max-all-reduce), root index within the
 * communicator (-1 for none), element count, stream (0 library stream,
 * 1 side stream).  Writes at most max_entries records; returns the total
 * number of records (>= 0) or a negative error.  Every member of a
 * communicator must produce the same sequence of records on it, else the
 * NCCL path would deadlock or mismatch counts (tests/test_gpu_dist.py). */
int stan_cl_dist_trace(int64_t n, int P, int Q, int p, int q, int adjoint, const double* L_local,
                       double* A_local, int64_t ld_local, int64_t* out, int64_t max_entries);
int stan_cl_dist_sim_cholesky_adjoint(int64_t n, int G, const double* const* L_locals, double* const* W_locals,
                                      int64_t ld_local);

/* ---- NEXT rows around the hot path ---- */

/*
 * Triangular solve with one right-hand side (the paper's triangular_solve,
 * PAPER.md:231-238 §3.3; NEXT-2):
 *   trans == 0:  x = L^-1 b        trans != 0:  x = L^-T b
 * L: n x n row-major (ld n), only the lower triangle is read; its diagonal must
 * be positive (a Cholesky factor): the first L[k][k] that is not finite and
 * > 0 returns k+1 (x unspecified).  b, x: n doubles; x may alias b (in place),
 * any other overlap -> STAN_CL_EINVAL.  Device pointers; synchronous.
 * Blocked substitution, one CTA per 64-row block, no inverse formed.
 */
int stan_cl_trsv(int64_t n, const double* L, const double* b, double* x, int trans);

/*
 * Lower triangular inverse X = L^-1 (the paper's lower_triangular_inverse,
 * PAPER.md:207-225 §3.2; NEXT-2).  Method: the paper's batched divide and
 * conquer -- the 128 x 128 diagonal blocks inverted by substitution, one CTA
 * per block (the paper's batch_identity + diag_inv), then log2(n/128) doubling
 * levels, each pair of adjacent inverted blocks [[C1, 0], [A3, C2]] completed
 * by C3 = -C2 A3 C1 on the FP64 tensor cores (batched 128^3 / 256^3 products,
 * persistent TMA GEMMs above).
 *   L  device, n x n, lower triangle read; its diagonal must be finite and > 0
 *      (the factors the library produces): the first L[k][k] that is not
 *      returns k+1 (X unspecified)
 *   X  device, n x n, written in full (strict upper +0.0); must not overlap L
 *      (STAN_CL_EINVAL).  Synchronous.
 */
int stan_cl_lower_triangular_inverse(int64_t n, const double* L, double* X);

/*
 * Triangular solve with m right-hand sides (the paper's general solver for
 * A x = b with triangular A, §3.2; NEXT-2):
 *   trans == 0:  X = L^-1 B        trans != 0:  X = L^-T B
 * L: n x n (lower triangle read, diagonal finite and > 0, else k+1 as
 * stan_cl_trsv); B, X: n x m row-major (ld m).  X may alias B (in place);
 * other overlaps -> STAN_CL_EINVAL.  Method: right-looking blocked
 * substitution over 256-row blocks (128 below n = 768) with the diagonal
 * blocks' explicit inverses -- per block S = D_i^-1 X_i (or D_i^-T X_i), then
 * the rank-256 update of the remaining rows on the FP64 tensor cores.
 * Synchronous.
 */
int stan_cl_trsm(int64_t n, int64_t m, const double* L, const double* B, double* X, int trans);

/*
 * Reverse mode of C = L^-1 B (the triangular solver's chain(), PAPER.md:231-238;
 * the listing's "A * adjB = adjC" read as A^T adjB = adjC, R17):
 *   B_bar = L^-T C_bar;    L_bar = tril(-B_bar C^T)
 * L, L_bar: n x n (L_bar written in full, strict upper +0.0); C, C_bar, B_bar:
 * n x m row-major.  B_bar may alias C_bar; every other overlap -> EINVAL.
 * m == 0: L_bar = 0.  Returns k+1 for a bad diagonal of L as stan_cl_trsm.
 * Synchronous.
 */
int stan_cl_trsm_adjoint(int64_t n, int64_t m, const double* L, const double* C, const double* C_bar,
                         double* L_bar, double* B_bar);
/* caller workspace (stan_cl_set_workspace) that suffices for stan_cl_trsm and
 * stan_cl_trsm_adjoint with n x m right-hand sides */
size_t stan_cl_trsm_workspace_bytes(int64_t n, int64_t m);

/*
 * Marginal log density of zero-mean GP regression and its gradient -- the
 * per-gradient work of the paper's GP example (§4.2, the model
 * y ~ multi_normal_cholesky(0, chol(K)); NEXT-1):
 *   K = alpha^2 exp((x_i - x_j)^2 (-0.5 / rho^2)) + sigma^2 [i == j]
 *   out[0] = log p(y) = -1/2 y^T K^-1 y - 1/2 log det K - n/2 log(2 pi)
 *   out[1], out[2], out[3] = d log p / d alpha, d rho, d sigma
 *   y_bar (may be NULL) = d log p / d y = -K^-1 y
 * The O(n^3) work is this library's Cholesky (stan_cl_cholesky) and its
 * adjoint (stan_cl_cholesky_adjoint) with L_bar = tril(a z^T) - diag(1 / L_ii),
 * z = L^-1 y, a = L^-T z; the hyperparameter gradient contracts A_bar's lower
 * triangle with dK/dtheta.  x, y: n doubles; out: 4 doubles; y_bar: n doubles;
 * all device pointers.  Returns 0, the Cholesky info k+1 if K is not positive
 * definite (out unspecified), STAN_CL_EINVAL for n < 0, NULL x/y/out with
 * n > 0, or rho == 0 / non-finite alpha, rho, sigma.  n == 0: out = {0, 0, 0, 0}.
 * Library-owned workspace: two n x n matrices + O(n).  Synchronous.
 */
int stan_cl_gp_lpdf_grad(int64_t n, const double* x, const double* y, double alpha, double rho, double sigma,
                         double* out, double* y_bar);

/*
 * Batched small matrices (NEXT-4; "batched linear algebra"; one
 * covariance per chain): batch independent n x n problems,
 * 1 <= n <= 128, stored contiguously (matrix b at offset b*n*n, row-major).
 *   stan_cl_cholesky_batched:         L_b = chol(A_b)                 (A may equal L)
 *   stan_cl_cholesky_adjoint_batched: A_bar_b = adjoint(L_b, L_bar_b) (any of the
 *                                     three may coincide; partial overlap -> EINVAL)
 * Same per-matrix semantics as the single-matrix calls (lower triangles read,
 * strict upper written +0.0).  info (device int[batch], may be NULL): LAPACK
 * info of each matrix (forward: first failing pivot + 1; adjoint: first
 * L[k][k] not finite and > 0, + 1).  Returns 0 when every matrix succeeded,
 * k > 0 when matrix k-1 is the first that failed, negative on errors
 * (n > 128 -> STAN_CL_EINVAL).  Kernels: n <= 32 one warp per matrix, n <= 64
 * two warps per matrix (rows in registers; forward bit-identical to the
 * single-matrix path), 64 < n <= 128 one CTA per matrix (the diagonal-tile
 * kernel, identity padded) and, for the adjoint, the paper's diagonal-block
 * step on 128 x 128 padded copies in chunks of 4096.  The single-matrix calls
 * use the n <= 64 kernels for n <= 64 as well.  Device pointers; synchronous.
 */
int stan_cl_cholesky_batched(int64_t batch, int64_t n, const double* A, double* L, int* info);
int stan_cl_cholesky_adjoint_batched(int64_t batch, int64_t n, const double* L, const double* L_bar,
                                     double* A_bar, int* info);

/*
 * Input checks of the paper's backend (§3.5: check_nan,
 * check_symmetric, check_diagonal_zeros; NEXT-3), one pass over the n x n
 * device matrix A (row-major, ld n), synchronous.  checks selects, the return
 * value reports (bitwise OR):
 *   1  some entry is NaN
 *   2  some |A[i][j] - A[j][i]| > tol (absolute tolerance, tol >= 0; a pair with
 *      a NaN or an infinite difference also counts)
 *   4  some diagonal entry is zero
 * Returns >= 0 (the bits found), or STAN_CL_EINVAL for n < 0, unknown bits in
 * checks, tol < 0 or NaN, or A == NULL with n > 0.  Flags are only ever set,
 * never cleared, by the CTAs (race-free, as the paper's kernels).
 */
int stan_cl_check_matrix(int64_t n, const double* A, int checks, double tol);

/* ---- control ---- */
int stan_cl_set_stream(void* cuda_stream); /* cudaStream_t; NULL = legacy default stream */
void* stan_cl_get_stream(void);
/* outer block size of the blocked Cholesky: 0 = auto (256 = two-level blocking
 * with 128-wide diagonal tiles for n >= 6144, else 128), 128 or 256; others ->
 * STAN_CL_EINVAL. */
int stan_cl_set_block_size(int nb);
int stan_cl_get_block_size(void);
/* block size of the blocked adjoint: 0 = auto (256 for n >= 768, else 128),
 * 128 or 256; others -> STAN_CL_EINVAL */
int stan_cl_set_adjoint_block_size(int nb);
/*
 * Caller-owned workspace (SURVEY.md §8(b) "lazily allocated ... or
 * caller-provided").  stan_cl_set_workspace(ptr, bytes): every device buffer
 * the library needs (status word, D^-1 blocks, split-K partials, padded
 * copies, GP matrices, the multi-GPU scratch) is carved from [ptr, ptr+bytes)
 * afresh by each call; the library then allocates no device memory of its own
 * (library-owned workspace is freed here) and never frees ptr.  ptr must be a
 * device pointer aligned to 256 bytes with bytes >= 256; NULL reverts to
 * library-owned workspace.  Synchronises the device.  A call whose needs
 * exceed bytes returns STAN_CL_ENOMEM and does nothing else (stan_cl_status_string
 * names the size it needed).  The buffer must stay allocated until
 * stan_cl_set_workspace(NULL, 0) or stan_cl_finalize.  Returns STAN_CL_EINVAL
 * for a misaligned / too small buffer.
 * stan_cl_workspace_bytes(n): bytes that suffice for every single-matrix entry
 * point at order n (cholesky, cholesky_adjoint, their _async and _host forms,
 * trsv, gp_lpdf_grad, lower_triangular_inverse; trsm: see
 * stan_cl_trsm_workspace_bytes) with the current block-size settings and 16-byte
 * aligned arguments (an unaligned argument takes the padded path: add
 * 2 * 8 * N^2, N = n rounded up to 256).
 * stan_cl_batched_workspace_bytes(batch, n, with_info): the same for the batched
 * calls (with_info != 0: the caller passes its own info array).
 */
int stan_cl_set_workspace(void* dev_ptr, size_t bytes);
size_t stan_cl_workspace_bytes(int64_t n);
size_t stan_cl_batched_workspace_bytes(int64_t batch, int64_t n, int with_info);
const char* stan_cl_status_string(int status);
/* number of CUDA kernel launches the library has issued so far (process-wide) */
long long stan_cl_kernel_launches(void);
/*
 * Per-kernel-class timing with CUDA events recorded on the launch stream around
 * the kernels the library issues (off by default; a few microseconds of host
 * overhead per recorded launch).  Classes (kind): 0 SYRK trailing update,
 * 1 adjoint DMMA GEMMs (B_bar, R_bar updates), 2 split-K long-K contraction,
 * 3 POTRF tile, 4 TRSM panel, 5 batched diagonal-block inverse, 6 128^3
 * products, 7 SE build, 8 other, 9 forward lookahead-column GEMMs,
 * 10 C_bar D^-1 products, 11 triangular solves and GP log-density /
 * gradient kernels.  stan_cl_profile_enable(on): 0 = off, 1 = every
 * class, otherwise (mask << 1) enables class k when bit k of mask is set.
 * stan_cl_profile_read synchronises on the recorded events and returns the
 * summed milliseconds, the summed algorithmic flops and the launch count of a
 * class since the last reset.
 */
int stan_cl_profile_enable(int on);  /* see above */
int stan_cl_profile_reset(void);
int stan_cl_profile_read(int kind, double* ms, double* flops, long long* launches);
/* summed algorithmic (minimum) HBM bytes of the recorded launches of a class */
int stan_cl_profile_read_bytes(int kind, double* bytes);
/*
 * Launch timeline (tracing).  stan_cl_trace_enable(1) records a
 * base event on the library stream and from then on brackets EVERY library
 * launch with CUDA events on its own stream (all classes; a few microseconds
 * of host overhead per launch); stan_cl_trace_enable(0) stops.
 * stan_cl_trace_read(out, max): 4 doubles per launch -- profiling class (as
 * above), stream id (0, 1, ... in order of first use: the library stream, the
 * lookahead side stream, copy streams), start and end in ms after the base
 * event; synchronises on the recorded events; returns the number of records
 * (writes at most max).
 */
int stan_cl_trace_enable(int on);
int stan_cl_trace_read(double* out, int max_records);
/* release library-owned device workspace; the library stays usable */
int stan_cl_finalize(void);
int stan_cl_version(void); /* major*10000 + minor*100 + patch */

#ifdef __cplusplus
}
#endif

#endif /* STAN_CL_H */
