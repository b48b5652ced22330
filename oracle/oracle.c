/*
 * oracle.c -- the CPU oracle for the FP64 Cholesky + adjoint hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1907_01063_b200/, libstancl.so) never links, loads
 * or calls it, and this file shares no code, header, table or helper with it.
 *
 * Plain, slow, obviously correct: single thread, IEEE binary64, loops in the
 * order written below, compiled with -O2 -ffp-contract=off (no FMA
 * contraction), no blocking, fusion or reordering.
 *
 * Paper: "GPU-based parallel computation support for Stan" (arXiv:1907.01063),
 * /root/reference/PAPER.md.  Each function cites the passage it follows.
 *
 * Parity status of each entry point (DESIGN.md §3 lists the pins):
 *   oracle_se_cov              pinned (symmetry, diagonal, closed-form entries)
 *   oracle_cholesky            pinned (closed forms, reconstruction, exact log-det,
 *                               integer-exact family, non-PD cases)
 *   oracle_cholesky_ld         long-double twin of oracle_cholesky, used only as a
 *                               truth proxy for rounding-floor studies; pinned by
 *                               the same closed forms
 *   oracle_cholesky_adjoint    pinned (closed-form 2x2, finite differences, log-det
 *                               and GP-density identities, paper's blocked algorithm,
 *                               torch autograd cross-check, integer-exact family)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define IDX(i, j) ((size_t)(i) * (size_t)n + (size_t)(j))

/*
 * Squared-exponential GP covariance (inputs of the paper's GP example,
 * PAPER.md:475 §4.2 "x ... independent draw from Unif(-10,+10)"; kernel form
 * per DESIGN.md reading R14, Stan's gp_exp_quad_cov):
 *   K[i][j] = alpha^2 * exp((x_i - x_j)^2 * (-0.5 / rho^2)) + jitter * [i == j]
 * Full symmetric n x n, row-major.
 */
void oracle_se_cov(int64_t n, const double* x, double alpha, double rho, double jitter,
                   double* K) {
  double sq_alpha = alpha * alpha;
  double neg_half_inv_rho2 = -0.5 / (rho * rho);
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t j = 0; j < n; ++j) {
      double d = x[i] - x[j];
      double v = sq_alpha * exp(d * d * neg_half_inv_rho2);
      if (i == j) v = v + jitter;
      K[IDX(i, j)] = v;
    }
  }
}

/*
 * Cholesky-Banachiewicz, the "classic sequential algorithm" the paper runs on
 * each diagonal block (§3.3.1), applied to the whole matrix; the
 * blocked algorithm of PAPER.md:246-248, 259-289 reaches the same L up to
 * rounding (L with positive diagonal is unique).
 * Reads only A[i][j], i >= j (reading R1).  Writes all of L, +0.0 in
 * the strict upper triangle ("filled with zeros"; reading R2).
 * Returns 0, or info = i+1 for the first row whose pivot s is not > 0 (NaN
 * included) (reading R4).  L may alias A.
 */
int oracle_cholesky(int64_t n, const double* A, double* L) {
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t j = 0; j <= i; ++j) {
      double s = A[IDX(i, j)];
      for (int64_t k = 0; k < j; ++k) {
        double p = L[IDX(i, k)] * L[IDX(j, k)];
        s = s - p;
      }
      if (i == j) {
        if (!(s > 0.0)) return (int)(i + 1);
        L[IDX(i, i)] = sqrt(s);
      } else {
        L[IDX(i, j)] = s / L[IDX(j, j)];
      }
    }
    for (int64_t j = i + 1; j < n; ++j) L[IDX(i, j)] = 0.0;
  }
  return 0;
}

/* Same algorithm in long double (x87 80-bit: 64-bit mantissa).  Input and
 * output are binary64; only used as a truth proxy for floor studies. */
int oracle_cholesky_ld(int64_t n, const double* A, double* L) {
  long double* W = (long double*)malloc(sizeof(long double) * (size_t)n * (size_t)n);
  if (!W && n > 0) return -2;
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t j = 0; j <= i; ++j) {
      long double s = (long double)A[IDX(i, j)];
      for (int64_t k = 0; k < j; ++k) s = s - W[IDX(i, k)] * W[IDX(j, k)];
      if (i == j) {
        if (!(s > 0.0L)) { free(W); return (int)(i + 1); }
        W[IDX(i, i)] = sqrtl(s);
      } else {
        W[IDX(i, j)] = s / W[IDX(j, j)];
      }
    }
  }
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) L[IDX(i, j)] = (j <= i) ? (double)W[IDX(i, j)] : 0.0;
  free(W);
  return 0;
}

/*
 * Reverse-mode adjoint of oracle_cholesky: the mechanical reverse sweep of the
 * loop above, statement by statement in reverse order.  This is the derivative
 * the paper's blocked gradient (§3.3.2, after Murray 2016)
 * computes, with Stan's convention (readings R5, R6): the strictly-lower entry
 * A_bar[i][j] is df/da_ij of the symmetric pair, the diagonal is df/da_ii, and
 * the strict upper triangle is +0.0 (PAPER.md:321 set_zeros_in_upper_tri).
 *
 * Forward statements, for row i ascending, j = 0..i:
 *   s = A[i][j] - sum_{k<j} L[i][k] L[j][k]
 *   L[i][i] = sqrt(s)          (i == j)
 *   L[i][j] = s / L[j][j]      (i >  j)
 * Reverse (M holds the running adjoint of L, initialised to tril(L_bar)):
 *   i == j: sbar = M[i][i] / (2 L[i][i])
 *   i >  j: sbar = M[i][j] / L[j][j];   M[j][j] -= M[i][j] * L[i][j] / L[j][j]
 *   A_bar[i][j] = sbar
 *   for k < j:  M[i][k] -= sbar * L[j][k];  M[j][k] -= sbar * L[i][k]
 * Reads only the lower triangles of L and L_bar.  Returns 0, or k+1 for the
 * first diagonal entry L[k][k] that is not finite and > 0.  A_bar may alias
 * L_bar (the upper triangle of L_bar is never read).
 */
int oracle_cholesky_adjoint(int64_t n, const double* L, const double* Lbar, double* Abar) {
  for (int64_t k = 0; k < n; ++k) {
    double d = L[IDX(k, k)];
    if (!(d > 0.0) || !isfinite(d)) return (int)(k + 1);
  }
  double* M = (double*)malloc(sizeof(double) * (size_t)n * (size_t)n);
  if (!M && n > 0) return -2;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) M[IDX(i, j)] = (j <= i) ? Lbar[IDX(i, j)] : 0.0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) Abar[IDX(i, j)] = 0.0;
  for (int64_t i = n - 1; i >= 0; --i) {
    for (int64_t j = i; j >= 0; --j) {
      double sbar;
      if (i == j) {
        sbar = M[IDX(i, i)] / (2.0 * L[IDX(i, i)]);
      } else {
        sbar = M[IDX(i, j)] / L[IDX(j, j)];
        double t = M[IDX(i, j)] * L[IDX(i, j)];
        t = t / L[IDX(j, j)];
        M[IDX(j, j)] = M[IDX(j, j)] - t;
      }
      Abar[IDX(i, j)] = sbar;
      for (int64_t k = 0; k < j; ++k) {
        double p = sbar * L[IDX(j, k)];
        M[IDX(i, k)] = M[IDX(i, k)] - p;
        double q = sbar * L[IDX(i, k)];
        M[IDX(j, k)] = M[IDX(j, k)] - q;
      }
    }
  }
  free(M);
  return 0;
}
