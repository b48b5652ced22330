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
 *   oracle_cholesky_par        oracle_cholesky with independent entries computed by
 *                               several threads; pinned by bit-identity with it
 *   oracle_cholesky_ld         long-double twin of oracle_cholesky, used only as a
 *                               truth proxy for rounding-floor studies; pinned by
 *                               the same closed forms
 *   oracle_cholesky_adjoint    pinned (closed-form 2x2, finite differences, log-det
 *                               and GP-density identities, paper's blocked algorithm,
 *                               torch autograd cross-check, integer-exact family)
 *   oracle_trsv                pinned (integer-exact round trips, independent
 *                               library solve)
 *   oracle_tri_inverse         pinned (integer-exact L X = I, exact reciprocal diagonal,
 *                               2 x 2 closed form, X L = I on SE factors)
 *   oracle_trsm                pinned (integer-exact round trips both ways, column
 *                               independence)
 *   oracle_trsm_adjoint        pinned (n = 1 closed form, finite differences of a
 *                               random functional of L^-1 B in B and in L)
 *   oracle_check_matrix        pinned (hand-built cases per bit, tolerance edge)
 *   oracle_gp_lpdf_grad        pinned (n = 1 closed form, independent Gaussian
 *                               log-density, trace-form gradient, finite differences)
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

/*
 * oracle_cholesky with its independent work spread over threads, bit for bit
 * the same result.  Each entry L[i][j] is computed by the same statements, in
 * the same order, from the same operands as in oracle_cholesky -- only the
 * order in which DIFFERENT entries are computed changes, and only among
 * entries whose operands are already final:
 *   for each block of 32 rows [r0, r1):
 *     (1) entries j < r0 of every row in the block, one row per thread (they
 *         need rows < r0, complete, and the row's own entries to their left);
 *     (2) entries r0 <= j <= i, rows in order (the block's own triangle),
 *         with the pivot test of oracle_cholesky.
 * So info (the first failing pivot row + 1) is oracle_cholesky's as well.
 * Used only to rebuild the oracle's L at n = 8192 / 16384 in a GPU test (a
 * single thread needs ~20 min at 16384); pinned by bit-identity with
 * oracle_cholesky (tests/test_oracle.py) and by the SHA-256 of the sequential
 * oracle's L stored in tests/golden/.
 */
int oracle_cholesky_par(int64_t n, const double* A, double* L, int nthreads) {
  const int64_t RB = 32;
  if (nthreads < 1) nthreads = 1;
  for (int64_t r0 = 0; r0 < n; r0 += RB) {
    const int64_t r1 = (r0 + RB < n) ? r0 + RB : n;
#pragma omp parallel for schedule(static, 1) num_threads(nthreads)
    for (int64_t i = r0; i < r1; ++i) {
      for (int64_t j = 0; j < r0; ++j) {
        double s = A[IDX(i, j)];
        for (int64_t k = 0; k < j; ++k) {
          double p = L[IDX(i, k)] * L[IDX(j, k)];
          s = s - p;
        }
        L[IDX(i, j)] = s / L[IDX(j, j)];
      }
    }
    for (int64_t i = r0; i < r1; ++i) {
      for (int64_t j = r0; j <= i; ++j) {
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

/*
 * Triangular solve with one right-hand side, the triangular_solve primitive of
 * the paper (§3.3 describes its blocked GPU form and reverse
 * mode), by plain substitution:
 *   trans == 0:  L x = b     x_i = (b_i - sum_{j<i} L[i][j] x_j) / L[i][i],  i ascending
 *   trans == 1:  L^T x = b   x_i = (b_i - sum_{j>i} L[j][i] x_j) / L[i][i],  i descending
 * Sums in ascending j.  Reads only the lower triangle of L.  Returns 0, or
 * k+1 for the first (in solve order) diagonal entry that is not finite and
 * nonzero.  x may alias b.
 */
int oracle_trsv(int64_t n, const double* L, const double* b, int trans, double* x) {
  for (int64_t k = 0; k < n; ++k) {
    double d = L[IDX(k, k)];
    if (d == 0.0 || !isfinite(d)) return (int)(k + 1);
  }
  if (x != b)
    for (int64_t i = 0; i < n; ++i) x[i] = b[i];
  if (!trans) {
    for (int64_t i = 0; i < n; ++i) {
      double s = x[i];
      for (int64_t j = 0; j < i; ++j) s = s - L[IDX(i, j)] * x[j];
      x[i] = s / L[IDX(i, i)];
    }
  } else {
    for (int64_t i = n - 1; i >= 0; --i) {
      double s = x[i];
      for (int64_t j = i + 1; j < n; ++j) s = s - L[IDX(j, i)] * x[j];
      x[i] = s / L[IDX(i, i)];
    }
  }
  return 0;
}

/*
 * Lower triangular inverse X = L^-1 (§3.2 "the lower
 * triangular inverse of A"), by its plain definition:
 * column j of X solves L x = e_j by forward substitution,
 *   X[j][j] = 1 / L[j][j]
 *   X[i][j] = -(sum_{k=j}^{i-1} L[i][k] X[k][j]) / L[i][i],   i = j+1 .. n-1
 * (the paper's divide-and-conquer C3 = -C2 A3 C1 reaches the same matrix up
 * to rounding).  Sums in ascending k.  Reads only the lower triangle of L;
 * writes all of X (+0.0 above the diagonal).  Returns 0, or k+1 for the first
 * diagonal entry that is not finite and nonzero.  X must not alias L.
 */
int oracle_tri_inverse(int64_t n, const double* L, double* X) {
  for (int64_t k = 0; k < n; ++k) {
    double d = L[IDX(k, k)];
    if (d == 0.0 || !isfinite(d)) return (int)(k + 1);
  }
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) X[IDX(i, j)] = 0.0;
  for (int64_t j = 0; j < n; ++j) {
    X[IDX(j, j)] = 1.0 / L[IDX(j, j)];
    for (int64_t i = j + 1; i < n; ++i) {
      double s = 0.0;
      for (int64_t k = j; k < i; ++k) {
        double p = L[IDX(i, k)] * X[IDX(k, j)];
        s = s + p;
      }
      X[IDX(i, j)] = -s / L[IDX(i, i)];
    }
  }
  return 0;
}

/*
 * Triangular solve with m right-hand sides, the paper's general solver for
 * A x = b with triangular A (§3.2; NEXT-2), by substitution,
 * one column c of B at a time (B, X: n x m row-major):
 *   trans == 0:  L X = B     X[i][c] = (B[i][c] - sum_{j<i} L[i][j] X[j][c]) / L[i][i],  i ascending
 *   trans == 1:  L^T X = B   X[i][c] = (B[i][c] - sum_{j>i} L[j][i] X[j][c]) / L[i][i],  i descending
 * Sums in ascending j.  Reads only the lower triangle of L.  Returns 0, or
 * k+1 for the first diagonal entry that is not finite and nonzero.  X may
 * alias B.
 */
int oracle_trsm(int64_t n, int64_t m, const double* L, const double* B, int trans, double* X) {
  for (int64_t k = 0; k < n; ++k) {
    double d = L[IDX(k, k)];
    if (d == 0.0 || !isfinite(d)) return (int)(k + 1);
  }
  if (X != B)
    for (int64_t i = 0; i < n; ++i)
      for (int64_t c = 0; c < m; ++c) X[(size_t)i * (size_t)m + (size_t)c] = B[(size_t)i * (size_t)m + (size_t)c];
  for (int64_t c = 0; c < m; ++c) {
    if (!trans) {
      for (int64_t i = 0; i < n; ++i) {
        double s = X[(size_t)i * (size_t)m + (size_t)c];
        for (int64_t j = 0; j < i; ++j) s = s - L[IDX(i, j)] * X[(size_t)j * (size_t)m + (size_t)c];
        X[(size_t)i * (size_t)m + (size_t)c] = s / L[IDX(i, i)];
      }
    } else {
      for (int64_t i = n - 1; i >= 0; --i) {
        double s = X[(size_t)i * (size_t)m + (size_t)c];
        for (int64_t j = i + 1; j < n; ++j) s = s - L[IDX(j, i)] * X[(size_t)j * (size_t)m + (size_t)c];
        X[(size_t)i * (size_t)m + (size_t)c] = s / L[IDX(i, i)];
      }
    }
  }
  return 0;
}

/*
 * Reverse mode of C = L^-1 B (the triangular solver's chain()
 * §3.2, read per DESIGN.md reading R17: the listing's "A * adjB = adjC" is the
 * transposed system A^T adjB = adjC, the derivative of C = A^-1 B):
 *   B_bar = L^-T C_bar                  (oracle_trsm, trans = 1)
 *   L_bar = tril(-B_bar C^T)            (only L's lower triangle is an input)
 *   L_bar[i][j] = -sum_c B_bar[i][c] C[j][c],  i >= j, sums in ascending c
 * C, C_bar, B_bar: n x m row-major; L, L_bar: n x n (+0.0 above the diagonal
 * of L_bar).  Returns 0, or k+1 for a bad diagonal of L.  B_bar may alias C_bar.
 */
int oracle_trsm_adjoint(int64_t n, int64_t m, const double* L, const double* C, const double* Cbar,
                        double* Lbar, double* Bbar) {
  int info = oracle_trsm(n, m, L, Cbar, 1, Bbar);
  if (info) return info;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double s = 0.0;
      if (j <= i)
        for (int64_t c = 0; c < m; ++c) {
          double p = Bbar[(size_t)i * (size_t)m + (size_t)c] * C[(size_t)j * (size_t)m + (size_t)c];
          s = s + p;
        }
      Lbar[IDX(i, j)] = (j <= i) ? -s : 0.0;
    }
  return 0;
}

/*
 * Input checks of the paper's OpenCL backend (§3.5 "Input
 * checking": check_nan, check_symmetric, check_diagonal_zeros), by their plain
 * definitions over the whole n x n matrix:
 *   bit 0 (1): some A[i][j] is NaN
 *   bit 1 (2): some |A[i][j] - A[j][i]| > tol (absolute; "within tolerance of
 *              zero"; a NaN pair also counts, since the comparison is false)
 *   bit 2 (4): some A[i][i] == 0
 * checks selects which bits are evaluated; returns the set bits.
 */
int oracle_check_matrix(int64_t n, const double* A, int checks, double tol) {
  int out = 0;
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t j = 0; j < n; ++j) {
      double a = A[IDX(i, j)];
      if ((checks & 1) && a != a) out |= 1;
      if ((checks & 2) && !(fabs(a - A[IDX(j, i)]) <= tol)) out |= 2;
      if ((checks & 4) && i == j && a == 0.0) out |= 4;
    }
  }
  return out;
}

/*
 * Marginal log density of a zero-mean GP regression and its gradient: the
 * per-gradient work of the paper's GP example (§4.2, the
 * model of Betancourt 2017: y ~ multi_normal_cholesky(0, chol(K))), whose
 * cost is the Cholesky + adjoint hot path:
 *   K     = SE(x; alpha, rho) + sigma^2 I                      (oracle_se_cov)
 *   L     = chol(K)                                            (oracle_cholesky)
 *   z     = L^-1 y                                             (oracle_trsv)
 *   lp    = -1/2 z.z - sum_i log L_ii - n/2 log(2 pi)
 *   a     = L^-T z  (= K^-1 y)                                 (oracle_trsv)
 *   L_bar = tril(a z^T) - diag(1 / L_ii)      (d lp / d L, lower part)
 *   A_bar = cholesky_adjoint(L, L_bar)                         (oracle_cholesky_adjoint)
 *   d lp / d theta = sum_{i >= j} A_bar[i][j] d K_ij / d theta  (A_bar's lower
 *     entries are the adjoints of the symmetric pairs, R5), with
 *     E_ij = exp((x_i - x_j)^2 (-0.5 / rho^2)):
 *     d K_ij / d alpha = 2 alpha E_ij,  d K_ij / d rho = alpha^2 E_ij (x_i - x_j)^2 / rho^3,
 *     d K_ij / d sigma = 2 sigma [i == j]
 *   d lp / d y = -a.
 * out[0] = lp, out[1..3] = d lp / d (alpha, rho, sigma); ybar (may be NULL) = -a.
 * Returns 0, the Cholesky info (k+1) if K is not positive definite, or -2 on
 * allocation failure.  Sums in ascending index order.
 */
int oracle_gp_lpdf_grad(int64_t n, const double* x, const double* y, double alpha, double rho, double sigma,
                        double* out, double* ybar) {
  size_t nn = (size_t)n * (size_t)n;
  double* K = (double*)malloc(sizeof(double) * (nn ? nn : 1));
  double* L = (double*)malloc(sizeof(double) * (nn ? nn : 1));
  double* z = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
  double* a = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
  if (!K || !L || !z || !a) {
    free(K); free(L); free(z); free(a);
    return -2;
  }
  oracle_se_cov(n, x, alpha, rho, sigma * sigma, K);
  int info = oracle_cholesky(n, K, L);
  if (info != 0) {
    free(K); free(L); free(z); free(a);
    return info;
  }
  oracle_trsv(n, L, y, 0, z);
  double zz = 0.0, logdet = 0.0;
  for (int64_t i = 0; i < n; ++i) zz = zz + z[i] * z[i];
  for (int64_t i = 0; i < n; ++i) logdet = logdet + log(L[IDX(i, i)]);
  const double log_2pi = 1.8378770664093454835606594728112;  /* log(2 pi) */
  out[0] = -0.5 * zz - logdet - 0.5 * (double)n * log_2pi;
  oracle_trsv(n, L, z, 1, a);
  /* L_bar into K (K is no longer needed); A_bar in place of L_bar */
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double v = 0.0;
      if (j < i) v = a[i] * z[j];
      if (j == i) v = a[i] * z[i] - 1.0 / L[IDX(i, i)];
      K[IDX(i, j)] = v;
    }
  info = oracle_cholesky_adjoint(n, L, K, K);
  if (info != 0) {
    free(K); free(L); free(z); free(a);
    return info;
  }
  double g_alpha = 0.0, g_rho = 0.0, g_sigma = 0.0;
  const double neg_half_inv_rho2 = -0.5 / (rho * rho);
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t j = 0; j <= i; ++j) {
      double d = x[i] - x[j];
      double e = exp(d * d * neg_half_inv_rho2);
      double ab = K[IDX(i, j)];
      g_alpha = g_alpha + ab * (2.0 * alpha * e);
      g_rho = g_rho + ab * (alpha * alpha * e * (d * d) / (rho * rho * rho));
      if (i == j) g_sigma = g_sigma + ab * (2.0 * sigma);
    }
  }
  out[1] = g_alpha;
  out[2] = g_rho;
  out[3] = g_sigma;
  if (ybar)
    for (int64_t i = 0; i < n; ++i) ybar[i] = -a[i];
  free(K); free(L); free(z); free(a);
  return 0;
}
