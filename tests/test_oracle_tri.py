"""Pins of the oracle's triangular primitives (NEXT-2, §3.2):
lower triangular inverse, multi-RHS triangular solve and its reverse mode.
Each pin is fixed by mathematics, not by re-running the oracle's own formula:
integer-exact round trips (any correct substitution returns the exact integers),
exact IEEE reciprocals, a 2 x 2 closed form, and finite differences."""
from __future__ import annotations

import numpy as np
import pytest
import scipy.linalg as sla

import oracle
from paper_1907_01063_b200 import inputs


def se_chol(n, jitter=1e-3, seed=42):
    return np.linalg.cholesky(oracle.se_cov(inputs.gp_x(n, seed), 1.0, 1.0, jitter))


# ------------------------------------------------------------ tri_inverse
def test_tri_inverse_2x2_closed_form():
    # [[a, 0], [b, c]]^-1 = [[1/a, 0], [-b/(a c), 1/c]], exact in binary64 here
    X = oracle.tri_inverse(np.array([[4.0, 0.0], [2.0, 8.0]]))
    assert np.array_equal(X, np.array([[0.25, 0.0], [-0.0625, 0.125]]))


@pytest.mark.parametrize("n,band", [(1, None), (7, None), (30, None), (300, 2), (257, 1)])
def test_tri_inverse_integer_exact(n, band):
    # unit-lower +-1 L: L^-1 is an integer matrix (|entries| < 2^53 here), so a
    # correct substitution returns it exactly and L X = X L = I with no rounding
    L = inputs.unit_lower_pm1(n, seed=n, band=band)
    X = oracle.tri_inverse(L)
    assert np.all(X == np.round(X)) and np.max(np.abs(X)) < 2.0 ** 50
    assert np.array_equal(L @ X, np.eye(n))
    assert np.array_equal(X @ L, np.eye(n))


def test_tri_inverse_se_factor():
    n = 200
    L = se_chol(n)
    X = oracle.tri_inverse(L)
    assert np.array_equal(np.diag(X), 1.0 / np.diag(L))          # IEEE-rounded reciprocals
    assert np.all(X[np.triu_indices(n, 1)] == 0.0) and not np.any(np.signbit(X[np.triu_indices(n, 1)]))
    assert np.linalg.norm(X @ L - np.eye(n)) <= 1e-10 * np.linalg.norm(X) * np.linalg.norm(L)


def test_tri_inverse_reads_lower_only_and_bad_diagonal():
    L = inputs.unit_lower_pm1(40, seed=3)
    G = L.copy()
    G[np.triu_indices(40, 1)] = np.nan
    assert np.array_equal(oracle.tri_inverse(G), oracle.tri_inverse(L))
    L[17, 17] = 0.0
    with pytest.raises(ValueError, match=r"L\[17\]\[17\]"):
        oracle.tri_inverse(L)


# ------------------------------------------------------------------- trsm
@pytest.mark.parametrize("n,m,band", [(1, 1, None), (5, 3, None), (200, 7, 2), (129, 64, 1), (64, 1, None)])
def test_trsm_integer_round_trip(n, m, band):
    L = inputs.unit_lower_pm1(n, seed=n + m, band=band)
    X0 = inputs.rng(5).integers(-5, 6, size=(n, m)).astype(np.float64)
    B = L @ X0                      # exact (integers far below 2^53)
    assert np.array_equal(oracle.trsm(L, B), X0)
    Bt = L.T @ X0
    assert np.array_equal(oracle.trsm(L, Bt, trans=True), X0)


def test_trsm_non_unit_diagonal_exact():
    # L = [[1,0,0],[2,3,0],[4,5,6]] (SURVEY.md §8(c) example) with B = L X0: the
    # substitution divides by 3 and 6 -- still exact for these right-hand sides
    L = np.array([[1.0, 0, 0], [2, 3, 0], [4, 5, 6]])
    X0 = np.array([[1.0, -2.0], [3.0, 0.5], [-1.0, 2.0]])
    assert np.array_equal(oracle.trsm(L, L @ X0), X0)
    assert np.array_equal(oracle.trsm(L, L.T @ X0, trans=True), X0)


def test_trsm_columns_independent_and_lower_only():
    n, m = 50, 6
    L = se_chol(n)
    B = inputs.rng(1).standard_normal((n, m))
    X = oracle.trsm(L, B)
    Lg = L.copy()
    Lg[np.triu_indices(n, 1)] = np.nan
    assert np.array_equal(oracle.trsm(Lg, B), X)
    for c in (0, 3, 5):
        assert np.array_equal(oracle.trsm(L, B[:, c:c + 1])[:, 0], X[:, c])
    assert np.linalg.norm(L @ X - B) <= 1e-12 * np.linalg.norm(L) * np.linalg.norm(X)


# ---------------------------------------------------------- trsm_adjoint
def test_trsm_adjoint_n1_closed_form():
    # C = B / l; B_bar = C_bar / l; L_bar = -sum_c B_bar_c C_c
    Lb, Bb = oracle.trsm_adjoint(np.array([[2.0]]), np.array([[1.5, 2.5]]), np.array([[1.0, -1.0]]))
    assert np.array_equal(Bb, np.array([[0.5, -0.5]]))
    assert np.array_equal(Lb, np.array([[0.5]]))


@pytest.mark.parametrize("n,m", [(6, 1), (12, 5), (20, 3)])
def test_trsm_adjoint_finite_differences(n, m):
    # f(L, B) = sum W o (L^-1 B): central differences in every B entry and every
    # lower L entry against (B_bar, L_bar) at C_bar = W
    L = se_chol(n, jitter=0.1, seed=n)
    B = inputs.rng(2).standard_normal((n, m))
    W = inputs.rng(3).standard_normal((n, m))

    def f(Lx, Bx):
        return float(np.sum(W * sla.solve_triangular(Lx, Bx, lower=True)))

    C = sla.solve_triangular(L, B, lower=True)
    Lbar, Bbar = oracle.trsm_adjoint(L, C, W)
    h = 1e-5
    fdB = np.zeros_like(B)
    for i in range(n):
        for c in range(m):
            e = np.zeros_like(B)
            e[i, c] = h
            fdB[i, c] = (f(L, B + e) - f(L, B - e)) / (2 * h)
    assert np.linalg.norm(fdB - Bbar) <= 1e-7 * np.linalg.norm(Bbar)
    fdL = np.zeros_like(L)
    for i in range(n):
        for j in range(i + 1):
            e = np.zeros_like(L)
            e[i, j] = h * max(1.0, abs(L[i, j]))
            fdL[i, j] = (f(L + e, B) - f(L - e, B)) / (2 * e[i, j])
    assert np.linalg.norm(fdL - Lbar) <= 1e-6 * np.linalg.norm(Lbar)
    assert np.all(Lbar[np.triu_indices(n, 1)] == 0.0)


# ----------------------------------------------------- input checks (NEXT-3)
def test_check_matrix_pins():
    # check_nan, check_symmetric (absolute tolerance), check_diagonal_zeros
    A = np.array([[4.0, 2.0, 1.0], [2.0, 5.0, 0.5], [1.0, 0.5, 3.0]])
    assert oracle.check_matrix(A) == 0
    B = A.copy()
    B[2, 0] = np.nan
    assert oracle.check_matrix(B) == 1 | 2              # a NaN pair is also not symmetric
    assert oracle.check_matrix(B, checks=1) == 1
    C = A.copy()
    C[0, 1] += 1e-9                                      # within 1e-8: symmetric
    assert oracle.check_matrix(C) == 0
    C[0, 1] += 2e-8                                      # now 3e-8 apart
    assert oracle.check_matrix(C) == 2
    assert oracle.check_matrix(C, tol=1e-7) == 0
    D = A.copy()
    D[1, 1] = 0.0
    assert oracle.check_matrix(D) == 4
    assert oracle.check_matrix(D, checks=3) == 0
    E = A.copy()
    E[1, 1] = -0.0                                       # -0.0 == 0: a zero on the diagonal
    assert oracle.check_matrix(E, checks=4) == 4
    assert oracle.check_matrix(np.zeros((0, 0))) == 0
    assert oracle.check_matrix(np.full((1, 1), np.inf)) == 2   # inf - inf is NaN: not within tol
