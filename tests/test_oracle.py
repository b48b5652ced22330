"""Pins for the CPU oracle (``oracle/``) against what the paper and mathematics fix.

None of these re-types the oracle's loops: each check is a closed form, an
identity, an exact (rational) computation, an independent library routine, the
paper's own blocked listing, or finite differences.  Runs on CPU (-m "not gpu").
"""
from __future__ import annotations

import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from paper_1907_01063_b200 import inputs
from tests.paper_blocked import blocked_adjoint, blocked_cholesky

GOLD = os.path.join(os.path.dirname(__file__), "golden", "cholesky_cases.json")


def relf(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def se(n, seed=42, alpha=1.0, rho=1.0, jitter=1e-6):
    return oracle.se_cov(inputs.gp_x(n, seed), alpha, rho, jitter)


# ---------------------------------------------------------------- golden cases
@pytest.fixture(scope="module")
def gold():
    with open(GOLD) as f:
        return json.load(f)


def test_forward_golden(gold):
    for case in gold["forward"]:
        L = oracle.cholesky(np.array(case["A"], float))
        assert np.array_equal(L, np.array(case["L"], float)), case["cite"]


def test_toeplitz3_closed_form(gold):
    A = np.array(gold["toeplitz3"]["A"], float)
    assert np.array_equal(A, inputs.toeplitz(3))          # the paper's generator at n=3
    r77 = math.sqrt(77.0)
    want = np.array([[3, 0, 0], [2 / 3, r77 / 3, 0], [1 / 3, 16 / (3 * r77), math.sqrt(656 / 77)]])
    L = oracle.cholesky(A)
    assert np.max(np.abs(L - want)) <= 4 * np.finfo(float).eps * 3


def test_identity_and_empty():
    assert np.array_equal(oracle.cholesky(np.eye(8)), np.eye(8))
    L, info = oracle.cholesky_info(np.zeros((0, 0)))
    assert info == 0 and L.shape == (0, 0)


def test_not_positive_definite(gold):
    for case in gold["not_pd"]:
        _, info = oracle.cholesky_info(np.array(case["A"], float))
        assert info == case["info"], case["cite"]
    A = inputs.toeplitz(6)
    A[3, 3] = np.nan
    assert oracle.cholesky_info(A)[1] == 4                             # NaN pivot fails (R4)
    A = inputs.toeplitz(6)
    A[4, 4] = -1e9
    assert oracle.cholesky_info(A)[1] == 5


def test_upper_triangle_ignored_and_zeroed():
    A = se(40)
    G = A.copy()
    G[np.triu_indices(40, 1)] = np.nan                                 # garbage above the diagonal
    L1 = oracle.cholesky(A)
    L2 = oracle.cholesky(G)
    assert np.array_equal(L1, L2)
    up = L1[np.triu_indices(40, 1)]
    assert np.all(up == 0) and not np.any(np.signbit(up))


@pytest.mark.parametrize("n", [64, 256, 700])
def test_reconstruction_se(n):
    # ||L L^T - A||_F / ||A||_F <= 1e-13 (BASELINE.json north_star); L L^T by numpy BLAS
    A = se(n)
    L = oracle.cholesky(A)
    assert relf(L @ L.T, A) <= 1e-13
    assert np.all(np.diag(L) > 0)


def test_reconstruction_toeplitz():
    A = inputs.toeplitz(300)
    L = oracle.cholesky(A)
    assert relf(L @ L.T, A) <= 1e-15


def _bareiss_det(A) -> Fraction:
    """Exact determinant of a binary64 matrix (fraction-free Bareiss on rationals)."""
    M = [[Fraction(float(v)) for v in row] for row in A]
    n = len(M)
    sign = 1
    prev = Fraction(1)
    for k in range(n - 1):
        if M[k][k] == 0:
            for r in range(k + 1, n):
                if M[r][k] != 0:
                    M[k], M[r] = M[r], M[k]
                    sign = -sign
                    break
            else:
                return Fraction(0)
        for i in range(k + 1, n):
            for j in range(k + 1, n):
                M[i][j] = (M[i][j] * M[k][k] - M[i][k] * M[k][j]) / prev
        prev = M[k][k]
    return sign * M[n - 1][n - 1]


def _log_fraction(f: Fraction) -> float:
    return math.log(f.numerator) - math.log(f.denominator)


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("n", [2, 5, 8])
def test_logdet_exact_se(n, seed):
    # 2 sum log L_ii = log det A (north_star), det exact over the rationals
    A = se(n, seed=seed)
    L = oracle.cholesky(A)
    got = 2.0 * float(np.sum(np.log(np.diag(L))))
    want = _log_fraction(_bareiss_det(A))
    assert abs(got - want) <= 1e-10 * max(1.0, abs(want))


@pytest.mark.parametrize("n", [3, 6, 8])
def test_logdet_exact_toeplitz(n):
    A = inputs.toeplitz(n)
    L = oracle.cholesky(A)
    got = 2.0 * float(np.sum(np.log(np.diag(L))))
    want = _log_fraction(_bareiss_det(A))
    assert abs(got - want) <= 1e-14 * abs(want)


@pytest.mark.parametrize("n,band", [(64, None), (200, None), (300, 2)])
def test_integer_exact_family(n, band):
    # every correct Cholesky of A = L L^T (L unit-lower, entries in {-1,0,1})
    # returns L bit-for-bit: all partial sums are integers below 2^53
    L0 = inputs.unit_lower_pm1(n, seed=n, band=band)
    A = inputs.gram_exact(L0)
    assert np.array_equal(oracle.cholesky(A), L0)


def test_power_of_two_scaling_equivariance():
    """chol(D A D) = D chol(A) for D = diag(2^e): every step of the method
    (products, sums, sqrt, division) commutes exactly with power-of-two scaling
    while intermediates stay normal, so the oracle must reproduce D L BIT FOR
    BIT; a transposed or mis-indexed operand breaks the row scaling."""
    n = 64
    A = inputs.toeplitz(n)
    e = np.random.default_rng(7).integers(-400, 401, n).astype(np.float64)
    d = np.exp2(e)
    L = oracle.cholesky(A)
    assert np.array_equal(oracle.cholesky(A * d[:, None] * d[None, :]), L * d[:, None])


def test_long_double_twin():
    A = np.array([[4.0, 2.0], [2.0, 5.0]])
    assert np.array_equal(oracle.cholesky_ld(A), np.array([[2.0, 0], [1.0, 2.0]]))
    A = se(300)
    Ld = oracle.cholesky_ld(A)
    assert relf(oracle.cholesky(A), Ld) <= 1e-11         # floor, SURVEY.md §0 finding 3
    assert relf(Ld @ Ld.T, A) <= 1e-15 * 300


@pytest.mark.parametrize("n", [17, 96])
def test_matches_paper_blocked_forward(n):
    # the paper's recursive blocked listing reaches the same L up to rounding
    A = se(n, jitter=1e-3)
    for part, mn in [(2, 4), (4, 8), (3, 3)]:  # min_L11 >= partition, else R10
        assert relf(oracle.cholesky(A), blocked_cholesky(A, part, mn)) <= 1e-12


# ------------------------------------------------------------------ SE builder
def test_se_builder_properties():
    x = inputs.gp_x(300)
    for alpha, rho, jit in [(1.0, 1.0, 1e-6), (2.5, 0.3, 0.0), (0.7, 5.5, 1e-3)]:
        K = oracle.se_cov(x, alpha, rho, jit)
        assert np.array_equal(K, K.T)                                  # exact symmetry
        assert np.all(np.diag(K) == alpha * alpha + jit)               # exp(0) = 1
        off = K[~np.eye(300, dtype=bool)]
        assert np.all(off >= 0) and np.all(off <= alpha * alpha)      # may underflow to +0


def test_se_builder_closed_form_points():
    # half height at |d| = rho sqrt(2 ln 2); e^{-1/2} at |d| = rho; e^{-2} at 2 rho
    rho, alpha = 1.7, 3.0
    x = np.array([0.0, rho * math.sqrt(2 * math.log(2)), rho, 2 * rho])
    K = oracle.se_cov(x, alpha, rho, 0.0)
    a2 = alpha * alpha
    assert abs(K[1, 0] - a2 * 0.5) <= 4e-16 * a2
    assert abs(K[2, 0] - a2 * 0.6065306597126334) <= 4e-16 * a2      # e^{-1/2}
    assert abs(K[3, 0] - a2 * 0.1353352832366127) <= 4e-16 * a2      # e^{-2}


def test_gp_inputs_distribution():
    x = inputs.gp_x(100000)
    assert x.min() >= -10 and x.max() < 10
    assert abs(x.mean()) < 0.1 and abs(x.var() - 400 / 12) < 0.3    # Unif(-10,10)


# -------------------------------------------------------------------- adjoint
def test_adjoint_golden(gold):
    for case in gold["adjoint"]:
        got = oracle.cholesky_adjoint(np.array(case["L"], float), np.array(case["Lbar"], float))
        assert np.array_equal(got, np.array(case["Abar"], float)), case["cite"]


@pytest.mark.parametrize("seed", range(5))
def test_adjoint_2x2_closed_form(seed):
    g = np.random.default_rng(seed)
    a, c = 1 + 3 * g.random(), 2 + 3 * g.random()
    b = (g.random() - 0.5) * math.sqrt(a * c)
    p, q, r = g.standard_normal(3)
    L = oracle.cholesky(np.array([[a, b], [b, c]]))
    L22 = math.sqrt(c - b * b / a)
    want = np.array([[p / (2 * math.sqrt(a)) - q * b / (2 * a ** 1.5) + r * b * b / (2 * a * a * L22), 0.0],
                     [q / math.sqrt(a) - r * b / (a * L22), r / (2 * L22)]])
    got = oracle.cholesky_adjoint(L, np.array([[p, 0], [q, r]]))
    assert np.max(np.abs(got - want)) <= 1e-14 * max(1, np.max(np.abs(want)))


def test_adjoint_zero_linear_and_upper():
    A = se(30, jitter=1e-3)
    L = oracle.cholesky(A)
    assert np.array_equal(oracle.cholesky_adjoint(L, np.zeros_like(L)), np.zeros_like(L))
    W1, W2 = inputs.lbar(30, 1), inputs.lbar(30, 2)
    lhs = oracle.cholesky_adjoint(L, 2.0 * W1 - 3.0 * W2)
    rhs = 2.0 * oracle.cholesky_adjoint(L, W1) - 3.0 * oracle.cholesky_adjoint(L, W2)
    assert relf(lhs, rhs) <= 1e-13
    G = W1.copy()
    G[np.triu_indices(30, 1)] = np.nan                                   # upper of L_bar ignored
    Lg = L.copy()
    Lg[np.triu_indices(30, 1)] = np.nan                                  # upper of L ignored
    out = oracle.cholesky_adjoint(Lg, G)
    assert np.array_equal(out, oracle.cholesky_adjoint(L, W1))
    assert np.all(out[np.triu_indices(30, 1)] == 0)


def test_adjoint_bad_diagonal():
    L = np.eye(4)
    L[2, 2] = 0.0
    assert oracle.cholesky_adjoint_info(L, np.eye(4))[1] == 3
    L[2, 2] = np.inf
    assert oracle.cholesky_adjoint_info(L, np.eye(4))[1] == 3


def _phi(X):
    P = np.tril(X).copy()
    P[np.diag_indices_from(P)] *= 0.5
    return P


@pytest.mark.parametrize("kind", ["toeplitz", "se"])
def test_adjoint_logdet_identity(kind):
    # f = log det A = 2 sum log L_ii  =>  L_bar = diag(2/L_ii), A_bar = Phi(2 A^-1)
    n = 80
    A = inputs.toeplitz(n) if kind == "toeplitz" else se(n, jitter=1e-2)
    L = oracle.cholesky(A)
    Lbar = np.diag(2.0 / np.diag(L))
    want = _phi(2.0 * np.linalg.inv(A))
    assert relf(oracle.cholesky_adjoint(L, Lbar), want) <= (1e-13 if kind == "toeplitz" else 1e-10)


def test_adjoint_gp_density_identity():
    # f = -1/2 y^T A^-1 y - 1/2 log det A: L_bar = tril(a z^T) - diag(1/L_ii),
    # z = L^-1 y, a = L^-T z; then A_bar = Phi(a a^T - A^-1)
    n = 64
    A = se(n, jitter=1e-2)
    y = np.random.default_rng(5).standard_normal(n)
    L = oracle.cholesky(A)
    import scipy.linalg as sla
    z = sla.solve_triangular(L, y, lower=True)
    a = sla.solve_triangular(L.T, z, lower=False)
    Lbar = np.tril(np.outer(a, z)) - np.diag(1.0 / np.diag(L))
    want = _phi(np.outer(a, a) - np.linalg.inv(A))
    assert relf(oracle.cholesky_adjoint(L, Lbar), want) <= 1e-10


def _f_weighted(A, W):
    L, info = oracle.cholesky_info(A)
    assert info == 0
    return float(np.sum(W * L))


@pytest.mark.parametrize("n", [2, 4, 8, 16, 32])
def test_adjoint_finite_differences_se(n):
    # 5-point central differences of f(A) = sum W o chol(A), perturbing the
    # symmetric pair (i,j),(j,i) together; h = 1e-2 * jitter (lambda_min >= jitter)
    jitter = 1e-6
    A = se(n, seed=100 + n, jitter=jitter)
    W = inputs.lbar(n, seed=200 + n)
    h = 1e-2 * jitter
    fd = np.zeros((n, n))
    for i in range(n):
        for j in range(i + 1):
            E = np.zeros((n, n))
            E[i, j] = 1.0
            E[j, i] = 1.0
            f = [_f_weighted(A + s * h * E, W) for s in (2, 1, -1, -2)]
            fd[i, j] = (-f[0] + 8 * f[1] - 8 * f[2] + f[3]) / (12 * h)
    got = oracle.cholesky_adjoint(oracle.cholesky(A), W)
    assert relf(got, fd) <= 1e-6                                         # north_star FD bar


def test_adjoint_finite_differences_toeplitz():
    n = 24
    A = inputs.toeplitz(n)
    W = inputs.lbar(n, seed=9)
    h = 1e-5 * np.max(np.abs(A))
    fd = np.zeros((n, n))
    for i in range(n):
        for j in range(i + 1):
            E = np.zeros((n, n))
            E[i, j] = E[j, i] = 1.0
            fd[i, j] = (_f_weighted(A + h * E, W) - _f_weighted(A - h * E, W)) / (2 * h)
    assert relf(oracle.cholesky_adjoint(oracle.cholesky(A), W), fd) <= 1e-8


@pytest.mark.parametrize("n", [1, 2, 5, 17, 32, 130])
def test_adjoint_matches_paper_blocked(n):
    # the paper's blocked gradient (reading R6) at several
    # block sizes equals the oracle's unblocked reverse sweep
    A = se(n, jitter=1e-3)
    L = oracle.cholesky(A)
    W = inputs.lbar(n, seed=n)
    want = oracle.cholesky_adjoint(L, W)
    for bs in (1, 3, 8, 64):
        assert relf(blocked_adjoint(L, W, bs), want) <= 1e-12, bs


def test_adjoint_integer_exact_band():
    # banded (<=2) unit-lower +-1 L with integer L_bar: every intermediate is a
    # multiple of 1/2 below 2^53, so any blocking returns the same bits
    n = 256
    L = inputs.unit_lower_pm1(n, seed=3, band=2)
    W = inputs.int_lbar(n, seed=4)
    want = oracle.cholesky_adjoint(L, W)
    assert np.all(np.abs(want) < 2.0 ** 52)
    for bs in (1, 7, 64, 128):
        assert np.array_equal(blocked_adjoint(L, W, bs), want), bs


def test_adjoint_torch_autograd_crosscheck():
    # torch.linalg.cholesky's backward returns the symmetric gradient S;
    # Stan's convention (R5) is Phi(2 S)
    import torch
    n = 40
    A = se(n, jitter=1e-2)
    W = inputs.lbar(n, seed=77)
    At = torch.tensor(A, dtype=torch.float64, requires_grad=True)
    Lt = torch.linalg.cholesky(At)
    (Lt * torch.tensor(W)).sum().backward()
    S = At.grad.numpy()
    S = 0.5 * (S + S.T)
    want = _phi(2.0 * S)
    got = oracle.cholesky_adjoint(oracle.cholesky(A), W)
    assert relf(got, want) <= 1e-9


@pytest.mark.parametrize("n", [0, 1, 2, 31, 32, 33, 100, 257, 700])
def test_cholesky_par_bit_identical(n):
    # oracle_cholesky_par only reorders the computation of DIFFERENT entries:
    # every entry's own statements and operands are oracle_cholesky's, so the
    # bits agree exactly (SE, Toeplitz and integer families, 1-8 threads)
    mats = [se(n) if n else np.zeros((0, 0)), inputs.toeplitz(n)]
    if n:
        mats.append(inputs.gram_exact(inputs.unit_lower_pm1(n, seed=n)))
    for A in mats:
        want, info = oracle.cholesky_info(A)
        for t in (1, 3, 8):
            got, info_p = oracle.cholesky_par_info(A, t)
            assert info_p == info == 0
            assert np.array_equal(got.view(np.int64), want.view(np.int64)), (n, t)


def test_cholesky_par_not_pd_info():
    for n, row in ((100, 0), (100, 40), (300, 299), (257, 64)):
        A = inputs.toeplitz(n)
        A[row, row] = -1e12
        assert oracle.cholesky_par_info(A, 4)[1] == oracle.cholesky_info(A)[1] == row + 1


def test_golden_adjoint_inputs_reproducible():
    # tests/golden/oracle_adj_se_n8192.npz stores the SHA-256 of the sequential
    # oracle's L (tools/make_golden_adjoint.py); the multi-threaded twin used by
    # the GPU test must rebuild exactly those bits
    import hashlib
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "oracle_adj_se_n8192.npz"))
    n = int(g["n"])
    K = oracle.se_cov(inputs.gp_x(n, int(g["x_seed"])), float(g["alpha"]), float(g["rho"]), float(g["jitter"]))
    L = oracle.cholesky_par(K)
    assert hashlib.sha256(L.tobytes()).hexdigest() == str(g["L_sha256"])
    # the sampled A_bar entries sit in the lower triangle; the rows are complete
    assert np.all(g["ii"] >= g["jj"])
    rv = g["row_vals"]
    for r, row in zip(g["rows"], rv):
        assert np.all(row[r + 1:] == 0.0) and row[r] == g["diag"][r]
