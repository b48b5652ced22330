"""Pins for the oracle's NEXT-1/NEXT-2 functions (oracle_trsv, oracle_gp_lpdf_grad)
and the GP data recipe, against closed forms, exact integer round trips,
independent library routines and finite differences (CPU, -m "not gpu").
"""
from __future__ import annotations

import math

import numpy as np
import pytest
import scipy.integrate
import scipy.linalg
import scipy.stats

import oracle
from paper_1907_01063_b200 import inputs


# ------------------------------------------------------------- data recipe
def test_gp_mean_function_moments():
    """alpha, beta such that E[f] = 0 and Var[f] = 1 under
    x ~ Unif(-10, 10).  E[g] = E[x^2] = 100/3 in closed form; the variance is
    checked with adaptive quadrature (independent of the module's Gauss-Legendre)."""
    assert abs(inputs.GP_F_ALPHA - 100.0 / 3.0) < 1e-10
    mean = scipy.integrate.quad(lambda t: inputs.gp_f(np.array([t]))[0] / 20.0, -10, 10, limit=500)[0]
    var = scipy.integrate.quad(lambda t: inputs.gp_f(np.array([t]))[0] ** 2 / 20.0, -10, 10, limit=500)[0]
    assert abs(mean) < 1e-9 and abs(var - 1.0) < 1e-9


def test_gp_y_noise_level():
    x = inputs.gp_x(200000)
    r = inputs.gp_y(x) - inputs.gp_f(x)
    assert abs(r.std() - 0.1) < 1e-3 and abs(r.mean()) < 1e-3


# ------------------------------------------------------------- triangular solve
@pytest.mark.parametrize("n,band", [(1, None), (7, None), (200, 2), (300, 1)])
def test_trsv_integer_round_trip(n, band):
    """Unit-lower L with entries in {-1, 0, 1} and integer x0: b = L x0 is exact
    in binary64, and substitution must return x0 bit for bit (both directions)."""
    L = inputs.unit_lower_pm1(n, seed=n, band=band)
    x0 = inputs.rng(n).integers(-5, 6, n).astype(np.float64)
    assert np.array_equal(oracle.trsv(L, L @ x0), x0)
    assert np.array_equal(oracle.trsv(L, L.T @ x0, trans=True), x0)


def test_trsv_vs_library():
    n = 60
    K = oracle.se_cov(inputs.gp_x(n), 1.0, 1.0, 0.01)
    L = oracle.cholesky(K)
    b = inputs.rng(5).standard_normal(n)
    for trans in (False, True):
        want = scipy.linalg.solve_triangular(L, b, lower=True, trans=1 if trans else 0)
        got = oracle.trsv(L, b, trans=trans)
        assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)


def test_trsv_reads_lower_only_and_errors():
    L = np.array([[2.0, 99.0], [1.0, 4.0]])
    assert np.allclose(oracle.trsv(L, np.array([2.0, 5.0])), [1.0, 1.0])
    with pytest.raises(ValueError):
        oracle.trsv(np.array([[1.0, 0.0], [1.0, 0.0]]), np.ones(2))


# ------------------------------------------------------------- GP log density
def _K(x, alpha, rho, sigma):
    d = x[:, None] - x[None, :]
    return alpha ** 2 * np.exp(-0.5 * d * d / rho ** 2) + sigma ** 2 * np.eye(x.shape[0])


def test_gp_n1_closed_form():
    """n = 1: K = alpha^2 + sigma^2, lp = -y^2/(2K) - log(K)/2 - log(2 pi)/2."""
    a, r, s, y = 1.3, 0.9, 0.2, 0.7
    K = a * a + s * s
    lp, g, yb = oracle.gp_lpdf_grad(np.array([0.3]), np.array([y]), a, r, s)
    dK = 0.5 * y * y / K ** 2 - 0.5 / K
    assert math.isclose(lp, -0.5 * y * y / K - 0.5 * math.log(K) - 0.5 * math.log(2 * math.pi), rel_tol=1e-15)
    assert math.isclose(g[0], dK * 2 * a, rel_tol=1e-14)
    assert g[1] == 0.0
    assert math.isclose(g[2], dK * 2 * s, rel_tol=1e-14)
    assert math.isclose(yb[0], -y / K, rel_tol=1e-15)


@pytest.mark.parametrize("n", [5, 30, 120])
def test_gp_lp_matches_independent_density(n):
    """lp against scipy's multivariate normal log density (eigen-based, no Cholesky)."""
    x = inputs.gp_x(n)
    y = inputs.gp_y(x)
    for a, r, s in [(1.0, 1.0, 0.1), (0.7, 2.5, 0.3)]:
        lp, _, _ = oracle.gp_lpdf_grad(x, y, a, r, s)
        want = scipy.stats.multivariate_normal(mean=np.zeros(n), cov=_K(x, a, r, s)).logpdf(y)
        assert math.isclose(lp, want, rel_tol=1e-10)


@pytest.mark.parametrize("n", [5, 30, 120])
def test_gp_gradient_trace_form(n):
    """d lp / d theta = 1/2 tr((a a^T - K^-1) dK/dtheta), a = K^-1 y, with an
    explicit inverse (independent of the Cholesky adjoint); d lp / d y = -a."""
    x = inputs.gp_x(n)
    y = inputs.gp_y(x)
    a_, r_, s_ = 0.8, 1.7, 0.15
    lp, g, yb = oracle.gp_lpdf_grad(x, y, a_, r_, s_)
    K = _K(x, a_, r_, s_)
    Ki = np.linalg.inv(K)
    a = Ki @ y
    W = np.outer(a, a) - Ki
    d = x[:, None] - x[None, :]
    E = np.exp(-0.5 * d * d / r_ ** 2)
    dK = [2 * a_ * E, a_ ** 2 * E * d * d / r_ ** 3, 2 * s_ * np.eye(n)]
    want = [0.5 * np.sum(W * D) for D in dK]
    for gi, wi in zip(g, want):
        assert math.isclose(gi, wi, rel_tol=1e-8, abs_tol=1e-10)
    assert np.linalg.norm(yb + a) <= 1e-9 * np.linalg.norm(a)


def test_gp_gradient_finite_differences():
    """5-point central differences of the oracle's own lp in alpha, rho, sigma, y."""
    n = 16
    x = inputs.gp_x(n)
    y = inputs.gp_y(x)
    th = np.array([0.9, 1.4, 0.2])
    lp0, g, yb = oracle.gp_lpdf_grad(x, y, *th)

    def f(t, yy=y):
        return oracle.gp_lpdf_grad(x, yy, *t)[0]

    for k in range(3):
        h = 1e-3 * th[k]
        e = np.zeros(3)
        e[k] = h
        fd = (-f(th + 2 * e) + 8 * f(th + e) - 8 * f(th - e) + f(th - 2 * e)) / (12 * h)
        assert math.isclose(g[k], fd, rel_tol=1e-7, abs_tol=1e-9)
    for i in (0, 7, 15):
        h = 1e-4
        e = np.zeros(n)
        e[i] = h
        fd = (-f(th, y + 2 * e) + 8 * f(th, y + e) - 8 * f(th, y - e) + f(th, y - 2 * e)) / (12 * h)
        assert math.isclose(yb[i], fd, rel_tol=1e-7, abs_tol=1e-9)


def test_gp_not_positive_definite():
    """Duplicate inputs with sigma = 0: K = [[1, 1], [1, 1]], second pivot exactly 0."""
    with pytest.raises(oracle.NotPositiveDefinite) as e:
        oracle.gp_lpdf_grad(np.array([0.5, 0.5]), np.array([1.0, 2.0]), 1.0, 1.0, 0.0)
    assert e.value.info == 2
