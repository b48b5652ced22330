"""GPU parity for the NEXT rows around the hot path: the triangular solve
(stan_cl_trsv, NEXT-2) and the GP log density + gradient (stan_cl_gp_lpdf_grad,
NEXT-1), against the oracle on the same seeded inputs.

Bars: solves 1e-11 relative 2-norm on SE factors (cond(L) <= 1e3 at sigma =
0.1), bit-exact on the integer family; lp 1e-10 relative; hyperparameter
gradients 1e-8 relative (they are A_bar-weighted sums, A_bar's bar is 1e-9);
y_bar 1e-10 relative.
"""
from __future__ import annotations

import math

import numpy as np
import pytest
import torch

import oracle
from paper_1907_01063_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sc():
    import paper_1907_01063_b200 as m
    m.load()
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("n", [1, 2, 63, 64, 65, 200, 1000, 4096])
def test_trsv_parity(sc, n):
    L = oracle.cholesky(oracle.se_cov(inputs.gp_x(n), 1.0, 1.0, 0.01))
    b = inputs.rng(n).standard_normal(n)
    Ld = dev(L)
    for trans in (False, True):
        got = sc.trsv(Ld, dev(b), trans=trans).cpu().numpy()
        assert rel(got, oracle.trsv(L, b, trans=trans)) <= 1e-11


@pytest.mark.parametrize("n,band", [(64, 2), (300, 1), (1000, 2), (5000, 2), (777, None)])
def test_trsv_integer_round_trip(sc, n, band):
    L = inputs.unit_lower_pm1(n, seed=n, band=band if band else None)
    if band is None:  # dense +-1 L: keep x0 tiny so |b| stays far below 2^53
        L = inputs.unit_lower_pm1(n, seed=n, band=8)
    x0 = inputs.rng(n).integers(-5, 6, n).astype(np.float64)
    Ld = dev(L)
    assert np.array_equal(sc.trsv(Ld, dev(L @ x0)).cpu().numpy(), x0)
    assert np.array_equal(sc.trsv(Ld, dev(L.T @ x0), trans=True).cpu().numpy(), x0)


def test_trsv_in_place_upper_garbage_and_errors(sc):
    n = 300
    L = oracle.cholesky(oracle.se_cov(inputs.gp_x(n), 1.0, 1.0, 0.01))
    Lg = L.copy()
    Lg[np.triu_indices(n, 1)] = np.nan  # upper triangle never read
    b = inputs.rng(1).standard_normal(n)
    bd = dev(b)
    sc.trsv(dev(Lg), bd, out=bd)
    assert rel(bd.cpu().numpy(), oracle.trsv(L, b)) <= 1e-11
    Lz = L.copy()
    Lz[7, 7] = 0.0
    with pytest.raises(ValueError):
        sc.trsv(dev(Lz), dev(b))
    lib = sc.load()
    assert lib.stan_cl_trsv(-1, None, None, None, 0) == -1
    assert lib.stan_cl_trsv(0, None, None, None, 0) == 0


def grad_term_scale(x, y, a, r, s):
    """S_theta = sum_{i>=j} |A_bar_ij dK_ij/dtheta| for theta = alpha, rho, sigma:
    the size of the terms the hyperparameter gradient sums (their cancellation is
    what makes |g| small), so the rounding error of any summation order is
    O(eps * n * S_theta) -- the scale the absolute tolerance is tied to (instead
    of |lp|).  A_bar from the oracle's pieces."""
    n = x.shape[0]
    K = oracle.se_cov(x, a, r, s * s)
    L = oracle.cholesky(K)
    z = oracle.trsv(L, y)
    al = oracle.trsv(L, z, trans=True)
    Lbar = np.tril(np.outer(al, z)) - np.diag(1.0 / np.diag(L))
    Ab = np.tril(oracle.cholesky_adjoint(L, Lbar))
    d = x[:, None] - x[None, :]
    E = np.exp(d * d * (-0.5 / (r * r)))
    dK = [2 * a * E, a * a * E * d * d / r ** 3, 2 * s * np.eye(n)]
    return [float(np.sum(np.abs(Ab * t))) for t in dK]


@pytest.mark.parametrize("n", [1, 2, 64, 100, 300, 1000, 2048])
def test_gp_lpdf_grad_parity(sc, n):
    x = inputs.gp_x(n)
    y = inputs.gp_y(x)
    for a, r, s in [(1.0, 1.0, 0.1), (0.8, 2.3, 0.25)]:
        lp_o, g_o, yb_o = oracle.gp_lpdf_grad(x, y, a, r, s)
        out, yb = sc.gp_lpdf_grad(dev(x), dev(y), a, r, s)
        out = out.cpu().numpy()
        assert math.isclose(out[0], lp_o, rel_tol=1e-10)
        S = grad_term_scale(x, y, a, r, s)
        for k in range(3):
            # relative 1e-8 of the value, or 1e-12 of the summed term magnitudes
            # (eps * sqrt(n) headroom: 2048 terms per row at 1.1e-16 ~ 5e-15 per term)
            assert math.isclose(out[1 + k], g_o[k], rel_tol=1e-8, abs_tol=1e-12 * S[k]), (k, out[1 + k], g_o[k], S[k])
        assert rel(yb.cpu().numpy(), yb_o) <= 1e-10


def test_gp_lpdf_grad_not_pd_and_errors(sc):
    with pytest.raises(sc.NotPositiveDefinite) as e:
        sc.gp_lpdf_grad(dev(np.array([0.5, 0.5])), dev(np.array([1.0, 2.0])), 1.0, 1.0, 0.0)
    assert e.value.info == 2
    lib = sc.load()
    t = torch.zeros(4, dtype=torch.float64, device="cuda")
    assert lib.stan_cl_gp_lpdf_grad(3, t.data_ptr(), t.data_ptr(), 1.0, 0.0, 0.1, t.data_ptr(), None) == -1
    assert lib.stan_cl_gp_lpdf_grad(-1, None, None, 1.0, 1.0, 0.1, None, None) == -1
    t.fill_(7.0)
    assert lib.stan_cl_gp_lpdf_grad(0, None, None, 1.0, 1.0, 0.1, t.data_ptr(), None) == 0
    torch.cuda.synchronize()
    assert torch.equal(t, torch.zeros_like(t))
