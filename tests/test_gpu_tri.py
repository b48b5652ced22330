"""GPU parity of the NEXT-2 triangular primitives (§3.2) through
the C ABI: lower_triangular_inverse, multi-RHS trsm (both transposes) and the
solve's reverse mode, against oracle/ (tests/test_oracle_tri.py pins the
oracle).  Bar: relative Frobenius 1e-11 (measured <= 1e-13 on SE factors with
jitter 1e-6 up to n = 3000, profiles/r02_tri_probe.jsonl); integer-exact
families bit for bit."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from paper_1907_01063_b200 import inputs

pytestmark = pytest.mark.gpu
TOL = 1e-11


@pytest.fixture(scope="module")
def sc():
    import paper_1907_01063_b200 as m
    m.load()
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def relf(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def se_L(n, jitter=1e-6, seed=inputs.X_SEED):
    return oracle.cholesky_par(oracle.se_cov(inputs.gp_x(n, seed), 1.0, 1.0, jitter))


NS = [1, 2, 63, 127, 128, 129, 255, 256, 300, 513, 767, 768, 1000, 1024, 1280, 2048, 2500]


@pytest.mark.parametrize("n", NS)
def test_tri_inverse_parity(sc, n):
    L = se_L(n)
    G = L.copy()
    G[np.triu_indices(n, 1)] = np.nan                 # upper triangle never read
    X = sc.lower_triangular_inverse(dev(G)).cpu().numpy()
    assert relf(X, oracle.tri_inverse(L)) <= TOL
    up = X[np.triu_indices(n, 1)]
    assert np.all(up == 0.0) and not np.any(np.signbit(up))


@pytest.mark.parametrize("n", [300, 1024, 3000, 4096])
def test_tri_inverse_integer_exact(sc, n):
    # unit-lower +-1 bidiagonal-band L: L^-1 has entries in {-1, 0, 1} and every
    # partial sum is an integer, so every correct blocking returns it exactly
    L = inputs.unit_lower_pm1(n, seed=n, band=1)
    X = sc.lower_triangular_inverse(dev(L)).cpu().numpy()
    assert np.array_equal(X, oracle.tri_inverse(L))
    assert np.array_equal(L @ X, np.eye(n))


@pytest.mark.parametrize("n", [1, 100, 128, 257, 768, 1000, 2048])
@pytest.mark.parametrize("m", [1, 7, 64, 100])
@pytest.mark.parametrize("trans", [False, True])
def test_trsm_parity(sc, n, m, trans):
    L = se_L(n)
    B = inputs.rng(n + m).standard_normal((n, m))
    X = sc.trsm(dev(L), dev(B), trans).cpu().numpy()
    assert relf(X, oracle.trsm(L, B, trans)) <= TOL


@pytest.mark.parametrize("n,m", [(300, 33), (1024, 64), (4096, 128), (5000, 3)])
def test_trsm_integer_round_trip(sc, n, m):
    L = inputs.unit_lower_pm1(n, seed=n, band=1)
    X0 = inputs.rng(5).integers(-5, 6, size=(n, m)).astype(np.float64)
    assert np.array_equal(sc.trsm(dev(L), dev(L @ X0)).cpu().numpy(), X0)
    assert np.array_equal(sc.trsm(dev(L), dev(L.T @ X0), True).cpu().numpy(), X0)


def test_trsm_in_place_and_errors(sc):
    n, m = 1024, 64
    L = se_L(n)
    B = inputs.rng(1).standard_normal((n, m))
    Bd = dev(B)
    sc.trsm(dev(L), Bd, out=Bd)
    assert relf(Bd.cpu().numpy(), oracle.trsm(L, B)) <= TOL
    Lz = L.copy()
    Lz[500, 500] = 0.0
    with pytest.raises(ValueError, match=r"L\[500\]\[500\]"):
        sc.trsm(dev(Lz), dev(B))
    with pytest.raises(ValueError, match=r"L\[500\]\[500\]"):
        sc.lower_triangular_inverse(dev(Lz))
    lib = sc.load()
    assert lib.stan_cl_trsm(-1, 1, None, None, None, 0) == -1
    assert lib.stan_cl_trsm(0, 5, None, None, None, 0) == 0
    assert lib.stan_cl_trsm(5, 0, None, None, None, 0) == 0
    Ld = dev(L)
    assert lib.stan_cl_lower_triangular_inverse(n, Ld.data_ptr(), Ld.data_ptr()) == -1   # no aliasing
    assert lib.stan_cl_lower_triangular_inverse(0, None, None) == 0


@pytest.mark.parametrize("n,m", [(1, 1), (5, 2), (128, 64), (300, 7), (1000, 100), (2048, 33)])
def test_trsm_adjoint_parity(sc, n, m):
    L = se_L(n)
    B = inputs.rng(n).standard_normal((n, m))
    C = oracle.trsm(L, B)
    W = inputs.rng(n + 1).standard_normal((n, m))
    Lbo, Bbo = oracle.trsm_adjoint(L, C, W)
    Lbg, Bbg = sc.trsm_adjoint(dev(L), dev(C), dev(W))
    Lbg = Lbg.cpu().numpy()
    assert relf(Lbg, Lbo) <= TOL
    assert relf(Bbg.cpu().numpy(), Bbo) <= TOL
    up = Lbg[np.triu_indices(n, 1)]
    assert np.all(up == 0.0) and not np.any(np.signbit(up))


def test_trsm_adjoint_integer_exact(sc):
    # integer L (band 1), C and C_bar: B_bar = L^-T C_bar and -B_bar C^T are exact
    n, m = 2048, 40
    L = inputs.unit_lower_pm1(n, seed=9, band=1)
    C = inputs.rng(2).integers(-3, 4, size=(n, m)).astype(np.float64)
    W = inputs.rng(3).integers(-3, 4, size=(n, m)).astype(np.float64)
    Lbo, Bbo = oracle.trsm_adjoint(L, C, W)
    Lbg, Bbg = sc.trsm_adjoint(dev(L), dev(C), dev(W))
    assert np.array_equal(Bbg.cpu().numpy(), Bbo)
    assert np.array_equal(Lbg.cpu().numpy(), Lbo)


def test_tri_primitives_in_caller_workspace(sc):
    n, m = 1000, 50
    buf = torch.empty(max(sc.workspace_bytes(n), int(sc.load().stan_cl_trsm_workspace_bytes(n, m))) // 8 + 1,
                      dtype=torch.float64, device="cuda")
    sc.set_workspace(buf)
    try:
        L = se_L(n)
        assert relf(sc.lower_triangular_inverse(dev(L)).cpu().numpy(), oracle.tri_inverse(L)) <= TOL
        B = inputs.rng(4).standard_normal((n, m))
        assert relf(sc.trsm(dev(L), dev(B)).cpu().numpy(), oracle.trsm(L, B)) <= TOL
        C = oracle.trsm(L, B)
        Lbo, Bbo = oracle.trsm_adjoint(L, C, B)
        Lbg, Bbg = sc.trsm_adjoint(dev(L), dev(C), dev(B))
        assert relf(Lbg.cpu().numpy(), Lbo) <= TOL and relf(Bbg.cpu().numpy(), Bbo) <= TOL
    finally:
        sc.set_workspace(None)
