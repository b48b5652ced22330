"""Seeded synthetic input generators shared by tests, bench.py and smoke().

This module holds NONE of the method's arithmetic (no covariance kernel, no
factorisation, no adjoint): it only draws the random numbers and builds the
integer test families.  Both the oracle and the CUDA path consume its output.

Recipes:
  * ``gp_x``      x_i ~ Unif(-10, 10) i.i.d., unsorted (§4.2).
  * ``gp_y``      y_i ~ N(f(x_i), sd 0.1), f(x) = beta (x + x^2 - x^3 + 100 sin 2x
    - alpha) with alpha, beta fixing E[f] = 0, Var[f] = 1 under Unif(-10, 10)
    ("1/10" read as the standard deviation, R16).
  * ``lbar``      L_bar = tril of N(0, 1) draws (the adjoint seed).
  * ``toeplitz``  A_ij = n - |i - j|, A_ii = n^2 (§3.3.3).
  * ``unit_lower_pm1``  unit-lower L with off-diagonal entries in {-1, 0, 1},
    optionally banded; A = L L^T is then factorised bit-exactly by every
    correct Cholesky (SURVEY.md §8(c) integer-exact family).
Generator: numpy PCG64 (a fixed, documented 64-bit generator; R15).
"""
from __future__ import annotations

import numpy as np

X_SEED = 42
LBAR_SEED = 43
Y_SEED = 44


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def gp_x(n: int, seed: int = X_SEED) -> np.ndarray:
    """n inputs x_i ~ Unif(-10, +10)."""
    return -10.0 + 20.0 * rng(seed).random(n)


def _gp_f_constants() -> tuple[float, float]:
    """alpha = E[g], beta = 1 / sd[g] for g(x) = x + x^2 - x^3 + 100 sin 2x,
    x ~ Unif(-10, 10), by 400-point Gauss-Legendre quadrature (exact for the
    polynomial part; the sin part converges far below 1e-14)."""
    t, w = np.polynomial.legendre.leggauss(400)
    xs = 10.0 * t
    w = w / 2.0  # density 1/20 times dx = 10 dt
    g = xs + xs ** 2 - xs ** 3 + 100.0 * np.sin(2.0 * xs)
    m = float(np.sum(w * g))
    v = float(np.sum(w * (g - m) ** 2))
    return m, 1.0 / np.sqrt(v)


GP_F_ALPHA, GP_F_BETA = _gp_f_constants()


def gp_f(x: np.ndarray) -> np.ndarray:
    """The paper's GP toy-data mean function."""
    return GP_F_BETA * (x + x ** 2 - x ** 3 + 100.0 * np.sin(2.0 * x) - GP_F_ALPHA)


def gp_y(x: np.ndarray, seed: int = Y_SEED, sd: float = 0.1) -> np.ndarray:
    """Targets y_i ~ N(f(x_i), sd)."""
    return gp_f(x) + sd * rng(seed).standard_normal(x.shape[0])


def lbar(n: int, seed: int = LBAR_SEED) -> np.ndarray:
    """Lower-triangular adjoint seed: tril of i.i.d. N(0,1); strict upper +0.0."""
    g = rng(seed)
    out = np.empty((n, n), dtype=np.float64)
    # row blocks keep the temporary small at large n
    step = max(1, (1 << 24) // max(n, 1))
    for r0 in range(0, n, step):
        r1 = min(n, r0 + step)
        blk = g.standard_normal((r1 - r0, n))
        ii = np.arange(r0, r1)[:, None]
        jj = np.arange(n)[None, :]
        blk[jj > ii] = 0.0
        out[r0:r1] = blk
    return out


def lbar_leading(n: int, m: int, seed: int = LBAR_SEED) -> np.ndarray:
    """lbar(n, seed)[:m, :m] without drawing the whole n x n matrix (the same
    row-block stream: only the blocks covering the first m rows are drawn)."""
    m = min(m, n)
    g = rng(seed)
    out = np.empty((m, m), dtype=np.float64)
    step = max(1, (1 << 24) // max(n, 1))
    for r0 in range(0, m, step):
        r1 = min(n, r0 + step)
        blk = g.standard_normal((r1 - r0, n))
        ii = np.arange(r0, r1)[:, None]
        jj = np.arange(n)[None, :]
        blk[jj > ii] = 0.0
        take = min(r1, m) - r0
        out[r0:r0 + take] = blk[:take, :m]
    return out


def toeplitz(n: int) -> np.ndarray:
    """The paper's Cholesky benchmark matrix."""
    i = np.arange(n)
    A = (n - np.abs(i[:, None] - i[None, :])).astype(np.float64)
    A[i, i] = float(n) * float(n)
    return A


def unit_lower_pm1(n: int, seed: int = 7, band: int | None = None, p_zero: float = 1.0 / 3.0) -> np.ndarray:
    """Unit-lower L, off-diagonal entries drawn from {-1, 0, +1}.

    ``band``: if given, only entries with 0 < i - j <= band are nonzero.
    """
    g = rng(seed)
    L = np.zeros((n, n), dtype=np.float64)
    step = max(1, (1 << 22) // max(n, 1))
    for r0 in range(0, n, step):
        r1 = min(n, r0 + step)
        vals = g.choice(np.array([-1.0, 0.0, 1.0]), size=(r1 - r0, n),
                        p=[(1 - p_zero) / 2, p_zero, (1 - p_zero) / 2])
        ii = np.arange(r0, r1)[:, None]
        jj = np.arange(n)[None, :]
        mask = jj < ii
        if band is not None:
            mask &= (ii - jj) <= band
        vals[~mask] = 0.0
        L[r0:r1] = vals
    L[np.arange(n), np.arange(n)] = 1.0
    return L


def int_lbar(n: int, seed: int = 11, lo: int = -3, hi: int = 3) -> np.ndarray:
    """Integer adjoint seed in {lo..hi}, lower triangular."""
    g = rng(seed)
    out = g.integers(lo, hi + 1, size=(n, n)).astype(np.float64)
    return np.tril(out)


def gram_exact(L: np.ndarray) -> np.ndarray:
    """A = L L^T for an integer L (exact: every partial sum is an integer < 2^53).

    Input construction only: any summation order gives the same bits here.
    """
    return L @ L.T
