"""CPU oracle for the FP64 Cholesky + adjoint hot path (arXiv:1907.01063).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_1907_01063_b200``) never imports it, and
the two share no code.

The arithmetic lives in ``oracle.c`` (plain C99, single thread, binary64,
``-O2 -ffp-contract=off``); this module only compiles it and marshals numpy
arrays through ctypes.  See ``oracle.c`` for the per-function citations.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-std=c99", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared"]

_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (gcc).  Returns the library path."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        D = ctypes.c_double
        lib.oracle_se_cov.argtypes = [I64, P, D, D, D, P]
        lib.oracle_se_cov.restype = None
        for name in ("oracle_cholesky", "oracle_cholesky_ld"):
            getattr(lib, name).argtypes = [I64, P, P]
            getattr(lib, name).restype = ctypes.c_int
        lib.oracle_cholesky_par.argtypes = [I64, P, P, ctypes.c_int]
        lib.oracle_cholesky_par.restype = ctypes.c_int
        lib.oracle_cholesky_adjoint.argtypes = [I64, P, P, P]
        lib.oracle_cholesky_adjoint.restype = ctypes.c_int
        lib.oracle_trsv.argtypes = [I64, P, P, ctypes.c_int, P]
        lib.oracle_trsv.restype = ctypes.c_int
        lib.oracle_tri_inverse.argtypes = [I64, P, P]
        lib.oracle_tri_inverse.restype = ctypes.c_int
        lib.oracle_trsm.argtypes = [I64, I64, P, P, ctypes.c_int, P]
        lib.oracle_trsm.restype = ctypes.c_int
        lib.oracle_trsm_adjoint.argtypes = [I64, I64, P, P, P, P, P]
        lib.oracle_trsm_adjoint.restype = ctypes.c_int
        lib.oracle_check_matrix.argtypes = [I64, P, ctypes.c_int, D]
        lib.oracle_check_matrix.restype = ctypes.c_int
        lib.oracle_gp_lpdf_grad.argtypes = [I64, P, P, D, D, D, P, P]
        lib.oracle_gp_lpdf_grad.restype = ctypes.c_int
        _lib = lib
    return _lib


def _c(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class NotPositiveDefinite(ValueError):
    def __init__(self, info: int):
        super().__init__(f"matrix not positive definite: first failing pivot at row {info - 1}")
        self.info = info


def se_cov(x, alpha: float = 1.0, rho: float = 1.0, jitter: float = 1e-6) -> np.ndarray:
    """K_ij = alpha^2 exp((x_i-x_j)^2 (-0.5/rho^2)) + jitter [i==j] (oracle.c)."""
    x = _c(x)
    n = x.shape[0]
    K = np.empty((n, n), dtype=np.float64)
    _load().oracle_se_cov(n, _ptr(x), float(alpha), float(rho), float(jitter), _ptr(K))
    return K


def cholesky_info(A) -> tuple[np.ndarray, int]:
    """(L, info): Cholesky-Banachiewicz; info = 0 or failing row + 1."""
    A = _c(A)
    n = A.shape[0]
    assert A.shape == (n, n)
    L = np.empty_like(A)
    info = _load().oracle_cholesky(n, _ptr(A), _ptr(L))
    return L, int(info)


def cholesky(A) -> np.ndarray:
    L, info = cholesky_info(A)
    if info != 0:
        raise NotPositiveDefinite(info)
    return L


def cholesky_par_info(A, nthreads: int = 0) -> tuple[np.ndarray, int]:
    """(L, info) of ``cholesky_info`` bit for bit, independent entries on
    ``nthreads`` threads (0 = all cores; oracle.c oracle_cholesky_par)."""
    A = _c(A)
    n = A.shape[0]
    assert A.shape == (n, n)
    L = np.empty_like(A)
    info = _load().oracle_cholesky_par(n, _ptr(A), _ptr(L), int(nthreads or os.cpu_count() or 1))
    return L, int(info)


def cholesky_par(A, nthreads: int = 0) -> np.ndarray:
    L, info = cholesky_par_info(A, nthreads)
    if info != 0:
        raise NotPositiveDefinite(info)
    return L


def cholesky_ld(A) -> np.ndarray:
    """Long-double twin of ``cholesky`` (truth proxy for floor studies)."""
    A = _c(A)
    n = A.shape[0]
    L = np.empty_like(A)
    info = _load().oracle_cholesky_ld(n, _ptr(A), _ptr(L))
    if info != 0:
        raise NotPositiveDefinite(info)
    return L


def cholesky_adjoint_info(L, Lbar) -> tuple[np.ndarray, int]:
    L = _c(L)
    Lbar = _c(Lbar)
    n = L.shape[0]
    assert L.shape == (n, n) and Lbar.shape == (n, n)
    Abar = np.empty_like(L)
    info = _load().oracle_cholesky_adjoint(n, _ptr(L), _ptr(Lbar), _ptr(Abar))
    return Abar, int(info)


def cholesky_adjoint(L, Lbar) -> np.ndarray:
    """A_bar given L and L_bar, Stan's Phi(G + G^T) convention (oracle.c)."""
    Abar, info = cholesky_adjoint_info(L, Lbar)
    if info != 0:
        raise ValueError(f"L[{info - 1}][{info - 1}] is not finite and > 0")
    return Abar


def trsv(L, b, trans: bool = False) -> np.ndarray:
    """x with L x = b (trans=False) or L^T x = b (trans=True); lower L (oracle.c)."""
    L = _c(L)
    b = _c(b)
    n = L.shape[0]
    assert L.shape == (n, n) and b.shape == (n,)
    x = np.empty_like(b)
    info = _load().oracle_trsv(n, _ptr(L), _ptr(b), int(bool(trans)), _ptr(x))
    if info != 0:
        raise ValueError(f"L[{info - 1}][{info - 1}] is zero or not finite")
    return x


def tri_inverse(L) -> np.ndarray:
    """X = L^-1 for lower-triangular L (oracle.c oracle_tri_inverse)."""
    L = _c(L)
    n = L.shape[0]
    assert L.shape == (n, n)
    X = np.empty_like(L)
    info = _load().oracle_tri_inverse(n, _ptr(L), _ptr(X))
    if info != 0:
        raise ValueError(f"L[{info - 1}][{info - 1}] is zero or not finite")
    return X


def trsm(L, B, trans: bool = False) -> np.ndarray:
    """X with L X = B (trans=False) or L^T X = B (trans=True); B n x m (oracle.c)."""
    L = _c(L)
    B = _c(B)
    n = L.shape[0]
    assert L.shape == (n, n) and B.ndim == 2 and B.shape[0] == n
    X = np.empty_like(B)
    info = _load().oracle_trsm(n, B.shape[1], _ptr(L), _ptr(B), int(bool(trans)), _ptr(X))
    if info != 0:
        raise ValueError(f"L[{info - 1}][{info - 1}] is zero or not finite")
    return X


def trsm_adjoint(L, C, Cbar) -> tuple[np.ndarray, np.ndarray]:
    """(L_bar, B_bar) of C = L^-1 B given C and C_bar (oracle.c oracle_trsm_adjoint)."""
    L = _c(L)
    C = _c(C)
    Cbar = _c(Cbar)
    n, m = C.shape
    assert L.shape == (n, n) and Cbar.shape == (n, m)
    Lbar = np.empty_like(L)
    Bbar = np.empty_like(C)
    info = _load().oracle_trsm_adjoint(n, m, _ptr(L), _ptr(C), _ptr(Cbar), _ptr(Lbar), _ptr(Bbar))
    if info != 0:
        raise ValueError(f"L[{info - 1}][{info - 1}] is zero or not finite")
    return Lbar, Bbar


def check_matrix(A, checks: int = 7, tol: float = 1e-8) -> int:
    """Bits: 1 NaN present, 2 not symmetric within tol, 4 zero on the diagonal (oracle.c)."""
    A = _c(A)
    n = A.shape[0]
    assert A.shape == (n, n)
    return int(_load().oracle_check_matrix(n, _ptr(A), int(checks), float(tol)))


def gp_lpdf_grad(x, y, alpha: float, rho: float, sigma: float) -> tuple[float, np.ndarray, np.ndarray]:
    """(lp, [d/d alpha, d/d rho, d/d sigma], d lp/d y) of the zero-mean GP
    regression log density with K = SE(x; alpha, rho) + sigma^2 I (oracle.c)."""
    x = _c(x)
    y = _c(y)
    n = x.shape[0]
    assert y.shape == (n,)
    out = np.empty(4, dtype=np.float64)
    ybar = np.empty(n, dtype=np.float64)
    info = _load().oracle_gp_lpdf_grad(n, _ptr(x), _ptr(y), float(alpha), float(rho), float(sigma),
                                       _ptr(out), _ptr(ybar))
    if info > 0:
        raise NotPositiveDefinite(info)
    if info < 0:
        raise MemoryError("oracle_gp_lpdf_grad: allocation failed")
    return float(out[0]), out[1:].copy(), ybar
