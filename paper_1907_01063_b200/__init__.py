"""paper_1907_01063_b200 -- B200-native FP64 Cholesky + adjoint (arXiv:1907.01063 hot path).

Thin ctypes binding over the C ABI in ``include/stan_cl.h`` (``libstancl.so``,
built in-tree for sm_100a).  This module only marshals arguments: every step of
the path runs in the library's CUDA kernels.  There is no CPU fallback: if the
library is missing or no CUDA device is present, calls raise.

PyTorch is used for device memory and streams only.

    import torch, paper_1907_01063_b200 as sc
    K = sc.gp_exp_quad_cov(x, alpha=1.0, rho=1.0, jitter=1e-6)   # x: cuda float64 [n]
    L = sc.cholesky(K)
    Abar = sc.cholesky_adjoint(L, Lbar)
"""
from __future__ import annotations

import ctypes
import os

import torch

__all__ = [
    "cholesky", "cholesky_adjoint", "gp_exp_quad_cov", "cholesky_async", "cholesky_adjoint_async",
    "cholesky_host", "cholesky_adjoint_host", "kernel_launches", "library_path", "load",
    "StanClError", "NotPositiveDefinite", "STATUS", "workspace_bytes", "finalize", "set_workspace",
    "batched_workspace_bytes",
    "profile_enable", "profile_reset", "profile_read", "PROFILE_KINDS",
]

_PKG = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_PKG, "libstancl.so")
_lib = None

STATUS = {0: "STAN_CL_OK", -1: "STAN_CL_EINVAL", -2: "STAN_CL_ENOMEM", -3: "STAN_CL_ECUDA",
          -4: "STAN_CL_ENCCL"}

# every entry point declared in include/stan_cl.h: (name, restype, argtypes)
_P, _I64, _D, _I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
SIGNATURES = {
    "stan_cl_cholesky": (_I, [_I64, _P, _P]),
    "stan_cl_cholesky_adjoint": (_I, [_I64, _P, _P, _P]),
    "stan_cl_gp_exp_quad_cov": (_I, [_I64, _P, _D, _D, _D, _P]),
    "stan_cl_trsv": (_I, [_I64, _P, _P, _P, _I]),
    "stan_cl_check_matrix": (_I, [_I64, _P, _I, _D]),
    "stan_cl_lower_triangular_inverse": (_I, [_I64, _P, _P]),
    "stan_cl_trsm": (_I, [_I64, _I64, _P, _P, _P, _I]),
    "stan_cl_trsm_adjoint": (_I, [_I64, _I64, _P, _P, _P, _P, _P]),
    "stan_cl_trsm_workspace_bytes": (ctypes.c_size_t, [_I64, _I64]),
    "stan_cl_cholesky_batched": (_I, [_I64, _I64, _P, _P, _P]),
    "stan_cl_cholesky_adjoint_batched": (_I, [_I64, _I64, _P, _P, _P, _P]),
    "stan_cl_gp_lpdf_grad": (_I, [_I64, _P, _P, _D, _D, _D, _P, _P]),
    "stan_cl_cholesky_async": (_I, [_I64, _P, _P, _P]),
    "stan_cl_cholesky_adjoint_async": (_I, [_I64, _P, _P, _P, _P]),
    "stan_cl_cholesky_host": (_I, [_I64, _P, _P]),
    "stan_cl_cholesky_adjoint_host": (_I, [_I64, _P, _P, _P]),
    "stan_cl_set_stream": (_I, [_P]),
    "stan_cl_get_stream": (_P, []),
    "stan_cl_set_block_size": (_I, [_I]),
    "stan_cl_get_block_size": (_I, []),
    "stan_cl_set_adjoint_block_size": (_I, [_I]),
    "stan_cl_workspace_bytes": (ctypes.c_size_t, [_I64]),
    "stan_cl_batched_workspace_bytes": (ctypes.c_size_t, [_I64, _I64, _I]),
    "stan_cl_set_workspace": (_I, [_P, ctypes.c_size_t]),
    "stan_cl_status_string": (ctypes.c_char_p, [_I]),
    "stan_cl_kernel_launches": (ctypes.c_longlong, []),
    "stan_cl_profile_enable": (_I, [_I]),
    "stan_cl_profile_reset": (_I, []),
    "stan_cl_profile_read": (_I, [_I, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                  ctypes.POINTER(ctypes.c_longlong)]),
    "stan_cl_profile_read_bytes": (_I, [_I, ctypes.POINTER(ctypes.c_double)]),
    "stan_cl_trace_enable": (_I, [_I]),
    "stan_cl_trace_read": (_I, [_P, _I]),
    "stan_cl_finalize": (_I, []),
    "stan_cl_dist_get_unique_id": (_I, [_P]),
    "stan_cl_dist_init": (_I, [_I, _I, _P, _I, _I]),
    "stan_cl_dist_cholesky": (_I, [_I64, _I, _P, _I64]),
    "stan_cl_dist_cholesky_adjoint": (_I, [_I64, _I, _P, _P, _I64]),
    "stan_cl_dist_finalize": (_I, []),
    "stan_cl_dist_trace": (_I, [_I64, _I, _I, _I, _I, _I, _P, _P, _I64, _P, _I64]),
    "stan_cl_dist_sim_cholesky": (_I, [_I64, _I, _P, _I64]),
    "stan_cl_gp_exp_quad_cov_cols": (_I, [_I64, _P, _D, _D, _D, _P, _I64, _I, _I]),
    "stan_cl_dist_sim_cholesky_adjoint": (_I, [_I64, _I, _P, _P, _I64]),
    "stan_cl_dist_sim2_cholesky": (_I, [_I64, _I, _I, _P, _I64]),
    "stan_cl_dist_sim2_cholesky_adjoint": (_I, [_I64, _I, _I, _P, _P, _I64]),
    "stan_cl_gp_exp_quad_cov_tiles": (_I, [_I64, _P, _D, _D, _D, _P, _I64, _I, _I, _I, _I]),
    "stan_cl_version": (_I, []),
}


class StanClError(RuntimeError):
    def __init__(self, fn: str, status: int, msg: str):
        super().__init__(f"{fn}: {STATUS.get(status, status)} ({msg})")
        self.status = status


class NotPositiveDefinite(ValueError):
    def __init__(self, info: int):
        super().__init__(f"matrix is not positive definite: first failing pivot at row {info - 1}")
        self.info = info


def library_path() -> str:
    return _LIB_PATH


def load():
    """Load libstancl.so (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} not built; run `python -m paper_1907_01063_b200._build`")
        lib = ctypes.CDLL(_LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _lib = lib
    return _lib


def _check(fn: str, rc: int):
    if rc < 0:
        raise StanClError(fn, rc, load().stan_cl_status_string(rc).decode())
    return rc


def _bind_stream(device: torch.device):
    s = torch.cuda.current_stream(device)
    load().stan_cl_set_stream(ctypes.c_void_p(s.cuda_stream))


def _dev_matrix(t: torch.Tensor, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype != torch.float64:
        raise ValueError(f"{name} must be float64")
    if t.dim() != 2 or t.shape[0] != t.shape[1]:
        raise ValueError(f"{name} must be square")
    return t.contiguous()


def _out(out: torch.Tensor | None, shape: tuple, device: torch.device, name: str = "out",
         dtype: torch.dtype = torch.float64) -> torch.Tensor:
    """A new output tensor, or the caller's one checked: CUDA, dtype, shape, same
    device and contiguous (the library writes a dense row-major block through its
    data pointer, so a strided view is refused rather than silently copied)."""
    if out is None:
        return torch.empty(shape, dtype=dtype, device=device)
    if not isinstance(out, torch.Tensor) or not out.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if out.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}")
    if tuple(out.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(out.shape)}")
    if out.device != device:
        raise ValueError(f"{name} is on {out.device}, the inputs on {device}")
    if not out.is_contiguous():
        raise ValueError(f"{name} must be contiguous (in-place / out= on a strided view is not supported)")
    return out


def cholesky(A: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """L = chol(A) (stan_cl_cholesky).  ``out`` may be ``A`` (in place)."""
    if out is not None and out is A and not A.is_contiguous():
        raise ValueError("in-place cholesky needs a contiguous A")
    A = _dev_matrix(A, "A")
    n = A.shape[0]
    L = _out(out, (n, n), A.device)
    with torch.cuda.device(A.device):
        _bind_stream(A.device)
        rc = _check("stan_cl_cholesky", load().stan_cl_cholesky(n, A.data_ptr(), L.data_ptr()))
    if rc > 0:
        raise NotPositiveDefinite(rc)
    return L


def cholesky_adjoint(L: torch.Tensor, Lbar: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """A_bar = Phi(G + G^T) (stan_cl_cholesky_adjoint).  ``out`` may be ``Lbar``."""
    L = _dev_matrix(L, "L")
    Lbar = _dev_matrix(Lbar, "Lbar")
    n = L.shape[0]
    if Lbar.shape[0] != n:
        raise ValueError("L and Lbar differ in shape")
    if Lbar.device != L.device:
        raise ValueError("L and Lbar are on different devices")
    Abar = _out(out, (n, n), L.device)
    with torch.cuda.device(L.device):
        _bind_stream(L.device)
        rc = _check("stan_cl_cholesky_adjoint",
                    load().stan_cl_cholesky_adjoint(n, L.data_ptr(), Lbar.data_ptr(), Abar.data_ptr()))
    if rc > 0:
        raise ValueError(f"L[{rc - 1}][{rc - 1}] is not finite and > 0")
    return Abar


def gp_exp_quad_cov(x: torch.Tensor, alpha: float = 1.0, rho: float = 1.0, jitter: float = 0.0,
                    out: torch.Tensor | None = None) -> torch.Tensor:
    """K_ij = alpha^2 exp((x_i-x_j)^2 (-0.5/rho^2)) + jitter [i==j] (stan_cl_gp_exp_quad_cov)."""
    if not x.is_cuda or x.dtype != torch.float64 or x.dim() != 1:
        raise ValueError("x must be a 1-D float64 CUDA tensor")
    x = x.contiguous()
    n = x.shape[0]
    K = _out(out, (n, n), x.device)
    with torch.cuda.device(x.device):
        _bind_stream(x.device)
        _check("stan_cl_gp_exp_quad_cov",
               load().stan_cl_gp_exp_quad_cov(n, x.data_ptr(), float(alpha), float(rho), float(jitter),
                                              K.data_ptr()))
    return K


def _dev_vector(t: torch.Tensor, name: str, n: int | None = None) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64 or t.dim() != 1:
        raise ValueError(f"{name} must be a 1-D float64 CUDA tensor")
    if n is not None and t.shape[0] != n:
        raise ValueError(f"{name} must have {n} entries")
    return t.contiguous()


def trsv(L: torch.Tensor, b: torch.Tensor, trans: bool = False, out: torch.Tensor | None = None) -> torch.Tensor:
    """x = L^-1 b (trans=False) or L^-T b (trans=True), L lower with positive
    diagonal (stan_cl_trsv).  ``out`` may be ``b`` (in place)."""
    L = _dev_matrix(L, "L")
    n = L.shape[0]
    b = _dev_vector(b, "b", n)
    if b.device != L.device:
        raise ValueError("L and b are on different devices")
    x = _out(out, (n,), L.device)
    with torch.cuda.device(L.device):
        _bind_stream(L.device)
        rc = _check("stan_cl_trsv", load().stan_cl_trsv(n, L.data_ptr(), b.data_ptr(), x.data_ptr(),
                                                        int(bool(trans))))
    if rc > 0:
        raise ValueError(f"L[{rc - 1}][{rc - 1}] is not finite and > 0")
    return x


def lower_triangular_inverse(L: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """X = L^-1, L lower with positive diagonal (stan_cl_lower_triangular_inverse)."""
    L = _dev_matrix(L, "L")
    n = L.shape[0]
    X = _out(out, (n, n), L.device)
    if X.data_ptr() == L.data_ptr() and n > 0:
        raise ValueError("lower_triangular_inverse is not in place")
    with torch.cuda.device(L.device):
        _bind_stream(L.device)
        rc = _check("stan_cl_lower_triangular_inverse",
                    load().stan_cl_lower_triangular_inverse(n, L.data_ptr(), X.data_ptr()))
    if rc > 0:
        raise ValueError(f"L[{rc - 1}][{rc - 1}] is not finite and > 0")
    return X


CHECK_NAN, CHECK_SYMMETRIC, CHECK_DIAGONAL_ZEROS = 1, 2, 4


def check_matrix(A: torch.Tensor, checks: int = 7, tol: float = 1e-8) -> int:
    """Bits found among 1 (NaN), 2 (not symmetric within tol), 4 (zero diagonal)
    (stan_cl_check_matrix)."""
    A = _dev_matrix(A, "A")
    with torch.cuda.device(A.device):
        _bind_stream(A.device)
        return _check("stan_cl_check_matrix",
                      load().stan_cl_check_matrix(A.shape[0], A.data_ptr(), int(checks), float(tol)))


def _dev_rect(t: torch.Tensor, name: str, n: int) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64 or t.dim() != 2 \
            or t.shape[0] != n:
        raise ValueError(f"{name} must be a ({n}, m) float64 CUDA tensor")
    return t.contiguous()


def trsm(L: torch.Tensor, B: torch.Tensor, trans: bool = False, out: torch.Tensor | None = None) -> torch.Tensor:
    """X = L^-1 B (trans=False) or L^-T B (trans=True), B n x m (stan_cl_trsm).
    ``out`` may be ``B`` (in place)."""
    if out is not None and out is B and not B.is_contiguous():
        raise ValueError("in-place trsm needs a contiguous B")
    L = _dev_matrix(L, "L")
    n = L.shape[0]
    B = _dev_rect(B, "B", n)
    if B.device != L.device:
        raise ValueError("L and B are on different devices")
    X = _out(out, tuple(B.shape), L.device)
    with torch.cuda.device(L.device):
        _bind_stream(L.device)
        rc = _check("stan_cl_trsm", load().stan_cl_trsm(n, B.shape[1], L.data_ptr(), B.data_ptr(), X.data_ptr(),
                                                        int(bool(trans))))
    if rc > 0:
        raise ValueError(f"L[{rc - 1}][{rc - 1}] is not finite and > 0")
    return X


def trsm_adjoint(L: torch.Tensor, C: torch.Tensor, Cbar: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """(L_bar, B_bar) of C = L^-1 B given C and C_bar (stan_cl_trsm_adjoint):
    B_bar = L^-T C_bar, L_bar = tril(-B_bar C^T)."""
    L = _dev_matrix(L, "L")
    n = L.shape[0]
    C = _dev_rect(C, "C", n)
    Cbar = _dev_rect(Cbar, "Cbar", n)
    if C.shape != Cbar.shape or C.device != L.device or Cbar.device != L.device:
        raise ValueError("C and Cbar must match in shape and sit on L's device")
    Lbar = torch.empty_like(L)
    Bbar = torch.empty_like(C)
    with torch.cuda.device(L.device):
        _bind_stream(L.device)
        rc = _check("stan_cl_trsm_adjoint", load().stan_cl_trsm_adjoint(
            n, C.shape[1], L.data_ptr(), C.data_ptr(), Cbar.data_ptr(), Lbar.data_ptr(), Bbar.data_ptr()))
    if rc > 0:
        raise ValueError(f"L[{rc - 1}][{rc - 1}] is not finite and > 0")
    return Lbar, Bbar


def gp_lpdf_grad(x: torch.Tensor, y: torch.Tensor, alpha: float, rho: float, sigma: float,
                 y_bar: bool = True) -> tuple[torch.Tensor, torch.Tensor | None]:
    """Zero-mean GP regression log density and gradient (stan_cl_gp_lpdf_grad):
    returns (out, ybar) with out = [lp, d/d alpha, d/d rho, d/d sigma] (cuda
    float64[4]) and ybar = d lp / d y (or None)."""
    x = _dev_vector(x, "x")
    n = x.shape[0]
    y = _dev_vector(y, "y", n)
    out = torch.empty(4, dtype=torch.float64, device=x.device)
    yb = torch.empty_like(y) if y_bar else None
    with torch.cuda.device(x.device):
        _bind_stream(x.device)
        rc = _check("stan_cl_gp_lpdf_grad", load().stan_cl_gp_lpdf_grad(
            n, x.data_ptr(), y.data_ptr(), float(alpha), float(rho), float(sigma), out.data_ptr(),
            None if yb is None else yb.data_ptr()))
    if rc > 0:
        raise NotPositiveDefinite(rc)
    return out, yb


def _dev_batch(t: torch.Tensor, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64 or t.dim() != 3 \
            or t.shape[1] != t.shape[2]:
        raise ValueError(f"{name} must be a (batch, n, n) float64 CUDA tensor")
    return t.contiguous()


def cholesky_batched(A: torch.Tensor, out: torch.Tensor | None = None) -> tuple[torch.Tensor, torch.Tensor]:
    """L_b = chol(A_b) for a (batch, n, n) tensor, n <= 128 (stan_cl_cholesky_batched).
    Returns (L, info) with info the per-matrix LAPACK code (cuda int32)."""
    A = _dev_batch(A, "A")
    batch, n = A.shape[0], A.shape[1]
    L = _out(out, tuple(A.shape), A.device)
    info = torch.empty(batch, dtype=torch.int32, device=A.device)
    with torch.cuda.device(A.device):
        _bind_stream(A.device)
        _check("stan_cl_cholesky_batched",
               load().stan_cl_cholesky_batched(batch, n, A.data_ptr(), L.data_ptr(), info.data_ptr()))
    return L, info


def cholesky_adjoint_batched(L: torch.Tensor, Lbar: torch.Tensor,
                             out: torch.Tensor | None = None) -> tuple[torch.Tensor, torch.Tensor]:
    """A_bar_b = adjoint(L_b, L_bar_b) for (batch, n, n) tensors, n <= 128
    (stan_cl_cholesky_adjoint_batched).  Returns (A_bar, info)."""
    L = _dev_batch(L, "L")
    Lbar = _dev_batch(Lbar, "Lbar")
    batch, n = L.shape[0], L.shape[1]
    if tuple(Lbar.shape) != tuple(L.shape) or Lbar.device != L.device:
        raise ValueError("L and Lbar differ in shape or device")
    Ab = _out(out, tuple(L.shape), L.device)
    info = torch.empty(batch, dtype=torch.int32, device=L.device)
    with torch.cuda.device(L.device):
        _bind_stream(L.device)
        _check("stan_cl_cholesky_adjoint_batched", load().stan_cl_cholesky_adjoint_batched(
            batch, n, L.data_ptr(), Lbar.data_ptr(), Ab.data_ptr(), info.data_ptr()))
    return Ab, info


def _async_args(mats, info):
    """The async wrappers pass raw pointers: every matrix must already be a square,
    contiguous float64 CUDA tensor of one shape on one device (no copies are made:
    a copy would be freed before the enqueued work reads it)."""
    dev = mats[0][0].device if isinstance(mats[0][0], torch.Tensor) else None
    for t, name in mats:
        if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64 or t.dim() != 2 \
                or t.shape[0] != t.shape[1] or not t.is_contiguous():
            raise ValueError(f"{name} must be a square contiguous float64 CUDA tensor")
        if t.device != dev or t.shape != mats[0][0].shape:
            raise ValueError(f"{name} differs in shape or device from {mats[0][1]}")
    if info is not None and (not isinstance(info, torch.Tensor) or not info.is_cuda or info.dtype != torch.int32
                             or info.numel() < 1 or info.device != dev):
        raise ValueError("info must be a cuda int32 tensor with >= 1 element on the inputs' device")


def cholesky_async(A: torch.Tensor, L: torch.Tensor, info: torch.Tensor | None = None) -> None:
    """Enqueue L = chol(A) without synchronising; ``info`` (cuda int32[1]) gets the status."""
    _async_args([(A, "A"), (L, "L")], info)
    n = A.shape[0]
    with torch.cuda.device(A.device):
        _bind_stream(A.device)
        _check("stan_cl_cholesky_async", load().stan_cl_cholesky_async(
            n, A.data_ptr(), L.data_ptr(), None if info is None else info.data_ptr()))


def cholesky_adjoint_async(L: torch.Tensor, Lbar: torch.Tensor, Abar: torch.Tensor,
                           info: torch.Tensor | None = None) -> None:
    _async_args([(L, "L"), (Lbar, "Lbar"), (Abar, "Abar")], info)
    n = L.shape[0]
    with torch.cuda.device(L.device):
        _bind_stream(L.device)
        _check("stan_cl_cholesky_adjoint_async", load().stan_cl_cholesky_adjoint_async(
            n, L.data_ptr(), Lbar.data_ptr(), Abar.data_ptr(), None if info is None else info.data_ptr()))


def _host_matrix(t: torch.Tensor, name: str) -> torch.Tensor:
    if t.is_cuda or t.dtype != torch.float64 or t.dim() != 2 or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous float64 CPU tensor")
    return t


def cholesky_host(A: torch.Tensor, L: torch.Tensor, device: int = 0) -> int:
    """Host buffers in, host buffer out (stan_cl_cholesky_host); returns info."""
    _host_matrix(A, "A")
    _host_matrix(L, "L")
    dev = torch.device("cuda", device)
    with torch.cuda.device(dev):
        _bind_stream(dev)
        return _check("stan_cl_cholesky_host", load().stan_cl_cholesky_host(A.shape[0], A.data_ptr(), L.data_ptr()))


def cholesky_adjoint_host(L: torch.Tensor, Lbar: torch.Tensor, Abar: torch.Tensor, device: int = 0) -> int:
    for t, nm in ((L, "L"), (Lbar, "Lbar"), (Abar, "Abar")):
        _host_matrix(t, nm)
    dev = torch.device("cuda", device)
    with torch.cuda.device(dev):
        _bind_stream(dev)
        return _check("stan_cl_cholesky_adjoint_host", load().stan_cl_cholesky_adjoint_host(
            L.shape[0], L.data_ptr(), Lbar.data_ptr(), Abar.data_ptr()))


# ------------------------------------------------------------------ multi-GPU
DIST_BLOCK = 256


def dist_owned_blocks(n: int, G: int, q: int) -> int:
    """Block indices I < n/256 with I % G == q (local block rows / columns of a grid index)."""
    T = n // DIST_BLOCK
    return (T - q + G - 1) // G if q < T else 0


def dist_grid(G: int) -> tuple[int, int]:
    """Default P x Q process grid for G ranks: 1x1, 1x2, 2x2, 2x4, ...
    P <= Q, P the largest divisor of G with P*P <= G."""
    P = max(d for d in range(1, int(G ** 0.5) + 1) if G % d == 0)
    return P, G // P


def dist_local_shape(n: int, P: int, Q: int, p: int, q: int) -> tuple[int, int]:
    """(rows, cols) of rank (p, q)'s local array: tiles (I, J), I % P == p, J % Q == q."""
    return dist_owned_blocks(n, P, p) * DIST_BLOCK, dist_owned_blocks(n, Q, q) * DIST_BLOCK


def _tiles(n: int, G: int, g: int) -> list:
    return list(range(g, n // DIST_BLOCK, G))


def dist_scatter2(A: torch.Tensor, P: int, Q: int, p: int, q: int, width: int | None = None) -> torch.Tensor:
    """Rank (p, q)'s local array of the 2-D block-cyclic layout (contiguous; optional
    zero-padded width = leading dimension)."""
    n = A.shape[0]
    rows, cols = dist_local_shape(n, P, Q, p, q)
    out = A.new_zeros((rows, width if width is not None else cols))
    B = DIST_BLOCK
    for li, I in enumerate(_tiles(n, P, p)):
        for lj, J in enumerate(_tiles(n, Q, q)):
            out[li * B:(li + 1) * B, lj * B:(lj + 1) * B] = A[I * B:(I + 1) * B, J * B:(J + 1) * B]
    return out


def dist_gather2(locals_: list, n: int, P: int, Q: int) -> torch.Tensor:
    """Inverse of dist_scatter2 over all P*Q ranks (locals_[p*Q + q])."""
    B = DIST_BLOCK
    out = locals_[0].new_zeros((n, n))
    for r, loc in enumerate(locals_):
        p, q = divmod(r, Q)
        for li, I in enumerate(_tiles(n, P, p)):
            for lj, J in enumerate(_tiles(n, Q, q)):
                out[I * B:(I + 1) * B, J * B:(J + 1) * B] = loc[li * B:(li + 1) * B, lj * B:(lj + 1) * B]
    return out


def dist_scatter(A: torch.Tensor, G: int, q: int) -> torch.Tensor:
    """Rank q's local array of the 1 x G grid (block columns J = q, q+G, ... of A)."""
    return dist_scatter2(A, 1, G, 0, q)


def dist_gather(locals_: list, n: int) -> torch.Tensor:
    """Inverse of dist_scatter over all ranks."""
    return dist_gather2(locals_, n, 1, len(locals_))


def _ptr_array(ts):
    arr = (ctypes.c_void_p * len(ts))(*[t.data_ptr() for t in ts])
    return arr


def _sim_ld(ts) -> int:
    ld = ts[0].stride(0)
    assert all(t.stride(0) == ld and t.stride(1) == 1 for t in ts), "equal leading dimensions, row-major"
    return ld


def dist_sim2_cholesky(A_locals: list, n: int, P: int, Q: int) -> int:
    """Distributed forward on a P x Q grid simulated on this device (A_locals[p*Q + q], in place)."""
    assert len(A_locals) == P * Q
    ld = _sim_ld(A_locals)
    with torch.cuda.device(A_locals[0].device):
        _bind_stream(A_locals[0].device)
        return _check("stan_cl_dist_sim2_cholesky", load().stan_cl_dist_sim2_cholesky(
            n, P, Q, ctypes.cast(_ptr_array(A_locals), ctypes.c_void_p), ld))


def dist_sim2_cholesky_adjoint(L_locals: list, W_locals: list, n: int, P: int, Q: int) -> int:
    assert len(L_locals) == len(W_locals) == P * Q
    ld = _sim_ld(list(L_locals) + list(W_locals))
    with torch.cuda.device(L_locals[0].device):
        _bind_stream(L_locals[0].device)
        return _check("stan_cl_dist_sim2_cholesky_adjoint", load().stan_cl_dist_sim2_cholesky_adjoint(
            n, P, Q, ctypes.cast(_ptr_array(L_locals), ctypes.c_void_p),
            ctypes.cast(_ptr_array(W_locals), ctypes.c_void_p), ld))


def dist_sim_cholesky(A_locals: list, n: int) -> int:
    """Distributed forward with len(A_locals) simulated ranks (1 x G grid) on this device."""
    return dist_sim2_cholesky(A_locals, n, 1, len(A_locals))


def dist_sim_cholesky_adjoint(L_locals: list, W_locals: list, n: int) -> int:
    return dist_sim2_cholesky_adjoint(L_locals, W_locals, n, 1, len(L_locals))


def dist_init_from_torch(group=None, P: int | None = None, Q: int | None = None) -> tuple[int, int]:
    """NCCL communicators for the library from an initialised torch.distributed group:
    rank 0 creates the id, torch ships it, every rank joins the P x Q grid
    (default dist_grid(world)); returns (P, Q).  Rank r is grid position (r // Q, r % Q)."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if P is None or Q is None:
        P, Q = dist_grid(world)
    try:
        import nvidia.nccl
        libdir = os.path.join(list(nvidia.nccl.__path__)[0], "lib", "libnccl.so.2")
        os.environ.setdefault("STAN_CL_NCCL_LIB", libdir)
    except Exception:
        pass
    buf = (ctypes.c_char * 128)()
    if rank == 0:
        _check("stan_cl_dist_get_unique_id", load().stan_cl_dist_get_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
    obj = [bytes(buf)]
    dist.broadcast_object_list(obj, src=0, group=group)
    idb = (ctypes.c_char * 128).from_buffer_copy(obj[0])
    _check("stan_cl_dist_init", load().stan_cl_dist_init(world, rank, ctypes.cast(idb, ctypes.c_void_p), P, Q))
    return P, Q


def gp_exp_quad_cov_tiles(x: torch.Tensor, K_local: torch.Tensor, P: int, Q: int, p: int, q: int,
                          alpha: float = 1.0, rho: float = 1.0, jitter: float = 0.0) -> torch.Tensor:
    """Rank (p, q)'s tiles of the SE covariance (2-D block-cyclic), into K_local (rows x ld)."""
    n = x.shape[0]
    with torch.cuda.device(x.device):
        _bind_stream(x.device)
        _check("stan_cl_gp_exp_quad_cov_tiles", load().stan_cl_gp_exp_quad_cov_tiles(
            n, x.data_ptr(), float(alpha), float(rho), float(jitter), K_local.data_ptr(), K_local.stride(0),
            P, Q, p, q))
    return K_local


def gp_exp_quad_cov_cols(x: torch.Tensor, K_local: torch.Tensor, G: int, q: int, alpha: float = 1.0,
                         rho: float = 1.0, jitter: float = 0.0) -> torch.Tensor:
    """Rank q's owned block columns of the SE covariance (1 x G grid), into K_local (n x ld)."""
    return gp_exp_quad_cov_tiles(x, K_local, 1, G, 0, q, alpha, rho, jitter)


def dist_cholesky(A_local: torch.Tensor, n: int) -> int:
    with torch.cuda.device(A_local.device):
        _bind_stream(A_local.device)
        return _check("stan_cl_dist_cholesky",
                      load().stan_cl_dist_cholesky(n, 0, A_local.data_ptr(), A_local.stride(0)))


def dist_cholesky_adjoint(L_local: torch.Tensor, W_local: torch.Tensor, n: int) -> int:
    assert L_local.stride(0) == W_local.stride(0), "L_local and W_local share the leading dimension"
    with torch.cuda.device(L_local.device):
        _bind_stream(L_local.device)
        return _check("stan_cl_dist_cholesky_adjoint", load().stan_cl_dist_cholesky_adjoint(
            n, 0, L_local.data_ptr(), W_local.data_ptr(), L_local.stride(0)))


def dist_trace(n: int, P: int, Q: int, p: int, q: int, adjoint: bool, A_local: torch.Tensor,
               L_local: torch.Tensor | None = None) -> list:
    """The NCCL calls rank (p, q) would issue, in order (stan_cl_dist_trace):
    [(comm_kind, comm_index, op, root, count, stream), ...]."""
    cap = 1 << 16
    buf = (ctypes.c_int64 * (6 * cap))()
    with torch.cuda.device(A_local.device):
        _bind_stream(A_local.device)
        m = _check("stan_cl_dist_trace", load().stan_cl_dist_trace(
            n, P, Q, p, q, int(bool(adjoint)), None if L_local is None else L_local.data_ptr(),
            A_local.data_ptr(), A_local.stride(0), ctypes.cast(buf, ctypes.c_void_p), cap))
    assert m <= cap
    return [tuple(buf[6 * i:6 * i + 6]) for i in range(m)]


def kernel_launches() -> int:
    return int(load().stan_cl_kernel_launches())


PROFILE_KINDS = ["syrk", "adj_gemm", "splitk", "potrf", "trsm", "tri_inverse", "gemm128", "se_cov", "other",
                 "lookahead", "trmm", "gp"]


def profile_enable(on: bool = True, kinds=None) -> None:
    """Record CUDA events around every launch (kinds=None) or only those classes."""
    if not on:
        load().stan_cl_profile_enable(0)
    elif kinds is None:
        load().stan_cl_profile_enable(1)
    else:
        mask = 0
        for k in kinds:
            mask |= 1 << PROFILE_KINDS.index(k)
        load().stan_cl_profile_enable(mask << 1)


def profile_reset() -> None:
    load().stan_cl_profile_reset()


def profile_read() -> dict:
    """{class: {"ms": summed event ms, "flops": algorithmic flops, "bytes": algorithmic
    HBM bytes, "launches": n}}"""
    out = {}
    for k, name in enumerate(PROFILE_KINDS):
        ms, fl, cnt, by = ctypes.c_double(), ctypes.c_double(), ctypes.c_longlong(), ctypes.c_double()
        load().stan_cl_profile_read(k, ctypes.byref(ms), ctypes.byref(fl), ctypes.byref(cnt))
        load().stan_cl_profile_read_bytes(k, ctypes.byref(by))
        out[name] = {"ms": ms.value, "flops": fl.value, "bytes": by.value, "launches": cnt.value}
    return out


def trace(on: bool = True) -> None:
    """Start (base event on the current stream) / stop the launch timeline."""
    _bind_stream(torch.device("cuda", torch.cuda.current_device()))
    load().stan_cl_trace_enable(int(bool(on)))


def trace_read() -> list:
    """[(class name, stream id, start ms, end ms), ...] of the traced launches."""
    n = int(load().stan_cl_trace_read(None, 0))
    buf = (ctypes.c_double * (4 * max(n, 1)))()
    n = int(load().stan_cl_trace_read(ctypes.cast(buf, ctypes.c_void_p), n))
    return [(PROFILE_KINDS[int(buf[4 * i])], int(buf[4 * i + 1]), buf[4 * i + 2], buf[4 * i + 3]) for i in range(n)]


def workspace_bytes(n: int) -> int:
    """Caller workspace that suffices for every single-matrix call at order n."""
    return int(load().stan_cl_workspace_bytes(n))


def batched_workspace_bytes(batch: int, n: int, with_info: bool = True) -> int:
    return int(load().stan_cl_batched_workspace_bytes(batch, n, int(bool(with_info))))


def set_workspace(buf: torch.Tensor | None) -> None:
    """Hand the library a caller-owned device buffer (stan_cl_set_workspace): every
    later call carves its device memory from it (None: back to library-owned).
    The tensor must stay alive until set_workspace(None) / finalize()."""
    if buf is None:
        _check("stan_cl_set_workspace", load().stan_cl_set_workspace(None, 0))
        return
    if not isinstance(buf, torch.Tensor) or not buf.is_cuda or not buf.is_contiguous():
        raise ValueError("workspace must be a contiguous CUDA tensor")
    with torch.cuda.device(buf.device):
        _check("stan_cl_set_workspace",
               load().stan_cl_set_workspace(buf.data_ptr(), buf.numel() * buf.element_size()))


def finalize() -> None:
    load().stan_cl_finalize()
