"""numpy transcriptions of the paper's two blocked listings (test helpers).

These are restatements of PAPER.md's pseudocode in numpy, used only to pin the
oracle against the algorithm the paper prints.  They share nothing with the
oracle (which is the unblocked definition) or with the CUDA path.

* ``blocked_cholesky``   PAPER.md:259-289 (§3.3.1), Louter-Nool recursion:
  L11 = chol(A11); L21 = A21 (L11^T)^-1; recurse on A22 - L21 L21^T.
* ``blocked_adjoint``    PAPER.md:297-323 (§3.3.2), Murray's blocked gradient,
  with DESIGN.md reading R6 for the garbled line 320
  (``D_adj = D_adj.diagonal() * 0.5`` = halve the diagonal in place).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla


def _small_chol(A: np.ndarray) -> np.ndarray:
    # "classic sequential algorithm", PAPER.md:250 (column-oriented here, so it
    # is a different summation order from the oracle's row-oriented loop)
    n = A.shape[0]
    L = np.zeros_like(A)
    for j in range(n):
        s = A[j, j] - np.dot(L[j, :j], L[j, :j])
        if not s > 0:
            raise np.linalg.LinAlgError("not PD")
        L[j, j] = np.sqrt(s)
        for i in range(j + 1, n):
            L[i, j] = (A[i, j] - np.dot(L[i, :j], L[j, :j])) / L[j, j]
    return L


def blocked_cholesky(A: np.ndarray, partition: int = 2, min_l11: int = 4) -> np.ndarray:
    """PAPER.md:259-289, with lower_triangular_inverse(L11) then multiply (line 277)."""
    A = np.array(A, dtype=np.float64, copy=True)
    n = A.shape[0]
    if n == 0:
        return A                                   # line 261-262
    if n <= min_l11:
        return _small_chol(np.tril(A) + np.tril(A, -1).T)   # line 264-266
    block = n // partition                          # line 268
    L11 = blocked_cholesky(A[:block, :block], partition, min_l11)   # 270-271
    A21 = A[block:, :block]
    L11inv = sla.solve_triangular(L11, np.eye(block), lower=True)   # lower_triangular_inverse
    L21 = A21 @ L11inv.T                            # line 277
    A22 = A[block:, block:]
    L22 = A22 - L21 @ L21.T                         # line 282 (multiply_transpose)
    Lrem = blocked_cholesky(L22, partition, min_l11)   # line 284
    out = np.zeros_like(A)
    out[:block, :block] = L11
    out[block:, :block] = L21
    out[block:, block:] = Lrem
    return out


def blocked_adjoint(L: np.ndarray, Lbar: np.ndarray, block_size: int = 128) -> np.ndarray:
    """PAPER.md:298-322 verbatim (working matrix M plays L_adj)."""
    L = np.asarray(L, dtype=np.float64)
    N = L.shape[0]
    M = np.tril(np.asarray(Lbar, dtype=np.float64)).copy()
    k = N
    while k > 0:                                     # for (k = N; k > 0; k -= block_size_)
        j = max(0, k - block_size)
        R = L[j:k, 0:j]
        D = L[j:k, j:k]
        B = L[k:N, 0:j]
        C = L[k:N, j:k]
        Dinv = sla.solve_triangular(D, np.eye(k - j), lower=True)   # lower_triangular_inverse(D)
        C_adj = M[k:N, j:k] @ Dinv                   # line 309
        M[k:N, j:k] = C_adj
        M[k:N, 0:j] = M[k:N, 0:j] - C_adj @ R        # line 310
        D_adj = M[j:k, j:k] - C_adj.T @ C            # line 311
        D_adj = D.T @ D_adj                          # line 313
        D_adj = np.tril(D_adj) + np.tril(D_adj, -1).T   # line 314 copy_lower_tri_to_upper_tri
        Dt = Dinv.T                                  # line 315 D = transpose(lower_triangular_inverse(D))
        D_adj = Dt @ (Dt @ D_adj).T                  # line 316
        D_adj = np.tril(D_adj) + np.tril(D_adj, -1).T   # line 317
        M[j:k, 0:j] = M[j:k, 0:j] - C_adj.T @ B - D_adj @ R   # line 319
        D_adj[np.arange(k - j), np.arange(k - j)] *= 0.5      # line 320 (reading R6)
        M[j:k, j:k] = np.tril(D_adj)                 # line 321 set_zeros_in_upper_tri
        k -= block_size
    return np.tril(M)
