"""Small invocations of every kernel added or changed in round 2, for
compute-sanitizer (memcheck / racecheck / synccheck):
    compute-sanitizer --tool racecheck python tools/sanitize_r2.py
w32 / w64 register kernels (single and batched), the blocked tri_inverse, the
fused R0 + reduce (in place and out of place), the two-stream pipelined sweep
(n <= 2048) and the merged single-stream sweep (n > 2048, one run at 2304),
the caller-owned workspace path, the NEXT-2 triangular primitives."""
from __future__ import annotations

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1907_01063_b200 as sc  # noqa: E402
from paper_1907_01063_b200 import inputs  # noqa: E402


def se(n):
    x = torch.from_numpy(inputs.gp_x(n)).cuda()
    return sc.gp_exp_quad_cov(x, 1.0, 1.0, 1e-6)


def main():
    sc.load()
    for n in (20, 48, 64, 300, 1024, 2304):
        K = se(n)
        L = sc.cholesky(K)
        W = torch.from_numpy(inputs.lbar(n)).cuda()
        A = sc.cholesky_adjoint(L, W)                 # out of place (fused R0 reads L_bar)
        sc.cholesky_adjoint(L, W, out=W)              # in place
        assert torch.allclose(A, W, rtol=0, atol=0) or n <= 64
        sc.cholesky(K, out=K)                         # in place (off-diagonal upper zeroing)
    for n in (48, 64):
        A = torch.stack([se(n) for _ in range(5)])
        Lb, info = sc.cholesky_batched(A)
        Wb = torch.stack([torch.from_numpy(inputs.lbar(n, seed=s)).cuda() for s in range(5)])
        sc.cholesky_adjoint_batched(Lb, Wb)
    n, m = 1000, 70
    L = sc.cholesky(se(n))
    sc.lower_triangular_inverse(L)
    B = torch.randn((n, m), dtype=torch.float64, device="cuda")
    C = sc.trsm(L, B)
    sc.trsm(L, B, True)
    sc.trsm_adjoint(L, C, B)
    buf = torch.empty(sc.workspace_bytes(300) // 8 + 1, dtype=torch.float64, device="cuda")
    sc.set_workspace(buf)
    K = se(300)
    L = sc.cholesky(K)
    sc.cholesky_adjoint(L, torch.from_numpy(inputs.lbar(300)).cuda())
    sc.set_workspace(None)
    torch.cuda.synchronize()
    print("sanitize_r2 ok")


if __name__ == "__main__":
    main()
