"""NEXT-4 measurement: batched small Cholesky + adjoint (n <= 128) on one GPU,
CUDA events, device-resident inputs.  Context: torch.linalg.cholesky on the
same batch (cuSOLVER batched) and its autograd backward.  One JSON line per
(batch, n)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1907_01063_b200 as sc  # noqa: E402
from paper_1907_01063_b200 import inputs  # noqa: E402


def ev_ms(fn, reps=7):
    fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


cases = [(4096, 32), (4096, 64), (4096, 128), (16384, 128)]
for batch, n in cases:
    x = torch.from_numpy(np.stack([inputs.gp_x(n, 1000 + b) for b in range(min(batch, 64))])).cuda()
    x = x.repeat((batch + 63) // 64, 1)[:batch]
    d = x[:, :, None] - x[:, None, :]
    A = torch.exp(-0.5 * d * d) + 1e-6 * torch.eye(n, dtype=torch.float64, device="cuda")
    del d
    W = torch.from_numpy(inputs.lbar(n)).cuda().expand(batch, n, n).contiguous()
    L, _ = sc.cholesky_batched(A)
    out = torch.empty_like(A)
    f_ms = ev_ms(lambda: sc.cholesky_batched(A, out=out))
    a_ms = ev_ms(lambda: sc.cholesky_adjoint_batched(L, W, out=out))
    t_f = ev_ms(lambda: torch.linalg.cholesky(A))

    def torch_bwd():
        Ar = A.clone().requires_grad_(True)
        Lr = torch.linalg.cholesky(Ar)
        torch.autograd.grad(Lr, Ar, grad_outputs=W)
    t_fb = ev_ms(torch_bwd, reps=3)
    fl = batch * n ** 3
    print(json.dumps({"batch": batch, "n": n, "fwd_ms": f_ms, "adj_ms": a_ms,
                      "matrices_per_s": batch / ((f_ms + a_ms) / 1e3),
                      "gflops_n3": fl / ((f_ms + a_ms) / 1e3) / 1e9,
                      "torch_cholesky_ms": t_f, "torch_fwd_plus_bwd_ms": t_fb}), flush=True)
