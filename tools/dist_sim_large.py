"""The 2-D block-cyclic multi-GPU schedule at the sharded size on ONE device
(BASELINE.json configs[4] is n = 65536 over 2/4/8 B200s; this box has one):
all P x Q ranks simulated in one process (stan_cl_dist_sim2_*: broadcasts
become device copies, the column reduce fixed-order additions -- the same
host schedule, kernels and buffers as the NCCL path).

  1. integer-exact forward: unit-lower +-1 L0 (on the device), A = L0 L0^T
     (exact), scattered over the grid; the distributed factor must return L0
     bit for bit (the oracle-free pin at n = 65536);
  2. integer-exact adjoint: banded (2) unit-lower L, integer L_bar; compared
     bit for bit with the single-GPU adjoint (every correct blocking returns
     the same bits for this family);
  3. SE forward + adjoint timing (x ~ U(-10, 10), jitter 1e-6; L_bar ~ N(0,1)).
    python tools/dist_sim_large.py [n] [P] [Q] > profiles/r02_dist_sim_65536.jsonl
"""
from __future__ import annotations

import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1907_01063_b200 as sc  # noqa: E402
from paper_1907_01063_b200 import inputs  # noqa: E402


def unit_lower_pm1_dev(n, seed, band=None):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    L = torch.randint(-1, 2, (n, n), generator=g, device="cuda", dtype=torch.int8).to(torch.float64)
    L.tril_(-1)
    if band is not None:
        L.triu_(-band)
    L.diagonal().fill_(1.0)
    return L


def scatter_all(A, n, P, Q):
    width = max(sc.dist_local_shape(n, P, Q, 0, q)[1] for q in range(Q))
    return [sc.dist_scatter2(A, P, Q, r // Q, r % Q, width).contiguous() for r in range(P * Q)]


def timed(fn):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    rc = fn()
    b.record()
    torch.cuda.synchronize()
    return rc, a.elapsed_time(b)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
    P = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    Q = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    sc.load()
    base = {"n": n, "grid": f"{P}x{Q}", "ranks_simulated_on_one_gpu": P * Q}
    # 1. integer-exact forward
    t0 = time.time()
    L0 = unit_lower_pm1_dev(n, seed=n)
    A = L0 @ L0.T                                   # integers, |partial sums| <= n: exact
    locs = scatter_all(A, n, P, Q)
    del A
    torch.cuda.empty_cache()
    rc, ms = timed(lambda: sc.dist_sim2_cholesky(locs, n, P, Q))
    got = sc.dist_gather2(locs, n, P, Q)
    del locs
    torch.cuda.empty_cache()
    exact = bool(torch.equal(torch.tril(got), L0))
    diag_up_zero = all(bool(torch.all(torch.triu(got[i:i + 256, i:i + 256], 1) == 0)) for i in range(0, n, 256))
    del got, L0
    torch.cuda.empty_cache()
    print(json.dumps({**base, "test": "integer-exact forward (unit-lower +-1, dense)", "status": rc,
                      "bit_exact": exact, "diag_tile_upper_zero": diag_up_zero, "ms": ms,
                      "wall_s": time.time() - t0}), flush=True)
    # 2. integer-exact adjoint vs the single-GPU adjoint (bit for bit)
    t0 = time.time()
    Li = unit_lower_pm1_dev(n, seed=3, band=2)
    g = torch.Generator(device="cuda")
    g.manual_seed(4)
    Wi = torch.randint(-3, 4, (n, n), generator=g, device="cuda", dtype=torch.int8).to(torch.float64).tril_()
    Ls, Ws = scatter_all(Li, n, P, Q), scatter_all(Wi, n, P, Q)
    rc, ms = timed(lambda: sc.dist_sim2_cholesky_adjoint(Ls, Ws, n, P, Q))
    del Ls
    got = sc.dist_gather2(Ws, n, P, Q)
    del Ws
    torch.cuda.empty_cache()
    sc.cholesky_adjoint(Li, Wi, out=Wi)             # single-GPU path, in place
    exact = bool(torch.equal(torch.tril(got), Wi))
    mx = float(Wi.abs().max())
    del got, Li, Wi
    torch.cuda.empty_cache()
    print(json.dumps({**base, "test": "integer-exact adjoint (band 2) vs single-GPU adjoint", "status": rc,
                      "bit_exact": exact, "max_abs": mx, "ms": ms, "wall_s": time.time() - t0}), flush=True)
    # 3. SE timing
    x = torch.from_numpy(inputs.gp_x(n)).cuda()
    width = max(sc.dist_local_shape(n, P, Q, 0, q)[1] for q in range(Q))
    Ks, Wb = [], []
    for r in range(P * Q):
        p, q = divmod(r, Q)
        rows, _ = sc.dist_local_shape(n, P, Q, p, q)
        K = torch.empty((rows, width), dtype=torch.float64, device="cuda")
        sc.gp_exp_quad_cov_tiles(x, K, P, Q, p, q, 1.0, 1.0, 1e-6)
        Ks.append(K)
        gg = torch.Generator(device="cuda")
        gg.manual_seed(inputs.LBAR_SEED + r)
        Wb.append(torch.randn((rows, width), dtype=torch.float64, device="cuda", generator=gg))
    rcf, msf = timed(lambda: sc.dist_sim2_cholesky(Ks, n, P, Q))
    rca, msa = timed(lambda: sc.dist_sim2_cholesky_adjoint(Ks, Wb, n, P, Q))
    fl = float(n) ** 3
    print(json.dumps({**base, "test": "SE forward + adjoint (timing)", "status": [rcf, rca],
                      "fwd_ms": msf, "adj_ms": msa, "tflops": fl / ((msf + msa) / 1e3) / 1e12,
                      "note": "all ranks' work serialised on one GPU: a correctness / scale run of the multi-GPU "
                              "schedule, not a scaling number"}), flush=True)


if __name__ == "__main__":
    main()
