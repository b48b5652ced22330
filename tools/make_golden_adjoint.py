"""Write sampled oracle values of A_bar = cholesky_adjoint(L, L_bar) at large n
into tests/golden/oracle_adj_se_n{n}.npz.

Calls only ``oracle/`` and the seeded generators (never the CUDA path):
    K     = oracle.se_cov(inputs.gp_x(n), 1, 1, 1e-6)
    L     = oracle.cholesky(K)                 (sequential oracle)
    L_bar = inputs.lbar(n)                     (seed 43)
    A_bar = oracle.cholesky_adjoint(L, L_bar)  (sequential oracle)
It also stores the SHA-256 of L's bytes: the GPU test rebuilds the oracle's L
with oracle.cholesky_par (bit-identical, multi-threaded), checks the hash, and
feeds those exact bits to the GPU adjoint (the A_bar bar of 1e-9 is stated for
the same L bits on both sides; a LAPACK L differing by ~1e-11 moves A_bar by
~1e-9 at n = 4096, SURVEY.md §8(c) / DESIGN.md §3).

    python tools/make_golden_adjoint.py 8192 16384

Cost (dev host, one core each): n = 8192 ~7 min, n = 16384 ~1 h.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1907_01063_b200 import inputs  # noqa: E402

ALPHA, RHO, JITTER = 1.0, 1.0, 1e-6


def sample_index(n: int, seed: int = 4321):
    g = np.random.Generator(np.random.PCG64(seed))
    rows = sorted({n - 1, n - 2, n // 2, 1000 % n, int(g.integers(0, n))})
    ri = g.integers(0, n, size=4096)
    rj = g.integers(0, n, size=4096)
    return rows, np.maximum(ri, rj), np.minimum(ri, rj)


def main(ns):
    for n in ns:
        t0 = time.time()
        K = oracle.se_cov(inputs.gp_x(n), ALPHA, RHO, JITTER)
        L = oracle.cholesky(K)
        t_chol = time.time() - t0
        sha = hashlib.sha256(L.tobytes()).hexdigest()
        t1 = time.time()
        Lp = oracle.cholesky_par(K)
        t_par = time.time() - t1
        if hashlib.sha256(Lp.tobytes()).hexdigest() != sha:
            raise SystemExit(f"n={n}: cholesky_par differs from cholesky")
        del Lp, K
        W = inputs.lbar(n)
        t2 = time.time()
        Ab = oracle.cholesky_adjoint(L, W)
        t_adj = time.time() - t2
        rows, ii, jj = sample_index(n)
        out = os.path.join(ROOT, "tests", "golden", f"oracle_adj_se_n{n}.npz")
        np.savez_compressed(out, n=n, alpha=ALPHA, rho=RHO, jitter=JITTER, x_seed=inputs.X_SEED,
                            lbar_seed=inputs.LBAR_SEED, L_sha256=sha,
                            rows=np.array(rows), row_vals=Ab[rows, :], diag=np.diag(Ab).copy(),
                            ii=ii, jj=jj, vals=Ab[ii, jj],
                            oracle_chol_seconds=t_chol, oracle_adj_seconds=t_adj, par_seconds=t_par)
        print(json.dumps({"n": n, "L_sha256": sha, "chol_s": t_chol, "par_s": t_par, "adj_s": t_adj,
                          "out": out}), flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [8192, 16384])
