"""Write sampled oracle values of L = chol(K) at large n into tests/golden/.

Calls only ``oracle/`` and the seeded generators (never the CUDA path).  The
GPU parity test at full size rebuilds the same K with the oracle's SE builder,
factors it on the GPU and compares the sampled entries.

    python tools/make_golden_large.py 8192 16384

Cost: single-threaded oracle, ~2.5 min at n=8192 and ~20 min at n=16384 on the
dev host (SURVEY.md §0 finding 4).
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1907_01063_b200 import inputs  # noqa: E402

ALPHA, RHO, JITTER = 1.0, 1.0, 1e-6


def sample_index(n: int, seed: int = 1234):
    g = np.random.Generator(np.random.PCG64(seed))
    rows = sorted({n - 1, n - 2, n // 2, int(g.integers(0, n)), int(g.integers(0, n))})
    ri = g.integers(0, n, size=4096)
    rj = g.integers(0, n, size=4096)
    ii = np.maximum(ri, rj)
    jj = np.minimum(ri, rj)
    return rows, ii, jj


def main(ns):
    for n in ns:
        t0 = time.time()
        K = oracle.se_cov(inputs.gp_x(n), ALPHA, RHO, JITTER)
        L = oracle.cholesky(K)
        dt = time.time() - t0
        rows, ii, jj = sample_index(n)
        out = os.path.join(ROOT, "tests", "golden", f"oracle_chol_se_n{n}.npz")
        np.savez_compressed(out, n=n, alpha=ALPHA, rho=RHO, jitter=JITTER, x_seed=inputs.X_SEED,
                            rows=np.array(rows), row_vals=L[rows, :], diag=np.diag(L).copy(),
                            ii=ii, jj=jj, vals=L[ii, jj], oracle_seconds=dt)
        print(f"n={n}: oracle {dt:.1f} s -> {out}", flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [8192, 16384])
