"""Measured parity margins of the CUDA path against the oracle (GPU run).

    python tools/parity_margins.py > profiles/r02_parity_margins.jsonl

For each n: relative Frobenius error of L = chol(K) (GPU fed the oracle's K) and
of A_bar (GPU fed the oracle's L and L_bar = inputs.lbar(n)), against the
BASELINE.json bars 1e-11 and 1e-9.  n <= 4096: full matrices (oracle L by the
bit-identical oracle.cholesky_par, oracle A_bar by the sequential oracle);
n = 8192 / 16384: the committed oracle samples in tests/golden/ (the oracle
adjoint takes ~1 h at 16384).  Test infrastructure: reads oracle/ only.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_1907_01063_b200 as sc  # noqa: E402
from paper_1907_01063_b200 import inputs  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")


def relf(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def main():
    sc.load()
    for n in (1024, 2048, 4096, 8192, 16384):
        t0 = time.time()
        K = oracle.se_cov(inputs.gp_x(n), 1.0, 1.0, 1e-6)
        Lo = oracle.cholesky_par(K)
        Lg = sc.cholesky(torch.from_numpy(K).cuda())
        rec = {"n": n, "L_bar": 1e-11, "A_bar_bar": 1e-9}
        W = inputs.lbar(n)
        if n <= 4096:
            rec["L_rel_frobenius"] = relf(np.tril(Lg.cpu().numpy()), Lo)
            rec["L_kind"] = "full matrix"
            Ao = oracle.cholesky_adjoint(Lo, W)
            Ag = sc.cholesky_adjoint(torch.from_numpy(Lo).cuda(), torch.from_numpy(W).cuda()).cpu().numpy()
            rec["A_bar_rel_frobenius"] = relf(Ag, Ao)
            rec["A_bar_kind"] = "full matrix"
        else:
            g = np.load(os.path.join(GOLD, f"oracle_chol_se_n{n}.npz"))
            Lc = Lg.cpu().numpy()
            got = np.concatenate([Lc[g["rows"]].ravel(), Lc[g["ii"], g["jj"]], np.diag(Lc)])
            want = np.concatenate([g["row_vals"].ravel(), g["vals"], g["diag"]])
            rec["L_rel_frobenius"] = relf(got, want)
            rec["L_kind"] = f"sampled: {len(g['rows'])} full rows + {len(g['ii'])} entries + diagonal"
            del Lc
            ga_path = os.path.join(GOLD, f"oracle_adj_se_n{n}.npz")
            if os.path.exists(ga_path):
                ga = np.load(ga_path)
                assert hashlib.sha256(Lo.tobytes()).hexdigest() == str(ga["L_sha256"])
                Ag = sc.cholesky_adjoint(torch.from_numpy(Lo).cuda(), torch.from_numpy(W).cuda()).cpu().numpy()
                got = np.concatenate([Ag[ga["rows"]].ravel(), Ag[ga["ii"], ga["jj"]], np.diag(Ag)])
                want = np.concatenate([ga["row_vals"].ravel(), ga["vals"], ga["diag"]])
                rec["A_bar_rel_frobenius"] = relf(got, want)
                rec["A_bar_kind"] = f"sampled: {len(ga['rows'])} full rows + {len(ga['ii'])} entries + diagonal"
                del Ag
        rec["L_margin"] = rec["L_bar"] / rec["L_rel_frobenius"]
        if "A_bar_rel_frobenius" in rec:
            rec["A_bar_margin"] = rec["A_bar_bar"] / rec["A_bar_rel_frobenius"]
        rec["seconds"] = time.time() - t0
        print(json.dumps(rec), flush=True)
        del Lg
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
