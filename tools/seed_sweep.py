"""L error vs the oracle over 24 SE seeds (GPU run): python tools/seed_sweep.py > profiles/r02_seed_sweep.txt."""
import sys, torch, numpy as np
sys.path.insert(0, '.')
import oracle, paper_1907_01063_b200 as sc
from paper_1907_01063_b200 import inputs
worst = {}
for n in (300, 1024, 2048):
    errs = []
    for seed in range(100, 124):
        K = oracle.se_cov(inputs.gp_x(n, seed), 1.0, 1.0, 1e-6)
        Lo = oracle.cholesky(K) if n <= 1024 else oracle.cholesky_par(K)
        Lg = sc.cholesky(torch.from_numpy(K).cuda()).cpu().numpy()
        lo = np.tril_indices(n)
        errs.append(float(np.linalg.norm(Lg[lo] - Lo[lo]) / np.linalg.norm(Lo[lo])))
    print(n, "max %.2e  median %.2e" % (max(errs), float(np.median(errs))), flush=True)
