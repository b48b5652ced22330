python -m pytest tests/test_gpu_fullsize.py -x -q -k "sampled_oracle" 2>&1 | grep -E "assert|Error|passed|failed" | head
python - <<'PY'
import sys, numpy as np, torch
sys.path.insert(0,'.')
import oracle, paper_1907_01063_b200 as sc
from paper_1907_01063_b200 import inputs
for n in (8192, 16384):
    g = np.load(f'tests/golden/oracle_chol_se_n{n}.npz')
    K = oracle.se_cov(inputs.gp_x(n), 1.0, 1.0, 1e-6)
    Kd = torch.from_numpy(K).cuda()
    for nb in (128, 256):
        sc.load().stan_cl_set_block_size(nb)
        L = sc.cholesky(Kd)
        rows = g['rows']; got = np.concatenate([L[torch.from_numpy(rows).cuda()].cpu().numpy().ravel(), L[torch.from_numpy(g['ii']).cuda(), torch.from_numpy(g['jj']).cuda()].cpu().numpy(), torch.diagonal(L).cpu().numpy()])
        want = np.concatenate([g['row_vals'].ravel(), g['vals'], g['diag']])
        print(n, nb, np.linalg.norm(got-want)/np.linalg.norm(want), flush=True)
PY
