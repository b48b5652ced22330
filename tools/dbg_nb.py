import sys, os, numpy as np, torch
sys.path.insert(0,'.')
import oracle, paper_1907_01063_b200 as sc
from paper_1907_01063_b200 import inputs
n = int(sys.argv[1])
g = np.load(f'tests/golden/oracle_chol_se_n{n}.npz')
K = oracle.se_cov(inputs.gp_x(n), 1.0, 1.0, 1e-6)
Kd = torch.from_numpy(K).cuda()
want = np.concatenate([g['row_vals'].ravel(), g['vals'], g['diag']])
res = []
for nb in [256, 128, 256, 256]:
    sc.load().stan_cl_set_block_size(nb)
    L = sc.cholesky(Kd)
    got = np.concatenate([L[torch.from_numpy(g['rows']).cuda()].cpu().numpy().ravel(), L[torch.from_numpy(g['ii']).cuda(), torch.from_numpy(g['jj']).cuda()].cpu().numpy(), torch.diagonal(L).cpu().numpy()])
    res.append(L.cpu())
    print(os.environ.get('TAG',''), n, nb, np.linalg.norm(got-want)/np.linalg.norm(want), flush=True)
print('256 runs identical:', torch.equal(res[0], res[2]), torch.equal(res[2], res[3]))
