"""Per-class event profile: single-GPU forward vs the distributed forward on a 1 x 1 grid (dev tool)."""
import sys, json
import torch
sys.path.insert(0, '.')
import paper_1907_01063_b200 as sc
from paper_1907_01063_b200 import inputs
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
x = torch.from_numpy(inputs.gp_x(n)).cuda()
K = sc.gp_exp_quad_cov(x, 1.0, 1.0, 1e-6)
L = torch.empty_like(K)
Kd = torch.empty_like(K)
for name, fn in [("single", lambda: sc.cholesky(K, out=L)),
                 ("dist11", lambda: (Kd.copy_(K), sc.dist_sim2_cholesky([Kd], n, 1, 1)))]:
    fn(); torch.cuda.synchronize()
    sc.profile_reset(); sc.profile_enable(True)
    fn(); torch.cuda.synchronize()
    sc.profile_enable(False)
    prof = sc.profile_read()
    print(name, json.dumps({k: [round(v["ms"], 2), v["launches"]] for k, v in prof.items() if v["launches"]}), flush=True)
