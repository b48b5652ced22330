"""One forward (and optionally adjoint) at n (dev tool for ncu launch lists)."""
import sys
import torch
sys.path.insert(0, '.')
import paper_1907_01063_b200 as sc
from paper_1907_01063_b200 import inputs
n = int(sys.argv[1])
x = torch.from_numpy(inputs.gp_x(n)).cuda()
K = sc.gp_exp_quad_cov(x, 1.0, 1.0, 1e-6)
L = torch.empty_like(K)
sc.cholesky(K, out=L)
torch.cuda.synchronize()
if len(sys.argv) > 2:
    W = torch.from_numpy(inputs.lbar(n)).cuda()
    Ab = torch.empty_like(K)
    sc.cholesky_adjoint(L, W, out=Ab)
    torch.cuda.synchronize()
