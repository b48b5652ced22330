"""Single-GPU adjoint vs the distributed adjoint on a 1 x 1 grid (same algorithm +
side-stream lookahead for the B_bar update) and the distributed forward on 1 x 1."""
import sys, json
import torch
sys.path.insert(0, '.')
import paper_1907_01063_b200 as sc
from paper_1907_01063_b200 import inputs

def ev(fn, reps=3):
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts)

for n in [int(v) for v in sys.argv[1:]] or [8192, 16384]:
    x = torch.from_numpy(inputs.gp_x(n)).cuda()
    K = sc.gp_exp_quad_cov(x, 1.0, 1.0, 1e-6)
    L = torch.empty_like(K)
    sc.cholesky(K, out=L)
    W0 = torch.from_numpy(inputs.lbar(n)).cuda()
    Ab = torch.empty_like(K)
    t_single = ev(lambda: sc.cholesky_adjoint(L, W0, out=Ab))
    Wd = torch.empty_like(K)
    def dist_adj():
        Wd.copy_(W0)
        sc.dist_sim2_cholesky_adjoint([L], [Wd], n, 1, 1)
    t_copy = ev(lambda: Wd.copy_(W0))
    t_dist = ev(dist_adj) - t_copy
    diff = float((torch.tril(Wd) - torch.tril(Ab)).abs().max() / Ab.abs().max())
    Kd = torch.empty_like(K)
    def dist_fwd():
        Kd.copy_(K)
        sc.dist_sim2_cholesky([Kd], n, 1, 1)
    t_dfwd = ev(dist_fwd) - t_copy
    t_fwd = ev(lambda: sc.cholesky(K, out=L))
    print(json.dumps({"n": n, "adj_single_ms": t_single, "adj_dist11_ms": t_dist, "rel_maxdiff": diff,
                      "fwd_single_ms": t_fwd, "fwd_dist11_ms": t_dfwd}), flush=True)
