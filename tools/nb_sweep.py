"""Forward outer block 128 vs 256 (stan_cl_set_block_size) at a few sizes (dev tool)."""
import sys, json
import torch
sys.path.insert(0, '.')
import paper_1907_01063_b200 as sc
from paper_1907_01063_b200 import inputs

def ev(fn, reps=5):
    fn()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts)

lib = sc.load()
for n in [int(v) for v in sys.argv[1:]] or [1024, 2048, 4096, 8192]:
    x = torch.from_numpy(inputs.gp_x(n)).cuda()
    K = sc.gp_exp_quad_cov(x, 1.0, 1.0, 1e-6)
    L = torch.empty_like(K)
    out = {"n": n}
    for nb in (128, 256):
        lib.stan_cl_set_block_size(nb)
        out[f"fwd_nb{nb}_ms"] = ev(lambda: sc.cholesky(K, out=L))
    lib.stan_cl_set_block_size(0)
    print(json.dumps(out), flush=True)

# adjoint block 128 vs 256 (stan_cl_set_adjoint_block_size)
for n in [int(v) for v in sys.argv[1:]] or [1024, 2048, 4096, 8192]:
    x = torch.from_numpy(inputs.gp_x(n)).cuda()
    K = sc.gp_exp_quad_cov(x, 1.0, 1.0, 1e-6)
    L = sc.cholesky(K)
    W = torch.from_numpy(inputs.lbar(n)).cuda()
    A = torch.empty_like(K)
    out = {"n": n}
    for nb in (128, 256):
        lib.stan_cl_set_adjoint_block_size(nb)
        out[f"adj_nb{nb}_ms"] = ev(lambda: sc.cholesky_adjoint(L, W, out=A))
    lib.stan_cl_set_adjoint_block_size(0)
    print(json.dumps(out), flush=True)
