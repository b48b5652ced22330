import sys, time, torch, numpy as np
sys.path.insert(0, '.')
import paper_1907_01063_b200 as sc
from paper_1907_01063_b200 import inputs
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
x = torch.from_numpy(inputs.gp_x(n)).cuda()
K = sc.gp_exp_quad_cov(x, 1, 1, 1e-6)
Kh = torch.empty((n, n), dtype=torch.float64).pin_memory(); Kh.copy_(K)
Lh = torch.empty_like(Kh).pin_memory(); Wh = torch.empty_like(Kh).pin_memory(); Wh.copy_(torch.from_numpy(inputs.lbar(n)))
Ah = torch.empty_like(Kh).pin_memory()
del K; torch.cuda.synchronize()
for it in range(3):
    t0 = time.perf_counter(); sc.cholesky_host(Kh, Lh); t1 = time.perf_counter()
    sc.cholesky_adjoint_host(Lh, Wh, Ah); t2 = time.perf_counter()
    print(f"iter {it}: chol_host {1e3*(t1-t0):.1f} ms  adjoint_host {1e3*(t2-t1):.1f} ms", flush=True)
