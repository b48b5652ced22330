"""Quick CUDA-event timing of the forward and adjoint at a few sizes (dev tool)."""
import sys, time, json
import numpy as np, torch
sys.path.insert(0, '.')
import paper_1907_01063_b200 as sc
from paper_1907_01063_b200 import inputs

def t_ev(fn, reps=3):
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts)

for n in [int(a) for a in sys.argv[1:]] or [1024, 4096, 8192, 16384]:
    x = torch.from_numpy(inputs.gp_x(n)).cuda()
    K = sc.gp_exp_quad_cov(x, 1.0, 1.0, 1e-6)
    L = torch.empty_like(K)
    W = torch.from_numpy(inputs.lbar(n)).cuda()
    Ab = torch.empty_like(K)
    sc.cholesky(K, out=L); sc.cholesky_adjoint(L, W, out=Ab)
    tf = t_ev(lambda: sc.cholesky(K, out=L))
    ta = t_ev(lambda: sc.cholesky_adjoint(L, W, out=Ab))
    fl_f, fl_a = n**3/3, 2*n**3/3
    print(json.dumps({"n": n, "fwd_ms": tf, "adj_ms": ta, "fwd_tflops": fl_f/tf/1e9, "adj_tflops": fl_a/ta/1e9,
                      "total_tflops": (fl_f+fl_a)/(tf+ta)/1e9}), flush=True)
