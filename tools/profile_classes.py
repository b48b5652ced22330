"""Per-kernel-class CUDA-event profile of one Cholesky + adjoint (dev tool)."""
import json, sys
import torch
sys.path.insert(0, '.')
import paper_1907_01063_b200 as sc
from paper_1907_01063_b200 import inputs
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
tag = sys.argv[2] if len(sys.argv) > 2 else ''
x = torch.from_numpy(inputs.gp_x(n)).cuda()
K = sc.gp_exp_quad_cov(x, 1, 1, 1e-6)
W = torch.from_numpy(inputs.lbar(n)).cuda()
L = torch.empty_like(K); A = torch.empty_like(K)
sc.cholesky(K, out=L); sc.cholesky_adjoint(L, W, out=A); torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
e[0].record(); sc.cholesky(K, out=L); e[1].record(); sc.cholesky_adjoint(L, W, out=A); e[2].record(); torch.cuda.synchronize()
tf, ta = e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2])
sc.profile_reset(); sc.profile_enable(True)
sc.cholesky(K, out=L); sc.cholesky_adjoint(L, W, out=A); torch.cuda.synchronize()
sc.profile_enable(False)
prof = sc.profile_read()
out = {"tag": tag, "n": n, "fwd_ms": tf, "adj_ms": ta, "total_tflops": n**3 / (tf + ta) / 1e9}
for k, v in prof.items():
    if v["launches"]:
        out[k] = [round(v["ms"], 2), round(v["flops"] / v["ms"] / 1e9, 2) if v["ms"] > 0 and v["flops"] > 0 else None]
print(json.dumps(out))
