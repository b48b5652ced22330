"""Single-GPU run at large n (BASELINE.json configs[4] size, 1-GPU baseline):
timing of SE build + Cholesky + adjoint, plus the integer-exact check at full size.
Inputs are generated on the device (seeded torch generator) to avoid a 34 GB host
round trip; the integer-exact Gram matrix A = L0 L0^T uses cuBLAS (exact for
integers, input construction only)."""
import json, sys, time
import torch
sys.path.insert(0, '.')
import paper_1907_01063_b200 as sc
from paper_1907_01063_b200 import inputs

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
dev = torch.device('cuda', 0)
out = {"n": n}
x = torch.from_numpy(inputs.gp_x(n)).to(dev)
K = torch.empty((n, n), dtype=torch.float64, device=dev)
g = torch.Generator(device=dev); g.manual_seed(43)
W = torch.randn((n, n), dtype=torch.float64, device=dev, generator=g).tril_()
Ab = torch.empty_like(K)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
for it in range(2):
    torch.cuda.synchronize()
    ev[0].record(); sc.gp_exp_quad_cov(x, 1.0, 1.0, 1e-6, out=K)
    ev[1].record(); sc.cholesky(K, out=K)
    ev[2].record(); sc.cholesky_adjoint(K, W, out=Ab)
    ev[3].record(); torch.cuda.synchronize()
out.update({"se_ms": ev[0].elapsed_time(ev[1]), "chol_ms": ev[1].elapsed_time(ev[2]), "adj_ms": ev[2].elapsed_time(ev[3])})
tot = out["chol_ms"] + out["adj_ms"]
out["tflops"] = n ** 3 / tot / 1e9
out["finite"] = bool(torch.isfinite(Ab).all().item())
# log-det from the diagonal (finite, positive)
out["logdet"] = float(2 * torch.log(torch.diagonal(K)).sum().item())
del W, Ab
torch.cuda.empty_cache()
# integer-exact family at full size
g.manual_seed(n)
L0 = torch.randint(-1, 2, (n, n), device=dev, generator=g, dtype=torch.int8).to(torch.float64).tril_(-1)
L0.diagonal().fill_(1.0)
torch.matmul(L0, L0.T, out=K)
sc.cholesky(K, out=K)
out["integer_exact_bitwise"] = bool(torch.equal(K, L0))
print(json.dumps(out), flush=True)
