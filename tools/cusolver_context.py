"""Context numbers: cuSOLVER via torch.linalg.cholesky and
torch autograd's Cholesky backward on the same SE workload, FP64, CUDA events.
Library code, NOT the product path; reported beside the bench line only."""
import json, sys
import torch
sys.path.insert(0, '.')
from paper_1907_01063_b200 import inputs

for n in [int(a) for a in sys.argv[1:]] or [4096, 16384]:
    x = torch.from_numpy(inputs.gp_x(n)).cuda()
    d = x[:, None] - x[None, :]
    K = torch.exp(d * d * -0.5)
    K.diagonal().add_(1e-6)
    del d
    Lbar = torch.from_numpy(inputs.lbar(n)).cuda()
    def fwd():
        return torch.linalg.cholesky(K)
    L = fwd()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    res = []
    for _ in range(3):
        Kr = K.clone().requires_grad_(True)
        torch.cuda.synchronize()
        ev[0].record()
        L = torch.linalg.cholesky(Kr)
        ev[1].record()
        (g,) = torch.autograd.grad(L, Kr, grad_outputs=Lbar)
        ev[2].record()
        torch.cuda.synchronize()
        res.append((ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])))
        del Kr, L, g
    f, b = min(r[0] for r in res), min(r[1] for r in res)
    print(json.dumps({"n": n, "impl": "torch.linalg.cholesky (cuSOLVER) + autograd backward",
                      "fwd_ms": f, "bwd_ms": b, "fwd_tflops": n ** 3 / 3 / f / 1e9,
                      "bwd_tflops_at_2n3_over_3": 2 * n ** 3 / 3 / b / 1e9}), flush=True)
