"""NEXT-1/NEXT-2 measurement: the GP log density + gradient and the triangular
solve on one GPU (CUDA events, device-resident inputs, warm-up first).

    python tools/bench_gp.py [n ...]     # default 4096 16384

Per n: total ms of stan_cl_gp_lpdf_grad, the hot path's share (cholesky +
adjoint classes), the per-class profile, and stan_cl_trsv (both directions)
with its algorithmic bytes (the lower triangle, n(n+1)/2 * 8) over time
against the measured HBM copy bandwidth.  One JSON line per n.
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1907_01063_b200 as sc  # noqa: E402
from paper_1907_01063_b200 import inputs  # noqa: E402

HBM_GBS = 6456.8  # MEASURED_PEAKS.json copy bandwidth (B200_PROFILING.md fallback if absent)
try:
    HBM_GBS = float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    pass


def ev_ms(fn, reps=5):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts)), float(min(ts))


for n in [int(a) for a in sys.argv[1:]] or [4096, 16384]:
    x = torch.from_numpy(inputs.gp_x(n)).cuda()
    y = torch.from_numpy(inputs.gp_y(inputs.gp_x(n))).cuda()
    a_, r_, s_ = 1.0, 1.0, 0.1
    sc.gp_lpdf_grad(x, y, a_, r_, s_)
    med, best = ev_ms(lambda: sc.gp_lpdf_grad(x, y, a_, r_, s_))
    sc.profile_reset()
    sc.profile_enable(True)
    sc.gp_lpdf_grad(x, y, a_, r_, s_)
    torch.cuda.synchronize()
    sc.profile_enable(False)
    prof = {k: round(v["ms"], 3) for k, v in sc.profile_read().items() if v["launches"]}
    # triangular solve alone, on the factor of the same K
    K = sc.gp_exp_quad_cov(x, a_, r_, s_ * s_)
    L = sc.cholesky(K)
    b = y.clone()
    out = torch.empty_like(b)
    tr = {}
    for trans in (False, True):
        m, bm = ev_ms(lambda: sc.trsv(L, b, trans=trans, out=out), reps=9)
        byt = 8.0 * n * (n + 1) / 2
        tr["trans" if trans else "lower"] = {"ms": m, "GBs": byt / (m / 1e3) / 1e9,
                                             "frac_hbm": byt / (m / 1e3) / 1e9 / HBM_GBS}
    line = {"n": n, "gp_lpdf_grad_ms": med, "gp_lpdf_grad_best_ms": best,
            "hot_path_tflops_equiv": n ** 3 / (med / 1e3) / 1e12,
            "profile_ms": prof, "trsv": tr, "hbm_peak_gbs": HBM_GBS}
    print(json.dumps(line), flush=True)
