"""Timing of the NEXT-2 triangular primitives on one GPU (CUDA events, median
of 5 after 2 warm-ups): lower_triangular_inverse (n^3/3 flops), trsm with m
right-hand sides (n^2 m flops), trsm_adjoint (n^2 m + n^2 m flops).
    python tools/bench_tri.py > profiles/r02_tri_bench.jsonl"""
from __future__ import annotations

import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1907_01063_b200 as sc  # noqa: E402


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    sc.load()
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    for n in (1024, 4096, 8192, 16384):
        x = torch.linspace(-10, 10, n, dtype=torch.float64, device="cuda")
        K = sc.gp_exp_quad_cov(x, 1.0, 1.0, 1e-2)
        L = sc.cholesky(K)
        X = torch.empty_like(L)
        ms = timed(lambda: sc.lower_triangular_inverse(L, out=X))
        print(json.dumps({"op": "lower_triangular_inverse", "n": n, "ms": ms,
                          "tflops": n ** 3 / 3 / ms / 1e9}), flush=True)
        for m in (64, 1024, n):
            B = torch.randn((n, m), dtype=torch.float64, device="cuda", generator=g)
            Y = torch.empty_like(B)
            ms = timed(lambda: sc.trsm(L, B, False, out=Y))
            ms_t = timed(lambda: sc.trsm(L, B, True, out=Y))
            ms_a = timed(lambda: sc.trsm_adjoint(L, Y, B))
            print(json.dumps({"op": "trsm", "n": n, "m": m, "ms": ms, "ms_trans": ms_t, "ms_adjoint": ms_a,
                              "tflops": n * n * m / ms / 1e9, "tflops_trans": n * n * m / ms_t / 1e9,
                              "tflops_adjoint": 2 * n * n * m / ms_a / 1e9}), flush=True)
            del B, Y
        del K, L, X
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
