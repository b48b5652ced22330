#!/usr/bin/env python
"""bench.py -- FP64 Cholesky + adjoint on B200 (arXiv:1907.01063 hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--n 16384] [--impl ours|reference]

One step = one pass of the whole hot path over one synthetic GP problem at
n = 16384 (BASELINE.json configs[3], the configuration the metric is quoted on):
SE covariance build from x (F0), Cholesky (F1-F4), adjoint (R0-R5), all through
the C ABI with device-resident inputs.  Flops counted: n^3/3 + 2n^3/3 (SURVEY.md
§8 convention; the O(n^2) SE build is timed but not counted).

Prints ONE JSON line on rank 0.  Multi-GPU (torchrun): replicas -- every rank
factors its own matrix, value = sum over ranks, time = max over
ranks.  ``--impl reference`` times the CPU oracle (oracle/, single thread) on a
bounded sample of the same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FP64 Cholesky+adjoint GFLOP/s and ms at n=16384; fraction of B200 FP64 peak"
UNIT = "GFLOP/s"
ALPHA, RHO, JITTER = 1.0, 1.0, 1e-6
# FP64 peak: DMMA (mma.sync .f64) register-resident microbenchmark on this pool's
# B200s, 37.15 TFLOP/s at 1965 MHz (profiles/fp64_peak_r01.jsonl; tools/fp64_peak.cu).
# MEASURED_PEAKS.json carries no FP64 figure; its bf16 numbers do not apply.
FP64_PEAK_TFLOPS = 37.1
PEAK_SOURCE = "measured: tools/fp64_peak.cu DMMA.8x8x4 loop, 148 SMs, profiles/fp64_peak_r01.jsonl"
ORACLE_SAMPLE_N = 2048

REASON_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}


def baseline_config_index(n: int, world: int) -> str:
    idx = {64: 0, 1024: 1, 8192: 2, 16384: 3, 65536: 4}.get(n)
    return f"BASELINE.json configs[{idx}]" if idx is not None else "not a BASELINE.json config"


L2_BYTES = 126 * 2 ** 20


def l2_resident(n: int) -> bool:
    """K/L, L_bar and A_bar of one step fit in L2 (n <= ~2300): time each step
    separately with an L2 flush before it (bench timing rule)."""
    return 3 * 8 * n * n < L2_BYTES


def config(n: int, world: int, mode: str = "single", grid: tuple = (1, 1)) -> dict:
    return {
        "workload": f"SE-kernel GP covariance n={n} (1-D x~U(-10,10), alpha=rho=1, jitter 1e-6): "
                    f"SE build + Cholesky + adjoint ({baseline_config_index(n, world)})",
        "n": n, "nb": (("forward: 256-wide outer blocks of 128-wide tiles (two-level); adjoint: " if n >= 6144
                        else "forward: 128-wide blocks; adjoint: ")
                       + ("256" if n >= 768 else "128") + "-wide blocks"),
        "flops_per_step": n ** 3,
        "flop_convention": "n^3/3 (Cholesky) + 2n^3/3 (adjoint)",
        "l2": ("inputs exceed L2 (one n x n FP64 matrix = %.2f GiB vs 126 MB L2); no flush needed" % (8 * n * n / 2 ** 30)
               if not l2_resident(n) else
               "the step's matrices fit in the 126 MB L2: a 256 MiB buffer is written before every timed step "
               "(outside the per-step events, which are summed)"),
        "parallelism": {"single": "single GPU",
                        "replicas": f"replicas: {world} independent problems, one per GPU",
                        "dist": f"2-D block-cyclic 256x256 tiles over {world} GPUs (P={grid[0]} x Q={grid[1]}), "
                                "NCCL row/column broadcasts of panels / C_bar D^-1 / L rows / sym(S), "
                                "column reductions of C_bar^T [B C]"}[mode],
    }


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], [], set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 4:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
                bits = int(parts[3], 16)
            except ValueError:
                continue
            for b, name in REASON_BITS.items():
                if bits & b and name != "gpu_idle":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


DMMA_CLASSES = ("syrk", "adj_gemm", "splitk", "lookahead", "trmm")
# roofline bound per library profiling class: FP64 tensor (DMMA) GEMMs, the
# FMA-bound latency kernels (POTRF / TRSM tiles, triangular inverses, the small
# register kernels), and the memory-bound O(n^2) passes
CLASS_BOUND = {"syrk": "tensor", "adj_gemm": "tensor", "splitk": "tensor", "lookahead": "tensor", "trmm": "tensor",
               "gemm128": "alu", "potrf": "alu", "trsm": "alu", "tri_inverse": "alu", "gp": "alu",
               "se_cov": "hbm", "other": "hbm"}
FP64_DFMA_PEAK_TFLOPS = 34.2   # measured (profiles/fp64_peak_r01.jsonl, DFMA loop)
HBM_PEAK_GBS = 6459.9          # MEASURED_PEAKS.json hbm_gbs (copy, read + write)


def traffic_from_profiles(kind: str):
    """Measured DRAM bytes (read + write) per launch of class `kind` from the committed
    ncu launch list summary (profiles/traffic.json, tools/traffic_from_launches.py)."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d["classes"][kind]["dram_bytes_per_launch"]
    except Exception:
        return None


def traffic_aggregate(kinds) -> float | None:
    """DRAM bytes per launch over the given classes from profiles/traffic.json (the
    ncu launch list classifies the C_bar D^-1 launches with the rank-256 updates:
    same kernel instantiation), launch-weighted."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            cl = json.load(f)["classes"]
    except Exception:
        return None
    keys = [k for k in kinds if k in cl]
    if len(kinds) == 1:
        return cl[kinds[0]]["dram_bytes_per_launch"] if keys else None
    tot = sum(cl[k]["dram_bytes_per_launch"] * cl[k]["launches"] for k in keys)
    cnt = sum(cl[k]["launches"] for k in keys)
    return tot / cnt if cnt else None


def host_path_bytes(n: int, adj_block: int) -> tuple[int, int]:
    """Bytes the host entry points move per call pair (include/stan_cl.h):
    lower-triangle rectangles, rows [r, r+128) x columns [0, r+128) for K (H2D),
    L (D2H), and L, L_bar (H2D); A_bar ships per adjoint block column j (width
    B): its diagonal block per 128-row slab, rows [r, r+128) x columns [j, r+128),
    then rows [j+B, n) x columns [j, j+B) (D2H)."""
    tri = sum(8 * (min(r + 128, n) - r) * min(r + 128, n) for r in range(0, n, 128))
    cols = 0
    for j in range(0, n, adj_block):
        k = min(j + adj_block, n)
        cols += sum(8 * (min(r + 128, n) - r) * (min(r + 128, n) - j) for r in range(j, k, 128))
        cols += 8 * (n - k) * (k - j)
    return 3 * tri, tri + cols


def max_over_ranks(value: float, world: int, device=None) -> float:
    """Max of a per-rank scalar over all ranks (timing rule: max over ranks)."""
    if world <= 1:
        return float(value)
    import torch
    t = torch.tensor([value], dtype=torch.float64, device=device)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def replica_seeds(rank: int) -> tuple[int, int]:
    """Per-rank input seeds of the replicas mode (independent problems per GPU)."""
    from paper_1907_01063_b200 import inputs
    return inputs.X_SEED + rank, inputs.LBAR_SEED + rank


def oracle_sample_inputs(n: int, n_s: int):
    """The bounded oracle sample of the order-n workload: the leading n_s x n_s
    block of the SAME synthetic problem -- K from x_1..x_{n_s} of the n-point
    draw (so the oracle's Cholesky-Banachiewicz rows 0..n_s-1 are exactly the
    first n_s rows of its order-n run) and the leading block of the same L_bar
    draw (the order-n adjoint of an L_bar supported on that block, restricted to
    it).  n_s = n when n <= n_s."""
    import oracle
    from paper_1907_01063_b200 import inputs
    n_s = min(n, n_s)
    K = oracle.se_cov(inputs.gp_x(n)[:n_s], ALPHA, RHO, JITTER)
    W = inputs.lbar_leading(n, n_s)
    return K, W


def run_oracle_sample(n: int, n_s: int) -> tuple[float, float]:
    """Oracle Cholesky + adjoint of the sample on one core: (seconds, flops)."""
    import oracle
    K, W = oracle_sample_inputs(n, n_s)
    t0 = time.perf_counter()
    L = oracle.cholesky(K)
    oracle.cholesky_adjoint(L, W)
    return time.perf_counter() - t0, float(K.shape[0]) ** 3


def sample_desc(n: int, n_s: int) -> str:
    m = min(n, n_s)
    if m == n:
        return f"the whole order-{n} workload (oracle Cholesky + adjoint), 1 thread"
    return (f"leading {m} x {m} block of the order-{n} workload (x_1..x_{m} of the same draw, leading block of "
            f"the same L_bar): the oracle's first {m} rows of L of the order-{n} problem plus the adjoint of "
            f"that block; {m ** 3 / n ** 3:.2e} of the step's flops, rate = sample flops / sample time, 1 thread")


def cpu_baseline_entry(n: int, n_sample: int) -> dict:
    secs, fl = run_oracle_sample(n, n_sample)
    return {"value": fl / secs / 1e9, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": sample_desc(n, n_sample) + f"; one run, {secs:.2f} s; host {os.cpu_count()} logical cores",
            "sample_n": min(n, n_sample), "sample_seconds": secs}


def bench_reference(args, rank: int, world: int):
    if rank != 0:
        return
    n_s = min(args.n, args.oracle_n)
    for _ in range(args.warmup):
        run_oracle_sample(args.n, n_s)
    times = []
    for _ in range(args.steps):
        s, fl = run_oracle_sample(args.n, n_s)
        times.append(s)
    ms = 1e3 * statistics.mean(times)
    val = float(n_s) ** 3 / (ms / 1e3) / 1e9
    cfg = config(args.n, world)
    cfg["sample"] = sample_desc(args.n, n_s)
    cfg["sample_n"] = n_s
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": cfg,
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": "each step = " + sample_desc(args.n, n_s)},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def setup_dist(sc, world: int, local_rank: int, grid=None) -> bool:
    """NCCL communicators of the library (P x Q grid); every rank must succeed, else replicas."""
    import torch
    ok = 1
    try:
        sc.dist_init_from_torch(None, *(grid or (None, None)))
    except Exception as e:  # noqa: BLE001
        print(f"[bench] dist init failed on this rank: {e}", file=sys.stderr, flush=True)
        ok = 0
    t = torch.tensor([ok], dtype=torch.int32, device=torch.device("cuda", local_rank))
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MIN)
    return bool(t.item())


def bench_ours(args, rank: int, world: int, local_rank: int):
    import numpy as np
    import torch
    import paper_1907_01063_b200 as sc
    from paper_1907_01063_b200 import inputs

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    n = args.n
    sc.load()
    mode = "single"
    if world > 1:
        mode = "replicas"
        grid = tuple(int(v) for v in args.grid.lower().split("x")) if args.grid else sc.dist_grid(world)
        if args.mode in ("auto", "dist") and n % sc.DIST_BLOCK == 0 and grid[0] * grid[1] == world \
                and setup_dist(sc, world, local_rank, grid):
            mode = "dist"
    e2e_fn = None
    if mode == "dist":
        # one problem of order n, 256 x 256 tiles 2-D block-cyclic over the P x Q grid (strong scaling)
        P, Q = grid
        gp, gq = divmod(rank, Q)
        x = torch.from_numpy(inputs.gp_x(n)).to(dev)
        hrows, w = sc.dist_local_shape(n, P, Q, gp, gq)
        # L_bar's local tiles ~ N(0, 1), drawn on the device per rank (seed 43 + rank):
        # the full n x n host matrix would be 32 GiB per rank at n = 65536; only
        # lower tiles are read (the tiles above the diagonal are ignored)
        gen = torch.Generator(device=dev)
        gen.manual_seed(inputs.LBAR_SEED + rank)
        Lbar_loc = torch.randn((hrows, w), dtype=torch.float64, device=dev, generator=gen)
        K_loc = torch.empty((hrows, w), dtype=torch.float64, device=dev)
        W_loc = torch.empty_like(K_loc)

        def step():
            sc.gp_exp_quad_cov_tiles(x, K_loc, P, Q, gp, gq, ALPHA, RHO, JITTER)  # F0 (owned tiles)
            sc.dist_cholesky(K_loc, n)                                          # F1-F4, NCCL panel broadcasts
            W_loc.copy_(Lbar_loc)
            sc.dist_cholesky_adjoint(K_loc, W_loc, n)                           # R0-R5, NCCL broadcasts

        def check_status():                                                      # the dist calls raise on failure
            pass

        # two pinned host buffers per rank: K in / L out share one (the upload
        # precedes the download on the stream), L_bar in / A_bar out the other
        Kh = torch.empty((hrows, w), dtype=torch.float64).pin_memory()
        Lbh = torch.empty((hrows, w), dtype=torch.float64).pin_memory()
        Lbh.copy_(Lbar_loc)
        Khost = torch.empty_like(Kh)
        sc.gp_exp_quad_cov_tiles(x, K_loc, P, Q, gp, gq, ALPHA, RHO, JITTER)
        Khost.copy_(K_loc)
        Lbhost = Lbh.clone()

        def e2e_fn():
            K_loc.copy_(Kh, non_blocking=True)
            sc.dist_cholesky(K_loc, n)
            Kh.copy_(K_loc, non_blocking=True)                 # L out
            W_loc.copy_(Lbh, non_blocking=True)
            sc.dist_cholesky_adjoint(K_loc, W_loc, n)
            Lbh.copy_(W_loc, non_blocking=True)                # A_bar out

        def e2e_reset():                                       # fresh inputs before each timed e2e step
            Kh.copy_(Khost)
            Lbh.copy_(Lbhost)
        e2e_bytes = (2 * 8 * hrows * w, 2 * 8 * hrows * w)
        e2e_path = "per rank: pinned H2D of its K and L_bar tiles, dist_cholesky + dist_cholesky_adjoint, D2H of L and A_bar"
    else:
        xs, ls = replica_seeds(rank)
        x = torch.from_numpy(inputs.gp_x(n, seed=xs)).to(dev)
        Lbar = torch.from_numpy(inputs.lbar(n, seed=ls)).to(dev)
        K = torch.empty((n, n), dtype=torch.float64, device=dev)
        Abar = torch.empty_like(K)

        info = torch.zeros(2, dtype=torch.int32, device=dev)

        def step():
            # the *_async entry points: enqueue only, the LAPACK-style status goes
            # to a device word (checked after the timed region) instead of a host
            # sync per call
            sc.gp_exp_quad_cov(x, ALPHA, RHO, JITTER, out=K)      # F0
            sc.cholesky_async(K, K, info[0:1])                    # F1-F4 (in place)
            sc.cholesky_adjoint_async(K, Lbar, Abar, info[1:2])   # R0-R5

        def check_status():
            st = info.tolist()
            if any(st):
                raise RuntimeError(f"bench step failed: cholesky info {st[0]}, adjoint info {st[1]}")

    def barrier():
        if world > 1:
            torch.distributed.barrier(device_ids=[local_rank])

    # warm-up; the last warm-up step is profiled for every kernel class (untimed):
    # it picks the dominant DMMA class, the only one events bracket in the timed region
    for i in range(args.warmup):
        if i == args.warmup - 1:
            torch.cuda.synchronize()
            sc.profile_reset()
            sc.profile_enable(True)
        step()
    torch.cuda.synchronize()
    sc.profile_enable(False)
    warm = sc.profile_read()
    # the dominant kernel of the step: when the DMMA GEMM classes take most of the
    # time, the one with the most algorithmic work (deterministic: the SYRK, the
    # split-K contraction and the rank-256 update each take ~30% of the n = 16384
    # step and tie within run-to-run noise in event time; the split-K
    # contraction carries the most flops); otherwise (n <= 64: the register
    # kernels) the class with the most event time.  Only that class is
    # event-bracketed inside the timed region (bracketing more launches breaks
    # the programmatic-dependent-launch overlap: +1.3 ms per step measured).
    dmma_ms = sum(warm[k]["ms"] for k in DMMA_CLASSES)
    if dmma_ms >= 0.5 * sum(v["ms"] for v in warm.values()):
        dom_kinds = [max(DMMA_CLASSES, key=lambda k: warm[k]["flops"])]
    else:
        dom_kinds = [max(warm, key=lambda k: warm[k]["ms"])]
    dom = dom_kinds[0]
    barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local_rank)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with sampler:
        time.sleep(0.3)
        launches0 = sc.kernel_launches()
        sc.profile_reset()
        sc.profile_enable(True, kinds=dom_kinds)
        if l2_resident(n):
            # small problems: flush L2 (write 256 MiB) before every step, time the
            # steps alone and sum them (the flush is not ours and not timed)
            flush = torch.empty(32 * 2 ** 20, dtype=torch.float64, device=dev)
            ea = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
            eb = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
            for i in range(args.steps):
                flush.fill_(float(i))
                ea[i].record()
                step()
                eb[i].record()
            torch.cuda.synchronize()
            step_ms = sum(a.elapsed_time(b) for a, b in zip(ea, eb)) / args.steps
            del flush
        else:
            e0.record()
            for _ in range(args.steps):
                step()
            e1.record()
            torch.cuda.synchronize()
            step_ms = e0.elapsed_time(e1) / args.steps
        sc.profile_enable(False)
        check_status()
        launches = sc.kernel_launches() - launches0
        prof = sc.profile_read()
    barrier()
    ms_max = max_over_ranks(step_ms, world, dev)
    flops = float(n) ** 3
    jobs = world if mode == "replicas" else 1                  # dist: one problem over all ranks
    value = jobs * flops / (ms_max / 1e3) / 1e9
    clocks = sampler.summary()

    # roofline of the dominant kernel class: algorithmic flops / event-timed duration
    # of its launches inside the timed region
    d = {key: sum(prof[k][key] for k in dom_kinds) for key in ("ms", "flops", "bytes", "launches")}
    nl = max(d["launches"], 1)
    bound = CLASS_BOUND.get(dom_kinds[0], "tensor")
    if bound == "hbm":
        achieved = d["bytes"] / (d["ms"] / 1e3) / 1e9 if d["ms"] > 0 else 0.0
        peak, unit, src = HBM_PEAK_GBS, "GB/s", "MEASURED_PEAKS.json hbm_gbs"
    else:
        achieved = d["flops"] / (d["ms"] / 1e3) / 1e12 if d["ms"] > 0 else 0.0
        peak, unit = (FP64_PEAK_TFLOPS, "TFLOP/s") if bound == "tensor" else (FP64_DFMA_PEAK_TFLOPS, "TFLOP/s")
        src = PEAK_SOURCE if bound == "tensor" else "measured: FP64 DFMA loop, profiles/fp64_peak_r01.jsonl"
    tr = traffic_aggregate(dom_kinds)
    roofline = {"bound": bound, "kernel": dom, "selection": "DMMA class with the most algorithmic flops per step",
                "achieved": achieved, "peak": peak,
                "unit": unit, "frac": achieved / peak,
                "traffic": tr, "algorithmic_bytes_per_launch": d["bytes"] / nl,
                "flops_per_launch": d["flops"] / nl, "peak_source": src,
                "per_launch_ms": d["ms"] / nl, "launches_per_step": d["launches"] // args.steps,
                "traffic_source": "profiles/traffic.json (ncu dram__bytes_read+write per launch)"}
    classes = {k: {"ms_per_step": v["ms"],
                   "tflops": (v["flops"] / (v["ms"] / 1e3) / 1e12) if v["ms"] > 0 and v["flops"] > 0 else None,
                   "hbm_gbs_algorithmic": (v["bytes"] / (v["ms"] / 1e3) / 1e9) if v["ms"] > 0 else None,
                   "launches_per_step": v["launches"]} for k, v in warm.items() if v["launches"]}

    # end-to-end through the public host-buffer API (pinned host in/out)
    e2e = None
    if args.e2e_steps > 0 and e2e_fn is not None:
        e2e_reset()
        e2e_fn()
        torch.cuda.synchronize()
        ems_l = []
        for _ in range(args.e2e_steps):
            e2e_reset()                                        # host-side refill, outside the timed region
            barrier()
            torch.cuda.synchronize()
            f0 = torch.cuda.Event(enable_timing=True)
            f1 = torch.cuda.Event(enable_timing=True)
            f0.record()
            e2e_fn()
            f1.record()
            torch.cuda.synchronize()
            ems_l.append(f0.elapsed_time(f1))
        ems = max_over_ranks(sum(ems_l) / len(ems_l), world, dev)
        e2e = {"value": flops / (ems / 1e3) / 1e9, "unit": UNIT, "ms_per_step": ems,
               "h2d_bytes_per_step": int(e2e_bytes[0]) * world, "d2h_bytes_per_step": int(e2e_bytes[1]) * world,
               "path": e2e_path}
    elif args.e2e_steps > 0:
        Kh = torch.empty((n, n), dtype=torch.float64).pin_memory()
        sc.gp_exp_quad_cov(x, ALPHA, RHO, JITTER, out=K)
        Kh.copy_(K)
        Lh = torch.empty_like(Kh).pin_memory()
        Lbh = torch.empty_like(Kh).pin_memory()
        Lbh.copy_(Lbar)
        Abh = torch.empty_like(Kh).pin_memory()
        torch.cuda.synchronize()

        def e2e_step():
            sc.cholesky_host(Kh, Lh, device=local_rank)
            sc.cholesky_adjoint_host(Lh, Lbh, Abh, device=local_rank)

        e2e_step()
        torch.cuda.synchronize()
        barrier()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(args.e2e_steps):
            e2e_step()
        f1.record()
        torch.cuda.synchronize()
        ems = max_over_ranks(f0.elapsed_time(f1) / args.e2e_steps, world, dev)
        hb = host_path_bytes(n, 256 if n >= 768 else 128)
        # the host path must reproduce the device-resident results (sampled lower entries;
        # K was overwritten with the covariance for the upload, so recompute on the device)
        step()
        torch.cuda.synchronize()
        rs = np.random.default_rng(7)
        ii = rs.integers(0, n, 4096)
        jj = (rs.random(4096) * (ii + 1)).astype(np.int64)
        idx = torch.from_numpy(ii * n + jj)
        Ld_s, Ad_s = K.flatten()[idx.to(dev)].cpu(), Abar.flatten()[idx.to(dev)].cpu()
        Lh_s, Ah_s = Lh.flatten()[idx], Abh.flatten()[idx]
        rel_L = float((Lh_s - Ld_s).norm() / Ld_s.norm())
        rel_A = float((Ah_s - Ad_s).norm() / Ad_s.norm())
        if not (rel_L <= 1e-13 and rel_A <= 1e-12):
            raise RuntimeError(f"host-path results differ from the device path: L {rel_L:.2e}, A_bar {rel_A:.2e}")
        e2e = {"value": jobs * flops / (ems / 1e3) / 1e9, "unit": UNIT, "ms_per_step": ems,
               "h2d_bytes_per_step": hb[0], "d2h_bytes_per_step": hb[1],
               "checked_vs_device": {"samples": 4096, "L_rel": rel_L, "A_bar_rel": rel_A},
               "path": "stan_cl_cholesky_host(K) + stan_cl_cholesky_adjoint_host(L, L_bar), pinned host buffers"}
        del Kh, Lh, Lbh, Abh

    if rank != 0:
        return
    cpu = None if args.no_cpu_baseline else cpu_baseline_entry(n, args.oracle_n)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
        "scaling": "strong" if mode == "dist" else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config(n, world, mode, grid if mode == "dist" else (1, 1)),
        "fp64_peak_frac": (jobs * flops / (ms_max / 1e3) / 1e12) / (FP64_PEAK_TFLOPS * world),
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": launches, "clocks": clocks,
        "kernel_classes_warmup_step": classes,
    }
    print(json.dumps(line), flush=True)


def dry_run(args, rank: int, world: int):
    """No device work: rendezvous over gloo, barrier, max over ranks of a per-rank
    number, one JSON line on rank 0 (tests/test_bench_cpu.py)."""
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("gloo")
    try:
        t0 = time.perf_counter()
        if world > 1:
            dist.barrier()
        for _ in range(args.warmup + args.steps):
            pass
        ms = (time.perf_counter() - t0) * 1e3
        if world > 1:
            t = torch.tensor([ms], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        if rank == 0:
            grid = dist_grid_default(world)
            print(json.dumps({"dry_run": True, "metric": METRIC, "value": None, "unit": UNIT, "n_gpus": world,
                              "steps": args.steps, "warmup": args.warmup, "ms_per_step": None,
                              "host_ms_max_over_ranks": ms, "higher_is_better": True,
                              "scaling": "strong" if world > 1 else "weak",
                              "config": config(args.n, world, "dist" if world > 1 else "single", grid)}),
                  flush=True)
    finally:
        if world > 1:
            dist.destroy_process_group()


def dist_grid_default(G: int) -> tuple:
    """Same rule as paper_1907_01063_b200.dist_grid (1x1, 1x2, 2x2, 2x4, ...)."""
    P = max(d for d in range(1, int(G ** 0.5) + 1) if G % d == 0)
    return P, G // P


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--n", type=int, default=None,
                    help="order (default: 16384 = BASELINE configs[3] at N=1; 65536 = configs[4] at N>1)")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU plumbing check: launch/rendezvous (gloo), barrier, max-over-ranks and the JSON "
                         "line, with no device work (value is null)")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--oracle-n", type=int, default=ORACLE_SAMPLE_N)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--grid", default="", help="N>1 dist mode: process grid PxQ (default: 1x2, 2x2, 2x4 ...)")
    ap.add_argument("--mode", choices=["auto", "dist", "replicas"], default="auto",
                    help="N>1: distributed (strong scaling, default) or independent replicas")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.n is None:
        args.n = 16384 if args.gpus == 1 else 65536
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-launch this script under torchrun (the driver
        # normally does this itself; a bare `bench.py --gpus N` must not silently
        # run one GPU)
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        print(f"[bench] launching {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"[bench] refusing to report: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr, flush=True)
        sys.exit(2)
    if args.dry_run:
        dry_run(args, rank, world)
        return
    if args.impl == "reference":
        bench_reference(args, rank, world)
        return
    if world > 1:
        import torch
        torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        bench_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch
            try:
                import paper_1907_01063_b200 as sc
                sc.load().stan_cl_dist_finalize()
            except Exception:  # noqa: BLE001
                pass
            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
