"""Launch timeline of one forward / adjoint call (stan_cl_trace_*): where the
critical chain of the blocked factorisation spends its time.

    python tools/timeline.py 4096 [adjoint]   > profiles/r02_timeline_n4096.txt

Prints every launch (class, stream, start, end, duration) and, for the
forward, the per-step chain: POTRF start -> panel (POTRF + TRSM) end on the
side stream -> lookahead GEMM start/end on the main stream -> next POTRF
start, with the gaps between them (launch latency + cross-stream event hops).
"""
from __future__ import annotations

import collections
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1907_01063_b200 as sc  # noqa: E402
from paper_1907_01063_b200 import inputs  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    which = sys.argv[2] if len(sys.argv) > 2 else "forward"
    sc.load()
    x = torch.from_numpy(inputs.gp_x(n)).cuda()
    K = sc.gp_exp_quad_cov(x, 1.0, 1.0, 1e-6)
    L = torch.empty_like(K)
    W = torch.from_numpy(inputs.lbar(n)).cuda()
    A = torch.empty_like(K)
    for _ in range(3):                     # warm: workspace, graphs (tracing disables graphs)
        sc.cholesky(K, out=L)
        sc.cholesky_adjoint(L, W, out=A)
    torch.cuda.synchronize()
    sc.trace(True)
    if which == "forward":
        sc.cholesky(K, out=L)
    else:
        sc.cholesky_adjoint(L, W, out=A)
    torch.cuda.synchronize()
    recs = sc.trace_read()
    sc.trace(False)
    t_end = max(r[3] for r in recs)
    t_beg = min(r[2] for r in recs)
    print(f"# {which} n={n}: {len(recs)} launches, {t_end - t_beg:.3f} ms first start -> last end")
    by = collections.defaultdict(lambda: [0, 0.0])
    for k, s, a, b in recs:
        by[(k, s)][0] += 1
        by[(k, s)][1] += b - a
    print("# class            stream  launches    busy ms")
    for (k, s), (c, ms) in sorted(by.items(), key=lambda x: -x[1][1]):
        print(f"  {k:16s} {s:6d} {c:9d} {ms:10.3f}")
    if os.environ.get("TIMELINE_RAW"):
        # every launch in start order: stream, class, start, duration, gap after the previous launch on its stream
        last = {}
        print("# stream class            start_ms   dur_us  gap_us")
        for k, s, a, b in sorted(recs, key=lambda r: r[2]):
            g = (a - last[s]) * 1e3 if s in last else float("nan")
            last[s] = b
            print(f"  {s:5d}  {k:14s} {a:9.4f} {1e3 * (b - a):8.1f} {g:7.1f}")
    if which == "forward" and any(r[0] == "lookahead" and r[1] == 0 for r in recs):
        # chain: POTRF launches mark the steps
        pot = [r for r in recs if r[0] == "potrf"]
        la = [r for r in recs if r[0] == "lookahead" and r[1] == 0]
        side = [r for r in recs if r[1] != 0]
        print("# step  potrf_start  potrf_ms  panel_end  la_start  la_ms  gap_panel_to_la  gap_la_to_next_potrf")
        gaps1, gaps2, pms, pans, las = [], [], [], [], []
        for i, p in enumerate(pot):
            pend = max((r[3] for r in side if p[2] <= r[2] and (i + 1 == len(pot) or r[2] < pot[i + 1][2])),
                       default=p[3])
            nxt = pot[i + 1][2] if i + 1 < len(pot) else None
            l = next((r for r in la if r[2] >= pend - 1e-3), None)
            g1 = (l[2] - pend) if l else float("nan")
            g2 = (nxt - l[3]) if (l and nxt) else float("nan")
            pms.append(p[3] - p[2])
            pans.append(pend - p[2])
            if l:
                las.append(l[3] - l[2])
            if l and nxt:
                gaps1.append(g1)
                gaps2.append(g2)
            if i < 6 or i + 3 > len(pot):
                print(f"  {i:4d} {p[2]:11.3f} {p[3] - p[2]:9.4f} {pend:10.3f} {l[2] if l else float('nan'):9.3f} "
                      f"{(l[3] - l[2]) if l else float('nan'):6.4f} {g1:16.4f} {g2:21.4f}")
        m = lambda v: sum(v) / max(len(v), 1)
        print(f"# mean per step: potrf {1e3 * m(pms):.1f} us, panel (potrf+trsm) {1e3 * m(pans):.1f} us, "
              f"lookahead GEMM {1e3 * m(las):.1f} us, panel->la gap {1e3 * m(gaps1):.1f} us, "
              f"la->next potrf gap {1e3 * m(gaps2):.1f} us")


if __name__ == "__main__":
    main()
