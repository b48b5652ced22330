"""Per-class FP64 tensor-pipe utilisation from an ncu launch list.

    ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed,\
sm__inst_executed_pipe_tensor_subpipe_dmma.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file L.csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline
    python tools/dmma_util_from_launches.py L.csv [out.txt]

SURVEY.md §8(d): the >= 60% bar is the DMMA-pipe utilisation of the trailing
updates (SYRK, split-K contraction, rank-B update), time-weighted over launches;
flops are counted from executed DMMA.8x8x4 instructions (512 flops each), so the
achieved TFLOP/s here is independent of the library's algorithmic count.
Representative launches (first, middle, last of the last step) are listed too.
"""
import collections
import csv
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from traffic_from_launches import UNITS, classify  # noqa: E402

PCT = "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed"
INST = "sm__inst_executed_pipe_tensor_subpipe_dmma.sum"


def main(path, out=None):
    recs = collections.OrderedDict()
    hdr = None
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        rec = recs.setdefault(d["ID"], {"name": d["Kernel Name"]})
        rec[d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) * UNITS.get(d["Metric Unit"], 1.0)
    byc = collections.defaultdict(list)
    for rec in recs.values():
        if rec.get(INST, 0) > 0:
            byc[classify(rec["name"])].append(rec)
    lines = [f"# {path}: DMMA-pipe utilisation per class (ncu, serialised, cold cache)",
             f"{'class':14s} {'launches':>8s} {'ms':>9s} {'DMMA %':>7s} {'TFLOP/s':>8s} {'min %':>6s} {'max %':>6s}"]
    for c, rs in sorted(byc.items(), key=lambda x: -sum(r["gpu__time_duration.sum"] for r in x[1])):
        ms = sum(r["gpu__time_duration.sum"] for r in rs)
        pct = sum(r[PCT] * r["gpu__time_duration.sum"] for r in rs) / ms
        fl = sum(r[INST] for r in rs) * 512.0
        lines.append(f"{c:14s} {len(rs):8d} {ms:9.2f} {pct:7.1f} {fl / ms / 1e9:8.2f} "
                     f"{min(r[PCT] for r in rs):6.1f} {max(r[PCT] for r in rs):6.1f}")
    lines.append("")
    lines.append("representative launches (last quarter of the list = the timed step):")
    for c, rs in byc.items():
        tail = rs[len(rs) * 3 // 4:]
        if not tail:
            continue
        for tag, r in (("early", tail[0]), ("middle", tail[len(tail) // 2]), ("late", tail[-1])):
            t = r["gpu__time_duration.sum"]
            lines.append(f"  {c:14s} {tag:6s} {t * 1e3:9.1f} us  DMMA {r[PCT]:5.1f}%  "
                         f"{r[INST] * 512 / t / 1e9:6.2f} TFLOP/s")
    txt = "\n".join(lines)
    print(txt)
    if out:
        open(out, "w").write(txt + "\n")


if __name__ == "__main__":
    main(*sys.argv[1:])
