"""Key metrics of every kernel in an .ncu-rep (details page) -> text table.

    python tools/ncu_summary.py gpurun_out/x.ncu-rep [more.ncu-rep ...]
"""
import csv, io, subprocess, sys

WANT = ["Duration", "SM Frequency", "DRAM Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Warp Cycles Per Issued Instruction", "Registers Per Thread", "Dynamic Shared Memory Per Block",
        "Achieved Occupancy", "L2 Hit Rate", "L1/TEX Hit Rate", "Grid Size", "Block Size"]


def summary(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    iid, ik, im, iu, iv = (hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    kern = {}
    for r in rows[1:]:
        if len(r) <= iv or r[im] not in WANT:
            continue
        d = kern.setdefault(r[iid], {"name": r[ik]})
        d.setdefault(r[im], f"{r[iv]} {r[iu]}".strip())
    lines = [f"# {path}"]
    for i, d in kern.items():
        lines.append(f"[{i}] {d['name'][:150]}")
        for k in WANT:
            if k in d:
                lines.append(f"    {k:38s} {d[k]}")
    return "\n".join(lines)


if __name__ == "__main__":
    print("\n".join(summary(p) for p in sys.argv[1:]))
