"""Per-class DRAM traffic per launch from an ncu launch list.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --csv --log-file launches.csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline
    python tools/traffic_from_launches.py launches.csv profiles/traffic.json

Kernel -> library profiling class (paper_1907_01063_b200.PROFILE_KINDS):
  gemm_dmma_kernel<..., 1, 1, 1> / gemm_tma_kernel<..., 1, 1, 1>   syrk      (MODE_LOWER)
  gemm_tma_fused_kernel<..., 1, 0>                                 adj_gemm  (fused: [R_bar; B_bar] update + next C_bar D^-1)
  gemm_tma_kernel<..., 1, 0, 0>                                    adj_gemm / trmm (unfused update; C_bar D^-1)
  gemm_tma_kernel<..., 0, 0, 2> / gemm_dmma_kernel<..., 0, 0, 2>   splitk
  gemm_tma_kernel<..., 1, 1, 0>                                    lookahead (main-stream column update)
  gemm_dmma_kernel<..., 1, 1, 0>                                   panel_gemm (side stream)
"""
import collections
import csv
import json
import re
import sys

UNITS = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
         "%": 1.0, "inst": 1.0, "cycle": 1.0, "": 1.0}


def classify(name: str):
    if "gemm_tma_fused_kernel" in name:  # the adjoint's update of step s + C_bar D^-1 of step s+1
        return "adj_gemm"
    m = re.search(r"(gemm_dmma_kernel|gemm_tma_kernel)<.*>, (\d), (\d), (\d)(?:, (\d))?>", name)
    if not m:
        return re.match(r"(?:void )?(?:\w+::)*(\w+)", name).group(1)
    kern, a, b, mode, fused = m.group(1), m.group(2), m.group(3), m.group(4), m.group(5)
    key = (a, b, mode)
    if fused == "1":  # the adjoint's update of step s + C_bar D^-1 of step s+1 (adj_update_fused_trmm)
        return "adj_gemm"
    if mode == "1":
        return "syrk"
    if mode == "2":
        return "splitk"
    if key == ("1", "0", "0"):
        return "adj_gemm" if kern == "gemm_tma_kernel" else "trmm"
    if key == ("1", "1", "0"):
        # TMA: main-stream lookahead column; one-tile-per-CTA: side-stream panel
        # GEMMs (in-panel lookahead, TRSM cross update)
        return "lookahead" if kern == "gemm_tma_kernel" else "panel_gemm"
    return kern


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
        rec[d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) * UNITS[d["Metric Unit"]]
    agg = collections.defaultdict(lambda: {"launches": 0, "ms": 0.0, "dram_bytes": 0.0})
    seq = list(recs.values())
    classes = [classify(r["name"]) for r in seq]
    # the adjoint's C_bar D^-1 product and its merged rank-256 update are the same
    # TMA instantiation; per step the order is C_bar D^-1 -> split-K -> ... ->
    # update, so a (1, 0, 0) launch whose next GEMM launch is split-K is the former
    gemm_like = {"adj_gemm", "splitk", "syrk", "lookahead", "panel_gemm"}
    for i, c in enumerate(classes):
        if c != "adj_gemm" or "gemm_tma_fused_kernel" in seq[i]["name"]:  # fused launches stay adj_gemm
            continue
        nxt = next((classes[j] for j in range(i + 1, len(classes)) if classes[j] in gemm_like), None)
        if nxt == "splitk":
            classes[i] = "trmm"
    for rec, c in zip(seq, classes):
        a = agg[c]
        a["launches"] += 1
        a["ms"] += rec.get("gpu__time_duration.sum", 0.0)
        a["dram_bytes"] += rec.get("dram__bytes_read.sum", 0.0) + rec.get("dram__bytes_write.sum", 0.0)
    res = {"source": path, "note": "ncu launch list (cold cache, serialised); dram bytes = read + write",
           "classes": {}}
    for c, a in sorted(agg.items(), key=lambda x: -x[1]["ms"]):
        res["classes"][c] = {"launches": a["launches"], "ms_total": round(a["ms"], 3),
                             "dram_bytes_per_launch": a["dram_bytes"] / a["launches"]}
        print(f"{c:28s} {a['launches']:6d} {a['ms']:10.2f} ms  {a['dram_bytes'] / a['launches'] / 1e6:10.2f} MB/launch")
    if out:
        json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:])
