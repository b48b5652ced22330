"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel."""
import collections, csv, sys

def main(path, out=None):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        v *= {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}[d["Metric Unit"]]
        k = d["Kernel Name"].split("(")[0]
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v[1] for v in agg.values())
    lines = [f"# {path}: {sum(v[0] for v in agg.values())} launches, {tot:.2f} ms total (ncu, cold-cache, serialised)",
             f"{'kernel':48s} {'launches':>8s} {'ms':>10s} {'share':>7s} {'ms/launch':>10s}"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{k:48s} {v[0]:8d} {v[1]:10.2f} {100 * v[1] / tot:6.1f}% {v[1] / v[0]:10.4f}")
    txt = "\n".join(lines)
    print(txt)
    if out:
        open(out, "w").write(txt + "\n")

if __name__ == "__main__":
    main(*sys.argv[1:])
