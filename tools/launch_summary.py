"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: launches and total/mean time per kernel."""
import collections
import csv
import sys


def summarise(path):
    hdr, agg = None, collections.defaultdict(lambda: [0, 0.0])
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(d["Metric Unit"], 1e-6)
        k = d["Kernel Name"].split("(")[0]
        agg[k][0] += 1
        agg[k][1] += v * scale
    total = sum(t for _, t in agg.values())
    lines = [f"{'kernel':48s} {'launches':>8s} {'total ms':>10s} {'mean ms':>10s} {'share':>6s}"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{k[:48]:48s} {c:8d} {t:10.3f} {t / c:10.4f} {t / total:6.1%}")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
