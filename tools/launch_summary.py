"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        if mi is not None and r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        agg[name][0] += 1
        agg[name][1] += v
        tot += v
    print("%-44s %6s %12s %10s %6s" % ("kernel", "n", "total_us", "avg_us", "share"))
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print("%-44s %6d %12.1f %10.2f %5.1f%%" % (k[:44], n, t, t / n, 100 * t / tot))
    print("total_us %.1f" % tot)


if __name__ == "__main__":
    main(sys.argv[1])
