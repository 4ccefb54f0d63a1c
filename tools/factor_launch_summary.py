"""Summarise an ncu launch list of tools/factor_times.py (second vb_factor): per-kernel time, share
and DMMA-pipe activity.  python tools/factor_launch_summary.py gpurun_out/factor_launches.csv"""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    L = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        d = L.setdefault(r[idi], {"k": r[ki]})
        d[r[mi]] = r[vi]
    items = list(L.values())
    idx = [i for i, d in enumerate(items) if d["k"].startswith("assemble_kernel")]
    it = items[idx[-1]:]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for d in it:
        n = d["k"].split("(")[0].replace("void ", "")
        n = n if "gemm2" in n else n.split("<")[0]
        t = float(d["gpu__time_duration.sum"].replace(",", "")) / 1e3
        dm = float(d.get("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed", "0").replace(",", ""))
        a = agg[n]
        a[0] += 1
        a[1] += t
        a[2] += t * dm
    tot = sum(a[1] for a in agg.values())
    gem = sum(a[1] for n, a in agg.items() if "gemm2" in n)
    gdm = sum(a[2] for n, a in agg.items() if "gemm2" in n)
    print("vb_factor (config 5, second call), ncu launch list: kernel total %.1f ms; DMMA GEMMs %.1f ms (%.0f%%), "
          "time-weighted DMMA-pipe active %.1f%%" % (tot / 1e3, gem / 1e3, 100 * gem / tot, gdm / gem))
    print("%-70s %5s %9s %6s %5s" % ("kernel", "n", "ms", "share", "dmma%"))
    for n, a in sorted(agg.items(), key=lambda x: -x[1][1])[:24]:
        print("%-70s %5d %9.1f %5.1f%% %5.1f" % (n[:70], a[0], a[1] / 1e3, 100 * a[1] / tot, a[2] / a[1] if a[1] else 0))


if __name__ == "__main__":
    main(sys.argv[1])
