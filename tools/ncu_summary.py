"""Summarise an `ncu --set full` report into JSON (per launch: duration, DRAM bytes, throughput
fractions, occupancy, L2 hit rate).

  python tools/ncu_summary.py report.ncu-rep ROLE0 ROLE1 ... > profiles/<name>.json
"""
import csv
import io
import json
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct"]


def main(path, roles):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    res = []
    for k, r in enumerate(rows[2:]):
        d = {"Kernel Name": r[head.index("Kernel Name")], "Grid Size": r[head.index("Grid Size")],
             "Block Size": r[head.index("Block Size")]}
        for m in METRICS:
            if m in head:
                i = head.index(m)
                d[m] = ("%s %s" % (r[i], units[i])).strip()
        if k < len(roles):
            d["role"] = roles[k]
        res.append(d)
    json.dump(res, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
