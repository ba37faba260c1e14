"""Aggregate an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv --log-file L ...`)
per kernel: launches, total ms, mean us, share of the listed time.

    python tools/launch_summary.py gpurun_out/launches_r02b_cfg4.csv > profiles/launches_r02b_cfg4.csv"""
import csv
import sys
from collections import OrderedDict

SCALE = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}


def main():
    rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
    h = rows[0]
    ik, im, iu, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    agg = OrderedDict()
    for r in rows[1:]:
        if r[im] != "gpu__time_duration.sum":
            continue
        ms = float(r[iv].replace(",", "")) * SCALE.get(r[iu], 1.0)
        k = agg.setdefault(r[ik], [0, 0.0])
        k[0] += 1
        k[1] += ms
    tot = sum(v[1] for v in agg.values())
    w = csv.writer(sys.stdout, lineterminator="\n")
    w.writerow(["kernel", "launches", "total_ms", "mean_us", "share"])
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        w.writerow([k, n, f"{ms:.4f}", f"{1e3 * ms / n:.2f}", f"{ms / tot:.4f}"])


if __name__ == "__main__":
    main()
