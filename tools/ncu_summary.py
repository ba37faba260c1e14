"""Summarise `ncu --set full` reports (gpurun_out/*.ncu-rep) into profiles/ncu_summary_<round>.json.

    python tools/ncu_summary.py r01 cfg4=gpurun_out/ncu_gram_cfg4.ncu-rep cfg5=... (or a --page raw --csv export)

Per report: kernel name, duration, DRAM bytes read+write (the `traffic` of bench.py's roofline
object), DMMA pipe utilisation, issue/stall ratios. Existing entries of the same file are kept.
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active": "dmma_pipe_active_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_active_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "lts__t_bytes.sum": "l2_bytes",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "nsecond": 1e-9,
         "Hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "KHz": 1e3, "MHz": 1e6, "GHz": 1e9}


def summarise(path):
    # a report, or its `ncu -i <rep> --page raw --csv` export (summarised on the GPU box)
    out = open(path).read() if path.endswith(".csv") else \
        subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    res = {"kernel": v[h.index("Kernel Name")], "report": os.path.basename(path)}
    stalls = {}
    for i, n in enumerate(h):
        try:
            x = float(v[i].replace(",", ""))
        except ValueError:
            continue
        if n in KEYS:
            res[KEYS[n]] = x * SCALE.get(u[i], 1.0)
        if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio") and x > 0.05:
            stalls[n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = x
    res["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
    res["dram_bytes_per_launch"] = res.get("dram_read", 0.0) + res.get("dram_write", 0.0)
    return res


def main():
    tag = sys.argv[1]
    dst = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                       f"ncu_summary_{tag}.json")
    data = json.load(open(dst)) if os.path.exists(dst) else {}
    for arg in sys.argv[2:]:
        name, path = arg.split("=", 1)
        data[name] = summarise(path)
    json.dump(data, open(dst, "w"), indent=1, sort_keys=True)
    for k, r in data.items():
        print(k, r["kernel"][:60], f"{r.get('duration', 0) * 1e3:.3f} ms", f"DRAM {r['dram_bytes_per_launch'] / 1e9:.2f} GB",
              f"DMMA {r.get('dmma_pipe_active_pct', 0):.1f}%")


if __name__ == "__main__":
    main()
