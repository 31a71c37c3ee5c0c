"""Summarise one kernel of an `ncu --set full` report into profiles/ncu_summary.json.

usage: python tools/ncu_summarize.py REPORT.ncu-rep KEY "SOURCE DESCRIPTION" [ALGORITHMIC_BYTES] [KERNEL_SUBSTRING]
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = {
    "gpu_time_ms": ("gpu__time_duration.sum", 1),
    "dram_read_GB": ("dram__bytes_read.sum", 1e-9),
    "dram_write_GB": ("dram__bytes_write.sum", 1e-9),
    "tensor_pipe_active_pct": ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", 1),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", 1),
    "dram_throughput_pct": ("dram__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "grid": ("launch__grid_size", 1),
    "registers_per_thread": ("launch__registers_per_thread", 1),
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1,
        "ns": 1e-6, "us": 1e-3, "ms": 1,
        "second": 1e3}


def main():
    rep, key, source = sys.argv[1], sys.argv[2], sys.argv[3]
    algo = float(sys.argv[4]) if len(sys.argv) > 4 and float(sys.argv[4]) > 0 else None
    match = sys.argv[5] if len(sys.argv) > 5 else ""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kn = hdr.index("Kernel Name")
    vals = next(r for r in rows[2:] if match in r[kn])
    col = {}
    for i, h in enumerate(hdr):        # raw-page names may carry a section prefix ("TPC.TriageCompute.")
        col.setdefault(h, i)
        col.setdefault(h.split(".", 2)[-1] if h.count(".") >= 3 and h.split(".")[0].isupper() else h, i)
    d = {"source": source, "kernel": vals[col["Kernel Name"]][:120]}
    for k, (m, scale) in METRICS.items():
        if m not in col:
            continue
        try:
            v = float(vals[col[m]].replace(",", ""))
        except ValueError:
            continue
        v *= UNIT.get(units[col[m]], 1)
        d[k] = round(v * scale, 6)
    if "dram_read_GB" in d and "dram_write_GB" in d:
        d["dram_bytes_per_launch"] = (d["dram_read_GB"] + d["dram_write_GB"]) * 1e9
    if algo:
        d["algorithmic_bytes_per_launch"] = algo
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summary = json.load(open(path)) if os.path.exists(path) else {}
    summary[key] = d
    json.dump(summary, open(path, "w"), indent=1)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main()
