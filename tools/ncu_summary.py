"""Text summaries of ncu output for profiles/ (development tool).

  python tools/ncu_summary.py launches LAUNCHES.csv      # per-kernel share of a launch list
  python tools/ncu_summary.py report REPORT.ncu-rep      # key metrics of a --set full capture
"""

import collections
import csv
import io
import subprocess
import sys

REPORT_METRICS = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[hi]
    col = {h: i for i, h in enumerate(hdr)}
    per = collections.defaultdict(lambda: [0, 0.0])
    total = 0.0
    unit = None
    for r in rows[hi + 1:]:
        if len(r) != len(hdr) or r[col["Metric Name"]] != "gpu__time_duration.sum":
            continue
        unit = r[col["Metric Unit"]]
        v = float(r[col["Metric Value"]].replace(",", ""))
        name = r[col["Kernel Name"]].split("(")[0]
        per[name][0] += 1
        per[name][1] += v
        total += v
    print(f"{sum(c for c, _ in per.values())} launches, total {total:.0f} {unit} (serialised, cold-cache)")
    print(f"{'kernel':60s} {'count':>6s} {'total':>12s} {'avg':>10s} {'share':>6s}")
    for name, (c, v) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        print(f"{name[:60]:60s} {c:6d} {v:12.0f} {v / c:10.0f} {100 * v / total:5.1f}%")


def report(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    for r in rows[2:]:
        print(f"== {r[col['Kernel Name']][:100]}")
        for m in REPORT_METRICS:
            if m in col:
                print(f"  {m:66s} {r[col[m]]:>16s} {units[col[m]]}")


if __name__ == "__main__":
    {"launches": launches, "report": report}[sys.argv[1]](sys.argv[2])
