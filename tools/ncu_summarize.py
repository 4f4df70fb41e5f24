"""Summarise an ncu report (``--set full`` capture or a launch-list CSV) into
the text kept under profiles/.  Usage:
    python tools/ncu_summarize.py report.ncu-rep > profiles/rNN/<name>.txt
    python tools/ncu_summarize.py launches.csv   > profiles/rNN/<name>.txt
"""
import csv
import re
import subprocess
import sys
from collections import defaultdict

KEYS = re.compile(r"^(gpu__time_duration.sum|dram__bytes_read.sum|dram__bytes_write.sum|"
                  r"gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed|"
                  r"sm__throughput.avg.pct_of_peak_sustained_elapsed|"
                  r"smsp__issue_active.avg.pct_of_peak_sustained_active|"
                  r"sm__warps_active.avg.pct_of_peak_sustained_active|launch__registers_per_thread|"
                  r"smsp__inst_executed.sum|sm__cycles_elapsed.avg.per_second|"
                  r"sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active|"
                  r"sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active|"
                  r"sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active|"
                  r"launch__grid_size|launch__block_size|launch__shared_mem_per_block_dynamic|"
                  r"launch__occupancy_limit_registers|launch__occupancy_limit_shared_mem|Kernel Name)$")


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        for i, h in enumerate(hdr):
            if KEYS.match(h):
                print(f"{h} = {vals[i]} {units[i]}".rstrip())
        st = [(h, vals[i]) for i, h in enumerate(hdr)
              if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("per_issue_active.ratio")]
        st = sorted(((float(v or 0), h) for h, v in st), reverse=True)[:8]
        print("top stall reasons (warps per issue):",
              ", ".join(f"{h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={v:.2f}"
                        for v, h in st))
        print()


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    d = defaultdict(list)
    for r in rows[1:]:
        d[r[ki].split("(")[0][:60]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in d.values())
    print(f"{'launches':>8} {'mean_us':>10} {'share':>7}  kernel  (gpu__time_duration.sum, cold-cache, serialised)")
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        print(f"{len(v):8d} {sum(v) / len(v) / 1e3:10.2f} {sum(v) / tot * 100:6.2f}%  {k}")


if __name__ == "__main__":
    p = sys.argv[1]
    (rep if p.endswith(".ncu-rep") else launches)(p)
