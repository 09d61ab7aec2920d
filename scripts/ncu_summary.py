"""Key metrics of ncu --set full reports (dev tool): python scripts/ncu_summary.py TAG=report.ncu-rep ..."""
import csv
import io
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "sm__cycles_active.avg", "gpc__cycles_elapsed.max",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "launch__registers_per_thread", "launch__grid_size", "sm__cycles_elapsed.avg.per_second"]
for arg in sys.argv[1:]:
    tag, path = arg.split("=", 1)
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        print(f"[{tag}] no data ({path})")
        continue
    h = rows[0]
    for r in rows[2:]:
        d = dict(zip(h, r))
        print(f"\n[{tag}] {d.get('Kernel Name', '')[:100]}")
        for m in METRICS:
            if m in d:
                print(f"  {m:72s} {d[m]}")
