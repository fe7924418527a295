"""Summarise an ncu --set full report (.ncu-rep) as JSON: the kernel, its duration,
DRAM traffic, grid / occupancy and issue metrics.  usage: python scripts/ncu_summary.py REP [ID]"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]

rep = sys.argv[1]
idx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units, vals = rows[0], rows[1], rows[2 + idx]
print(json.dumps({k: (vals[h.index(k)] + (" " + units[h.index(k)] if units[h.index(k)] else "")).strip()
                  for k in KEYS if k in h}, indent=1))
