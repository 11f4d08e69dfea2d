"""Key metrics of the first kernel in an ncu report (raw page)."""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, v = rows[0], rows[-1]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__inst_executed.avg.per_cycle_active", "lts__t_sectors.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex__t_sector_hit_rate.pct"]
for i, h in enumerate(hdr):
    if h in keys:
        print(f"{h:55s} {v[i]}")
    elif "pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued"):
        try:
            if float(v[i]) > 0.03 * 1e9 or float(v[i]) > 150:
                print(f"{h:55s} {v[i]}")
        except ValueError:
            pass
