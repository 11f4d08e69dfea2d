"""Per-source-line warp instructions and stall samples of one kernel from an
ncu report (ncu --page source --print-source cuda,sass).
usage: ncu_lines.py <report.ncu-rep> [top_n] [norm]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
norm = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
ins, smp, src = defaultdict(int), defaultdict(int), {}
cur = None
fname = ""
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 2 and r[0] == "Line No":
        hdr = r
        ie = hdr.index("Instructions Executed")
        isamp = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) < len(hdr) - 1:
        continue
    if r[0]:
        cur = (fname, int(r[0]))
        src[cur] = r[1].strip()[:80]
    elif cur is not None:
        try:
            ins[cur] += int(float(r[ie] or 0))
            smp[cur] += int(float(r[isamp] or 0))
        except ValueError:
            pass
ti, ts = sum(ins.values()), sum(smp.values())
print(f"total warp instructions {ti} ({ti / norm:.2f} per norm unit), stall samples {ts}")
for ln in sorted(ins, key=lambda k: -ins[k])[:top]:
    print(f"{ln[0][:12]:12s}:{ln[1]:4d} ins {ins[ln]:10d} ({100 * ins[ln] / max(ti, 1):5.1f}%) samp {smp[ln]:7d} "
          f"({100 * smp[ln] / max(ts, 1):5.1f}%)  {src.get(ln, '')}")
