"""Top SASS lines by warp-stall samples (with their main stall reasons) from
`ncu -i X --page source --csv --print-source sass` output, plus the kernel's
stall-reason totals.  usage: python scripts/ncu_hot.py file.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, ist = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
reasons = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
data, tot_r = [], {}
for r in rows[2:]:
    try:
        s = int(r[ist] or 0)
    except (ValueError, IndexError):
        continue
    rs = {hdr[i][6:]: int(r[i] or 0) for i in reasons}
    for k, v in rs.items():
        tot_r[k] = tot_r.get(k, 0) + v
    data.append((s, r[ia], r[isrc], rs))
tot = sum(d[0] for d in data)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print("total samples", tot, " by reason:",
      ", ".join(f"{k}={v}" for k, v in sorted(tot_r.items(), key=lambda kv: -kv[1]) if v))
for s, a, src, rs in sorted(data, key=lambda d: -d[0])[:n]:
    top = ", ".join(f"{k}={v}" for k, v in sorted(rs.items(), key=lambda kv: -kv[1])[:2] if v)
    print(f"{s:7d} {100.0 * s / max(tot, 1):5.1f}%  {a[-5:]}  {src.strip()[:60]:60s} {top}")
