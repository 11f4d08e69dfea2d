#!/usr/bin/env python
"""Summarise ncu captures for profiles/ (run here, no GPU needed).

usage: python scripts/ncu_summary.py <dir with unit_<cfg>.ncu-rep / launches_<cfg>.csv> <out.md>

For every config found: the top metrics of the --set full capture of the
SpMV kernel (duration, DRAM bytes -> traffic per launch, DRAM / L2 / SM
throughput %, occupancy, stall reasons) and, from the --metrics
gpu__time_duration.sum launch list, the SpMV kernel's share of the device
time of one timed bench step (cold-cache, serialised: compare shares).
"""
import csv
import glob
import io
import json
import os
import re
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum",
]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6,
        "usecond": 1e-6, "nsecond": 1e-9, "ms": 1e-3, "msecond": 1e-3}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {}
        for i, k in enumerate(h):
            d[k] = (v[i], units[i])
        res.append(d)
    return res


def num(d, k):
    v, u = d.get(k, ("", ""))
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return None
    return x * UNIT.get(u, 1.0)


def launch_shares(path):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(io.StringIO("".join(lines))):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            rows.append((r["Kernel Name"], float(r["Metric Value"].replace(",", "")) *
                         UNIT.get(r["Metric Unit"], 1.0)))
    return rows


def main():
    d, out = sys.argv[1], sys.argv[2]
    lines = [f"# ncu summary: {d}", ""]
    traffic = {}
    for rep in sorted(glob.glob(os.path.join(d, "unit_*.ncu-rep"))):
        cfg = re.sub(r"^unit_|\.ncu-rep$", "", os.path.basename(rep))
        lines.append(f"## {cfg}: `ncu --set full` of the SpMV kernel")
        for i, k in enumerate(raw(rep)):
            name = k.get("Kernel Name", ("?", ""))[0]
            lines.append(f"### launch {i}: {name}")
            for key in KEYS:
                if key in k:
                    lines.append(f"- {key}: {k[key][0]} {k[key][1]}")
            rd, wr = num(k, "dram__bytes_read.sum"), num(k, "dram__bytes_write.sum")
            if rd is not None and wr is not None:
                # one SpMV = the captured launches of one step: sum them
                traffic[cfg] = traffic.get(cfg, 0) + int(rd + wr)
                lines.append(f"- traffic (read+write): {int(rd + wr)} B")
            l2s = num(k, "lts__t_sectors_srcunit_tex_op_read.sum")
            if l2s is not None and rd:
                # L1 -> L2 read sectors (32 B) per DRAM byte read: > 1 means
                # the kernel's reads are served from L2 more than once (the
                # remainder's x gathers: 4 useful bytes per 32-byte sector)
                lines.append(f"- L2 read sectors x 32 B / DRAM bytes read: {l2s * 32 / rd:.2f}")
            stalls = sorted(((float(v[0]), kk) for kk, v in k.items()
                             if kk.startswith("smsp__pcsamp_warps_issue_stalled_")
                             and not kk.endswith("_not_issued") and v[0] not in ("",)),
                            reverse=True)[:6]
            if stalls:
                lines.append("- top stall samples: " + ", ".join(
                    f"{kk.replace('smsp__pcsamp_warps_issue_stalled_', '')}={int(v)}"
                    for v, kk in stalls))
        lines.append("")
    for lf in sorted(glob.glob(os.path.join(d, "launches_*.csv"))):
        cfg = re.sub(r"^launches_|\.csv$", "", os.path.basename(lf))
        rows = launch_shares(lf)
        uk = [t for n, t in rows if "unit_kernel" in n]
        lines.append(f"## {cfg}: launch list ({len(rows)} launches)")
        med = lambda v: sorted(v)[len(v) // 2] if v else 0.0  # noqa: E731
        if uk:
            # one SpMV step = one unit_kernel launch (+ the L2 scrub, not ours)
            timed = [t for n, t in rows if "unit_kernel" in n or "elementwise" in n or
                     "reduce" in n]
            lines.append(f"- unit_kernel launches: {len(uk)}, median {med(uk) * 1e6:.2f} us; "
                         f"share of the device time of a timed step (SpMV + L2 scrub): "
                         f"{sum(uk) / max(sum(timed), 1e-12):.2f}")
        tot = {}
        for n, t in rows:
            short = n.split("(")[0]
            tot[short] = tot.get(short, 0.0) + t
        for n, t in sorted(tot.items(), key=lambda kv: -kv[1])[:8]:
            lines.append(f"- {n}: {t * 1e6:.1f} us total")
        lines.append("")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    tj = os.path.join(os.path.dirname(out), "traffic.json")
    old = json.load(open(tj)) if os.path.exists(tj) else {}
    old.update(traffic)
    json.dump(old, open(tj, "w"), indent=1, sort_keys=True)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
