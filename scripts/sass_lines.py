#!/usr/bin/env python
"""Per-source-line instruction counts and stall samples of a kernel from an
ncu --page source CSV (SASS view) joined with nvdisasm -g line info.
usage: sass_lines.py <ncu_source.csv> <nvdisasm -g output> <kernel-substring> [n_items]"""
import csv
import re
import sys
from collections import defaultdict

src, dis, kname = sys.argv[1], sys.argv[2], sys.argv[3]
norm = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
# offset -> line for the kernel
off2line, cur, inside = {}, None, False
for ln in open(dis):
    if ln.startswith(".text.") and kname in ln:
        inside = True
        continue
    if inside and ln.startswith(".text.") and kname not in ln:
        break
    if not inside:
        continue
    m = re.search(r'line (\d+)', ln)
    if m and "## File" in ln:
        cur = int(m.group(1))
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/', ln)
    if m:
        off2line[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(src)))
h = rows[1]
data = rows[2:]
ia, ie, ist = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
base = int(data[0][ia], 16)
per_e, per_s = defaultdict(int), defaultdict(int)
for r in data:
    off = int(r[ia], 16) - base
    line = off2line.get(off)
    per_e[line] += int(r[ie] or 0)
    per_s[line] += int(r[ist] or 0)
te, ts = sum(per_e.values()), sum(per_s.values())
print(f"total warp instructions {te} ({te / norm:.1f} per unit), samples {ts}")
lines = open(re.sub(r'^.*?File "', '', '')) if False else None
for line in sorted(per_e, key=lambda k: (k is None, k)):
    if per_e[line] > 0.005 * te or per_s[line] > 0.01 * ts:
        print(f"line {line}: instr {per_e[line]:>10} ({100 * per_e[line] / te:4.1f}%)  {per_e[line] / norm:7.1f}/unit  samples {per_s[line]:>6} ({100 * per_s[line] / ts:4.1f}%)")
