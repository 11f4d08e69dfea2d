#!/usr/bin/env python
"""Probe one calibration matrix: dense-arm time vs area and executor knobs.
usage: python scripts/calib_probe.py h w fill [area_log2 ...]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen.calib as gc  # noqa: E402
from paper_2407_00829_b200 import sable  # noqa: E402

scrub = torch.empty(128 << 20, dtype=torch.float32, device="cuda")
sink = torch.empty((), dtype=torch.float32, device="cuda")


def timeit(A, x, y, reps=15, flush=True):
    st = torch.cuda.current_stream()
    for _ in range(3):
        A.spmv(x, y)
    ts = []
    for _ in range(reps):
        if flush:
            scrub.zero_()
            torch.sum(scrub, dim=0, out=sink)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        A.spmv(x, y)
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return sorted(ts)[len(ts) // 2]


h, w, f = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
for lg in [int(a) for a in sys.argv[4:]] or [23]:
    s = gc.shape_grid(h, w, f, area=1 << lg)
    inp = s.vbr_input("all_vbr")
    arrays = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in inp.items()
              if isinstance(v, np.ndarray)}
    x = torch.from_numpy(s.x).cuda()
    y = torch.empty(s.nrows, dtype=torch.float32, device="cuda")
    for delta in [int(d) for d in os.environ.get("PROBE_DELTAS", "0,101").split(",")]:
        A = sable.VbrMatrix(arrays, s.nrows, s.ncols, delta=delta)
        i = A.info
        r = dict(h=h, w=w, fill=f, area_log2=lg, delta=delta, arch=os.environ.get("SABLE_ARCH", "1"),
                 us=round(timeit(A, x, y), 2), us_noflush=round(timeit(A, x, y, flush=False), 2),
                 n_items=i["n_items"], n_chunks=i["n_chunks"], n_tasks=i["n_tasks"],
                 grid=i["exec_grid"], groups=i["n_groups"], rem_packets=i["rem_packets"],
                 bytes_alg=i["bytes_alg"])
        print(json.dumps(r), flush=True)
        A.close()
