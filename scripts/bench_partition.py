#!/usr/bin/env python
"""Time the GPU partitioner (sable_partition_grid, Alg. 1) at a
config's full size with device-resident CSR input; one JSON line per config.

usage: python scripts/bench_partition.py [c2 c3 c4] [--reps R]
Traffic model: the row pass reads rowptr (8 B/row) and every
column index about twice (row i as u, row i+1 as v: 8 B/nnz); the column pass
sorts nnz 64-bit keys (radix passes, not counted) and repeats the row pass on
A^T -- algorithmic bytes = 2 * (8 n + 8 nnz)."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import gen  # noqa: E402
from paper_2407_00829_b200 import sable  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    reps = 5
    if "--reps" in sys.argv:
        reps = int(sys.argv[sys.argv.index("--reps") + 1])
    for name in args or ["c2"]:
        t0 = time.time()
        s = gen.make(name)
        gen_s = time.time() - t0
        o = np.lexsort((s.J, s.I))
        rp = np.zeros(s.nrows + 1, np.int64)
        np.cumsum(np.bincount(s.I, minlength=s.nrows), out=rp[1:])
        rpd = torch.from_numpy(rp).cuda()
        cid = torch.from_numpy(s.J[o].astype(np.int32)).cuda()
        torch.cuda.synchronize()
        out = None
        ts = []
        for r in range(reps + 1):
            t = time.perf_counter()
            out = sable.partition_grid(rpd, cid, s.ncols, 1, 2, True)
            torch.cuda.synchronize()
            if r:
                ts.append(time.perf_counter() - t)
        ms = 1e3 * float(np.median(ts))
        nnz = int(len(s.I))
        alg = 2 * (8 * (s.nrows + s.ncols) + 8 * nnz)
        print(json.dumps({"bench": "partition_grid", "config": name, "nrows": s.nrows,
                          "nnz": nnz, "t": "1/2", "shifts": True, "ms": round(ms, 3),
                          "gnnz_per_s": round(nnz / ms / 1e6, 3),
                          "alg_gbs": round(alg / ms / 1e6, 1),
                          "nbrows": len(out[0]) - 1, "nbcols": len(out[1]) - 1,
                          "gen_s": round(gen_s, 1)}), flush=True)


if __name__ == "__main__":
    main()
