#!/usr/bin/env python
"""Per-shard SpMV times of the row partition on ONE GPU (no collective, no
kernel waits on another): for P in 1, 2, 4, 8 the P sharded handles (rank r of
P, sable_shard_bounds by stored entries) are created one after the other and
each shard's SpMV is timed alone.  The compute part of the multi-GPU step is
the slowest shard; with the exchange (n * s_v * (P-1)/P bytes per GPU per
step) it gives the projected strong-scaling curve this pool cannot measure.

usage: python scripts/shard_balance.py [--config c5] [--out profiles/x.json]
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
from paper_2407_00829_b200 import sable  # noqa: E402

NVLINK_GBS = 900.0  # per direction, /opt/skills/guides (nominal, not measured here)


def time_spmv(A, x, y, flush, reps=20):
    scrub = time_spmv.scrub
    ev = []
    for i in range(reps + 3):
        if flush:
            scrub.zero_()
            scrub.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        A.spmv(x, y)
        b.record()
        ev.append((a, b))
    torch.cuda.synchronize()
    return statistics.mean(a.elapsed_time(b) for a, b in ev[3:])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    s = gen.make(args.config)
    arrays = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda()
              for k, v in s.vbr_input("rect").items() if isinstance(v, np.ndarray)}
    x = torch.from_numpy(s.x).cuda()
    time_spmv.scrub = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    sv = 8 if s.dtype == np.float64 else 4
    res = {"config": args.config, "n": s.nrows, "nnz": int(s.nnz), "P": {}}
    t1 = None
    for P in (1, 2, 4, 8):
        shards = []
        for r in range(P):
            A = sable.VbrMatrix(arrays, s.nrows, s.ncols, delta=s.delta, rank=r, world=P)
            i = A.info
            nloc = i["row_end"] - i["row_begin"]
            y = torch.empty(nloc, dtype=x.dtype, device="cuda")
            kept = time_spmv(A, x, y, False)
            fl = time_spmv(A, x, y, True)
            shards.append({"rank": r, "rows": int(nloc), "bytes_alg": int(i["bytes_alg"]),
                           "ms_l2_kept": round(kept, 5), "ms_l2_flushed": round(fl, 5)})
            A.close()
        mx = max(q["ms_l2_kept"] for q in shards)
        mean = statistics.mean(q["ms_l2_kept"] for q in shards)
        if P == 1:
            t1 = mx
        egress_ms = s.ncols * sv * (P - 1) / P / (NVLINK_GBS * 1e9) * 1e3
        res["P"][str(P)] = {
            "shards": shards, "max_ms": round(mx, 5), "mean_ms": round(mean, 5),
            "imbalance_max_over_mean": round(mx / mean, 4),
            "compute_speedup_vs_P1": round(t1 / mx, 3),
            "exchange_egress_ms_at_nominal_nvlink": round(egress_ms, 5),
            "projected_speedup_overlapped": round(t1 / max(mx, egress_ms), 3),
            "projected_speedup_serialized": round(t1 / (mx + egress_ms), 3),
        }
        print(P, json.dumps({k: v for k, v in res["P"][str(P)].items() if k != "shards"}), flush=True)
    if args.out:
        json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
