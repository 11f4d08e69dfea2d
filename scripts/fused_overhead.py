#!/usr/bin/env python
"""Kernel-side cost of the fused exchange epilogue on ONE GPU: for every shard
of P ranks, the step with the y rows stored to P - 1 extra destinations (other
buffers of the same GPU standing in for the peers' x_next: HBM writes here,
NVLink stores on a multi-GPU box) against the plain step (no peers).  The
ranks run one at a time; nothing waits on anything.

usage: python scripts/fused_overhead.py [--config c5] [--world 8] [--out f.json]
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


def timed(fn, reps=30):
    ev = []
    for _ in range(reps + 5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        ev.append((a, b))
    torch.cuda.synchronize()
    return statistics.mean(a.elapsed_time(b) for a, b in ev[5:])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    s = gen.make(args.config)
    arrays = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda()
              for k, v in s.vbr_input("rect").items() if isinstance(v, np.ndarray)}
    x = torch.from_numpy(s.x).cuda()
    P = args.world
    xa = [x.clone() for _ in range(P)]
    xb = [torch.empty_like(x) for _ in range(P)]
    plain_next = torch.empty_like(x)
    rows = []
    for r in range(P):
        A = sable.VbrMatrix(arrays, s.nrows, s.ncols, delta=s.delta, rank=r, world=P)
        # plain step of a world-P handle needs a registration too (no communicator here):
        # zero peers = the SpMV written into x_next's local rows only
        A.comm_set_peers(xa[r], plain_next, [], [])
        t_plain = timed(lambda: A.spmv_allgather(xa[r], plain_next))
        others = [q for q in range(P) if q != r]
        A.comm_set_peers(xa[r], xb[r], [xa[q] for q in others], [xb[q] for q in others])
        t_fused = timed(lambda: A.spmv_allgather(xa[r], xb[r]))
        i = A.info
        rows.append({"rank": r, "rows": int(i["row_end"] - i["row_begin"]),
                     "ms_plain": round(t_plain, 5), "ms_fused_local_peers": round(t_fused, 5)})
        print(rows[-1], flush=True)
        A.close()
    res = {"config": args.config, "world": P, "shards": rows,
           "max_ms_plain": max(q["ms_plain"] for q in rows),
           "max_ms_fused_local_peers": max(q["ms_fused_local_peers"] for q in rows)}
    print(json.dumps({k: v for k, v in res.items() if k != "shards"}))
    if args.out:
        json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
