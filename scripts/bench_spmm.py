#!/usr/bin/env python
"""Time sable_spmm (Y = A X, k right-hand sides) against k
separate sable_spmv calls at a config's full size; L2 flushed before each
timed call, CUDA events on the launching stream.  One JSON line per (config, k).
k = 1..8 run on the CUDA cores, k = 16..128 (fp32) on the tensor cores.
usage: python scripts/bench_spmm.py [c2 c4 ...]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import gen  # noqa: E402
from paper_2407_00829_b200 import sable  # noqa: E402

scrub = torch.empty(128 << 20, dtype=torch.float32, device="cuda")
sink = torch.empty((), dtype=torch.float32, device="cuda")


def timed(fn, reps=20):
    st = torch.cuda.current_stream()
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        scrub.zero_()
        torch.sum(scrub, dim=0, out=sink)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


for name in sys.argv[1:] or ["c2"]:
    s = gen.make(name)
    inp = s.vbr_input("rect")
    arrays = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in inp.items()
              if isinstance(v, np.ndarray)}
    A = sable.VbrMatrix(arrays, s.nrows, s.ncols, delta=s.delta)
    del arrays
    tdt = torch.float64 if s.dtype == np.float64 else torch.float32
    ks = (1, 2, 4, 8, 16, 32, 64, 128) if tdt == torch.float32 else (1, 2, 4, 8)
    for k in ks:
        X = torch.randn((s.ncols, k), dtype=tdt, device="cuda")
        Y = torch.empty((s.nrows, k), dtype=tdt, device="cuda")
        xcols = [X[:, j].contiguous() for j in range(k)]
        ys = [torch.empty(s.nrows, dtype=tdt, device="cuda") for _ in range(k)]
        t_mm = timed(lambda: A.spmm(X, Y))

        def kspmv():
            for j in range(k):
                A.spmv(xcols[j], ys[j])
        t_k = timed(kspmv, reps=5 if k > 8 else 20)
        flops = 2.0 * s.nnz * k
        print(json.dumps({"bench": "spmm", "config": name, "k": k, "spmm_ms": round(t_mm, 4),
                          "k_spmv_ms": round(t_k, 4), "spmm_gflops": round(flops / t_mm / 1e6, 1),
                          "k_spmv_gflops": round(flops / t_k / 1e6, 1),
                          "speedup": round(t_k / t_mm, 3),
                          "path": "tensor cores (tcgen05 kind::tf32, 3xTF32)" if k >= 16 else
                                  "CUDA cores (unit_kernel, k accumulators)",
                          "bytes_alg_once": A.info["bytes_alg"],
                          "alg_gbs_spmm": round((A.info["bytes_alg"] +
                                                 (k - 1) * (s.ncols + s.nrows) *
                                                 (8 if tdt == torch.float64 else 4)) / t_mm / 1e6, 1)}),
              flush=True)
    A.close()
