#!/usr/bin/env python
"""Per-shape delta calibration and sparsity ablation on B200.

The paper decides dense-vs-sparse per block with a regression model trained
on CPU timings of its own machine (Fig. 7 heatmap); the
north star replaces it by the delta rule.  This script measures the B200
version of that heatmap with the library itself: for one matrix, the same
VBR input is inspected twice, with delta = 0 (every block a dense tile) and
delta = 101 (every block's non-zeros in the CSR remainder), and both SpMVs are
timed (CUDA events on the launching stream, L2 flushed before every SpMV).
speedup = t_csr / t_dense; the per-shape crossover delta* is the smallest
fill at which the dense tile is at least as fast -- the delta a user should
pass for blocks of that shape.  The Fig. 10 ablation
repeats the comparison on 10000^2 / 50x50 splits / 500 blocks over a
sparsity sweep.

The measured crossovers become a per-shape delta policy (reading R22,
sable_vbr_create_policy): one rule per measured shape over the shape bucket
around it (geometric midpoints between the measured sizes), delta = the
crossover (101 where the dense tile never wins), default delta 50.  The
64-aligned C4 stress case (gen c4a) is then timed and partitioned under
delta = 50 and under the policy.

usage: python scripts/calibrate.py [--quick] [--out profiles/r02_f2_calibration]
writes <out>.json, <out>.md and <out>_policy.json.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = [(4, 4), (8, 8), (16, 16), (32, 32), (64, 64), (128, 128), (4, 64), (64, 4),
          (16, 128), (128, 16)]
FILLS = [0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9, 1.0]
SPARSITIES = [0.0, 0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9, 0.95, 0.99]


def crossover(fills, speedups):
    """Smallest fill f such that the dense tile is at least as fast at f and at
    every larger measured fill (speedup >= 1 from there on); None if never."""
    best = None
    for f, s in sorted(zip(fills, speedups), reverse=True):
        if s >= 1.0:
            best = f
        else:
            break
    return best


def delta_of(fill):
    """delta (percent, integer) that makes exactly the fills >= `fill` dense."""
    return None if fill is None else int(round(100 * fill))


def size_buckets(sizes):
    """Inclusive [lo, hi] bucket of each measured size: edges at the
    geometric midpoints between consecutive sizes, open at both ends."""
    sizes = sorted(set(int(v) for v in sizes))
    out = {}
    for i, v in enumerate(sizes):
        lo = 1 if i == 0 else int((sizes[i - 1] * v) ** 0.5) + 1
        hi = 2 ** 31 - 1 if i == len(sizes) - 1 else int((v * sizes[i + 1]) ** 0.5)
        out[v] = (lo, hi)
    return out


def policy_from_heatmap(heat, default_delta=50):
    """Rules (h_min, h_max, w_min, w_max, delta) from the heatmap rows (dicts
    with h, w, delta_star): delta_star, or 101 where dense never won."""
    hb = size_buckets([r["h"] for r in heat])
    wb = size_buckets([r["w"] for r in heat])
    rules = []
    for r in heat:
        d = r["delta_star"] if r["delta_star"] is not None else 101
        rules.append((hb[r["h"]][0], hb[r["h"]][1], wb[r["w"]][0], wb[r["w"]][1], int(d)))
    return dict(delta=default_delta, min_area=0, rules=rules)


def monotone_violations(xs, ys, increasing=True, slack=0.1):
    """Adjacent pairs that move against the expected trend by more than `slack`
    (relative) -- timing noise below that is tolerated."""
    bad = []
    for (x0, y0), (x1, y1) in zip(zip(xs, ys), list(zip(xs, ys))[1:]):
        if increasing and y1 < y0 * (1 - slack):
            bad.append((x0, x1))
        if not increasing and y1 > y0 * (1 + slack):
            bad.append((x0, x1))
    return bad


def time_one(A, x, y, reps, flush):
    """Median us of `reps` SpMVs (CUDA events, L2 flushed before each)."""
    import torch
    st = torch.cuda.current_stream()
    for _ in range(3):
        A.spmv(x, y)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(reps)]
    for e0, e1 in ev:
        flush()
        e0.record(st)
        A.spmv(x, y)
        e1.record(st)
    torch.cuda.synchronize()
    t = sorted(e0.elapsed_time(e1) * 1e3 for e0, e1 in ev)
    return t[len(t) // 2]


def time_policies(s, policies, reps, flush, split="all_vbr"):
    """Per (name, delta, policy): SpMV us and partition stats of matrix s."""
    import torch

    from paper_2407_00829_b200 import sable
    inp = s.vbr_input(split)
    arrays = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in inp.items()
              if isinstance(v, np.ndarray)}
    x = torch.from_numpy(s.x).cuda()
    y = torch.empty(s.nrows, dtype=x.dtype, device="cuda")
    out = []
    for name, delta, pol in policies:
        A = sable.VbrMatrix(arrays, s.nrows, s.ncols, delta=delta, policy=pol)
        i = A.info
        out.append(dict(policy=name, us=round(time_one(A, x, y, reps, flush), 2),
                        n_dense=i["n_dense"], tile_elems=i["tile_elems"], rem_nnz=i["rem_nnz"],
                        bytes_alg=i["bytes_alg"], nnz=i["nnz"]))
        A.close()
    return out


def time_pair(s, reps, flush):
    """(t_dense_us, t_csr_us, nnz) for the matrix s, through libsable.so."""
    import torch

    from paper_2407_00829_b200 import sable
    inp = s.vbr_input("all_vbr")
    arrays = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in inp.items()
              if isinstance(v, np.ndarray)}
    x = torch.from_numpy(s.x).cuda()
    out = []
    for delta in (0, 101):
        A = sable.VbrMatrix(arrays, s.nrows, s.ncols, delta=delta)
        y = torch.empty(s.nrows, dtype=torch.float32, device="cuda")
        st = torch.cuda.current_stream()
        for _ in range(3):
            A.spmv(x, y)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(reps)]
        for e0, e1 in ev:
            flush()
            e0.record(st)
            A.spmv(x, y)
            e1.record(st)
        torch.cuda.synchronize()
        t = sorted(e0.elapsed_time(e1) * 1e3 for e0, e1 in ev)
        out.append(t[len(t) // 2])
        A.close()
    return out[0], out[1], s.nnz


def main():
    import torch

    import gen.calib as gc
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--reps", type=int, default=15)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_f2_calibration"))
    ap.add_argument("--c4a-scale", type=float, default=1.0)
    a = ap.parse_args()
    scrub = torch.empty(128 << 20, dtype=torch.float32, device="cuda")
    sink = torch.empty((), dtype=torch.float32, device="cuda")

    def flush():
        scrub.zero_()
        torch.sum(scrub, dim=0, out=sink)

    shapes = SHAPES[:3] if a.quick else SHAPES
    fills = FILLS[::3] if a.quick else FILLS
    heat = []
    for h, w in shapes:
        row = []
        for f in fills:
            s = gc.shape_grid(h, w, f)
            td, tc, nnz = time_pair(s, a.reps, flush)
            row.append(dict(h=h, w=w, fill=f, nnz=nnz, t_dense_us=round(td, 2),
                            t_csr_us=round(tc, 2), speedup=round(tc / td, 3)))
            print(json.dumps(row[-1]), flush=True)
        xf = crossover([r["fill"] for r in row], [r["speedup"] for r in row])
        heat.append(dict(h=h, w=w, points=row, crossover_fill=xf, delta_star=delta_of(xf)))
    abl = []
    for sp in (SPARSITIES[::3] if a.quick else SPARSITIES):
        s = gc.fig10(sp)
        td, tc, nnz = time_pair(s, a.reps, flush)
        abl.append(dict(sparsity=sp, nnz=nnz, t_dense_us=round(td, 2), t_csr_us=round(tc, 2),
                        speedup=round(tc / td, 3)))
        print(json.dumps(abl[-1]), flush=True)
    policy = policy_from_heatmap(heat)
    with open(a.out + "_policy.json", "w") as fp:
        json.dump(policy, fp, indent=1)
    import gen
    s4a = gen.make("c4a", scale=a.c4a_scale)
    stress = time_policies(s4a, [("delta=50", 50, None),
                                 ("calibrated", policy["delta"], policy),
                                 ("delta=0", 0, None), ("delta=101", 101, None)],
                           a.reps, flush, split="rect")
    for r in stress:
        print(json.dumps(dict(c4a=r)), flush=True)
    res = dict(heatmap=heat, fig10=abl, policy=policy, c4a_stress=stress, reps=a.reps,
               timing="median of per-SpMV CUDA events, L2 flushed (512 MiB scrub) before each SpMV",
               device=torch.cuda.get_device_name(0))
    with open(a.out + ".json", "w") as fjs:
        json.dump(res, fjs, indent=1)
    lines = ["# f2: per-shape delta calibration and sparsity ablation (B200)", "",
             "speedup = t(delta=101, all CSR remainder) / t(delta=0, all dense tiles), "
             "same VBR input; " + res["timing"] + ".", "",
             "## Fig. 7 analogue: speedup of the dense tile over CSR, by block shape and fill", "",
             "| h x w | " + " | ".join(f"{f:.1f}" for f in fills) + " | crossover fill | delta* |",
             "|---|" + "---|" * len(fills) + "---|---|"]
    for r in heat:
        lines.append(f"| {r['h']}x{r['w']} | " + " | ".join(f"{p['speedup']:.2f}"
                                                            for p in r["points"]) +
                     f" | {r['crossover_fill']} | {r['delta_star']} |")
    lines += ["", "## Fig. 10 analogue: 10000^2, 50x50 splits, 500 blocks", "",
              "| sparsity | nnz | dense us | CSR us | speedup |", "|---|---|---|---|---|"]
    for r in abl:
        lines.append(f"| {r['sparsity']:.2f} | {r['nnz']} | {r['t_dense_us']} | "
                     f"{r['t_csr_us']} | {r['speedup']:.2f} |")
    lines += ["", "## Calibrated policy (reading R22; sable_vbr_create_policy)", "",
              f"default delta {policy['delta']}, min_area {policy['min_area']}; rules "
              "(h range, w range, delta):", ""]
    for r in policy["rules"]:
        lines.append(f"- h {r[0]}..{r[1]}, w {r[2]}..{r[3]}: delta {r[4]}")
    lines += ["", f"## 64-aligned C4 stress case (gen c4a, scale {a.c4a_scale})", "",
              "| policy | SpMV us | dense tiles | tile elems | remainder nnz | alg. bytes |",
              "|---|---|---|---|---|---|"]
    for r in stress:
        lines.append(f"| {r['policy']} | {r['us']} | {r['n_dense']} | {r['tile_elems']} | "
                     f"{r['rem_nnz']} | {r['bytes_alg']} |")
    with open(a.out + ".md", "w") as fmd:
        fmd.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
