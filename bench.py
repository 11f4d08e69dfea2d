#!/usr/bin/env python
"""bench.py -- VBR SpMV on B200 through libsable.so (the C-ABI).

Metric (BASELINE.json): "VBR SpMV GFLOP/s and achieved HBM GB/s (% of
roofline) at 1/2/4/8 B200".  value = useful GFLOP/s = 2 * nnz / step time,
nnz = true non-zeros of the whole matrix (all ranks).

A step is one pass of the executor over the whole matrix, y = A x (SURVEY
8(a) a6); with N > 1 GPUs the matrix is row-sharded (north_star s7) and a step
is one iterated-SpMV step (a6 + a7): the local SpMV written into x_next and
its rows exchanged -- by the fused epilogue (the kernel stores each y row into
every peer's x_next over NVLink, sable_comm_fuse; self-checked against the
NCCL step before timing) or else by the pipelined NCCL all-gather.  The inspector (a1..a5, sable_vbr_create)
runs once before the timed region -- compile once, run many
-- and its time is reported as inspect_ms.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2]
                       [--impl reference]
For N > 1 launch with torch.distributed.run (one process per GPU).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "VBR SpMV GFLOP/s and achieved HBM GB/s (% of roofline) at 1/2/4/8 B200"
WORKLOADS = {
    "c1": "configs[0]: fp32 VBR SpMV 2000^2, 12 blocks + 0.2% scatter, delta=50",
    "c2": "configs[1]: fp32 VBR SpMV 200000^2 block-diagonal-plus-off-diagonal, 5000 blocks "
          "log-U[4,128] + 1e-4 scatter, delta=50",
    "c3": "configs[2]: fp64 VBR SpMV 500000^2 power-grid-like block-tridiagonal + 3 couplings/row",
    "c4": "configs[3]: fp32 VBR SpMV 2^20 pruned-NN-like 64x64-aligned sub-blocks (~60M nnz)",
    "c5": "configs[4]: fp32 iterated VBR SpMV 2^23, 40% blocks log-U[4,256] + 60% power-law CSR",
}
L2_FLUSH_BYTES = 512 << 20  # > 2x the 126 MB L2
L2_BYTES = 126 << 20  # B200 L2 capacity (B200_PROFILING.md)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def traffic_for(config: str):
    """DRAM bytes (read + write) of one SpMV -- the remainder and the dense-tile
    executor launches of one step -- from the committed ncu capture
    (profiles/traffic.json, written by scripts/ncu_summary.py), or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        return json.load(open(p)).get(config)
    return None


class ClockSampler:
    """Poll NVML (the data behind nvidia-smi's clocks line) during the timed region."""

    def __init__(self, dev_index: int, period_s: float = 0.005):
        self.samples, self.reasons = [], set()
        self.period = period_s
        self.ok = False
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False
        self._stop = threading.Event()

    _NAMES = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
              0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
              0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
              0x100: "display_clock_setting"}

    def _run(self):
        while not self._stop.is_set():
            try:
                mhz = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                util = self.nv.nvmlDeviceGetUtilizationRates(self.h).gpu
                self.samples.append((mhz, util))
                for bit, name in self._NAMES.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        loaded = [m for m, u in self.samples if u > 0] or [m for m, _ in self.samples]
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def make_input(config: str):
    """The seeded synthetic matrix of a config and its VBR input split.  With
    SABLE_GEN_CACHE=<dir> the generated matrix is saved there once and reused
    by later runs of the same gpurun call (C5 takes minutes to generate);
    nothing depends on the cache surviving between calls."""
    import gen
    t = time.time()
    cache = os.environ.get("SABLE_GEN_CACHE")
    path = os.path.join(cache, f"{config}.npz") if cache else None
    if path and os.path.exists(path):
        z = np.load(path, allow_pickle=False)
        s = gen.Synth(name=config, nrows=int(z["nrows"]), ncols=int(z["ncols"]),
                      dtype=z["V"].dtype.type, delta=int(z["delta"]), rpntr=z["rpntr"],
                      cpntr=z["cpntr"], rects=z["rects"], I=z["I"], J=z["J"], V=z["V"], x=z["x"],
                      in_rect=z["in_rect"], iterations=int(z["iterations"]))
    else:
        s = gen.make(config)
        if path:
            os.makedirs(cache, exist_ok=True)
            np.savez(path, nrows=s.nrows, ncols=s.ncols, delta=s.delta, rpntr=s.rpntr,
                     cpntr=s.cpntr, rects=s.rects, I=s.I, J=s.J, V=s.V, x=s.x, in_rect=s.in_rect,
                     iterations=s.iterations)
    inp = s.vbr_input("rect")
    return s, inp, time.time() - t


# --------------------------------------------------------------------- our arm

def run_sable(args):
    import torch
    import torch.distributed as dist

    from paper_2407_00829_b200 import sable

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)

    s, inp, gen_s = make_input(args.config)
    arrays = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in inp.items()
              if isinstance(v, np.ndarray)}
    torch.cuda.synchronize()
    A = sable.VbrMatrix(arrays, s.nrows, s.ncols, delta=s.delta, rank=rank, world=world)
    del arrays
    info = A.info
    if world > 1:
        uid = [sable.sable_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        A.comm_init(uid[0])

    tdt = torch.float64 if s.dtype == np.float64 else torch.float32
    sv = 8 if s.dtype == np.float64 else 4
    x = torch.from_numpy(s.x).to(dev)
    nloc = info["row_end"] - info["row_begin"]
    y = torch.empty(nloc, dtype=tdt, device=dev)
    xn = torch.empty_like(x)
    # L2 between timed steps: flushed, or kept when the SpMV's working set is
    # larger than twice the 126 MB L2 (the streamed bytes cannot be L2 hits;
    # what survives is x and metadata, as in an iterated SpMV) -- "auto"
    if args.l2 == "auto":
        flush_l2 = info["bytes_alg"] <= 2 * L2_BYTES
    else:
        flush_l2 = args.l2 == "flush"
    scrub = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    scrub_sink = torch.empty((), dtype=torch.float32, device=dev)

    def flush():
        # write 512 MiB (> 4x the 126 MB L2), then read it back, so L2 holds
        # only clean lines of the scrub buffer: none of the SpMV's data, and no
        # dirty write-back of the scrub's own lines inside the timed region
        scrub.zero_()
        torch.sum(scrub, dim=0, out=scrub_sink)
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream

    # N > 1: the fused exchange epilogue (peer stores from the SpMV kernel,
    # sable_comm_fuse) when every rank can map its peers and one fused step
    # reproduces the NCCL pipeline's x_next bit for bit; else the NCCL pipeline
    exchange, exchange_note = "none", ""
    if world > 1:
        exchange = "nccl"
        ref = torch.empty_like(x)
        A.spmv_allgather(x, ref, sp)  # unregistered buffers: the NCCL pipeline
        ok = torch.ones(1, dtype=torch.int32, device=dev)
        if args.exchange in ("auto", "fused"):
            try:
                A.comm_fuse(x, xn)
            except sable.SableError as e:
                ok.zero_()
                exchange_note = str(e)
        else:
            ok.zero_()
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()):
            A.spmv_allgather(x, xn, sp)  # xn is registered: the fused step
            torch.cuda.synchronize()
            ok.fill_(int(torch.equal(ref, xn)))
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if int(ok.item()):
                exchange = "fused"
            else:
                exchange_note = "fused step differed from the NCCL step (self-check): NCCL used"
        if exchange != "fused":
            A.comm_unfuse()
        del ref

    def step():
        if world > 1:
            A.spmv_allgather(x, xn, sp)
        else:
            A.spmv(x, y, sp)

    def timed_loop(fn, k, flush_each=None):
        fl = flush_l2 if flush_each is None else flush_each
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(k)]
        for i in range(k):
            if fl:
                flush()
            ev[i][0].record(stream)
            fn()
            ev[i][1].record(stream)
        return ev

    for _ in range(args.warmup):
        if flush_l2:
            flush()
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev = timed_loop(step, args.steps)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    times = [a.elapsed_time(b) for a, b in ev]
    ms = sum(times) / len(times)

    # the SpMV kernel alone (roofline of the dominant kernel), same protocol
    evk = timed_loop(lambda: A.spmv(x, y, sp), max(args.steps, 20))
    torch.cuda.synchronize()
    kt = [a.elapsed_time(b) for a, b in evk]
    k_ms = sum(kt) / len(kt)
    # when L2 is kept between steps, the same kernel with L2 flushed too
    # (reported beside the headline, roofline.frac_l2_flushed)
    kf_ms = None
    if not flush_l2:
        evf = timed_loop(lambda: A.spmv(x, y, sp), max(args.steps, 20), flush_each=True)
        torch.cuda.synchronize()
        kf_ms = statistics.mean(a.elapsed_time(b) for a, b in evf)

    # end to end through the C-ABI with pinned host buffers (H2D x, SpMV, D2H y)
    xh = torch.from_numpy(s.x.copy()).pin_memory()
    yh = torch.empty(nloc, dtype=tdt).pin_memory()
    for _ in range(3):
        sable.sable_spmv_host(A.handle, xh.data_ptr(), yh.data_ptr(), sp)
    e2e_ev = timed_loop(lambda: sable.sable_spmv_host(A.handle, xh.data_ptr(), yh.data_ptr(), sp),
                        max(args.steps, 20))
    torch.cuda.synchronize()
    e2e_ms = statistics.mean(a.elapsed_time(b) for a, b in e2e_ev)

    # our kernels per step: one unit-executor launch (sable::unit_kernel)
    launches_per_step = int(info["n_unit_batches"] > 0) * (8 if exchange == "nccl" else 1)
    red = torch.tensor([ms, k_ms, e2e_ms, info["bytes_alg"], kf_ms or 0.0], dtype=torch.float64,
                       device=dev)
    if world > 1:
        mx = red.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        tot = torch.tensor([float(info["bytes_alg"])], dtype=torch.float64, device=dev)
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        ms, k_ms, e2e_ms = float(mx[0]), float(mx[1]), float(mx[2])
        bytes_alg_local_max = float(mx[3])
        kf_ms = float(mx[4]) if kf_ms is not None else None
    else:
        bytes_alg_local_max = float(info["bytes_alg"])

    if rank == 0:
        peak, peak_kind = peaks()
        nnz = s.nnz
        gflops = 2.0 * nnz / (ms * 1e-3) / 1e9
        ach = bytes_alg_local_max / (k_ms * 1e-3) / 1e9
        line = {
            "metric": METRIC,
            "value": round(gflops, 3),
            "unit": "GFLOP/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms, 6),
            "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None,
            "dtype": "f64" if s.dtype == np.float64 else "f32",
            "data": "synthetic (seeded gen/ recipe of BASELINE.json config; SuiteSparse stand-in)",
            "config": {
                "workload": f"{args.config} -- {WORKLOADS[args.config]}",
                "n": s.nrows, "nnz": nnz, "delta": s.delta, "input_split": "rect",
                "grid": [len(s.rpntr) - 1, len(s.cpntr) - 1],
                "n_cells": info["n_cells"], "n_dense_tiles": info["n_dense"],
                "tile_elems": info["tile_elems"], "rem_nnz": info["rem_nnz"],
                "executor": "unit executor (one launch per SpMV)",
                "n_units": info["n_units"], "warps": info["n_unit_batches"],
                "n_combine": info["n_combine"], "panel_elems": info["panel_elems"],
                "xmap_entries": info["xmap_entries"], "exec_grid": info["exec_grid"],
                "l2": ("flushed between timed steps (512 MiB write, then read)" if flush_l2 else
                       "not flushed: working set > 2x L2 (iterated SpMV, cache behaviour is real)"),
                "parallelism": f"row-sharded x{world}" + {
                    "none": "", "nccl": " + NCCL broadcast pipeline (8 slices overlapped)",
                    "fused": " + fused NVLink epilogue (peer stores from the SpMV kernel) + "
                             "one-word all-reduce barrier"}[exchange],
                **({"exchange_note": exchange_note} if exchange_note else {}),
                "bytes_alg_per_step": info["bytes_alg"] if world == 1 else None,
            },
            "roofline": {
                "bound": "hbm", "achieved": round(ach, 2), "peak": peak, "unit": "GB/s",
                "frac": round(ach / peak, 4), "traffic": traffic_for(args.config),
                "peak_kind": peak_kind,
                "kernel": "one SpMV = one sable::unit_kernel launch",
                "kernel_ms": round(k_ms, 6),
                "bytes_alg_per_launch": bytes_alg_local_max,
                "l2": "kept between steps" if not flush_l2 else "flushed between steps",
            },
            "e2e": {"value": round(2.0 * nnz / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GFLOP/s",
                    "h2d_bytes_per_step": int(s.ncols * sv), "d2h_bytes_per_step": int(nloc * sv),
                    "ms_per_step": round(e2e_ms, 6), "api": "sable_spmv_host (C-ABI, pinned host x/y)"},
            "gpu_launches": args.steps * launches_per_step,
            **({"l2_flushed": {
                "kernel_ms": round(kf_ms, 6),
                "frac": round(bytes_alg_local_max / (kf_ms * 1e-3) / 1e9 / peak, 4),
                "note": "the same SpMV with L2 flushed (512 MiB scrub) before every launch"}}
               if kf_ms else {}),
            "inspect_ms": round(info["inspect_ms"], 3),
            "gen_s": round(gen_s, 2),
            "clocks": clk.summary(),
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(s)
        print(json.dumps(line), flush=True)
    A.close()
    if world > 1:
        dist.destroy_process_group()


# --------------------------------------------------------------- oracle timing

def host_info():
    """nproc and the CPU model of this host."""
    model = "unknown"
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return os.cpu_count() or 1, model


def oracle_sample(s, max_nnz: int):
    """The first rows of the matrix holding at most max_nnz non-zeros."""
    rp = s.rowptr()
    r = int(np.searchsorted(rp, max_nnz, side="right") - 1)
    r = max(1, min(r, s.nrows))
    k = int(rp[r])
    return r, k, rp[: r + 1]


def time_oracle(rp, J, V, x, r, nthreads, reps=5, budget_s=20.0):
    """Median ms of `reps` oracle SpMVs (after one warm-up), fewer if the
    budget runs out."""
    import oracle
    oracle.spmv_csr_mt(rp, J, V, x, r, nthreads)  # warm-up
    ts = []
    t_all = time.perf_counter()
    for _ in range(reps):
        t0 = time.perf_counter()
        oracle.spmv_csr_mt(rp, J, V, x, r, nthreads)
        ts.append((time.perf_counter() - t0) * 1e3)
        if time.perf_counter() - t_all > budget_s:
            break
    return statistics.median(ts), len(ts)


def cpu_baseline(s, max_nnz: int = 64_000_000, partition: bool = True):
    """The oracle's fp64 SpMV (plain C, oracle/sable_oracle.c) on this host:
    median of 5 after a warm-up, single-threaded and row-parallel on all
    cores (OpenMP; bitwise the same y), on the first rows of the matrix
    holding <= max_nnz non-zeros (all of C1..C4); plus the oracle's
    partition time next to the GPU inspector's."""
    import oracle
    nproc, model = host_info()
    r, k, rp = oracle_sample(s, max_nnz)
    J = np.ascontiguousarray(s.J[:k], dtype=np.int64)
    V = np.ascontiguousarray(s.V[:k], dtype=np.float64)
    x = s.x.astype(np.float64)
    ms1, n1 = time_oracle(rp, J, V, x, r, 1)
    msn, nn = time_oracle(rp, J, V, x, r, nproc)
    out = {"value": round(2.0 * k / (msn * 1e-3) / 1e9, 4), "unit": "GFLOP/s", "cores": nproc,
           "kind": "oracle",
           "sample": f"oracle_spmv_csr_mt (fp64) over rows [0,{r}) = {k} of {s.nnz} nnz; "
                     f"median of {nn} after 1 warm-up, {nproc} OpenMP threads: {msn:.2f} ms",
           "single_thread": {"value": round(2.0 * k / (ms1 * 1e-3) / 1e9, 4), "unit": "GFLOP/s",
                             "ms": round(ms1, 3), "reps": n1},
           "all_cores_ms": round(msn, 3), "nproc": nproc, "cpu_model": model}
    if partition:
        t0 = time.perf_counter()
        oracle.partition(s.nrows, s.ncols, s.I, s.J, s.V.astype(np.float64), s.rpntr, s.cpntr,
                         s.delta)
        out["oracle_partition_ms"] = round((time.perf_counter() - t0) * 1e3, 1)
    return out


def run_reference(args):
    """--impl reference: the oracle as it stands, on all host cores (OpenMP,
    row-parallel; the reference arm of this tier is the oracle)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    s, _, _ = make_input(args.config)
    nproc, model = host_info()
    r, k, rp = oracle_sample(s, 64_000_000)
    J = np.ascontiguousarray(s.J[:k], dtype=np.int64)
    V = np.ascontiguousarray(s.V[:k], dtype=np.float64)
    x = s.x.astype(np.float64)
    for _ in range(args.warmup):
        oracle.spmv_csr_mt(rp, J, V, x, r, nproc)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.spmv_csr_mt(rp, J, V, x, r, nproc)
    ms = (time.perf_counter() - t0) * 1e3 / args.steps
    v = 2.0 * k / (ms * 1e-3) / 1e9
    sample = (f"oracle_spmv_csr_mt (fp64, {nproc} OpenMP threads) over rows [0,{r}) = {k} of "
              f"{s.nnz} nnz per step")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": "GFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "config": {"workload": f"{args.config} -- {WORKLOADS[args.config]}",
                                                         "n": s.nrows, "nnz": s.nnz},
        "cpu_baseline": {"value": round(v, 4), "unit": "GFLOP/s", "cores": nproc, "kind": "oracle",
                         "sample": sample, "cpu_model": model},
        "e2e": {"value": round(v, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="sable", choices=["sable", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--exchange", default="auto", choices=["auto", "fused", "nccl"],
                    help="N > 1: fused NVLink epilogue (self-checked, falls back) or NCCL pipeline")
    ap.add_argument("--l2", default="auto", choices=["auto", "flush", "keep"],
                    help="L2 between timed steps: flush, keep, or auto (keep when the "
                         "SpMV's algorithmic bytes exceed 2x L2)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_sable(args)


if __name__ == "__main__":
    main()
