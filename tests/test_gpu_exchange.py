"""The exchange step through the C-ABI.

* one GPU: sable_spmv_iterate (one CUDA graph) equals the step-by-step loop
  bit for bit, graph relaunch and re-capture (new buffers / iteration count)
  included; the slice launches of the pipelined multi-GPU step tile the rows
  (SABLE_SLICED=1 runs them back to back on one GPU);
* two or more GPUs (skipped on a one-GPU box): world-size-2 processes over
  NCCL, sharded handles, sable_comm_init, then iterated steps checked against
  the oracle applied to the GPU's own x_k, and bitwise equal to the one-GPU
  result (P-invariance of the row sums).
"""
import os
import socket

import numpy as np
import pytest

import gen
import oracle
from parity import assert_y_close

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def sable():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2407_00829_b200 import sable as s
    return s


def make(sable, s, rank=0, world=1):
    arrays = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda()
              for k, v in s.vbr_input("rect").items() if isinstance(v, np.ndarray)}
    return sable.VbrMatrix(arrays, s.nrows, s.ncols, delta=s.delta, rank=rank, world=world)


def steps(A, x0, k):
    cur = x0.clone()
    nxt = torch.empty_like(cur)
    for _ in range(k):
        A.spmv_allgather(cur, nxt)
        cur, nxt = nxt, cur
    return cur


@pytest.mark.parametrize("sliced", [0, 1])
def test_iterate_graph_matches_steps(sable, monkeypatch, sliced):
    monkeypatch.setenv("SABLE_SLICED", str(sliced))
    s = gen.make("c5", scale=1 / 128)
    A = make(sable, s)
    try:
        x0 = torch.from_numpy(s.x).cuda()
        ref = steps(A, x0, 7)
        for k in (7, 7, 3, 7):  # capture, relaunch, re-capture, re-capture
            xa = x0.clone()
            xb = torch.empty_like(xa)
            res = A.iterate(xa, xb, k)
            if k == 7:
                assert torch.equal(res, ref)
            else:
                assert torch.equal(res, steps(A, x0, k))
        # one step against the oracle
        y = steps(A, x0, 1).cpu().numpy()
        yo, so = oracle.spmv(s.nrows, s.I, s.J, s.V.astype(np.float64), s.x.astype(np.float64))
        assert_y_close(y, yo, so, np.float32, "step")
    finally:
        A.close()


def test_sliced_step_equals_spmv(sable, monkeypatch):
    """The slice launches write every row exactly once: bitwise the single
    launch (the rows' summation order does not depend on the launch)."""
    for name, scale in (("c2", 0.03), ("c5", 1 / 256)):
        s = gen.make(name, scale=scale)
        if s.nrows != s.ncols:
            continue
        monkeypatch.setenv("SABLE_SLICED", "1")
        A = make(sable, s)
        try:
            x = torch.from_numpy(s.x).cuda()
            xn = torch.full_like(x, float("nan"))
            A.spmv_allgather(x, xn)
            assert torch.equal(xn, A.spmv(x))
        finally:
            A.close()


def test_comm_check_world1(sable):
    s = gen.make("c1")
    A = make(sable, s)
    try:
        A.comm_check()  # no communicator: OK
        A.comm_init(sable.sable_nccl_unique_id())
        A.comm_check()
    finally:
        A.close()


def _free_port() -> int:
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    return port


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2407_00829_b200 import dist as sdist
        from paper_2407_00829_b200 import sable
        s = gen.make("c5", scale=1 / 128)
        A = make(sable, s, rank, world)
        A.comm_init(sdist.broadcast_nccl_id(rank))
        x0 = torch.from_numpy(s.x).cuda()
        xs = [steps(A, x0, k).cpu().numpy() for k in (1, 2, 5)]
        xa = x0.clone()
        xb = torch.empty_like(xa)
        it = A.iterate(xa, xb, 5).cpu().numpy()
        A.close()
        if rank == 0:
            out.put((xs, it))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs two GPUs")
def test_two_gpu_exchange(sable):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pc = mp.start_processes(_worker, args=(2, _free_port(), q), nprocs=2, join=False,
                            start_method="spawn")
    xs, it = q.get(timeout=600)
    while not pc.join():
        pass
    s = gen.make("c5", scale=1 / 128)
    A = make(sable, s)
    x0 = torch.from_numpy(s.x).cuda()
    for k, xk in zip((1, 2, 5), xs):
        assert np.array_equal(xk, steps(A, x0, k).cpu().numpy())  # bitwise P-invariant
    assert np.array_equal(it, xs[-1])
    xprev = steps(A, x0, 4).cpu().numpy().astype(np.float64)
    yo, so = oracle.spmv(s.nrows, s.I, s.J, s.V.astype(np.float64), xprev)
    assert_y_close(xs[-1], yo, so, np.float32, "2-GPU step 5")
    A.close()
