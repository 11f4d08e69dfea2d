"""The exchange step through the C-ABI.

* one GPU: sable_spmv_iterate (one CUDA graph) equals the step-by-step loop
  bit for bit, graph relaunch and re-capture (new buffers / iteration count)
  included; the slice launches of the pipelined multi-GPU step tile the rows
  (SABLE_SLICED=1 runs them back to back on one GPU);
* the fused exchange epilogue (sable_comm_set_peers / sable_comm_fuse): P
  virtual ranks on one GPU, every rank's kernel storing its rows into all P
  "peer" buffers (here: other buffers of the same GPU, the ranks run one after
  the other on one stream): every buffer ends up with the full next x, bitwise
  the one-GPU step, over several ping-pong steps, fp32 and fp64, with long
  rows split into combine groups; world 1 fused = the plain step; argument
  errors; a step on an unregistered buffer falls back to the NCCL path's
  argument check;
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


@pytest.mark.parametrize("name,scale,world", [("c5", 1 / 128, 3), ("c3", 0.02, 2), ("c2", 0.03, 4),
                                              ("c5", 1 / 512, 8)])
def test_fused_epilogue_virtual_ranks(sable, name, scale, world):
    """KC2 on one GPU: rank r's launch writes its rows into its own x_next and
    into the x_next of every other rank; after all ranks ran, every rank's
    x_next is the full A x -- bitwise the one-GPU result, step after step."""
    s = gen.make(name, scale=scale)
    full = make(sable, s)
    ranks = [make(sable, s, r, world) for r in range(world)]
    try:
        x0 = torch.from_numpy(s.x).cuda()
        # each rank's ping-pong pair; the initial x replicated in every a-buffer
        xa = [x0.clone() for _ in range(world)]
        xb = [torch.full_like(x0, float("nan")) for _ in range(world)]
        for r, A in enumerate(ranks):
            others = [q for q in range(world) if q != r]
            A.comm_set_peers(xa[r], xb[r], [xa[q] for q in others], [xb[q] for q in others])
        cur, nxt = xa, xb
        ref = x0
        for k in range(4):
            for r, A in enumerate(ranks):  # one stream: the ranks in turn
                A.spmv_allgather(cur[r], nxt[r])
            ref = steps(full, ref, 1)
            for r in range(world):
                assert torch.equal(nxt[r], ref), (k, r)
            cur, nxt = nxt, cur
        # the graph iterate on fused buffers (no communicator: caller-ordered;
        # one rank alone only fills its own rows everywhere)
        for r in range(world):
            xa[r].copy_(x0)
            xb[r].fill_(0)
        res = ranks[0].iterate(xa[0], xb[0], 1)
        lo, hi = ranks[0].info["row_begin"], ranks[0].info["row_end"]
        one = steps(full, x0, 1)
        assert res.data_ptr() == xb[0].data_ptr()
        for r in range(world):
            assert torch.equal(xb[r][lo:hi], one[lo:hi])
            assert not xb[r][hi:].any() and not xb[r][:lo].any()
        # unfuse: a world > 1 handle without a communicator refuses the step
        ranks[0].comm_unfuse()
        with pytest.raises(sable.SableError):
            ranks[0].spmv_allgather(xa[0], xb[0])
    finally:
        for A in ranks:
            A.close()
        full.close()


def test_fused_world1_and_errors(sable):
    s = gen.make("c5", scale=1 / 256)
    A = make(sable, s)
    try:
        x0 = torch.from_numpy(s.x).cuda()
        ref = steps(A, x0, 3)
        xa, xb = x0.clone(), torch.empty_like(x0)
        A.comm_fuse(xa, xb)  # world 1: no peers, the plain step
        assert torch.equal(A.iterate(xa, xb, 3), ref)
        other = torch.empty_like(x0)
        assert torch.equal(steps(A, x0, 3), ref)  # unregistered buffers: unchanged path
        with pytest.raises(sable.SableError):
            A.comm_fuse(xa, xa)
        with pytest.raises(sable.SableError):
            A.comm_set_peers(xa, xb, [xa], [other])  # a peer aliasing the local buffer
        with pytest.raises(sable.SableError):
            A.comm_set_peers(xa, xb, [other] * 8, [other] * 8)  # more than 7 peers
        A.comm_unfuse()
        assert torch.equal(A.iterate(xa.copy_(x0), xb, 3), ref)
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
        # the fused epilogue over CUDA IPC peer mappings (plain cudaMalloc
        # buffers: torch's caching allocator hands out cudaMalloc blocks)
        fa = x0.clone()
        fb = torch.empty_like(fa)
        A.comm_fuse(fa, fb)
        fused = A.iterate(fa, fb, 5).cpu().numpy()
        torch.cuda.synchronize()
        dist.barrier()
        A.close()
        if rank == 0:
            out.put((xs, it, fused))
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
    xs, it, fused = q.get(timeout=600)
    while not pc.join():
        pass
    s = gen.make("c5", scale=1 / 128)
    A = make(sable, s)
    x0 = torch.from_numpy(s.x).cuda()
    for k, xk in zip((1, 2, 5), xs):
        assert np.array_equal(xk, steps(A, x0, k).cpu().numpy())  # bitwise P-invariant
    assert np.array_equal(it, xs[-1])
    assert np.array_equal(fused, xs[-1])  # fused epilogue = NCCL path, bitwise
    xprev = steps(A, x0, 4).cpu().numpy().astype(np.float64)
    yo, so = oracle.spmv(s.nrows, s.I, s.J, s.V.astype(np.float64), xprev)
    assert_y_close(xs[-1], yo, so, np.float32, "2-GPU step 5")
    A.close()
