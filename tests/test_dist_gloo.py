"""Multi-process (world size 2, gloo, CPU) tests of the multi-GPU plumbing
(BASELINE.json north_star s7).

No GPU here: each rank computes its y slice with the CPU oracle (test
infrastructure) and the slices are all-gathered with torch.distributed over
gloo.  What is under test is the protocol the GPU path implements with NCCL
inside libsable.so: block-row shard bounds from sable_shard_bounds (the host
function the inspector calls) agree on every rank, the ranks' row ranges tile
the rows, and the rank-ordered concatenation of the slices -- the all-gather
into the next x -- reproduces A x and, iterated, the oracle's iteration.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _case():
    import gen
    import oracle

    s = gen.make("c5", scale=1 / 512)  # square, column-stochastic, power-law rows
    part = oracle.partition(s.nrows, s.ncols, s.I, s.J, s.V.astype(np.float64), s.rpntr, s.cpntr,
                            s.delta)
    nbr = len(s.rpntr) - 1
    h = np.diff(s.rpntr).astype(np.int64)
    w = np.diff(s.cpntr).astype(np.int64)
    dense = part["cell_dense"].astype(bool)
    area = np.zeros(nbr, np.int64)
    np.add.at(area, part["cell_br"][dense], h[part["cell_br"][dense]] * w[part["cell_bc"][dense]])
    rem_per_row = np.diff(part["rem_indptr"])
    return s, area, rem_per_row


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2407_00829_b200 import dist as sdist

        s, area, rem_per_row = _case()
        weights = sdist.block_row_weights(len(s.rpntr) - 1, s.rpntr, area, rem_per_row)
        bounds = sdist.shard_bounds(weights, world)
        # every rank derived the same bounds
        allb = [torch.zeros(world + 1, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(allb, torch.from_numpy(bounds.astype(np.int32)))
        same = all(torch.equal(b, allb[0]) for b in allb)
        ranges = sdist.row_ranges(s.rpntr, bounds)
        # the rows libsable.so's all-gather broadcasts for every rank
        # (sable_exchange_rows: the host layout comm.cu follows)
        ex = sdist.sable.sable_exchange_rows(weights, s.rpntr, world)
        layout_ok = [(int(ex[q]), int(ex[q + 1])) for q in range(world)] == ranges
        r0, r1 = ranges[rank]
        rp = s.rowptr()
        x = s.x.astype(np.float64)
        xs = [x]
        for _ in range(3):  # iterated SpMV: local rows, then the all-gather
            y_loc, _ = oracle.spmv_rows(rp, s.J, s.V.astype(np.float64), x, np.arange(r0, r1))
            sizes = [b - a for a, b in ranges]
            pad = max(sizes)
            buf = torch.zeros(pad, dtype=torch.float64)
            buf[: r1 - r0] = torch.from_numpy(y_loc)
            gathered = [torch.zeros(pad, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(gathered, buf)
            x = np.concatenate([g[:n].numpy() for g, n in zip(gathered, sizes)])
            xs.append(x)
        if rank == 0:
            out.put((same and layout_ok, bounds.tolist(), ranges, [v.tolist() for v in xs]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_iteration_matches_oracle(world):
    import oracle

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pc = mp.start_processes(_worker, args=(world, _free_port(), q), nprocs=world, join=False,
                            start_method="spawn")
    same, bounds, ranges, xs = q.get(timeout=240)  # before join: the queue must drain
    while not pc.join():
        pass
    assert same, "ranks derived different shard bounds or exchange rows"
    s, area, rem_per_row = _case()
    nbr = len(s.rpntr) - 1
    assert bounds[0] == 0 and bounds[-1] == nbr and all(a <= b for a, b in zip(bounds, bounds[1:]))
    # the row ranges tile [0, nrows) in rank order
    assert ranges[0][0] == 0 and ranges[-1][1] == s.nrows
    assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
    # balance: no rank holds more than its share plus the heaviest block row
    from paper_2407_00829_b200 import dist as sdist
    w = sdist.block_row_weights(nbr, s.rpntr, area, rem_per_row)
    per = [int(w[bounds[q]:bounds[q + 1]].sum()) for q in range(world)]
    assert max(per) <= w.sum() / world + w.max()
    # x_{k+1} = A x_k, gathered from the slices, equals the oracle's product
    x = s.x.astype(np.float64)
    for k in range(1, len(xs)):
        y, sc = oracle.spmv(s.nrows, s.I, s.J, s.V.astype(np.float64), x)
        np.testing.assert_allclose(np.asarray(xs[k]), y, rtol=0, atol=1e-12 * max(1.0, sc.max()))
        x = y
    # column-stochastic A conserves sum(x)
    assert abs(sum(xs[-1]) - sum(xs[0])) <= 1e-9 * abs(sum(xs[0]))


def _worker_fused(rank, world, port, out):
    """The fused exchange protocol (KC2) over gloo: every
    rank keeps two full ping-pong buffers; a step computes the local rows from
    the current buffer, stores them at their global row offset into its own
    next buffer and into every peer's next buffer (here: point-to-point sends
    the peer places at the sender's row range -- the peer stores of the
    kernel's epilogue), and ends with a one-word all-reduce (the barrier)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2407_00829_b200 import dist as sdist

        s, area, rem_per_row = _case()
        weights = sdist.block_row_weights(len(s.rpntr) - 1, s.rpntr, area, rem_per_row)
        ex = sdist.sable.sable_exchange_rows(weights, s.rpntr, world)  # libsable's row layout
        ranges = [(int(ex[q]), int(ex[q + 1])) for q in range(world)]
        r0, r1 = ranges[rank]
        rp = s.rowptr()
        cur = torch.from_numpy(s.x.astype(np.float64).copy())
        nxt = torch.full_like(cur, float("nan"))
        xs = []
        for k in range(3):
            y_loc, _ = oracle.spmv_rows(rp, s.J, s.V.astype(np.float64), cur.numpy(),
                                        np.arange(r0, r1))
            mine = torch.from_numpy(y_loc)
            nxt[r0:r1] = mine  # the local store
            reqs = [dist.isend(mine, q) for q in range(world) if q != rank]  # the peer stores
            for q in range(world):
                if q != rank:
                    a, b = ranges[q]
                    dist.recv(nxt[a:b], q)  # lands at the sender's global rows
            for r in reqs:
                r.wait()
            flag = torch.zeros(1, dtype=torch.int32)
            dist.all_reduce(flag, op=dist.ReduceOp.MAX)  # the step barrier
            assert not torch.isnan(nxt).any()  # every row arrived before the barrier ended
            xs.append(nxt.clone())
            cur, nxt = nxt, cur
            nxt.fill_(float("nan"))  # the buffer the next step overwrites is free
        out.put((rank, [v.tolist() for v in xs]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_fused_exchange_protocol(world):
    import oracle

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pc = mp.start_processes(_worker_fused, args=(world, _free_port(), q), nprocs=world,
                            join=False, start_method="spawn")
    got = dict(q.get(timeout=240) for _ in range(world))
    while not pc.join():
        pass
    s, _, _ = _case()
    x = s.x.astype(np.float64)
    for k in range(3):
        y, sc = oracle.spmv(s.nrows, s.I, s.J, s.V.astype(np.float64), x)
        for r in range(world):  # every rank holds the full next x after every step
            np.testing.assert_allclose(np.asarray(got[r][k]), y, rtol=0,
                                       atol=1e-12 * max(1.0, sc.max()))
        assert all(got[r][k] == got[0][k] for r in range(world))  # and the same bits
        x = y
