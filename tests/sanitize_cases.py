"""Small cases for compute-sanitizer runs (tests/test_gpu_sanitize.py): C1,
random grids in fp32/fp64, long remainder rows split into pieces, tiny unit
budgets (column chunks, many combine groups), SpMM k = 4, tensor-core SpMM
k = 16 and 128 (fp32), an iterated exchange step and the fused exchange
epilogue with virtual ranks.  Exits 0 when every
result matches the oracle."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import gen  # noqa: E402
import oracle  # noqa: E402
from parity import assert_partition_equal, assert_y_close  # noqa: E402


def run(s, split="rect"):
    from paper_2407_00829_b200 import sable
    arrays = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda()
              for k, v in s.vbr_input(split).items() if isinstance(v, np.ndarray)}
    A = sable.VbrMatrix(arrays, s.nrows, s.ncols, delta=s.delta)
    got = A.export()
    want = oracle.partition(s.nrows, s.ncols, s.I, s.J, s.V.astype(np.float64), s.rpntr, s.cpntr,
                            s.delta)
    assert_partition_equal(got, want, s.dtype, s.name)
    x = torch.from_numpy(s.x).cuda()
    y = A.spmv(x).cpu().numpy()
    yo, so = oracle.spmv(s.nrows, s.I, s.J, s.V.astype(np.float64), s.x.astype(np.float64))
    assert_y_close(y, yo, so, s.dtype, s.name)
    X = torch.stack([x, 2 * x, -x, x], dim=1).contiguous()
    Y = A.spmm(X).cpu().numpy()
    assert_y_close(Y[:, 1] / 2, yo, so, s.dtype, s.name + " spmm")
    if s.dtype == np.float32:  # the tensor-core path (k = 16 and 128)
        for kk in (16, 128):
            Xk = torch.stack([x * (1 + (j % 3)) for j in range(kk)], dim=1).contiguous()
            Yk = A.spmm(Xk).cpu().numpy()
            assert_y_close(Yk[:, kk - 2] / (1 + (kk - 2) % 3), yo, so, s.dtype, s.name + f" mma{kk}")
    if s.nrows == s.ncols:
        xn = torch.empty_like(x)
        A.spmv_allgather(x, xn)
        assert torch.equal(xn, A.spmv(x))
        xa, xb = x.clone(), torch.empty_like(x)
        A.iterate(xa, xb, 3)
    img = A.serialize()
    B = sable.VbrMatrix.from_image(img)
    assert torch.equal(B.spmv(x), A.spmv(x))
    B.close()
    A.close()
    torch.cuda.synchronize()


def run_fused(s, world=3):
    """The fused exchange epilogue with `world` virtual ranks on one GPU:
    every rank stores its rows into all the ranks' x_next."""
    from paper_2407_00829_b200 import sable
    arrays = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda()
              for k, v in s.vbr_input("rect").items() if isinstance(v, np.ndarray)}
    full = sable.VbrMatrix(arrays, s.nrows, s.ncols, delta=s.delta)
    ranks = [sable.VbrMatrix(arrays, s.nrows, s.ncols, delta=s.delta, rank=r, world=world)
             for r in range(world)]
    x = torch.from_numpy(s.x).cuda()
    xa = [x.clone() for _ in range(world)]
    xb = [torch.empty_like(x) for _ in range(world)]
    for r, A in enumerate(ranks):
        o = [q for q in range(world) if q != r]
        A.comm_set_peers(xa[r], xb[r], [xa[q] for q in o], [xb[q] for q in o])
    for r, A in enumerate(ranks):
        A.spmv_allgather(xa[r], xb[r])
    want = full.spmv(x)
    for r in range(world):
        assert torch.equal(xb[r], want)
    for A in ranks + [full]:
        A.close()
    torch.cuda.synchronize()


def main():
    from test_gpu_parity import long_rows_synth
    cases = [gen.make("c1"), gen.make("c5", scale=1 / 512), long_rows_synth()]
    for seed, shape in enumerate([(300, 280, 23, 19), (64, 5000, 2, 3), (1000, 800, 7, 5)]):
        cases.append(gen.random_small(60 + seed, *shape, dtype=np.float64 if seed % 2 else np.float32,
                                      density=0.2, dense_cells=0.5))
    for s in cases:
        run(s)
    for s in cases:
        if s.nrows == s.ncols:
            run_fused(s)
    os.environ["SABLE_USTAGE"] = "1024"  # tiny units: pieces, column chunks, combine groups
    os.environ["SABLE_UBATCH_UNITS"] = "3"
    for s in cases[1:4]:
        run(s, "all_rem")
    for s in cases[1:4]:
        if s.nrows == s.ncols:
            run_fused(s, world=2)
    print("sanitize cases ok")


if __name__ == "__main__":
    main()
