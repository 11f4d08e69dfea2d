"""Multi-vector products (sable_spmm): Y = A X for k
right-hand sides.  Pin: Y[:, j] is the product with column j, so every column
is checked against the oracle's SpMV of that column (north_star tolerance,
per-row scale sum|a||x_j|).  Inputs: seeded generators of gen/."""
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


def make(sable, s, split="rect", rank=0, world=1):
    inp = s.vbr_input(split)
    arrays = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in inp.items()
              if isinstance(v, np.ndarray)}
    return sable.VbrMatrix(arrays, s.nrows, s.ncols, delta=s.delta, rank=rank, world=world)


def xs(s, k, seed=3):
    g = np.random.default_rng(seed)
    X = g.uniform(-1, 1, (s.ncols, k)).astype(s.dtype)
    X[:, 0] = s.x
    return X


def check(sable, s, k, split="rect", rank=0, world=1):
    A = make(sable, s, split, rank, world)
    try:
        X = xs(s, k)
        Y = A.spmm(torch.from_numpy(X).cuda()).cpu().numpy()
        r0, r1 = A.info["row_begin"], A.info["row_end"]
        rp = s.rowptr()
        for j in range(k):
            yo, so = oracle.spmv_rows(rp, s.J, s.V.astype(np.float64), X[:, j].astype(np.float64),
                                      np.arange(r0, r1))
            assert_y_close(Y[:, j], yo, so, s.dtype, f"{s.name}/{split}/k{k}/col{j}")
        # deterministic run to run
        Y2 = A.spmm(torch.from_numpy(X).cuda()).cpu().numpy()
        np.testing.assert_array_equal(Y.view(np.uint8), Y2.view(np.uint8))
        return Y
    finally:
        A.close()


@pytest.mark.parametrize("k", [1, 2, 4, 8])
def test_c1(sable, k):
    check(sable, gen.make("c1"), k)


@pytest.mark.parametrize("name,scale", [("c2", 0.03), ("c3", 0.01), ("c4", 0.02), ("c5", 1 / 512)])
def test_configs(sable, name, scale):
    s = gen.make(name, scale=scale)
    check(sable, s, 4)
    check(sable, s, 8, split="all_rem")


@pytest.mark.parametrize("seed", range(6))
def test_random_small(sable, seed):
    s = gen.random_small(40 + seed, 300 + 37 * seed, 250 + 11 * seed, 9, 7,
                         dtype=np.float64 if seed % 2 else np.float32, density=0.2,
                         dense_cells=0.5)
    check(sable, s, [1, 2, 4, 8][seed % 4])


def test_long_rows_and_shard(sable):
    from test_gpu_parity import long_rows_synth
    s = long_rows_synth()
    check(sable, s, 8)
    check(sable, s, 2, split="all_rem")
    c3 = gen.make("c3", scale=0.01)
    check(sable, c3, 4, rank=1, world=3)


def test_k_one_is_spmv(sable):
    s = gen.make("c2", scale=0.02)
    A = make(sable, s)
    try:
        x = torch.from_numpy(s.x).cuda()
        y = A.spmv(x).cpu().numpy()
        Y = A.spmm(x.reshape(-1, 1).contiguous()).cpu().numpy()[:, 0]
        yo, so = oracle.spmv(s.nrows, s.I, s.J, s.V.astype(np.float64), s.x.astype(np.float64))
        assert_y_close(y, yo, so, s.dtype, "spmv")
        assert np.array_equal(Y.view(np.uint8), y.view(np.uint8))  # same kernel, same order
    finally:
        A.close()


@pytest.mark.parametrize("k", [16, 32, 64, 128])
def test_tensor_core_k(sable, k):
    """k >= 16 on the tensor cores (tcgen05.mma kind::tf32, 3xTF32): every
    column within the SpMV tolerance of the oracle, deterministic."""
    check(sable, gen.make("c1"), k)
    check(sable, gen.random_small(70, 300, 280, 23, 19, density=0.3, dense_cells=0.5), k,
          split="all_vbr")


@pytest.mark.parametrize("name,scale", [("c2", 0.02), ("c4", 0.01), ("c5", 1 / 512)])
def test_tensor_core_configs(sable, name, scale):
    check(sable, gen.make(name, scale=scale), 32)


def test_tensor_core_long_rows_and_wide_panels(sable, monkeypatch):
    from test_gpu_parity import long_rows_synth
    check(sable, long_rows_synth(), 64)  # remainder pieces meet in the combine scratch
    monkeypatch.setenv("SABLE_USTAGE", "1024")  # panels cut into column chunks
    check(sable, gen.random_small(71, 64, 3000, 2, 3, density=0.2, dense_cells=0.7), 16)


def test_tensor_core_needs_fp32(sable):
    s = gen.random_small(72, 100, 90, 7, 6, dtype=np.float64)
    A = make(sable, s)
    try:
        X = torch.zeros((s.ncols, 16), dtype=torch.float64, device="cuda")
        with pytest.raises(sable.SableError) as e:
            A.spmm(X)
        assert e.value.status == sable.SABLE_E_UNSUPPORTED
    finally:
        A.close()


def test_bad_k(sable):
    s = gen.make("c1")
    A = make(sable, s)
    try:
        X = torch.zeros((s.ncols, 3), dtype=torch.float32, device="cuda")
        with pytest.raises(sable.SableError) as e:
            A.spmm(X)
        assert e.value.status == sable.SABLE_E_UNSUPPORTED
    finally:
        A.close()
