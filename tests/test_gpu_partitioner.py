"""Parity of the GPU partitioner (sable_partition_grid, Alg. 1 PAPER.md:381-416,
SURVEY 8(f) row f1) with the oracle's Alg. 1 (oracle_alg1): the row and column
grids must be identical (integer work: bit-exact).  Inputs are the seeded
generators of gen/ and tiny hand cases (paper examples, empty runs)."""
from fractions import Fraction

import numpy as np
import pytest

import gen
import oracle
from golden_io import coo, load

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def sable():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2407_00829_b200 import sable as s
    return s


def csr(nrows, I, J):
    I = np.asarray(I, np.int64)
    J = np.asarray(J, np.int64)
    o = np.lexsort((J, I))
    rp = np.zeros(nrows + 1, np.int64)
    np.cumsum(np.bincount(I, minlength=nrows), out=rp[1:])
    return rp, J[o].astype(np.int32)


def compare(sable, nrows, ncols, I, J, t, shifts, on_device=True):
    t = Fraction(t)
    rp, ci = csr(nrows, I, J)
    if on_device:
        r, c = sable.partition_grid(torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda(),
                                    ncols, t.numerator, t.denominator, shifts)
    else:
        r, c = sable.partition_grid(rp, ci, ncols, t.numerator, t.denominator, shifts)
    wr, wc = oracle.partition_grid(nrows, ncols, I, J, t.numerator, t.denominator, shifts)
    np.testing.assert_array_equal(r, wr)
    np.testing.assert_array_equal(c, wc)
    return r, c


@pytest.mark.parametrize("shifts", [False, True])
@pytest.mark.parametrize("t", [Fraction(1, 2), Fraction(9, 20), Fraction(4, 9), Fraction(0),
                               Fraction(1), Fraction(7, 10)])
def test_fig2(sable, t, shifts):
    A = load("fig2_vbr.txt")["A"]
    I, J, _ = coo(A)
    r, c = compare(sable, 11, 11, I, J, t, shifts)
    if t == Fraction(1, 2) and not shifts:
        assert r.tolist() == [0, 2, 5, 6, 9, 11] == c.tolist()  # the grid Fig. 2 draws


def test_sec5_example_and_edges(sable):
    A = np.array([[0, 1, 0, 0, 0], [1, 0, 0, 0, 0], [0, 1, 0, 0, 0]], dtype=float)
    for shifts in (False, True):
        compare(sable, 3, 5, *coo(A)[:2], Fraction(1, 2), shifts)
    # all-zero, one row, one column, empty runs at both ends
    compare(sable, 4, 6, [], [], Fraction(1, 2), True)
    compare(sable, 1, 1, [0], [0], Fraction(1, 2), True)
    compare(sable, 1, 9, [0, 0, 0], [1, 2, 8], Fraction(1, 2), False)
    compare(sable, 9, 1, [2, 3, 8], [0, 0, 0], Fraction(1, 2), False)
    compare(sable, 12, 7, [5, 5, 6], [0, 1, 1], Fraction(1, 2), True)


@pytest.mark.parametrize("seed", range(10))
def test_random_patterns(sable, seed):
    g = np.random.default_rng(100 + seed)
    m, n = int(g.integers(1, 400)), int(g.integers(1, 400))
    M = g.random((m, n)) < g.choice([0.002, 0.02, 0.2, 0.7])
    M[g.integers(0, m, m // 5)] = False  # empty-row runs
    I, J = np.nonzero(M)
    t = Fraction(int(g.integers(0, 21)), 20)
    compare(sable, m, n, I, J, t, bool(seed % 2), on_device=bool(seed % 3))


def test_long_rows(sable):
    # rows longer than a warp's stride and a dense band with +-1 shifts
    g = np.random.default_rng(7)
    n = 5000
    I, J = [], []
    for i in range(40):
        cols = np.sort(g.choice(n, 3000, replace=False)) if i % 7 else np.arange(i, n - 40 + i)
        I += [i] * len(cols)
        J += cols.tolist()
    for shifts in (False, True):
        compare(sable, 40, n, np.array(I), np.array(J), Fraction(1, 3), shifts)


@pytest.mark.parametrize("name", ["c1", "c2", "c5"])
def test_generated_configs(sable, name):
    s = gen.make(name, scale={"c1": 1.0, "c2": 0.05, "c5": 1 / 256}[name])
    for t, shifts in ((Fraction(1, 2), True), (Fraction(3, 10), False)):
        compare(sable, s.nrows, s.ncols, s.I, s.J, t, shifts)


def test_bad_arguments(sable):
    rp = np.array([0, 1], np.int64)
    ci = np.array([0], np.int32)
    with pytest.raises(sable.SableError):
        sable.partition_grid(rp, ci, 1, 1, 0, True)  # t_den = 0
