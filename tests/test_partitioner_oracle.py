"""Pins for the oracle's Alg. 1 partitioner (oracle_alg1 in
oracle/sable_oracle.c) -- against what the paper fixes:

* Fig. 2: the grid the paper draws, Rpntr = Cpntr =
  [0,2,5,6,9,11], is what Alg. 1 with Eq. 1 produces for
  thresholds t in (4/9, 1/2]; outside that window it is not (the boundary
  ratios 4/9 and 1/2 are the Fig. 2 row pairs (8,9)/(1,2) similarities);
* the shifted-rows example of Sec. 5: Eq. 1 "would register
  zero similarity between consecutive rows" (three row blocks), Eq. 2
   captures the block (one row block);
* the zero-row rule (Alg. 1 lines "if row i is empty"): runs of
  empty rows extend one block, the all-zero matrix is one block;
* brute force on tiny dense 0/1 matrices: the similarity from dense vectors
  and shifted copies (numpy), Alg. 1 stepped literally with exact fractions.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from golden_io import coo, load


def grid(A, t, shifts):
    t = Fraction(t)
    I, J, _ = coo(A)
    r, c = oracle.partition_grid(A.shape[0], A.shape[1], I, J, t.numerator, t.denominator, shifts)
    return r.tolist(), c.tolist()


# ---------------------------------------------------------------- brute force


def sim_dense(u, v, shifts):
    """Eq. 1 / Eq. 2 on dense 0/1 vectors; shifts move u one place right/left."""
    u = (u != 0).astype(np.int64)
    v = (v != 0).astype(np.int64)
    dots = [int(u @ v)]
    if shifts:
        right = np.concatenate([[0], u[:-1]])
        left = np.concatenate([u[1:], [0]])
        dots += [int(right @ v), int(left @ v)]
    den = max(int(u.sum()), int(v.sum()))
    return Fraction(max(dots), den) if den else Fraction(0)


def alg1_dense(M, t, shifts):
    """Alg. 1 stepped literally on the rows of dense M."""
    n = M.shape[0]
    cuts = []
    i = 0
    while i < n - 1:
        if not M[i].any():
            while i < n - 1 and not M[i + 1].any():
                i += 1
            cuts.append(i + 1)
        elif sim_dense(M[i], M[i + 1], shifts) < t:
            cuts.append(i + 1)
        i += 1
    cuts.append(n)
    out = [0]
    for c in cuts:  # reading R19: a cut equal to the previous one is not a new block
        if c != out[-1]:
            out.append(c)
    return out


# ------------------------------------------------------------- paper examples


@pytest.mark.parametrize("t", [Fraction(1, 2), Fraction(9, 20), Fraction(4, 9) + Fraction(1, 1000)])
def test_fig2_grid_from_eq1(t):
    A = load("fig2_vbr.txt")["A"]
    r, c = grid(A, t, False)
    assert r == [0, 2, 5, 6, 9, 11] and c == [0, 2, 5, 6, 9, 11]


@pytest.mark.parametrize("t", [Fraction(4, 9), Fraction(5, 9), Fraction(1, 10), Fraction(9, 10)])
def test_fig2_grid_outside_window_differs(t):
    A = load("fig2_vbr.txt")["A"]
    r, _ = grid(A, t, False)
    assert r != [0, 2, 5, 6, 9, 11]


def test_fig2_eq2_merges_shifted_columns():
    """Eq. 2 at 1/2 keeps the Fig. 2 rows but merges column blocks 2 and 3
    (columns 5 and 6..8 are +-1 shifts of each other)."""
    A = load("fig2_vbr.txt")["A"]
    r, c = grid(A, Fraction(1, 2), True)
    assert r == [0, 2, 5, 6, 9, 11]
    assert c == [0, 2, 5, 9, 11]


def test_sec5_shifted_rows_example():
    A = np.array([[0, 1, 0, 0, 0], [1, 0, 0, 0, 0], [0, 1, 0, 0, 0]], dtype=float)
    r1, c1 = grid(A, Fraction(1, 2), False)
    assert r1 == [0, 1, 2, 3]  # Eq. 1: zero similarity between consecutive rows
    r2, c2 = grid(A, Fraction(1, 2), True)
    assert r2 == [0, 3]  # Eq. 2: one block row
    # columns: 0 and 1 are shifts of each other; 2..4 are empty and extend a block
    assert c1 == [0, 1, 2, 5] and c2 == [0, 2, 5]


def test_zero_matrix_is_one_block():
    A = np.zeros((4, 6))
    assert grid(A, Fraction(1, 2), False) == ([0, 4], [0, 6])
    assert grid(A, Fraction(1, 2), True) == ([0, 4], [0, 6])


def test_identity():
    A = np.eye(4)
    assert grid(A, Fraction(1, 2), False) == ([0, 1, 2, 3, 4], [0, 1, 2, 3, 4])
    assert grid(A, Fraction(1, 2), True) == ([0, 4], [0, 4])


def test_empty_rows_extend_block():
    A = np.zeros((7, 3))
    A[0, 0] = A[4, 1] = A[5, 1] = 1
    r, _ = grid(A, Fraction(1, 2), False)
    # row 0 vs empty row 1: similarity 0 -> cut at 1; rows 1..3 empty -> one
    # block ending before row 4; rows 4,5 identical; row 5 vs empty row 6:
    # similarity 0 -> cut at 6
    assert r == [0, 1, 4, 6, 7]


def test_single_row_and_column():
    A = np.ones((1, 1))
    assert grid(A, Fraction(1, 2), True) == ([0, 1], [0, 1])
    A = np.array([[1, 0, 1, 1]], dtype=float)
    assert grid(A, Fraction(1, 2), False) == ([0, 1], [0, 1, 2, 4])


def test_threshold_zero_never_cuts_between_nonempty_rows():
    g = np.random.default_rng(5)
    A = (g.random((30, 20)) < 0.4).astype(float)
    A[A.sum(1) == 0, 0] = 1
    r, _ = grid(A, Fraction(0), False)
    assert r == [0, 30]


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("shifts", [False, True])
def test_brute_force_tiny(seed, shifts):
    g = np.random.default_rng(seed)
    m, n = g.integers(1, 14, 2)
    # banded / blocky / empty-run structure so that all branches of Alg. 1 run
    dens = g.choice([0.05, 0.2, 0.5, 0.8])
    M = g.random((m, n)) < dens
    if seed % 3 == 0:
        M[g.integers(0, m, 2)] = False
        M[:, g.integers(0, n, 2)] = False
    t = Fraction(int(g.integers(0, 11)), 10)
    r, c = grid(M.astype(float), t, shifts)
    assert r == alg1_dense(M, t, shifts)
    assert c == alg1_dense(M.T, t, shifts)
