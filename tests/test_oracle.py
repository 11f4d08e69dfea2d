"""Pins for the CPU oracle (oracle/sable_oracle.c) against what the paper and
the mathematics fix -- never against the oracle's own formulas.

* worked examples printed in the paper: Fig. 2, Fig. 3
  (PAPER.md:285-321), Fig. 4a/Fig. 6, Listing 2
  (PAPER.md:598-604);
* closed forms: y on the worked examples, dense brute force (numpy slicing of
  the dense matrix, an independent definition of the cell counts, tiles and
  remainder), scipy CSR matvec at delta = 101, GEMV for one full block, the
  diagonal for 1x1 blocks;
* invariants of BASELINE.json north_star s10 and SURVEY 8(c).
"""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle
from golden_io import coo, load

# ---------------------------------------------------------------- helpers


def brute_partition(A, rpntr, cpntr, delta, min_area=0, rules=()):
    """The partition by definition, on a dense matrix: slice every grid cell.
    min_area / rules: the per-shape policy of reading R22 (first matching
    (h_min, h_max, w_min, w_max, delta) rule, else `delta`)."""
    cells, tiles, offs, ub = [], [], [0], []
    mask_rem = np.zeros(A.shape, dtype=bool)
    for a in range(len(rpntr) - 1):
        for b in range(len(cpntr) - 1):
            sub = A[rpntr[a]:rpntr[a + 1], cpntr[b]:cpntr[b + 1]]
            cnt = int(np.count_nonzero(sub))
            if cnt == 0:
                continue
            h, w = sub.shape
            d = next((r[4] for r in rules if r[0] <= h <= r[1] and r[2] <= w <= r[3]), delta)
            dense = h * w >= min_area and cnt * 100 >= d * h * w
            if dense:
                tiles.append(sub.flatten(order="F"))
                offs.append(offs[-1] + h * w)
            else:
                ub.append(len(cells))
                mask_rem[rpntr[a]:rpntr[a + 1], cpntr[b]:cpntr[b + 1]] = True
            cells.append((a, b, cnt, int(dense)))
    R = sp.csr_matrix(np.where(mask_rem, A, 0.0))
    R.sort_indices()
    return dict(
        cells=np.array(cells, dtype=np.int64).reshape(-1, 4),
        tile_val=np.concatenate(tiles) if tiles else np.zeros(0),
        tile_off=np.array(offs, dtype=np.int64), ublocks=np.array(ub, dtype=np.int64),
        rem_indptr=R.indptr.astype(np.int64), rem_indices=R.indices.astype(np.int64),
        rem_val=R.data)


def run(A, rpntr, cpntr, delta, a0=0, a1=None, min_area=0, rules=None):
    I, J, V = coo(A)
    return oracle.partition(A.shape[0], A.shape[1], I, J, V, rpntr, cpntr, delta, a0, a1,
                            min_area=min_area, rules=rules)


def cells_of(p):
    return np.stack([p["cell_br"], p["cell_bc"], p["cell_cnt"], p["cell_dense"]],
                    axis=1).astype(np.int64).reshape(-1, 4)


def assert_same(p, b):
    np.testing.assert_array_equal(cells_of(p), b["cells"])
    np.testing.assert_array_equal(p["tile_off"], b["tile_off"])
    np.testing.assert_array_equal(p["tile_val"], b["tile_val"])
    np.testing.assert_array_equal(p["ublocks"], b["ublocks"])
    np.testing.assert_array_equal(p["rem_indptr"], b["rem_indptr"])
    np.testing.assert_array_equal(p["rem_indices"], b["rem_indices"])
    np.testing.assert_array_equal(p["rem_val"], b["rem_val"])


def random_case(seed, m, n, nbr, nbc, dens=0.3, ints=True):
    g = np.random.default_rng(seed)
    rp = np.concatenate([[0], np.sort(g.choice(np.arange(1, m), nbr - 1, replace=False)), [m]])
    cp = np.concatenate([[0], np.sort(g.choice(np.arange(1, n), nbc - 1, replace=False)), [n]])
    # cell-wise densities so that dense, sparse and empty cells all occur
    cd = g.choice([0.0, 0.1, 0.5, 0.9, 1.0], size=(nbr, nbc))
    P = np.repeat(np.repeat(cd, np.diff(rp), 0), np.diff(cp), 1)
    M = g.random((m, n)) < P * (dens / 0.3)
    if ints:
        A = np.where(M, g.integers(1, 9, (m, n)) * g.choice([-1, 1], (m, n)), 0).astype(float)
    else:
        A = np.where(M, g.standard_normal((m, n)), 0.0)
    return A, rp.astype(np.int32), cp.astype(np.int32)


# ---------------------------------------------------------- worked examples


def test_fig2_vbr_arrays_verbatim():
    """Fig. 2b: with every non-empty cell kept dense
    (delta = 0), the tiles are Val, their offsets Indx, their block columns
    Bindx, and the per-block-row counts give Bpntrb / Bpntre."""
    g = load("fig2_vbr.txt")
    p = run(g["A"], g["Rpntr"], g["Cpntr"], 0)
    assert p["n_cells"] == 13 and p["n_dense"] == 13
    np.testing.assert_array_equal(p["tile_val"], g["Val"])
    np.testing.assert_array_equal(p["tile_off"], g["Indx"])
    np.testing.assert_array_equal(p["cell_bc"], g["Bindx"])
    per_row = np.bincount(p["cell_br"], minlength=len(g["Rpntr"]) - 1)
    bpntre = np.cumsum(per_row)
    np.testing.assert_array_equal(bpntre, g["Bpntre"])
    np.testing.assert_array_equal(bpntre - per_row, g["Bpntrb"])
    # 51 stored values, 47 of them non-zero (the 4 zeros sit in green, pink,
    # CadetBlue and Thistle)
    assert p["tile_elems"] == 51 and p["nnz"] == 47 and p["cell_cnt"].sum() == 47


@pytest.mark.parametrize("delta", [67, 75, 88])
def test_fig3_vbrc_arrays(delta):
    """Fig. 3b is reproduced by every integer delta in
    [67, 88] (reading R2)."""
    g = load("fig3_vbrc.txt")
    p = run(g["A"], g["Rpntr"], g["Cpntr"], delta)
    np.testing.assert_array_equal(p["ublocks"], g["ublocks"])
    np.testing.assert_array_equal(p["rem_indptr"], g["indptr"])
    np.testing.assert_array_equal(p["rem_indices"], g["indices"])
    np.testing.assert_array_equal(p["rem_val"], g["csr_val"])
    np.testing.assert_array_equal(p["tile_val"], g["Val"])
    np.testing.assert_array_equal(p["tile_off"], [0, 4, 6, 15, 17, 20, 21, 24, 33, 37])


@pytest.mark.parametrize("delta,ub", [(0, []), (50, []), (51, [2, 12]), (66, [2, 12]),
                                      (67, [2, 4, 9, 12]), (89, [2, 4, 9, 10, 12]),
                                      (101, list(range(13)))])
def test_fig3_delta_sweep(delta, ub):
    """Tie rule 'at least delta %' (reading R1): green and
    Gray are exactly 50% dense, pink and CadetBlue 66.7%, Thistle 88.9%."""
    g = load("fig3_vbrc.txt")
    p = run(g["A"], g["Rpntr"], g["Cpntr"], delta)
    np.testing.assert_array_equal(p["ublocks"], ub)


def test_fig4_fig6_tile_offsets():
    """Fig. 6 reads A_val at offsets 0, 8, 14, 18."""
    g = load("fig4_fig6.txt")
    for delta in (0, 50, 66):
        p = run(g["A"], g["Rpntr"], g["Cpntr"], delta)
        np.testing.assert_array_equal(p["tile_off"], g["tile_off"])
    # at 67 the 2x3 blue block (4/6 = 66.7%) leaves for the remainder
    p = run(g["A"], g["Rpntr"], g["Cpntr"], 67)
    np.testing.assert_array_equal(p["tile_off"], [0, 8, 12, 15])
    np.testing.assert_array_equal(p["rem_indices"], [7, 8, 6, 8])


def test_listing2_offset_arithmetic():
    """Listing 2: element (i, j) of the 50x60 block at rows
    640..689, cols 4175..4234 is val[69722 + (j-4175)*50 + i-640]; the next
    block starts at 72722."""
    rp = np.array([0, 2, 640, 690], dtype=np.int32)
    cp = np.array([0, 4175, 4235, 34861], dtype=np.int32)
    I1, J1 = np.meshgrid(np.arange(2), np.arange(34861), indexing="ij")
    I2, J2 = np.meshgrid(np.arange(640, 690), np.arange(4175, 4235), indexing="ij")
    I = np.concatenate([I1.ravel(), I2.ravel()]).astype(np.int64)
    J = np.concatenate([J1.ravel(), J2.ravel()]).astype(np.int64)
    V = (I * 100000 + J + 1).astype(np.float64)
    o = np.lexsort((J, I))
    p = oracle.partition(690, 34861, I[o], J[o], V[o], rp, cp, 50)
    np.testing.assert_array_equal(p["tile_off"], [0, 8350, 8470, 69722, 72722])
    for i in (640, 641, 689):
        for j in (4175, 4200, 4234):
            assert p["tile_val"][69722 + (j - 4175) * 50 + i - 640] == i * 100000 + j + 1


def test_y_worked_examples():
    """Closed forms (SURVEY 8(c) 'y, from worked examples')."""
    A2 = load("fig2_vbr.txt")["A"]
    A3 = load("fig3_vbrc.txt")["A"]
    one = np.ones(11)
    y, s = oracle.spmv(11, *coo(A2), one)
    np.testing.assert_array_equal(y, [7, 7, 11, 10, 13, 34, 23, 20, 9, 40, 21])
    np.testing.assert_array_equal(s, [9, 9, 11, 10, 15, 34, 23, 20, 9, 40, 25])
    y, _ = oracle.spmv(11, *coo(A2), np.arange(1, 12, dtype=float))
    np.testing.assert_array_equal(y, [15, 12, 44, 39, 68, 184, 165, 154, 77, 299, 216])
    y, _ = oracle.spmv(11, *coo(A3), one)
    np.testing.assert_array_equal(y, [8, 7, 11, 10, 13, 34, 23, 20, 9, 37, 9])


def test_fig3_dense_remainder_split_of_y():
    """y splits into the dense-tile part and the remainder part at delta=75:
    y_dense = [7,8,9,10,10,34,19,17,9,12,1], y_rem = [1,-1,2,0,3,0,4,3,0,25,8]."""
    g = load("fig3_vbrc.txt")
    p = run(g["A"], g["Rpntr"], g["Cpntr"], 75)
    R = sp.csr_matrix((p["rem_val"], p["rem_indices"], p["rem_indptr"]), shape=(11, 11))
    np.testing.assert_array_equal(R @ np.ones(11), [1, -1, 2, 0, 3, 0, 4, 3, 0, 25, 8])
    # dense part = y - remainder, via the tiles placed back
    D = np.zeros((11, 11))
    k = 0
    for (a, b, _, d) in cells_of(p):
        if d:
            r0, r1, c0, c1 = g["Rpntr"][a], g["Rpntr"][a + 1], g["Cpntr"][b], g["Cpntr"][b + 1]
            D[r0:r1, c0:c1] = p["tile_val"][p["tile_off"][k]:p["tile_off"][k + 1]].reshape(
                (r1 - r0, c1 - c0), order="F")
            k += 1
    np.testing.assert_array_equal(D @ np.ones(11), [7, 8, 9, 10, 10, 34, 19, 17, 9, 12, 1])


# ------------------------------------------------------------- brute force


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("delta", [0, 30, 50, 75, 100, 101])
def test_partition_matches_dense_brute_force(seed, delta):
    g = np.random.default_rng(1000 + seed)
    m, n = int(g.integers(1, 60)), int(g.integers(1, 60))
    nbr, nbc = int(g.integers(1, m + 1)), int(g.integers(1, n + 1))
    A, rp, cp = random_case(seed, m, n, nbr, nbc) if m > 1 and n > 1 else (
        np.where(g.random((m, n)) < 0.5, 1.0, 0.0), np.array([0, m], np.int32),
        np.array([0, n], np.int32))
    assert_same(run(A, rp, cp, delta), brute_partition(A, rp, cp, delta))


@pytest.mark.parametrize("seed", range(8))
def test_y_matches_dense_matvec(seed):
    A, rp, cp = random_case(seed, 48, 37, 7, 5, ints=True)
    x = np.random.default_rng(seed).integers(-8, 9, 37).astype(float)
    y, s = oracle.spmv(48, *coo(A), x)
    np.testing.assert_array_equal(y, A @ x)       # small integers: exact
    np.testing.assert_array_equal(s, np.abs(A) @ np.abs(x))
    A, rp, cp = random_case(seed, 48, 37, 7, 5, ints=False)
    x = np.random.default_rng(seed).standard_normal(37)
    y, s = oracle.spmv(48, *coo(A), x)
    assert np.all(np.abs(y - A @ x) <= 1e-14 * (s + 1e-300))


# ---------------------------------------------------------- special cases


def test_delta101_is_the_input_csr():
    """delta = 101: nothing is dense, the remainder is the whole CSR matrix
    (SPEC 'decide == Sparse'); its product is scipy's CSR matvec."""
    A, rp, cp = random_case(3, 40, 50, 6, 6, ints=False)
    p = run(A, rp, cp, 101)
    C = sp.csr_matrix(A)
    C.sort_indices()
    np.testing.assert_array_equal(p["rem_indptr"], C.indptr)
    np.testing.assert_array_equal(p["rem_indices"], C.indices)
    np.testing.assert_array_equal(p["rem_val"], C.data)
    assert p["n_dense"] == 0 and len(p["tile_val"]) == 0
    x = np.random.default_rng(0).standard_normal(50)
    y, s = oracle.spmv(40, *coo(A), x)
    np.testing.assert_allclose(y, C @ x, rtol=0, atol=1e-13 * s.max())


def test_delta0_every_candidate_dense():
    A, rp, cp = random_case(4, 40, 40, 8, 8)
    p = run(A, rp, cp, 0)
    assert p["n_dense"] == p["n_cells"] and p["rem_nnz"] == 0
    assert np.all(p["cell_cnt"] >= 1)


def test_single_full_block_is_gemv():
    g = np.random.default_rng(7)
    A = g.integers(1, 9, (13, 17)).astype(float)
    x = g.integers(-8, 9, 17).astype(float)
    p = run(A, [0, 13], [0, 17], 100)
    assert p["n_dense"] == 1
    np.testing.assert_array_equal(p["tile_val"], A.flatten(order="F"))
    y, _ = oracle.spmv(13, *coo(A), x)
    np.testing.assert_array_equal(y, A @ x)


def test_diagonal_1x1_blocks():
    """1x1 blocks on the diagonal: y_i = a_ii x_i; unit values give y = x."""
    d = np.arange(1, 10, dtype=float)
    A = np.diag(d)
    grid = np.arange(10, dtype=np.int32)
    p = run(A, grid, grid, 50)
    assert p["n_dense"] == 9 and p["rem_nnz"] == 0
    np.testing.assert_array_equal(p["tile_val"], d)
    x = np.arange(9, dtype=float) - 4
    y, _ = oracle.spmv(9, *coo(A), x)
    np.testing.assert_array_equal(y, d * x)
    y, _ = oracle.spmv(9, *coo(np.eye(9)), x)
    np.testing.assert_array_equal(y, x)


def test_empty_matrix_and_empty_rows():
    A = np.zeros((5, 7))
    p = run(A, [0, 2, 5], [0, 3, 7], 50)
    assert p["n_cells"] == 0 and p["rem_nnz"] == 0
    np.testing.assert_array_equal(p["rem_indptr"], np.zeros(6))
    y, s = oracle.spmv(5, *coo(A), np.ones(7))
    assert not y.any() and not s.any()


# ------------------------------------------------------------- invariants


@pytest.mark.parametrize("seed", range(6))
def test_invariants(seed):
    """north_star s10: block nnz + remainder nnz = nnz; every dense block meets
    delta, every other candidate does not; zero fill = area - cnt; dense sets
    shrink as delta grows."""
    A, rp, cp = random_case(50 + seed, 64, 64, 9, 11)
    prev = None
    for delta in range(0, 102, 17):
        p = run(A, rp, cp, delta)
        h = np.diff(rp)[p["cell_br"]].astype(np.int64)
        w = np.diff(cp)[p["cell_bc"]].astype(np.int64)
        d = p["cell_dense"].astype(bool)
        assert p["cell_cnt"][d].sum() + p["rem_nnz"] == np.count_nonzero(A)
        assert np.all(100 * p["cell_cnt"][d] >= delta * h[d] * w[d])
        assert np.all(100 * p["cell_cnt"][~d] < delta * h[~d] * w[~d])
        assert np.count_nonzero(p["tile_val"] == 0) == (h[d] * w[d] - p["cell_cnt"][d]).sum()
        np.testing.assert_array_equal(np.flatnonzero(~d), p["ublocks"])
        key = set(zip(p["cell_br"][d].tolist(), p["cell_bc"][d].tolist()))
        if prev is not None:
            assert key <= prev
        prev = key


def test_block_row_ranges_concatenate_to_full():
    """Shard exports (block-row ranges) concatenate to the full export."""
    A, rp, cp = random_case(9, 70, 60, 10, 8)
    full = run(A, rp, cp, 50)
    parts = [run(A, rp, cp, 50, a0, a1) for a0, a1 in [(0, 3), (3, 3), (3, 7), (7, 10)]]
    cells = np.concatenate([cells_of(q) for q in parts])
    np.testing.assert_array_equal(cells, cells_of(full))
    base, ub = 0, []
    for q in parts:
        ub.append(q["ublocks"] + base)
        base += q["n_cells"]
    np.testing.assert_array_equal(np.concatenate(ub), full["ublocks"])
    np.testing.assert_array_equal(np.concatenate([q["tile_val"] for q in parts]), full["tile_val"])
    ptr = [np.zeros(1, np.int64)]
    off = 0
    for q in parts:
        ptr.append(q["rem_indptr"][1:] + off)
        off += q["rem_nnz"]
    np.testing.assert_array_equal(np.concatenate(ptr), full["rem_indptr"])
    np.testing.assert_array_equal(np.concatenate([q["rem_val"] for q in parts]), full["rem_val"])


# ------------------------------------------------------------ normalisation


def test_normalize_sorts_drops_zeros_rejects_duplicates():
    I = [2, 0, 1, 0, 1]
    J = [1, 3, 0, 1, 2]
    V = [1.0, -0.0, 3.0, 0.0, float("nan")]
    I2, J2, V2 = oracle.normalize(3, 4, I, J, V)
    np.testing.assert_array_equal(I2, [1, 1, 2])
    np.testing.assert_array_equal(J2, [0, 2, 1])
    assert V2[0] == 3.0 and np.isnan(V2[1]) and V2[2] == 1.0
    with pytest.raises(oracle.OracleError):
        oracle.normalize(3, 4, [0, 0], [1, 1], [1.0, 2.0])
    with pytest.raises(oracle.OracleError):
        oracle.normalize(3, 4, [3], [0], [1.0])
    with pytest.raises(oracle.OracleError):
        oracle.partition(3, 4, [0], [0], [1.0], [0, 2, 2, 3], [0, 4], 50)  # not strictly increasing


def test_spmv_rows_sample_equals_full():
    A, rp, cp = random_case(11, 50, 50, 5, 5, ints=False)
    I, J, V = coo(A)
    x = np.random.default_rng(1).standard_normal(50)
    y, s = oracle.spmv(50, I, J, V, x)
    rows = np.array([0, 7, 7, 49, 23])
    ys, ss = oracle.spmv_rows(oracle.rowptr(50, I), J, V, x, rows)
    np.testing.assert_array_equal(ys, y[rows])
    np.testing.assert_array_equal(ss, s[rows])


# ------------------------------------------------- per-shape delta policy (f2)


def random_rules(g, k):
    rules = []
    for _ in range(k):
        h0, w0 = int(g.integers(1, 6)), int(g.integers(1, 6))
        rules.append((h0, h0 + int(g.integers(0, 6)), w0, w0 + int(g.integers(0, 6)),
                      int(g.choice([0, 25, 50, 67, 80, 101]))))
    return rules


@pytest.mark.parametrize("seed", range(12))
def test_policy_matches_brute_force(seed):
    """Reading R22 on random grids: the first matching shape rule's delta,
    min_area, cell counts by slicing the dense matrix."""
    g = np.random.default_rng(100 + seed)
    A, rp, cp = random_case(100 + seed, 40, 37, 9, 8)
    rules = random_rules(g, int(g.integers(1, 5)))
    min_area = int(g.choice([0, 1, 4, 9, 30]))
    delta = int(g.choice([0, 50, 75, 101]))
    assert_same(run(A, rp, cp, delta, min_area=min_area, rules=rules),
                brute_partition(A, rp, cp, delta, min_area, rules))


@pytest.mark.parametrize("delta", [0, 50, 67, 101])
def test_policy_special_cases(delta):
    A, rp, cp = random_case(7, 50, 45, 10, 9)
    plain = run(A, rp, cp, delta)
    # a rule over every shape, or min_area 1 with no rule: the plain delta rule
    assert_same(run(A, rp, cp, 3, rules=[(1, 50, 1, 45, delta)]), brute_partition(A, rp, cp, delta))
    assert_same(run(A, rp, cp, delta, min_area=1), brute_partition(A, rp, cp, delta))
    for k in ("cell_dense", "tile_val", "rem_indices"):
        np.testing.assert_array_equal(run(A, rp, cp, delta, min_area=1)[k], plain[k])
    # min_area above every cell: nothing dense, the remainder is the input CSR
    big = run(A, rp, cp, delta, min_area=50 * 45 + 1)
    assert big["n_dense"] == 0
    R = sp.csr_matrix(A)
    np.testing.assert_array_equal(big["rem_indptr"], R.indptr)
    np.testing.assert_array_equal(big["rem_indices"], R.indices)


def test_policy_first_rule_wins_and_monotone():
    A, rp, cp = random_case(8, 60, 60, 12, 12)
    r_lo = [(1, 60, 1, 60, 30)]
    r_hi = [(1, 60, 1, 60, 90)]
    lo = run(A, rp, cp, 50, rules=r_lo + r_hi)
    assert_same(lo, brute_partition(A, rp, cp, 30))
    hi = run(A, rp, cp, 50, rules=r_hi + r_lo)
    assert_same(hi, brute_partition(A, rp, cp, 90))
    # delta-monotone under a policy too: raising every rule's delta keeps a subset dense
    d_lo, d_hi = lo["cell_dense"].astype(bool), hi["cell_dense"].astype(bool)
    assert np.all(d_hi <= d_lo)
