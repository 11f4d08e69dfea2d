"""Parity of the CUDA path (through the C-ABI) with the CPU oracle.

Partition: byte-identical canonical export (cells, tiles, ublocks, remainder).
y: |y_gpu - y_oracle| <= tol * sum|a||x| (1e-5 fp32, 1e-12 fp64), bitwise for
small integers.  Inputs are the seeded generators of gen/ (never a GPU
output), at sizes the oracle finishes in seconds that span many work items
and ragged tails, plus the paper's worked examples and edge cases.
"""
import numpy as np
import pytest

import gen
import oracle
from golden_io import load
from parity import (assert_partition_equal, assert_y_close, oracle_partition,
                    slice_export)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def sable():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2407_00829_b200 import sable as s
    return s


def from_dense(A, rpntr, cpntr, dtype=np.float32, delta=50, x=None, name="dense"):
    I, J = np.nonzero(A)
    V = A[I, J].astype(dtype)
    if x is None:
        x = np.arange(1, A.shape[1] + 1).astype(dtype)
    s = gen.Synth(name=name, nrows=A.shape[0], ncols=A.shape[1], dtype=dtype, delta=delta,
                  rpntr=np.asarray(rpntr, np.int32), cpntr=np.asarray(cpntr, np.int32),
                  rects=np.zeros((0, 4), np.int64), I=I.astype(np.int64), J=J.astype(np.int64),
                  V=V, x=np.asarray(x, dtype), in_rect=np.zeros(len(I), bool))
    return s


def to_dev(inp):
    return {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in inp.items()
            if isinstance(v, np.ndarray)}


def handle(sable, s, split="rect", delta=None, on_device=True, rank=0, world=1, inp=None):
    inp = inp if inp is not None else s.vbr_input(split)
    arrays = to_dev(inp) if on_device else {k: v for k, v in inp.items() if isinstance(v, np.ndarray)}
    return sable.VbrMatrix(arrays, s.nrows, s.ncols, delta=s.delta if delta is None else delta,
                           rank=rank, world=world)


def check(sable, s, split="rect", delta=None, on_device=True, exact=False):
    d = s.delta if delta is None else delta
    A = handle(sable, s, split, d, on_device)
    try:
        got = A.export()
        want = oracle.partition(s.nrows, s.ncols, s.I, s.J, s.V.astype(np.float64), s.rpntr,
                                s.cpntr, d)
        assert_partition_equal(got, want, s.dtype, f"{s.name}/{split}/d{d}")
        y = A.spmv(torch.from_numpy(s.x).cuda()).cpu().numpy()
        yo, so = oracle.spmv(s.nrows, s.I, s.J, s.V.astype(np.float64), s.x.astype(np.float64))
        if exact:
            np.testing.assert_array_equal(y.astype(np.float64), yo)
        else:
            assert_y_close(y, yo, so, s.dtype, f"{s.name}/{split}/d{d}")
        info = A.info
        assert info["nnz"] == s.nnz
        assert info["n_dense"] == len(want["tile_off"]) - 1
        return A, y
    except Exception:
        A.close()
        raise


# ------------------------------------------------------------------ worked examples

@pytest.mark.parametrize("delta", [0, 50, 75, 89, 101])
@pytest.mark.parametrize("split", ["all_vbr", "all_rem", "rect"])
def test_fig2_fig3(sable, split, delta):
    for name in ("fig2_vbr.txt", "fig3_vbrc.txt"):
        g = load(name)
        s = from_dense(g["A"], g["Rpntr"], g["Cpntr"], np.float32, delta, np.ones(11, np.float32),
                       name=name)
        s.in_rect = (s.I + s.J) % 2 == 0  # an arbitrary split: the partition must not care
        A, y = check(sable, s, split, exact=True)
        A.close()


def test_fig3_paper_arrays_from_gpu(sable):
    """The Fig. 3b VBR-C arrays come out of the GPU
    inspector at delta = 75, from the Fig. 2-style VBR input that still stores
    the sparse blocks with their zeros."""
    g = load("fig3_vbrc.txt")
    s = from_dense(g["A"], g["Rpntr"], g["Cpntr"], np.float32, 75, np.ones(11, np.float32))
    inp = s.vbr_input("all_vbr")
    A = handle(sable, s, inp=inp)
    got = A.export()
    np.testing.assert_array_equal(got["ublocks"], g["ublocks"])
    np.testing.assert_array_equal(got["rem_indptr"], g["indptr"])
    np.testing.assert_array_equal(got["rem_indices"], g["indices"])
    np.testing.assert_array_equal(got["rem_val"], g["csr_val"])
    np.testing.assert_array_equal(got["tile_val"], g["Val"])
    np.testing.assert_array_equal(A.spmv(torch.ones(11, device="cuda")).cpu().numpy(),
                                  [8, 7, 11, 10, 13, 34, 23, 20, 9, 37, 9])
    A.close()


# ------------------------------------------------------------------ C1 and random cases

@pytest.mark.parametrize("split", ["rect", "all_vbr", "all_rem"])
@pytest.mark.parametrize("delta", [0, 50, 75, 101])
def test_c1(sable, split, delta):
    s = gen.make("c1")
    A, _ = check(sable, s, split, delta)
    A.close()


@pytest.mark.parametrize("seed", range(16))
def test_random_small(sable, seed):
    g = np.random.default_rng(seed)
    m, n = int(g.integers(1, 300)), int(g.integers(1, 300))
    nbr, nbc = int(g.integers(1, max(2, m // 2))), int(g.integers(1, max(2, n // 2)))
    dt = np.float64 if seed % 2 else np.float32
    s = gen.random_small(seed, m, n, min(nbr, m), min(nbc, n), dtype=dt,
                         values="int" if seed % 3 == 0 else "u11",
                         delta=int(g.choice([0, 30, 50, 80, 101])))
    for split in ("rect", "all_rem", "all_vbr"):
        A, _ = check(sable, s, split, exact=seed % 3 == 0)
        A.close()


@pytest.mark.parametrize("shape", [
    (1000, 800, 7, 5),      # tall block rows: h >> 32 (several row groups)
    (64, 5000, 2, 3),       # wide panels: W > 512 columns (split pieces)
    (300, 300, 300, 300),   # 1x1 cells everywhere (nr = 1 groups)
    (1, 1000, 1, 10),       # a single row
    (1000, 1, 10, 1),       # a single column
])
@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_shapes(sable, shape, dt):
    m, n, nbr, nbc = shape
    s = gen.random_small(7, m, n, nbr, nbc, dtype=dt, density=0.2, dense_cells=0.5)
    A, _ = check(sable, s, "rect")
    A.close()


def long_rows_synth():
    g = np.random.default_rng(3)
    A_ = np.zeros((40, 20000))
    A_[5, :] = g.integers(1, 4, 20000)            # a full row (remainder at delta = 101)
    A_[7, g.choice(20000, 9000, replace=False)] = 2.0
    A_[20:23, :] = (g.random((3, 20000)) < 0.1) * 3.0
    A_[30:40, :50] = g.integers(1, 3, (10, 50))   # medium rows: warp-cooperative sums
    rp = [0, 5, 6, 7, 8, 40]
    cp = [0, 5000, 10000, 15000, 20000]
    return from_dense(A_, rp, cp, np.float32, 101, g.integers(-2, 3, 20000).astype(np.float32),
                      name="longrows")


def test_long_remainder_rows(sable):
    """Rows with thousands of remainder entries are split over several work
    items and combined in a fixed order (bitwise equal to the oracle on small
    integers)."""
    s = long_rows_synth()
    M, _ = check(sable, s, "all_rem", exact=True)
    assert M.info["n_combine"] > 0  # rows split over several units
    M.close()


def test_integer_values_bitwise(sable):
    s = gen.random_small(11, 257, 263, 17, 19, dtype=np.float32, values="int")
    for split in ("rect", "all_rem"):
        A, _ = check(sable, s, split, exact=True)
        A.close()


# ------------------------------------------------------------------ edge cases

@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("split", ["rect", "all_rem", "all_vbr"])
def test_special_values(sable, dt, split):
    """Reading R4 on the GPU: a non-zero is any bit pattern but +-0, so NaN
    and subnormal values count (and are stored bit-exactly) while -0 and +0
    stored in val or the remainder do not; a row holding a NaN is NaN in y
    (x finite), every other row within the tolerance."""
    s = gen.random_small(41, 301, 277, 23, 19, dtype=dt, density=0.3, dense_cells=0.4)
    g = np.random.default_rng(41)
    n = s.nnz
    pick = g.permutation(n)
    tiny = np.finfo(dt).tiny
    V = s.V.copy()
    V[pick[:5]] = dt(np.nan)
    V[pick[5:40]] = (tiny * g.uniform(0.01, 0.9, 35)).astype(dt)   # subnormal
    V[pick[40:60]] = dt(-0.0)
    V[pick[60:80]] = dt(0.0)
    assert np.isnan(V).sum() == 5 and (np.abs(V[pick[5:40]]) < tiny).all()
    s.V = V
    inp = s.vbr_input(split)  # +-0 entries stay stored in val / the remainder
    A = handle(sable, s, inp=inp)
    try:
        got = A.export()
        keep = ~((V == 0) & ~np.isnan(V))
        want = oracle.partition(s.nrows, s.ncols, s.I[keep], s.J[keep], V[keep].astype(np.float64),
                                s.rpntr, s.cpntr, s.delta)
        assert_partition_equal(got, want, dt, f"special/{split}")
        assert A.info["nnz"] == int(keep.sum())
        y = A.spmv(torch.from_numpy(s.x).cuda()).cpu().numpy().astype(np.float64)
        yo, so = oracle.spmv(s.nrows, s.I[keep], s.J[keep], V[keep].astype(np.float64),
                             s.x.astype(np.float64))
        nan = np.isnan(yo)
        assert nan.sum() >= 1 and np.array_equal(np.isnan(y), nan)
        assert_y_close(y[~nan], yo[~nan], so[~nan], dt, f"special/{split}")
    finally:
        A.close()


def test_empty_matrix(sable):
    s = from_dense(np.zeros((33, 17)), [0, 10, 33], [0, 17])
    A, y = check(sable, s, "rect")
    assert A.info["n_cells"] == 0 and not y.any()
    A.close()


def test_stored_zero_blocks_and_negative_zero(sable):
    """A stored block holding only zeros (+0 and -0) is not a candidate
    (PAPER.md:130, 275); -0 fill inside a dense block exports as +0."""
    A_ = np.zeros((6, 6), np.float32)
    A_[0:3, 0:3] = 1
    A_[1, 1] = 0
    s = from_dense(A_, [0, 3, 6], [0, 3, 6])
    inp = s.vbr_input("all_vbr")
    # add a stored all-zero block (block row 1, block col 1) by hand
    inp["bpntr"] = np.array([0, 1, 2], np.int64)
    inp["bindx"] = np.array([0, 1], np.int32)
    inp["indx"] = np.array([0, 9, 18], np.int64)
    val = np.zeros(18, np.float32)
    val[:9] = inp["val"][:9]
    val[4] = -0.0
    val[9:] = -0.0
    inp["val"] = val
    M = handle(sable, s, inp=inp)
    got = M.export()
    want = oracle_partition(s)
    assert_partition_equal(got, want, np.float32)
    assert M.info["n_cells"] == 1
    assert not np.signbit(got["tile_val"]).any()
    M.close()


@pytest.mark.parametrize("kind", ["dup", "indx", "bindx", "rem_order", "rem_range", "rpntr"])
def test_format_errors(sable, kind):
    s = gen.random_small(5, 50, 50, 5, 5, dtype=np.float32, dense_cells=0.6)
    inp = s.vbr_input("rect")
    want = sable.SABLE_E_FORMAT
    if kind == "dup":
        k = 0  # a VBR non-zero also present in the remainder
        rp, cp = inp["rpntr"], inp["cpntr"]
        a = int(np.searchsorted(inp["bpntr"], 0, side="right") - 1)
        b = int(inp["bindx"][0])
        blk = inp["val"][inp["indx"][0]:inp["indx"][1]]
        e = int(np.flatnonzero(blk)[0])
        h = rp[a + 1] - rp[a]
        i, j = rp[a] + e % h, cp[b] + e // h
        ii = np.repeat(np.arange(s.nrows), np.diff(inp["rem_indptr"]))
        I = np.concatenate([ii, [i]])
        J = np.concatenate([inp["rem_indices"], [j]])
        V = np.concatenate([inp["rem_val"], [np.float32(5)]])
        o = np.lexsort((J, I))
        inp["rem_indices"] = J[o].astype(np.int32)
        inp["rem_val"] = V[o].astype(np.float32)
        inp["rem_indptr"] = np.concatenate([[0], np.cumsum(np.bincount(I, minlength=s.nrows))])
        want = sable.SABLE_E_DUPLICATE
        del k
    elif kind == "indx":
        inp["indx"] = inp["indx"].copy()
        inp["indx"][1] += 1
    elif kind == "bindx":
        a = int(np.argmax(np.diff(inp["bpntr"]) >= 2))
        k = int(inp["bpntr"][a])
        inp["bindx"] = inp["bindx"].copy()
        inp["bindx"][k], inp["bindx"][k + 1] = inp["bindx"][k + 1], inp["bindx"][k]
    elif kind == "rem_order":
        r = int(np.argmax(np.diff(inp["rem_indptr"]) >= 2))
        p = int(inp["rem_indptr"][r])
        inp["rem_indices"] = inp["rem_indices"].copy()
        inp["rem_indices"][p], inp["rem_indices"][p + 1] = inp["rem_indices"][p + 1], inp["rem_indices"][p]
    elif kind == "rem_range":
        inp["rem_indices"] = inp["rem_indices"].copy()
        inp["rem_indices"][-1] = s.ncols
    elif kind == "rpntr":
        inp["rpntr"] = inp["rpntr"].copy()
        inp["rpntr"][2] = inp["rpntr"][1]
    for on_device in (True, False):
        with pytest.raises(sable.SableError) as e:
            handle(sable, s, inp=dict(inp), on_device=on_device)
        assert e.value.status == want, str(e.value)


# ------------------------------------------------------------------ API behaviour

def test_host_inputs_and_host_spmv(sable):
    s = gen.make("c1")
    A, y = check(sable, s, "rect", on_device=False)
    y2 = A.spmv_host(s.x.copy())
    np.testing.assert_array_equal(y, y2)
    A.close()


def test_deterministic_and_split_invariant_y(sable):
    """The work decomposition depends on the matrix only; repeated calls give
    the same bits."""
    s = gen.make("c2", scale=0.05)
    A = handle(sable, s, "rect")
    x = torch.from_numpy(s.x).cuda()
    y1 = A.spmv(x).clone()
    y2 = A.spmv(x)
    assert torch.equal(y1, y2)
    A.close()


@pytest.mark.parametrize("world", [2, 3, 5])
def test_shards_concatenate_to_full(sable, world):
    s = gen.make("c2", scale=0.02)
    full = handle(sable, s, "rect")
    fe = full.export()
    x = torch.from_numpy(s.x).cuda()
    yf = full.spmv(x).cpu().numpy()
    parts, ys = [], []
    for r in range(world):
        h = handle(sable, s, "rect", rank=r, world=world)
        i = h.info
        e = h.export()
        assert i["cell_base"] == np.searchsorted(fe["cell_br"], i["br_begin"])
        e["ublocks"] = e["ublocks"] + i["cell_base"]
        parts.append(e)
        ys.append(h.spmv(x).cpu().numpy())
        h.close()
    for k in ("cell_br", "cell_bc", "cell_cnt", "cell_dense", "tile_val", "ublocks",
              "rem_indices", "rem_val"):
        np.testing.assert_array_equal(np.concatenate([p[k] for p in parts]), fe[k], err_msg=k)
    np.testing.assert_array_equal(np.concatenate(ys), yf)  # bitwise P-invariance
    full.close()


def test_iterate_world1(sable):
    """x_{k+1} = A x_k through sable_spmv_iterate; every step checked against
    the oracle applied to the GPU's own x_k."""
    s = gen.make("c5", scale=1 / 256)
    A = handle(sable, s, "rect")
    xa = torch.from_numpy(s.x).cuda()
    xb = torch.empty_like(xa)
    xs = [s.x.astype(np.float64)]
    cur = xa
    for k in range(4):
        nxt = xb if cur is xa else xa
        A.spmv_allgather(cur, nxt)
        xs.append(nxt.cpu().numpy())
        yo, so = oracle.spmv(s.nrows, s.I, s.J, s.V.astype(np.float64), np.asarray(xs[-2], np.float64))
        assert_y_close(xs[-1], yo, so, np.float32, f"iter {k}")
        cur = nxt
    xa2 = torch.from_numpy(s.x).cuda()
    xb2 = torch.empty_like(xa2)
    res = A.iterate(xa2, xb2, 4)
    assert torch.equal(res, cur)
    A.close()


def test_comm_world1(sable):
    s = gen.make("c1")
    A = handle(sable, s, "rect")
    A.comm_init(sable.sable_nccl_unique_id())
    x = torch.from_numpy(s.x).cuda()
    xn = torch.empty_like(x)
    A.spmv_allgather(x, xn)
    assert torch.equal(xn, A.spmv(x))
    A.close()


# ------------------------------------------------------------------ full-size configs

# ------------------------------------------------------------------ executor shapes

EXEC_CFGS = {
    "unit": {},
    # tiny unit budget: remainders cut into many pieces, wide panels cut into
    # column chunks, few rows per remainder unit, one unit per warp
    "unit_small": dict(SABLE_USTAGE=1024, SABLE_UREM_ROWS=3, SABLE_UBATCH_UNITS=1),
    "unit_mid": dict(SABLE_USTAGE=4096, SABLE_UBATCH_UNITS=7),
    # long warp batches, no L2 prefetch
    "unit_long_batches": dict(SABLE_UBATCH_UNITS=64, SABLE_XPREFETCH=0),
    # lanes per row = the largest power of two <= the panel width (every lane busy)
    "unit_lpr1": dict(SABLE_LPR=1),
    "unit_lpr1_small": dict(SABLE_LPR=1, SABLE_USTAGE=2048, SABLE_UBATCH_UNITS=2),
}


@pytest.mark.parametrize("cfg", sorted(EXEC_CFGS))
def test_executor_configurations(sable, monkeypatch, cfg):
    """The same parity bar under other executor shapes (SABLE_* overrides):
    chunk boundaries, split groups and the stage ring at every position."""
    for k, v in EXEC_CFGS[cfg].items():
        monkeypatch.setenv(k, str(v))
    cases = [gen.make("c1"), gen.make("c2", scale=0.02)]
    for seed, shape in enumerate([(1000, 800, 7, 5), (64, 5000, 2, 3), (300, 300, 300, 300),
                                  (517, 611, 40, 3)]):
        cases.append(gen.random_small(20 + seed, *shape, dtype=np.float64 if seed % 2 else np.float32,
                                      density=0.2, dense_cells=0.5,
                                      values="int" if seed == 3 else "u11"))
    cases.append(long_rows_synth())
    for s in cases:
        for split in ("rect", "all_rem"):
            A, _ = check(sable, s, split, exact=s.name in ("rand23", "longrows"))
            A.close()


@pytest.mark.parametrize("env", [dict(SABLE_USTAGE=512), dict(SABLE_USTAGE=1000),
                                 dict(SABLE_ARCH=1), dict(SABLE_UREM_ROWS=33),
                                 dict(SABLE_UBATCH_UNITS=0)])
def test_executor_config_rejected(sable, monkeypatch, env):
    for k, v in env.items():  # below the minimum / not 16-aligned / no such executor
        monkeypatch.setenv(k, str(v))
    s = gen.make("c1")
    with pytest.raises(sable.SableError) as e:
        handle(sable, s, "rect")
    assert e.value.status == sable.SABLE_E_INVALID_ARG


# ------------------------------------------------------------------ per-shape delta policy

@pytest.mark.parametrize("seed", range(6))
def test_delta_policy(sable, seed):
    """sable_vbr_create_policy (reading R22): the partition equals the
    oracle's under the same rules and min_area, y within the tolerance."""
    g = np.random.default_rng(500 + seed)
    dt = np.float64 if seed % 2 else np.float32
    s = gen.random_small(500 + seed, 400, 380, 40, 35, dtype=dt, density=0.3, dense_cells=0.5)
    rules = []
    for _ in range(int(g.integers(1, 5))):
        h0, w0 = int(g.integers(1, 12)), int(g.integers(1, 12))
        rules.append((h0, h0 + int(g.integers(0, 10)), w0, w0 + int(g.integers(0, 10)),
                      int(g.choice([0, 30, 50, 80, 101]))))
    min_area = int(g.choice([0, 4, 16, 64]))
    inp = s.vbr_input("rect")
    arrays = to_dev(inp)
    A = sable.VbrMatrix(arrays, s.nrows, s.ncols, delta=s.delta,
                        policy=dict(min_area=min_area, rules=rules))
    try:
        got = A.export()
        want = oracle.partition(s.nrows, s.ncols, s.I, s.J, s.V.astype(np.float64), s.rpntr,
                                s.cpntr, s.delta, min_area=min_area, rules=rules)
        assert_partition_equal(got, want, dt, f"policy{seed}")
        y = A.spmv(torch.from_numpy(s.x).cuda()).cpu().numpy()
        yo, so = oracle.spmv(s.nrows, s.I, s.J, s.V.astype(np.float64), s.x.astype(np.float64))
        assert_y_close(y, yo, so, dt, f"policy{seed}")
    finally:
        A.close()


def test_delta_policy_rejected(sable):
    s = gen.make("c1")
    for pol in (dict(min_area=-1), dict(rules=[(1, 9, 1, 9, 102)]),
                dict(rules=[(1, 2, 1, 2, 50)] * 65)):
        with pytest.raises(sable.SableError) as e:
            sable.VbrMatrix(to_dev(s.vbr_input("rect")), s.nrows, s.ncols, delta=50, policy=pol)
        assert e.value.status == sable.SABLE_E_INVALID_ARG
