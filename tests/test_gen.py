"""The seeded generators: determinism, structure, and that the VBR encoding
decodes back to the matrix (Fig. 2 column-major addressing)."""
import numpy as np
import pytest

import gen
from gen.configs import c5_dmin, log_uniform_int, rng
from golden_io import load


def decode(d):
    """VBR + remainder arrays -> dense, by the Fig. 2 definitions."""
    A = np.zeros((d["nrows"], d["ncols"]))
    rp, cp = d["rpntr"], d["cpntr"]
    for a in range(len(rp) - 1):
        for k in range(d["bpntr"][a], d["bpntr"][a + 1]):
            b = d["bindx"][k]
            h, w = rp[a + 1] - rp[a], cp[b + 1] - cp[b]
            blk = d["val"][d["indx"][k]:d["indx"][k + 1]].reshape((h, w), order="F")
            A[rp[a]:rp[a + 1], cp[b]:cp[b + 1]] += blk
    for i in range(d["nrows"]):
        for k in range(d["rem_indptr"][i], d["rem_indptr"][i + 1]):
            A[i, d["rem_indices"][k]] += d["rem_val"][k]
    return A


def dense(s):
    A = np.zeros((s.nrows, s.ncols))
    A[s.I, s.J] = s.V
    return A


def test_fig2_encodes_to_paper_arrays():
    g = load("fig2_vbr.txt")
    A = g["A"]
    I, J = np.nonzero(A)
    d = gen.encode_vbr(11, 11, g["Rpntr"], g["Cpntr"], I, J, A[I, J], np.ones(len(I), bool))
    np.testing.assert_array_equal(d["val"], g["Val"])
    np.testing.assert_array_equal(d["indx"], g["Indx"])
    np.testing.assert_array_equal(d["bindx"], g["Bindx"])
    np.testing.assert_array_equal(d["bpntr"][:-1], g["Bpntrb"])
    np.testing.assert_array_equal(d["bpntr"][1:], g["Bpntre"])


@pytest.mark.parametrize("split", ["rect", "all_vbr", "all_rem"])
def test_encode_roundtrip(split):
    s = gen.random_small(3, 40, 33, 6, 5)
    np.testing.assert_array_equal(decode(s.vbr_input(split)), dense(s))


def test_c1_shape_and_determinism():
    a, b = gen.make("c1"), gen.make("c1")
    for k in ("I", "J", "V", "x", "rpntr", "cpntr", "in_rect"):
        np.testing.assert_array_equal(getattr(a, k), getattr(b, k))
    assert a.V.dtype == np.float32 and a.nrows == 2000 and len(a.rects) == 12
    assert np.all(np.diff(a.I * a.ncols + a.J) > 0)  # sorted, no duplicates
    assert np.all(a.V != 0)
    r = a.rects
    assert np.all((r[:, 2] >= 8) & (r[:, 2] <= 64) & (r[:, 3] >= 8) & (r[:, 3] <= 64))
    # 0.2% of 2000^2 = 8000 scattered; the few that land inside a rectangle join its cells
    assert 7900 <= (~a.in_rect).sum() <= 8000
    np.testing.assert_array_equal(decode(a.vbr_input()), dense(a))
    c = gen.make("c1", seed=7)
    assert not np.array_equal(c.I, a.I)


@pytest.mark.parametrize("name,scale", [("c2", 0.02), ("c3", 0.01), ("c4", 1 / 16), ("c5", 1 / 512)])
def test_scaled_configs(name, scale):
    s = gen.make(name, scale=scale)
    assert np.all(np.diff(s.I * s.ncols + s.J) > 0)
    assert np.all(s.V != 0) and s.nnz > 0
    assert s.rpntr[0] == 0 and s.rpntr[-1] == s.nrows and np.all(np.diff(s.rpntr) > 0)
    d = s.vbr_input()
    assert len(d["val"]) >= int(s.in_rect.sum())
    assert len(d["rem_indices"]) == int((~s.in_rect).sum())
    if name == "c3":
        inband = np.abs(s.I - s.J) <= 31
        assert np.all(s.in_rect == inband)
        assert np.all(np.bincount(s.I[~inband], minlength=s.nrows) == 3)
    if name == "c5":
        colsum = np.bincount(s.J, weights=s.V.astype(np.float64), minlength=s.ncols)
        nz = colsum > 0
        assert np.allclose(colsum[nz], 1.0, rtol=1e-5)
        assert s.iterations == 100


def test_log_uniform_and_dmin():
    v = log_uniform_int(rng(0, 9), 4, 128, 100000)
    assert v.min() == 4 and v.max() == 128
    d = c5_dmin(1 << 16)
    k = np.arange(1, (1 << 16) + 1)
    assert abs(np.minimum(1, (d / k) ** 1.5).sum() - 16) < 1e-6
