"""Host logic of the f2 calibration (scripts/calibrate.py) and
the structure of its seeded workloads (gen/calib.py): Fig. 10's 10000^2 /
50x50 splits / 500 blocks with an exact per-block sparsity,
the one-shape grids of the Fig. 7 analogue.  The GPU leg
checks that both arms the calibration times (delta = 0: all tiles; delta =
101: all remainder) compute the oracle's y."""
import importlib.util
import os

import numpy as np
import pytest

import gen.calib as gc
import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
_spec = importlib.util.spec_from_file_location(
    "calibrate", os.path.join(HERE, "..", "scripts", "calibrate.py"))
calibrate = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(calibrate)


def test_crossover():
    f = [0.1, 0.2, 0.3, 0.4, 0.5]
    assert calibrate.crossover(f, [0.5, 0.8, 1.1, 1.3, 2.0]) == 0.3
    assert calibrate.crossover(f, [0.5, 1.2, 0.9, 1.3, 2.0]) == 0.4  # must hold from there on
    assert calibrate.crossover(f, [0.5, 0.6, 0.7, 0.8, 0.9]) is None
    assert calibrate.crossover(f, [1.0] * 5) == 0.1
    assert calibrate.delta_of(0.3) == 30 and calibrate.delta_of(None) is None


def test_monotone_violations():
    assert calibrate.monotone_violations([1, 2, 3], [1.0, 1.05, 2.0]) == []
    assert calibrate.monotone_violations([1, 2, 3], [1.0, 0.5, 2.0]) == [(1, 2)]
    assert calibrate.monotone_violations([1, 2], [2.0, 1.0], increasing=False) == []


@pytest.mark.parametrize("sp", [0.0, 0.5, 0.99])
def test_fig10_structure(sp):
    s = gc.fig10(sp)
    assert s.nrows == s.ncols == 10000
    assert len(s.rpntr) == len(s.cpntr) == 201 and np.all(np.diff(s.rpntr) == 50)
    cell = (s.I // 50) * 200 + s.J // 50
    cells, cnt = np.unique(cell, return_counts=True)
    assert len(cells) == 500
    assert np.all(cnt == max(1, round((1 - sp) * 2500)))
    assert np.all(s.V != 0) and np.all(np.diff(s.I * s.ncols + s.J) > 0)


@pytest.mark.parametrize("h,w,fill", [(4, 4, 0.1), (16, 128, 0.5), (64, 4, 1.0)])
def test_shape_grid_structure(h, w, fill):
    s = gc.shape_grid(h, w, fill, area=1 << 16)
    cell = (s.I // h) * (s.ncols // w) + s.J // w
    cells, cnt = np.unique(cell, return_counts=True)
    assert len(cells) == max(8, (1 << 16) // (h * w))
    per_row = np.bincount(cells // (s.ncols // w))
    assert np.all(per_row == 8)
    dens = cnt.sum() / (len(cells) * h * w)
    assert abs(dens - fill) < 0.05 + 1.0 / (h * w)


def test_delta_extremes_split_on_oracle():
    s = gc.shape_grid(8, 8, 0.6, area=1 << 12)
    p0 = oracle.partition(s.nrows, s.ncols, s.I, s.J, s.V.astype(float), s.rpntr, s.cpntr, 0)
    p1 = oracle.partition(s.nrows, s.ncols, s.I, s.J, s.V.astype(float), s.rpntr, s.cpntr, 101)
    assert p0["n_dense"] == p0["n_cells"] and len(p0["rem_val"]) == 0
    assert p1["n_dense"] == 0 and len(p1["rem_val"]) == s.nnz


@pytest.mark.gpu
@pytest.mark.parametrize("delta", [0, 101])
def test_both_arms_match_oracle(delta):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2407_00829_b200 import sable
    from parity import assert_y_close
    for s in (gc.shape_grid(16, 128, 0.3, area=1 << 18), gc.fig10(0.8)):
        inp = s.vbr_input("all_vbr")
        arrays = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in inp.items()
                  if isinstance(v, np.ndarray)}
        A = sable.VbrMatrix(arrays, s.nrows, s.ncols, delta=delta)
        y = A.spmv(torch.from_numpy(s.x).cuda()).cpu().numpy()
        A.close()
        yo, so = oracle.spmv(s.nrows, s.I, s.J, s.V.astype(np.float64), s.x.astype(np.float64))
        assert_y_close(y, yo, so, np.float32, f"{s.name}/d{delta}")


def test_policy_from_heatmap():
    b = calibrate.size_buckets([4, 16, 64])
    assert b == {4: (1, 8), 16: (9, 32), 64: (33, 2 ** 31 - 1)}
    heat = [dict(h=4, w=4, delta_star=None), dict(h=16, w=64, delta_star=70),
            dict(h=64, w=16, delta_star=40)]
    pol = calibrate.policy_from_heatmap(heat)
    assert pol["delta"] == 50 and pol["min_area"] == 0
    assert pol["rules"][0] == (1, 8, 1, 8, 101)
    assert pol["rules"][1] == (9, 32, 33, 2 ** 31 - 1, 70)
    assert pol["rules"][2] == (33, 2 ** 31 - 1, 9, 32, 40)


def test_c4a_structure():
    import gen
    s = gen.make("c4a", scale=1 / 32)
    assert np.all(np.diff(s.rpntr) == 64) and np.array_equal(s.rpntr, s.cpntr)
    assert not s.in_rect.any()
    c4 = gen.make("c4", scale=1 / 32)
    assert s.nnz == c4.nnz  # the same matrix on another grid
