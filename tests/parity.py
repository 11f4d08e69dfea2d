"""Comparison helpers for the CUDA path vs the oracle (tests only).

Partition arrays must be byte-identical (values compared as bit patterns in
the config dtype); y must satisfy |y_gpu - y| <= tol * s with s = sum |a||x|
(BASELINE.json north_star s11: 1e-5 for fp32, 1e-12 for fp64), and y_gpu must
be exactly 0 where s = 0.
"""
import numpy as np

import oracle

TOL = {np.float32: 1e-5, np.float64: 1e-12}
INT_KEYS = ("cell_br", "cell_bc", "cell_cnt", "cell_dense", "tile_off", "ublocks",
            "rem_indptr", "rem_indices")
VAL_KEYS = ("tile_val", "rem_val")


def bits(a, dtype):
    a = np.ascontiguousarray(np.asarray(a).astype(dtype))
    return a.view(np.uint32 if np.dtype(dtype).itemsize == 4 else np.uint64)


def assert_partition_equal(got: dict, want: dict, dtype, where=""):
    for k in INT_KEYS:
        g = np.asarray(got[k]).astype(np.int64)
        w = np.asarray(want[k]).astype(np.int64)
        assert g.shape == w.shape, f"{where} {k}: shape {g.shape} != {w.shape}"
        if not np.array_equal(g, w):
            bad = np.flatnonzero(g != w)[:5]
            raise AssertionError(f"{where} {k} differs at {bad}: got {g[bad]} want {w[bad]}")
    for k in VAL_KEYS:
        g, w = bits(got[k], dtype), bits(want[k], dtype)
        assert g.shape == w.shape, f"{where} {k}: shape {g.shape} != {w.shape}"
        if not np.array_equal(g, w):
            bad = np.flatnonzero(g != w)[:5]
            raise AssertionError(f"{where} {k} bits differ at {bad}")


def oracle_partition(s, a0=0, a1=None):
    return oracle.partition(s.nrows, s.ncols, s.I, s.J, s.V.astype(np.float64), s.rpntr,
                            s.cpntr, s.delta, a0, a1)


def slice_export(exp: dict, a0: int, a1: int, rpntr) -> dict:
    """Restrict a full-matrix export to block rows [a0, a1) (local ordinals)."""
    br = exp["cell_br"]
    c0, c1 = np.searchsorted(br, a0), np.searchsorted(br, a1)
    dense = exp["cell_dense"].astype(bool)
    t0, t1 = int(dense[:c0].sum()), int(dense[:c1].sum())
    to = exp["tile_off"]
    ub = np.flatnonzero(~dense[c0:c1]).astype(np.int64)
    r0, r1 = int(rpntr[a0]), int(rpntr[a1])
    ip = exp["rem_indptr"]
    return dict(cell_br=br[c0:c1], cell_bc=exp["cell_bc"][c0:c1], cell_cnt=exp["cell_cnt"][c0:c1],
                cell_dense=exp["cell_dense"][c0:c1], tile_off=to[t0:t1 + 1] - to[t0],
                tile_val=exp["tile_val"][to[t0]:to[t1]], ublocks=ub,
                rem_indptr=ip[r0:r1 + 1] - ip[r0], rem_indices=exp["rem_indices"][ip[r0]:ip[r1]],
                rem_val=exp["rem_val"][ip[r0]:ip[r1]])


def assert_y_close(y_gpu, y, s, dtype, where=""):
    y_gpu = np.asarray(y_gpu).astype(np.float64)
    tol = TOL[np.dtype(dtype).type]
    err = np.abs(y_gpu - y)
    zero = s == 0
    assert np.all(y_gpu[zero] == 0), f"{where}: nonzero y where s = 0"
    ok = err <= tol * s
    if not np.all(ok):
        bad = np.flatnonzero(~ok)[:5]
        raise AssertionError(f"{where}: y off at rows {bad}: rel {(err[bad] / s[bad])}")
