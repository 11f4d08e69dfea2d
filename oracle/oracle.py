"""ctypes marshalling for oracle/sable_oracle.c (test infrastructure only).

Each wrapper converts numpy arrays to the C types, calls the C function, and
copies the result into numpy arrays; there is no arithmetic here.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sable_oracle.c")
_LIB = os.path.join(_HERE, "libsable_oracle.so")
_lib = None

_ERRS = {1: "index out of range", 2: "duplicate (i,j)", 3: "bad cut grid",
         4: "out of memory", 5: "bad argument"}


class OracleError(RuntimeError):
    pass


def build(force: bool = False) -> str:
    """Compile the oracle shared library in-tree (gcc, fp64, no contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-std=c11", "-Wall",
                               "-fopenmp", "-shared", "-fPIC", "-o", _LIB, _SRC, "-lm"])
    return _LIB


class _Partition(C.Structure):
    _fields_ = [
        ("n_cells", C.c_int64), ("n_dense", C.c_int64), ("tile_elems", C.c_int64),
        ("rem_nnz", C.c_int64), ("nnz", C.c_int64),
        ("row_begin", C.c_int64), ("row_end", C.c_int64),
        ("cell_br", C.POINTER(C.c_int32)), ("cell_bc", C.POINTER(C.c_int32)),
        ("cell_cnt", C.POINTER(C.c_int64)), ("cell_dense", C.POINTER(C.c_uint8)),
        ("tile_off", C.POINTER(C.c_int64)), ("tile_val", C.POINTER(C.c_double)),
        ("ublocks", C.POINTER(C.c_int64)),
        ("rem_indptr", C.POINTER(C.c_int64)), ("rem_indices", C.POINTER(C.c_int32)),
        ("rem_val", C.POINTER(C.c_double)),
    ]


def _load():
    global _lib
    if _lib is None:
        build()
        lib = C.CDLL(_LIB)
        P = C.c_void_p
        lib.oracle_normalize.restype = C.c_int64
        lib.oracle_normalize.argtypes = [C.c_int64, C.c_int64, C.c_int64, P, P, P,
                                         C.POINTER(C.c_int)]
        lib.oracle_partition.restype = C.POINTER(_Partition)
        lib.oracle_partition.argtypes = [C.c_int64, C.c_int64, C.c_int64, P, P, P,
                                         C.c_int32, P, C.c_int32, P, C.c_int32,
                                         C.c_int32, C.c_int32, C.POINTER(C.c_int)]
        lib.oracle_partition_policy.restype = C.POINTER(_Partition)
        lib.oracle_partition_policy.argtypes = [C.c_int64, C.c_int64, C.c_int64, P, P, P,
                                                C.c_int32, P, C.c_int32, P, C.c_int32,
                                                C.c_int64, C.c_int32, P, C.c_int32,
                                                C.c_int32, C.POINTER(C.c_int)]
        lib.oracle_partition_free.restype = None
        lib.oracle_partition_free.argtypes = [C.POINTER(_Partition)]
        lib.oracle_spmv.restype = None
        lib.oracle_spmv.argtypes = [C.c_int64, C.c_int64, P, P, P, P, P, P]
        lib.oracle_spmv_rows.restype = None
        lib.oracle_spmv_rows.argtypes = [P, P, P, P, C.c_int64, P, P, P]
        lib.oracle_spmv_csr_mt.restype = None
        lib.oracle_spmv_csr_mt.argtypes = [P, P, P, P, C.c_int64, C.c_int32, P, P]
        lib.oracle_rowptr.restype = None
        lib.oracle_rowptr.argtypes = [C.c_int64, C.c_int64, P, P]
        lib.oracle_alg1.restype = C.c_int64
        lib.oracle_alg1.argtypes = [C.c_int64, P, P, C.c_uint32, C.c_uint32, C.c_int32, P]
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def normalize(nrows: int, ncols: int, I, J, V):
    """range check, sort by (i,j), reject duplicates,
    drop v == 0.  Returns new (I, J, V) arrays (int64, int64, float64)."""
    lib = _load()
    I = np.array(I, dtype=np.int64, copy=True)
    J = np.array(J, dtype=np.int64, copy=True)
    V = np.array(V, dtype=np.float64, copy=True)
    err = C.c_int(0)
    n = lib.oracle_normalize(nrows, ncols, len(I), _p(I), _p(J), _p(V), C.byref(err))
    if n < 0:
        raise OracleError(_ERRS.get(err.value, str(err.value)))
    return I[:n].copy(), J[:n].copy(), V[:n].copy()


def _arr(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


def partition(nrows: int, ncols: int, I, J, V, rpntr, cpntr, delta: int,
              a0: int = 0, a1: int | None = None, min_area: int = 0, rules=None) -> dict:
    """SURVEY 8(c) steps 3-6 over block rows [a0, a1) of normalised COO.

    min_area / rules: the per-shape delta policy (reading R22): rules is a
    sequence of (h_min, h_max, w_min, w_max, delta), the first match wins;
    `delta` is the default for unmatched shapes.

    Returns the canonical export: cell_br, cell_bc,
    cell_cnt, cell_dense, tile_off, tile_val (float64), ublocks, rem_indptr,
    rem_indices, rem_val (float64), plus the sizes.
    """
    lib = _load()
    I = _c(I, np.int64)
    J = _c(J, np.int64)
    V = _c(V, np.float64)
    rp = _c(rpntr, np.int32)
    cp = _c(cpntr, np.int32)
    nbr, nbc = len(rp) - 1, len(cp) - 1
    if a1 is None:
        a1 = nbr
    err = C.c_int(0)
    if min_area or rules:
        rr = _c(np.asarray(rules if rules else np.zeros((0, 5)), np.int64).reshape(-1, 5),
                np.int32)
        res = lib.oracle_partition_policy(nrows, ncols, len(I), _p(I), _p(J), _p(V), nbr,
                                          _p(rp), nbc, _p(cp), int(delta), int(min_area),
                                          len(rr), _p(rr), int(a0), int(a1), C.byref(err))
    else:
        res = lib.oracle_partition(nrows, ncols, len(I), _p(I), _p(J), _p(V), nbr, _p(rp),
                                   nbc, _p(cp), int(delta), int(a0), int(a1), C.byref(err))
    if not res:
        raise OracleError(_ERRS.get(err.value, str(err.value)))
    try:
        p = res.contents
        nloc = p.row_end - p.row_begin
        out = dict(
            n_cells=p.n_cells, n_dense=p.n_dense, tile_elems=p.tile_elems,
            rem_nnz=p.rem_nnz, nnz=p.nnz, row_begin=p.row_begin, row_end=p.row_end,
            cell_br=_arr(p.cell_br, p.n_cells, np.int32),
            cell_bc=_arr(p.cell_bc, p.n_cells, np.int32),
            cell_cnt=_arr(p.cell_cnt, p.n_cells, np.int64),
            cell_dense=_arr(p.cell_dense, p.n_cells, np.uint8),
            tile_off=_arr(p.tile_off, p.n_dense + 1, np.int64),
            tile_val=_arr(p.tile_val, p.tile_elems, np.float64),
            ublocks=_arr(p.ublocks, p.n_cells - p.n_dense, np.int64),
            rem_indptr=_arr(p.rem_indptr, nloc + 1, np.int64),
            rem_indices=_arr(p.rem_indices, p.rem_nnz, np.int32),
            rem_val=_arr(p.rem_val, p.rem_nnz, np.float64),
        )
    finally:
        lib.oracle_partition_free(res)
    return out


def spmv(nrows: int, I, J, V, x):
    """y = A x row by row in fp64, and s = |A| |x|."""
    lib = _load()
    I = _c(I, np.int64)
    J = _c(J, np.int64)
    V = _c(V, np.float64)
    x = _c(x, np.float64)
    y = np.empty(nrows, dtype=np.float64)
    s = np.empty(nrows, dtype=np.float64)
    lib.oracle_spmv(nrows, len(I), _p(I), _p(J), _p(V), _p(x), _p(y), _p(s))
    return y, s


def rowptr(nrows: int, I) -> np.ndarray:
    lib = _load()
    I = _c(I, np.int64)
    rp = np.empty(nrows + 1, dtype=np.int64)
    lib.oracle_rowptr(nrows, len(I), _p(I), _p(rp))
    return rp


def spmv_rows(rp, J, V, x, rows):
    """y_i and s_i for a sample of rows (full-size configurations)."""
    lib = _load()
    rp = _c(rp, np.int64)
    J = _c(J, np.int64)
    V = _c(V, np.float64)
    x = _c(x, np.float64)
    rows = _c(rows, np.int64)
    y = np.empty(len(rows), dtype=np.float64)
    s = np.empty(len(rows), dtype=np.float64)
    lib.oracle_spmv_rows(_p(rp), _p(J), _p(V), _p(x), len(rows), _p(rows), _p(y), _p(s))
    return y, s


def spmv_csr_mt(rp, J, V, x, nrows: int, nthreads: int):
    """y, s for rows [0, nrows) on `nthreads` OpenMP threads (timing only)."""
    lib = _load()
    rp = _c(rp, np.int64)
    J = _c(J, np.int64)
    V = _c(V, np.float64)
    x = _c(x, np.float64)
    y = np.empty(nrows, dtype=np.float64)
    s = np.empty(nrows, dtype=np.float64)
    lib.oracle_spmv_csr_mt(_p(rp), _p(J), _p(V), _p(x), nrows, nthreads, _p(y), _p(s))
    return y, s


def alg1_cuts(n: int, rowptr, J, t_num: int, t_den: int, shifts: bool) -> np.ndarray:
    """Alg. 1 on a CSR pattern: the grid 0 = g0 < g1 < ...
    < gk = n (0 followed by the algorithm's cuts), Eq. 1 similarity, or Eq. 2
    with the +-1 shifts when `shifts`; threshold t_num / t_den, exact."""
    lib = _load()
    rp = _c(rowptr, np.int64)
    J = _c(J, np.int64)
    cuts = np.zeros(max(n, 1), dtype=np.int32)
    m = lib.oracle_alg1(n, _p(rp), _p(J), t_num, t_den, 1 if shifts else 0, _p(cuts))
    return np.concatenate([[0], cuts[:m]]).astype(np.int32)


def partition_grid(nrows: int, ncols: int, I, J, t_num: int, t_den: int, shifts: bool):
    """(rpntr, cpntr) of Alg. 1 for the pattern of COO triples: rows on A,
    then "the same procedure on the columns" on the pattern of A^T."""
    I = np.asarray(I, np.int64)
    J = np.asarray(J, np.int64)
    o = np.lexsort((J, I))
    rp = np.zeros(nrows + 1, np.int64)
    np.cumsum(np.bincount(I, minlength=nrows), out=rp[1:])
    rows = alg1_cuts(nrows, rp, J[o], t_num, t_den, shifts)
    o2 = np.lexsort((I, J))
    cp = np.zeros(ncols + 1, np.int64)
    np.cumsum(np.bincount(J, minlength=ncols), out=cp[1:])
    cols = alg1_cuts(ncols, cp, I[o2], t_num, t_den, shifts)
    return rows, cols
