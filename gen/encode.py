"""Encode COO triples in the paper's VBR input format (input preparation only).

VBR (Fig. 2): ``val`` holds each stored block column-major
(``val[indx[k] + (j-c0)*h + (i-r0)]``, Listing 2), ``indx`` is
"inclusive of the length of the Val array", ``bindx`` is the block column of
each block, and the block-row pointers are given CSR-style as
``bpntr[nbr+1]`` (reading R9; ``bpntrb[a]=bpntr[a]`` or -1 when empty,
``bpntre[a]=bpntr[a+1]``).  Triples the caller does not route to VBR form a
CSR remainder (Fig. 3 indptr/indices/csr_val).

Which triples go to ``val`` is the caller's choice (the "split"); the method
must give the same partition for every split (reading R5).
"""
from __future__ import annotations

import numpy as np


def encode_vbr(nrows: int, ncols: int, rpntr, cpntr, I, J, V, to_vbr) -> dict:
    """Return the VBR + remainder input arrays for sorted, duplicate-free COO.

    ``to_vbr`` is a boolean mask over the triples: True sends a triple to the
    VBR block of its grid cell (every cell holding such a triple becomes a
    stored block), False to the CSR remainder.
    """
    rpntr = np.asarray(rpntr, dtype=np.int32)
    cpntr = np.asarray(cpntr, dtype=np.int32)
    I = np.asarray(I, dtype=np.int64)
    J = np.asarray(J, dtype=np.int64)
    V = np.asarray(V)
    to_vbr = np.asarray(to_vbr, dtype=bool)
    nbr, nbc = len(rpntr) - 1, len(cpntr) - 1

    Iv, Jv, Vv = I[to_vbr], J[to_vbr], V[to_vbr]
    br = np.searchsorted(rpntr, Iv, side="right") - 1
    bc = np.searchsorted(cpntr, Jv, side="right") - 1
    key = br.astype(np.int64) * nbc + bc
    blocks, inv = np.unique(key, return_inverse=True)
    bbr = (blocks // nbc).astype(np.int64)
    bbc = (blocks % nbc).astype(np.int64)
    h = (rpntr[bbr + 1] - rpntr[bbr]).astype(np.int64)
    w = (cpntr[bbc + 1] - cpntr[bbc]).astype(np.int64)
    indx = np.zeros(len(blocks) + 1, dtype=np.int64)
    np.cumsum(h * w, out=indx[1:])
    val = np.zeros(int(indx[-1]), dtype=V.dtype)
    pos = indx[inv] + (Jv - cpntr[bbc[inv]]) * h[inv] + (Iv - rpntr[bbr[inv]])
    val[pos] = Vv
    bpntr = np.searchsorted(bbr, np.arange(nbr + 1), side="left").astype(np.int64)

    Ir, Jr, Vr = I[~to_vbr], J[~to_vbr], V[~to_vbr]
    rem_indptr = np.zeros(nrows + 1, dtype=np.int64)
    np.cumsum(np.bincount(Ir, minlength=nrows), out=rem_indptr[1:])
    return dict(
        nrows=int(nrows), ncols=int(ncols), rpntr=rpntr, cpntr=cpntr,
        bpntr=bpntr, bindx=bbc.astype(np.int32), indx=indx, val=val,
        rem_indptr=rem_indptr, rem_indices=Jr.astype(np.int32),
        rem_val=np.ascontiguousarray(Vr),
    )
