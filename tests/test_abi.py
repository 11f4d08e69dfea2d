"""CPU-only checks of the C-ABI library: it loads, exports every symbol that
include/sable.h declares, and its host-only logic (argument checking, status
strings, shard bounds) behaves as documented.  No compute call needs a GPU."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def sable():
    from paper_2407_00829_b200 import build
    build.build()
    from paper_2407_00829_b200 import sable as s
    return s


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "sable.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sable_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_symbols()
    for n in ("sable_vbr_create", "sable_spmv", "sable_destroy"):  # north_star s3
        assert n in names


def test_library_exports_every_declared_symbol(sable):
    lib = C.CDLL(sable.LIB_PATH)
    for n in declared_symbols():
        assert hasattr(lib, n), n
    assert set(declared_symbols()) == set(sable.EXPORTS)


def test_library_is_sm100a(sable):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", sable.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_status_strings_and_version(sable):
    assert sable.sable_abi_version() == 2
    assert sable.sable_status_string(0) == "SABLE_OK"
    assert sable.sable_status_string(sable.SABLE_E_DUPLICATE) == "SABLE_E_DUPLICATE"


def test_create_rejects_bad_arguments_before_touching_the_gpu(sable):
    d = sable.sable_vbr_desc()
    with pytest.raises(sable.SableError) as e:
        sable.sable_vbr_create(d, 102)
    assert e.value.status == sable.SABLE_E_INVALID_ARG
    d.nrows = d.ncols = 4
    d.nbrows = d.nbcols = 1
    d.dtype, d.mem = 7, 0
    with pytest.raises(sable.SableError) as e:
        sable.sable_vbr_create(d, 50)
    assert e.value.status == sable.SABLE_E_INVALID_ARG and "dtype" in str(e.value)
    d.dtype = 0
    d.nrows = 0
    with pytest.raises(sable.SableError) as e:
        sable.sable_vbr_create(d, 50)
    assert e.value.status == sable.SABLE_E_DIM
    d.nrows = 4
    with pytest.raises(sable.SableError) as e:  # NULL arrays
        sable.sable_vbr_create(d, 50)
    assert e.value.status == sable.SABLE_E_INVALID_ARG
    rp = np.array([0, 4], np.int32)
    bp = np.array([0, 0], np.int64)
    ix = np.array([0], np.int64)
    d.rpntr = d.cpntr = rp.ctypes.data
    d.bpntr, d.indx = bp.ctypes.data, ix.ctypes.data
    with pytest.raises(sable.SableError) as e:
        sable.sable_vbr_create(d, 50, rank=2, world=2)
    assert e.value.status == sable.SABLE_E_INVALID_ARG and "shard" in str(e.value)
    d.rem_nnz = 3
    with pytest.raises(sable.SableError) as e:
        sable.sable_vbr_create(d, 50)
    assert e.value.status == sable.SABLE_E_INVALID_ARG


def test_null_handles(sable):
    sable.sable_destroy(0)  # NULL is a no-op
    with pytest.raises(sable.SableError):
        sable.sable_get_info(0)
    with pytest.raises(sable.SableError):
        sable.sable_spmv(0, 0, 0)
    # the fused-exchange registration checks its arguments before any device work
    with pytest.raises(sable.SableError) as e:
        sable.sable_comm_fuse(0, 0, 0)
    assert e.value.status == sable.SABLE_E_INVALID_ARG
    with pytest.raises(sable.SableError) as e:
        sable.sable_comm_set_peers(0, 16, 32, [], [])
    assert e.value.status == sable.SABLE_E_INVALID_ARG
    with pytest.raises(sable.SableError):
        sable.sable_comm_unfuse(0)


def brute_bounds(w, world):
    """Definition: boundary k = first a with sum(w[:a]) >= k * total / world."""
    total = sum(int(v) for v in w)
    pre = np.concatenate([[0], np.cumsum(np.asarray(w, dtype=np.int64))])
    out = [0]
    for k in range(1, world):
        a = 0
        while a < len(w) and pre[a] * world < k * total:
            a += 1
        out.append(max(a, out[-1]))
    out.append(len(w))
    return out


@pytest.mark.parametrize("seed", range(20))
def test_shard_bounds_definition(sable, seed):
    g = np.random.default_rng(seed)
    nbr = int(g.integers(1, 60))
    w = g.integers(0, 1000, nbr) * (g.random(nbr) < 0.8)
    for world in (1, 2, 3, 4, 8, 64):
        b = sable.sable_shard_bounds(w, world)
        assert list(b) == brute_bounds(w, world)
        assert b[0] == 0 and b[-1] == nbr and np.all(np.diff(b) >= 0)


def test_shard_bounds_balance(sable):
    w = np.full(1000, 7, np.int64)
    b = sable.sable_shard_bounds(w, 8)
    assert np.all(np.diff(b) == 125)
    with pytest.raises(sable.SableError):
        sable.sable_shard_bounds(np.array([-1], np.int64), 2)
