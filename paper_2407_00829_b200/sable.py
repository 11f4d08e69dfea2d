"""Thin ctypes binding of libsable.so (include/sable.h) -- argument
marshalling only.  Every step of the hot path runs in the library's CUDA
kernels; PyTorch is used only for device memory, streams and process groups.

There is no fallback: if libsable.so is missing or does not load, importing
this module raises ImportError (build it with ``python -m
paper_2407_00829_b200.build`` or ``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# SABLE_LIB=<variant> loads an in-tree A/B build libsable_<variant>.so (build.py)
LIB_PATH = os.path.join(_PKG, f"libsable_{os.environ['SABLE_LIB']}.so" if os.environ.get("SABLE_LIB")
                        else "libsable.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libsable.so not built at {LIB_PATH}; run __graft_entry__.build()")
try:
    _lib = C.CDLL(LIB_PATH)
except OSError as e:  # pragma: no cover - loud failure, no CPU fallback
    raise ImportError(f"cannot load {LIB_PATH}: {e}") from e

SABLE_OK, SABLE_E_INVALID_ARG, SABLE_E_FORMAT, SABLE_E_DIM, SABLE_E_DUPLICATE, \
    SABLE_E_OOM, SABLE_E_CUDA, SABLE_E_NCCL, SABLE_E_UNSUPPORTED = range(9)
SABLE_F32, SABLE_F64 = 0, 1
SABLE_MEM_HOST, SABLE_MEM_DEVICE = 0, 1

#: every symbol declared in include/sable.h
EXPORTS = ("sable_vbr_create", "sable_spmv", "sable_spmv_host", "sable_destroy",
           "sable_get_info", "sable_export_partition", "sable_shard_bounds",
           "sable_nccl_unique_id", "sable_comm_init", "sable_spmv_allgather",
           "sable_spmv_iterate", "sable_status_string", "sable_last_error",
           "sable_abi_version", "sable_partition_grid", "sable_serialize",
           "sable_deserialize", "sable_spmm", "sable_comm_check", "sable_exchange_rows",
           "sable_vbr_create_policy", "sable_comm_fuse", "sable_comm_set_peers",
           "sable_comm_unfuse")


class sable_vbr_desc(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64),
                ("nbrows", C.c_int32), ("nbcols", C.c_int32),
                ("nblocks", C.c_int64), ("val_len", C.c_int64), ("rem_nnz", C.c_int64),
                ("dtype", C.c_int32), ("mem", C.c_int32),
                ("rpntr", C.c_void_p), ("cpntr", C.c_void_p), ("bpntr", C.c_void_p),
                ("bindx", C.c_void_p), ("indx", C.c_void_p), ("val", C.c_void_p),
                ("rem_indptr", C.c_void_p), ("rem_indices", C.c_void_p),
                ("rem_val", C.c_void_p)]


class sable_shard(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32)]


class sable_delta_rule(C.Structure):
    _fields_ = [("h_min", C.c_int32), ("h_max", C.c_int32), ("w_min", C.c_int32),
                ("w_max", C.c_int32), ("delta_pct", C.c_uint32)]


class sable_delta_policy(C.Structure):
    _fields_ = [("delta_pct", C.c_uint32), ("min_area", C.c_int64), ("n_rules", C.c_int32),
                ("rules", C.POINTER(sable_delta_rule))]


class sable_info(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64),
                ("nbrows", C.c_int32), ("nbcols", C.c_int32),
                ("br_begin", C.c_int32), ("br_end", C.c_int32),
                ("row_begin", C.c_int64), ("row_end", C.c_int64),
                ("nnz", C.c_int64), ("n_cells", C.c_int64), ("cell_base", C.c_int64),
                ("n_dense", C.c_int64), ("tile_elems", C.c_int64), ("rem_nnz", C.c_int64),
                ("n_dense_global", C.c_int64), ("bytes_alg", C.c_int64),
                ("dtype", C.c_int32), ("delta", C.c_int32), ("suitable", C.c_int32),
                ("world", C.c_int32), ("rank", C.c_int32), ("inspect_ms", C.c_double),
                ("exec_grid", C.c_int32), ("unit_bytes", C.c_int32), ("n_units", C.c_int64),
                ("n_unit_batches", C.c_int64), ("n_combine", C.c_int64),
                ("panel_elems", C.c_int64), ("xmap_entries", C.c_int64)]


class sable_partition_host(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("cell_br", "cell_bc", "cell_cnt", "cell_dense",
                                           "tile_off", "tile_val", "ublocks", "rem_indptr",
                                           "rem_indices", "rem_val")]


_H = C.c_void_p
_P = C.c_void_p
_sig = {
    "sable_vbr_create": [C.POINTER(sable_vbr_desc), C.c_uint32, C.POINTER(sable_shard), _P,
                         C.POINTER(_H)],
    "sable_spmv": [_H, _P, _P, _P],
    "sable_spmv_host": [_H, _P, _P, _P],
    "sable_destroy": [_H],
    "sable_get_info": [_H, C.POINTER(sable_info)],
    "sable_export_partition": [_H, C.POINTER(sable_partition_host)],
    "sable_shard_bounds": [_P, C.c_int32, C.c_int32, _P],
    "sable_nccl_unique_id": [_P],
    "sable_comm_init": [_H, _P],
    "sable_spmv_allgather": [_H, _P, _P, _P],
    "sable_spmv_iterate": [_H, _P, _P, C.c_int32, _P, C.POINTER(C.c_int32)],
    "sable_partition_grid": [C.c_int64, C.c_int64, C.c_int64, _P, _P, C.c_int32, C.c_uint32,
                             C.c_uint32, C.c_int32, _P, _P, C.POINTER(C.c_int32), _P,
                             C.POINTER(C.c_int32)],
    "sable_serialize": [_H, _P, C.c_int64, C.POINTER(C.c_int64)],
    "sable_spmm": [_H, _P, _P, C.c_int32, _P],
    "sable_deserialize": [_P, C.c_int64, _P, C.POINTER(_H)],
    "sable_comm_check": [_H],
    "sable_vbr_create_policy": [C.POINTER(sable_vbr_desc), C.POINTER(sable_delta_policy),
                                C.POINTER(sable_shard), _P, C.POINTER(_H)],
    "sable_exchange_rows": [_P, C.c_int32, _P, C.c_int32, _P],
    "sable_comm_fuse": [_H, _P, _P],
    "sable_comm_set_peers": [_H, _P, _P, _P, _P, C.c_int32],
    "sable_comm_unfuse": [_H],
}
for _name, _args in _sig.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = C.c_int
_lib.sable_status_string.argtypes = [C.c_int]
_lib.sable_status_string.restype = C.c_char_p
_lib.sable_last_error.argtypes = []
_lib.sable_last_error.restype = C.c_char_p
_lib.sable_abi_version.argtypes = []
_lib.sable_abi_version.restype = C.c_int32


class SableError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = _lib.sable_last_error().decode()
        super().__init__(f"{where}: {_lib.sable_status_string(status).decode()}: {msg}")


def _check(status: int, where: str):
    if status != SABLE_OK:
        raise SableError(status, where)


# ------------------------------------------------------------------ raw calls
# Same names as the C-ABI; pointers are plain integers (device or host).

def sable_vbr_create(desc: sable_vbr_desc, delta_pct: int, rank: int = 0, world: int = 1,
                     stream: int = 0) -> int:
    h = _H()
    sh = sable_shard(rank, world)
    _check(_lib.sable_vbr_create(C.byref(desc), delta_pct, C.byref(sh), _P(stream), C.byref(h)),
           "sable_vbr_create")
    return h.value


def sable_vbr_create_policy(desc: sable_vbr_desc, delta_pct: int, min_area: int = 0,
                            rules=(), rank: int = 0, world: int = 1, stream: int = 0) -> int:
    """sable_vbr_create under a per-shape delta policy: rules is a sequence
    of (h_min, h_max, w_min, w_max, delta), the first match wins (R22)."""
    h = _H()
    sh = sable_shard(rank, world)
    arr = (sable_delta_rule * max(1, len(rules)))(*[sable_delta_rule(*map(int, r)) for r in rules])
    pol = sable_delta_policy(delta_pct, int(min_area), len(rules), arr)
    _check(_lib.sable_vbr_create_policy(C.byref(desc), C.byref(pol), C.byref(sh), _P(stream),
                                        C.byref(h)), "sable_vbr_create_policy")
    return h.value


def sable_spmv(h: int, x_ptr: int, y_ptr: int, stream: int = 0) -> None:
    _check(_lib.sable_spmv(_H(h), _P(x_ptr), _P(y_ptr), _P(stream)), "sable_spmv")


def sable_spmv_host(h: int, x_ptr: int, y_ptr: int, stream: int = 0) -> None:
    _check(_lib.sable_spmv_host(_H(h), _P(x_ptr), _P(y_ptr), _P(stream)), "sable_spmv_host")


def sable_destroy(h: int) -> None:
    _check(_lib.sable_destroy(_H(h)), "sable_destroy")


def sable_get_info(h: int) -> dict:
    info = sable_info()
    _check(_lib.sable_get_info(_H(h), C.byref(info)), "sable_get_info")
    return {k: getattr(info, k) for k, _ in sable_info._fields_}


def sable_export_partition(h: int, out: sable_partition_host) -> None:
    _check(_lib.sable_export_partition(_H(h), C.byref(out)), "sable_export_partition")


def sable_shard_bounds(weights, world: int) -> np.ndarray:
    w = np.ascontiguousarray(weights, dtype=np.int64)
    b = np.zeros(world + 1, dtype=np.int32)
    _check(_lib.sable_shard_bounds(_P(w.ctypes.data), len(w), world, _P(b.ctypes.data)),
           "sable_shard_bounds")
    return b


def sable_exchange_rows(weights, rpntr, world: int) -> np.ndarray:
    """Global row bounds of every rank's slice of y in the all-gather (host)."""
    w = np.ascontiguousarray(weights, dtype=np.int64)
    rp = np.ascontiguousarray(rpntr, dtype=np.int32)
    out = np.zeros(world + 1, dtype=np.int64)
    _check(_lib.sable_exchange_rows(_P(w.ctypes.data), len(w), _P(rp.ctypes.data), world,
                                    _P(out.ctypes.data)), "sable_exchange_rows")
    return out


def sable_comm_check(h: int) -> None:
    _check(_lib.sable_comm_check(_H(h)), "sable_comm_check")


def sable_nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    _check(_lib.sable_nccl_unique_id(C.cast(buf, _P)), "sable_nccl_unique_id")
    return bytes(buf)


def sable_comm_init(h: int, uid: bytes) -> None:
    buf = (C.c_char * 128).from_buffer_copy(uid)
    _check(_lib.sable_comm_init(_H(h), C.cast(buf, _P)), "sable_comm_init")


def sable_comm_fuse(h: int, xa_ptr: int, xb_ptr: int) -> None:
    _check(_lib.sable_comm_fuse(_H(h), _P(xa_ptr), _P(xb_ptr)), "sable_comm_fuse")


def sable_comm_set_peers(h: int, xa_ptr: int, xb_ptr: int, peers_a, peers_b) -> None:
    n = len(peers_a)
    assert len(peers_b) == n
    pa = (C.c_void_p * max(n, 1))(*peers_a)
    pb = (C.c_void_p * max(n, 1))(*peers_b)
    _check(_lib.sable_comm_set_peers(_H(h), _P(xa_ptr), _P(xb_ptr), C.cast(pa, _P),
                                     C.cast(pb, _P), n), "sable_comm_set_peers")


def sable_comm_unfuse(h: int) -> None:
    _check(_lib.sable_comm_unfuse(_H(h)), "sable_comm_unfuse")


def sable_spmv_allgather(h: int, x_ptr: int, xn_ptr: int, stream: int = 0) -> None:
    _check(_lib.sable_spmv_allgather(_H(h), _P(x_ptr), _P(xn_ptr), _P(stream)),
           "sable_spmv_allgather")


def sable_spmv_iterate(h: int, xa_ptr: int, xb_ptr: int, iters: int, stream: int = 0) -> bool:
    r = C.c_int32(0)
    _check(_lib.sable_spmv_iterate(_H(h), _P(xa_ptr), _P(xb_ptr), iters, _P(stream), C.byref(r)),
           "sable_spmv_iterate")
    return bool(r.value)


def sable_partition_grid(nrows: int, ncols: int, nnz: int, rowptr_ptr: int, colidx_ptr: int,
                         mem: int, t_num: int, t_den: int, shifts: bool,
                         stream: int = 0) -> tuple:
    """Alg. 1 on the device: (rpntr, cpntr) as int32 arrays."""
    rp = np.zeros(nrows + 1, dtype=np.int32)
    cp = np.zeros(ncols + 1, dtype=np.int32)
    nbr, nbc = C.c_int32(0), C.c_int32(0)
    _check(_lib.sable_partition_grid(nrows, ncols, nnz, _P(rowptr_ptr), _P(colidx_ptr), mem,
                                     t_num, t_den, 1 if shifts else 0, _P(stream),
                                     _P(rp.ctypes.data), C.byref(nbr), _P(cp.ctypes.data),
                                     C.byref(nbc)), "sable_partition_grid")
    return rp[:nbr.value + 1].copy(), cp[:nbc.value + 1].copy()


def sable_spmm(h: int, x_ptr: int, y_ptr: int, k: int, stream: int = 0) -> None:
    _check(_lib.sable_spmm(_H(h), _P(x_ptr), _P(y_ptr), k, _P(stream)), "sable_spmm")


def sable_serialize(h: int) -> bytes:
    """The handle's image (SABLEVC1) as bytes."""
    n = C.c_int64(0)
    _check(_lib.sable_serialize(_H(h), None, 0, C.byref(n)), "sable_serialize")
    buf = (C.c_char * n.value)()
    _check(_lib.sable_serialize(_H(h), C.cast(buf, _P), n.value, C.byref(n)), "sable_serialize")
    return bytes(buf)


def sable_deserialize(image: bytes, stream: int = 0) -> int:
    h = _H()
    buf = C.create_string_buffer(image, len(image))
    _check(_lib.sable_deserialize(C.cast(buf, _P), len(image), _P(stream), C.byref(h)),
           "sable_deserialize")
    return h.value


def sable_status_string(s: int) -> str:
    return _lib.sable_status_string(s).decode()


def sable_last_error() -> str:
    return _lib.sable_last_error().decode()


def sable_abi_version() -> int:
    return int(_lib.sable_abi_version())


# ------------------------------------------------------------ torch front-end

def _dtype_code(dt) -> int:
    import torch
    if isinstance(dt, torch.dtype):
        ok = {torch.float32: SABLE_F32, torch.float64: SABLE_F64}
    else:
        dt = np.dtype(dt)
        ok = {np.dtype(np.float32): SABLE_F32, np.dtype(np.float64): SABLE_F64}
    if dt not in ok:
        raise TypeError(f"values must be float32 or float64, got {dt}")
    return ok[dt]


class VbrMatrix:
    """A handle over libsable.so.  ``arrays`` is a dict with rpntr, cpntr,
    bpntr, bindx, indx, val and optionally rem_indptr, rem_indices, rem_val
    (numpy arrays or CUDA torch tensors, all of the same kind)."""

    def __init__(self, arrays: dict, nrows: int, ncols: int, delta: int = 50,
                 rank: int = 0, world: int = 1, device=None, policy: dict | None = None):
        import torch
        self.device = torch.device(device or "cuda")
        keep = []
        first = arrays["val"]
        on_dev = isinstance(first, torch.Tensor) and first.is_cuda

        tdt = {np.int32: torch.int32, np.int64: torch.int64, np.float32: torch.float32,
               np.float64: torch.float64}

        def ptr(name, dt):
            a = arrays.get(name)
            if a is None:
                return None, 0
            if on_dev:
                # every array in its ABI dtype on this handle's device (a
                # wrong width would be read as another type by the library)
                if not (isinstance(a, torch.Tensor) and a.is_cuda):
                    raise TypeError(f"{name}: all arrays must be CUDA tensors when val is")
                t = a.to(device=self.device, dtype=tdt[dt]).contiguous()
                keep.append(t)
                return t.data_ptr(), t.numel()
            n = np.ascontiguousarray(a, dtype=dt)
            keep.append(n)
            return n.ctypes.data, n.size

        vdt = np.float64 if _dtype_code(first.dtype) == SABLE_F64 else np.float32
        d = sable_vbr_desc()
        d.nrows, d.ncols = nrows, ncols
        d.rpntr, nrp = ptr("rpntr", np.int32)
        d.cpntr, ncp = ptr("cpntr", np.int32)
        d.bpntr, _ = ptr("bpntr", np.int64)
        d.bindx, nblk = ptr("bindx", np.int32)
        d.indx, _ = ptr("indx", np.int64)
        d.val, nval = ptr("val", vdt)
        d.rem_indptr, _ = ptr("rem_indptr", np.int64)
        d.rem_indices, nrem = ptr("rem_indices", np.int32)
        d.rem_val, _ = ptr("rem_val", vdt)
        d.nbrows, d.nbcols = nrp - 1, ncp - 1
        d.nblocks, d.val_len, d.rem_nnz = nblk, nval, nrem
        d.dtype = SABLE_F64 if vdt == np.float64 else SABLE_F32
        d.mem = SABLE_MEM_DEVICE if on_dev else SABLE_MEM_HOST
        self.dtype = torch.float64 if vdt == np.float64 else torch.float32
        self.np_dtype = vdt
        with torch.cuda.device(self.device):
            stream = torch.cuda.current_stream().cuda_stream
            if policy:
                self.handle = sable_vbr_create_policy(d, int(delta), policy.get("min_area", 0),
                                                      policy.get("rules", ()), rank, world,
                                                      stream)
            else:
                self.handle = sable_vbr_create(d, int(delta), rank, world, stream)
        self.info = sable_get_info(self.handle)
        del keep

    # -- products
    def spmv(self, x, y=None, stream=None):
        import torch
        nloc = self.info["row_end"] - self.info["row_begin"]
        if y is None:
            y = torch.empty(nloc, dtype=self.dtype, device=self.device)
        assert x.dtype == self.dtype and y.dtype == self.dtype and x.is_cuda and y.is_cuda
        assert x.is_contiguous() and y.is_contiguous() and x.numel() == self.info["ncols"]
        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        sable_spmv(self.handle, x.data_ptr(), y.data_ptr(), s)
        return y

    def spmm(self, X, Y=None, stream=None):
        """Y = A X for X of shape (ncols, k), k in {1, 2, 4, 8} (row-major)."""
        import torch
        nloc = self.info["row_end"] - self.info["row_begin"]
        k = X.shape[1]
        if Y is None:
            Y = torch.empty((nloc, k), dtype=self.dtype, device=self.device)
        assert X.dtype == self.dtype and Y.dtype == self.dtype and X.is_cuda and Y.is_cuda
        assert X.is_contiguous() and Y.is_contiguous() and X.shape[0] == self.info["ncols"]
        assert Y.shape == (nloc, k)
        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        sable_spmm(self.handle, X.data_ptr(), Y.data_ptr(), k, s)
        return Y

    def spmv_host(self, x: np.ndarray, y: np.ndarray | None = None, stream=None) -> np.ndarray:
        import torch
        nloc = self.info["row_end"] - self.info["row_begin"]
        if y is None:
            y = np.empty(nloc, dtype=self.np_dtype)
        assert x.dtype == self.np_dtype and y.dtype == self.np_dtype
        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        sable_spmv_host(self.handle, x.ctypes.data, y.ctypes.data, s)
        return y

    def comm_init(self, uid: bytes):
        sable_comm_init(self.handle, uid)

    def comm_check(self):
        sable_comm_check(self.handle)

    def comm_fuse(self, x_a, x_b):
        """Register the ping-pong buffers for the fused exchange epilogue
        (collective; plain cudaMalloc memory)."""
        sable_comm_fuse(self.handle, x_a.data_ptr(), x_b.data_ptr())

    def comm_set_peers(self, x_a, x_b, peers_a, peers_b):
        sable_comm_set_peers(self.handle, x_a.data_ptr(), x_b.data_ptr(),
                             [p.data_ptr() for p in peers_a], [p.data_ptr() for p in peers_b])

    def comm_unfuse(self):
        sable_comm_unfuse(self.handle)

    def spmv_allgather(self, x, x_next, stream=None):
        import torch
        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        sable_spmv_allgather(self.handle, x.data_ptr(), x_next.data_ptr(), s)
        return x_next

    def iterate(self, x_a, x_b, iters: int, stream=None):
        import torch
        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        in_b = sable_spmv_iterate(self.handle, x_a.data_ptr(), x_b.data_ptr(), iters, s)
        return x_b if in_b else x_a

    # -- images (compile once, run many)
    def serialize(self) -> bytes:
        return sable_serialize(self.handle)

    @classmethod
    def from_image(cls, image: bytes, device=None) -> "VbrMatrix":
        """A handle loaded from sable_serialize's image, without re-inspection."""
        import torch
        self = cls.__new__(cls)
        self.device = torch.device(device or "cuda")
        with torch.cuda.device(self.device):
            self.handle = sable_deserialize(image, torch.cuda.current_stream().cuda_stream)
        self.info = sable_get_info(self.handle)
        f64 = self.info["dtype"] == SABLE_F64
        self.dtype = torch.float64 if f64 else torch.float32
        self.np_dtype = np.float64 if f64 else np.float32
        return self

    # -- parity export
    def export(self) -> dict:
        i = self.info
        nc, nd, te, rn = i["n_cells"], i["n_dense"], i["tile_elems"], i["rem_nnz"]
        nloc = i["row_end"] - i["row_begin"]
        out = dict(cell_br=np.zeros(nc, np.int32), cell_bc=np.zeros(nc, np.int32),
                   cell_cnt=np.zeros(nc, np.int64), cell_dense=np.zeros(nc, np.uint8),
                   tile_off=np.zeros(nd + 1, np.int64), tile_val=np.zeros(te, self.np_dtype),
                   ublocks=np.zeros(nc - nd, np.int64), rem_indptr=np.zeros(nloc + 1, np.int64),
                   rem_indices=np.zeros(rn, np.int32), rem_val=np.zeros(rn, self.np_dtype))
        p = sable_partition_host(**{k: v.ctypes.data for k, v in out.items()})
        sable_export_partition(self.handle, p)
        return out

    def close(self):
        if getattr(self, "handle", None):
            sable_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def partition_grid(rowptr, colidx, ncols: int, t_num: int, t_den: int, shifts: bool = True,
                   stream=None) -> tuple:
    """Alg. 1 on the GPU for a CSR pattern: rowptr (int64,
    nrows+1) and colidx (int32), both CUDA tensors or both numpy arrays.
    Returns (rpntr, cpntr) as int32 numpy arrays (readings R17, R19-R21)."""
    import torch
    on_dev = isinstance(rowptr, torch.Tensor) and rowptr.is_cuda
    if on_dev:
        rp = rowptr.to(torch.int64).contiguous()
        ci = colidx.to(torch.int32).contiguous()
        rp_ptr, ci_ptr, nrows, nnz = rp.data_ptr(), ci.data_ptr(), rp.numel() - 1, ci.numel()
        mem = SABLE_MEM_DEVICE
    else:
        rp = np.ascontiguousarray(rowptr, dtype=np.int64)
        ci = np.ascontiguousarray(colidx, dtype=np.int32)
        rp_ptr, ci_ptr, nrows, nnz = rp.ctypes.data, ci.ctypes.data, rp.size - 1, ci.size
        mem = SABLE_MEM_HOST
    s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    return sable_partition_grid(nrows, ncols, nnz, rp_ptr, ci_ptr, mem, t_num, t_den, shifts, s)
