"""Build libsable.so in-tree with nvcc for sm_100a (no torch extension
machinery: the library has a plain C ABI, include/sable.h)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libsable.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    import nvidia.nccl  # torch's bundled NCCL (2.28) ships its headers too

    base = list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def build(force: bool = False, verbose: bool = False, variant: str = "",
          extra: tuple = ()) -> str:
    """Build libsable.so; `variant` + `extra` nvcc flags build an A/B variant
    libsable_<variant>.so (selected at import with SABLE_LIB=<variant>)."""
    srcs = sources()
    LIB = os.path.join(PKG, f"libsable_{variant}.so" if variant else "libsable.so")
    bdir = os.path.join(PKG, "build" + (f"_{variant}" if variant else ""))
    deps = srcs + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "sable.h")]
    if (not force and os.path.exists(LIB)
            and os.path.getmtime(LIB) >= max(os.path.getmtime(p) for p in deps)):
        return LIB
    inc, lib = _nccl_dirs()
    nvcc = os.environ.get("NVCC", "nvcc")
    os.makedirs(bdir, exist_ok=True)
    cmds, objs = [], []
    for s in srcs:
        o = os.path.join(bdir, os.path.basename(s) + ".o")
        cmd = [nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-I", CSRC,
               "-I", inc, *extra, "-c", s, "-o", o]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        cmds.append(cmd)
        objs.append(o)
    # one nvcc per source, in parallel (they are independent translation units)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 4)) as ex:
        list(ex.map(subprocess.check_call, cmds))
    cmd = [nvcc, *ARCH, "-shared", "-o", LIB, *objs, "-L", lib, "-l:libnccl.so.2",
           "-Xlinker", "-rpath=" + lib, "-lcudart"]
    subprocess.check_call(cmd)
    return LIB


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if a not in ("--force", "-v")]
    # python build.py [--force] [-v] [variant -DFLAG=...]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv,
                variant=args[0] if args else "", extra=tuple(args[1:])))
