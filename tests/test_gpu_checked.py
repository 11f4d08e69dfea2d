"""The bounds-checked build (libsable_checked.so, -DSABLE_CHECKED): every
index the executors follow -- unit ranges, panel vectors, x-map and side-map
columns, remainder columns, row ranges, combine slots and counters -- is
checked on the device and a violation traps.  compute-sanitizer is closed on
this pool (tests/test_gpu_sanitize.py), so this is the memory-safety evidence:
tests/sanitize_cases.py (C1, random grids fp32/fp64, long rows in pieces, tiny
unit budgets with column chunks and combine groups, SpMM k = 4 and tensor-core
k = 16/128, an iterated exchange step) runs on the checked library in a
subprocess and must match the oracle without a trap."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def test_checked_build_runs_clean():
    lib = os.path.join(ROOT, "paper_2407_00829_b200", "libsable_checked.so")
    if not os.path.exists(lib):
        from paper_2407_00829_b200 import build as b
        b.build(variant="checked", extra=("-DSABLE_CHECKED",))
    env = dict(os.environ, SABLE_LIB="checked")
    code = ("import runpy, sys; sys.argv = ['sanitize_cases.py'];"
            f"runpy.run_path({os.path.join(HERE, 'sanitize_cases.py')!r}, run_name='__main__');"
            "from paper_2407_00829_b200 import sable;"
            "assert sable.LIB_PATH.endswith('libsable_checked.so'), sable.LIB_PATH;"
            "print('checked library:', sable.LIB_PATH)")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=1500,
                       env=env, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "libsable_checked.so" in r.stdout
