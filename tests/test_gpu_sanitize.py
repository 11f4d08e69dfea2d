"""compute-sanitizer over the CUDA path (memcheck, racecheck, synccheck) on
small cases (tests/sanitize_cases.py), one tool per run.  Opt-in: set
SABLE_SANITIZE to a tool name (the B200 profiling guide allows one sanitizer
tool per GPU call); the logs of the committed runs are under profiles/."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

TOOL = os.environ.get("SABLE_SANITIZE", "")


@pytest.mark.skipif(TOOL not in ("memcheck", "racecheck", "synccheck", "initcheck"),
                    reason="set SABLE_SANITIZE=memcheck|racecheck|synccheck|initcheck")
def test_sanitizer():
    here = os.path.dirname(os.path.abspath(__file__))
    log = os.environ.get("SABLE_SANITIZE_LOG", f"/tmp/sanitize_{TOOL}.log")
    cmd = ["compute-sanitizer", f"--tool={TOOL}", "--error-exitcode=99", "--print-limit=50",
           "--log-file", log, sys.executable, os.path.join(here, "sanitize_cases.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500)
    text = open(log).read() if os.path.exists(log) else ""
    assert r.returncode == 0, f"{TOOL}: rc {r.returncode}\n{text[-4000:]}\n{r.stdout[-2000:]}{r.stderr[-2000:]}"
    assert "ERROR SUMMARY: 0 errors" in text, text[-4000:]
