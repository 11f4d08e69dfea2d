"""Seeded synthetic inputs for the SABLE VBR SpMV path (C1..C5 of BASELINE.json).

This module is shared by the tests, ``bench.py`` and ``smoke()``: it serves
both the oracle and the CUDA path and therefore holds NONE of the method's
arithmetic (no counting, classification, packing or multiplication).  It only
draws matrices and encodes them in the paper's input format (VBR arrays,
PAPER.md:221-228, plus an optional CSR remainder) -- see DESIGN.md "Inputs".
"""
from .configs import CONFIGS, Synth, make, random_small  # noqa: F401
from .encode import encode_vbr  # noqa: F401
