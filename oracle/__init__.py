"""CPU oracle for the SABLE VBR SpMV hot path (arXiv 2407.00829).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_2407_00829_b200`` never imports it and
shares no code with it.

The arithmetic lives in ``sable_oracle.c`` (plain C, fp64, one translation
unit, ``-O2 -ffp-contract=off``); this module is only the ctypes marshalling.
See the header of ``sable_oracle.c`` for the passage each step follows and
DESIGN.md "Readings" for the interpretations R1..R18.
"""
from .oracle import (  # noqa: F401
    OracleError,
    alg1_cuts,
    build,
    partition_grid,
    normalize,
    partition,
    rowptr,
    spmv_csr_mt,
    spmv,
    spmv_rows,
)
