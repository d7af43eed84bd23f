"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the ParDNN weighted-level sweep.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  It
shares no code with ``paper_2008_08636_b200`` (the CUDA path); see
``oracle/oracle.c`` for the definitions and their PAPER.md citations.
"""
from .oracle import (  # noqa: F401
    OracleGraph,
    OracleError,
    build_lib,
    REMOVED,
    UNASSIGNED,
    KIND_NORMAL,
    KIND_RESIDUAL,
    KIND_REFERENCE,
    EVAL_DTYPE,
)
