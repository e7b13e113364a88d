"""CPU oracle for the PRNGD hot path (Demchik & Gulov, arXiv 1401.8230).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package.  The product package
``paper_1401_8230_b200`` never imports it, and it never imports the product.

The arithmetic lives in ``prngd_oracle.c`` (plain C, one IEEE binary64 RN rounding per
operation, ``-ffp-contract=off``); this module only builds it and marshals numpy arrays.
"""
from .oracle import *  # noqa: F401,F403
