"""CPU oracle for the fused SpMM-Legendre recurrence -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline.  The product package (paper_1509_08360_b200) never
imports it.  See oracle/csemb_oracle.c for the reference file:line map and
tests/test_oracle.py for the pins against the reference's golden vectors.
"""

from .oracle import *  # noqa: F401,F403
