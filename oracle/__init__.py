"""fp64 CPU oracle — TEST INFRASTRUCTURE ONLY (see fdpd_oracle.py header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package.  The product path never does.
"""
from . import fdpd_oracle  # noqa: F401
