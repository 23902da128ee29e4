"""CPU float64 oracle for the SOFA exact k-NN path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
may import this package.  See sofa_oracle.py for the per-function citations.
"""
from . import sofa_oracle  # noqa: F401
