"""CPU oracle for the homomorphic linear layer -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this package.  It is independent of the CUDA path (see oracle/ref.py).
"""
from . import ref  # noqa: F401
