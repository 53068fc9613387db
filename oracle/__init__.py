"""SOCKET CPU oracle (float64).  TEST INFRASTRUCTURE ONLY -- see socket_oracle.py header.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl
reference) may import this package; the product path never does.
"""
from .socket_oracle import *  # noqa: F401,F403
from .socket_oracle import GROUP_KV_SHARED, GROUP_PER_QHEAD  # noqa: F401
