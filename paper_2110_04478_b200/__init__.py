"""paper_2110_04478_b200 — B200-native Themis chunked hierarchical All-Reduce.

libthemis.so (C ABI, include/themis.h) holds the exact-integer Themis planner
(Algorithm 1 + intra-dimension pre-simulation) and the sm_100a executor
kernel; ``themis`` is the ctypes binding.  See DESIGN.md.
"""

from .themis import *  # noqa: F401,F403
from .themis import __all__  # noqa: F401
