"""B200-native OCCL hot path (arXiv 2303.06324): a persistent, preemptible sm_100a
daemon kernel running ring AllReduce / AllGather / ReduceScatter / Broadcast over
peer memory, behind the C-ABI in include/occl.h.  See DESIGN.md.
"""
from . import occl  # noqa: F401
from .occl import Comm, local_group, process_group, occlConfigDefault  # noqa: F401
