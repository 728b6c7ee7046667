"""B200-native batched limit-order-book engine (the data-parallel hot path of JAX-LOB,
arXiv 2308.13289, Section 4).

The product is ``liblob.so`` behind the C ABI in ``include/lob.h``; this package is
its thin binding.  See DESIGN.md.
"""
from .lob import (LIB_PATH, LOB_NSTATS, MAX_CAPACITY, MAX_L2_LEVELS, STAT_NAMES, EnvConfig, LobBatch,
                  LobEnv, LobError, LobSession, build_id, launch_count, lib)

__all__ = ["LobBatch", "LobEnv", "LobSession", "EnvConfig", "LobError", "lib", "launch_count", "build_id", "LIB_PATH", "LOB_NSTATS",
           "STAT_NAMES", "MAX_CAPACITY", "MAX_L2_LEVELS"]
