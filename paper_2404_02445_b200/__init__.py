"""B200-native PRNet pattern-attention forward (arXiv 2404.02445).

The product is libprnet.so (C ABI, include/prnet.h) built from csrc/ for
sm_100a; this package is its thin Python binding plus the data-parallel
sharding helpers.  See DESIGN.md.
"""
from .prnet import PRNet, PrnetConfig, PrnetError, load_library, EXPORTS  # noqa: F401
from .sharding import shard_windows, all_reduce_error_sums  # noqa: F401

__all__ = ["PRNet", "PrnetConfig", "PrnetError", "load_library", "EXPORTS", "shard_windows",
           "all_reduce_error_sums"]
