"""B200-native segment x triangle-mesh intersection (arXiv 2305.01867 hot path).

The product is the C-ABI library lib/librsi.so (include/rsi.h, CUDA sm_100a);
this package is its thin Python binding plus the multi-GPU driver.
"""
from .rsi import (  # noqa: F401
    MODES, Handle, Options, RsiError, alloc_outputs, load, rsi_build, rsi_bvh_download, rsi_bvh_info,
    rsi_compact_hits, rsi_free, rsi_get_stats, rsi_intersect, rsi_rebuild, rsi_reset_stats, rsi_test,
    rsi_validate, rsi_version, sparse_barycentric,
)
