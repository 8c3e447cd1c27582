"""B200-native (sm_100a) online-normalizer softmax and fused softmax+TopK.

A drop-in for the hot path of the reference library ``osmx``
(arXiv 1805.02867): the C-ABI ``include/osmx_b200.h`` implemented by
``libosmx_b200.so`` (hand-written CUDA for sm_100a), with the reference's
API mirrored in ``paper_1805_02867_b200.osmx`` and the multi-GPU row
sharder / V-split combine in ``paper_1805_02867_b200.shard``.
"""
from ._lib import LIB_PATH, OsmxLibraryError, launch_count, load  # noqa: F401

__all__ = ["LIB_PATH", "OsmxLibraryError", "launch_count", "load"]
