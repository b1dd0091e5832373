"""B200-native AttentionPack KV-cache path (arXiv 2603.23914).

Drop-in for the reference ``kvpack`` hot path: prefill compaction (truncated
SVD of head-combined K/V segments) and decode attention over the compressed
cache, as hand-written sm_100a kernels behind the C-ABI in include/kvp_b200.h.
"""
__version__ = "0.1.0"
