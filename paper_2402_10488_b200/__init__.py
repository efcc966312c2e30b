"""B200-native batched parametric source iteration (arxiv 2402.10488 hot path).

The compute path is librte_b200.so (hand-written sm_100a CUDA kernels behind
the C-ABI of include/rte_b200.h); ``rte`` mirrors the reference's host API.
"""
from . import capi  # noqa: F401

__all__ = ["capi", "rte", "build"]
