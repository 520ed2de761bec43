"""zkl: a B200-native implementation of zkLLM's tlookup prover hot path (arXiv 2404.16109, §4).

The compute path is libzkl.so (hand-written sm_100a CUDA behind the C ABI in include/zkl.h);
`paper_2404_16109_b200.zkl` is the ctypes binding.  See DESIGN.md.
"""
from . import zkl  # noqa: F401

__all__ = ["zkl"]
