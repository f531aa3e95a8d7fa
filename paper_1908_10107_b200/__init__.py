"""B200-native ORCA step (arXiv 1908.10107) behind the liborca C-ABI.

Importing the package is cheap; ``paper_1908_10107_b200.orca`` loads the CUDA library
(and fails loudly if it is missing -- there is no CPU fallback).
"""
__all__ = ["orca", "workloads"]
