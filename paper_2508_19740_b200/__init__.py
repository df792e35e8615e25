"""B200-native Spotlight Attention decode-time retrieval (arXiv 2508.19740).

The product is the sm_100a CUDA library behind include/spl_c.h
(paper_2508_19740_b200/lib/libspl.so) and the C++ drop-in of the reference's
spotlight:: API on top of it. This Python package is host glue: `capi` binds
the C-ABI with ctypes for tests, the bench and multi-GPU (torch.distributed)
orchestration.
"""
__all__ = ["capi"]
