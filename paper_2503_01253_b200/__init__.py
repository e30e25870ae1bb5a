"""B200-native vector-wise N:M SpMM (NM-SpMM, arXiv 2503.01253).

The compute path lives in ``libnmspmm.so`` (hand-written sm_100a CUDA behind
the C ABI declared in ``include/nmspmm.h``); ``nmspmm`` is its thin Python
binding.  Importing this package does not load the library; the first call
into ``nmspmm`` does, and fails loudly if it is missing.
"""
__all__ = ["nmspmm", "synth"]
