"""paper_1308_5626_b200 -- B200-native PSP-GMRES hot path (arXiv 1308.5626).

The compute path is libpspgmres.so (hand-written CUDA for sm_100a behind the C ABI in
include/pspgmres.h); ``pspgmres`` is its thin ctypes binding.  Importing this package does
not load the library; ``pspgmres.lib()`` does, and fails loudly if it is missing.
"""
__all__ = ["inputs", "pspgmres"]
