"""B200-native Bi-cADMM hot path (arXiv 2405.16267).

The compute path is the C-ABI library ``libbicadmm.so`` (CUDA, sm_100a) declared
in ``include/bicadmm.h``; ``paper_2405_16267_b200.bicadmm`` is its thin ctypes
binding.  Importing this package does not load the library; ``bicadmm.lib()``
does, and raises if the extension has not been built.
"""
__all__ = ["bicadmm", "datagen"]
