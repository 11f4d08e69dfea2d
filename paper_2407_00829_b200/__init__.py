"""SABLE (arXiv 2407.00829) VBR SpMV hot path, B200-native.

The product is ``libsable.so`` (C-ABI in ``include/sable.h``, CUDA sources in
``csrc/``); ``sable`` is its thin ctypes binding.  Importing ``sable`` fails
loudly when the library is not built -- there is no CPU fallback.
"""
__all__ = ["sable", "build"]
