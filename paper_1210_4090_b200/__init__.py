"""B200-native Lax-Oleinik min-plus hot path (arXiv 1210.4090 reference `laxol`).

The product is the in-tree CUDA library ``lib/liblaxol_b200.so`` (C-ABI in
``include/laxol_b200.h``); ``api`` mirrors the reference's stepping API over it.
"""
from . import _capi  # noqa: F401

__all__ = ["api"]
