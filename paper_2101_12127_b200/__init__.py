"""B200-native engine for the tf.data (arXiv 2101.12127) fused
shuffle -> map -> batch -> prefetch path.

The product is ``lib/libdpcuda.so`` (sm_100a kernels + C++ host engine behind
the C ABI in ``include/``).  This package only binds it; importing fails
loudly when the library has not been built.
"""
from ._capi import lib, check, DpError, LIB_PATH  # noqa: F401

__all__ = ["lib", "check", "DpError", "LIB_PATH"]
