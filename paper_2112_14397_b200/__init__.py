"""B200-native DTS-Gate MoE layer (EvoMoE, arXiv 2112.14397).

The product is libmoe_dts.so (csrc/, C ABI in include/moe_dts.h); this package holds
its ctypes binding (_lib) and the call-sequence driver (layer.DTSMoELayer).  Importing
the binding raises if the library is not built -- there is no CPU fallback.
"""
from . import _lib  # noqa: F401

__all__ = ["_lib"]
