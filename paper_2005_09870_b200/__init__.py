"""B200-native exact wavelet decomposition of product-convolution operators (arxiv 2005.09870).

The product is libpcwd.so (C ABI, include/pcwd.h) with its sm_100a kernels; this package
is the thin Python binding.  See DESIGN.md.
"""
from .pcwd import Decomposition, PcwdError, Spec, lib, num_subbands, plan_shard, plan_stencil, validate  # noqa: F401

__all__ = ["Decomposition", "PcwdError", "Spec", "lib", "plan_shard", "plan_stencil", "validate", "num_subbands"]
