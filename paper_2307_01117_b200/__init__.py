"""libheat1d: B200-native explicit 1D periodic heat-equation stencil (arxiv 2307.01117 §2).

The product is the C-ABI shared library ``libheat1d.so`` (include/heat1d.h,
sources in csrc/); this package is its thin Python binding.
"""
from .heat1d import (  # noqa: F401
    EXPORTS,
    Heat1D,
    Heat1DError,
    buffer_len,
    default_opts,
    get_unique_id,
    load,
    partition,
    plan_exchange,
    strerror,
)

__all__ = ["Heat1D", "Heat1DError", "load", "partition", "plan_exchange", "get_unique_id",
           "buffer_len", "default_opts", "strerror", "EXPORTS"]
