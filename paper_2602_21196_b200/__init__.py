"""B200-native UPipe (Untied Ulysses, arXiv 2602.21196): headwise-chunked Ulysses
context-parallel attention layer, forward and backward, on hand-written sm_100a
kernels (libupipe.so, C ABI in include/upipe.h)."""
from . import upipe  # noqa: F401
from .layer import UPipeAttention  # noqa: F401

__all__ = ["upipe", "UPipeAttention"]
