"""B200-native GS-Scale hot path: cull, forwarding gather, tile rasterizer, deferred Adam.

The compute lives in libgss_b200.so (hand-written sm_100a CUDA behind a C ABI, include/gss_b200.h);
this package is the reference-shaped host API over it (see gss.py).
"""
from ._abi import ConfigError, GssError, InvariantViolation, ParseError, lib  # noqa: F401
from .gss import *  # noqa: F401,F403

__all__ = [n for n in dir() if not n.startswith("_")]
