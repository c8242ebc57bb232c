"""B200-native InstantAvatar per-ray render/train hot path (arXiv 2212.10550).

The compute path is libarfx.so (hand-written sm_100a CUDA behind the C-ABI in
include/arfx.h); this package is the Python mirror of the reference `arf` API
over that library. Importing does not touch the GPU; every compute call raises
if the library or the GPU is missing (no CPU fallback).
"""
from . import arf, fixtures  # noqa: F401
from ._lib import ArfxError, InvalidArgument, DomainError, NumericError, DataError, NoDevice  # noqa: F401

__all__ = ["arf", "fixtures", "ArfxError", "InvalidArgument", "DomainError", "NumericError", "DataError",
           "NoDevice"]
