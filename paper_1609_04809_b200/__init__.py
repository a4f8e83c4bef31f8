"""B200-native (sm_100a) geometric-multigrid V-cycle hot path of arXiv:1609.04809.

The compute lives in ``libpf_gpu.so`` (paper_1609_04809_b200/csrc, C ABI in
include/pf_gpu.h); ``gmg`` mirrors the reference's multigrid / linear-algebra /
communicator API on top of it and ``levels.StructuredSetup`` is the product's own
communication-free hierarchy setup (include/pf_setup.h).
"""
from . import _lib  # noqa: F401

__all__ = ["_lib", "gmg", "levels"]
