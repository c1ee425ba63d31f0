"""B200-native batched SLO-attainment simulator for AlpaServe's placement
search (arXiv 2302.11665).

The hot path -- candidate encoding, the per-(request, candidate) dispatch /
pipeline / admission loop, per-run argmax and the greedy search driver --
runs in libasim.so (include/asim.h): a C++ host runtime plus hand-written
sm_100a CUDA kernels.  This package is its Python binding; it raises on
import if the library is missing (no CPU fallback).
"""

from .api import SearchHandle, SearchResult, Simulator  # noqa: F401
from ._abi import AsimError  # noqa: F401

__all__ = ["Simulator", "SearchHandle", "SearchResult", "AsimError"]
