"""sliceeig-b200: B200-native polynomial-filtering hot path of EVSL (arXiv 1802.05215).

The compute path is libsliceeig_cuda.so (hand-written sm_100a kernels + C++ host engine behind the
C ABI in include/sliceeig_cuda.h).  ``api`` mirrors the reference's sliceeig API in Python;
``pipeline`` is the sliced-solve pipeline (bounds -> KPM DOS -> slicing -> per-slice filtered
Lanczos) with one process per GPU.
"""
from ._lib import LIB_PATH, LibraryNotBuilt  # noqa: F401

__all__ = ["api", "pipeline", "LIB_PATH", "LibraryNotBuilt"]
