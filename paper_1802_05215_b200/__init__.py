"""sliceeig-b200: B200-native polynomial-filtering hot path of EVSL (arXiv 1802.05215).

The compute path is libsliceeig_cuda.so (hand-written sm_100a kernels + C++ host engine behind the
C ABI in include/sliceeig_cuda.h).  ``api`` mirrors the reference's sliceeig API in Python;
``pipeline`` is the sliced-solve pipeline (bounds -> KPM DOS -> slicing -> per-slice filtered
Lanczos) with one process per GPU.
"""
import os as _os

# Up to 32 hardware work queues (default 8): the slice contexts sharing a GPU each drive two
# streams, and with 8 queues a high-priority stream's small synchronising work would sit behind
# another stream's bandwidth-bound kernels.  Must be set before CUDA initialises.
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

from ._lib import LIB_PATH, LibraryNotBuilt  # noqa: F401

__all__ = ["api", "pipeline", "LIB_PATH", "LibraryNotBuilt"]
