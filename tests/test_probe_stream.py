"""Host probe generation (se_probe_block): probes [first, first+count) of Rng(seed)'s stream,
row-major.  Threads start their probes by MT19937-64 jump-ahead (mt64.cpp) and ranks skip the
probes they do not own the same way; the values must equal the reference Rng's serial draw
(rng.hpp:43-58, via oracle/_ref) bit for bit, on both sides of the parallel/jump thresholds."""
import ctypes as C

import numpy as np
import pytest

from oracle import reflib
from paper_1802_05215_b200 import _lib


def probes(seed, kind, n, first, count):
    out = np.empty(n * count)
    _lib.call("se_probe_block", seed, 1 if kind == "normal" else 0, n, first, count,
              out.ctypes.data_as(C.POINTER(C.c_double)))
    return out.reshape(n, count)


@pytest.mark.parametrize("seed,kind,n,first,count", [
    (1, "rademacher", 1000, 0, 5),        # serial
    (3, "normal", 1001, 2, 7),            # odd n: Box-Muller spare crosses probes (serial)
    (7, "rademacher", 131072, 0, 20),     # parallel jump-ahead fill, two device blocks
    (9, "normal", 131072, 3, 17),         # parallel Gaussian (n even, no pending spare)
    (11, "rademacher", 131072, 130, 16),  # rank skip by jump-ahead (17M draws)
    (13, "normal", 131071, 1, 16),        # odd n at parallel size: serial fallback
    (15, "normal", 131072, 129, 3),       # Gaussian skip by jump-ahead
])
def test_probe_block_matches_reference_stream(seed, kind, n, first, count):
    got = probes(seed, kind, n, first, count)
    ref = reflib.rng_vectors(seed, kind, n, first + count)[first:].reshape(count, n).T
    assert np.array_equal(got, ref)


def test_probe_block_rejects_bad_arguments():
    with pytest.raises(ValueError):
        probes(1, "rademacher", 0, 0, 1)
    with pytest.raises(ValueError):
        probes(1, "rademacher", 10, -1, 1)
