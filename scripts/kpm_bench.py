"""KPM moment throughput (BASELINE cfg3: 160^3, 300 moments, probes in blocks of 16)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1802_05215_b200 import api
dims = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "160,160,160").split(",")]
m = int(sys.argv[2]) if len(sys.argv) > 2 else 300
nprobe = int(sys.argv[3]) if len(sys.argv) > 3 else 16
A = api.DeviceCsr.laplacian(dims)
b = api.SpectralBounds(0.0, 12.0)
api.kpm_moments(A, b, 4, 16, seed=0, count=16)  # warm
import ctypes as C
from paper_1802_05215_b200 import _lib
ctx = api.default_context(0)
_lib.call("se_ctx_filter_timing", ctx.handle, 1, None, None, None)
t = time.perf_counter()
z = api.kpm_moments(A, b, m, nprobe, seed=0)
el = time.perf_counter() - t
ms, nl, byt = C.c_double(), C.c_long(), C.c_double()
_lib.call("se_ctx_filter_timing", ctx.handle, 0, C.byref(ms), C.byref(nl), C.byref(byt))
print(f"device: {ms.value:.1f} ms for {nl.value} block-steps = {ms.value/nl.value*1e3:.1f} us/step, "
      f"{byt.value/(ms.value*1e-3)/1e9:.0f} GB/s algorithmic ({100*byt.value/(ms.value*1e-3)/1e9/6550.7:.1f}% of 6550.7)")
ab = 12.0 * A.nnz + 4.0 * (A.n + 1)
blocks = (nprobe + 15) // 16
by = blocks * m * (ab + 32.0 * A.n * 16)
print(f"{dims} m={m} probes={nprobe}: {el:.3f} s wall (incl. host probe generation), "
      f"{by/el/1e9:.0f} GB/s algorithmic, {el/(blocks*m)*1e6:.1f} us per block-step")
