"""Time the fused Chebyshev-filter SpMV as it runs in production (graph-captured, warm L2)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_05215_b200 import _lib, api
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
if len(sys.argv) > 3:
    api.set_resident_filter(int(sys.argv[3]))  # 0: one launch per degree, 1: resident (default)
ctx = api.default_context(0)
for spec in (sys.argv[1] if len(sys.argv) > 1 else "160,160,160").split(";"):
    dims = [int(x) for x in spec.split(",")]
    A = api.DeviceCsr.laplacian(dims, ctx)
    f = api.find_pol(1.1691525, 1.2, api.SpectralBounds(0.0, 12.0 if len(dims) == 3 else 8.0))
    s, keep = f._c()
    ms, nl, by = C.c_double(), C.c_long(), C.c_double()
    _lib.call("se_filter_bench", ctx.handle, A.handle, C.byref(s), reps, C.byref(ms), C.byref(nl), C.byref(by))
    print(f"dims {dims} n={A.n} nnz={A.nnz} deg {f.k}: {ms.value/nl.value*1e3:.2f} us/launch, "
          f"{by.value/(ms.value*1e-3)/1e9:.1f} GB/s algorithmic ({by.value/nl.value/1e6:.1f} MB/launch)")
    A.free()
