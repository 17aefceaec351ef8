"""CGS2 step: two unfused passes (4 reads of W) vs the fused path (3 reads)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_05215_b200 import _lib, api
ctx = api.default_context(0)
for spec in (sys.argv[1] if len(sys.argv) > 1 else "262144,1440").split(";"):
    n, k = (int(x) for x in spec.split(","))
    res = {}
    for mode in (0, 1):
        ms = C.c_double()
        _lib.call("se_cgs2_bench", ctx.handle, n, k, 10, mode, C.byref(ms))
        res[mode] = ms.value / 10
    by4 = 32.0 * n * k  # four reads of W (8 B each)
    print(f"n={n} k={k}: unfused {res[0]*1e3:.0f} us ({by4/(res[0]*1e-3)/1e9:.0f} GB/s eff), fused {res[1]*1e3:.0f} us "
          f"(speed-up {res[0]/res[1]:.2f}x; {by4/(res[1]*1e-3)/1e9:.0f} GB/s of 4-read-equivalent)")
