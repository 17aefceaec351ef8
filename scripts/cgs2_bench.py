"""CGS2 step (re-pass forced): two column-major passes (4 reads of W) vs the product's row-major
three-read step (T1 + fused MID + N2, rowgs.cu).  python scripts/cgs2_bench.py "n,k;n,k" """
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_05215_b200 import _lib, api
ctx = api.default_context(0)
for spec in (sys.argv[1] if len(sys.argv) > 1 else "262144,1440").split(";"):
    n, k = (int(x) for x in spec.split(","))
    res = {}
    for mode in (0, 2):
        ms = C.c_double()
        _lib.call("se_cgs2_bench", ctx.handle, n, k, 10, mode, C.byref(ms))
        res[mode] = ms.value / 10
    by4 = 32.0 * n * k  # four reads of W (8 B each)
    by3 = 24.0 * n * k
    print(f"n={n} k={k}: column-major 4-read {res[0]*1e3:.0f} us ({by4/(res[0]*1e-3)/1e9:.0f} GB/s), "
          f"row-major 3-read {res[2]*1e3:.0f} us ({by3/(res[2]*1e-3)/1e9:.0f} GB/s of its 3 reads; "
          f"speed-up {res[0]/res[2]:.2f}x)", flush=True)
