"""Time one reorthogonalisation pass (GEMV-T + GEMV-N) against an n x k basis (production graph)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_05215_b200 import _lib, api
ctx = api.default_context(0)
peak = 6550.7
for spec in (sys.argv[1] if len(sys.argv) > 1 else "262144,1440").split(";"):
    n, k = (int(x) for x in spec.split(","))
    ms = C.c_double()
    reps = 20
    _lib.call("se_cgs_bench", ctx.handle, n, k, reps, C.byref(ms))
    per = ms.value / reps
    by = 16.0 * n * k + 24.0 * n
    print(f"n={n} k={k}: {per*1e3:.1f} us/pass  {by/(per*1e-3)/1e9:.0f} GB/s  ({100*by/(per*1e-3)/1e9/peak:.1f}% of {peak})")
