import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_05215_b200 import _lib, api
ctx = api.default_context(0)
for spec in sys.argv[1].split(";"):
    dims = [int(x) for x in spec.split(",")]
    A = api.DeviceCsr.laplacian(dims, ctx)
    for nv in (1, 2, 4, 8):
        ms = C.c_double()
        _lib.call("se_multi_filter_bench", ctx.handle, A.handle, nv, 100, 5, C.byref(ms))
        per = ms.value / 500 * 1e3
        print(f"{dims} nv={nv}: {per:.2f} us/degree ({per/nv:.2f} us per vector-degree)")
    ms = C.c_double()
    _lib.call("se_block_filter_bench", ctx.handle, A.handle, 100, 5, C.byref(ms))
    per = ms.value / 500 * 1e3
    nnz = A.nnz
    gb = (12.0 * nnz + 4.0 * (A.n + 1) + 40.0 * A.n * 8) / 1e9
    print(f"{dims} row-major block kernel, 8 vectors: {per:.2f} us/degree ({per/8:.2f} us per vector-degree, "
          f"{gb / (per * 1e-6):.0f} GB/s algorithmic)")
    A.free()
