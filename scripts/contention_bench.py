"""Filter-chain latency under reorthogonalisation load: time the graph-replayed filter (64^3,
degree ~368) alone, then while T other threads replay CGS passes (n = 262144, k = 1440) on
their own contexts -- the situation of 8 slices sharing one GPU."""
import ctypes as C, os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_05215_b200 import _lib, api

def filt(ctx, A, f, reps):
    s, keep = f._c()
    ms, nl, by = C.c_double(), C.c_long(), C.c_double()
    _lib.call("se_filter_bench", ctx.handle, A.handle, C.byref(s), reps, C.byref(ms), C.byref(nl), C.byref(by))
    return ms.value / nl.value * 1e3

ctx = api.Context(0)
A = api.DeviceCsr.laplacian([64, 64, 64], ctx)
f = api.find_pol(1.1691525, 1.2, api.SpectralBounds(0.0, 12.0))
print(f"alone: {filt(ctx, A, f, 5):.2f} us/launch")
for T in (1, 3, 7):
    stop = threading.Event()
    def load():
        c2 = api.Context(0)
        ms = C.c_double()
        while not stop.is_set():
            _lib.call("se_cgs_bench", c2.handle, 262144, 1440, 3000, C.byref(ms))
        c2.close()
    th = [threading.Thread(target=load) for _ in range(T)]
    for t in th: t.start()
    time.sleep(4.0)
    us = filt(ctx, A, f, 5)
    stop.set()
    for t in th: t.join()
    print(f"with {T} CGS threads: {us:.2f} us/launch")

# Reverse direction: the CGS pass (HBM-bound) while T threads replay filter chains -- if the
# filters' matrix/vector traffic reaches HBM under load, the pass slows by that bandwidth share.
def cgs(ctx, reps=40):
    ms = C.c_double()
    _lib.call("se_cgs_bench", ctx.handle, 262144, 1440, reps, C.byref(ms))
    return ms.value / reps * 1e3

print(f"CGS pass alone: {cgs(ctx):.1f} us")
for T in (1, 3, 7):
    stop = threading.Event()
    def fload():
        c2 = api.Context(0)
        A2 = api.DeviceCsr.laplacian([64, 64, 64], c2)
        while not stop.is_set():
            filt(c2, A2, f, 2)
        c2.close()
    th = [threading.Thread(target=fload) for _ in range(T)]
    for t in th: t.start()
    time.sleep(4.0)
    us = cgs(ctx)
    stop.set()
    for t in th: t.join()
    print(f"CGS pass with {T} filter threads: {us:.1f} us")
