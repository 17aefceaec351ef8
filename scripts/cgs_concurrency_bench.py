"""Aggregate reorthogonalisation throughput when T slices' CGS passes run concurrently (one
context + basis per thread, as when 8 slices share a GPU): does HBM stay saturated?"""
import ctypes as C, os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_05215_b200 import _lib, api

n, k, reps = 262144, int(sys.argv[1]) if len(sys.argv) > 1 else 1440, int(sys.argv[2]) if len(sys.argv) > 2 else 1500
by = 16.0 * n * k + 24.0 * n
for T in (1, 2, 4, 8):
    ctxs = [api.Context(0) for _ in range(T)]
    ms = [C.c_double() for _ in range(T)]
    bar = threading.Barrier(T + 1)
    def run(i):
        bar.wait()
        _lib.call("se_cgs_bench", ctxs[i].handle, n, k, reps, C.byref(ms[i]))
    th = [threading.Thread(target=run, args=(i,)) for i in range(T)]
    for t in th: t.start()
    bar.wait()
    t0 = time.perf_counter()
    for t in th: t.join()
    el = time.perf_counter() - t0
    # each thread's device-timed window covers its own passes; long runs make the windows
    # overlap almost entirely (per-thread setup is < 1 s), so total bytes / longest window is the
    # aggregate rate
    agg = T * reps * by / (max(m.value for m in ms) * 1e-3) / 1e9
    print(f"T={T}: per-thread {[round(m.value/reps) for m in ms]} ms... us/pass "
          f"{[round(m.value/reps*1e3) for m in ms]}, aggregate {agg:.0f} GB/s ({100*agg/6548.5:.0f}% of 6548.5)")
    for c in ctxs: c.close()
