"""Rayleigh-Ritz contraction (k_ritz_gemm, DMMA) timing on the workload shapes.

    python scripts/gemm_bench.py

U = W Y with W the row-major Krylov basis (n x steps) and Y the candidate Ritz coefficients
(steps x nc): cfg2 slice 0 (n = 262,144, steps 2,880, ~720 candidates), a mid slice, the cfg4/cfg5
chunk shape (n ~ 2M, steps 2,504, 250 candidates per chunk), and the subspace-iteration Gram
(q x q over n rows, split-K)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_05215_b200 import api  # noqa: E402

ctx = api.default_context(0)
for m, n, k, row, what in [(262144, 720, 2880, True, "cfg2 slice 0: U = W Y"),
                           (262144, 280, 1184, True, "cfg2 slice 4: U = W Y"),
                           (262144, 1440, 2880, True, "cfg2 slice 0: thick-restart vectors"),
                           (2097152, 250, 2504, True, "cfg5 chunk: U = W Y"),
                           (400, 400, 262144, True, "cheb_si Gram T^T (A T), q = 400 (split-K)"),
                           (262144, 400, 400, False, "cheb_si rotation Y = T V, q = 400")]:
    ms = api.mult_cols_bench(m, n, k, a_rowmajor=row, reps=3, ctx=ctx)
    tf = 2.0 * m * n * k / (ms * 1e-3) / 1e12
    print(f"{what}: M={m} N={n} K={k}: {ms:.2f} ms, {tf:.1f} TFLOP/s fp64")
