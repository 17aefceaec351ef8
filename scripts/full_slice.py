"""One full DOS slice of BASELINE cfg5 (or a bounded part of a cfg4 slice) at FULL size through the
product pipeline (pipeline.run) on one GPU, with the memory plan: the slice is solved as DOS-mass
windows (m = 4 est each, est <= the device-memory / dense_sym_eig limit), eigenvectors streamed
window by window to a sink that re-checks a sample with rayleigh_and_residual and drops them.

    python scripts/full_slice.py cfg5 [--slice 0] [--out gpurun_out/full_slice_cfg5.json]
    python scripts/full_slice.py cfg4 [--slice 0] [--max-windows 1]

Reported: bounds, DOS breakpoints / estimates (same recipe as scripts/full_configs.py), per window
(interval, DOS estimate, degree, found, iterations, seconds), the slice's total count vs its DOS
estimate, every device residual vs tol max(1, |lambda|), the sampled re-checks, eigenpairs/s.
"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_05215_b200 import api  # noqa: E402
from paper_1802_05215_b200.pipeline import (GpuBackend, Plan, run, window_breakpoints,  # noqa: E402
                                            window_estimate)


def cfg4_window(backend, seed):
    """Middle 2% of the DOS-estimated spectrum (count reading): [t_0.49, t_0.51]."""
    lmin, lmax = backend.bounds(seed)
    z = api.kpm_moments(backend.A, api.SpectralBounds(lmin, lmax), 100, 40, seed=seed)
    c = api.kpm_curve(z / (40.0 * backend.n), backend.n, api.SpectralBounds(lmin, lmax), 3000)
    x, y = np.asarray(c.xdos), np.asarray(c.ydos)
    cum = np.concatenate([[0.0], np.cumsum(0.5 * (y[1:] + y[:-1]) * np.diff(x))])
    cum /= cum[-1]
    return float(x[np.argmax(cum >= 0.49)]), float(x[np.argmax(cum >= 0.51)])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", choices=["cfg4", "cfg5"])
    ap.add_argument("--slice", type=int, default=0)
    ap.add_argument("--max-windows", type=int, default=0, help="cfg4: solve only the first W windows")
    ap.add_argument("--sample", type=int, default=16, help="re-checked vectors per window")
    ap.add_argument("--max-its", type=int, default=0,
                    help="Lanczos step budget (SolverConfig.max_its): a bounded partial solve that "
                         "returns the pairs converged so far with hit_max_its, as the reference does")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    out_path = a.out or f"gpurun_out/full_slice_{a.which}.json"
    t0 = time.perf_counter()
    if a.which == "cfg5":
        A = api.DeviceCsr.laplacian([128, 128, 128])
        _, d = api.mass_scaling(A.n, 1234)
        A.scale_sym(d)
        plan = Plan(xi=1.0, eta=2.0, ns=8, solver="tr", damping="sigma", dos_m=100, dos_nvec=40,
                    probes="rademacher", tol=1e-8, seed=1234, only=[a.slice], want_vectors=True,
                    solver_max_its=a.max_its)
        desc = ("cfg5: D A D, A = 128^3 Laplacian, lumped mass uniform [0.5, 1.5] (seed 1234), "
                "[1, 2] in 8 DOS slices, ChebLanTr tol 1e-8")
    else:
        host = api.gen_random_sparse(2_000_000, 1234)
        A = api.DeviceCsr.upload(host)
        del host
        be0 = GpuBackend(matrix=A)
        xi, eta = cfg4_window(be0, 1234)
        plan = Plan(xi=xi, eta=eta, ns=8, solver="tr", damping="sigma", dos_m=100, dos_nvec=40,
                    dos_npts=3000, probes="rademacher", tol=1e-9, seed=1234, only=[a.slice],
                    want_vectors=False, solver_max_its=a.max_its)
        api.SAMPLE_VECTORS = a.sample  # 83 GB of eigenvectors stay on the device; a sample is checked
        desc = ("cfg4: random banded (half-width 3) + 8 extras, n = 2,000,000 (seed 1234), middle 2% "
                "of the DOS ([t_0.49, t_0.51]) in 8 DOS slices, ChebLanTr tol 1e-9")
    t_setup = time.perf_counter() - t0
    be = GpuBackend(matrix=A)
    checks = []
    tol = plan.tol

    nwin = [0]

    def sink(si, wi, win, vals, res, vecs):
        nwin[0] += 1
        if isinstance(vecs, tuple):  # (positions, sample vectors): the result stayed on the device
            pairs = [(int(j), vecs[1][:, q]) for q, j in enumerate(vecs[0])]
        else:
            step = max(1, vals.size // a.sample)
            pairs = [(j, vecs[:, j]) for j in range(0, vals.size, step)]
        for j, u in pairs:
            lam, r = api.rayleigh_and_residual(A, None, np.ascontiguousarray(u))
            checks.append({"window": wi, "lambda": float(vals[j]), "lambda_recheck": float(lam),
                           "residual_device": float(res[j]), "residual_recheck": float(r)})
        rec = {"window": wi, "lo": win.lo, "hi": win.hi, "est": round(win.est, 1),
               "degree": win.degree, "found": win.found, "niter": win.niter,
               "seconds": round(win.seconds, 1), "hit_max_its": win.hit_max_its}
        print(json.dumps(rec), flush=True)
        return bool(a.max_windows and nwin[0] >= a.max_windows)

    t1 = time.perf_counter()
    res = run(plan, be, sink=sink)
    el = time.perf_counter() - t1
    s = res.slices[0]
    lam, rr = s.eigenvalues, s.residuals
    rec = {
        "config": desc, "n": A.n, "nnz": A.nnz, "bounds": [res.lmin, res.lmax],
        "breakpoints": res.breakpoints.tolist(), "est_counts": [round(float(v), 1) for v in res.est_counts],
        "slice": a.slice, "interval": [s.lo, s.hi], "dos_estimate": round(s.est, 1),
        "window_est_cap": round(window_estimate(A.n, be.memory(), 1), 1),
        "windows": [vars(w) for w in s.windows], "error": s.error,
        "found": int(lam.size), "partial": bool(a.max_windows) or bool(s.hit_max_its),
        "max_its": a.max_its or None,
        "found_vs_estimate": round(lam.size / s.est, 4) if s.est else None,
        "niter": s.niter, "n_A_matvec": s.n_A_matvec, "hit_max_its": s.hit_max_its,
        "max_residual_rel": float(np.max(rr / np.maximum(1.0, np.abs(lam)))) if lam.size else None,
        "all_within_tol": bool(np.all(rr <= tol * np.maximum(1.0, np.abs(lam)))) if lam.size else None,
        "in_interval": bool(np.all((lam >= s.lo - 1e-9) & (lam <= s.hi + 1e-9))) if lam.size else None,
        "sorted_unique": bool(np.all(np.diff(lam) >= 0)) if lam.size else None,
        "rechecks": checks,
        "recheck_max_rel_lambda_diff": max((abs(c["lambda"] - c["lambda_recheck"]) / abs(c["lambda"])
                                            for c in checks), default=None),
        "recheck_max_residual_rel": max((c["residual_recheck"] / max(1.0, abs(c["lambda"]))
                                         for c in checks), default=None),
        "t_setup_s": round(t_setup, 2), "t_bounds_s": round(res.t_bounds, 2),
        "t_dos_s": round(res.t_dos, 2), "t_solve_s": round(res.t_solve, 1), "wall_s": round(el, 1),
        "eigenpairs_per_s": round(lam.size / el, 3) if el > 0 else None,
        "orth_bytes": s.orth_bytes, "t_mv_s": round(s.t_mv, 1), "t_orth_s": round(s.t_orth, 1),
    }
    os.makedirs(os.path.dirname(out_path) or ".", exist_ok=True)
    with open(out_path, "w") as fh:
        json.dump(rec, fh, indent=1)
    print(json.dumps({k: rec[k] for k in ("found", "dos_estimate", "all_within_tol", "wall_s",
                                          "eigenpairs_per_s", "max_residual_rel", "error")}))


if __name__ == "__main__":
    main()
