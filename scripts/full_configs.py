"""BASELINE configs[3] (cfg4) and configs[4] (cfg5) at FULL size on one GPU: matrix generation,
bounds, KPM DOS, window / slicing, filter degrees and per-slice DOS estimates for all 8 slices,
then one sub-window of slice 0 solved with ChebLanTr (the full slices hold ~5,000 (cfg4) and
~10,000 (cfg5) eigenpairs each, hours of GPU time and beyond the reference's dense_sym_eig guard
at its default m = 4 est).  Residuals come back from the device and a sample is re-checked with
rayleigh_and_residual; the sub-window count is compared with the DOS estimate.

    python scripts/full_configs.py [cfg4|cfg5|both] [--sub 16] [--out path.json]
"""
import argparse, json, math, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_05215_b200 import api
from paper_1802_05215_b200.pipeline import slice_clipped


def dos_window(curve, q0, q1):
    """First DOS grid points with normalised cumulative mass >= q0 / q1."""
    x, y = np.asarray(curve.xdos), np.asarray(curve.ydos)
    cum = np.concatenate([[0.0], np.cumsum(0.5 * (y[1:] + y[:-1]) * np.diff(x))])
    cum /= cum[-1]
    return float(x[np.argmax(cum >= q0)]), float(x[np.argmax(cum >= q1)])


def staged(name, A, seed, window, tol, sub, analytic=None, dos_m=100, dos_nvec=40, npts=3000):
    rec = {"config": name, "n": A.n, "nnz": A.nnz}
    t = time.perf_counter()
    b = api.lan_tr_bounds(A, 1e-4, 60, 40, seed)
    rec["bounds"] = [b.lmin, b.lmax]
    rec["t_bounds_s"] = round(time.perf_counter() - t, 3)
    t = time.perf_counter()
    z = api.kpm_moments(A, b, dos_m, dos_nvec, seed=seed)
    curve = api.kpm_curve(z / (dos_nvec * float(A.n)), A.n, b, npts)
    rec["t_dos_s"] = round(time.perf_counter() - t, 3)
    rec["dos"] = {"m": dos_m, "n_vec": dos_nvec, "npts": npts, "probes": "rademacher", "seed": seed}
    xi, eta = window(curve) if callable(window) else window
    rec["window"] = [xi, eta]
    bp, est = slice_clipped(curve, xi, eta, 8)
    rec["breakpoints"] = [float(v) for v in bp]
    rec["est_counts"] = [round(float(v), 1) for v in est]
    rec["degrees"] = [api.find_pol(bp[i], bp[i + 1], b).k for i in range(8)]
    if analytic is not None:
        rec["analytic_count_window_B_eq_I"] = analytic
    if sub <= 0:
        return rec
    # one sub-window of slice 0
    lo = float(bp[0])
    hi = lo + (float(bp[1]) - lo) / sub
    f = api.find_pol(lo, hi, b)
    est_sub = api.dos_count(curve, lo, hi)
    cfg = api.SolverConfig(res_tol=tol, seed=seed, est_count=max(1, int(math.ceil(est_sub))))
    t = time.perf_counter()
    r = api.cheb_lan_tr(A, None, f, lo, hi, cfg, want_vectors=True)
    el = time.perf_counter() - t
    lam = np.asarray(r.eigenvalues)
    res = np.asarray(r.residuals)
    chk = []
    for i in range(0, lam.size, max(1, lam.size // 8)):
        l2, r2 = api.rayleigh_and_residual(A, None, r.vectors[:, i])
        chk.append([float(lam[i]), float(l2), float(r2)])
    rec["sub_window"] = {
        "slice": 0, "fraction": f"1/{sub}", "interval": [lo, hi], "degree": f.k,
        "dos_estimate": round(float(est_sub), 1), "found": int(lam.size), "niter": int(r.niter),
        "n_A_matvec": int(r.counters.n_A_matvec), "seconds": round(el, 2),
        "eigenpairs_per_s": round(lam.size / el, 2),
        "max_residual_rel": float(np.max(res / np.maximum(1.0, np.abs(lam)))) if lam.size else None,
        "all_within_tol": bool(np.all(res <= tol * np.maximum(1.0, np.abs(lam)))),
        "in_interval": bool(np.all((lam >= lo) & (lam <= hi))),
        "recheck_lambda_lambda2_res": chk,
    }
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", nargs="?", default="both")
    ap.add_argument("--sub", type=int, default=16)
    ap.add_argument("--out", default="gpurun_out/full_configs.json")
    a = ap.parse_args()
    out = []
    if a.which in ("cfg4", "both"):
        t = time.perf_counter()
        host = api.gen_random_sparse(2_000_000, 1234)
        A = api.DeviceCsr.upload(host)
        tg = time.perf_counter() - t
        rec = staged("cfg4: random banded (half-width 3) + 8 extras, n = 2,000,000, tol 1e-9",
                     A, 1234, lambda c: dos_window(c, 0.49, 0.51), 1e-9, a.sub)
        rec["t_generate_upload_s"] = round(tg, 2)
        out.append(rec)
        print(json.dumps(rec), flush=True)
        A.free()
    if a.which in ("cfg5", "both"):
        t = time.perf_counter()
        A = api.DeviceCsr.laplacian([128, 128, 128])
        _, d = api.mass_scaling(A.n, 1234)
        A.scale_sym(d)
        tg = time.perf_counter() - t
        ev = api.laplacian_analytic_eigs([128, 128, 128])
        rec = staged("cfg5: D A D, A = 128^3 Laplacian, lumped mass uniform [0.5, 1.5], [1, 2], tol 1e-8",
                     A, 1234, (1.0, 2.0), 1e-8, a.sub,
                     analytic=int(api.count_in_interval(ev, 1.0, 2.0)), npts=300)
        rec["t_generate_scale_s"] = round(tg, 2)
        out.append(rec)
        print(json.dumps(rec), flush=True)
        A.free()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
