"""Run one BASELINE config through the GPU pipeline and print per-stage / per-slice timing."""
import argparse, json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_05215_b200 import api
from paper_1802_05215_b200.pipeline import Plan, GpuBackend, run

CFGS = {
    "cfg1": dict(dims=[100, 100], plan=dict(xi=0.4, eta=1.6, ns=2, solver="nr", damping="jackson",
                 dos_m=80, dos_nvec=20, probes="rademacher", tol=1e-8, seed=0)),
    "cfg2": dict(dims=[64, 64, 64], plan=dict(xi=0.6, eta=1.2, ns=8, solver="tr", damping="sigma",
                 dos_m=100, dos_nvec=40, probes="gaussian", tol=1e-8, seed=1234)),
}
ap = argparse.ArgumentParser()
ap.add_argument("cfg")
ap.add_argument("--repeat", type=int, default=1)
ap.add_argument("--jobs", type=int, default=0)
ap.add_argument("--solver", default=None)
ap.add_argument("--only", default=None)
ap.add_argument("--resident", type=int, default=1, help="resident filter: 0 off, 1 on (default)")
a = ap.parse_args()
api.set_resident_filter(a.resident)
c = CFGS[a.cfg]
p = dict(c["plan"])
if a.solver:
    p["solver"] = a.solver
plan = Plan(**p, jobs=a.jobs, only=[int(q) for q in a.only.split(",")] if a.only else None)
be = GpuBackend(dims=c["dims"])
ev = api.laplacian_analytic_eigs(c["dims"])
for rep in range(a.repeat):
    t0 = time.time()
    r = run(plan, be)
    el = time.time() - t0
    print(f"[{a.cfg}] total {el:.2f}s bounds {r.t_bounds:.2f} dos {r.t_dos:.2f} solve {r.t_solve:.2f} "
          f"found {r.n_found} -> {r.n_found/el:.1f} eig/s  bounds=({r.lmin!r},{r.lmax!r})")
    for s in r.slices:
        lo, hi = s.lo, s.hi
        truth = int(np.sum((ev > lo + (1e-10*(r.lmax-r.lmin) if s.index > 0 else -1e300)) & (ev <= hi + (1e-10*(r.lmax-r.lmin) if s.index + 1 < len(r.slices) else 1e300)) & (ev >= lo) & (ev <= hi)))
        maxerr = 0.0
        if s.eigenvalues.size:
            # nearest analytic eigenvalue
            idx = np.searchsorted(ev, s.eigenvalues)
            cand = np.stack([ev[np.clip(idx-1,0,ev.size-1)], ev[np.clip(idx,0,ev.size-1)]])
            maxerr = float(np.min(np.abs(cand - s.eigenvalues), axis=0).max() / max(1e-300, np.abs(s.eigenvalues).max()))
        print(f"  slice {s.index} [{lo:.8f},{hi:.8f}] est {s.est:.1f} deg {s.degree} found {s.eigenvalues.size} truth {truth} "
              f"niter {s.niter} nmv {s.n_A_matvec} {s.seconds:.2f}s (start {s.t_start:.2f} mv {s.t_mv:.2f} orth {s.t_orth:.2f}) maxrelerr {maxerr:.2e} maxres {s.residuals.max() if s.residuals.size else 0:.1e} err={s.error}")
print("launches", be.launches())
