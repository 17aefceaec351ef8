"""Time the UNMODIFIED reference (oracle/_ref, the reference headers compiled in place) on the full
BASELINE cfg2 workload once, on this container's host cores, and cache the result with the machine
string ("time cfg2/cfg3 once and cache the result with machine details").

  python scripts/cpu_reference_cfg2.py [--jobs 8] [--out profiles/r2_cpu_reference_cfg2.json]

The recipe is bench.py's CFG2 (64^3 Laplacian, bounds by lan_tr_bounds, KPM 100 moments x 40
Gaussian probes, [0.6, 1.2] in 8 DOS slices, ChebLanTr sigma damping, tol 1e-8, seed 1234) through
the reference `sliceeig solve` semantics (tools/sliceeig_main.cpp:464-619: slices on a std::thread
pool of `--jobs` workers).  Test/measurement infrastructure only: bench.py reads the cached JSON.
"""
import argparse
import json
import os
import platform
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import reflib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--jobs", type=int, default=8)
ap.add_argument("--dims", default="64,64,64")
ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_cpu_reference_cfg2.json"))
a = ap.parse_args()
dims = [int(x) for x in a.dims.split(",")]

try:
    cpu = [ln.split(":", 1)[1].strip() for ln in subprocess.run(
        ["lscpu"], capture_output=True, text=True).stdout.splitlines() if ln.startswith("Model name")][0]
except Exception:
    cpu = platform.processor()

rp, ci, v = reflib.laplacian(dims)
t0 = time.perf_counter()
res = reflib.solve(rp, ci, v, 0.6, 1.2, 8, "tr", "sigma", 100, 40, 300, "normal", 1e-8, 1234,
                   jobs=a.jobs)
wall = time.perf_counter() - t0
found = int(sum(len(s["eigenvalues"]) for s in res["slices"]))
out = {
    "workload": f"cfg2: {dims[0]}^3 7-pt Laplacian, KPM 100x40 Gaussian, [0.6,1.2] in 8 slices, "
                "ChebLanTr (sigma) tol 1e-8, seed 1234",
    "impl": "reference (oracle/_ref: /root/reference/proj/include compiled -O3 -DNDEBUG, ref_solve = "
            "sliceeig solve semantics)",
    "machine": {"cpu": cpu, "cores": os.cpu_count(), "jobs": a.jobs, "host": platform.node()},
    "wall_s": round(wall, 2), "eigenpairs": found, "eigenpairs_per_s": round(found / wall, 4),
    "t_bounds": round(res["t_bounds"], 2), "t_dos": round(res["t_dos"], 2),
    "t_solve": round(res["t_solve"], 2), "lmin": res["lmin"], "lmax": res["lmax"],
    "breakpoints": [float(x) for x in res["breakpoints"]],
    "est_counts": [float(x) for x in res["est_counts"]],
    "slices": [{"slice": i, "found": int(len(s["eigenvalues"])), "niter": s["niter"],
                "n_A_matvec": s["n_A_matvec"], "degree": s["degree"],
                "hit_max_its": s["hit_max_its"], "t_mv": round(s["t_mv"], 2),
                "t_orth": round(s["t_orth"], 2), "t_total": round(s["t_total"], 2),
                "max_residual": float(np.max(s["residuals"])) if len(s["residuals"]) else 0.0,
                "error": s["error"]}
               for i, s in enumerate(res["slices"])],
    "eigenvalues": [[float(x) for x in s["eigenvalues"]] for s in res["slices"]],
    "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
}
with open(a.out, "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps({k: out[k] for k in ("wall_s", "eigenpairs", "eigenpairs_per_s", "machine")}))
