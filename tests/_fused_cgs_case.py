"""Run in a subprocess by test_gpu_parity.py::test_fused_cgs2_opt_in_matches_reference with
SE_CGS_FUSED=1 (the engine reads the switch once per process): the cfg5 proxy slices through the
fused CGS2 path must match the reference exactly like the default path does."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_05215_b200 import api  # noqa: E402

g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cfg5p.npz"))
A = api.DeviceCsr.laplacian([24, 24, 24])
A.scale_sym(g["d"])
lo, hi = g["bounds"]
bp, est = g["bp"], g["est"]
for s in (2, 7):
    f = api.find_pol(bp[s], bp[s + 1], api.SpectralBounds(lo, hi))
    r = api.cheb_lan_tr(A, None, f, bp[s], bp[s + 1],
                        api.SolverConfig(res_tol=1e-8, est_count=int(np.ceil(est[s])), seed=5))
    ref = g[f"slice{s}_vals"]
    assert r.eigenvalues.size == ref.size, (s, r.eigenvalues.size, ref.size)
    assert np.all(np.abs(r.eigenvalues - ref) <= 1e-10 * np.abs(ref))
    assert np.all(r.residuals <= 1e-8 * np.maximum(1.0, np.abs(r.eigenvalues)))
print("fused-ok")
