"""Subprocess body for test_kpm_kernel_variants (SE_KPM_KERNEL is read once per process):
prints the max scaled moment error of each case against the oracle."""
import json
import sys

import numpy as np

from oracle import clib
from paper_1802_05215_b200 import api


def irregular(n, seed):
    """Symmetric matrix with 0..8 entries per row (some empty rows): the ELL path's padding."""
    rng = np.random.default_rng(seed)
    deg = np.zeros(n, int)
    rows, cols, vals = [], [], []
    for i in range(n):
        if i % 11 == 5:
            continue  # empty row (and column)
        rows.append(i); cols.append(i); vals.append(2.0 + rng.random())
        deg[i] += 1
    for i in range(n):
        for _ in range(int(rng.integers(0, 5))):
            j = int(rng.integers(0, n))
            if j == i or i % 11 == 5 or j % 11 == 5 or deg[i] >= 8 or deg[j] >= 8:
                continue
            if any(r == i and c == j for r, c in zip(rows[-8:], cols[-8:])):
                continue
            v = float(rng.standard_normal()) * 0.3
            rows += [i, j]; cols += [j, i]; vals += [v, v]
            deg[i] += 1; deg[j] += 1
    a = api.CsrMatrix.from_triplets(n, rows, cols, vals)
    return a


out = {}
cases = [("lap20", api.gen_laplacian([20, 20, 20]), (0.0, 12.0)),
         ("lap2d", api.gen_laplacian([37, 23]), (0.0, 8.0)),
         ("irr", irregular(3001, 7), (-4.0, 6.0))]
for name, a, (lo, hi) in cases:
    assert name != "irr" or max(np.diff(a.row_ptr)) <= 8
    for nvec in (16, 21, 6):
        z = api.kpm_moments(a, api.SpectralBounds(lo, hi), 40, nvec, seed=3)
        zr = clib.kpm_moments(a.row_ptr, a.col_idx, a.vals, lo, hi, 40, nvec, 3)
        zn, zrn = z / (nvec * a.n), zr / (nvec * a.n)
        err = np.abs(zn - zrn) / np.maximum(np.abs(zrn), abs(zrn[0]))
        out[f"{name}/{nvec}"] = float(err.max())
print(json.dumps(out))
