"""BASELINE configs 4 and 5 inputs (generators the reference lacks): structural
properties on CPU, pinned to the checksums stored with the reference-solved golden proxies."""
import numpy as np
import pytest
import scipy.sparse as sp

from paper_1802_05215_b200 import api


def _sp(a):
    return sp.csr_matrix((a.vals, a.col_idx, a.row_ptr), shape=(a.n, a.n))


def test_random_sparse_structure():
    a = api.gen_random_sparse(3000, 11)
    M = _sp(a)
    assert abs(M - M.T).max() == 0.0  # exactly symmetric
    rp, ci = a.row_ptr, a.col_idx
    for i in range(0, a.n, 37):
        cols = ci[rp[i]:rp[i + 1]]
        assert np.all(np.diff(cols) > 0)  # sorted, no duplicates
        band = [j for j in range(max(0, i - 3), min(a.n, i + 4))]
        assert set(band) <= set(cols)  # |i-j| <= 3 (diagonal included)
        assert len(cols) >= len(band) + 8  # at least its own 8 extras
    # diagonal = N(0,1) + 0.1 * sum_j |a_ij|  => residual has unit-normal statistics
    D = M.diagonal()
    off = np.asarray(abs(M).sum(axis=1)).ravel() - np.abs(D)
    z = D - 0.1 * off
    assert abs(z.mean()) < 0.1 and abs(z.std() - 1.0) < 0.1
    assert 22.0 < a.nnz / a.n < 24.0  # ~ 7 + 8 + 8 per row (~46 M at n = 2 M)
    # deterministic in the seed
    b = api.gen_random_sparse(3000, 11)
    assert np.array_equal(a.vals, b.vals) and np.array_equal(a.col_idx, b.col_idx)


def test_random_sparse_pinned_to_golden(golden):
    g = golden("cfg4p")
    a = api.gen_random_sparse(20000, 4)
    assert a.nnz == int(g["nnz"])
    assert [int(a.row_ptr[-1]), int(a.col_idx.sum() % 1000003)] == list(g["rp_check"])
    assert [float(a.vals.sum()), float(np.abs(a.vals).sum())] == list(g["v_check"])


def test_mass_scaling_and_congruence(golden):
    b, d = api.mass_scaling(1000, 5)
    assert np.all((b >= 0.5) & (b < 1.5)) and np.allclose(d, 1.0 / np.sqrt(b), rtol=0, atol=0)
    L = api.gen_laplacian([6, 5, 4])
    b, d = api.mass_scaling(L.n, 3)
    S = api.scale_sym_host(L, d)
    ref = sp.diags(d) @ _sp(L) @ sp.diags(d)
    assert abs(_sp(S) - ref).max() <= 1e-15
    g = golden("cfg5p")
    L24 = api.gen_laplacian([24, 24, 24])
    _, d24 = api.mass_scaling(L24.n, 5)
    assert np.array_equal(d24, g["d"])
    assert np.array_equal(api.scale_sym_host(L24, d24).vals, g["vals_scaled"])
