"""Pin the oracle (oracle/sliceeig_oracle.c, the C restatement used as the GPU checker) to the
golden fixtures generated from the unmodified reference (tests/golden/make_golden.py).  CPU only.
Integer/index work and every bitwise-reproducible float path must match exactly."""
import numpy as np
import pytest

from oracle import clib

INTS = [(-0.4, 0.4), (0.2, 0.4), (0.0, 0.3), (-0.5, 0.5), (-0.9, -0.85), (0.61, 0.62)]


@pytest.fixture(scope="module")
def g(golden):
    return golden("kats")


def test_rng_streams(g):
    assert np.array_equal(clib.rng_vectors(7, "normal", 257, 3), g["rng_normal_7"])
    assert np.array_equal(clib.rng_vectors(7, "rademacher", 257, 3), g["rng_rademacher_7"])


@pytest.mark.parametrize("dims", [[7], [5, 4], [4, 3, 5], [20, 20]])
def test_laplacian_csr_and_spectrum(g, dims):
    tag = "x".join(map(str, dims))
    rp, ci, v = clib.laplacian(dims)
    assert np.array_equal(rp, g[f"lap_{tag}_rp"])
    assert np.array_equal(ci, g[f"lap_{tag}_ci"])
    assert np.array_equal(v, g[f"lap_{tag}_v"])
    assert np.array_equal(clib.laplacian_eigs(dims), g[f"lapeig_{tag}"])


def test_laplacian_nnz_kats():
    # test_matrix_core.cpp:45-69 anchors: 343^2 -> nnz 586,873 ; 49^3 -> 809,137
    assert clib.lib().or_laplacian_nnz(2, np.array([343, 343], np.int32)) == 586873
    assert clib.lib().or_laplacian_nnz(3, np.array([49, 49, 49], np.int32)) == 809137


@pytest.mark.parametrize("damp", ["none", "sigma", "jackson"])
def test_damping_and_coeffs(g, damp):
    for k in (1, 2, 8, 40):
        assert np.array_equal(clib.damping(k, damp), g[f"damp_{damp}_{k}"])
    assert np.array_equal(clib.normalized_coeffs(16, 0.3, damp), g[f"ncoef_{damp}_16"])
    assert np.array_equal(clib.normalized_coeffs(5, -0.7, damp), g[f"ncoef_{damp}_5"])


@pytest.mark.parametrize("damp", ["none", "sigma", "jackson"])
@pytest.mark.parametrize("q", range(len(INTS)))
def test_find_pol(g, damp, q):
    a, b = INTS[q]
    f = clib.find_pol(a, b, -1.0, 1.0, damping=damp)
    assert f["k"] == int(g[f"findpol_{damp}_{q}_k"])
    assert np.array_equal(f["mu"], g[f"findpol_{damp}_{q}_mu"])
    sc = g[f"findpol_{damp}_{q}_scalars"]
    assert [f["gamma"], f["ta"], f["tb"], f["bar"], f["c"], f["d"], float(f["cap_reached"])] == list(sc)


def test_find_pol_boundary_slices(g):
    for q, (a, b) in enumerate([(0.0, 0.5), (7.5, 8.0), (3.0, 4.0), (0.4, 1.0443178519)]):
        f = clib.find_pol(a, b, 0.0, 8.0)
        assert f["k"] == int(g[f"findpol_b8_{q}_k"])
        assert np.array_equal(f["mu"], g[f"findpol_b8_{q}_mu"])
    assert clib.balance_center(16, 0.2, 0.4, "sigma") == float(g["balance_16_02_04_sigma"])


def test_apply_pol_and_matvec(g):
    rp, ci, v = clib.laplacian([20, 20])
    x = g["ap_x"]
    assert np.array_equal(clib.matvec(rp, ci, v, x), g["ap_Ax"])
    for damp in ("sigma", "jackson"):
        c, d = g[f"ap_{damp}_cd"]
        y = clib.apply_pol(rp, ci, v, g[f"ap_{damp}_mu"], c, d, x)
        assert np.array_equal(y, g[f"ap_{damp}_y"])


def test_kpm_moments_curve_slicing(g):
    rp, ci, v = clib.laplacian([25, 25])
    for kind in ("rademacher", "normal"):
        z = clib.kpm_moments(rp, ci, v, 0.0, 8.0, 60, 8, 777, kind)
        assert np.array_equal(z, g[f"kpm25_zeta_{kind}"])
    z = g["kpm25_zeta_rademacher"] / (8.0 * 625)
    x, y, nev = clib.kpm_curve(z, 625, 0.0, 8.0, 300)
    assert np.array_equal(x, g["kpm25_x"]) and np.array_equal(y, g["kpm25_y"])
    assert nev == float(g["kpm25_nev"])
    bp, est = clib.slice_spectrum(x, y, 625, 0.0, 8.0, 4)
    assert np.array_equal(bp, g["kpm25_bp4"]) and np.array_equal(est, g["kpm25_est4"])
    assert clib.dos_count(x, y, 625, 1.0, 3.0) == float(g["kpm25_count_1_3"])


def test_paired_cgs2(g):
    t, h, passes = clib.paired_cgs2(g["cgs_W"], g["cgs_t"])
    assert np.array_equal(t, g["cgs_t_out"]) and np.array_equal(h, g["cgs_h"])


def test_cfg1_pipeline_stages(golden):
    """BASELINE configs[0]: moments, curve, breakpoints and Jackson degrees from the reference."""
    c = golden("cfg1")
    rp, ci, v = clib.laplacian([100, 100])
    lo, hi = c["bounds"]
    z = clib.kpm_moments(rp, ci, v, lo, hi, 80, 20, 0, "rademacher")
    assert np.array_equal(z, c["zeta"])
    x, y, nev = clib.kpm_curve(z / (20.0 * 10000), 10000, lo, hi, 300)
    assert np.array_equal(y, c["y"]) and nev == float(c["nev"])
    bp, est = clib.slice_spectrum(x, y, 10000, 0.4, 1.6, 2)
    assert np.array_equal(bp, c["bp"]) and np.array_equal(est, c["est"])
    degs = [clib.find_pol(bp[i], bp[i + 1], lo, hi, damping="jackson")["k"] for i in range(2)]
    assert degs == list(c["degrees"])
    # the reference's own solve found exactly the analytic eigenvalues of each slice
    ev = clib.laplacian_eigs([100, 100])
    delta = 1e-10 * (c["solve_bounds"][1] - c["solve_bounds"][0])
    b1 = c["solve_bp"][1]
    truths = [ev[(ev >= 0.4) & (ev <= b1 + delta)], ev[(ev > b1 + delta) & (ev <= 1.6)]]
    for i in range(2):
        vals = c[f"slice{i}_vals"]
        truth = truths[i]
        assert vals.size == truth.size
        assert np.max(np.abs(vals - truth)) <= 1e-12


def test_cfg2_kpm_gaussian_and_slices(golden):
    """BASELINE configs[1]: 64^3, 100 moments x 40 Gaussian probes (seed 1234)."""
    c = golden("cfg2")
    rp, ci, v = clib.laplacian([64, 64, 64])
    lo, hi = c["bounds"]
    z = clib.kpm_moments(rp, ci, v, lo, hi, 100, 40, 1234, "normal")
    assert np.array_equal(z, c["zeta"])
    x, y, nev = clib.kpm_curve(z / (40.0 * 262144), 262144, lo, hi, 300)
    assert np.array_equal(y, c["y"])
    bp, est = clib.slice_spectrum(x, y, 262144, 0.6, 1.2, 8)
    assert np.array_equal(bp, c["bp"]) and np.array_equal(est, c["est"])
    degs = [clib.find_pol(bp[i], bp[i + 1], lo, hi)["k"] for i in range(8)]
    assert degs == list(c["degrees"]) == [67, 115, 121, 126, 260, 133, 138, 367]


@pytest.mark.skipif(not __import__("oracle.reflib", fromlist=["available"]).available(),
                    reason="oracle/_ref (the reference build) not present")
def test_pencil_golden_reproduced_by_reference(golden):
    """tests/golden/pencil.npz is the reference's own B-weighted cheb_lan_tr/nr (b != nullptr) on
    (16^3 Laplacian, diag B): rerunning it reproduces the stored eigenvalues bitwise."""
    from oracle import reflib
    from paper_1802_05215_b200 import api
    g = golden("pencil")
    L = api.gen_laplacian([16, 16, 16])
    assert np.array_equal(api.mass_scaling(L.n, 7)[0], g["b"])
    r = reflib.cheb_lan_pencil(L.row_ptr, L.col_idx, L.vals, g["b"], "tr", *g["window"], *g["bounds"],
                               est_count=80, seed=7)
    assert np.array_equal(r["eigenvalues"], g["tr_vals"])
