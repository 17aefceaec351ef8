"""Host-side logic of the PRODUCT library (libsliceeig_cuda.so host-only C-ABI entry points, no GPU
needed): filters, DOS curve, slicing, small eigensolvers, matrix generators, error types --
checked against the golden fixtures of the unmodified reference.  CPU only."""
import ctypes as C
import re

import numpy as np
import pytest

from paper_1802_05215_b200 import _lib, api

INTS = [(-0.4, 0.4), (0.2, 0.4), (0.0, 0.3), (-0.5, 0.5), (-0.9, -0.85), (0.61, 0.62)]


@pytest.fixture(scope="module")
def g(golden):
    return golden("kats")


def test_library_exports_every_declared_symbol():
    """The C-ABI library loads and exports exactly what include/sliceeig_cuda.h declares."""
    import os
    hdr = open(os.path.join(os.path.dirname(__file__), "..", "include", "sliceeig_cuda.h")).read()
    declared = set(re.findall(r"SE_API\s+(?:int|const char\*)\s+(se_\w+)\s*\(", hdr))
    L = _lib.lib()
    assert declared, "no declarations parsed"
    missing = [s for s in declared if not hasattr(L, s)]
    assert not missing, missing
    assert set(_lib.SIGNATURES) | {"se_last_error", "se_version"} == declared
    assert b"sm_100a" in L.se_version()


@pytest.mark.parametrize("dims", [[7], [5, 4], [4, 3, 5], [20, 20]])
def test_gen_laplacian_host_bitwise(g, dims):
    tag = "x".join(map(str, dims))
    a = api.gen_laplacian(dims)
    assert np.array_equal(a.row_ptr, g[f"lap_{tag}_rp"])
    assert np.array_equal(a.col_idx, g[f"lap_{tag}_ci"])
    assert np.array_equal(a.vals, g[f"lap_{tag}_v"])
    assert np.array_equal(api.laplacian_analytic_eigs(dims), g[f"lapeig_{tag}"])


def test_laplacian_counts_kats():
    # test_matrix_core.cpp:45-69: 343 eigenvalues of 49^3 in [0.40, 0.570]; 1,971 in [0, 1]
    e = api.laplacian_analytic_eigs([49, 49, 49])
    assert api.count_in_interval(e, 0.40, 0.570) == 343
    assert api.count_in_interval(e, 0.0, 1.0) == 1971
    with pytest.raises(ValueError):
        api.gen_laplacian([])
    with pytest.raises(ValueError):
        api.gen_laplacian([0, 3])


@pytest.mark.parametrize("damp", ["none", "sigma", "jackson"])
def test_filter_coefficients(g, damp):
    for k in (1, 2, 8, 40):
        assert np.array_equal(api.damping_multipliers(k, damp), g[f"damp_{damp}_{k}"])
    assert np.array_equal(api.normalized_filter_coeffs(16, 0.3, damp), g[f"ncoef_{damp}_16"])
    for q, (a, b) in enumerate(INTS):
        f = api.find_pol(a, b, api.SpectralBounds(-1.0, 1.0), api.PolyOpts(damping=damp))
        assert f.k == int(g[f"findpol_{damp}_{q}_k"])
        assert np.array_equal(f.mu, g[f"findpol_{damp}_{q}_mu"])
        assert [f.gamma, f.ta, f.tb, f.bar, f.c, f.d, float(f.cap_reached)] == \
            list(g[f"findpol_{damp}_{q}_scalars"])


def test_filter_kats_and_errors():
    # test_filters.cpp:24-68: mu(0,2) = (1/2, 0, -1); sigma_1(k=1) = 2/pi; rho(t) = 1 - 4t^2/3
    mu = api.chebyshev_coeffs(0.0, 2)
    assert mu[0] == 0.5 and abs(mu[1]) <= 1e-16 and abs(mu[2] + 1.0) <= 1e-15
    assert abs(api.damping_multipliers(1, "sigma")[1] - 2.0 / np.pi) <= 1e-14 * 2.0 / np.pi
    f = api.PolynomialFilter(k=2, mu=api.normalized_filter_coeffs(2, 0.0, "none"))
    for t in (-0.9, -0.3, 0.2, 0.7):
        assert abs(api.eval_pol(f, t) - (1.0 - 4.0 / 3.0 * t * t)) <= 1e-14
    with pytest.raises(ValueError):
        api.eval_pol(f, 1.2)
    with pytest.raises(ValueError):
        api.chebyshev_coeffs(1.0, 3)
    b = api.SpectralBounds(0.0, 8.0)
    with pytest.raises(ValueError):
        api.find_pol(0.5, 0.5, b)
    with pytest.raises(ValueError):
        api.find_pol(9.0, 10.0, b)
    # minimality: one degree lower cannot satisfy tau (test_filters.cpp:118-122)
    fp = api.find_pol(0.2, 0.4, api.SpectralBounds(-1.0, 1.0))
    capped = api.find_pol(0.2, 0.4, api.SpectralBounds(-1.0, 1.0), api.PolyOpts(max_deg=fp.k - 1))
    assert capped.cap_reached and not fp.cap_reached


def test_kpm_curve_and_slicer(g):
    z = g["kpm25_zeta_rademacher"] / (8.0 * 625)
    c = api.kpm_curve(z, 625, api.SpectralBounds(0.0, 8.0), 300)
    assert np.array_equal(c.xdos, g["kpm25_x"]) and np.array_equal(c.ydos, g["kpm25_y"])
    assert c.nev_est == float(g["kpm25_nev"])
    s = api.slice_spectrum(c, 0.0, 8.0, 4)
    assert np.array_equal(s.breakpoints, g["kpm25_bp4"])
    assert np.array_equal(s.est_counts, g["kpm25_est4"])
    assert api.dos_count(c, 1.0, 3.0) == float(g["kpm25_count_1_3"])


def test_slicer_kats_and_errors():
    # test_dos.cpp:254-283 / 350-361
    x = np.array([1.0 * i / 100 for i in range(101)])
    c = api.DosCurve(x, np.ones(101), 100.0, 100)
    s = api.slice_spectrum(c, 0.0, 1.0, 2)
    assert s.breakpoints[0] == 0.0 and s.breakpoints[-1] == 1.0
    assert abs(s.breakpoints[1] - 0.5) <= 0.0101
    s1 = api.slice_spectrum(api.DosCurve(np.linspace(0, 2, 50), np.full(50, 0.5), 0, 10), 0.25, 1.75, 1)
    assert list(s1.breakpoints) == [0.25, 1.75]
    c5 = api.DosCurve(np.array([0.0, 0.25, 0.5, 0.75, 1.0]), np.ones(5), 5.0, 5)
    for bad in ((0.0, 1.0, 0), (0.5, 0.5, 1), (-0.5, 1.0, 2), (0.0, 1.0, 5)):
        with pytest.raises(ValueError):
            api.slice_spectrum(c5, *bad)
    api.slice_spectrum(c5, 0.0, 1.0, 4)
    with pytest.raises(ValueError):
        api.dos_count(c5, -1.0, 0.5)
    with pytest.raises(RuntimeError):  # dos_finalize: vanishing density (dos.hpp:57)
        api.kpm_curve(np.zeros(5), 10, api.SpectralBounds(0.0, 1.0), 20)


def test_small_eigensolvers(g):
    vals, vecs = api.sym_tridiag_eig(g["trid_a"], g["trid_b"], True)
    assert np.max(np.abs(vals - g["trid_vals"])) <= 1e-13
    ref = g["trid_vecs"]
    assert np.max(np.abs(np.abs(vecs) - np.abs(ref))) <= 1e-10
    dv, dvec = api.dense_sym_eig(g["dense_S"], True)
    assert np.max(np.abs(dv - g["dense_vals"])) <= 1e-12
    S = g["dense_S"]
    assert np.max(np.abs(S @ dvec - dvec * dv)) <= 1e-11
    with pytest.raises(ValueError):
        api.dense_sym_eig(np.eye(6), False, size_guard=5)


@pytest.mark.parametrize("l", [0, 1, 2, 7, 40])
def test_arrow_to_tridiag_preserves_spectrum(l):
    rng = np.random.default_rng(l)
    th = rng.standard_normal(l)
    s = rng.standard_normal(l)
    al = 0.3
    d = np.empty(l + 1)
    o = np.empty(max(l, 1))
    _lib.call("se_arrow_tridiag", l, th.ctypes.data_as(C.POINTER(C.c_double)),
              s.ctypes.data_as(C.POINTER(C.c_double)), al, d.ctypes.data_as(C.POINTER(C.c_double)),
              o.ctypes.data_as(C.POINTER(C.c_double)))
    H = np.zeros((l + 1, l + 1))
    H[np.arange(l), np.arange(l)] = th
    H[:l, l] = H[l, :l] = s
    H[l, l] = al
    T = np.diag(d) + np.diag(o[:l], 1) + np.diag(o[:l], -1)
    assert np.allclose(np.linalg.eigvalsh(H), np.linalg.eigvalsh(T), atol=1e-12)


def test_csr_from_triplets_semantics():
    # csr.hpp:29-58: sorted, duplicates summed, explicit zeros dropped, range checked
    a = api.CsrMatrix.from_triplets(3, [2, 0, 0, 1, 1], [0, 2, 2, 1, 2], [1.0, 2.0, 3.0, 0.0, 4.0])
    assert list(a.row_ptr) == [0, 1, 2, 3]
    assert list(a.col_idx) == [2, 2, 0] and list(a.vals) == [5.0, 4.0, 1.0]
    with pytest.raises(IndexError):
        api.CsrMatrix.from_triplets(2, [0], [2], [1.0])
    with pytest.raises(ValueError):
        api.CsrMatrix.from_triplets(-1, [], [], [])


@pytest.mark.parametrize("q", [0, 1, 2, 3])
def test_ls_pol_approx_matches_reference(golden, q):
    """ls_pol_approx (cheb_approx.hpp:40-88, host): degree and coefficients of the reference's
    fits (tests/golden/pencil_general.npz)."""
    g = golden("pencil_general")
    fun, a, b, tol, ach = g[f"lsq{q}_meta"]
    co, got = api.ls_pol_approx("inverse_sqrt" if fun else "inverse", api.SpectralBounds(a, b), tol)
    ref = g[f"lsq{q}_coeff"]
    assert co.size == ref.size
    assert np.max(np.abs(co - ref)) <= 1e-14 * np.max(np.abs(ref))
    assert got <= tol and abs(got - ach) <= 1e-3 * tol
    with pytest.raises(ValueError):
        api.ls_pol_approx("inverse", api.SpectralBounds(-0.5, 2.0), 1e-8)
    with pytest.raises(RuntimeError):
        api.ls_pol_approx("inverse", api.SpectralBounds(1e-4, 1.0), 1e-14, 6)
