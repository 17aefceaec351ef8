"""GPU parity of the core kernels and drivers against the oracle (C restatement) and, where its
prebuilt library is present, the reference itself (oracle/_ref)."""
import numpy as np
import pytest

from oracle import clib

pytestmark = pytest.mark.gpu


def _api():
    from paper_1802_05215_b200 import api
    return api


CFG1_BOUNDS = (0.0010977890680629611, 7.99911827091601)  # reference lan_tr_bounds, cfg1 (seed 0)


def test_spmv_bitwise(gpu_ctx):
    api = _api()
    a = api.gen_laplacian([100, 100])
    x = clib.rng_vectors(5, "normal", a.n)[0]
    y = a.matvec(x)
    ref = clib.matvec(a.row_ptr, a.col_idx, a.vals, x)
    assert np.array_equal(y, ref)


def test_device_laplacian_generator_bitwise(gpu_ctx):
    api = _api()
    for dims in ([7], [5, 4], [4, 3, 5], [64, 64, 64]):
        d = api.DeviceCsr.laplacian(dims).download()
        rp, ci, v = clib.laplacian(dims)
        assert np.array_equal(d.row_ptr, rp) and np.array_equal(d.col_idx, ci)
        assert np.array_equal(d.vals, v)


@pytest.mark.parametrize("dims,slice_,damping", [
    ([100, 100], (0.4, 1.0443178519), "jackson"),
    ([100, 100], (1.0443178519, 1.6), "jackson"),
    ([64, 64, 64], (0.6, 0.7), "sigma"),
])
def test_apply_pol_bitwise(gpu_ctx, dims, slice_, damping):
    api = _api()
    a = api.gen_laplacian(dims)
    lo, hi = CFG1_BOUNDS if len(dims) == 2 else (0.0, 12.0)
    f = api.find_pol(slice_[0], slice_[1], api.SpectralBounds(lo, hi), api.PolyOpts(damping=damping))
    x = clib.rng_vectors(11, "normal", a.n)[0]
    cnt = api.Counters()
    out = api.apply_pol(f, a, x, cnt)
    ref = clib.apply_pol(a.row_ptr, a.col_idx, a.vals, f.mu, f.c, f.d, x)
    assert cnt.n_A_matvec == f.k
    assert np.array_equal(out, ref), np.max(np.abs(out - ref))


def test_apply_pol_block_bitwise(gpu_ctx):
    """Block application (multi-vector fused kernel, 8 columns per launch; used by cheb_si):
    every column bitwise the reference's apply_pol (9 columns: a full group of 8 plus a tail)."""
    api = _api()
    a = api.gen_laplacian([40, 40])
    f = api.find_pol(0.5, 0.6, api.SpectralBounds(0.0, 8.0))
    X = clib.rng_vectors(5, "normal", a.n, 9)
    cnt = api.Counters()
    out = api.apply_pol(f, a, X, cnt)
    assert cnt.n_A_matvec == 9 * f.k
    for j in range(9):
        ref = clib.apply_pol(a.row_ptr, a.col_idx, a.vals, f.mu, f.c, f.d, X[j])
        assert np.array_equal(out[j], ref), (j, np.max(np.abs(out[j] - ref)))


def test_kpm_moments_match_oracle(gpu_ctx):
    api = _api()
    a = api.gen_laplacian([100, 100])
    lo, hi = CFG1_BOUNDS
    for probes in ("rademacher", "gaussian"):
        z = api.kpm_moments(a, api.SpectralBounds(lo, hi), 80, 20, seed=0, probes=probes)
        zr = clib.kpm_moments(a.row_ptr, a.col_idx, a.vals, lo, hi, 80, 20, 0,
                              kind="normal" if probes == "gaussian" else "rademacher")
        zn, zrn = z / (20 * a.n), zr / (20 * a.n)
        tol = 1e-12 * np.maximum(np.abs(zrn), abs(zrn[0]))
        assert np.all(np.abs(zn - zrn) <= tol), np.max(np.abs(zn - zrn) / np.abs(zrn[0]))


def test_lan_tr_bounds_encloses_spectrum(gpu_ctx):
    api = _api()
    a = api.gen_laplacian([100, 100])
    b = api.lan_tr_bounds(a, 1e-4, 60, 40, seed=0)
    ev = api.laplacian_analytic_eigs([100, 100])
    assert b.lmin <= ev[0] + 1e-3 and b.lmax >= ev[-1] - 1e-6
    spread = CFG1_BOUNDS[1] - CFG1_BOUNDS[0]
    assert abs(b.lmin - CFG1_BOUNDS[0]) <= 1e-4 * spread and abs(b.lmax - CFG1_BOUNDS[1]) <= 1e-4 * spread


def test_diagonal_slice(gpu_ctx):
    api = _api()
    a = api.CsrMatrix.diag([0.1, 0.5, 0.9])
    f = api.find_pol(0.4, 0.6, api.SpectralBounds(0.05, 0.95))
    for drv in (api.cheb_lan_nr, api.cheb_lan_tr):
        r = drv(a, None, f, 0.4, 0.6)
        assert len(r.eigenvalues) == 1
        assert abs(r.eigenvalues[0] - 0.5) <= 1e-12
        assert r.residuals[0] <= 1e-12
        assert abs(abs(r.vectors[1, 0]) - 1.0) <= 1e-10
        assert r.counters.t_total > 0 and not r.hit_max_its


@pytest.mark.parametrize("driver", ["nr", "tr"])
def test_laplacian_60x60_window(gpu_ctx, driver):
    api = _api()
    a = api.gen_laplacian([60, 60])
    allv = api.laplacian_analytic_eigs([60, 60])
    oracle = allv[(allv >= 0.4) & (allv <= 0.6)]
    assert oracle.size == 62
    f = api.find_pol(0.4, 0.6, api.SpectralBounds(allv[0] - 1e-8, allv[-1] + 1e-8))
    cfg = api.SolverConfig(est_count=62)
    drv = api.cheb_lan_nr if driver == "nr" else api.cheb_lan_tr
    r = drv(a, None, f, 0.4, 0.6, cfg)
    assert r.eigenvalues.size == 62
    assert np.max(np.abs(r.eigenvalues - oracle)) <= 1e-8
    assert np.all(r.residuals <= cfg.res_tol)
    G = r.vectors.T @ r.vectors
    assert np.max(np.abs(G - np.eye(62))) <= 1e-8
    assert r.counters.n_A_matvec >= f.k * r.niter
    for i in range(0, 62, 7):
        lam, res = api.rayleigh_and_residual(a, None, r.vectors[:, i])
        assert abs(lam - r.eigenvalues[i]) <= 1e-10
        assert abs(res - r.residuals[i]) <= 1e-10


def _irregular(n, seed, maxdeg):
    """Symmetric matrix with 0..maxdeg entries per row (some empty rows)."""
    rng = np.random.default_rng(seed)
    deg = np.zeros(n, int)
    rows, cols, vals = [], [], []
    seen = set()
    for i in range(n):
        if i % 11 == 5:
            continue  # empty row (and column)
        rows.append(i); cols.append(i); vals.append(2.0 + rng.random())
        deg[i] += 1
    for i in range(n):
        for _ in range(int(rng.integers(0, maxdeg // 2 + 1))):
            j = int(rng.integers(0, n))
            if j == i or i % 11 == 5 or j % 11 == 5 or deg[i] >= maxdeg or deg[j] >= maxdeg:
                continue
            if (min(i, j), max(i, j)) in seen:
                continue
            seen.add((min(i, j), max(i, j)))
            v = float(rng.standard_normal()) * 0.3
            rows += [i, j]; cols += [j, i]; vals += [v, v]
            deg[i] += 1; deg[j] += 1
    return _api().CsrMatrix.from_triplets(n, rows, cols, vals)


@pytest.mark.parametrize("case", ["lap20", "lap2d", "irr8", "irr24", "banded"])
def test_kpm_block_kernels(gpu_ctx, case):
    """Both block-KPM kernels against the oracle: the padded-row kernel (rows <= 8: stencils and
    an irregular matrix with 0..8 entries per row, empty rows included) and the CSR-stream
    kernel (longer rows: an irregular matrix with up to 24 per row, a cfg4-recipe random banded
    matrix), with full (16), ragged (21 = 16 + 5) and narrow (6) probe blocks."""
    api = _api()
    if case == "lap20":
        a, (lo, hi) = api.gen_laplacian([20, 20, 20]), (0.0, 12.0)
    elif case == "lap2d":
        a, (lo, hi) = api.gen_laplacian([37, 23]), (0.0, 8.0)
    elif case == "irr8":
        a, (lo, hi) = _irregular(3001, 7, 8), (-4.0, 6.0)
    elif case == "irr24":
        a, (lo, hi) = _irregular(2003, 9, 24), (-6.0, 8.0)
    else:
        a = api.gen_random_sparse(4000, 11)
        rows = np.repeat(np.arange(a.n), np.diff(a.row_ptr))
        diag = np.zeros(a.n)
        diag[rows[a.col_idx == rows]] = a.vals[a.col_idx == rows]
        rad = np.bincount(rows, weights=np.abs(a.vals), minlength=a.n) - np.abs(diag)
        lo, hi = float(np.min(diag - rad)), float(np.max(diag + rad))  # Gershgorin
    mx = int(np.max(np.diff(a.row_ptr)))
    assert (mx <= 8) == (case in ("lap20", "lap2d", "irr8")), mx
    for nvec in (16, 21, 6):
        z = api.kpm_moments(a, api.SpectralBounds(lo, hi), 40, nvec, seed=3)
        zr = clib.kpm_moments(a.row_ptr, a.col_idx, a.vals, lo, hi, 40, nvec, 3)
        zn, zrn = z / (nvec * a.n), zr / (nvec * a.n)
        err = np.abs(zn - zrn) / np.maximum(np.abs(zrn), abs(zrn[0]))
        assert err.max() <= 1e-12, (case, nvec, err.max())


def test_kpm_rademacher_threaded_bits_match_oracle(gpu_ctx):
    """Large enough (n b >= 2^21) that the host draws each probe's sign bits on its own thread
    from a jumped-ahead stream: moments still match the oracle's serial draws; a ragged second
    block (16 + 3) and a later first probe (rank offset) too."""
    api = _api()
    a = api.gen_laplacian([64, 64, 64])
    lo, hi = 0.0, 12.0
    z = api.kpm_moments(a, api.SpectralBounds(lo, hi), 12, 19, seed=5)
    zr = clib.kpm_moments(a.row_ptr, a.col_idx, a.vals, lo, hi, 12, 19, 5)
    tol = 1e-12 * np.maximum(np.abs(zr), abs(zr[0]))
    assert np.all(np.abs(z - zr) <= tol), np.max(np.abs(z - zr) / abs(zr[0]))
    z2 = api.kpm_moments(a, api.SpectralBounds(lo, hi), 12, 19, seed=5, first=3, count=16)
    zr2 = clib.kpm_moments(a.row_ptr, a.col_idx, a.vals, lo, hi, 12, 19, 5, first=3, count=16)
    tol2 = 1e-12 * np.maximum(np.abs(zr2), abs(zr2[0]))
    assert np.all(np.abs(z2 - zr2) <= tol2)


@pytest.mark.parametrize("n,k,repass", [(4097, 1, True), (5000, 300, True), (5000, 300, False),
                                        (20001, 1300, True), (3000, 2900, True), (9000, 6000, True)])
def test_paired_cgs2_row_major_vs_numpy(gpu_ctx, n, k, repass):
    """The product CGS2 (row-major basis, T1 + fused N1/T2 + N2, rowgs.cu) against a numpy
    restatement of paired_cgs2 (orth.hpp:63-80), with and without the DGKS re-pass, across the
    register-column templates (k = 1 .. 6000)."""
    api = _api()
    rng = np.random.default_rng(n + k)
    Q, _ = np.linalg.qr(rng.standard_normal((n, k)))
    t = rng.standard_normal(n)
    if repass:
        t = t + Q @ rng.standard_normal(k) * 50.0
    h = np.zeros(k)
    before = np.linalg.norm(t)
    c1 = Q.T @ t
    t1 = t - Q @ c1
    h += c1
    if not np.linalg.norm(t1) > 0.70710678118654752 * before:
        c2 = Q.T @ t1
        t1 = t1 - Q @ c2
        h += c2
        assert repass
    else:
        assert not repass
    tg, hg = api.paired_cgs2(t, np.ascontiguousarray(Q.T), np.zeros(k))
    assert np.max(np.abs(tg - t1)) <= 1e-12 * before
    assert np.max(np.abs(hg - h)) <= 1e-12 * before


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,k,rowmajor", [(1000, 37, 129, True), (517, 5, 33, True),
                                            (300, 70, 64, False), (129, 130, 7, False),
                                            (40, 40, 20011, True), (64, 3, 1, True)])
def test_ritz_gemm_matches_numpy(gpu_ctx, m, n, k, rowmajor):
    """The DMMA Rayleigh-Ritz contraction (ritz_gemm.cu) against numpy: ragged tiles in every
    dimension, odd K (8-byte tail copies), both A layouts, and the split-K Gram shape."""
    from paper_1802_05215_b200 import api
    rng = np.random.default_rng(5)
    a = rng.standard_normal((m, k))
    b = rng.standard_normal((k, n))
    out = api.mult_cols(a, b, a_rowmajor=rowmajor, ctx=gpu_ctx)
    ref = a @ b
    scale = np.abs(a) @ np.abs(b)
    assert np.all(np.abs(out - ref) <= 4e-16 * k * scale + 1e-300)


@pytest.mark.parametrize("case,degree", [("lap3d", 0), ("lap2d", 0), ("irr8", 0), ("irr24", 0),
                                         ("banded", 0), ("lap2d", 1), ("lap2d", 2), ("tiny", 0)])
def test_resident_filter_bitwise(gpu_ctx, case, degree):
    """The resident filter (resident.cu: every degree in one cooperative launch, matrix tiles in
    shared memory, neighbour hand-off through L2) against the oracle's apply_pol and against the
    per-degree kernels: bit-identical on stencils (neighbour tiles only), irregular matrices with
    empty rows and a random banded matrix (every tile a neighbour), a one-tile matrix, and the
    degree-1 / degree-2 edge cases."""
    api = _api()
    if case == "lap3d":
        a, (lo, hi) = api.gen_laplacian([30, 28, 26]), (0.0, 12.0)
    elif case == "lap2d":
        a, (lo, hi) = api.gen_laplacian([130, 90]), (0.0, 8.0)
    elif case == "tiny":
        a, (lo, hi) = api.gen_laplacian([9, 7]), (0.0, 8.0)
    elif case == "irr8":
        a, (lo, hi) = _irregular(30011, 7, 8), (-4.0, 6.0)
    elif case == "irr24":
        a, (lo, hi) = _irregular(20001, 8, 24), (-6.0, 9.0)
    else:
        a, (lo, hi) = api.gen_random_sparse(40000, 3), (-12.0, 18.0)
    f = api.find_pol(lo + 0.31 * (hi - lo), lo + 0.36 * (hi - lo), api.SpectralBounds(lo, hi))
    if degree:  # truncate the series: degree 1 and 2 take the kernel's short paths
        f = api.PolynomialFilter(k=degree, gamma=f.gamma, mu=f.mu[:degree + 1].copy(), c=f.c, d=f.d,
                                 tau=f.tau, ta=f.ta, tb=f.tb, bar=f.bar, damping=f.damping,
                                 cap_reached=f.cap_reached)
    x = clib.rng_vectors(3, "normal", a.n)[0]
    assert api.resident_tiles(a) > 0
    out = api.apply_pol(f, a, x)
    ref = clib.apply_pol(a.row_ptr, a.col_idx, a.vals, f.mu, f.c, f.d, x)
    assert np.array_equal(out, ref), np.max(np.abs(out - ref))
    api.set_resident_filter(False)
    try:
        assert api.resident_tiles(a) == 0
        out2 = api.apply_pol(f, a, x)
    finally:
        api.set_resident_filter(True)
    assert np.array_equal(out, out2)
    # a second application on the same matrix (the tile counters keep advancing)
    assert np.array_equal(api.apply_pol(f, a, x), ref)


def test_resident_filter_in_the_slice_solve(gpu_ctx):
    """cheb_lan_tr with the resident filter on and off: identical eigenvalues, residuals and
    iteration counts (the filter output is bit-identical, so the whole recurrence is)."""
    api = _api()
    a = api.gen_laplacian([40, 40])
    f = api.find_pol(0.5, 0.9, api.SpectralBounds(0.0, 8.0))
    cfg = api.SolverConfig(est_count=60)
    r1 = api.cheb_lan_tr(a, None, f, 0.5, 0.9, cfg)
    api.set_resident_filter(False)
    try:
        r0 = api.cheb_lan_tr(a, None, f, 0.5, 0.9, cfg)
    finally:
        api.set_resident_filter(True)
    assert r1.niter == r0.niter and np.array_equal(r1.eigenvalues, r0.eigenvalues)
    assert np.array_equal(r1.residuals, r0.residuals)


@pytest.mark.parametrize("case,ncols", [("irr8", 11), ("lap3d", 8), ("lap2d", 3), ("banded", 5)])
def test_block_filter_bitwise(gpu_ctx, case, ncols):
    """Block apply_pol: the row-major 8-vector block kernel on padded-row matrices (stencils, an
    irregular matrix with 0..8 entries per row and empty rows; full, split and narrow groups) and
    the CSR multi-vector kernel on longer rows -- every column bitwise the oracle's apply_pol."""
    api = _api()
    if case == "lap3d":
        a, (lo, hi) = api.gen_laplacian([17, 13, 11]), (0.0, 12.0)
    elif case == "lap2d":
        a, (lo, hi) = api.gen_laplacian([33, 29]), (0.0, 8.0)
    elif case == "irr8":
        a, (lo, hi) = _irregular(3001, 7, 8), (-4.0, 6.0)
    else:
        a, (lo, hi) = api.gen_random_sparse(3000, 3), (-12.0, 18.0)
    f = api.find_pol(lo + 0.31 * (hi - lo), lo + 0.40 * (hi - lo), api.SpectralBounds(lo, hi))
    X = clib.rng_vectors(9, "normal", a.n, ncols)
    out = api.apply_pol(f, a, X)
    for j in range(ncols):
        ref = clib.apply_pol(a.row_ptr, a.col_idx, a.vals, f.mu, f.c, f.d, X[j])
        assert np.array_equal(out[j], ref), (j, np.max(np.abs(out[j] - ref)))
