"""General SPD-B pencils (A, B) on the device: S = P A P with P ~ B^-1/2 a
Chebyshev series in B (ls_pol_approx / apply_cheb, cheb_approx.hpp), against the reference's own
Cholesky-backed B-weighted drivers (eigensolvers.hpp:640-732) on a non-diagonal SPD B: the 2-D
Laplacian with B = M1 (x) M1 (linear-element mass), whose spectrum is known in closed form
(tests/golden/pencil_general.npz, made by oracle/_ref)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _api():
    from paper_1802_05215_b200 import api
    return api


def _problem(golden):
    api = _api()
    g = golden("pencil_general")
    a = api.gen_laplacian([30, 30])
    b = api.CsrMatrix(a.n, g["brp"], g["bci"], g["bv"])
    return api, g, a, b


def _dense(m):
    d = np.zeros((m.n, m.n))
    for i in range(m.n):
        for p in range(m.row_ptr[i], m.row_ptr[i + 1]):
            d[i, m.col_idx[p]] = m.vals[p]
    return d


@pytest.mark.parametrize("q", [0, 1, 2, 3])
def test_apply_cheb_matches_reference(gpu_ctx, golden, q):
    """apply_cheb (cheb_approx.hpp:91-112) on the device: the reference's y = p(B) x."""
    api, g, a, b = _problem(golden)
    fun, lo, hi, tol, _ = g[f"lsq{q}_meta"]
    x = np.cos(np.arange(a.n) * 0.37)
    y = api.apply_cheb(g[f"lsq{q}_coeff"], api.SpectralBounds(lo, hi), b, x)
    ref = g[f"lsq{q}_apply"]
    assert np.max(np.abs(y - ref)) <= 1e-13 * np.max(np.abs(ref))


@pytest.mark.parametrize("solver", ["tr", "nr"])
@pytest.mark.parametrize("q", [0, 1])
def test_general_pencil_matches_reference(gpu_ctx, golden, solver, q):
    """cheb_lan_tr / cheb_lan_nr(A, &B, ...) with a non-diagonal SPD B: identical counts and
    eigenvalues within 1e-10 relative of the reference (and of the closed form); returned
    vectors B-orthonormal with ||A x - lambda B x|| <= tol max(1, |lambda|)."""
    api, g, a, b = _problem(golden)
    niter, nmv, degree, hit, xi, eta, est = g[f"{solver}{q}_meta"]
    lo, hi = g["bounds"]
    f = api.find_pol(xi, eta, api.SpectralBounds(lo, hi))
    assert f.k == int(degree)
    cfg = api.SolverConfig(est_count=int(est), res_tol=1e-8, seed=1234)
    drv = api.cheb_lan_tr if solver == "tr" else api.cheb_lan_nr
    r = drv(a, b, f, xi, eta, cfg)
    ref = g[f"{solver}{q}_vals"]
    ev = g["analytic"]
    truth = ev[(ev >= xi) & (ev <= eta)]
    assert r.eigenvalues.size == ref.size == truth.size, (r.eigenvalues.size, ref.size)
    assert np.all(np.abs(r.eigenvalues - ref) <= 1e-10 * np.abs(ref))
    assert np.all(np.abs(r.eigenvalues - truth) <= 1e-10 * np.abs(truth))
    assert np.all(r.residuals <= 1e-8 * np.maximum(1.0, np.abs(r.eigenvalues)))
    A, B = _dense(a), _dense(b)
    X = r.vectors
    G = X.T @ B @ X
    assert np.max(np.abs(G - np.eye(X.shape[1]))) <= 1e-8
    R = A @ X - (B @ X) * r.eigenvalues
    res = np.linalg.norm(R, axis=0)
    assert np.all(res <= 1e-8 * np.maximum(1.0, np.abs(r.eigenvalues)))
    assert np.allclose(res, r.residuals, rtol=1e-3, atol=1e-12)


def test_pencil_bounds_and_density(gpu_ctx, golden):
    """lan_tr_bounds in the B inner product and dos_generalized (dos.hpp:160-184) for the
    pencil: bounds within the reference's settle tolerance of the reference's and enclosing the
    closed-form spectrum; the density integrates to n and counts within 15% of the truth."""
    api, g, a, b = _problem(golden)
    ev = g["analytic"]
    rlo, rhi = g["bounds"]
    bd = api.lan_tr_bounds_pencil(a, b, 1e-4, 60, 40, 1234)
    spread = rhi - rlo
    assert abs(bd.lmin - rlo) <= 1e-3 * spread and abs(bd.lmax - rhi) <= 1e-3 * spread
    assert bd.lmin <= ev[0] + 1e-3 * spread and bd.lmax >= ev[-1] - 1e-3 * spread
    c = api.dos_generalized(a, b, api.SpectralBounds(rlo, rhi),
                            api.DosConfig(method="lanczos", m=60, n_vec=40, seed=1234))
    assert abs(c.nev_est - a.n) <= 1e-6 * a.n
    for lo, hi in ((2.0, 6.0), (10.0, 20.0), (30.0, 50.0)):
        t = int(((ev >= lo) & (ev <= hi)).sum())
        assert abs(api.dos_count(c, lo, hi) - t) <= max(0.15 * t, 10.0), (lo, hi, t)
        gx, gy = g["dos_x"], g["dos_y"]
        ref_c = api.DosCurve(gx, gy, float(g["dos_nev"]), a.n)
        assert abs(api.dos_count(ref_c, lo, hi) - t) <= max(0.15 * t, 10.0)


def test_general_pencil_errors(gpu_ctx, golden):
    api, g, a, b = _problem(golden)
    f = api.find_pol(2.0, 3.0, api.SpectralBounds(*g["bounds"]))
    neg = api.CsrMatrix(a.n, b.row_ptr, b.col_idx, -b.vals)
    with pytest.raises(ValueError):  # B not positive definite
        api.cheb_lan_tr(a, neg, f, 2.0, 3.0, api.SolverConfig(est_count=50))
    small = api.gen_laplacian([10, 10])
    with pytest.raises(ValueError):  # size mismatch
        api.cheb_lan_tr(a, small, f, 2.0, 3.0, api.SolverConfig(est_count=50))
