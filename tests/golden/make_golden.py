"""Generate the committed golden fixtures from the UNMODIFIED reference (oracle/_ref, compiled from
/root/reference/proj/include by oracle/Makefile).  Run in the build container (the reference is
absent on the GPU box):

    python tests/golden/make_golden.py [--skip-solve]

Outputs tests/golden/*.npz.  Every eigen/DOS/filter array is produced by calling the reference
library; the cfg4/cfg5 input matrices (generators the reference lacks) come from
the product's host-only generator, whose structural properties tests/test_configs.py checks.
"""
import argparse
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import reflib  # noqa: E402


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **{k: np.asarray(v) for k, v in arrays.items()})
    print("wrote", path, f"{os.path.getsize(path) / 1024:.1f} KiB")


def kats():
    out = {}
    # filter coefficient KATs (filter_poly.hpp)
    ints = [(-0.4, 0.4), (0.2, 0.4), (0.0, 0.3), (-0.5, 0.5), (-0.9, -0.85), (0.61, 0.62)]
    for damp in ("none", "sigma", "jackson"):
        for q, (a, b) in enumerate(ints):
            f = reflib.find_pol(a, b, -1.0, 1.0, damping=damp)
            out[f"findpol_{damp}_{q}_k"] = f["k"]
            out[f"findpol_{damp}_{q}_scalars"] = [f["gamma"], f["ta"], f["tb"], f["bar"], f["c"], f["d"],
                                                  float(f["cap_reached"])]
            out[f"findpol_{damp}_{q}_mu"] = f["mu"]
        for k in (1, 2, 8, 40):
            out[f"damp_{damp}_{k}"] = reflib.damping_multipliers(k, damp)
        for k, g in ((16, 0.3), (5, -0.7)):
            out[f"ncoef_{damp}_{k}"] = reflib.normalized_coeffs(k, g, damp)
    out["findpol_bounds"] = [0.0, 8.0]
    for q, (a, b) in enumerate([(0.0, 0.5), (7.5, 8.0), (3.0, 4.0), (0.4, 1.0443178519)]):
        f = reflib.find_pol(a, b, 0.0, 8.0)
        out[f"findpol_b8_{q}_k"] = f["k"]
        out[f"findpol_b8_{q}_mu"] = f["mu"]
        out[f"findpol_b8_{q}_scalars"] = [f["gamma"], f["ta"], f["tb"], f["bar"], f["c"], f["d"],
                                          float(f["cap_reached"])]
    out["balance_16_02_04_sigma"] = reflib.balance_center(16, 0.2, 0.4, "sigma")
    # rng streams (rng.hpp)
    out["rng_normal_7"] = reflib.rng_vectors(7, "normal", 257, 3)
    out["rng_rademacher_7"] = reflib.rng_vectors(7, "rademacher", 257, 3)
    out["rng_uniform_7"] = reflib.rng_uniform(7, 100)
    # matrices + analytic spectra (laplacian.hpp)
    for dims in ([7], [5, 4], [4, 3, 5], [20, 20]):
        tag = "x".join(map(str, dims))
        rp, ci, v = reflib.laplacian(dims)
        out[f"lap_{tag}_rp"], out[f"lap_{tag}_ci"], out[f"lap_{tag}_v"] = rp, ci, v
        out[f"lapeig_{tag}"] = reflib.laplacian_eigs(dims)
    # apply_pol / matvec on the 20x20 Laplacian (filter_poly.hpp:256-277)
    rp, ci, v = reflib.laplacian([20, 20])
    x = reflib.rng_vectors(3, "normal", 400, 1)[0]
    out["ap_x"] = x
    out["ap_Ax"] = reflib.matvec(rp, ci, v, x)
    for damp in ("sigma", "jackson"):
        f = reflib.find_pol(1.0, 1.5, 0.0, 8.0, damping=damp)
        y, nmv = reflib.apply_pol(rp, ci, v, f["mu"], f["c"], f["d"], x)
        out[f"ap_{damp}_mu"], out[f"ap_{damp}_cd"] = f["mu"], [f["c"], f["d"]]
        out[f"ap_{damp}_y"], out[f"ap_{damp}_nmv"] = y, nmv
    # KPM moments / curve / slicing on 25x25 (dos.hpp, slicer.hpp)
    rp, ci, v = reflib.laplacian([25, 25])
    for kind in ("rademacher", "normal"):
        out[f"kpm25_zeta_{kind}"] = reflib.kpm_moments(rp, ci, v, 0.0, 8.0, 60, 8, 777, kind)
    x25, y25, nev25 = reflib.kpm_dos(rp, ci, v, 0.0, 8.0, 60, 8, 300, 777)
    out["kpm25_x"], out["kpm25_y"], out["kpm25_nev"] = x25, y25, nev25
    out["kpm25_bp4"], out["kpm25_est4"] = reflib.slice_spectrum(x25, y25, 625, 0.0, 8.0, 4)
    out["kpm25_count_1_3"] = reflib.dos_count(x25, y25, 625, 1.0, 3.0)
    # CGS2 (orth.hpp:70-80)
    rng = np.random.default_rng(0)
    W = np.linalg.qr(rng.standard_normal((300, 25)))[0].T.copy()
    t = rng.standard_normal(300)
    out["cgs_W"], out["cgs_t"] = W, t
    out["cgs_t_out"], out["cgs_h"] = reflib.paired_cgs2(W, t)
    # small eigensolvers (tridiag_eig.hpp, dense_eig.hpp)
    a = rng.standard_normal(30)
    b = rng.standard_normal(29)
    out["trid_a"], out["trid_b"] = a, b
    out["trid_vals"], out["trid_vecs"] = reflib.sym_tridiag_eig(a, b, True)
    S = rng.standard_normal((24, 24))
    S = S + S.T
    out["dense_S"] = S
    out["dense_vals"], out["dense_vecs"] = reflib.dense_sym_eig(S, True)
    # lanczos_run on 20x20 (lanczos.hpp:37-118)
    rp, ci, v = reflib.laplacian([20, 20])
    st = reflib.rng_vectors(5, "normal", 400, 1)[0]
    lr = reflib.lanczos_run(rp, ci, v, st, 30)
    out["lanczos_start"], out["lanczos_alpha"], out["lanczos_beta"] = st, lr["alpha"], lr["beta"]
    out["lanczos_next_beta"] = lr["next_beta"]
    save("kats", **out)


def cfg1(skip_solve):
    # BASELINE configs[0]: 100x100, KPM 80 x 20 Rademacher seed 0, [0.4,1.6] in 2, Jackson, NR 1e-8
    rp, ci, v = reflib.laplacian([100, 100])
    lo, hi = reflib.lan_tr_bounds(rp, ci, v, 1e-4, 60, 40, 0)
    zeta = reflib.kpm_moments(rp, ci, v, lo, hi, 80, 20, 0, "rademacher")
    x, y, nev = reflib.kpm_dos(rp, ci, v, lo, hi, 80, 20, 300, 0)
    bp, est = reflib.slice_spectrum(x, y, 10000, 0.4, 1.6, 2)
    degs = [reflib.find_pol(bp[i], bp[i + 1], lo, hi, damping="jackson")["k"] for i in range(2)]
    out = dict(bounds=[lo, hi], zeta=zeta, x=x, y=y, nev=nev, bp=bp, est=est, degrees=degs)
    if not skip_solve:
        t0 = time.time()
        r = reflib.solve(rp, ci, v, 0.4, 1.6, 2, "nr", "jackson", 80, 20, 300, "rademacher", 1e-8, 0,
                         jobs=2)
        print(f"cfg1 reference solve {time.time() - t0:.1f} s")
        for i, s in enumerate(r["slices"]):
            out[f"slice{i}_vals"] = s["eigenvalues"]
            out[f"slice{i}_res"] = s["residuals"]
            out[f"slice{i}_meta"] = [s["niter"], s["n_A_matvec"], s["degree"], int(s["hit_max_its"])]
        out["solve_bp"] = r["breakpoints"]
        out["solve_bounds"] = [r["lmin"], r["lmax"]]
    save("cfg1", **out)


def cfg2():
    # BASELINE configs[1]: 64^3, KPM 100 x 40 Gaussian seed 1234, [0.6,1.2] in 8 (sigma damping)
    rp, ci, v = reflib.laplacian([64, 64, 64])
    t0 = time.time()
    lo, hi = reflib.lan_tr_bounds(rp, ci, v, 1e-4, 60, 40, 1234)
    zeta = reflib.kpm_moments(rp, ci, v, lo, hi, 100, 40, 1234, "normal")
    x, y, nev = reflib.curve_from_moments(zeta / (40.0 * 262144), 262144, lo, hi, 300)
    bp, est = reflib.slice_spectrum(x, y, 262144, 0.6, 1.2, 8)
    degs = [reflib.find_pol(bp[i], bp[i + 1], lo, hi)["k"] for i in range(8)]
    print(f"cfg2 bounds+kpm {time.time() - t0:.1f} s; degrees {degs}")
    save("cfg2", bounds=[lo, hi], zeta=zeta, x=x, y=y, nev=nev, bp=bp, est=est, degrees=degs)


def cfg4p():
    """BASELINE configs[3] proxy: random banded + 8 extras, n = 20,000 (seed 4); window = middle 2%
    of the KPM DOS (first grid points with cumulative mass >= 0.49 / 0.51, npts 3000), 8 slices,
    ChebLanTr tol 1e-9; the reference's slice 3 solve."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from paper_1802_05215_b200 import api  # host-only generator (no GPU needed)
    a = api.gen_random_sparse(20000, 4)
    rp, ci, v = a.row_ptr, a.col_idx, a.vals
    lo, hi = reflib.lan_tr_bounds(rp, ci, v, 1e-4, 60, 40, 4)
    zeta = reflib.kpm_moments(rp, ci, v, lo, hi, 60, 40, 4, "rademacher")
    x, y, nev = reflib.curve_from_moments(zeta / (40.0 * 20000), 20000, lo, hi, 3000)
    cum = np.concatenate([[0.0], np.cumsum(0.5 * (y[1:] + y[:-1]) * np.diff(x))])
    cum /= cum[-1]
    w0, w1 = x[np.argmax(cum >= 0.49)], x[np.argmax(cum >= 0.51)]
    bp, est = reflib.slice_spectrum(x, y, 20000, w0, w1, 8)
    t0 = time.time()
    r = reflib.cheb_lan(rp, ci, v, "tr", bp[3], bp[4], lo, hi, res_tol=1e-9,
                        est_count=int(np.ceil(est[3])), seed=4)
    print(f"cfg4p slice 3: {len(r['eigenvalues'])} pairs, deg {r['degree']}, {time.time() - t0:.0f} s")
    save("cfg4p", bounds=[lo, hi], zeta=zeta, window=[w0, w1], bp=bp, est=est,
         slice3_vals=r["eigenvalues"], slice3_res=r["residuals"],
         slice3_meta=[r["niter"], r["n_A_matvec"], r["degree"]], nnz=a.nnz,
         rp_check=[int(rp[-1]), int(ci.sum() % 1000003)], v_check=[float(v.sum()), float(np.abs(v).sum())])


def cfg5p():
    """BASELINE configs[4] proxy: 24^3 Laplacian scaled to D A D, d = (0.5 + uniform)^-1/2
    (seed 5); [1, 2] in 8 DOS slices; the reference's ChebLanTr on slices 2 and 7 (tol 1e-8)."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from paper_1802_05215_b200 import api
    L = api.gen_laplacian([24, 24, 24])
    b, d = api.mass_scaling(L.n, 5)
    S = api.scale_sym_host(L, d)
    rp, ci, v = S.row_ptr, S.col_idx, S.vals
    lo, hi = reflib.lan_tr_bounds(rp, ci, v, 1e-4, 60, 40, 5)
    zeta = reflib.kpm_moments(rp, ci, v, lo, hi, 60, 40, 5, "rademacher")
    x, y, nev = reflib.curve_from_moments(zeta / (40.0 * L.n), L.n, lo, hi, 300)
    bp, est = reflib.slice_spectrum(x, y, L.n, 1.0, 2.0, 8)
    out = dict(bounds=[lo, hi], zeta=zeta, bp=bp, est=est, d=d, vals_scaled=v)
    for s in (2, 7):
        r = reflib.cheb_lan(rp, ci, v, "tr", bp[s], bp[s + 1], lo, hi, res_tol=1e-8,
                            est_count=int(np.ceil(est[s])), seed=5)
        out[f"slice{s}_vals"] = r["eigenvalues"]
        out[f"slice{s}_res"] = r["residuals"]
    save("cfg5p", **out)


def pencil():
    """Generalized pencil (A, B), A = 16^3 Laplacian, B = diag(0.5 + uniform) (seed 7): the
    reference's own B-weighted cheb_lan_tr / cheb_lan_nr / cheb_si (b != nullptr, SpdFactor solves) on
    [1.0, 1.4] with bounds fixed to [0, 24] (lambda(A, B) <= 12 / 0.5)."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from paper_1802_05215_b200 import api
    L = api.gen_laplacian([16, 16, 16])
    b, _ = api.mass_scaling(L.n, 7)
    out = dict(b=b, window=[1.0, 1.4], bounds=[0.0, 24.0])
    for solver in ("tr", "nr", "si"):
        r = reflib.cheb_lan_pencil(L.row_ptr, L.col_idx, L.vals, b, solver, 1.0, 1.4, 0.0, 24.0,
                                   est_count=80 if solver != "si" else 60, seed=7)
        out[f"{solver}_vals"] = r["eigenvalues"]
        out[f"{solver}_res"] = r["residuals"]
        out[f"{solver}_meta"] = [r["niter"], r["n_A_matvec"], r["degree"]]
    save("pencil", **out)


def landos():
    """lan_dos (dos.hpp:136-154, add_ritz_gaussians :63-75): the reference's Lanczos-quadrature
    curves on seeded Gaussian probes, plus the slicing the CLI would derive from them."""
    out = {}
    cases = [("l20", [20, 20, 20], 40, 12, 1234, 0.0),
             ("l60", [60, 60], 50, 16, 7, 0.0),
             ("l60s", [60, 60], 30, 8, 99, 0.05)]   # explicit sigma
    for tag, dims, m, nvec, seed, sigma in cases:
        rp, ci, v = reflib.laplacian(dims)
        lo, hi = reflib.lan_tr_bounds(rp, ci, v, 1e-4, 60, 40, seed)
        x, y, nev = reflib.lan_dos(rp, ci, v, lo, hi, m=m, n_vec=nvec, npts=300, sigma=sigma, seed=seed)
        xi, eta = lo + 0.1 * (hi - lo), lo + 0.4 * (hi - lo)
        bp, est = reflib.slice_spectrum(x, y, len(v) and len(rp) - 1, xi, eta, 4)
        out[f"{tag}_meta"] = [m, nvec, seed, sigma, lo, hi, nev, xi, eta]
        out[f"{tag}_dims"] = dims
        out[f"{tag}_x"] = x
        out[f"{tag}_y"] = y
        out[f"{tag}_bp"] = bp
        out[f"{tag}_est"] = est
    save("landos", **out)


def kron_mass(nx):
    """B = M1 (x) M1, M1 = tridiag(1, 4, 1) / 6 (1-D linear-element mass matrix): a 9-point SPD
    matrix whose eigenvectors are those of the 2-D Laplacian (sine products), so the pencil
    (Laplacian, B) has the closed-form spectrum (t_i + t_j) / (m_i m_j)."""
    m1 = np.diag(np.full(nx, 4.0 / 6.0)) + np.diag(np.full(nx - 1, 1.0 / 6.0), 1) + \
        np.diag(np.full(nx - 1, 1.0 / 6.0), -1)
    Bd = np.kron(m1, m1)
    rows, cols = np.nonzero(Bd)
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    rp = np.zeros(nx * nx + 1, np.int32)
    np.add.at(rp, rows + 1, 1)
    return np.cumsum(rp).astype(np.int32), cols.astype(np.int32), Bd[rows, cols].astype(np.float64)


def pencil_general():
    """The reference's B-weighted drivers (Cholesky B-solves) on a non-diagonal SPD B."""
    nx = 30
    rp, ci, v = reflib.laplacian([nx, nx])
    brp, bci, bv = kron_mass(nx)
    th = np.arange(1, nx + 1) * np.pi / (nx + 1)
    t = 2.0 - 2.0 * np.cos(th)
    m = (4.0 + 2.0 * np.cos(th)) / 6.0
    ev = np.sort(((t[:, None] + t[None, :]) / (m[:, None] * m[None, :])).ravel())
    lo, hi = reflib.pencil_bounds(rp, ci, v, brp, bci, bv, seed=1234)
    x, y, nev = reflib.pencil_dos(rp, ci, v, brp, bci, bv, lo, hi, m=60, n_vec=40, npts=300, seed=1234)
    out = dict(brp=brp, bci=bci, bv=bv, analytic=ev, bounds=[lo, hi], dos_x=x, dos_y=y, dos_nev=nev)
    for q, (xi, eta) in enumerate([(2.0, 3.0), (10.0, 11.5)]):
        est = int(((ev >= xi) & (ev <= eta)).sum())
        for solver in ("tr", "nr"):
            r = reflib.cheb_lan_pencil_csr(rp, ci, v, brp, bci, bv, solver, xi, eta, lo, hi,
                                           est_count=est, seed=1234)
            out[f"{solver}{q}_vals"] = r["eigenvalues"]
            out[f"{solver}{q}_res"] = r["residuals"]
            out[f"{solver}{q}_meta"] = [r["niter"], r["n_A_matvec"], r["degree"],
                                        int(r["hit_max_its"]), xi, eta, est]
    # ls_pol_approx KATs (test_operators.cpp:162-225 shapes)
    for q, (fun, a, b, tol) in enumerate([("inverse", 1.0, 2.0, 1e-8), ("inverse_sqrt", 0.5, 2.0, 1e-9),
                                          ("inverse", 1.0 / 3.0 - 1e-3, 1.0 + 1e-3, 1e-12),
                                          ("inverse_sqrt", 0.1, 1.05, 1e-13)]):
        co, ach = reflib.ls_pol_approx(fun, a, b, tol)
        out[f"lsq{q}_coeff"] = co
        out[f"lsq{q}_meta"] = [1.0 if fun == "inverse_sqrt" else 0.0, a, b, tol, ach]
        xv = np.cos(np.arange(brp.size - 1) * 0.37)
        out[f"lsq{q}_apply"] = reflib.apply_cheb(brp, bci, bv, fun, a, b, co, xv)
    save("pencil_general", **out)


def cli():
    """`sliceeig solve --dims 30,30 --interval 0.4,0.6 --slices 4 [--solver tr]` with the CLI
    defaults (KPM deg 60 x 40 Rademacher probes, sigma damping, tol 1e-8, seed 1234): the
    reference's cmd_solve semantics (tools/sliceeig_main.cpp:464-619) via the harness."""
    rp, ci, v = reflib.laplacian([30, 30])
    out = {}
    for solver in ("nr", "tr", "si"):
        r = reflib.solve(rp, ci, v, 0.4, 0.6, 4, solver=solver, jobs=4)
        out[f"{solver}_bp"] = r["breakpoints"]
        out[f"{solver}_est"] = r["est_counts"]
        out[f"{solver}_bounds"] = [r["lmin"], r["lmax"]]
        for i, s in enumerate(r["slices"]):
            assert s["error"] is None
            out[f"{solver}_slice{i}_vals"] = s["eigenvalues"]
            out[f"{solver}_slice{i}_meta"] = [s["niter"], s["n_A_matvec"], s["degree"], int(s["hit_max_its"])]
    # cheb_si directly (eigensolvers.hpp:760-940) on a 60x60 window with the bounds fixed
    rp6, ci6, v6 = reflib.laplacian([60, 60])
    b6 = reflib.lan_tr_bounds(rp6, ci6, v6, 1e-4, 60, 40, 1234)
    for q, (lo, hi, est) in enumerate([(0.5, 0.6, 20), (1.0, 1.1, 25)]):
        r = reflib.cheb_lan(rp6, ci6, v6, "si", lo, hi, b6[0], b6[1], est_count=est, seed=1234)
        out[f"si60_{q}_vals"] = r["eigenvalues"]
        out[f"si60_{q}_res"] = r["residuals"]
        out[f"si60_{q}_meta"] = [r["niter"], r["n_A_matvec"], r["degree"], int(r["hit_max_its"]), lo, hi, est,
                                 b6[0], b6[1]]
    save("cli", **out)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-solve", action="store_true")
    ap.add_argument("--only", default="kats,cfg1,cfg2,cfg4p,cfg5p,cli,pencil,landos,pencil_general")
    a = ap.parse_args()
    only = a.only.split(",")
    if "kats" in only:
        kats()
    if "cfg2" in only:
        cfg2()
    if "cfg1" in only:
        cfg1(a.skip_solve)
    if "cfg4p" in only:
        cfg4p()
    if "cfg5p" in only:
        cfg5p()
    if "cli" in only:
        cli()
    if "pencil" in only:
        pencil()
    if "landos" in only:
        landos()
    if "pencil_general" in only:
        pencil_general()
