"""TEST INFRASTRUCTURE ONLY: numpy-facing wrapper of oracle/_ref/libsliceeig_ref.so, i.e. the
UNMODIFIED reference headers (/root/reference/proj/include/sliceeig) compiled in place by
oracle/Makefile through the C-ABI harness oracle/ref_harness.cpp.

On the GPU box /root/reference is absent, but the prebuilt .so travels with the repo snapshot;
``available()`` reports whether it can be loaded.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_ref", "libsliceeig_ref.so")
_lib = None

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_PD = C.POINTER(C.c_double)
_PI = C.POINTER(C.c_int)
_PL = C.POINTER(C.c_long)

DAMPING = {"none": 0, "sigma": 1, "jackson": 2}
SOLVER = {"nr": 0, "tr": 1, "si": 2}
PROBES = {"rademacher": 0, "normal": 1}


class RefError(RuntimeError):
    pass


def build() -> str:
    if os.path.isdir("/root/reference/proj/include"):
        subprocess.run(["make", "-s", "-C", _HERE, "ref"], check=True)
    return _SO


def available() -> bool:
    try:
        lib()
        return True
    except OSError:
        return False


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        L = C.CDLL(_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_cheb_lan.restype = C.c_void_p
        L.ref_cheb_lan.argtypes = [C.c_int, _ip, _ip, _dp, C.c_int, C.c_double, C.c_double,
                                   C.c_double, C.c_double, C.c_int, C.c_int, C.c_long, C.c_int,
                                   C.c_double, C.c_double, C.c_int, C.c_uint64]
        L.ref_cheb_lan_pencil.restype = C.c_void_p
        L.ref_cheb_lan_pencil.argtypes = [C.c_int, _ip, _ip, _dp, _dp, C.c_int, C.c_double,
                                          C.c_double, C.c_double, C.c_double, C.c_int, C.c_double,
                                          C.c_int, C.c_uint64]
        L.ref_cheb_lan_pencil_csr.restype = C.c_void_p
        L.ref_cheb_lan_pencil_csr.argtypes = [C.c_int, _ip, _ip, _dp, _ip, _ip, _dp, C.c_int,
                                              C.c_double, C.c_double, C.c_double, C.c_double,
                                              C.c_int, C.c_double, C.c_int, C.c_uint64]
        L.ref_solve.restype = C.c_void_p
        L.ref_solve.argtypes = [C.c_int, _ip, _ip, _dp, C.c_double, C.c_double, C.c_int, C.c_int,
                                C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                C.c_uint64, C.c_int, C.c_double, C.c_double]
        L.ref_results_nslices.argtypes = [C.c_void_p]
        L.ref_results_slice.argtypes = [C.c_void_p, C.c_int, _PI, _PL, _PL, _PI, _PI, _dp]
        L.ref_results_values.argtypes = [C.c_void_p, C.c_int, _dp, _dp, C.c_void_p]
        L.ref_results_pipeline.argtypes = [C.c_void_p, _dp, C.c_void_p, C.c_void_p]
        L.ref_results_free.argtypes = [C.c_void_p]
        L.ref_rng_normal.argtypes = [C.c_uint64, C.c_int, C.c_int, _dp]
        L.ref_rng_rademacher.argtypes = [C.c_uint64, C.c_int, C.c_int, _dp]
        L.ref_rng_uniform.argtypes = [C.c_uint64, C.c_int, _dp]
        L.ref_kpm_moments.argtypes = [C.c_int, _ip, _ip, _dp, C.c_double, C.c_double, C.c_int,
                                      C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_int, _dp]
        _lib = L
    return _lib


def _chk(rc):
    if rc != 0:
        msg = lib().ref_last_error().decode()
        raise (ValueError if rc == -1 else RefError)(msg)


def laplacian(dims):
    d = np.asarray(dims, np.int32)
    n = C.c_int()
    nnz = C.c_long()
    _chk(lib().ref_laplacian(len(d), d.ctypes.data_as(_PI), C.byref(n), C.byref(nnz), None, None,
                             None))
    rp = np.empty(n.value + 1, np.int32)
    ci = np.empty(nnz.value, np.int32)
    v = np.empty(nnz.value, np.float64)
    _chk(lib().ref_laplacian(len(d), d.ctypes.data_as(_PI), C.byref(n), C.byref(nnz),
                             rp.ctypes.data_as(_PI), ci.ctypes.data_as(_PI), v.ctypes.data_as(_PD)))
    return rp, ci, v


def laplacian_eigs(dims):
    d = np.asarray(dims, np.int32)
    out = np.empty(int(np.prod(d)), np.float64)
    _chk(lib().ref_laplacian_eigs(len(d), d.ctypes.data_as(_PI), out.ctypes.data_as(_PD)))
    return out


def _csr_args(rp, ci, v):
    return (C.c_int(len(rp) - 1), rp.ctypes.data_as(_PI), ci.ctypes.data_as(_PI),
            v.ctypes.data_as(_PD))


def matvec(rp, ci, v, x):
    x = np.ascontiguousarray(x, np.float64)
    y = np.empty(len(rp) - 1, np.float64)
    _chk(lib().ref_matvec(*_csr_args(rp, ci, v), x.ctypes.data_as(_PD), y.ctypes.data_as(_PD)))
    return y


def rng_vectors(seed, kind, n, count=1):
    out = np.empty(n * count, np.float64)
    f = lib().ref_rng_normal if kind == "normal" else lib().ref_rng_rademacher
    _chk(f(seed, n, count, out))
    return out.reshape(count, n)


def rng_uniform(seed, n):
    out = np.empty(n, np.float64)
    _chk(lib().ref_rng_uniform(seed, n, out))
    return out


def find_pol(xi, eta, lmin, lmax, tau=0.8, max_deg=3000, damping="sigma"):
    mu = np.empty(max_deg + 1, np.float64)
    k, cap = C.c_int(), C.c_int()
    g, ta, tb, bar, c, d = (C.c_double() for _ in range(6))
    _chk(lib().ref_find_pol(C.c_double(xi), C.c_double(eta), C.c_double(lmin), C.c_double(lmax),
                            C.c_double(tau), C.c_int(max_deg), C.c_int(DAMPING[damping]),
                            C.c_int(max_deg + 1), C.byref(k), C.byref(g), mu.ctypes.data_as(_PD),
                            C.byref(ta), C.byref(tb), C.byref(bar), C.byref(cap), C.byref(c),
                            C.byref(d)))
    return {"k": k.value, "gamma": g.value, "ta": ta.value, "tb": tb.value, "bar": bar.value,
            "c": c.value, "d": d.value, "cap_reached": bool(cap.value),
            "mu": mu[: k.value + 1].copy()}


def balance_center(k, ta, tb, damping):
    g = C.c_double()
    _chk(lib().ref_balance_center(C.c_int(k), C.c_double(ta), C.c_double(tb),
                                  C.c_int(DAMPING[damping]), C.byref(g)))
    return g.value


def damping_multipliers(k, damping):
    out = np.empty(k + 1, np.float64)
    _chk(lib().ref_damping(C.c_int(k), C.c_int(DAMPING[damping]), out.ctypes.data_as(_PD)))
    return out


def normalized_coeffs(k, gamma, damping):
    out = np.empty(k + 1, np.float64)
    _chk(lib().ref_normalized_coeffs(C.c_int(k), C.c_double(gamma), C.c_int(DAMPING[damping]),
                                     out.ctypes.data_as(_PD)))
    return out


def eval_series(mu, t):
    mu = np.ascontiguousarray(mu, np.float64)
    out = C.c_double()
    _chk(lib().ref_eval_series(C.c_int(len(mu) - 1), mu.ctypes.data_as(_PD), C.c_double(t),
                               C.byref(out)))
    return out.value


def apply_pol(rp, ci, v, mu, c, d, x):
    mu = np.ascontiguousarray(mu, np.float64)
    x = np.ascontiguousarray(x, np.float64)
    out = np.empty(len(rp) - 1, np.float64)
    nmv = C.c_long()
    _chk(lib().ref_apply_pol(*_csr_args(rp, ci, v), C.c_int(len(mu) - 1), mu.ctypes.data_as(_PD),
                             C.c_double(c), C.c_double(d), x.ctypes.data_as(_PD),
                             out.ctypes.data_as(_PD), C.byref(nmv)))
    return out, nmv.value


def kpm_moments(rp, ci, v, lmin, lmax, m, n_vec, seed, kind="rademacher", first=0, count=None):
    z = np.empty(m + 1, np.float64)
    count = n_vec if count is None else count
    _chk(lib().ref_kpm_moments(len(rp) - 1, rp, ci, v, lmin, lmax, m, n_vec, seed, PROBES[kind],
                               first, count, z))
    return z


def kpm_dos(rp, ci, v, lmin, lmax, m=60, n_vec=40, npts=300, seed=1234):
    x = np.empty(npts, np.float64)
    y = np.empty(npts, np.float64)
    nev = C.c_double()
    _chk(lib().ref_kpm_dos(*_csr_args(rp, ci, v), C.c_double(lmin), C.c_double(lmax), C.c_int(m),
                           C.c_int(n_vec), C.c_int(npts), C.c_uint64(seed), x.ctypes.data_as(_PD),
                           y.ctypes.data_as(_PD), C.byref(nev)))
    return x, y, nev.value


def curve_from_moments(zeta, n, lmin, lmax, npts=300):
    zeta = np.ascontiguousarray(zeta, np.float64)
    x = np.empty(npts, np.float64)
    y = np.empty(npts, np.float64)
    nev = C.c_double()
    _chk(lib().ref_curve_from_moments(C.c_int(len(zeta) - 1), zeta.ctypes.data_as(_PD), C.c_int(n),
                                      C.c_double(lmin), C.c_double(lmax), C.c_int(npts),
                                      x.ctypes.data_as(_PD), y.ctypes.data_as(_PD), C.byref(nev)))
    return x, y, nev.value


def lan_dos(rp, ci, v, lmin, lmax, m=60, n_vec=40, npts=300, sigma=0.0, seed=1234):
    x = np.empty(npts, np.float64)
    y = np.empty(npts, np.float64)
    nev = C.c_double()
    _chk(lib().ref_lan_dos(*_csr_args(rp, ci, v), C.c_double(lmin), C.c_double(lmax), C.c_int(m),
                           C.c_int(n_vec), C.c_int(npts), C.c_double(sigma), C.c_uint64(seed),
                           x.ctypes.data_as(_PD), y.ctypes.data_as(_PD), C.byref(nev)))
    return x, y, nev.value


def dos_count(x, y, n, xi, eta):
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    out = C.c_double()
    _chk(lib().ref_dos_count(C.c_int(len(x)), C.c_int(n), x.ctypes.data_as(_PD),
                             y.ctypes.data_as(_PD), C.c_double(xi), C.c_double(eta), C.byref(out)))
    return out.value


def slice_spectrum(x, y, n, xi, eta, ns):
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    bp = np.empty(ns + 1, np.float64)
    est = np.empty(ns, np.float64)
    _chk(lib().ref_slice_spectrum(C.c_int(len(x)), C.c_int(n), x.ctypes.data_as(_PD),
                                  y.ctypes.data_as(_PD), C.c_double(xi), C.c_double(eta),
                                  C.c_int(ns), bp.ctypes.data_as(_PD), est.ctypes.data_as(_PD)))
    return bp, est


def lan_tr_bounds(rp, ci, v, tol=1e-4, restart=60, max_restarts=40, seed=1234):
    lo, hi = C.c_double(), C.c_double()
    _chk(lib().ref_lan_tr_bounds(*_csr_args(rp, ci, v), C.c_double(tol), C.c_int(restart),
                                 C.c_int(max_restarts), C.c_uint64(seed), C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def lanczos_run(rp, ci, v, start, m, want_basis=False):
    n = len(rp) - 1
    start = np.ascontiguousarray(start, np.float64)
    mm = min(m, n)
    alpha = np.zeros(mm, np.float64)
    beta = np.zeros(max(mm - 1, 1), np.float64)
    basis = np.zeros((mm, n), np.float64) if want_basis else None
    steps, brk = C.c_int(), C.c_int()
    nb = C.c_double()
    _chk(lib().ref_lanczos_run(*_csr_args(rp, ci, v), start.ctypes.data_as(_PD), C.c_int(m),
                               alpha.ctypes.data_as(_PD), beta.ctypes.data_as(_PD), C.byref(steps),
                               C.byref(brk), C.byref(nb),
                               basis.ctypes.data_as(_PD) if want_basis else None))
    s = steps.value
    return {"alpha": alpha[:s], "beta": beta[: max(s - 1, 0)], "steps": s,
            "breakdown": bool(brk.value), "next_beta": nb.value,
            "basis": basis[:s] if want_basis else None}


def paired_cgs2(W, t, h=None):
    W = np.ascontiguousarray(W, np.float64)
    k, n = W.shape
    t = np.array(t, np.float64, copy=True)
    hh = np.zeros(k, np.float64) if h is None else np.array(h, np.float64, copy=True)
    _chk(lib().ref_paired_cgs2(C.c_int(n), C.c_int(k), W.ctypes.data_as(_PD), t.ctypes.data_as(_PD),
                               hh.ctypes.data_as(_PD)))
    return t, hh


def sym_tridiag_eig(alpha, beta, want=True):
    m = len(alpha)
    a = np.ascontiguousarray(alpha, np.float64)
    b = np.ascontiguousarray(beta if m > 1 else np.zeros(1), np.float64)
    vals = np.empty(m, np.float64)
    vecs = np.empty((m, m), np.float64)
    _chk(lib().ref_sym_tridiag_eig(C.c_int(m), a.ctypes.data_as(_PD), b.ctypes.data_as(_PD),
                                   C.c_int(int(want)), vals.ctypes.data_as(_PD),
                                   vecs.ctypes.data_as(_PD)))
    return vals, (vecs.T.copy() if want else None)  # vecs[:, j] = eigenvector j


def dense_sym_eig(A, want=True):
    A = np.asfortranarray(A, np.float64)
    m = A.shape[0]
    vals = np.empty(m, np.float64)
    vecs = np.empty((m, m), np.float64)
    _chk(lib().ref_dense_sym_eig(C.c_int(m), A.ctypes.data_as(_PD), C.c_int(int(want)),
                                 vals.ctypes.data_as(_PD), vecs.ctypes.data_as(_PD)))
    return vals, (vecs.T.copy() if want else None)


def _collect(h, with_pipeline):
    L = lib()
    try:
        out = {"slices": []}
        for s in range(L.ref_results_nslices(h)):
            cnt, hit, deg = C.c_int(), C.c_int(), C.c_int()
            niter, nmv = C.c_long(), C.c_long()
            times = np.zeros(3, np.float64)
            rc = L.ref_results_slice(h, s, C.byref(cnt), C.byref(niter), C.byref(nmv),
                                     C.byref(hit), C.byref(deg), times)
            rec = {"error": L.ref_last_error().decode() if rc else None}
            vals = np.empty(cnt.value, np.float64)
            res = np.empty(cnt.value, np.float64)
            L.ref_results_values(h, s, vals, res, None)
            rec.update(eigenvalues=vals, residuals=res, niter=niter.value, n_A_matvec=nmv.value,
                       hit_max_its=bool(hit.value), degree=deg.value, t_mv=times[0],
                       t_orth=times[1], t_total=times[2])
            out["slices"].append(rec)
        if with_pipeline:
            sc = np.zeros(6, np.float64)
            ns = len(out["slices"])
            bp = np.empty(ns + 1, np.float64)
            est = np.empty(ns, np.float64)
            L.ref_results_pipeline(h, sc, bp.ctypes.data_as(C.c_void_p),
                                   est.ctypes.data_as(C.c_void_p))
            out.update(lmin=sc[0], lmax=sc[1], t_bounds=sc[2], t_dos=sc[3], t_solve=sc[4],
                       t_total=sc[5], breakpoints=bp, est_counts=est)
        return out
    finally:
        L.ref_results_free(h)


def cheb_lan(rp, ci, v, solver, xi, eta, lmin, lmax, damping="sigma", m=0, max_its=0, ncycle=30,
             tau1=0.0, res_tol=1e-8, est_count=20, seed=1234):
    h = lib().ref_cheb_lan(len(rp) - 1, rp, ci, v, SOLVER[solver], xi, eta, lmin, lmax,
                           DAMPING[damping], m, max_its, ncycle, tau1, res_tol, est_count, seed)
    if not h:
        msg = lib().ref_last_error().decode()
        raise RefError(msg)
    return _collect(h, False)["slices"][0]


def cheb_lan_pencil(rp, ci, v, bdiag, solver, xi, eta, lmin, lmax, damping="sigma",
                    res_tol=1e-8, est_count=20, seed=1234):
    """The reference's B-weighted cheb_lan_nr/tr on (A, diag(bdiag))."""
    h = lib().ref_cheb_lan_pencil(len(rp) - 1, rp, ci, v, np.ascontiguousarray(bdiag, np.float64),
                                  SOLVER[solver], xi, eta, lmin, lmax, DAMPING[damping], res_tol,
                                  est_count, seed)
    if not h:
        raise RefError(lib().ref_last_error().decode())
    return _collect(h, False)["slices"][0]


def solve(rp, ci, v, xi, eta, ns, solver="nr", damping="sigma", dos_m=60, dos_nvec=40,
          dos_npts=300, probes="rademacher", tol=1e-8, seed=1234, jobs=1, bounds=None):
    lo, hi = bounds if bounds is not None else (0.0, 0.0)
    h = lib().ref_solve(len(rp) - 1, rp, ci, v, xi, eta, ns, SOLVER[solver], DAMPING[damping],
                        dos_m, dos_nvec, dos_npts, PROBES[probes], tol, seed, jobs, lo, hi)
    if not h:
        raise RefError(lib().ref_last_error().decode())
    return _collect(h, True)


# ---- general SPD-B pencils (the reference's Cholesky-backed path) --------------------------------
def ls_pol_approx(fun, lmin, lmax, tol, max_deg=300):
    """cheb_approx.hpp:40-88.  fun: "inverse" | "inverse_sqrt".  Returns (coeff, achieved)."""
    cap = max_deg + 1
    co = np.empty(cap, np.float64)
    deg, ach = C.c_int(), C.c_double()
    _chk(lib().ref_ls_pol_approx(C.c_int(1 if fun == "inverse_sqrt" else 0), C.c_double(lmin),
                                 C.c_double(lmax), C.c_double(tol), C.c_int(max_deg), C.c_int(cap),
                                 C.byref(deg), co.ctypes.data_as(_PD), C.byref(ach)))
    return co[: deg.value + 1].copy(), ach.value


def apply_cheb(rp, ci, v, fun, lmin, lmax, coeff, x):
    """cheb_approx.hpp:91-112: y = p(B) x."""
    coeff = np.ascontiguousarray(coeff, np.float64)
    x = np.ascontiguousarray(x, np.float64)
    y = np.empty_like(x)
    _chk(lib().ref_apply_cheb(*_csr_args(rp, ci, v), C.c_int(1 if fun == "inverse_sqrt" else 0),
                              C.c_double(lmin), C.c_double(lmax), C.c_int(coeff.size - 1),
                              coeff.ctypes.data_as(_PD), x.ctypes.data_as(_PD), y.ctypes.data_as(_PD)))
    return y


def _csr_b(brp, bci, bv):
    return (brp.ctypes.data_as(_PI), bci.ctypes.data_as(_PI), bv.ctypes.data_as(_PD))


def pencil_bounds(rp, ci, v, brp, bci, bv, seed=1234):
    lo, hi = C.c_double(), C.c_double()
    _chk(lib().ref_pencil_bounds(*_csr_args(rp, ci, v), *_csr_b(brp, bci, bv), C.c_uint64(seed),
                                 C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def pencil_dos(rp, ci, v, brp, bci, bv, lmin, lmax, m=60, n_vec=40, npts=300, seed=1234):
    x = np.empty(npts, np.float64)
    y = np.empty(npts, np.float64)
    nev = C.c_double()
    _chk(lib().ref_pencil_dos(*_csr_args(rp, ci, v), *_csr_b(brp, bci, bv), C.c_double(lmin),
                              C.c_double(lmax), C.c_int(m), C.c_int(n_vec), C.c_int(npts),
                              C.c_uint64(seed), x.ctypes.data_as(_PD), y.ctypes.data_as(_PD),
                              C.byref(nev)))
    return x, y, nev.value


def cheb_lan_pencil_csr(rp, ci, v, brp, bci, bv, solver, xi, eta, lmin, lmax, damping="sigma",
                        res_tol=1e-8, est_count=20, seed=1234):
    """The reference's B-weighted cheb_lan_nr/tr/cheb_si on (A, B), B a general sparse SPD CSR
    (Cholesky-backed B-solves, eigensolvers.hpp:640-732)."""
    h = lib().ref_cheb_lan_pencil_csr(len(rp) - 1, rp, ci, v, brp, bci, bv, SOLVER[solver], xi, eta,
                                      lmin, lmax, DAMPING[damping], res_tol, est_count, seed)
    if not h:
        raise RefError(lib().ref_last_error().decode())
    return _collect(h, False)["slices"][0]
