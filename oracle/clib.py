"""TEST INFRASTRUCTURE ONLY: numpy-facing wrapper of the C restatement oracle/sliceeig_oracle.c.

Every function mirrors the reference function cited in the C file (header:line).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")


class OrFilter(C.Structure):
    _fields_ = [("k", C.c_int), ("gamma", C.c_double), ("ta", C.c_double), ("tb", C.c_double),
                ("bar", C.c_double), ("c", C.c_double), ("d", C.c_double),
                ("cap_reached", C.c_int)]


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE, "oracle"], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        L = C.CDLL(_SO)
        L.or_rng_vectors.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, _dp]
        L.or_laplacian_nnz.argtypes = [C.c_int, _ip]
        L.or_laplacian_nnz.restype = C.c_long
        L.or_laplacian.argtypes = [C.c_int, _ip, _ip, _ip, _dp]
        L.or_matvec.argtypes = [C.c_int, _ip, _ip, _dp, _dp, _dp]
        L.or_damping.argtypes = [C.c_int, C.c_int, _dp]
        L.or_cheb_series.argtypes = [C.c_int, _dp, C.c_double]
        L.or_cheb_series.restype = C.c_double
        L.or_eval_pol.argtypes = [C.c_int, _dp, C.c_double]
        L.or_eval_pol.restype = C.c_double
        L.or_balance_center.argtypes = [C.c_int, C.c_double, C.c_double, C.c_int,
                                        C.POINTER(C.c_double)]
        L.or_normalized_coeffs.argtypes = [C.c_int, C.c_double, C.c_int, _dp]
        L.or_find_pol.argtypes = [C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                                  C.c_int, C.c_int, C.POINTER(OrFilter), _dp]
        L.or_apply_pol.argtypes = [C.c_int, _ip, _ip, _dp, C.c_int, _dp, C.c_double, C.c_double,
                                   _dp, _dp]
        L.or_kpm_moments.argtypes = [C.c_int, _ip, _ip, _dp, C.c_double, C.c_double, C.c_int,
                                     C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_int, _dp]
        L.or_kpm_curve.argtypes = [C.c_int, _dp, C.c_int, C.c_double, C.c_double, C.c_int, _dp, _dp]
        L.or_kpm_curve.restype = C.c_double
        L.or_dos_count.argtypes = [C.c_int, C.c_int, _dp, _dp, C.c_double, C.c_double]
        L.or_dos_count.restype = C.c_double
        L.or_slice_spectrum.argtypes = [C.c_int, C.c_int, _dp, _dp, C.c_double, C.c_double, C.c_int,
                                        _dp, _dp]
        L.or_cgs_pass.argtypes = [C.c_int, C.c_int, _dp, _dp, C.c_void_p]
        L.or_paired_cgs2.argtypes = [C.c_int, C.c_int, _dp, _dp, C.c_void_p]
        L.or_laplacian_eigs_unsorted.argtypes = [C.c_int, _ip, _dp]
        _lib = L
    return _lib


DAMPING = {"none": 0, "sigma": 1, "jackson": 2}


def rng_vectors(seed: int, kind: str, n: int, count: int = 1) -> np.ndarray:
    out = np.empty(n * count, dtype=np.float64)
    lib().or_rng_vectors(seed, 1 if kind == "normal" else 0, n, count, out)
    return out.reshape(count, n)


def laplacian(dims):
    d = np.asarray(dims, dtype=np.int32)
    n = int(np.prod(d))
    nnz = lib().or_laplacian_nnz(len(d), d)
    rp = np.empty(n + 1, np.int32)
    ci = np.empty(nnz, np.int32)
    v = np.empty(nnz, np.float64)
    lib().or_laplacian(len(d), d, rp, ci, v)
    return rp, ci, v


def laplacian_eigs(dims) -> np.ndarray:
    d = np.asarray(dims, dtype=np.int32)
    out = np.empty(int(np.prod(d)), np.float64)
    lib().or_laplacian_eigs_unsorted(len(d), d, out)
    return np.sort(out, kind="stable")


def matvec(rp, ci, v, x):
    y = np.empty(len(rp) - 1, np.float64)
    lib().or_matvec(len(rp) - 1, rp, ci, v, np.ascontiguousarray(x, np.float64), y)
    return y


def damping(k: int, kind: str) -> np.ndarray:
    s = np.empty(k + 1, np.float64)
    lib().or_damping(k, DAMPING[kind], s)
    return s


def balance_center(k, ta, tb, kind):
    g = C.c_double()
    rc = lib().or_balance_center(k, ta, tb, DAMPING[kind], C.byref(g))
    if rc == -1:
        raise ValueError("balance_center: bad mapped interval")
    if rc:
        raise RuntimeError("balance_center: no balanced center found")
    return g.value


def normalized_coeffs(k, gamma, kind):
    mu = np.empty(k + 1, np.float64)
    if lib().or_normalized_coeffs(k, gamma, DAMPING[kind], mu):
        raise RuntimeError("find_pol: degenerate normalization")
    return mu


def eval_pol(mu, t):
    mu = np.ascontiguousarray(mu, np.float64)
    return lib().or_eval_pol(len(mu) - 1, mu, t)


def find_pol(xi, eta, lmin, lmax, tau=0.8, max_deg=3000, damping="sigma"):
    f = OrFilter()
    mu = np.empty(max_deg + 1, np.float64)
    rc = lib().or_find_pol(xi, eta, lmin, lmax, tau, max_deg, DAMPING[damping], C.byref(f), mu)
    if rc == -1:
        raise ValueError("find_pol: invalid interval")
    if rc:
        raise RuntimeError("find_pol: numerical failure")
    return {"k": f.k, "gamma": f.gamma, "ta": f.ta, "tb": f.tb, "bar": f.bar, "c": f.c, "d": f.d,
            "cap_reached": bool(f.cap_reached), "mu": mu[: f.k + 1].copy()}


def apply_pol(rp, ci, v, mu, c, d, x):
    out = np.empty(len(rp) - 1, np.float64)
    mu = np.ascontiguousarray(mu, np.float64)
    lib().or_apply_pol(len(rp) - 1, rp, ci, v, len(mu) - 1, mu, c, d,
                       np.ascontiguousarray(x, np.float64), out)
    return out


def kpm_moments(rp, ci, v, lmin, lmax, m, n_vec, seed, kind="rademacher", first=0, count=None):
    z = np.empty(m + 1, np.float64)
    count = n_vec if count is None else count
    lib().or_kpm_moments(len(rp) - 1, rp, ci, v, lmin, lmax, m, n_vec, seed,
                         1 if kind == "normal" else 0, first, count, z)
    return z


def kpm_curve(zeta, n, lmin, lmax, npts=300):
    zeta = np.ascontiguousarray(zeta, np.float64)
    x = np.empty(npts, np.float64)
    y = np.empty(npts, np.float64)
    nev = lib().or_kpm_curve(len(zeta) - 1, zeta, n, lmin, lmax, npts, x, y)
    if np.isnan(nev):
        raise RuntimeError("dos: vanishing density estimate")
    return x, y, nev


def dos_count(x, y, n, xi, eta):
    return lib().or_dos_count(len(x), n, np.ascontiguousarray(x), np.ascontiguousarray(y), xi, eta)


def slice_spectrum(x, y, n, xi, eta, ns):
    bp = np.empty(ns + 1, np.float64)
    est = np.empty(ns, np.float64)
    rc = lib().or_slice_spectrum(len(x), n, np.ascontiguousarray(x), np.ascontiguousarray(y),
                                 xi, eta, ns, bp, est)
    if rc == -1:
        raise ValueError("slice_spectrum: invalid argument")
    if rc:
        raise RuntimeError("slice_spectrum: curve grid too coarse")
    return bp, est


def paired_cgs2(W, t, h=None):
    """W: (k, n) rows = basis columns.  Returns (t_out, h_out, passes)."""
    W = np.ascontiguousarray(W, np.float64)
    k, n = W.shape
    t = np.array(t, np.float64, copy=True)
    hh = np.zeros(k, np.float64) if h is None else np.array(h, np.float64, copy=True)
    passes = lib().or_paired_cgs2(n, k, W.reshape(-1), t, hh.ctypes.data_as(C.c_void_p))
    return t, hh, passes
