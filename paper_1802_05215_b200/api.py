"""Python mirror of the reference's polynomial-filtering API (namespace ``sliceeig``,
/root/reference/proj/include/sliceeig/*.hpp), backed by libsliceeig_cuda.so.

Same names, argument meaning and error behaviour as the reference:
``std::invalid_argument`` -> ``ValueError``, ``std::out_of_range`` -> ``IndexError``,
``std::runtime_error`` -> ``RuntimeError``.  Everything that touches an O(n) vector runs on the
GPU through the C ABI; there is no host fallback.
"""
from __future__ import annotations

import ctypes as C
import math
import threading
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import call, lib

_PD = C.POINTER(C.c_double)
_PI = C.POINTER(C.c_int)


def _pd(a: np.ndarray):
    return a.ctypes.data_as(_PD)


def _pi(a: np.ndarray):
    return a.ctypes.data_as(_PI)


def _f64(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.float64)


# ---- device contexts -------------------------------------------------------------------------
class Context:
    """One CUDA stream + cuBLAS/cuSOLVER handles on one device (se_ctx).  One per host thread."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        call("se_ctx_create", device, C.byref(h))
        self.handle = h
        self.device = device

    def synchronize(self):
        call("se_ctx_synchronize", self.handle)

    def set_candidate_budget(self, nbytes: int):
        """Device bytes the drivers' Ritz-candidate evaluation may hold at once (default 8 GB);
        larger candidate sets are evaluated in column chunks."""
        call("se_ctx_set_candidate_budget", self.handle, int(nbytes))

    def kernel_launches(self) -> int:
        v = C.c_long()
        call("se_ctx_kernel_launches", self.handle, C.byref(v))
        return v.value

    def close(self):
        if self.handle:
            call("se_ctx_destroy", self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_tls = threading.local()


def default_context(device: Optional[int] = None) -> Context:
    dev = 0 if device is None else device
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if dev not in ctxs:
        ctxs[dev] = Context(dev)
    return ctxs[dev]


def device_count() -> int:
    v = C.c_int()
    call("se_device_count", C.byref(v))
    return v.value


def device_memory(device: int = 0) -> tuple[int, int]:
    """(free, total) bytes of a device's memory."""
    f, t = C.c_size_t(), C.c_size_t()
    call("se_device_memory", device, C.byref(f), C.byref(t))
    return f.value, t.value


# ---- matrices (csr.hpp, laplacian.hpp) ------------------------------------------------------------
class DeviceCsr:
    """A CSR matrix resident in HBM (se_csr)."""

    def __init__(self, handle, ctx: Context):
        self.handle = handle
        self.ctx = ctx
        n, nnz = C.c_int(), C.c_long()
        call("se_csr_info", handle, C.byref(n), C.byref(nnz))
        self.n, self.nnz = n.value, nnz.value

    @classmethod
    def upload(cls, a: "CsrMatrix", ctx: Optional[Context] = None) -> "DeviceCsr":
        ctx = ctx or default_context()
        h = C.c_void_p()
        call("se_csr_upload", ctx.handle, a.n, _pi(a.row_ptr), _pi(a.col_idx), _pd(a.vals),
             C.byref(h))
        return cls(h, ctx)

    @classmethod
    def laplacian(cls, dims: Sequence[int], ctx: Optional[Context] = None) -> "DeviceCsr":
        """Device generator kernel for gen_laplacian (laplacian.hpp:19-48)."""
        ctx = ctx or default_context()
        d = np.asarray(dims, np.int32)
        h = C.c_void_p()
        call("se_csr_gen_laplacian", ctx.handle, len(d), _pi(d), C.byref(h))
        return cls(h, ctx)

    def download(self) -> "CsrMatrix":
        rp = np.empty(self.n + 1, np.int32)
        ci = np.empty(self.nnz, np.int32)
        v = np.empty(self.nnz, np.float64)
        call("se_csr_download", self.ctx.handle, self.handle, _pi(rp), _pi(ci), _pd(v))
        return CsrMatrix(self.n, rp, ci, v)

    def scale_sym(self, d: np.ndarray):
        d = _f64(d)
        call("se_csr_scale_sym", self.ctx.handle, self.handle, _pd(d))

    def set_residual_weight(self, w: Optional[np.ndarray]):
        """Candidate residuals ||w .* (A u - lambda u)|| / sqrt(u.u) (None clears)."""
        wf = None if w is None else _f64(w)
        call("se_csr_set_residual_weight", self.ctx.handle, self.handle,
             _pd(wf) if wf is not None else None)

    def free(self):
        if self.handle:
            call("se_csr_free", self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class CsrMatrix:
    """Host CSR (csr.hpp:23-162): int32 row_ptr / col_idx, f64 vals, sorted unique columns."""

    def __init__(self, n: int, row_ptr, col_idx, vals):
        self.n = int(n)
        self.row_ptr = np.ascontiguousarray(row_ptr, np.int32)
        self.col_idx = np.ascontiguousarray(col_idx, np.int32)
        self.vals = _f64(vals)
        self._dev = {}

    @property
    def nnz(self) -> int:
        return int(self.vals.size)

    @staticmethod
    def from_triplets(n: int, rows, cols, vals) -> "CsrMatrix":
        """csr.hpp:29-58: sort by (row, col), sum duplicates (in input order), drop zeros."""
        if n < 0:
            raise ValueError("CsrMatrix: negative dimension")
        r = np.asarray(rows, np.int64)
        c = np.asarray(cols, np.int64)
        v = np.asarray(vals, np.float64)
        if r.size and (r.min() < 0 or r.max() >= n or c.min() < 0 or c.max() >= n):
            raise IndexError("CsrMatrix: triplet index out of range")
        order = np.lexsort((c, r))  # stable: equal keys keep input order, as std::sort groups them
        r, c, v = r[order], c[order], v[order]
        key = r * max(n, 1) + c
        starts = np.flatnonzero(np.r_[True, key[1:] != key[:-1]]) if key.size else np.array([], int)
        sums = np.empty(starts.size, np.float64)
        for q, s in enumerate(starts):  # sequential sum in sorted order
            e = starts[q + 1] if q + 1 < starts.size else key.size
            acc = v[s]
            for t in range(s + 1, e):
                acc += v[t]
            sums[q] = acc
        keep = sums != 0.0
        rr, cc, vv = r[starts][keep], c[starts][keep], sums[keep]
        rp = np.zeros(n + 1, np.int64)
        np.add.at(rp, rr + 1, 1)
        return CsrMatrix(n, np.cumsum(rp).astype(np.int32), cc.astype(np.int32), vv)

    @staticmethod
    def diag(d) -> "CsrMatrix":
        d = _f64(d)
        idx = np.arange(d.size)
        return CsrMatrix.from_triplets(d.size, idx, idx, d)

    @staticmethod
    def identity(n: int) -> "CsrMatrix":
        return CsrMatrix.diag(np.ones(n))

    @staticmethod
    def tridiag_toeplitz(n: int, e: float, d: float) -> "CsrMatrix":
        rows, cols, vals = [], [], []
        for i in range(n):
            if i > 0:
                rows.append(i); cols.append(i - 1); vals.append(e)
            rows.append(i); cols.append(i); vals.append(d)
            if i < n - 1:
                rows.append(i); cols.append(i + 1); vals.append(e)
        return CsrMatrix.from_triplets(n, rows, cols, vals)

    def device(self, ctx: Optional[Context] = None) -> DeviceCsr:
        ctx = ctx or default_context()
        key = id(ctx)
        if key not in self._dev:
            self._dev[key] = DeviceCsr.upload(self, ctx)
        return self._dev[key]

    def matvec(self, x) -> np.ndarray:
        """y = A x on the GPU (csr.hpp:98-105; bit-identical row sums)."""
        x = _f64(x)
        if x.size != self.n:
            raise ValueError("matvec: size mismatch")
        y = np.empty(self.n, np.float64)
        d = self.device()
        call("se_spmv", d.ctx.handle, d.handle, _pd(x), _pd(y))
        return y

    def to_dense(self) -> np.ndarray:
        A = np.zeros((self.n, self.n))
        for i in range(self.n):
            for p in range(self.row_ptr[i], self.row_ptr[i + 1]):
                A[i, self.col_idx[p]] = self.vals[p]
        return A


def gen_laplacian(dims: Sequence[int]) -> CsrMatrix:
    """laplacian.hpp:19-48 (host closed form, bit-identical to the reference's CSR)."""
    d = np.asarray(list(dims), np.int32)
    if d.size == 0 or d.size > 3:
        raise ValueError("gen_laplacian: need 1 to 3 grid dimensions")
    n, nnz = C.c_int(), C.c_long()
    call("se_laplacian_host", len(d), _pi(d), C.byref(n), C.byref(nnz), None, None, None)
    rp = np.empty(n.value + 1, np.int32)
    ci = np.empty(nnz.value, np.int32)
    v = np.empty(nnz.value, np.float64)
    call("se_laplacian_host", len(d), _pi(d), C.byref(n), C.byref(nnz), _pi(rp), _pi(ci), _pd(v))
    return CsrMatrix(n.value, rp, ci, v)


def gen_random_sparse(n: int, seed: int = 1234, halfband: int = 3, extras: int = 8,
                      diag_frac: float = 0.1) -> CsrMatrix:
    """BASELINE cfg4 generator (random banded + extras, symmetric; see sliceeig_cuda.h)."""
    nnz = C.c_long()
    call("se_gen_random_sparse", n, seed, halfband, extras, diag_frac, C.byref(nnz), None, None, None)
    rp = np.empty(n + 1, np.int32)
    ci = np.empty(nnz.value, np.int32)
    v = np.empty(nnz.value, np.float64)
    call("se_gen_random_sparse", n, seed, halfband, extras, diag_frac, C.byref(nnz), _pi(rp), _pi(ci),
         _pd(v))
    return CsrMatrix(n, rp, ci, v)


def mass_scaling(n: int, seed: int = 1234):
    """BASELINE cfg5: lumped mass b_i = 0.5 + uniform (Rng(seed)), d = b^-1/2."""
    b = np.empty(n)
    d = np.empty(n)
    call("se_mass_scaling", n, seed, _pd(b), _pd(d))
    return b, d


def scale_sym_host(a: CsrMatrix, d) -> CsrMatrix:
    """Host D A D (vals[p] = (a_ij d_i) d_j), the reference of DeviceCsr.scale_sym."""
    d = _f64(d)
    rows = np.repeat(np.arange(a.n), np.diff(a.row_ptr))
    return CsrMatrix(a.n, a.row_ptr, a.col_idx, (a.vals * d[rows]) * d[a.col_idx])


def laplacian_analytic_eigs(dims: Sequence[int]) -> np.ndarray:
    """laplacian.hpp:51-86."""
    d = np.asarray(list(dims), np.int32)
    if d.size == 0 or d.size > 3:
        raise ValueError("laplacian_analytic_eigs: need 1 to 3 grid dimensions")
    out = np.empty(int(np.prod(d.astype(np.int64))) if (d > 0).all() else 0, np.float64)
    call("se_laplacian_eigs", len(d), _pi(d), _pd(out))
    return out


def count_in_interval(sorted_vals, lo: float, hi: float) -> int:
    """laplacian.hpp:89-93 (closed interval)."""
    s = np.asarray(sorted_vals)
    return int(np.searchsorted(s, hi, side="right") - np.searchsorted(s, lo, side="left"))


# ---- operators / counters (operators.hpp) -----------------------------------------------------------
@dataclass
class Counters:
    n_A_matvec: int = 0
    n_B_matvec: int = 0
    n_B_solve: int = 0
    n_shift_solve: int = 0
    t_mv: float = 0.0
    t_orth: float = 0.0
    t_sv: float = 0.0
    t_total: float = 0.0


@dataclass
class Operator:
    """make_operator(a) (operators.hpp:34-36): the CSR-backed operator the device path consumes."""
    n: int
    csr: CsrMatrix


def make_operator(a: CsrMatrix) -> Operator:
    return Operator(a.n, a)


def _dev(op) -> DeviceCsr:
    if isinstance(op, DeviceCsr):
        return op
    if isinstance(op, Operator):
        return op.csr.device()
    if isinstance(op, CsrMatrix):
        return op.device()
    raise TypeError("expected CsrMatrix, Operator or DeviceCsr (matrix-free operators are not "
                    "supported on the device path)")


# ---- filters (filter_poly.hpp) ---------------------------------------------------------------------
@dataclass
class SpectralBounds:
    lmin: float = 0.0
    lmax: float = 0.0


@dataclass
class PolyOpts:
    tau: float = 0.8
    max_deg: int = 3000
    damping: str = "sigma"


@dataclass
class PolynomialFilter:
    k: int = 0
    gamma: float = 0.0
    mu: np.ndarray = field(default_factory=lambda: np.zeros(0))
    c: float = 0.0
    d: float = 1.0
    tau: float = 0.8
    ta: float = -1.0
    tb: float = 1.0
    bar: float = 0.0
    damping: str = "sigma"
    cap_reached: bool = False

    def to_ref(self, lam: float) -> float:
        return (lam - self.c) / self.d

    def _c(self):
        mu = _f64(self.mu)
        s = _lib.SePolyFilter(self.k, self.gamma, self.c, self.d, self.tau, self.ta, self.tb,
                              self.bar, _lib.DAMPING[self.damping], int(self.cap_reached),
                              _pd(mu), mu.size)
        return s, mu  # keep mu alive


def damping_multipliers(k: int, kind: str) -> np.ndarray:
    out = np.empty(k + 1, np.float64)
    call("se_damping_multipliers", k, _lib.DAMPING[kind], _pd(out))
    return out


def chebyshev_coeffs(gamma: float, k: int) -> np.ndarray:
    out = np.empty(max(k + 1, 1), np.float64)
    call("se_chebyshev_coeffs", gamma, k, _pd(out))
    return out


def normalized_filter_coeffs(k: int, gamma: float, kind: str) -> np.ndarray:
    out = np.empty(k + 1, np.float64)
    call("se_normalized_filter_coeffs", k, gamma, _lib.DAMPING[kind], _pd(out))
    return out


def balance_center(k: int, ta: float, tb: float, kind: str) -> float:
    g = C.c_double()
    call("se_balance_center", k, ta, tb, _lib.DAMPING[kind], C.byref(g))
    return g.value


def find_pol(xi: float, eta: float, bounds: SpectralBounds, opts: PolyOpts = PolyOpts()
             ) -> PolynomialFilter:
    """filter_poly.hpp:198-253."""
    mu = np.empty(opts.max_deg + 1 if opts.max_deg >= 2 else 3, np.float64)
    s = _lib.SePolyFilter(0, 0.0, 0.0, 1.0, 0.8, -1.0, 1.0, 0.0, 0, 0, _pd(mu), mu.size)
    call("se_find_pol", xi, eta, bounds.lmin, bounds.lmax, opts.tau, opts.max_deg,
         _lib.DAMPING[opts.damping], C.byref(s))
    return PolynomialFilter(s.k, s.gamma, mu[: s.k + 1].copy(), s.c, s.d, s.tau, s.ta, s.tb, s.bar,
                            opts.damping, bool(s.cap_reached))


def eval_pol(f: PolynomialFilter, t: float) -> float:
    s, _keep = f._c()
    out = C.c_double()
    call("se_eval_pol", C.byref(s), t, C.byref(out))
    return out.value


def apply_pol(f: PolynomialFilter, op, v, counters: Optional[Counters] = None) -> np.ndarray:
    """out = rho(Ahat) v on the GPU (filter_poly.hpp:256-277): exactly k A-products, bitwise the
    reference's result.  v may be (n,) or (nvec, n)."""
    d = _dev(op)
    V = _f64(v)
    nvec = 1 if V.ndim == 1 else V.shape[0]
    if V.size != d.n * nvec:
        raise ValueError("apply_pol: size mismatch")
    out = np.empty_like(V)
    s, _keep = f._c()
    nmv = C.c_long(0)
    call("se_cheb_apply", d.ctx.handle, d.handle, C.byref(s), nvec, _pd(V), _pd(out), C.byref(nmv))
    if counters is not None:
        counters.n_A_matvec += nmv.value
    return out


# ---- density of states (dos.hpp) / slicing (slicer.hpp) ----------------------------------------------
@dataclass
class DosConfig:
    method: str = "kpm"
    m: int = 60
    n_vec: int = 40
    npts: int = 300
    gaussian_sigma: float = 0.0
    seed: int = 1234
    probes: str = "rademacher"  # extension for BASELINE cfg2 ("gaussian"); reference: Rademacher


@dataclass
class DosCurve:
    xdos: np.ndarray
    ydos: np.ndarray
    nev_est: float
    n: int


def kpm_moments(op, bounds: SpectralBounds, m: int, n_vec: int, seed: int = 1234,
                probes: str = "rademacher", first: int = 0, count: Optional[int] = None
                ) -> np.ndarray:
    """Unnormalised moment sums over probes [first, first+count) (dos.hpp:96-109) on the GPU."""
    d = _dev(op)
    count = n_vec - first if count is None else count
    z = np.empty(m + 1, np.float64)
    call("se_kpm_moments", d.ctx.handle, d.handle, bounds.lmin, bounds.lmax, m, n_vec,
         _lib.PROBES[probes], seed, first, count, _pd(z))
    return z


def kpm_moments_probes(op, bounds: SpectralBounds, m: int, n_vec: int, seed: int = 1234,
                       probes: str = "rademacher", first: int = 0, count: Optional[int] = None
                       ) -> np.ndarray:
    """Per-probe moments (count, m+1) for probes [first, first+count) of the Rng(seed) stream."""
    d = _dev(op)
    count = n_vec - first if count is None else count
    out = np.empty((max(count, 1), m + 1), np.float64)
    call("se_kpm_moments_probes", d.ctx.handle, d.handle, bounds.lmin, bounds.lmax, m, n_vec,
         _lib.PROBES[probes], seed, first, count, _pd(out))
    return out[:count]


def kpm_curve(zeta_normalised, n: int, bounds: SpectralBounds, npts: int = 300) -> DosCurve:
    z = _f64(zeta_normalised)
    x = np.empty(npts, np.float64)
    y = np.empty(npts, np.float64)
    nev = C.c_double()
    call("se_kpm_curve", z.size - 1, _pd(z), n, bounds.lmin, bounds.lmax, npts, _pd(x), _pd(y),
         C.byref(nev))
    return DosCurve(x, y, nev.value, n)


def kpm_dos(op, bounds: SpectralBounds, cfg: DosConfig = DosConfig()) -> DosCurve:
    """dos.hpp:82-132."""
    d = _dev(op)
    x = np.empty(max(cfg.npts, 0), np.float64)
    y = np.empty(max(cfg.npts, 0), np.float64)
    nev = C.c_double()
    call("se_kpm_dos", d.ctx.handle, d.handle, bounds.lmin, bounds.lmax, cfg.m, cfg.n_vec, cfg.npts,
         cfg.seed, _lib.PROBES[cfg.probes], _pd(x), _pd(y), C.byref(nev))
    return DosCurve(x, y, nev.value, d.n)


def _one_nccl_per_process():
    """The library resolves NCCL at run time and reuses a copy already in the process.  torch
    links its own NCCL under the same soname, so import torch (when present) first: its copy is
    then the one both use, instead of a system copy shadowing it for a later torch import."""
    try:
        import torch  # noqa: F401
    except ImportError:
        pass


def kpm_dos_devices(a: "CsrMatrix", bounds: SpectralBounds, cfg: DosConfig,
                    devices: Sequence[int]) -> DosCurve:
    """kpm_dos (dos.hpp:82-132) with the probes split over several GPUs of this process and the
    per-probe moments combined by one NCCL all-reduce (se_kpm_dos_multi); bit-identical to
    kpm_dos on one GPU."""
    _one_nccl_per_process()
    devs = np.ascontiguousarray(devices, np.int32)
    x = np.empty(max(cfg.npts, 0), np.float64)
    y = np.empty(max(cfg.npts, 0), np.float64)
    nev = C.c_double()
    call("se_kpm_dos_multi", int(devs.size), _pi(devs), a.n, _pi(a.row_ptr), _pi(a.col_idx),
         _pd(a.vals), bounds.lmin, bounds.lmax, cfg.m, cfg.n_vec, cfg.npts, cfg.seed,
         _lib.PROBES[cfg.probes], _pd(x), _pd(y), C.byref(nev))
    return DosCurve(x, y, nev.value, a.n)


def nccl_version() -> int:
    """The NCCL the library resolves at run time (e.g. 22809), or raises when absent."""
    _one_nccl_per_process()
    v = C.c_int()
    call("se_nccl_version", C.byref(v))
    return v.value


def lan_dos(op, bounds: SpectralBounds, cfg: DosConfig = DosConfig()) -> DosCurve:
    """dos.hpp:136-154."""
    d = _dev(op)
    x = np.empty(max(cfg.npts, 0), np.float64)
    y = np.empty(max(cfg.npts, 0), np.float64)
    nev = C.c_double()
    call("se_lan_dos", d.ctx.handle, d.handle, bounds.lmin, bounds.lmax, cfg.m, cfg.n_vec, cfg.npts,
         cfg.gaussian_sigma, cfg.seed, _pd(x), _pd(y), C.byref(nev))
    return DosCurve(x, y, nev.value, d.n)


def ls_pol_approx(fun: str, bounds: SpectralBounds, tol: float, max_deg: int = 300):
    """cheb_approx.hpp:40-88: Chebyshev least-squares fit of 1/t ("inverse") or 1/sqrt(t)
    ("inverse_sqrt") on bounds.  Returns (coefficients, achieved relative error)."""
    co = np.empty(max_deg + 1)
    deg, ach = C.c_int(), C.c_double()
    call("se_ls_pol_approx", 1 if fun == "inverse_sqrt" else 0, bounds.lmin, bounds.lmax, tol,
         max_deg, max_deg + 1, C.byref(deg), _pd(co), C.byref(ach))
    return co[: deg.value + 1].copy(), ach.value


def apply_cheb(coeff, bounds: SpectralBounds, b, v) -> np.ndarray:
    """cheb_approx.hpp:91-112: y = p(B) v (v: n or n x k), on the GPU."""
    d = _dev(b)
    co = _f64(coeff)
    v = np.asarray(v, np.float64)
    vv = np.asfortranarray(v.reshape(d.n, -1))
    out = np.empty_like(vv, order="F")
    call("se_apply_cheb", d.ctx.handle, d.handle, bounds.lmin, bounds.lmax, co.size - 1, _pd(co),
         vv.shape[1], vv.ctypes.data_as(_PD), out.ctypes.data_as(_PD))
    return out.reshape(v.shape)


def lan_tr_bounds_pencil(a, b, tol: float = 1e-4, restart_dim: int = 60, max_restarts: int = 40,
                         seed: int = 1234) -> SpectralBounds:
    """lan_tr_bounds(op_a, {B, B-solve}, ...) (lanczos.hpp:148-277) for a general SPD B."""
    d = _dev(a)
    pen = Pencil(b, d.ctx)
    try:
        lo, hi = C.c_double(), C.c_double()
        call("se_lan_tr_bounds_pencil", d.ctx.handle, d.handle, pen.handle, tol, restart_dim,
             max_restarts, seed, C.byref(lo), C.byref(hi))
        return SpectralBounds(lo.value, hi.value)
    finally:
        pen.close()


def dos_generalized(a, b, bounds: SpectralBounds, cfg: DosConfig = DosConfig()) -> DosCurve:
    """dos.hpp:160-184: the Lanczos density of the pencil (A, B), B sparse SPD."""
    d = _dev(a)
    pen = Pencil(b, d.ctx)
    try:
        x = np.empty(max(cfg.npts, 0))
        y = np.empty(max(cfg.npts, 0))
        nev = C.c_double()
        call("se_lan_dos_pencil", d.ctx.handle, d.handle, pen.handle, bounds.lmin, bounds.lmax,
             cfg.m, cfg.n_vec, cfg.npts, cfg.gaussian_sigma, cfg.seed, _pd(x), _pd(y), C.byref(nev))
        return DosCurve(x, y, nev.value, d.n)
    finally:
        pen.close()


def dos_count(c: DosCurve, xi: float, eta: float) -> float:
    """dos.hpp:212-218."""
    out = C.c_double()
    x, y = _f64(c.xdos), _f64(c.ydos)
    call("se_dos_count", x.size, c.n, _pd(x), _pd(y), xi, eta, C.byref(out))
    return out.value


@dataclass
class SliceSet:
    breakpoints: np.ndarray
    est_counts: np.ndarray

    def ns(self) -> int:
        return len(self.breakpoints) - 1


def slice_spectrum(c: DosCurve, xi: float, eta: float, ns: int) -> SliceSet:
    """slicer.hpp:18-64."""
    x, y = _f64(c.xdos), _f64(c.ydos)
    bp = np.empty(max(ns + 1, 1), np.float64)
    est = np.empty(max(ns, 1), np.float64)
    call("se_slice_spectrum", x.size, c.n, _pd(x), _pd(y), xi, eta, ns, _pd(bp), _pd(est))
    return SliceSet(bp, est[:ns])


# ---- Krylov building blocks (lanczos.hpp, orth.hpp, tridiag_eig.hpp, dense_eig.hpp) -----------------
def lan_tr_bounds(op, tol: float, restart_dim: int, max_restarts: int = 40, seed: int = 1234
                  ) -> SpectralBounds:
    """lanczos.hpp:148-277 (euclidean inner product)."""
    d = _dev(op)
    lo, hi = C.c_double(), C.c_double()
    call("se_lan_tr_bounds", d.ctx.handle, d.handle, tol, restart_dim, max_restarts, seed,
         C.byref(lo), C.byref(hi))
    return SpectralBounds(lo.value, hi.value)


@dataclass
class LanczosState:
    alpha: np.ndarray
    beta: np.ndarray
    steps: int
    breakdown: bool
    next_beta: float
    next_w: Optional[np.ndarray]
    basis: Optional[np.ndarray]  # (steps, n): row j = basis column j


def lanczos_run(op, start, m: int, want_basis: bool = False) -> LanczosState:
    """lanczos.hpp:37-118 (euclidean)."""
    d = _dev(op)
    s = _f64(start)
    if s.size != d.n:
        raise ValueError("lanczos_run: bad start vector size")
    mm = min(m, d.n)
    alpha = np.zeros(max(mm, 1))
    beta = np.zeros(max(mm, 1))
    nw = np.zeros(d.n)
    basis = np.zeros((max(mm, 1), d.n)) if want_basis else None
    steps, brk = C.c_int(), C.c_int()
    nb = C.c_double()
    call("se_lanczos_run", d.ctx.handle, d.handle, _pd(s), m, _pd(alpha), _pd(beta), C.byref(steps),
         C.byref(brk), C.byref(nb), _pd(nw), _pd(basis) if want_basis else None)
    k = steps.value
    return LanczosState(alpha[:k].copy(), beta[: max(k - 1, 0)].copy(), k, bool(brk.value),
                        nb.value, None if brk.value else nw,
                        basis[:k].copy() if want_basis else None)


def paired_cgs2(t, W, h=None, ctx: Optional[Context] = None):
    """orth.hpp:70-80 on the GPU.  W: (k, n) rows = basis columns.  Returns (t, h)."""
    ctx = ctx or default_context()
    W = _f64(W)
    k, n = (0, np.asarray(t).size) if W.size == 0 else W.shape
    tt = np.array(t, np.float64, copy=True)
    hh = np.zeros(max(k, 1)) if h is None else np.array(h, np.float64, copy=True)
    call("se_paired_cgs2", ctx.handle, n, k, _pd(W) if k else None, _pd(tt), _pd(hh))
    return tt, hh[:k]


def sym_tridiag_eig(alpha, beta, want_vectors: bool = True):
    """tridiag_eig.hpp:111-131.  Returns (values, vectors[:, j])."""
    a = _f64(alpha)
    b = _f64(beta) if a.size > 1 else np.zeros(1)
    m = a.size
    vals = np.empty(m)
    vecs = np.empty((m, m)) if want_vectors else None
    call("se_sym_tridiag_eig", m, _pd(a), _pd(b), int(want_vectors), _pd(vals),
         _pd(vecs) if want_vectors else None)
    return vals, (vecs.T.copy() if want_vectors else None)


def dense_sym_eig(A, want_vectors: bool = True, size_guard: int = 5000):
    """dense_eig.hpp:114-139.  Returns (values, vectors[:, j])."""
    A = np.asfortranarray(A, np.float64)
    m = A.shape[0]
    vals = np.empty(m)
    vecs = np.empty((m, m)) if want_vectors else None
    call("se_dense_sym_eig", m, A.ctypes.data_as(_PD), int(want_vectors), size_guard, _pd(vals),
         _pd(vecs) if want_vectors else None)
    return vals, (vecs.T.copy() if want_vectors else None)


# ---- slice drivers (eigensolvers.hpp) ----------------------------------------------------------------
@dataclass
class SolverConfig:
    m: int = 0
    max_its: int = 0
    ncycle: int = 30
    tau1: float = 0.0
    res_tol: float = 1e-8
    est_count: int = 20
    seed: int = 1234


@dataclass
class DeflationSet:
    u: np.ndarray  # (n, k) column-major semantics: u[:, j]
    values: np.ndarray

    def count(self) -> int:
        return 0 if self.u is None else self.u.shape[1]


@dataclass
class OrthStats:
    """Reorthogonalisation accounting of a device slice solve (extension, measurement only)."""
    passes: int = 0
    cols: int = 0
    bytes: float = 0.0


@dataclass
class EigenResults:
    eigenvalues: np.ndarray
    vectors: Optional[np.ndarray]  # (n, nev): column i pairs with eigenvalues[i]
    residuals: np.ndarray
    niter: int
    counters: Counters
    hit_max_its: bool
    orth: OrthStats = field(default_factory=OrthStats)
    sample_index: Optional[np.ndarray] = None    # with want_vectors=False and SAMPLE_VECTORS > 0
    sample_vectors: Optional[np.ndarray] = None  # (n, len(sample_index))


def _host_buffer(shape):
    """Page-locked host array when torch is importable (D2H of eigenvectors at PCIe speed), else
    an ordinary numpy array."""
    try:
        import torch
        if torch.cuda.is_available():
            return torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()
    except Exception:
        pass
    return np.empty(shape, np.float64)


def _cheb_lan(solver: int, a, b, f: PolynomialFilter, xi, eta, cfg: SolverConfig,
              locked: Optional[DeflationSet], want_vectors: bool) -> EigenResults:
    who = "cheb_lan_tr" if solver == 1 else "cheb_lan_nr"
    d = _dev(a)
    if b is not None:
        return _cheb_lan_pencil(solver, a, d, b, f, xi, eta, cfg, locked, want_vectors, who)
    s, _keep = f._c()
    c = _lib.SeSolverCfg(cfg.m, cfg.max_its, cfg.ncycle, cfg.tau1, cfg.res_tol, cfg.est_count,
                         cfg.seed)
    nd = 0
    du = dv = None
    if locked is not None and locked.count() > 0:
        if locked.u.shape[0] != d.n:
            raise ValueError(f"{who}: deflation size mismatch")
        if len(locked.values) != locked.u.shape[1]:
            raise ValueError(f"{who}: deflation values/vectors mismatch")
        nd = locked.u.shape[1]
        du = np.asfortranarray(locked.u, np.float64)
        dv = _f64(locked.values)
    h = C.c_void_p()
    call("se_cheb_lan", d.ctx.handle, d.handle, C.byref(s), xi, eta, C.byref(c), solver, nd,
         du.ctypes.data_as(_PD) if nd else None, _pd(dv) if nd else None, int(want_vectors),
         C.byref(h))
    return _collect_results(h, d, want_vectors)


def _pencil_diag(b, n: int, who: str) -> np.ndarray:
    """The diagonal of an SPD diagonal B (CsrMatrix or DeviceCsr); anything else raises."""
    if getattr(b, "n", n) != n:
        raise ValueError(f"{who}: pencil size mismatch")
    hb = b.download() if isinstance(b, DeviceCsr) else b
    rp, ci, v = np.asarray(hb.row_ptr), np.asarray(hb.col_idx), np.asarray(hb.vals, np.float64)
    if not (np.all(np.diff(rp) == 1) and np.array_equal(ci, np.arange(n)) and np.all(v > 0.0)):
        raise ValueError(f"{who}: generalized pencils need a diagonal SPD B on the device path")
    return v.copy()


def _pencil_scaled(a, d, b, who, solve, want_vectors=True):
    """(A, B) with diagonal SPD B = D^-2: `solve(S, dsc)` on the standard matrix D A D (a scaled
    device copy); its eigenpairs (lambda, y) give the pencil's (lambda, D y), B-normalised, with
    residuals reported as the reference's ||A x - lambda B x|| (eigensolvers.hpp:289-316).  The
    reference runs its B-weighted recurrence with Cholesky solves of B (eigensolvers.hpp:640-690);
    a non-diagonal B would need a sparse Cholesky, outside the device path."""
    bd = _pencil_diag(b, d.n, who)
    dsc = 1.0 / np.sqrt(bd)
    host = a if isinstance(a, CsrMatrix) else (a.csr if isinstance(a, Operator) else d.download())
    S = DeviceCsr.upload(host, d.ctx)
    try:
        S.scale_sym(dsc)
        # candidates are judged (and reported) on the pencil residual
        # ||A x - lambda B x|| / sqrt(x'Bx) = ||D^-1 (S y - lambda y)|| / sqrt(y'y), x = D y
        S.set_residual_weight(np.sqrt(bd))
        r = solve(S, dsc)
    finally:
        S.free()
    x = r.vectors * dsc[:, None] if (want_vectors and r.vectors is not None) else None
    return EigenResults(r.eigenvalues, x, r.residuals, r.niter, r.counters, r.hit_max_its, r.orth)


def _is_diagonal(b, n: int) -> bool:
    hb = b.download() if isinstance(b, DeviceCsr) else b
    rp, ci = np.asarray(hb.row_ptr), np.asarray(hb.col_idx)
    return bool(np.all(np.diff(rp) == 1) and np.array_equal(ci, np.arange(n)))


class Pencil:
    """A general SPD-B pencil on the device (se_pencil): B's spectrum, the Chebyshev fit
    P ~ B^-1/2 (ls_pol_approx, cheb_approx.hpp:40-88) used to solve S = P A P."""

    def __init__(self, b, ctx: Optional[Context] = None, tol: float = 0.0, max_deg: int = 0):
        ctx = ctx or default_context()
        self.B = b if isinstance(b, DeviceCsr) else DeviceCsr.upload(b, ctx)
        self._owns = not isinstance(b, DeviceCsr)
        h = C.c_void_p()
        call("se_pencil_create", self.B.ctx.handle, self.B.handle, tol, max_deg, C.byref(h))
        self.handle = h
        deg, lo, hi, ach = C.c_int(), C.c_double(), C.c_double(), C.c_double()
        call("se_pencil_info", h, C.byref(deg), C.byref(lo), C.byref(hi), C.byref(ach))
        self.degree, self.bmin, self.bmax, self.achieved = deg.value, lo.value, hi.value, ach.value

    def close(self):
        if getattr(self, "handle", None):
            call("se_pencil_free", self.handle)
            self.handle = None
        if getattr(self, "_owns", False) and self.B is not None:
            self.B.free()
            self.B = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _cheb_lan_general_pencil(solver, d, b, f, xi, eta, cfg, locked, want_vectors, who):
    if locked is not None and locked.count() > 0:
        raise ValueError(f"{who}: a preloaded deflation set is not supported for a non-diagonal B")
    pen = Pencil(b, d.ctx)
    try:
        s, _keep = f._c()
        c = _lib.SeSolverCfg(cfg.m, cfg.max_its, cfg.ncycle, cfg.tau1, cfg.res_tol, cfg.est_count,
                             cfg.seed)
        h = C.c_void_p()
        call("se_cheb_lan_pencil", d.ctx.handle, d.handle, pen.handle, C.byref(s), xi, eta,
             C.byref(c), solver, C.byref(h))
        return _collect_results(h, d, want_vectors)
    finally:
        pen.close()


def _cheb_lan_pencil(solver, a, d, b, f, xi, eta, cfg, locked, want_vectors, who):
    if getattr(b, "n", d.n) != d.n:
        raise ValueError(f"{who}: pencil size mismatch")
    if not _is_diagonal(b, d.n):  # general SPD B: S = P A P with P ~ B^-1/2 on the device
        return _cheb_lan_general_pencil(solver, d, b, f, xi, eta, cfg, locked, want_vectors, who)

    def solve(S, dsc):
        ly = None
        if locked is not None and locked.count() > 0:  # locked pencil vectors x -> y = D^-1 x
            ly = DeflationSet(np.asarray(locked.u, np.float64) / dsc[:, None], locked.values)
        return _cheb_lan(solver, S, None, f, xi, eta, cfg, ly, want_vectors)
    return _pencil_scaled(a, d, b, who, solve, want_vectors)


def _d_matvec(d: "DeviceCsr", x) -> np.ndarray:
    """y = A x on the GPU (csr.hpp:98-105)."""
    x = _f64(x)
    y = np.empty(d.n)
    call("se_spmv", d.ctx.handle, d.handle, _pd(x), _pd(y))
    return y


# With want_vectors=False a driver still returns this many evenly spaced eigenvectors
# (EigenResults.sample_index / sample_vectors) for spot checks of results too large to download
# whole (SURVEY.md §8c, cfg4/cfg5 at full size).  0: none.
SAMPLE_VECTORS = 0


def set_resident_filter(on) -> None:
    """Process-wide switch of the resident (one launch for all degrees) filter; results are
    bit-identical either way.  Default on."""
    call("se_resident_filter", int(on))


def resident_tiles(d) -> int:
    """Row tiles of the matrix' resident-filter plan (0: the per-degree kernels run)."""
    t = C.c_int()
    call("se_csr_resident_tiles", _dev(d).handle, C.byref(t))
    return t.value


def resident_tile_smem(d) -> int:
    """Shared-memory bytes one tile of the resident filter holds (0: no plan)."""
    b = C.c_size_t()
    call("se_csr_resident_smem", _dev(d).handle, C.byref(b))
    return int(b.value)


def mult_cols(a: np.ndarray, b: np.ndarray, a_rowmajor: bool = True, ctx=None) -> np.ndarray:
    """out = A @ B on the GPU's fp64 tensor cores (mult_cols vecops.hpp:81-89; the Ritz
    combination U = W Y of eigensolvers.hpp:275-283).  a: (m, k) C-contiguous (the row-major
    Krylov-basis layout) or, with a_rowmajor=False, F-contiguous; b: (k, n), returned (m, n)."""
    ctx = ctx or default_context(0)
    a = np.asarray(a, np.float64)
    m, k = a.shape
    a = np.ascontiguousarray(a) if a_rowmajor else np.asfortranarray(a)
    bf = np.asfortranarray(np.asarray(b, np.float64))
    n = bf.shape[1]
    out = np.empty((m, n), order="F")
    call("se_mult_cols", ctx.handle, m, n, k, a.ctypes.data_as(_PD), k if a_rowmajor else m,
         int(a_rowmajor), bf.ctypes.data_as(_PD), k, out.ctypes.data_as(_PD), m, 0, None)
    return out


def mult_cols_bench(m: int, n: int, k: int, a_rowmajor: bool = True, reps: int = 5, ctx=None) -> float:
    """Mean device milliseconds of one (m x k)(k x n) Ritz contraction on synthetic operands."""
    ctx = ctx or default_context(0)
    ms = C.c_double()
    dummy = np.zeros(1)
    call("se_mult_cols", ctx.handle, m, n, k, None, k + (k & 1) if a_rowmajor else m, int(a_rowmajor),
         None, k, dummy.ctypes.data_as(_PD), m, reps, C.byref(ms))
    return ms.value


def _collect_results(h, d, want_vectors: bool) -> "EigenResults":
    sample_idx, sample_vecs = None, None
    try:
        nev = C.c_int()
        call("se_results_count", h, C.byref(nev))
        k = nev.value
        vals = np.empty(k)
        res = np.empty(k)
        vecs = _host_buffer((k, d.n)) if (want_vectors and k) else None
        call("se_results_copy", h, _pd(vals) if k else None, _pd(res) if k else None,
             _pd(vecs) if vecs is not None else None)
        if not want_vectors and SAMPLE_VECTORS > 0 and k:
            sample_idx = np.unique(np.linspace(0, k - 1, min(k, SAMPLE_VECTORS)).astype(np.int64))
            sample_vecs = np.empty((sample_idx.size, d.n))
            for q, j in enumerate(sample_idx):
                call("se_results_vector", h, int(j), _pd(sample_vecs[q]))
        niter, hit = C.c_long(), C.c_int()
        cn = _lib.SeCounters()
        call("se_results_info", h, C.byref(niter), C.byref(hit), C.byref(cn))
        op, oc, ob = C.c_longlong(), C.c_longlong(), C.c_double()
        call("se_results_orth", h, C.byref(op), C.byref(oc), C.byref(ob))
    finally:
        call("se_results_free", h)
    counters = Counters(cn.n_A_matvec, cn.n_B_matvec, cn.n_B_solve, cn.n_shift_solve, cn.t_mv,
                        cn.t_orth, cn.t_sv, cn.t_total)
    return EigenResults(vals, vecs.T if vecs is not None else (np.zeros((d.n, 0)) if want_vectors else None),
                        res, niter.value, counters, bool(hit.value),
                        OrthStats(op.value, oc.value, ob.value), sample_idx,
                        sample_vecs.T if sample_vecs is not None else None)


def cheb_si(a, b, f: PolynomialFilter, xi: float, eta: float, est_count: int,
            cfg: SolverConfig = SolverConfig(), want_vectors: bool = True) -> EigenResults:
    """Filtered subspace iteration on a block of ceil(1.3 est_count) + 8 vectors
    (eigensolvers.hpp:760-940); raises RuntimeError when the block saturates above the bar."""
    d = _dev(a)
    if b is not None:  # diagonal SPD B: the scaled standard problem (_pencil_scaled)
        return _pencil_scaled(a, d, b, "cheb_si",
                              lambda S, dsc: cheb_si(S, None, f, xi, eta, est_count, cfg,
                                                     want_vectors),
                              want_vectors)
    s, _keep = f._c()
    c = _lib.SeSolverCfg(cfg.m, cfg.max_its, cfg.ncycle, cfg.tau1, cfg.res_tol, cfg.est_count, cfg.seed)
    h = C.c_void_p()
    call("se_cheb_si", d.ctx.handle, d.handle, C.byref(s), xi, eta, int(est_count), C.byref(c), C.byref(h))
    return _collect_results(h, d, want_vectors)


def cheb_lan_nr(a, b, f: PolynomialFilter, xi: float, eta: float, cfg: SolverConfig = SolverConfig(),
                locked: Optional[DeflationSet] = None, want_vectors: bool = True) -> EigenResults:
    """Polynomial filtered non-restarted Lanczos (eigensolvers.hpp:703-716)."""
    return _cheb_lan(0, a, b, f, xi, eta, cfg, locked, want_vectors)


def cheb_lan_tr(a, b, f: PolynomialFilter, xi: float, eta: float, cfg: SolverConfig = SolverConfig(),
                locked: Optional[DeflationSet] = None, want_vectors: bool = True) -> EigenResults:
    """Polynomial filtered thick-restart Lanczos with locking (eigensolvers.hpp:719-732)."""
    return _cheb_lan(1, a, b, f, xi, eta, cfg, locked, want_vectors)


def rayleigh_and_residual(a, b, u) -> tuple[float, float]:
    """eigensolvers.hpp:86-106 (standard problem) on the GPU."""
    d = _dev(a)
    u = _f64(u)
    if u.size != d.n:
        raise ValueError("rayleigh_and_residual: vector size mismatch")
    if b is not None:  # lambda = u'Au / u'Bu, r = ||Au - lambda Bu|| (eigensolvers.hpp:86-106)
        db = _dev(b)
        if db.n != d.n:
            raise ValueError("rayleigh_and_residual: pencil size mismatch")
        au, bu = _d_matvec(d, u), _d_matvec(db, u)
        uu = float(np.dot(u, bu))
        if not uu > 0.0:
            raise ValueError("rayleigh_and_residual: zero (or B-degenerate) vector")
        lam = float(np.dot(u, au)) / uu
        return lam, float(np.linalg.norm(au - lam * bu))
    lam, res = C.c_double(), C.c_double()
    call("se_rayleigh_residual", d.ctx.handle, d.handle, _pd(u), C.byref(lam), C.byref(res))
    return lam.value, res.value
