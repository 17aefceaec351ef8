"""ctypes binding of libsliceeig_cuda.so (the C ABI in include/sliceeig_cuda.h).

There is no fallback: if the in-tree library is missing or fails to load, every call raises
``LibraryNotBuilt`` (build it with ``python -m paper_1802_05215_b200.build``).
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsliceeig_cuda.so")

SE_OK, SE_EINVAL, SE_ENUMERIC, SE_ECUDA, SE_ENOMEM, SE_ERANGE = 0, -1, -2, -3, -4, -5
DAMPING = {"none": 0, "sigma": 1, "jackson": 2}
PROBES = {"rademacher": 0, "gaussian": 1, "normal": 1}


class LibraryNotBuilt(RuntimeError):
    pass


class CudaError(RuntimeError):
    pass


class SePolyFilter(C.Structure):
    _fields_ = [("k", C.c_int), ("gamma", C.c_double), ("c", C.c_double), ("d", C.c_double),
                ("tau", C.c_double), ("ta", C.c_double), ("tb", C.c_double), ("bar", C.c_double),
                ("damping", C.c_int), ("cap_reached", C.c_int), ("mu", C.POINTER(C.c_double)),
                ("mu_cap", C.c_int)]


class SeSolverCfg(C.Structure):
    _fields_ = [("m", C.c_int), ("max_its", C.c_long), ("ncycle", C.c_int), ("tau1", C.c_double),
                ("res_tol", C.c_double), ("est_count", C.c_int), ("seed", C.c_uint64)]


class SeCounters(C.Structure):
    _fields_ = [("n_A_matvec", C.c_long), ("n_B_matvec", C.c_long), ("n_B_solve", C.c_long),
                ("n_shift_solve", C.c_long), ("t_mv", C.c_double), ("t_orth", C.c_double),
                ("t_sv", C.c_double), ("t_total", C.c_double)]


_VP = C.c_void_p
_PD = C.POINTER(C.c_double)
_PI = C.POINTER(C.c_int)
_PL = C.POINTER(C.c_long)

# name -> argtypes (all return int status)
SIGNATURES = {
    "se_device_count": [_PI],
    "se_ctx_create": [C.c_int, C.POINTER(_VP)],
    "se_ctx_set_candidate_budget": [_VP, C.c_size_t],
    "se_ctx_destroy": [_VP],
    "se_ctx_synchronize": [_VP],
    "se_ctx_kernel_launches": [_VP, _PL],
    "se_ctx_filter_timing": [_VP, C.c_int, _PD, _PL, _PD],
    "se_laplacian_host": [C.c_int, _PI, _PI, _PL, _PI, _PI, _PD],
    "se_laplacian_eigs": [C.c_int, _PI, _PD],
    "se_gen_random_sparse": [C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_double, _PL, _PI, _PI, _PD],
    "se_mass_scaling": [C.c_int, C.c_uint64, _PD, _PD],
    "se_csr_upload": [_VP, C.c_int, _PI, _PI, _PD, C.POINTER(_VP)],
    "se_csr_gen_laplacian": [_VP, C.c_int, _PI, C.POINTER(_VP)],
    "se_csr_info": [_VP, _PI, _PL],
    "se_csr_download": [_VP, _VP, _PI, _PI, _PD],
    "se_csr_scale_sym": [_VP, _VP, _PD],
    "se_csr_set_residual_weight": [_VP, _VP, _PD],
    "se_csr_free": [_VP],
    "se_spmv": [_VP, _VP, _PD, _PD],
    "se_cheb_apply": [_VP, _VP, C.POINTER(SePolyFilter), C.c_int, _PD, _PD, _PL],
    "se_cheb_apply_dev": [_VP, _VP, C.POINTER(SePolyFilter), C.c_int, _VP, _VP],
    "se_filter_bench": [_VP, _VP, C.POINTER(SePolyFilter), C.c_int, _PD, _PL, _PD],
    "se_cgs_bench": [_VP, C.c_int, C.c_int, C.c_int, _PD],
    "se_multi_filter_bench": [_VP, _VP, C.c_int, C.c_int, C.c_int, _PD],
    "se_block_filter_bench": [_VP, _VP, C.c_int, C.c_int, _PD],
    "se_resident_filter": [C.c_int],
    "se_csr_resident_tiles": [_VP, _PI],
    "se_csr_resident_smem": [_VP, C.POINTER(C.c_size_t)],
    "se_mult_cols": [_VP, C.c_int, C.c_int, C.c_int, _PD, C.c_long, C.c_int, _PD, C.c_long, _PD,
                     C.c_long, C.c_int, _PD],
    "se_cgs2_bench": [_VP, C.c_int, C.c_int, C.c_int, C.c_int, _PD],
    "se_damping_multipliers": [C.c_int, C.c_int, _PD],
    "se_chebyshev_coeffs": [C.c_double, C.c_int, _PD],
    "se_normalized_filter_coeffs": [C.c_int, C.c_double, C.c_int, _PD],
    "se_balance_center": [C.c_int, C.c_double, C.c_double, C.c_int, _PD],
    "se_find_pol": [C.c_double, C.c_double, C.c_double, C.c_double, C.c_double, C.c_int, C.c_int,
                    C.POINTER(SePolyFilter)],
    "se_eval_pol": [C.POINTER(SePolyFilter), C.c_double, _PD],
    "se_kpm_moments": [_VP, _VP, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int, C.c_uint64,
                       C.c_int, C.c_int, _PD],
    "se_kpm_moments_probes": [_VP, _VP, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int,
                              C.c_uint64, C.c_int, C.c_int, _PD],
    "se_probe_block": [C.c_uint64, C.c_int, C.c_int, C.c_long, C.c_int, _PD],
    "se_kpm_moments_multi": [C.c_int, _PI, C.c_int, _PI, _PI, _PD, C.c_double, C.c_double, C.c_int,
                             C.c_int, C.c_int, C.c_uint64, _PD],
    "se_kpm_dos_multi": [C.c_int, _PI, C.c_int, _PI, _PI, _PD, C.c_double, C.c_double, C.c_int,
                         C.c_int, C.c_int, C.c_uint64, C.c_int, _PD, _PD, _PD],
    "se_nccl_version": [_PI],
    "se_ls_pol_approx": [C.c_int, C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, _PI, _PD,
                         _PD],
    "se_apply_cheb": [_VP, _VP, C.c_double, C.c_double, C.c_int, _PD, C.c_int, _PD, _PD],
    "se_pencil_create": [_VP, _VP, C.c_double, C.c_int, C.POINTER(_VP)],
    "se_pencil_info": [_VP, _PI, _PD, _PD, _PD],
    "se_pencil_free": [_VP],
    "se_lan_tr_bounds_pencil": [_VP, _VP, _VP, C.c_double, C.c_int, C.c_int, C.c_uint64, _PD, _PD],
    "se_lan_dos_pencil": [_VP, _VP, _VP, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int,
                          C.c_double, C.c_uint64, _PD, _PD, _PD],
    "se_cheb_lan_pencil": [_VP, _VP, _VP, C.POINTER(SePolyFilter), C.c_double, C.c_double,
                           C.POINTER(SeSolverCfg), C.c_int, C.POINTER(_VP)],
    "se_kpm_curve": [C.c_int, _PD, C.c_int, C.c_double, C.c_double, C.c_int, _PD, _PD, _PD],
    "se_kpm_dos": [_VP, _VP, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int,
                   _PD, _PD, _PD],
    "se_lan_dos": [_VP, _VP, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int, C.c_double,
                   C.c_uint64, _PD, _PD, _PD],
    "se_results_orth": [_VP, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong), _PD],
    "se_device_memory": [C.c_int, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)],
    "se_dos_count": [C.c_int, C.c_int, _PD, _PD, C.c_double, C.c_double, _PD],
    "se_slice_spectrum": [C.c_int, C.c_int, _PD, _PD, C.c_double, C.c_double, C.c_int, _PD, _PD],
    "se_lan_tr_bounds": [_VP, _VP, C.c_double, C.c_int, C.c_int, C.c_uint64, _PD, _PD],
    "se_lanczos_run": [_VP, _VP, _PD, C.c_int, _PD, _PD, _PI, _PI, _PD, _PD, _PD],
    "se_paired_cgs2": [_VP, C.c_int, C.c_int, _PD, _PD, _PD],
    "se_sym_tridiag_eig": [C.c_int, _PD, _PD, C.c_int, _PD, _PD],
    "se_arrow_tridiag": [C.c_int, _PD, _PD, C.c_double, _PD, _PD],
    "se_dense_sym_eig": [C.c_int, _PD, C.c_int, C.c_int, _PD, _PD],
    "se_cheb_si": [_VP, _VP, C.POINTER(SePolyFilter), C.c_double, C.c_double, C.c_int,
                   C.POINTER(SeSolverCfg), C.POINTER(_VP)],
    "se_cheb_lan": [_VP, _VP, C.POINTER(SePolyFilter), C.c_double, C.c_double,
                    C.POINTER(SeSolverCfg), C.c_int, C.c_int, _PD, _PD, C.c_int, C.POINTER(_VP)],
    "se_results_count": [_VP, _PI],
    "se_results_copy": [_VP, _PD, _PD, _PD],
    "se_results_vector": [_VP, C.c_int, _PD],
    "se_results_info": [_VP, _PL, _PI, C.POINTER(SeCounters)],
    "se_results_free": [_VP],
    "se_rayleigh_residual": [_VP, _VP, _PD, _PD, _PD],
}

_lib = None
_lock = threading.Lock()


def lib():
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise LibraryNotBuilt(
                        f"{LIB_PATH} is missing; run `python -m paper_1802_05215_b200.build`")
                try:
                    L = C.CDLL(LIB_PATH)
                except OSError as e:
                    raise LibraryNotBuilt(f"cannot load {LIB_PATH}: {e}") from e
                L.se_last_error.restype = C.c_char_p
                L.se_version.restype = C.c_char_p
                for name, args in SIGNATURES.items():
                    fn = getattr(L, name)
                    fn.argtypes = args
                    fn.restype = C.c_int
                _lib = L
    return _lib


def check(rc: int):
    """Map a C-ABI status to the reference's exception types (include/sliceeig_cuda.h)."""
    if rc == SE_OK:
        return
    msg = lib().se_last_error().decode()
    if rc == SE_EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    if rc == SE_ERANGE:
        raise IndexError(msg)  # std::out_of_range
    if rc in (SE_ECUDA, SE_ENOMEM):
        raise CudaError(msg)
    raise RuntimeError(msg)  # std::runtime_error


def call(name: str, *args):
    check(getattr(lib(), name)(*args))
