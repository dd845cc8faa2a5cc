"""ctypes binding of libchebstep_gpu.so (include/chebstep_gpu.h).

The library is the product: hand-written sm_100a kernels behind a C ABI.
Importing this module loads it from paper_2603_09790_b200/lib/ and fails
loudly if it is missing -- there is no Python or CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

LIB_PATH = os.environ.get("CS_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                    "lib", "libchebstep_gpu.so")

CS_OK = 0
CS_CHECK_STRUCTURE, CS_CHECK_SYMMETRIC, CS_CHECK_SPD_DIAGONAL = 0, 1, 2
CS_ERR_DIMENSION = 1
CS_ERR_INVALID_MATRIX = 2
CS_ERR_NOT_SPD = 3
CS_ERR_BASIS_BREAKDOWN = 4
CS_ERR_SOLVER_BREAKDOWN = 5
CS_ERR_GUARD_EXCEEDED = 6
CS_ERR_PARSE = 7
CS_ERR_INVALID_ARGUMENT = 8
CS_ERR_GENERIC = 9
CS_ERR_CUDA = 10
CS_ERR_NCCL = 11

CS_PRECOND_IDENTITY, CS_PRECOND_JACOBI, CS_PRECOND_BLOCK_JACOBI, CS_PRECOND_DEVICE_FN = 0, 1, 2, 3
# int (*)(void* user, const double* in, double* out, int64_t n, void* stream)
PRECOND_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)
CS_GEN_POISSON27, CS_GEN_STENCIL7 = 0, 1
CS_GRAM_FGS, CS_GRAM_CHOLESKY = 0, 1
CS_MODE_FAST, CS_MODE_REFERENCE = 0, 1
CS_VAR_EXPLICIT_W, CS_VAR_RECUR_W, CS_VAR_REF_FGS, CS_VAR_REF_MPK, CS_VAR_TREE = 1, 2, 4, 8, 16
CS_VAR_P_FROM_Z, CS_VAR_P_STORED, CS_VAR_TRUE_R, CS_VAR_RECUR_R, CS_VAR_STORED_R = 32, 64, 128, 256, 512
PHASES = ("spmv", "reduce", "small", "update", "lanczos", "comm", "other")

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_dp = C.POINTER(C.c_double)
_vp = C.c_void_p


class CsConfig(C.Structure):
    _fields_ = [("s", C.c_int), ("tol", C.c_double), ("max_outer", C.c_int), ("nu", C.c_int),
                ("gram", C.c_int), ("has_spectrum", C.c_int), ("lambda_min", C.c_double),
                ("lambda_max", C.c_double), ("lanczos_steps", C.c_int), ("seed", C.c_uint64),
                ("mode", C.c_int), ("check_every", C.c_int),
                ("collect_gram", C.c_int), ("track_true_residual", C.c_int),
                ("error_reference", C.c_void_p), ("collect_iterates", C.c_int),
                ("variant", C.c_int)]


class CsReport(C.Structure):
    _fields_ = [("converged", C.c_int), ("outer_iters", C.c_int), ("spmv_count", C.c_int64),
                ("precond_count", C.c_int64), ("allreduce_count", C.c_int64),
                ("local_update_flops", C.c_double), ("gram_solve_flops", C.c_double),
                ("lambda_min", C.c_double), ("lambda_max", C.c_double), ("cap", C.c_int),
                ("n_rel", C.c_int), ("n_da", C.c_int), ("n_db", C.c_int),
                ("rel_residual", _dp), ("delta_alpha", _dp), ("delta_beta", _dp),
                ("device_allreduces", C.c_int64), ("kernel_launches", C.c_int64),
                ("t_lanczos_ms", C.c_double), ("t_solve_ms", C.c_double),
                ("n_kappa", C.c_int), ("n_true", C.c_int), ("n_aerr", C.c_int), ("n_iter", C.c_int),
                ("kappa_w", _dp), ("gram_history", _dp), ("true_rel_residual", _dp),
                ("a_norm_error", _dp), ("iterates", _dp), ("schedule", C.c_int)]


# name -> (restype, argtypes); every symbol of include/chebstep_gpu.h
SIGNATURES = {
    "cs_last_error": (C.c_char_p, [C.POINTER(C.c_int)]),
    "cs_version": (C.c_int, []),
    "cs_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "cs_ctx_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "cs_ctx_destroy": (C.c_int, [_vp]),
    "cs_ctx_set_timing": (C.c_int, [_vp, C.c_int]),
    "cs_ctx_reset_timing": (C.c_int, [_vp]),
    "cs_ctx_get_timing": (C.c_int, [_vp, C.c_int, _dp, C.POINTER(C.c_int64)]),
    "cs_ctx_launch_count": (C.c_int, [_vp, C.POINTER(C.c_int64)]),
    "cs_ctx_synchronize": (C.c_int, [_vp]),
    "cs_ctx_stream": (C.c_int, [_vp, C.POINTER(_vp)]),
    "cs_comm_unique_id": (C.c_int, [C.c_char_p]),
    "cs_ctx_comm_init": (C.c_int, [_vp, C.c_int, C.c_int, C.c_char_p]),
    "cs_ctx_allreduce_max": (C.c_int, [_vp, _dp]),
    "cs_partition_rows": (C.c_int, [C.c_int64, C.c_int64, C.c_int, C.c_int,
                                    C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "cs_halo_map_csr": (C.c_int, [C.c_int64, C.c_int64, _i64p, _i64p, C.POINTER(C.c_int64),
                                  _vp, C.c_int64, _vp]),
    "cs_problem_generate": (C.c_int, [_vp, C.c_int, C.c_int64, C.c_int64, C.c_int64, _vp,
                                      C.POINTER(_vp)]),
    "cs_problem_upload_csr": (C.c_int, [_vp, C.c_int64, _vp, _vp, _vp, C.POINTER(_vp)]),
    "cs_problem_upload_csr_block": (C.c_int, [_vp, C.c_int64, C.c_int64, C.c_int64, _vp, _vp, _vp,
                                              C.POINTER(_vp)]),
    "cs_problem_read_mm": (C.c_int, [_vp, C.c_char_p, C.c_int, C.POINTER(_vp)]),
    "cs_fgs_rate": (C.c_int, [C.c_int, _vp, _dp, _dp]),
    "cs_kappa_sym": (C.c_int, [C.c_int, _vp, _dp]),
    "cs_mm_read": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(_vp), C.POINTER(C.c_int64),
                             C.POINTER(C.c_int64)]),
    "cs_csr_host_rows": (C.c_int, [_vp, C.c_int64, C.c_int64, _vp, _vp, _vp]),
    "cs_csr_host_free": (C.c_int, [_vp]),
    "cs_mm_write": (C.c_int, [C.c_char_p, C.c_int64, _vp, _vp, _vp]),
    "cs_csr_validate": (C.c_int, [C.c_int64, _vp, _vp, _vp, C.c_int]),
    "cs_problem_destroy": (C.c_int, [_vp]),
    "cs_problem_info": (C.c_int, [_vp, _i64p]),
    "cs_problem_halo_mode": (C.c_int, [_vp, C.POINTER(C.c_int)]),
    "cs_problem_download_csr": (C.c_int, [_vp, _i64p, _i64p, _f64p]),
    "cs_problem_ghosts": (C.c_int, [_vp, _i64p]),
    "cs_problem_set_precond": (C.c_int, [_vp, C.c_int]),
    "cs_problem_inv_diag": (C.c_int, [_vp, _f64p]),
    "cs_problem_set_precond_block_jacobi": (C.c_int, [_vp, C.c_int, _f64p]),
    "cs_problem_set_precond_fn": (C.c_int, [_vp, _vp, _vp]),
    "cs_spmv": (C.c_int, [_vp, _f64p, _f64p]),
    "cs_mpk": (C.c_int, [_vp, _f64p, C.c_int, C.c_double, C.c_double, _f64p, _f64p]),
    "cs_block_gram": (C.c_int, [_vp, C.c_int64, C.c_int, C.c_int, _f64p, _f64p, _f64p, C.c_int]),
    "cs_block_update": (C.c_int, [_vp, C.c_int64, C.c_int, C.c_int, _f64p, _f64p, _f64p, _f64p]),
    "cs_assemble_gram": (C.c_int, [_vp, C.c_int64, C.c_int, _f64p, _f64p, _f64p, C.c_int]),
    "cs_fgs_solve": (C.c_int, [_vp, C.c_int, _f64p, C.c_int, _f64p, C.c_int, _f64p, _dp]),
    "cs_cholesky_solve": (C.c_int, [_vp, C.c_int, _f64p, C.c_int, _f64p, _f64p]),
    "cs_random_vector": (C.c_int, [_vp, C.c_int64, C.c_uint64, _f64p]),
    "cs_tridiag_eigvals": (C.c_int, [C.c_int, _f64p, _f64p, _f64p]),
    "cs_estimate_interval": (C.c_int, [_vp, C.c_int, C.c_uint64, C.c_int, _dp, _dp]),
    "cs_bench_spmv": (C.c_int, [_vp, C.c_int, C.c_int, _dp]),
    "cs_config_default": (None, [C.POINTER(CsConfig)]),
    "cs_pcg_s_solve": (C.c_int, [_vp, _f64p, _f64p, C.POINTER(CsConfig), _f64p,
                                 C.POINTER(CsReport)]),
    "cs_pcg_solve": (C.c_int, [_vp, _f64p, _f64p, C.c_double, C.c_int, C.c_int, _f64p,
                               C.POINTER(CsReport)]),
    "cs_pcg_solve_cfg": (C.c_int, [_vp, _f64p, _f64p, C.POINTER(CsConfig), _f64p,
                                   C.POINTER(CsReport)]),
    "cs_pcg_s_solve_device": (C.c_int, [_vp, _vp, _vp, C.POINTER(CsConfig), _vp,
                                        C.POINTER(CsReport)]),
    "cs_pcg_solve_device": (C.c_int, [_vp, _vp, _vp, C.c_double, C.c_int, C.c_int, _vp,
                                      C.POINTER(CsReport)]),
    "cs_pcg_s_solve_csr": (C.c_int, [_vp, C.c_int64, _vp, _vp, _vp, C.c_int, _vp, _vp,
                                     C.POINTER(CsConfig), _vp, C.POINTER(CsReport)]),
    "cs_pcg_solve_csr": (C.c_int, [_vp, C.c_int64, _vp, _vp, _vp, C.c_int, _vp, _vp, C.c_double,
                                   C.c_int, _vp, C.POINTER(CsReport)]),
}

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python paper_2603_09790_b200/build.py` "
        "(the CUDA library is the product; there is no CPU fallback)")

lib = C.CDLL(LIB_PATH)
for _name, (_res, _args) in SIGNATURES.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


def last_error():
    payload = C.c_int(0)
    msg = lib.cs_last_error(C.byref(payload)).decode()
    return msg, payload.value
