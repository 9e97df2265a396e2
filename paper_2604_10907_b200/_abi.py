"""ctypes binding of the C-ABI in include/rw_b200.h (librw_b200.so, built in-tree).

The product path is CUDA only: if the library is missing or no GPU is present the
entry points raise — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "librw_b200.so")

RW_MAX_MODELS = 32
RW_OK, RW_ERR_VALIDATION, RW_ERR_CONFIG, RW_ERR_CUDA, RW_ERR_NCCL, RW_ERR_UNSUPPORTED = range(6)

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_lp = C.POINTER(C.c_int64)


class rw_subgradient_params(C.Structure):
    _fields_ = [("eta0", C.c_double), ("max_iters", C.c_int32), ("residual_tol", C.c_double),
                ("polish_passes", C.c_int32)]


class rw_pga_params(C.Structure):
    _fields_ = [("eta", C.c_double), ("max_iters", C.c_int32), ("w_tol", C.c_double),
                ("dual", rw_subgradient_params)]


class rw_beta_params(C.Structure):
    _fields_ = [("beta_min", C.c_double), ("beta_max", C.c_double), ("epsilon", C.c_double),
                ("pga", rw_pga_params)]


class rw_opt_context(C.Structure):
    _fields_ = [("lambda_rps", C.c_double), ("tau_ms", C.c_double), ("kappa", C.c_double)]


class rw_dual_solution(C.Structure):
    _fields_ = [("alpha_star", C.c_double * RW_MAX_MODELS),
                ("count_residual", C.c_double * RW_MAX_MODELS),
                ("counts", C.c_int32 * RW_MAX_MODELS), ("score", C.c_double),
                ("dual_bound", C.c_double), ("duality_gap", C.c_double),
                ("iterations", C.c_int32), ("converged", C.c_int32),
                ("eval_passes", C.c_int64)]


class rw_relaxed_result(C.Structure):
    _fields_ = [("w", C.c_double * RW_MAX_MODELS), ("objective", C.c_double),
                ("score", C.c_double), ("latency_ms", C.c_double), ("iterations", C.c_int32),
                ("converged", C.c_int32), ("out_of_range", C.c_uint32), ("pad_", C.c_int32),
                ("eval_passes", C.c_int64)]


class rw_beta_step(C.Structure):
    _fields_ = [("beta", C.c_double), ("score", C.c_double), ("latency_ms", C.c_double),
                ("feasible", C.c_int32), ("pad_", C.c_int32)]


class rw_beta_result(C.Structure):
    _fields_ = [("feasible", C.c_int32), ("has_beta_star", C.c_int32),
                ("beta_star", C.c_double), ("w_star", C.c_double * RW_MAX_MODELS),
                ("best", rw_relaxed_result), ("n_trace", C.c_int32), ("pad_", C.c_int32),
                ("eval_passes", C.c_int64)]


class rw_setup_record(C.Structure):
    _fields_ = [("setup_id", C.c_int64), ("feasible", C.c_int32), ("status", C.c_int32),
                ("score", C.c_double), ("latency_ms", C.c_double), ("beta", C.c_double),
                ("tau_ms", C.c_double), ("w", C.c_double * RW_MAX_MODELS),
                ("out_of_range", C.c_uint32),
                ("bisect_steps", C.c_int32), ("eval_passes", C.c_int64),
                ("polish_passes", C.c_int64), ("repair_calls", C.c_int64),
                ("exec_passes", C.c_int64)]


# numpy view of rw_setup_record (same layout) for zero-copy record arrays
RECORD_DTYPE = np.dtype([("setup_id", "<i8"), ("feasible", "<i4"), ("status", "<i4"),
                         ("score", "<f8"), ("latency_ms", "<f8"), ("beta", "<f8"),
                         ("tau_ms", "<f8"), ("w", "<f8", (RW_MAX_MODELS,)), ("out_of_range", "<u4"),
                         ("bisect_steps", "<i4"), ("eval_passes", "<i8"),
                         ("polish_passes", "<i8"), ("repair_calls", "<i8"),
                         ("exec_passes", "<i8")])
assert RECORD_DTYPE.itemsize == C.sizeof(rw_setup_record)

_LIB = None


def lib():
    """Load librw_b200.so (raises if it was not built — no fallback)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing; build it with "
                              "`python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        L.rw_last_error.restype = C.c_char_p
        L.rw_reduce_records.restype = C.c_int64
        L.rw_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
        L.rw_destroy.argtypes = [C.c_void_p]
        L.rw_last_error.argtypes = [C.c_void_p]
        L.rw_set_stream.argtypes = [C.c_void_p, C.c_void_p]
        L.rw_last_kernel_ms.argtypes = [C.c_void_p, _dp]
        L.rw_set_profiling.argtypes = [C.c_void_p, C.c_int]
        L.rw_get_profile.argtypes = [C.c_void_p, _lp]
        L.rw_bench_passes.argtypes = [C.c_void_p, _dp, _dp, C.c_int32, _dp]
        L.rw_load_scores.argtypes = [C.c_void_p, C.c_int32, C.c_int32, _dp]
        L.rw_bind_scores_device.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]
        L.rw_load_profiles.argtypes = [C.c_void_p, C.c_int32, _lp, _dp, _dp]
        L.rw_dual_objective.argtypes = [C.c_void_p, _dp, _dp, _dp]
        L.rw_assign_prompts.argtypes = [C.c_void_p, C.c_int32, _dp, _ip, _ip]
        L.rw_solve_dual.argtypes = [C.c_void_p, _dp, C.POINTER(rw_subgradient_params), _dp,
                                    C.POINTER(rw_dual_solution), _ip]
        L.rw_winner_policy.argtypes = [C.c_void_p, C.c_int32, _dp,
                                       C.POINTER(rw_subgradient_params),
                                       C.POINTER(rw_dual_solution), _ip]
        L.rw_project_simplex.argtypes = [C.c_void_p, C.c_int32, _dp, _dp]
        L.rw_system_latency_eval.argtypes = [C.c_void_p, _ip, _dp, C.c_double, C.c_double,
                                             _dp, _dp, _dp, _ip, _dp]
        L.rw_optimize_fractions.argtypes = [C.c_void_p, _ip, C.c_double,
                                            C.POINTER(rw_opt_context),
                                            C.POINTER(rw_pga_params),
                                            C.POINTER(rw_relaxed_result)]
        L.rw_optimize_beta.argtypes = [C.c_void_p, _ip, C.POINTER(rw_opt_context),
                                       C.POINTER(rw_beta_params), C.POINTER(rw_beta_result),
                                       C.c_int32, C.POINTER(rw_beta_step)]
        L.rw_sweep.argtypes = [C.c_void_p, C.c_int64, _lp, _ip, C.POINTER(rw_opt_context),
                               C.POINTER(rw_beta_params), C.c_int32, C.c_int32, C.c_void_p,
                               _lp]
        L.rw_sweep_async.argtypes = [C.c_void_p, C.c_int64, _lp, _ip,
                                     C.POINTER(rw_opt_context), C.POINTER(rw_beta_params),
                                     C.c_int32, C.c_int32]
        L.rw_sweep_slo.argtypes = [C.c_void_p, C.c_int64, _lp, _ip, C.c_int32, _dp,
                                   C.POINTER(rw_opt_context), C.POINTER(rw_beta_params),
                                   C.c_int32, C.c_int32, C.c_void_p, _lp]
        L.rw_sweep_slo_async.argtypes = [C.c_void_p, C.c_int64, _lp, _ip, C.c_int32, _dp,
                                         C.POINTER(rw_opt_context), C.POINTER(rw_beta_params),
                                         C.c_int32, C.c_int32]
        L.rw_sweep_fetch.argtypes = [C.c_void_p, C.c_void_p, _lp]
        L.rw_sweep_spec.argtypes = [C.c_void_p, C.c_int64, _lp, _ip, C.c_int32, _dp,
                                    C.POINTER(rw_opt_context), C.POINTER(rw_beta_params),
                                    C.c_int32, C.c_void_p, _lp]
        L.rw_sweep_multi.argtypes = [C.POINTER(C.c_void_p), C.c_int32, C.c_int64, _lp, _ip,
                                     C.c_int32, _dp, C.POINTER(rw_opt_context),
                                     C.POINTER(rw_beta_params), C.c_void_p]
        L.rw_set_records_device.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        L.rw_reduce_records.argtypes = [C.c_int64, C.c_void_p]
        L.rw_write_scores_f64.argtypes = [C.c_char_p, C.c_int64, C.c_int32,
                                          C.POINTER(C.c_char_p), _dp]
        L.rw_read_scores_f64.argtypes = [C.c_char_p, _lp, _ip, _dp, C.c_int64, C.c_char_p,
                                         C.c_int64]
        L.rw_host_last_error.restype = C.c_char_p
        L.rw_synth_scores.argtypes = [C.c_int32, C.c_int32, _dp, _dp, C.c_uint64, _dp]
        L.rw_enumerate_retain.argtypes = [C.c_int32, _ip, _ip, _ip, _ip, _dp, C.c_int32, _ip,
                                          _ip, _dp, C.c_int32, C.c_double, C.c_int64, _lp, _ip,
                                          _ip, _dp]
        _LIB = L
    return _LIB


def dptr(a):
    return a.ctypes.data_as(_dp) if a is not None else None


def iptr(a):
    return a.ctypes.data_as(_ip) if a is not None else None


def lptr(a):
    return a.ctypes.data_as(_lp) if a is not None else None
