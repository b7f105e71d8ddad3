"""ctypes binding of the C-ABI (include/alsncg_capi.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_1508_03110_b200/csrc``).  There is no fallback: if it is
missing, importing the device API raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ALSNCG_LIB") or os.path.join(HERE, "libalsncg_b200.so")  # ALSNCG_LIB: development A/B builds

OK, EINVAL, EDATA, EDUP, ECUDA, ENCCL, ENOMEM, EUNSUPPORTED, ELOGIC = range(9)


class Config(C.Structure):
    _fields_ = [("lambda_", C.c_double), ("n_f", C.c_int), ("max_iters", C.c_int),
                ("tol", C.c_double), ("seed", C.c_uint64), ("alpha0", C.c_double),
                ("armijo_c", C.c_double), ("tau", C.c_double), ("max_backtracks", C.c_int),
                ("n_blocks", C.c_int), ("n_workers", C.c_int), ("trace_every", C.c_int),
                ("snapshot_every", C.c_int), ("paper_timing", C.c_int),
                ("has_fixed_alpha", C.c_int), ("fixed_alpha", C.c_double),
                ("force_beta_zero", C.c_int)]


class TraceRecordC(C.Structure):
    _fields_ = [("iter", C.c_int), ("loss", C.c_double), ("grad_norm", C.c_double),
                ("elapsed_seconds", C.c_double), ("backtracks", C.c_int),
                ("shuffled_columns", C.c_int64), ("restarted", C.c_int)]


class ResultC(C.Structure):
    _fields_ = [("converged", C.c_int), ("iterations", C.c_int), ("final_loss", C.c_double),
                ("final_grad_norm", C.c_double), ("restarts", C.c_int),
                ("fallback_steps", C.c_int), ("fallback_columns", C.c_int)]


SNAPSHOT_FN = C.CFUNCTYPE(None, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double),
                          C.POINTER(C.c_double), C.c_void_p)

vp, dp, ip, lp = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_int64)
i64, f64, i32 = C.c_int64, C.c_double, C.c_int

# name -> (restype, argtypes)
SIGNATURES = {
    "alsncg_last_error": (C.c_char_p, []),
    "alsncg_abi_version": (i32, []),
    "alsncg_row_stride": (i32, [i32]),
    "alsncg_max_rank": (i32, []),
    "alsncg_csr_build": (i32, [i32, i32, i64, vp, vp, vp, i32, vp, vp, vp, vp, vp, vp, ip, ip]),
    "alsncg_random_init": (i32, [i32, i32, i32, C.c_uint64, vp, vp]),
    "alsncg_synth_generate": (i32, [i32, i32, i64, i32, C.c_uint64, vp, vp, vp]),
    "alsncg_backtracking_search": (i32, [vp, f64, f64, f64, f64, i32, dp, ip]),
    "alsncg_ctx_create": (i32, [i32, C.POINTER(vp)]),
    "alsncg_nccl_unique_id": (i32, [vp]),
    "alsncg_ctx_create_dist": (i32, [i32, i32, i32, vp, C.POINTER(vp)]),
    "alsncg_loopgroup_create": (i32, [i32, C.POINTER(vp)]),
    "alsncg_write_trace_csv": (i32, [C.c_char_p, vp, i32]),
    "alsncg_mean_ranking_accuracy": (i32, [vp, i32, i32, i32, vp, vp, vp, vp, i32, dp]),
    "alsncg_read_trace_csv": (i32, [C.c_char_p, vp, i32, ip]),
    "alsncg_loopgroup_destroy": (i32, [vp]),
    "alsncg_ctx_create_loopback": (i32, [i32, i32, vp, C.POINTER(vp)]),
    "alsncg_ctx_destroy": (i32, [vp]),
    "alsncg_ctx_info": (i32, [vp, ip, ip, ip]),
    "alsncg_ctx_stream": (vp, [vp]),
    "alsncg_ctx_synchronize": (i32, [vp]),
    "alsncg_ctx_set_profiling": (i32, [vp, i32]),
    "alsncg_ctx_reset_stats": (i32, [vp]),
    "alsncg_ctx_stat_count": (i32, [vp]),
    "alsncg_ctx_stat": (i32, [vp, i32, C.POINTER(C.c_char_p), lp, dp]),
    "alsncg_ctx_launches": (i64, [vp]),
    "alsncg_ratings_upload": (i32, [vp, i32, i32, i64, vp, vp, vp, vp, vp, vp, C.POINTER(vp)]),
    "alsncg_ratings_download": (i32, [vp, vp, vp, vp, vp, vp, vp]),
    "alsncg_ratings_shard": (i32, [vp, ip, ip, ip, ip]),
    "alsncg_partition_rows": (i32, [i32, vp, i32, i32, vp]),
    "alsncg_ratings_free": (i32, [vp]),
    "alsncg_loss": (i32, [vp, i32, vp, f64, dp]),
    "alsncg_gradient": (i32, [vp, i32, vp, f64, vp]),
    "alsncg_quartic": (i32, [vp, i32, vp, vp, f64, vp]),
    "alsncg_half_sweep": (i32, [vp, i32, i32, vp, f64, vp, ip]),
    "alsncg_als_sweep": (i32, [vp, i32, vp, f64, vp, ip]),
    "alsncg_dev_loss": (i32, [vp, i32, vp, f64, dp]),
    "alsncg_dev_gradient": (i32, [vp, i32, vp, f64, vp]),
    "alsncg_dev_quartic": (i32, [vp, i32, vp, vp, f64, vp]),
    "alsncg_dev_half_sweep": (i32, [vp, i32, i32, vp, f64, vp, ip]),
    "alsncg_dev_dot": (i32, [vp, i64, vp, vp, dp]),
    "alsncg_dev_dot_seq": (i32, [vp, i64, vp, vp, dp]),
    "alsncg_dev_beta_bar_seq": (i32, [vp, i64, vp, vp, vp, vp, dp]),
    "alsncg_dev_axpby": (i32, [vp, i64, f64, vp, f64, vp, vp]),
    "alsncg_dev_beta_bar": (i32, [vp, i64, vp, vp, vp, vp, dp]),
    "alsncg_dev_malloc": (i32, [vp, C.c_size_t, C.POINTER(vp)]),
    "alsncg_dev_free": (i32, [vp, vp]),
    "alsncg_memcpy_h2d": (i32, [vp, vp, vp, C.c_size_t]),
    "alsncg_memcpy_d2h": (i32, [vp, vp, vp, C.c_size_t]),
    "alsncg_flat_h2d": (i32, [vp, i32, i32, i32, vp, vp]),
    "alsncg_flat_d2h": (i32, [vp, i32, i32, i32, vp, vp]),
    "alsncg_ncg_solve": (i32, [vp, C.POINTER(Config), SNAPSHOT_FN, vp, C.POINTER(ResultC), vp,
                               C.POINTER(TraceRecordC), i32, ip]),
    "alsncg_als_solve": (i32, [vp, C.POINTER(Config), SNAPSHOT_FN, vp, C.POINTER(ResultC), vp,
                               C.POINTER(TraceRecordC), i32, ip]),
    "alsncg_solver_create": (i32, [vp, C.POINTER(Config), C.POINTER(vp)]),
    "alsncg_solver_step": (i32, [vp, i32, ip]),
    "alsncg_solver_state": (i32, [vp, ip, ip, dp, ip, ip, ip]),
    "alsncg_solver_trace": (i32, [vp, C.POINTER(TraceRecordC), i32, ip]),
    "alsncg_solver_model": (i32, [vp, vp]),
    "alsncg_solver_destroy": (i32, [vp]),
}

_lib = None


class AlsncgError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is not built; run __graft_entry__.build() "
                "(the B200 path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(status):
    """Maps a C-ABI status to the reference's exception types."""
    if status == OK:
        return
    msg = lib().alsncg_last_error().decode(errors="replace")
    from . import ratings  # local import: DataError types live there
    if status == EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    if status == EDATA:
        raise ratings.DataError(msg)
    if status == ELOGIC:
        raise AssertionError(msg)  # std::logic_error
    raise AlsncgError(status, msg)


def ptr(a):
    """Raw data pointer of a C-contiguous numpy array (or None)."""
    return None if a is None else a.ctypes.data_as(C.c_void_p)
