"""ctypes binding of libcnmf_b200.so (include/cnmf_b200.h).

The CUDA library is the product: there is no CPU fallback. Importing this
module without the built library, or calling into it without a CUDA device,
raises immediately.
"""

import ctypes
import os

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CNMF_LIB_PATH") or os.path.join(_HERE, "libcnmf_b200.so")  # override: A/B tools only

c_i64 = ctypes.c_int64
c_int = ctypes.c_int
c_u64 = ctypes.c_uint64
c_dbl = ctypes.c_double
c_size = ctypes.c_size_t
vp = ctypes.c_void_p
c_i64p = ctypes.POINTER(ctypes.c_int64)
c_intp = ctypes.POINTER(ctypes.c_int)

# name -> (restype, argtypes); mirrors include/cnmf_b200.h exactly
SIGNATURES = {
    "cnmf_abi_version": (c_int, []),
    "cnmf_last_error": (ctypes.c_char_p, []),
    "cnmf_panel_ld": (c_int, [c_int]),
    "cnmf_launch_count": (c_i64, []),
    "cnmf_set_pass_profiling": (None, [c_int]),
    "cnmf_set_pass_impl": (None, [c_int]),
    "cnmf_pass_stats": (c_int, [ctypes.POINTER(c_dbl), c_i64p, ctypes.POINTER(c_dbl)]),
    "cnmf_child_seed": (c_u64, [c_u64, ctypes.c_char_p]),
    "cnmf_gaussian_fill": (c_int, [c_u64, c_i64, c_i64, c_i64, c_int, vp, c_i64, vp]),
    "cnmf_uniform_fill": (c_int, [c_u64, c_i64, c_i64, c_dbl, c_dbl, c_int, c_int, vp, vp]),
    "cnmf_uniform_fill_at": (c_int, [c_u64, c_i64, c_i64, c_i64, c_dbl, c_dbl, c_int, c_int, vp, vp]),
    "cnmf_normal_fill_at": (c_int, [c_u64, c_i64, c_i64, c_int, vp, vp, vp]),
    "cnmf_pass_forward": (c_int, [vp, c_i64, c_i64, c_i64, vp, c_int, vp, vp]),
    "cnmf_pass_transpose": (c_int, [vp, c_i64, c_i64, c_i64, vp, c_int, vp, vp]),
    "cnmf_pass_pair": (c_int, [vp, c_i64, c_i64, c_i64, vp, vp, vp, vp, c_int, vp]),
    "cnmf_admm_full_workspace": (c_size, [c_i64, c_i64, c_int]),
    "cnmf_admm_full_run": (c_int, [vp, c_i64, c_i64, c_i64, c_int, vp, vp, vp, vp, vp, vp, c_dbl, c_dbl, c_dbl, c_int,
                                   c_dbl, vp, vp, c_intp, c_intp, c_int, c_int, vp, c_size, vp]),
    "cnmf_compress_workspace": (c_size, [c_i64, c_i64, c_int]),
    "cnmf_structured_compress": (c_int, [vp, c_i64, c_i64, c_i64, c_int, c_int, c_u64, c_int, vp, vp, c_size, vp]),
    "cnmf_structured_compress_async": (c_int, [vp, c_i64, c_i64, c_i64, c_int, c_int, c_u64, c_int, vp, vp, c_size,
                                               vp]),
    "cnmf_compress_pair_async": (c_int, [vp, c_i64, c_i64, c_i64, c_int, c_int, c_u64, c_u64, vp, vp, vp, vp,
                                         c_size, vp]),
    "cnmf_compress_check": (c_int, [vp, c_i64, c_i64, c_int, vp]),
    "cnmf_orthonormalize": (c_int, [vp, c_i64, c_int, vp, vp, c_size, vp]),
    "cnmf_cholesky_inverse": (c_int, [vp, c_int, c_int, vp, vp, vp]),
    "cnmf_small_workspace": (c_size, [c_int]),
    "cnmf_status_reset": (c_int, [vp, c_int, vp]),
    "cnmf_status_check": (c_int, [vp, c_int, vp]),
    "cnmf_orthonormalize_async": (c_int, [vp, c_i64, c_int, vp, vp, c_size, vp]),
    "cnmf_cholesky_inverse_async": (c_int, [vp, c_int, c_int, vp, vp, vp, vp]),
    "cnmf_panel_apply": (c_int, [vp, c_i64, c_int, vp, vp]),
    "cnmf_spa_workspace": (c_size, [c_i64, c_int]),
    "cnmf_panel_to_f64": (c_int, [vp, c_i64, c_int, vp, c_i64, vp]),
    "cnmf_select_spa": (c_int, [vp, c_i64, c_int, c_i64, c_int, c_i64p, c_intp, vp, c_size, vp]),
    "cnmf_select_xray": (c_int, [vp, c_i64, c_int, c_i64, c_int, vp, c_dbl, c_i64p, c_intp, vp]),
    "cnmf_right_factor": (c_int, [vp, c_i64, c_int, c_i64, vp, c_int, c_dbl, vp, c_i64p, vp]),
    "cnmf_refit_norms": (c_int, [vp, c_i64, c_int, c_i64, vp, c_int, vp, vp, vp]),
    "cnmf_nnls_gram": (c_int, [vp, vp, c_i64, c_int, c_dbl, c_int, vp, c_i64p, vp]),
    "cnmf_gram_f64": (c_int, [vp, c_i64, c_int, vp, c_int, vp, vp]),
    "cnmf_panel_cross": (c_int, [vp, vp, c_i64, c_int, vp, vp]),
    "cnmf_residual_norms": (c_int, [vp, c_i64, c_i64, c_i64, vp, vp, vp, c_int, vp, vp]),
    "cnmf_admm_workspace": (c_size, [c_i64, c_i64, c_int, c_int]),
    "cnmf_compress_f64_workspace": (c_size, [c_i64, c_i64, c_int]),
    "cnmf_structured_compress_f64": (c_int, [vp, c_i64, c_i64, c_i64, c_int, c_int, c_u64, c_int, vp, vp, c_size,
                                             vp]),
    "cnmf_pass_transpose_f64": (c_int, [vp, c_i64, c_i64, c_i64, vp, c_int, vp, vp]),
    "cnmf_residual_norms_f64": (c_int, [vp, c_i64, c_i64, c_i64, vp, vp, vp, c_int, vp, vp]),
    "cnmf_admm_shard_workspace": (c_size, [c_int, c_int]),
    "cnmf_admm_shard_sums_offset": (c_size, []),
    "cnmf_admm_shard_begin": (c_int, [vp, c_int, c_int, vp, vp, c_int, vp]),
    "cnmf_admm_shard_sweep": (c_int, [vp, vp, c_i64, vp, c_i64, c_int, c_int, vp, vp, vp, vp, c_dbl, c_dbl, c_dbl,
                                      c_int, vp]),
    "cnmf_admm_shard_core": (c_int, [vp, vp, vp, vp, c_int, c_int, c_dbl, c_dbl, c_dbl, c_dbl, vp, vp, c_int, c_int,
                                     c_int, c_int, vp]),
    "cnmf_admm_shard_status": (c_int, [vp, c_intp, vp]),
    "cnmf_shard_argmax": (c_int, [vp, c_i64, vp, vp, vp, vp, vp]),
    "cnmf_spa_shard_step": (c_int, [vp, c_i64, c_int, c_i64, vp, vp, vp, vp]),
    "cnmf_xray_shard_scores": (c_int, [vp, c_i64, c_int, c_i64, vp, vp, vp, vp]),
    "cnmf_col_mass": (c_int, [vp, c_i64, c_int, c_i64, vp, vp, vp]),
    "cnmf_right_factor_given": (c_int, [vp, c_i64, c_int, c_i64, vp, c_int, c_dbl, vp, c_i64p, vp]),
    "cnmf_refit_given": (c_int, [vp, c_i64, c_int, c_i64, vp, c_int, vp, vp, vp, vp, vp]),
    "cnmf_admm_run": (c_int, [vp, vp, c_i64, vp, c_i64, c_int, c_int, vp, vp, vp, vp, vp, vp, c_dbl, c_dbl,
                              c_dbl, c_int, c_dbl, vp, vp, c_intp, c_intp, c_int, c_int, vp, c_size, vp]),
}

_STATUS = {
    1: errors.ArgumentError,
    2: errors.InfeasibleRankError,
    3: errors.NumericError,
    4: errors.RankDeficiencyError,
    5: errors.ConvergenceError,
    6: errors.DivergenceError,
    7: errors.UndefinedMetricError,
    8: errors.DeviceError,
}

_lib = None


def load():
    """Load the library (once). Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(make -C paper_1505_04650_b200/csrc). There is no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error():
    return load().cnmf_last_error().decode("utf-8", "replace")


def check(status, **extra):
    """Map a cnmf_status onto the reference's exception classes (errors.py)."""
    if status == 0:
        return
    cls = _STATUS.get(status, errors.CnmfError)
    msg = last_error()
    if cls is errors.RankDeficiencyError:
        raise cls(msg, picks=extra.get("picks"))
    if cls is errors.DivergenceError:
        raise cls(msg, trace=extra.get("trace"))
    if cls is errors.ConvergenceError:
        raise cls(msg, best=extra.get("best"))
    raise cls(msg)


def call(name, *args, **extra):
    check(getattr(load(), name)(*args), **extra)
