"""ctypes binding of the laxol_b200 C-ABI (include/laxol_b200.h).

The product path is the in-tree CUDA library ``lib/liblaxol_b200.so``.  There
is no CPU fallback: if the library cannot be loaded, or no CUDA device is
present, every compute call raises.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int64, c_size_t, c_uint64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "liblaxol_b200.so")
# the seeded synthetic-workload generators (include/laxol_b200_configs.h): host code, no device
CONFIGS_PATH = os.path.join(_HERE, "lib", "liblaxol_configs.so")

LOB_OK = 0
LOB_INVALID_INPUT = 1
LOB_EVALUATION_ERROR = 2
LOB_CUDA_ERROR = 3

ENGINE_DIRECT = 0
ENGINE_FAST = 1
ENGINE_RELAXED = 2
FAST_STATS_VALID = 1
FAST_CHAINED = 2
FAST_STATS_CHECK = 4
DIRECT_SCREENED = 0
DIRECT_PLAIN = 1
POTENTIAL_ZERO, POTENTIAL_CONST, POTENTIAL_COSINE = 0, 1, 2
TMOD_NONE, TMOD_SIN, TMOD_COS = 0, 1, 2


class LobPotential(ctypes.Structure):
    """lob_potential (include/laxol_b200.h)"""
    _fields_ = [("kind", c_int), ("value", c_double), ("offset", c_double), ("amplitude", c_double),
                ("frequency", c_int), ("tmod", c_int), ("omega", c_double)]

# name -> (restype, argtypes); every symbol declared in include/laxol_b200.h.
_P = c_void_p
SIGNATURES = {
    "lob_ctx_create": (c_int, [c_int, POINTER(c_void_p)]),
    "lob_ctx_destroy": (c_int, [_P]),
    "lob_last_error": (c_char_p, [_P]),
    "lob_version": (c_char_p, []),
    "lob_minplus_direct_f64": (c_int, [_P, _P, _P, c_int64, c_int64, _P, c_int64, _P, _P, c_int64, _P]),
    "lob_minplus_direct_f32": (c_int, [_P, _P, _P, c_int64, c_int64, _P, c_int64, _P, _P]),
    "lob_minplus_window_f64": (c_int, [_P, _P, _P, c_int64, c_int64, c_int64, _P, c_int64, _P, _P, c_int64, _P]),
    "lob_fast_workspace_bytes": (c_int, [c_int64, c_int64, POINTER(c_size_t)]),
    "lob_minplus_fast_f64": (c_int, [_P, _P, _P, c_int64, c_int64, _P, c_double, _P, c_int64, c_double,
                                     _P, _P, c_size_t, c_int, _P]),
    "lob_split_step_2d_f64": (c_int, [_P, _P, _P, _P, c_int64, c_double, c_double, c_double, _P, _P,
                                      c_double, c_int, _P, c_size_t, _P]),
    "lob_evolve_f64": (c_int, [_P, _P, _P, c_int64, c_int64, _P, c_double, _P, c_int64, c_double, c_int,
                               c_int64, _P, _P, POINTER(c_int64), _P, c_size_t, _P]),
    "lob_step_host_f64": (c_int, [_P, _P, _P, c_int64, c_int64, _P, c_double, _P, c_int64, c_double, c_int, _P]),
    "lob_kernel_mech_host": (c_int, [_P, c_int64, c_double, c_double, _P, POINTER(c_int64), POINTER(c_int64),
                                     POINTER(c_double)]),
    "lob_kernel_tabulated_host": (c_int, [_P, c_int64, c_double, _P, c_int64, c_double, c_double, _P,
                                          POINTER(c_int64), POINTER(c_int64)]),
    "lob_minplus_fast_window_f64": (c_int, [_P, _P, _P, c_int64, c_int64, _P, c_int64, _P, c_double, _P, c_int64,
                                            c_double, _P, _P, c_size_t, c_int, _P]),
    "lob_slab_pack_f64": (c_int, [_P, _P, c_int64, c_int64, _P, _P]),
    "lob_slab_unpack_f64": (c_int, [_P, _P, c_int64, c_int64, _P, _P]),
    "lob_slab_push_f64": (c_int, [_P, _P, c_int64, c_int64, c_int, _P, _P]),
    "lob_ctx_set_fast_delta": (c_int, [_P, c_double]),
    "lob_fast_diagnostics": (c_int, [_P, _P, c_int64, c_int64, _P]),
    "lob_block_counts": (c_int, [_P, _P, c_int64, c_int64, c_double, _P, _P]),
    "lob_bench_fp64": (c_int, [_P, POINTER(c_double), POINTER(c_double), POINTER(c_double)]),
    "lob_launch_count": (c_int64, [_P]),
    "lob_ctx_set_direct_mode": (c_int, [_P, c_int]),
    "lob_ctx_set_evolve_resident": (c_int, [_P, c_int]),
    "lob_ctx_set_fast_line": (c_int, [_P, c_int]),
    "lob_direct_stats": (c_int, [_P, POINTER(c_uint64), POINTER(c_uint64), c_int]),
    # weak-KAM consumers (proj/src/weakkam.cpp)
    "lob_minplus_gemm_f64": (c_int, [_P, _P, c_int64, _P, c_int64, _P, c_int64, c_int64, c_int64, c_int64, _P]),
    "lob_period_kinetic_host": (c_int, [_P, c_int64, c_int64, _P]),
    "lob_period_matrix_f64": (c_int, [_P, _P, _P, c_int64, c_int64, _P, _P, _P]),
    "lob_eigenvalue_karp_f64": (c_int, [_P, _P, c_int64, POINTER(c_double), _P]),
    "lob_hbar_drift_host_f64": (c_int, [_P, _P, c_int64, c_double, c_double, _P, c_int64, c_int, c_int, c_double,
                                        POINTER(c_double), POINTER(c_double), POINTER(c_int64), POINTER(c_int),
                                        _P]),
    "lob_fixed_point_residual_host_f64": (c_int, [_P, _P, c_int64, c_double, c_double, c_double, _P, c_int64,
                                                  c_int, POINTER(c_double)]),
    "lob_step_semidiscrete_f64": (c_int, [_P, _P, _P, c_int64, c_int64, c_int64, c_int, c_double, _P, c_int64,
                                          c_double, c_double, _P, c_int, _P]),
    "lob_relaxed_workspace_bytes": (c_int, [c_int64, c_int64, POINTER(c_size_t)]),
    "lob_minplus_relaxed_f64": (c_int, [_P, _P, _P, c_int64, c_int64, _P, c_int64, _P, _P, c_int64, c_double, _P,
                                        _P, c_size_t, _P]),
    "lob_split_step_nd_f64": (c_int, [_P, _P, _P, _P, c_int, c_int64, c_double, _P, _P, _P, _P, c_double, c_int,
                                      _P, c_size_t, _P]),
    "lob_split_step_nd_window_f64": (c_int, [_P, _P, _P, _P, c_int, _P, c_int64, c_double, _P, _P, _P, _P]),
    "lob_potential2d_rows_f64": (c_int, [_P, _P, c_int64, c_int64, _P, _P, c_double, c_double, _P]),
    "lob_minplus_conv_naive_f64": (c_int, [_P, _P, c_int64, _P, c_int64, _P, _P]),
    "lob_decompose_f64": (c_int, [_P, _P, c_int64, c_double, _P, _P, _P, c_int64, POINTER(c_int64), _P]),
    "lob_conv_fast_f64": (c_int, [_P, _P, c_int64, _P, c_int64, c_double, _P, POINTER(c_int64), _P]),
    # synthetic workloads (include/laxol_b200_configs.h)
}

_lib = None
_cfg = None

# include/laxol_b200_configs.h (liblaxol_configs.so)
CONFIG_SIGNATURES = {
    "lob_gen_sin": (None, [c_int64, _P]),
    "lob_gen_cos": (None, [c_int64, _P]),
    "lob_gen_potential": (None, [c_int, c_int64, _P]),
    "lob_gen_c2_drifts": (None, [c_int64, _P]),
    "lob_gen_c3_lines": (None, [c_int64, c_int64, c_int64, c_uint64, _P]),
    "lob_gen_c4_u0": (None, [c_int64, _P]),
    "lob_c4_time_term": (c_double, [c_double]),
    "lob_gen_c5_lines": (None, [c_int64, c_int64, c_int64, c_uint64, _P, c_int]),
}


class LaxolError(RuntimeError):
    """Base error; subclasses mirror the reference's exception types."""


class InvalidInput(LaxolError):
    """proj/include/laxol/errors.hpp:9-11"""


class EvaluationError(LaxolError):
    """proj/include/laxol/errors.hpp:15-17"""


class CudaError(LaxolError):
    pass


def load(path: str | None = None, required_symbols=None):
    """Load the CUDA library; raises OSError if it was not built."""
    global _lib
    if path is None:
        path = LIB_PATH
    if _lib is not None and path == LIB_PATH:
        return _lib
    if not os.path.exists(path):
        raise OSError(f"laxol_b200 CUDA library not built: {path} (run __graft_entry__.build())")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        if required_symbols is not None and name not in required_symbols:
            continue
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path == LIB_PATH:
        _lib = lib
    return lib


def load_configs(path: str | None = None):
    """Load the synthetic-workload generator library (host code only)."""
    global _cfg
    if _cfg is not None and path is None:
        return _cfg
    p = path or CONFIGS_PATH
    if not os.path.exists(p):
        raise OSError(f"laxol_b200 generator library not built: {p} (run __graft_entry__.build())")
    lib = ctypes.CDLL(p)
    for name, (res, args) in CONFIG_SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _cfg = lib
    return lib


def check(status: int, ctx=None, where: str = ""):
    if status == LOB_OK:
        return
    msg = ""
    if ctx is not None:
        raw = load().lob_last_error(ctx)
        msg = raw.decode() if raw else ""
    text = f"{where}: {msg}" if where else msg
    if status == LOB_INVALID_INPUT:
        raise InvalidInput(text)
    if status == LOB_EVALUATION_ERROR:
        raise EvaluationError(text)
    raise CudaError(text or "CUDA error / no device")
