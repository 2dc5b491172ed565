"""ctypes binding of libpnx.so (include/pnx.h). Loads the in-tree library and
fails loudly if it is missing -- the product path has no CPU fallback."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PNX_LIB_PATH") or os.path.join(HERE, "libpnx.so")  # override: dev A/B builds

_lib = None

# Every symbol include/pnx.h declares (checked by tests/test_capi_host.py).
EXPORTS = [
    "pnx_create", "pnx_destroy", "pnx_last_error", "pnx_create_error", "pnx_param_count",
    "pnx_set_points", "pnx_set_ic", "pnx_set_bc", "pnx_step", "pnx_step_device", "pnx_check",
    "pnx_adam_step_device", "pnx_set_engine", "pnx_set_chunk_rows", "pnx_last_launch_count",
    "pnx_capture_residuals", "pnx_copy_residuals", "pnx_profile", "pnx_profile_read",
    "pnx_step_terms", "pnx_step_terms_device", "pnx_set_causality", "pnx_set_poynting", "pnx_last_penalty",
    "pnx_adam_step_device_state",
    "pnx_device_count", "pnx_dp_create", "pnx_dp_destroy", "pnx_dp_last_error", "pnx_dp_size", "pnx_dp_rank_ctx",
    "pnx_dp_set_points", "pnx_dp_set_ic", "pnx_dp_set_bc", "pnx_dp_set_params", "pnx_dp_get_params",
    "pnx_dp_set_optimizer", "pnx_dp_set_graph", "pnx_dp_step", "pnx_dp_step_terms", "pnx_dp_apply_gradient",
    "pnx_dp_check", "pnx_sample_points", "pnx_dp_sample_points", "pnx_copy_points",
]


class ModelDesc(C.Structure):
    _fields_ = [("in_dim", C.c_int32), ("hidden_dim", C.c_int32), ("depth", C.c_int32),
                ("out_dim", C.c_int32), ("activation", C.c_int32), ("sine_w0", C.c_double),
                ("n_periodic_axes", C.c_int32), ("periodic", C.POINTER(C.c_int32)),
                ("period", C.POINTER(C.c_double)), ("period_trainable", C.POINTER(C.c_int32)),
                ("rff_width", C.c_int32), ("rff_B", C.POINTER(C.c_double)), ("rwf", C.c_int32)]


class ProblemDesc(C.Structure):
    _fields_ = [("pde", C.c_int32), ("advection_c", C.c_double), ("epsilon", C.c_double),
                ("mu", C.c_double), ("reynolds", C.c_double), ("bc", C.c_int32)]


def load(path: str = LIB_PATH):
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} not built: run `python -m paper_2604_15645_b200.build` "
                           "(the B200 path has no CPU fallback)")
    lib = C.CDLL(path)
    vp, i32, i64, dp = C.c_void_p, C.c_int32, C.c_int64, C.POINTER(C.c_double)
    lib.pnx_create.argtypes = [C.POINTER(ModelDesc), C.POINTER(ProblemDesc), C.c_int, C.POINTER(vp)]
    lib.pnx_create.restype = C.c_int
    lib.pnx_destroy.argtypes = [vp]
    lib.pnx_destroy.restype = None
    lib.pnx_last_error.argtypes = [vp]
    lib.pnx_last_error.restype = C.c_char_p
    lib.pnx_create_error.argtypes = []
    lib.pnx_create_error.restype = C.c_char_p
    lib.pnx_param_count.argtypes = [vp, C.POINTER(i64)]
    lib.pnx_set_points.argtypes = [vp, dp, i64, i32]
    lib.pnx_set_ic.argtypes = [vp, dp, dp, i64]
    lib.pnx_set_bc.argtypes = [vp, dp, dp, dp, i64]
    lib.pnx_step.argtypes = [vp, dp, dp, dp, dp]
    lib.pnx_step_device.argtypes = [vp, vp, dp, vp, vp, vp]
    lib.pnx_check.argtypes = [vp]
    lib.pnx_adam_step_device.argtypes = [vp, vp, vp, vp, vp, i64, C.c_double, C.c_double, C.c_double,
                                         C.c_double, i64, C.c_double, vp]
    lib.pnx_set_engine.argtypes = [vp, C.c_int]
    lib.pnx_set_chunk_rows.argtypes = [vp, i64]
    lib.pnx_last_launch_count.argtypes = [vp, C.POINTER(i64)]
    lib.pnx_capture_residuals.argtypes = [vp, C.c_int]
    lib.pnx_copy_residuals.argtypes = [vp, dp]
    lib.pnx_profile.argtypes = [vp, C.c_int]
    lib.pnx_profile_read.argtypes = [vp, dp, C.POINTER(i64), C.c_int]
    lib.pnx_step_terms.argtypes = [vp, dp, dp, dp]
    lib.pnx_step_terms_device.argtypes = [vp, vp, vp, vp, vp]
    lib.pnx_set_causality.argtypes = [vp, i32, C.c_double, C.c_double, C.c_double]
    lib.pnx_set_poynting.argtypes = [vp, C.c_double, i32, i32, dp]
    lib.pnx_last_penalty.argtypes = [vp, dp]
    lib.pnx_adam_step_device_state.argtypes = [vp, vp, vp, vp, vp, i64, vp, C.c_double, C.c_double, C.c_double,
                                               C.c_double, C.c_double, C.c_double, vp]
    ip = C.POINTER(C.c_int)
    lib.pnx_device_count.argtypes = [ip]
    lib.pnx_dp_create.argtypes = [C.POINTER(ModelDesc), C.POINTER(ProblemDesc), ip, C.c_int, C.POINTER(vp)]
    lib.pnx_dp_destroy.argtypes = [vp]
    lib.pnx_dp_destroy.restype = None
    lib.pnx_dp_last_error.argtypes = [vp]
    lib.pnx_dp_last_error.restype = C.c_char_p
    lib.pnx_dp_size.argtypes = [vp, ip, ip]
    lib.pnx_dp_rank_ctx.argtypes = [vp, C.c_int, C.POINTER(vp)]
    lib.pnx_dp_set_points.argtypes = [vp, dp, i64, i32]
    lib.pnx_dp_set_ic.argtypes = [vp, dp, dp, i64]
    lib.pnx_dp_set_bc.argtypes = [vp, dp, dp, dp, i64]
    lib.pnx_dp_set_params.argtypes = [vp, dp]
    lib.pnx_dp_get_params.argtypes = [vp, C.c_int, dp]
    lib.pnx_dp_set_optimizer.argtypes = [vp] + [C.c_double] * 5
    lib.pnx_dp_set_graph.argtypes = [vp, C.c_int]
    lib.pnx_dp_step.argtypes = [vp, dp, C.c_int, dp, dp]
    lib.pnx_dp_step_terms.argtypes = [vp, dp, dp]
    lib.pnx_dp_apply_gradient.argtypes = [vp, dp]
    lib.pnx_dp_check.argtypes = [vp]
    lp = C.POINTER(C.c_int64)
    lib.pnx_sample_points.argtypes = [vp, i32, dp, lp, i64, C.c_uint64, i64, i64]
    lib.pnx_copy_points.argtypes = [vp, dp]
    lib.pnx_dp_sample_points.argtypes = [vp, i32, dp, lp, i64, C.c_uint64]
    for name in EXPORTS:
        if name not in ("pnx_destroy", "pnx_last_error", "pnx_create_error", "pnx_dp_destroy", "pnx_dp_last_error"):
            getattr(lib, name).restype = C.c_int
    _lib = lib
    return lib
