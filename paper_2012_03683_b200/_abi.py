"""ctypes mirror of the POD descriptors in include/kreg_b200.h.

Shared by the product binding (paper_2012_03683_b200.api) and the test-only
checker bindings (tests/_checkers.py), which use the same descriptor layout.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

KREG_OK = 0
KREG_INVALID_ARGUMENT = 1
KREG_NO_OVERLAP = 2
KREG_CUDA_ERROR = 3
KREG_OUT_OF_MEMORY = 4
KREG_RUNTIME_ERROR = 5
KREG_NO_DEVICE = 6
KREG_PARSE_ERROR = 7

KREG_EVAL_GRAD = 1
KREG_EVAL_DISP = 2

dptr = C.POINTER(C.c_double)
i64ptr = C.POINTER(C.c_int64)
i32ptr = C.POINTER(C.c_int32)
u8ptr = C.POINTER(C.c_uint8)


class kreg_channel(C.Structure):
    _fields_ = [("name", C.c_char_p), ("dim", C.c_int32), ("kind", C.c_int32)]


class kreg_cloud_view(C.Structure):
    _fields_ = [
        ("xyz", dptr),
        ("n", C.c_int32),
        ("features", dptr),
        ("dim", C.c_int32),
        ("channels", C.POINTER(kreg_channel)),
        ("n_channels", C.c_int32),
    ]


class kreg_channel_params(C.Structure):
    _fields_ = [("sigma", C.c_double), ("lengthscale", C.c_double), ("form", C.c_int32)]


class kreg_kernel_params(C.Structure):
    _fields_ = [
        ("sigma", C.c_double),
        ("lengthscale", C.c_double),
        ("per_channel", C.POINTER(kreg_channel_params)),
        ("n_channels", C.c_int32),
    ]


class kreg_registration_config(C.Structure):
    _fields_ = [
        ("init_lengthscale", C.c_double),
        ("subsequent_lengthscale", C.c_double),
        ("min_lengthscale", C.c_double),
        ("decay_factor", C.c_double),
        ("stabilization_window", C.c_int32),
        ("stabilization_rel_tol", C.c_double),
        ("max_iterations", C.c_int32),
        ("step_init", C.c_double),
        ("step_shrink", C.c_double),
        ("step_grow", C.c_double),
        ("max_backtracks", C.c_int32),
        ("convergence_twist_norm", C.c_double),
        ("cutoff_multiplier", C.c_double),
        ("c_min", C.c_double),
    ]


class kreg_registration_result(C.Structure):
    _fields_ = [
        ("transform", C.c_double * 12),
        ("converged", C.c_int32),
        ("iterations", C.c_int32),
        ("final_indicator", C.c_double),
        ("trace_capacity", C.c_int32),
        ("objective_trace", dptr),
        ("indicator_trace", dptr),
        ("lengthscale_trace", dptr),
        ("step_trace", dptr),
        ("twist_norm_trace", dptr),
        ("pair_count_trace", i64ptr),
        ("rebuild_trace", u8ptr),
        ("sweeps", C.c_int32),
        ("rebuilds", C.c_int32),
    ]


class kreg_sequence_result(C.Structure):
    _fields_ = [
        ("relative", dptr),
        ("trajectory", dptr),
        ("fallback", u8ptr),
        ("converged", u8ptr),
        ("final_indicator", dptr),
        ("iterations", i32ptr),
    ]


class kreg_camera_intrinsics(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("depth_scale", C.c_double), ("max_depth", C.c_double), ("skip_top_rows", C.c_int32)]


class kreg_selector_config(C.Structure):
    _fields_ = [("target_min", C.c_int32), ("target_max", C.c_int32), ("initial_threshold", C.c_double),
                ("adjust_factor", C.c_double), ("max_adjust_rounds", C.c_int32)]


class kreg_selection_info(C.Structure):
    _fields_ = [("count", C.c_int64), ("threshold", C.c_double), ("in_band", C.c_int32), ("fallback", C.c_int32),
                ("valid_pixels", C.c_int64)]


def as_ptr(a: np.ndarray, ctype=C.c_double):
    return a.ctypes.data_as(C.POINTER(ctype))


class TraceBuffers:
    """Owns numpy arrays backing a kreg_registration_result's traces."""

    def __init__(self, capacity: int):
        self.capacity = capacity
        self.objective = np.zeros(capacity)
        self.indicator = np.zeros(capacity)
        self.lengthscale = np.zeros(capacity)
        self.step = np.zeros(capacity)
        self.twist_norm = np.zeros(capacity)
        self.pair_count = np.zeros(capacity, dtype=np.int64)
        self.rebuild = np.zeros(capacity, dtype=np.uint8)
        self.struct = kreg_registration_result()
        s = self.struct
        s.trace_capacity = capacity
        s.objective_trace = as_ptr(self.objective)
        s.indicator_trace = as_ptr(self.indicator)
        s.lengthscale_trace = as_ptr(self.lengthscale)
        s.step_trace = as_ptr(self.step)
        s.twist_norm_trace = as_ptr(self.twist_norm)
        s.pair_count_trace = as_ptr(self.pair_count, C.c_int64)
        s.rebuild_trace = as_ptr(self.rebuild, C.c_uint8)
