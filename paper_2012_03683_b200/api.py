"""Python mirror of the reference's public API on top of the B200 engine.

Same names, argument order and meaning as /root/reference/proj/include/kreg/
inner_product.hpp:50-87 and registration.hpp:42-100; errors map to the
reference's exceptions (std::invalid_argument -> ValueError,
kreg::NoOverlapError -> NoOverlapError). Everything here calls the C-ABI of
libkreg_b200.so (include/kreg_b200.h); there is no CPU fallback — without the
library or a CUDA device every call raises.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
import threading

import numpy as np

from . import _abi
from .types import (CameraIntrinsics, Channel, ChannelKind, FeatureSchema, Isometry, KernelParams, PointCloud,
                    RegistrationConfig, RegistrationResult, Selection, SelectorConfig, SequenceBuffers, SequenceResult,
                    raise_for)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KREG_LIB") or os.path.join(_HERE, "libkreg_b200.so")

_lib = None
_lib_lock = threading.Lock()

P = C.c_void_p
D = C.c_double
VP = C.POINTER(_abi.kreg_cloud_view)
KP = C.POINTER(_abi.kreg_kernel_params)
CP = C.POINTER(_abi.kreg_registration_config)
RP = C.POINTER(_abi.kreg_registration_result)
VP_ = C.c_void_p
# kreg_collective_fn: int32 (*)(void*, double* sums, int32 n_sums, double* maxes, int32 n_maxes)
COLLECTIVE_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.POINTER(C.c_double), C.c_int32, C.POINTER(C.c_double),
                            C.c_int32)


def lib():
    """Load libkreg_b200.so (fails loudly when it was not built)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2012_03683_b200.build` "
                              "(the engine has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.kreg_last_error.restype = C.c_char_p
        L.kreg_abi_version.restype = C.c_int32
        L.kreg_ctx_create.argtypes = [C.c_int32, C.POINTER(P)]
        L.kreg_ctx_destroy.argtypes = [P]
        L.kreg_ctx_synchronize.argtypes = [P]
        L.kreg_ctx_kernel_launches.argtypes = [P]
        L.kreg_ctx_kernel_launches.restype = C.c_int64
        L.kreg_ctx_sweep_stats.argtypes = [P, _abi.dptr, _abi.i64ptr, _abi.i64ptr]
        L.kreg_ctx_set_profiling.argtypes = [P, C.c_int32]
        L.kreg_ctx_timer_mark.argtypes = [P, C.c_int32]
        L.kreg_ctx_screen_stats.argtypes = [P, _abi.i64ptr]
        L.kreg_ctx_timer_elapsed.argtypes = [P, _abi.dptr]
        L.kreg_ctx_set_max_active.argtypes = [P, C.c_int32]
        L.kreg_ctx_host_stats.argtypes = [P, _abi.dptr]
        L.kreg_ctx_stats.argtypes = [P, _abi.dptr]
        L.kreg_ctx_reset_stats.argtypes = [P]
        L.kreg_ctx_io_stats.argtypes = [P, _abi.i64ptr]
        L.kreg_ctx_set_memory_budget.argtypes = [P, C.c_int64]
        L.kreg_ctx_admission_stats.argtypes = [P, _abi.i64ptr]
        L.kreg_ctx_set_candidate_skin.argtypes = [P, D]
        L.kreg_ctx_set_chunk_units.argtypes = [P, C.c_int32]
        L.kreg_ctx_build_stats.argtypes = [P, _abi.i64ptr]
        L.kreg_ctx_build_profile.argtypes = [P, _abi.dptr]
        L.kreg_rebuild_pairs.argtypes = [P, P, _abi.dptr, KP, D, D, _abi.i64ptr]
        L.kreg_cloud_create.argtypes = [P, VP, C.POINTER(P)]
        L.kreg_cloud_destroy.argtypes = [P]
        L.kreg_cloud_size.argtypes = [P]
        L.kreg_cloud_read_ply.argtypes = [P, C.c_char_p, C.POINTER(P), C.c_char_p, C.c_int32]
        L.kreg_cloud_schema.argtypes = [P, _abi.i32ptr, _abi.i32ptr, _abi.i32ptr, _abi.i32ptr, C.c_int32]
        L.kreg_cloud_download.argtypes = [P, _abi.dptr, _abi.dptr]
        L.kreg_build_pairs.argtypes = [P, P, P, _abi.dptr, KP, D, D, C.POINTER(P), _abi.i64ptr]
        L.kreg_pairs_destroy.argtypes = [P]
        L.kreg_pairs_size.argtypes = [P]
        L.kreg_pairs_size.restype = C.c_int64
        L.kreg_pairs_export.argtypes = [P, P, _abi.i64ptr, _abi.i32ptr, _abi.dptr]
        L.kreg_pairs_info.argtypes = [P, _abi.i64ptr]
        L.kreg_inner_product.argtypes = [P, P, P, P, _abi.dptr, KP, _abi.dptr]
        L.kreg_objective_and_gradient.argtypes = [P, P, P, P, _abi.dptr, KP, _abi.dptr]
        L.kreg_eval_transforms.argtypes = [P, P, P, P, _abi.dptr, C.c_int32, KP, C.c_uint32, _abi.dptr]
        L.kreg_directional_terms.argtypes = [P, P, P, P, _abi.dptr, _abi.dptr, KP, _abi.dptr]
        L.kreg_evaluate_alignment.argtypes = [P, P, P, P, _abi.dptr, KP, _abi.dptr, _abi.dptr, _abi.i64ptr]
        L.kreg_indicator.argtypes = [P, P, P, _abi.dptr, KP, D, D, _abi.dptr]
        L.kreg_max_point_displacement.argtypes = [P, P, _abi.dptr, _abi.dptr, _abi.dptr]
        L.kreg_check_config.argtypes = [CP]
        L.kreg_registration_config_default.argtypes = [CP]
        L.kreg_anneal_step.argtypes = [D, _abi.dptr, C.c_int32, CP, _abi.dptr]
        L.kreg_line_search.argtypes = [P, P, P, _abi.dptr, _abi.dptr, KP, P, CP, _abi.dptr]
        L.kreg_register_clouds.argtypes = [P, P, P, _abi.dptr, KP, CP, RP]
        L.kreg_register_clouds_host.argtypes = [P, VP, VP, _abi.dptr, KP, CP, RP]
        L.kreg_register_batch.argtypes = [P, C.c_int32, C.POINTER(P), C.POINTER(P), _abi.dptr, KP, CP, RP, _abi.i32ptr]
        L.kreg_register_batch_host.argtypes = [P, C.c_int32, VP, VP, _abi.dptr, KP, CP, RP, _abi.i32ptr]
        L.kreg_register_sequence.argtypes = [P, C.POINTER(P), C.c_int32, KP, CP, C.POINTER(_abi.kreg_sequence_result)]
        L.kreg_register_sequence_chains.argtypes = [P, C.POINTER(P), C.c_int32, C.c_int32, KP, CP,
                                                    C.POINTER(_abi.kreg_sequence_result)]
        L.kreg_register_sequence_host.argtypes = [P, C.POINTER(_abi.kreg_cloud_view), C.c_int32, C.c_int32, KP, CP,
                                                  C.POINTER(_abi.kreg_sequence_result)]
        L.kreg_register_sequence_spans.argtypes = [P, C.POINTER(P), C.c_int32, _abi.i32ptr, _abi.i32ptr, C.c_int32, KP,
                                                   CP, C.POINTER(_abi.kreg_sequence_result)]
        L.kreg_register_clouds_rows.argtypes = [P, P, P, C.c_int64, _abi.dptr, KP, CP, RP]
        L.kreg_ctx_set_collective.argtypes = [P, COLLECTIVE_FN, VP_]
        L.kreg_nccl_unique_id.argtypes = [C.c_void_p]
        L.kreg_ctx_set_nccl.argtypes = [P, C.c_void_p, C.c_int32, C.c_int32, C.c_int32]
        L.kreg_ctx_nccl_calls.argtypes = [P]
        L.kreg_ctx_nccl_calls.restype = C.c_int64
        L.kreg_exact_cosine.argtypes = [P, VP, VP, _abi.dptr, KP, _abi.dptr, _abi.dptr]
        L.kreg_select_points.argtypes = [P, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                         C.POINTER(_abi.kreg_selector_config), C.c_void_p, C.c_int64,
                                         C.POINTER(_abi.kreg_selection_info)]
        L.kreg_depth_rgb_to_cloud.argtypes = [P, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int32,
                                              C.c_int32, C.POINTER(_abi.kreg_camera_intrinsics),
                                              C.POINTER(_abi.kreg_selector_config), _abi.dptr, _abi.dptr, C.c_int64,
                                              C.POINTER(_abi.kreg_selection_info)]
        L.kreg_indicator_sweep.argtypes = [P, VP, KP, C.c_int32, D, C.c_int32, D, D, _abi.dptr, _abi.dptr]
        L.kreg_se3_exp.argtypes = [_abi.dptr, _abi.dptr]
        L.kreg_se3_compose.argtypes = [_abi.dptr, _abi.dptr, _abi.dptr]
        L.kreg_se3_inverse.argtypes = [_abi.dptr, _abi.dptr]
        L.kreg_cloud_diameter.argtypes = [VP]
        L.kreg_cloud_diameter.restype = D
        _lib = L
        return L


def _check(rc: int):
    if rc != 0:
        raise_for(rc, lib().kreg_last_error().decode())


def _t12(T):
    a = T.as12() if isinstance(T, Isometry) else np.ascontiguousarray(np.asarray(T, dtype=np.float64).reshape(12))
    return a, _abi.as_ptr(a)


class Context:
    """One CUDA device + stream (kreg_ctx). Not thread-safe."""

    def __init__(self, device: int = 0):
        h = P()
        _check(lib().kreg_ctx_create(int(device), C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            lib().kreg_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self):
        _check(lib().kreg_ctx_synchronize(self.h))

    def kernel_launches(self) -> int:
        return int(lib().kreg_ctx_kernel_launches(self.h))

    def set_profiling(self, on: bool):
        _check(lib().kreg_ctx_set_profiling(self.h, int(on)))

    def screen_stats(self) -> dict:
        """Displacement screen: sweep requests asked / answered by the bound."""
        out = np.zeros(2, dtype=np.int64)
        _check(lib().kreg_ctx_screen_stats(self.h, _abi.as_ptr(out, C.c_int64)))
        return {"asked": int(out[0]), "screened": int(out[1])}

    def timer_mark(self, which: int):
        """Record the start (0) / stop (1) CUDA event on the context's stream."""
        _check(lib().kreg_ctx_timer_mark(self.h, int(which)))

    def timer_ms(self) -> float:
        """Device milliseconds between the start and stop marks."""
        v = C.c_double()
        _check(lib().kreg_ctx_timer_elapsed(self.h, C.byref(v)))
        return v.value

    def reset_stats(self):
        _check(lib().kreg_ctx_reset_stats(self.h))

    def set_max_active(self, n: int):
        """Lockstep window of register_batch (0 = all registrations at once)."""
        _check(lib().kreg_ctx_set_max_active(self.h, int(n)))

    def set_candidate_skin(self, skin: float):
        """Candidate-list radius R_s = cutoff * (1 + skin); 0 = grid search every build."""
        _check(lib().kreg_ctx_set_candidate_skin(self.h, float(skin)))

    def set_chunk_units(self, units: int):
        """Sweep chunk size (2-step units) of lists built from now on: 48 for
        throughput (default), ~10 for single-registration latency."""
        _check(lib().kreg_ctx_set_chunk_units(self.h, int(units)))

    def build_stats(self):
        out = np.zeros(2, dtype=np.int64)
        _check(lib().kreg_ctx_build_stats(self.h, _abi.as_ptr(out, C.c_int64)))
        prof = np.zeros(9)
        _check(lib().kreg_ctx_build_profile(self.h, _abi.as_ptr(prof)))
        return {"grid_builds": int(out[0]), "filter_builds": int(out[1]), "build_ms": float(prof[0]),
                "build_rounds": int(prof[1]), "filter_entries": int(prof[2]), "built_slots": int(prof[3]),
                "grid_why": {"no_list": int(prof[4]), "forced": int(prof[5]), "moved": int(prof[6]),
                             "other": int(prof[7])}, "refilter_builds": int(prof[8])}

    def host_stats(self):
        out = np.zeros(8)
        _check(lib().kreg_ctx_host_stats(self.h, _abi.as_ptr(out)))
        return {"rounds": int(out[0]), "t_prepare_s": float(out[1]), "t_wait_s": float(out[2]),
                "t_build_prep_s": float(out[3]), "t_sweep_prep_s": float(out[4]), "t_solver_s": float(out[5]),
                "device_allocs": int(out[6]), "device_alloc_s": float(out[7])}

    def set_memory_budget(self, nbytes: int):
        """Workspace bytes registrations may hold at once (0 = free device memory)."""
        _check(lib().kreg_ctx_set_memory_budget(self.h, int(nbytes)))

    def admission_stats(self):
        out = np.zeros(2, dtype=np.int64)
        _check(lib().kreg_ctx_admission_stats(self.h, _abi.as_ptr(out, C.c_int64)))
        return {"peak_in_flight": int(out[0]), "deferred": int(out[1])}

    def io_stats(self):
        out = np.zeros(2, dtype=np.int64)
        _check(lib().kreg_ctx_io_stats(self.h, _abi.as_ptr(out, C.c_int64)))
        return {"h2d_bytes": int(out[0]), "d2h_bytes": int(out[1])}

    def sweep_stats(self):
        o = np.zeros(8)
        _check(lib().kreg_ctx_stats(self.h, _abi.as_ptr(o)))
        return {"sweep_ms": float(o[0]), "sweep_rounds": int(o[1]), "pair_evals": int(o[2]),
                "pairs_streamed": int(o[3]), "slots_streamed": int(o[4]), "rounds": int(o[5])}


_default_ctx = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(int(os.environ.get("KREG_DEVICE", "0")))
    return _default_ctx


class DeviceCloud:
    """Device-resident SoA copy of a PointCloud (kreg_cloud)."""

    def __init__(self, cloud: PointCloud, ctx: Context | None = None, handle=None):
        self.ctx = ctx or default_context()
        self.cloud = cloud
        if handle is None:
            handle = P()
            _check(lib().kreg_cloud_create(self.ctx.h, cloud.view(), C.byref(handle)))
        self.h = handle

    def size(self):
        return self.cloud.size()

    def __del__(self):
        try:
            lib().kreg_cloud_destroy(self.h)
        except Exception:
            pass


_KIND_NAMES = {0: "color", 1: "intensity", 2: "semantic", 3: "custom"}


def read_ply(path: str, ctx: Context | None = None, warnings: list | None = None) -> DeviceCloud:
    """read_cloud for .ply (cloud_io.cpp:141-297) straight into a device cloud:
    the vertex block is read once into pinned memory and decoded, ordered and
    laid out on the device. `.cloud` is the host view (positions exact,
    features the device's FP32 values). Raises ParseError like the reference."""
    from .types import Channel, ChannelKind, FeatureSchema
    ctx = ctx or default_context()
    h = P()
    wbuf = C.create_string_buffer(1 << 16)
    _check(lib().kreg_cloud_read_ply(ctx.h, os.fsencode(path), C.byref(h), wbuf, len(wbuf)))
    if warnings is not None:
        warnings.extend(w for w in wbuf.value.decode().split("\n") if w)
    n = lib().kreg_cloud_size(h)
    dim, nch = np.zeros(1, np.int32), np.zeros(1, np.int32)
    dims, kinds = np.zeros(8, np.int32), np.zeros(8, np.int32)
    _check(lib().kreg_cloud_schema(h, _abi.as_ptr(dim, C.c_int32), _abi.as_ptr(nch, C.c_int32),
                                   _abi.as_ptr(dims, C.c_int32), _abi.as_ptr(kinds, C.c_int32), 8))
    xyz = np.zeros((n, 3))
    feat = np.zeros((n, int(dim[0])))
    _check(lib().kreg_cloud_download(h, _abi.as_ptr(xyz), _abi.as_ptr(feat) if dim[0] else None))
    schema = FeatureSchema([Channel(_KIND_NAMES[int(kinds[k])], int(dims[k]), ChannelKind(int(kinds[k])))
                            for k in range(int(nch[0]))])
    return DeviceCloud(PointCloud(xyz, schema, feat), ctx, handle=h)


def device_cloud(c, ctx: Context | None = None) -> DeviceCloud:
    """Upload once per (cloud, context); PointCloud is immutable."""
    if isinstance(c, DeviceCloud):
        return c
    ctx = ctx or default_context()
    cache = c.__dict__.setdefault("_device", {})
    dc = cache.get(id(ctx))
    if dc is None:
        dc = DeviceCloud(c, ctx)
        cache[id(ctx)] = dc
    return dc


class PairList:
    """kreg::PairList (inner_product.hpp:18-32), device resident."""

    def __init__(self, h, X: DeviceCloud, Z: DeviceCloud, n: int, params: KernelParams, T, cutoff_multiplier, c_min):
        self.h, self.X, self.Z = h, X, Z
        self.n = n
        self.built_at_lengthscale = params.lengthscale
        self.cutoff_radius = cutoff_multiplier * params.lengthscale
        self.c_min = c_min
        self.build_transform = T if isinstance(T, Isometry) else Isometry.from12(T)
        self.n_x = X.size()
        self.n_z = Z.size()

    def size(self) -> int:
        return self.n

    def empty(self) -> bool:
        return self.n == 0

    def rebuild(self, T, params: KernelParams, cutoff_multiplier: float, c_min: float) -> "PairList":
        """build_pairs(X, Z, T, ...) into this list (registration.cpp:126), reusing
        its candidate list when that provably covers the new list."""
        t, tp = _t12(T)
        n = C.c_int64()
        _check(lib().kreg_rebuild_pairs(self.X.ctx.h, self.h, tp, params.cstruct(), cutoff_multiplier, c_min,
                                        C.byref(n)))
        self.n = n.value
        self.built_at_lengthscale = params.lengthscale
        self.cutoff_radius = cutoff_multiplier * params.lengthscale
        self.c_min = c_min
        self.build_transform = T if isinstance(T, Isometry) else Isometry.from12(T)
        return self

    def info(self) -> dict:
        """Device layout: pairs, sliced-ELL slots (incl. padding), tiles, grid cells."""
        out = np.zeros(4, dtype=np.int64)
        _check(lib().kreg_pairs_info(self.h, _abi.as_ptr(out, C.c_int64)))
        return {"pairs": int(out[0]), "slots": int(out[1]), "tiles": int(out[2]), "cells": int(out[3])}

    def export(self):
        """(offsets, x_index, coeff) in the reference layout."""
        off = np.zeros(self.n_z + 1, dtype=np.int64)
        idx = np.zeros(max(self.n, 1), dtype=np.int32)
        cf = np.zeros(max(self.n, 1))
        _check(lib().kreg_pairs_export(self.X.ctx.h, self.h, _abi.as_ptr(off, C.c_int64), _abi.as_ptr(idx, C.c_int32),
                                       _abi.as_ptr(cf)))
        return off, idx[: self.n], cf[: self.n]

    def __del__(self):
        try:
            lib().kreg_pairs_destroy(self.h)
        except Exception:
            pass


@dataclasses.dataclass
class Evaluation:
    value: float
    grad: np.ndarray  # twist (omega[3], v[3])


@dataclasses.dataclass
class AlignmentReport:
    value_F: float
    indicator: float
    pair_count: int


def build_pairs(X, Z, T, params: KernelParams, cutoff_multiplier: float, c_min: float, ctx=None) -> PairList:
    dx, dz = device_cloud(X, ctx), device_cloud(Z, ctx)
    t, tp = _t12(T)
    h = P()
    n = C.c_int64()
    _check(lib().kreg_build_pairs(dx.ctx.h, dx.h, dz.h, tp, params.cstruct(), cutoff_multiplier, c_min, C.byref(h),
                                  C.byref(n)))
    return PairList(h, dx, dz, n.value, params, T, cutoff_multiplier, c_min)


def eval_transforms(pairs: PairList, X, Z, Ts, params: KernelParams) -> np.ndarray:
    """K transforms in one device pass -> (K, 8): F, omega, v, displacement."""
    dx, dz = device_cloud(X, pairs.X.ctx), device_cloud(Z, pairs.X.ctx)
    Ts = [T.as12() if isinstance(T, Isometry) else np.asarray(T, dtype=np.float64).reshape(12) for T in Ts]
    arr = np.ascontiguousarray(np.stack(Ts)) if Ts else np.zeros((0, 12))
    out = np.zeros((len(Ts), 8))
    _check(lib().kreg_eval_transforms(dx.ctx.h, pairs.h, dx.h, dz.h, _abi.as_ptr(arr), len(Ts), params.cstruct(),
                                      _abi.KREG_EVAL_GRAD | _abi.KREG_EVAL_DISP, _abi.as_ptr(out)))
    return out


def inner_product(pairs: PairList, X, Z, T, params: KernelParams) -> float:
    return float(eval_transforms(pairs, X, Z, [T], params)[0, 0])


def objective_and_gradient(pairs: PairList, X, Z, T, params: KernelParams) -> Evaluation:
    o = eval_transforms(pairs, X, Z, [T], params)[0]
    return Evaluation(float(o[0]), o[1:7].copy())


def directional_terms(pairs: PairList, X, Z, T, xi, params: KernelParams) -> np.ndarray:
    """{F, dF/d eps, d2F/d eps2} at eps = 0 for F(eps) = inner_product at
    exp(eps xi) T, pair list fixed: the second-order step-size terms (a
    diagnostic; no reference counterpart)."""
    t, tp = _t12(T)
    x = np.ascontiguousarray(np.asarray(xi, dtype=np.float64).reshape(6))
    out = np.zeros(3)
    _check(lib().kreg_directional_terms(pairs.X.ctx.h, pairs.h, pairs.X.h, pairs.Z.h, tp, _abi.as_ptr(x),
                                        params.cstruct(), _abi.as_ptr(out)))
    return out


def gradient(pairs, X, Z, T, params) -> np.ndarray:
    return objective_and_gradient(pairs, X, Z, T, params).grad


def evaluate_alignment(pairs: PairList, X, Z, T, params: KernelParams) -> AlignmentReport:
    F = inner_product(pairs, X, Z, T, params)
    denom = np.sqrt(float(pairs.n_x) * float(pairs.n_z))
    return AlignmentReport(F, F / denom if denom > 0 else 0.0, pairs.size())


def indicator(X, Z, T, params: KernelParams, cutoff_multiplier: float = 3.0, c_min: float = 1e-4, ctx=None) -> float:
    dx, dz = device_cloud(X, ctx), device_cloud(Z, ctx)
    t, tp = _t12(T)
    out = np.zeros(1)
    _check(lib().kreg_indicator(dx.ctx.h, dx.h, dz.h, tp, params.cstruct(), cutoff_multiplier, c_min, _abi.as_ptr(out)))
    return float(out[0])


def max_point_displacement(Z, built, now, ctx=None) -> float:
    dz = device_cloud(Z, ctx)
    a, ap = _t12(built)
    b, bp = _t12(now)
    out = np.zeros(1)
    _check(lib().kreg_max_point_displacement(dz.ctx.h, dz.h, ap, bp, _abi.as_ptr(out)))
    return float(out[0])


def check_config(config: RegistrationConfig):
    _check(lib().kreg_check_config(C.byref(config.cstruct())))


def anneal_step(lengthscale: float, history, config: RegistrationConfig) -> float:
    h = np.ascontiguousarray(history, dtype=np.float64)
    out = np.zeros(1)
    _check(lib().kreg_anneal_step(lengthscale, _abi.as_ptr(h), len(h), C.byref(config.cstruct()), _abi.as_ptr(out)))
    return float(out[0])


def line_search(X, Z, T, g, params: KernelParams, pairs: PairList, config: RegistrationConfig) -> float:
    dx, dz = device_cloud(X, pairs.X.ctx), device_cloud(Z, pairs.X.ctx)
    t, tp = _t12(T)
    gg = np.ascontiguousarray(g, dtype=np.float64)
    out = np.zeros(1)
    _check(lib().kreg_line_search(dx.ctx.h, dx.h, dz.h, tp, _abi.as_ptr(gg), params.cstruct(), pairs.h,
                                  C.byref(config.cstruct()), _abi.as_ptr(out)))
    return float(out[0])


def register_clouds(X, Z, initial, params: KernelParams, config: RegistrationConfig, ctx=None,
                    trace_capacity: int | None = None) -> RegistrationResult:
    dx, dz = device_cloud(X, ctx), device_cloud(Z, ctx)
    buf = _abi.TraceBuffers(trace_capacity or config.max_iterations)
    t, tp = _t12(initial)
    cfg = config.cstruct()
    _check(lib().kreg_register_clouds(dx.ctx.h, dx.h, dz.h, tp, params.cstruct(), C.byref(cfg), C.byref(buf.struct)))
    return RegistrationResult.from_buffers(buf)


def register_clouds_host(X: PointCloud, Z: PointCloud, initial, params: KernelParams, config: RegistrationConfig,
                         ctx=None, trace_capacity: int | None = None) -> RegistrationResult:
    """End-to-end call: host clouds in, uploads inside the call."""
    ctx = ctx or default_context()
    buf = _abi.TraceBuffers(trace_capacity or config.max_iterations)
    t, tp = _t12(initial)
    cfg = config.cstruct()
    _check(lib().kreg_register_clouds_host(ctx.h, X.view(), Z.view(), tp, params.cstruct(), C.byref(cfg),
                                           C.byref(buf.struct)))
    return RegistrationResult.from_buffers(buf)


def register_batch(Xs, Zs, initials, params: KernelParams, config: RegistrationConfig, ctx=None,
                   trace_capacity: int | None = None):
    """Independent registrations in lockstep on one device.
    Returns (results, statuses); results[k] is None when statuses[k] != 0."""
    ctx = ctx or default_context()
    n = len(Xs)
    dxs = [device_cloud(x, ctx) for x in Xs]
    dzs = [device_cloud(z, ctx) for z in Zs]
    xh = (P * n)(*[d.h for d in dxs])
    zh = (P * n)(*[d.h for d in dzs])
    inits = np.ascontiguousarray(np.stack([T.as12() if isinstance(T, Isometry) else np.asarray(T, np.float64).reshape(12)
                                           for T in initials])) if n else np.zeros((0, 12))
    bufs = [_abi.TraceBuffers(trace_capacity or config.max_iterations) for _ in range(n)]
    res = (_abi.kreg_registration_result * max(n, 1))(*[b.struct for b in bufs])
    st = np.zeros(max(n, 1), dtype=np.int32)
    cfg = config.cstruct()
    _check(lib().kreg_register_batch(ctx.h, n, xh, zh, _abi.as_ptr(inits), params.cstruct(), C.byref(cfg), res,
                                     _abi.as_ptr(st, C.c_int32)))
    out = []
    for k in range(n):
        bufs[k].struct = res[k]
        out.append(RegistrationResult.from_buffers(bufs[k]) if st[k] == 0 else None)
    return out, st[:n].copy()


def register_batch_host(Xs, Zs, initials, params: KernelParams, config: RegistrationConfig, ctx=None,
                        trace_capacity: int | None = None):
    """End-to-end throughput call: host clouds in (uploaded inside the call).
    Returns (results, statuses)."""
    ctx = ctx or default_context()
    n = len(Xs)
    xv = (_abi.kreg_cloud_view * max(n, 1))(*[x.view() for x in Xs])
    zv = (_abi.kreg_cloud_view * max(n, 1))(*[z.view() for z in Zs])
    inits = np.ascontiguousarray(np.stack([T.as12() if isinstance(T, Isometry) else np.asarray(T, np.float64).reshape(12)
                                           for T in initials])) if n else np.zeros((0, 12))
    bufs = [_abi.TraceBuffers(trace_capacity or config.max_iterations) for _ in range(n)]
    res = (_abi.kreg_registration_result * max(n, 1))(*[b.struct for b in bufs])
    st = np.zeros(max(n, 1), dtype=np.int32)
    cfg = config.cstruct()
    _check(lib().kreg_register_batch_host(ctx.h, n, xv, zv, _abi.as_ptr(inits), params.cstruct(), C.byref(cfg), res,
                                          _abi.as_ptr(st, C.c_int32)))
    out = []
    for k in range(n):
        bufs[k].struct = res[k]
        out.append(RegistrationResult.from_buffers(bufs[k]) if st[k] == 0 else None)
    return out, st[:n].copy()


def register_sequence(frames, params: KernelParams, config: RegistrationConfig, ctx=None,
                      chains: int | None = None) -> SequenceResult:
    ctx = ctx or default_context()
    n = len(frames)
    ds = [device_cloud(f, ctx) for f in frames]
    fh = (P * max(n, 1))(*[d.h for d in ds])
    sb = SequenceBuffers(max(n, 1))
    cfg = config.cstruct()
    if chains is None:
        _check(lib().kreg_register_sequence(ctx.h, fh, n, params.cstruct(), C.byref(cfg), C.byref(sb.struct)))
    else:
        _check(lib().kreg_register_sequence_chains(ctx.h, fh, n, int(chains), params.cstruct(), C.byref(cfg),
                                                   C.byref(sb.struct)))
    return sb.result()


def register_sequence_host(frames, params: KernelParams, config: RegistrationConfig, ctx=None,
                           chains: int = 1) -> SequenceResult:
    """End-to-end sequence call: host frames in, uploaded inside the call
    while the first pairs run (chains = 1: register_sequence's semantics)."""
    ctx = ctx or default_context()
    n = len(frames)
    fv = (_abi.kreg_cloud_view * max(n, 1))(*[f.view() for f in frames])
    sb = SequenceBuffers(max(n, 1))
    cfg = config.cstruct()
    _check(lib().kreg_register_sequence_host(ctx.h, fv, n, int(chains), params.cstruct(), C.byref(cfg),
                                             C.byref(sb.struct)))
    return sb.result()


def register_sequence_spans(frames, spans, params: KernelParams, config: RegistrationConfig, ctx=None) -> SequenceResult:
    """Chains over explicit pair spans [(begin, end), ...] (pair p registers
    frame p -> p + 1): a rank's share of a distributed sequence (parallel.py).
    Pairs outside the spans come back as identity, fallback 0, 0 iterations."""
    ctx = ctx or default_context()
    n = len(frames)
    ds = [device_cloud(f, ctx) for f in frames]
    fh = (P * max(n, 1))(*[d.h for d in ds])
    sb = SequenceBuffers(max(n, 1))
    cfg = config.cstruct()
    b = np.ascontiguousarray([s[0] for s in spans], dtype=np.int32)
    e = np.ascontiguousarray([s[1] for s in spans], dtype=np.int32)
    _check(lib().kreg_register_sequence_spans(ctx.h, fh, n, _abi.as_ptr(b, C.c_int32), _abi.as_ptr(e, C.c_int32),
                                              len(spans), params.cstruct(), C.byref(cfg), C.byref(sb.struct)))
    return sb.result()


def register_clouds_rows(X, Z_rows, n_z_total: int, initial, params: KernelParams, config: RegistrationConfig,
                         ctx=None, collective=None, trace_capacity: int | None = None) -> RegistrationResult:
    """One rank's share of a row-sharded registration: Z_rows
    are this rank's source rows, n_z_total the whole source's size. Every
    round's sums / maxima are combined through `collective` (a kreg_collective_fn
    wrapper, e.g. parallel.TorchCollective), so all ranks run the identical
    replicated host loop."""
    ctx = ctx or default_context()
    dx, dz = device_cloud(X, ctx), device_cloud(Z_rows, ctx)
    t, tp = _t12(initial)
    buf = _abi.TraceBuffers(trace_capacity or config.max_iterations)
    cfg = config.cstruct()
    if getattr(collective, "native", False):  # parallel.NcclCollective: NCCL inside the engine
        collective.attach(ctx)
    else:
        fn = collective.c_fn if collective is not None else COLLECTIVE_FN()
        _check(lib().kreg_ctx_set_collective(ctx.h, fn, None))
    try:
        _check(lib().kreg_register_clouds_rows(ctx.h, dx.h, dz.h, int(n_z_total), tp, params.cstruct(), C.byref(cfg),
                                               C.byref(buf.struct)))
    finally:
        if not getattr(collective, "native", False):  # an NCCL communicator stays with its context
            lib().kreg_ctx_set_collective(ctx.h, COLLECTIVE_FN(), None)
    return RegistrationResult.from_buffers(buf)


def indicator_sweep(cloud: PointCloud, params: KernelParams, axis: str, range_: float, steps: int,
                    cutoff_multiplier: float = 3.0, c_min: float = 1e-4, ctx=None):
    """reference eval.cpp:198-235: [(magnitude, indicator)] of the cloud against
    perturbed copies of itself (axis "rotation" about z through the centroid, or
    "translation" along +x); one batched device round."""
    ctx = ctx or default_context()
    if axis not in ("rotation", "translation"):
        raise ValueError("indicator_sweep: axis must be 'rotation' or 'translation'")
    n = max(int(steps), 1)
    mags, inds = np.zeros(n), np.zeros(n)
    _check(lib().kreg_indicator_sweep(ctx.h, cloud.view(), params.cstruct(), 0 if axis == "rotation" else 1,
                                      float(range_), int(steps), float(cutoff_multiplier), float(c_min),
                                      _abi.as_ptr(mags), _abi.as_ptr(inds)))
    k = 1 if range_ == 0.0 else int(steps)
    return list(zip(mags[:k].tolist(), inds[:k].tolist()))


def exact_cosine(X: PointCloud, Z: PointCloud, T, params: KernelParams, ctx=None, parts: bool = False):
    """reference inner_product.cpp:203-236: dense all-pairs cosine between f_X
    and f_TZ, FP64 on the device (K4). parts=True also returns (cross,
    |f_X|^2, |f_Z|^2)."""
    ctx = ctx or default_context()
    t, tp = _t12(T)
    out = np.zeros(1)
    pr = np.zeros(3)
    _check(lib().kreg_exact_cosine(ctx.h, X.view(), Z.view(), tp, params.cstruct(), _abi.as_ptr(out), _abi.as_ptr(pr)))
    return (float(out[0]), tuple(pr)) if parts else float(out[0])


def _selection_note(info, sel) -> str:
    # selector.cpp:112-123 (the reference's warning strings)
    if info.fallback:
        return (f"selector fallback: {info.valid_pixels} valid-depth pixels returned without corner filtering")
    if not info.in_band:
        return f"selector accepted out-of-band count {info.count} after {sel.max_adjust_rounds} rounds"
    return ""


def _image_u8(rgb):
    a = np.ascontiguousarray(rgb, dtype=np.uint8)
    if a.ndim == 2:
        a = a[:, :, None]
    if a.ndim != 3 or a.shape[2] not in (1, 3):
        raise ValueError("image: expected h x w (x 1 or 3) uint8")
    return a


def select_points(rgb, valid_depth, sel: SelectorConfig | None = None, ctx=None) -> Selection:
    """reference selector.cpp:63-125 (budgeted FAST corners over valid-depth
    pixels): FAST scores and their histogram on the device, the reference's
    threshold rounds replayed from the histogram, ordered compaction."""
    ctx = ctx or default_context()
    sel = sel or SelectorConfig()
    img = _image_u8(rgb)
    h, w, ch = img.shape
    mask = np.ascontiguousarray(valid_depth, dtype=np.uint8)
    if mask.size != w * h:
        raise ValueError("select_points: mask size does not match image")
    info = _abi.kreg_selection_info()
    cs = sel.cstruct()
    _check(lib().kreg_select_points(ctx.h, img.ctypes.data_as(C.c_void_p), ch, w, h, mask.ctypes.data_as(C.c_void_p),
                                    C.byref(cs), None, 0, C.byref(info)))
    px = np.zeros((max(info.count, 1), 2), dtype=np.int32)
    if info.count:
        _check(lib().kreg_select_points(ctx.h, img.ctypes.data_as(C.c_void_p), ch, w, h,
                                        mask.ctypes.data_as(C.c_void_p), C.byref(cs), px.ctypes.data_as(C.c_void_p),
                                        info.count, C.byref(info)))
    return Selection(pixels=[(int(u), int(v)) for u, v in px[:info.count]], threshold=float(info.threshold),
                     in_band=bool(info.in_band), note=_selection_note(info, sel))


def depth_rgb_to_cloud(depth, rgb, semantics, intr: CameraIntrinsics, sel: SelectorConfig | None = None, ctx=None,
                       warnings: list | None = None) -> PointCloud:
    """reference projection.cpp:30-75: valid-depth pixels (row >= skip_top_rows,
    d != 0, d * scale <= max_depth) -> budgeted FAST selection -> back-projected
    cloud with colour (rgb / 255) and optional class-probability channels,
    bit-identical to the reference, on the device."""
    ctx = ctx or default_context()
    sel = sel or SelectorConfig()
    d = np.ascontiguousarray(depth, dtype=np.uint16)
    img = _image_u8(rgb)
    if d.shape != img.shape[:2]:
        raise ValueError("depth_rgb_to_cloud: depth and rgb resolutions differ")
    h, w, ch = img.shape
    sem = None
    n_sem = 0
    if semantics is not None:
        sem = np.ascontiguousarray(semantics, dtype=np.float32)
        if sem.ndim == 2:
            sem = sem[:, :, None]
        if sem.shape[:2] != d.shape:
            raise ValueError("depth_rgb_to_cloud: semantics resolution differs")
        n_sem = sem.shape[2]
    info = _abi.kreg_selection_info()
    ci, cs = intr.cstruct(), sel.cstruct()
    sem_p = sem.ctypes.data_as(C.c_void_p) if sem is not None else None
    # one call when the selection fits the guess (the band's upper end, or the
    # previous frame's count); otherwise a second call with the exact size
    cap = max(int(sel.target_max), getattr(ctx, "_ingest_cap", 0))
    for _ in range(2):
        xyz = np.zeros((cap, 3))
        feat = np.zeros((cap, 3 + n_sem))
        _check(lib().kreg_depth_rgb_to_cloud(ctx.h, d.ctypes.data_as(C.c_void_p), img.ctypes.data_as(C.c_void_p), ch,
                                             sem_p, n_sem, w, h, C.byref(ci), C.byref(cs), _abi.as_ptr(xyz),
                                             _abi.as_ptr(feat), cap, C.byref(info)))
        n = int(info.count)
        if n <= cap:
            break
        cap = n
    ctx._ingest_cap = max(getattr(ctx, "_ingest_cap", 0), n)
    note = _selection_note(info, sel)
    if warnings is not None and note:
        warnings.append(note)
    chans = [Channel("color", 3, ChannelKind.color)]
    if n_sem:
        chans.append(Channel("semantic", n_sem, ChannelKind.semantic))
    return PointCloud(xyz[:n], FeatureSchema(chans), feat[:n])


def se3_exp(xi) -> Isometry:
    xi = np.ascontiguousarray(xi, dtype=np.float64)
    out = np.zeros(12)
    _check(lib().kreg_se3_exp(_abi.as_ptr(xi), _abi.as_ptr(out)))
    return Isometry.from12(out)


def se3_compose(a, b) -> Isometry:
    x, xp = _t12(a)
    y, yp = _t12(b)
    out = np.zeros(12)
    lib().kreg_se3_compose(xp, yp, _abi.as_ptr(out))
    return Isometry.from12(out)
