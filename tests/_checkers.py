"""TEST INFRASTRUCTURE: ctypes bindings to the two CPU checkers.

  oracle/liboracle.so       plain-C restatement (oracle/kreg_oracle.c)
  oracle/_ref/libkreg_ref.so the unmodified reference compiled from its sources
                             (oracle/Makefile; present only where the reference
                             tree was available at build time)

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2012_03683_b200 import _abi
from paper_2012_03683_b200.types import (Isometry, KernelParams, PointCloud, RegistrationConfig,
                                         RegistrationResult, SequenceBuffers, raise_for)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libkreg_ref.so")

D = C.c_double
P = C.c_void_p
VP = C.POINTER(_abi.kreg_cloud_view)
KP = C.POINTER(_abi.kreg_kernel_params)
CP = C.POINTER(_abi.kreg_registration_config)
RP = C.POINTER(_abi.kreg_registration_result)


def _img(rgb):
    a = np.ascontiguousarray(rgb, dtype=np.uint8)
    return a[:, :, None] if a.ndim == 2 else a


def _d12(T):
    a = (T.as12() if isinstance(T, Isometry) else np.ascontiguousarray(T, dtype=np.float64).reshape(12))
    return a, _abi.as_ptr(a)


def build_oracle():
    if not os.path.exists(ORACLE_SO):
        subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "oracle"])


class Oracle:
    """Plain-C restatement (kreg_oracle.h)."""

    def __init__(self):
        build_oracle()
        L = self.lib = C.CDLL(ORACLE_SO)
        L.ko_last_error.restype = C.c_char_p
        L.ko_build_pairs.argtypes = [VP, VP, _abi.dptr, KP, D, D, C.c_int, C.POINTER(P), C.POINTER(C.c_int64)]
        L.ko_pairs_destroy.argtypes = [P]
        L.ko_pairs_export.argtypes = [P, _abi.i64ptr, _abi.i32ptr, _abi.dptr]
        L.ko_inner_product.argtypes = [P, VP, VP, _abi.dptr, KP]
        L.ko_inner_product.restype = D
        L.ko_objective_and_gradient.argtypes = [P, VP, VP, _abi.dptr, KP, _abi.dptr]
        L.ko_max_point_displacement.argtypes = [VP, _abi.dptr, _abi.dptr]
        L.ko_directional_terms.argtypes = [P, VP, VP, _abi.dptr, _abi.dptr, KP, _abi.dptr]
        L.ko_max_point_displacement.restype = D
        L.ko_diameter.argtypes = [VP]
        L.ko_diameter.restype = D
        L.ko_anneal_step.argtypes = [D, _abi.dptr, C.c_int, CP]
        L.ko_anneal_step.restype = D
        L.ko_register_clouds.argtypes = [VP, VP, _abi.dptr, KP, CP, RP]
        L.ko_se3_exp.argtypes = [_abi.dptr, _abi.dptr]
        L.ko_se3_compose.argtypes = [_abi.dptr, _abi.dptr, _abi.dptr]
        L.ko_se3_inverse.argtypes = [_abi.dptr, _abi.dptr]
        L.ko_feature_coefficient.argtypes = [_abi.dptr, _abi.dptr, VP, KP]
        L.ko_feature_coefficient.restype = D
        L.ko_set_iteration_log.argtypes = [P, P, P, C.c_int]

    def _err(self, rc):
        raise_for(rc, self.lib.ko_last_error().decode())

    # frame ingest (selector.cpp / projection.cpp restated in C)
    def select_points(self, rgb, valid, sel):
        img = _img(rgb)
        h, w, ch = img.shape
        m = np.ascontiguousarray(valid, dtype=np.uint8)
        px = np.zeros((w * h + 1, 2), dtype=np.int32)
        thr, ib, fb = C.c_double(), C.c_int(), C.c_int()
        cs = sel.cstruct()
        L = self.lib
        L.ko_select_points.restype = C.c_long
        n = L.ko_select_points(img.ctypes.data_as(C.c_void_p), ch, w, h, m.ctypes.data_as(C.c_void_p), C.byref(cs),
                               px.ctypes.data_as(C.c_void_p), C.byref(thr), C.byref(ib), C.byref(fb))
        return [tuple(map(int, p)) for p in px[:n]], thr.value, bool(ib.value), bool(fb.value)

    def depth_rgb_to_cloud(self, depth, rgb, sem, intr, sel):
        d = np.ascontiguousarray(depth, dtype=np.uint16)
        img = _img(rgb)
        h, w, ch = img.shape
        s = None if sem is None else np.ascontiguousarray(sem, dtype=np.float32)
        sc = 0 if s is None else (1 if s.ndim == 2 else s.shape[2])
        xyz = np.zeros((w * h + 1, 3))
        feat = np.zeros((w * h + 1, 3 + sc))
        ib, fb = C.c_int(), C.c_int()
        ci, cs = intr.cstruct(), sel.cstruct()
        L = self.lib
        L.ko_depth_rgb_to_cloud.restype = C.c_long
        n = L.ko_depth_rgb_to_cloud(d.ctypes.data_as(C.c_void_p), img.ctypes.data_as(C.c_void_p), ch,
                                    None if s is None else s.ctypes.data_as(C.c_void_p), sc, w, h, C.byref(ci),
                                    C.byref(cs), _abi.as_ptr(xyz), _abi.as_ptr(feat), C.byref(fb), C.byref(ib))
        return xyz[:n], feat[:n], bool(fb.value)

    def build_pairs(self, X, Z, T, params: KernelParams, cutoff=3.0, c_min=1e-4, dense=False):
        h = P()
        n = C.c_int64()
        t, tp = _d12(T)
        kp = params.cstruct()
        self._err(self.lib.ko_build_pairs(X.view(), Z.view(), tp, kp, cutoff, c_min, int(dense), C.byref(h), C.byref(n)))
        off = np.zeros(Z.size() + 1, dtype=np.int64)
        idx = np.zeros(max(n.value, 1), dtype=np.int32)
        cf = np.zeros(max(n.value, 1))
        self.lib.ko_pairs_export(h, _abi.as_ptr(off, C.c_int64), _abi.as_ptr(idx, C.c_int32), _abi.as_ptr(cf))
        return _OraclePairs(self, h, off, idx[: n.value], cf[: n.value])

    def inner_product(self, pairs, X, Z, T, params):
        t, tp = _d12(T)
        return self.lib.ko_inner_product(pairs.h, X.view(), Z.view(), tp, params.cstruct())

    def objective_and_gradient(self, pairs, X, Z, T, params):
        t, tp = _d12(T)
        out = np.zeros(7)
        self.lib.ko_objective_and_gradient(pairs.h, X.view(), Z.view(), tp, params.cstruct(), _abi.as_ptr(out))
        return out

    def max_point_displacement(self, Z, built, now):
        a, ap = _d12(built)
        b, bp = _d12(now)
        return self.lib.ko_max_point_displacement(Z.view(), ap, bp)

    def directional_terms(self, pairs, X, Z, T, xi, params):
        t, tp = _d12(T)
        x = np.ascontiguousarray(np.asarray(xi, dtype=np.float64).reshape(6))
        out = np.zeros(3)
        self.lib.ko_directional_terms(pairs.h, X.view(), Z.view(), tp, _abi.as_ptr(x), params.cstruct(),
                                      _abi.as_ptr(out))
        return out

    def diameter(self, X):
        return self.lib.ko_diameter(X.view())

    def anneal_step(self, l, history, config: RegistrationConfig):
        h = np.ascontiguousarray(history, dtype=np.float64)
        return self.lib.ko_anneal_step(l, _abi.as_ptr(h), len(h), C.byref(config.cstruct()))

    def exp(self, xi):
        xi = np.ascontiguousarray(xi, dtype=np.float64)
        out = np.zeros(12)
        self._err(self.lib.ko_se3_exp(_abi.as_ptr(xi), _abi.as_ptr(out)))
        return Isometry.from12(out)

    def compose(self, a, b):
        x, xp = _d12(a)
        y, yp = _d12(b)
        out = np.zeros(12)
        self.lib.ko_se3_compose(xp, yp, _abi.as_ptr(out))
        return Isometry.from12(out)

    def register_clouds(self, X, Z, initial, params, config, capacity=None):
        buf = _abi.TraceBuffers(capacity or config.max_iterations)
        t, tp = _d12(initial)
        cfg = config.cstruct()
        self._err(self.lib.ko_register_clouds(X.view(), Z.view(), tp, params.cstruct(), C.byref(cfg), C.byref(buf.struct)))
        return RegistrationResult.from_buffers(buf)


    def register_clouds_logged(self, X, Z, initial, params, config, capacity=None):
        """register_clouds plus the replay log: per iteration the evaluated T,
        the pair list's build transform and the lengthscale."""
        cap = capacity or config.max_iterations
        T = np.zeros((cap, 12))
        Tb = np.zeros((cap, 12))
        ls = np.zeros(cap)
        self.lib.ko_set_iteration_log(T.ctypes.data, Tb.ctypes.data, ls.ctypes.data, cap)
        try:
            res = self.register_clouds(X, Z, initial, params, config, capacity)
        finally:
            self.lib.ko_set_iteration_log(None, None, None, 0)
        n = res.iterations
        return res, T[:n], Tb[:n], ls[:n]


class _OraclePairs:
    def __init__(self, owner, h, off, idx, cf):
        self.owner, self.h, self.offsets, self.x_index, self.coeff = owner, h, off, idx, cf

    def size(self):
        return len(self.x_index)

    def __del__(self):
        try:
            self.owner.lib.ko_pairs_destroy(self.h)
        except Exception:
            pass


def ref_available() -> bool:
    return os.path.exists(REF_SO)


class Reference:
    """The compiled reference (oracle/_ref/libkreg_ref.so) via ref_capi.cpp."""

    def __init__(self):
        if not ref_available():
            raise FileNotFoundError(REF_SO)
        L = self.lib = C.CDLL(REF_SO)
        L.kref_last_error.restype = C.c_char_p
        L.kref_set_threads.argtypes = [C.c_int]
        L.kref_build_pairs.argtypes = [VP, VP, _abi.dptr, KP, D, D, C.c_int, C.POINTER(P), C.POINTER(C.c_int64)]
        L.kref_pairs_destroy.argtypes = [P]
        L.kref_pairs_export.argtypes = [P, _abi.i64ptr, _abi.i32ptr, _abi.dptr]
        L.kref_objective_and_gradient.argtypes = [P, VP, VP, _abi.dptr, KP, C.c_int, _abi.dptr]
        L.kref_inner_product.argtypes = [P, VP, VP, _abi.dptr, KP, _abi.dptr]
        L.kref_dense_inner_product.argtypes = [VP, VP, _abi.dptr, KP, _abi.dptr]
        L.kref_max_point_displacement.argtypes = [VP, _abi.dptr, _abi.dptr, _abi.dptr]
        L.kref_indicator.argtypes = [VP, VP, _abi.dptr, KP, D, D, _abi.dptr]
        L.kref_exact_cosine.argtypes = [VP, VP, _abi.dptr, KP, _abi.dptr]
        L.kref_register_clouds.argtypes = [VP, VP, _abi.dptr, KP, CP, RP]
        L.kref_register_batch.argtypes = [C.c_int, VP, VP, _abi.dptr, KP, CP, RP, _abi.i32ptr, _abi.dptr]
        L.kref_register_sequence.argtypes = [VP, C.c_int, KP, CP, C.POINTER(_abi.kreg_sequence_result)]
        L.kref_anneal_step.argtypes = [D, _abi.dptr, C.c_int, CP, _abi.dptr]
        L.kref_line_search.argtypes = [VP, VP, _abi.dptr, _abi.dptr, KP, P, CP, _abi.dptr]
        L.kref_check_config.argtypes = [CP]
        L.kref_se3_exp.argtypes = [_abi.dptr, _abi.dptr]
        L.kref_se3_compose.argtypes = [_abi.dptr, _abi.dptr, _abi.dptr]
        L.kref_diameter.argtypes = [VP]
        L.kref_diameter.restype = D
        L.kref_make_box_cloud.argtypes = [C.c_uint64, C.c_int, C.c_int, _abi.dptr, _abi.dptr]
        L.kref_make_ring_cloud.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, _abi.dptr, _abi.dptr]
        L.kref_max_threads.restype = C.c_int
        L.kref_write_ply.argtypes = [VP, C.c_char_p, C.c_int]
        L.kref_read_ply.argtypes = [C.c_char_p, C.POINTER(P), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                    C.POINTER(C.c_int), C.c_char_p, C.c_int]
        L.kref_cloud_copy.argtypes = [P, _abi.dptr, _abi.dptr, _abi.i32ptr, _abi.i32ptr]
        L.kref_cloud_destroy.argtypes = [P]

    def _err(self, rc):
        raise_for(rc, self.lib.kref_last_error().decode())

    # cloud file I/O: the reference's write_ply / read_cloud (cloud_io.cpp)
    def write_ply(self, cloud, path, binary=True):
        self._err(self.lib.kref_write_ply(cloud.view(), os.fsencode(path), int(binary)))

    def read_ply(self, path):
        """Returns (PointCloud with FP64 features, warnings list)."""
        from paper_2012_03683_b200.types import Channel, ChannelKind, FeatureSchema
        h, n, dim, nch = P(), C.c_int(), C.c_int(), C.c_int()
        w = C.create_string_buffer(1 << 16)
        self._err(self.lib.kref_read_ply(os.fsencode(path), C.byref(h), C.byref(n), C.byref(dim), C.byref(nch),
                                         w, len(w)))
        xyz = np.zeros((n.value, 3))
        feat = np.zeros((n.value, max(dim.value, 1)))
        dims = np.zeros(8, np.int32)
        kinds = np.zeros(8, np.int32)
        self.lib.kref_cloud_copy(h, _abi.as_ptr(xyz), _abi.as_ptr(feat), _abi.as_ptr(dims, C.c_int32),
                                 _abi.as_ptr(kinds, C.c_int32))
        self.lib.kref_cloud_destroy(h)
        warns = [x for x in w.value.decode().split("\n") if x]
        if nch.value == 0:
            return PointCloud(xyz), warns
        names = {0: "color", 1: "intensity", 2: "semantic", 3: "custom"}
        schema = FeatureSchema([Channel(names[int(kinds[k])], int(dims[k]), ChannelKind(int(kinds[k])))
                                for k in range(nch.value)])
        return PointCloud(xyz, schema, feat[:, :dim.value]), warns

    # frame ingest: the reference's select_points / depth_rgb_to_cloud
    def select_points(self, rgb, valid, sel):
        img = _img(rgb)
        h, w, ch = img.shape
        m = np.ascontiguousarray(valid, dtype=np.uint8)
        px = np.zeros((w * h + 1, 2), dtype=np.int32)
        info = _abi.kreg_selection_info()
        note = C.create_string_buffer(256)
        cs = sel.cstruct()
        self._err(self.lib.kref_select_points(img.ctypes.data_as(C.c_void_p), ch, w, h, m.ctypes.data_as(C.c_void_p),
                                              C.byref(cs), px.ctypes.data_as(C.c_void_p), C.c_int64(w * h + 1),
                                              C.byref(info), note, 256))
        return ([tuple(map(int, p)) for p in px[:info.count]], info.threshold, bool(info.in_band),
                note.value.decode())

    def depth_rgb_to_cloud(self, depth, rgb, sem, intr, sel):
        d = np.ascontiguousarray(depth, dtype=np.uint16)
        img = _img(rgb)
        h, w, ch = img.shape
        s = None if sem is None else np.ascontiguousarray(sem, dtype=np.float32)
        sc = 0 if s is None else (1 if s.ndim == 2 else s.shape[2])
        xyz = np.zeros((w * h + 1, 3))
        feat = np.zeros((w * h + 1, 3 + sc))
        n = C.c_int64()
        note = C.create_string_buffer(256)
        ci, cs = intr.cstruct(), sel.cstruct()
        self._err(self.lib.kref_depth_rgb_to_cloud(
            d.ctypes.data_as(C.c_void_p), img.ctypes.data_as(C.c_void_p), ch,
            None if s is None else s.ctypes.data_as(C.c_void_p), sc, w, h, C.byref(ci), C.byref(cs),
            _abi.as_ptr(xyz), _abi.as_ptr(feat), C.c_int64(w * h + 1), C.byref(n), note, 256))
        return xyz[:n.value], feat[:n.value], note.value.decode()

    def set_threads(self, n):
        self.lib.kref_set_threads(int(n))

    def max_threads(self):
        return self.lib.kref_max_threads()

    def build_pairs(self, X, Z, T, params, cutoff=3.0, c_min=1e-4, dense=False):
        h = P()
        n = C.c_int64()
        t, tp = _d12(T)
        self._err(self.lib.kref_build_pairs(X.view(), Z.view(), tp, params.cstruct(), cutoff, c_min, int(dense), C.byref(h), C.byref(n)))
        off = np.zeros(Z.size() + 1, dtype=np.int64)
        idx = np.zeros(max(n.value, 1), dtype=np.int32)
        cf = np.zeros(max(n.value, 1))
        self.lib.kref_pairs_export(h, _abi.as_ptr(off, C.c_int64), _abi.as_ptr(idx, C.c_int32), _abi.as_ptr(cf))
        return _RefPairs(self, h, off, idx[: n.value], cf[: n.value])

    def objective_and_gradient(self, pairs, X, Z, T, params, serial=False):
        t, tp = _d12(T)
        out = np.zeros(7)
        self._err(self.lib.kref_objective_and_gradient(pairs.h, X.view(), Z.view(), tp, params.cstruct(), int(serial), _abi.as_ptr(out)))
        return out

    def inner_product(self, pairs, X, Z, T, params):
        t, tp = _d12(T)
        out = np.zeros(1)
        self._err(self.lib.kref_inner_product(pairs.h, X.view(), Z.view(), tp, params.cstruct(), _abi.as_ptr(out)))
        return float(out[0])

    def dense_inner_product(self, X, Z, T, params):
        t, tp = _d12(T)
        out = np.zeros(1)
        self._err(self.lib.kref_dense_inner_product(X.view(), Z.view(), tp, params.cstruct(), _abi.as_ptr(out)))
        return float(out[0])

    def max_point_displacement(self, Z, built, now):
        a, ap = _d12(built)
        b, bp = _d12(now)
        out = np.zeros(1)
        self._err(self.lib.kref_max_point_displacement(Z.view(), ap, bp, _abi.as_ptr(out)))
        return float(out[0])

    def indicator(self, X, Z, T, params, cutoff=3.0, c_min=1e-4):
        t, tp = _d12(T)
        out = np.zeros(1)
        self._err(self.lib.kref_indicator(X.view(), Z.view(), tp, params.cstruct(), cutoff, c_min, _abi.as_ptr(out)))
        return float(out[0])

    def exact_cosine(self, X, Z, T, params):
        t, tp = _d12(T)
        out = np.zeros(1)
        self._err(self.lib.kref_exact_cosine(X.view(), Z.view(), tp, params.cstruct(), _abi.as_ptr(out)))
        return float(out[0])

    def register_clouds(self, X, Z, initial, params, config, capacity=None):
        buf = _abi.TraceBuffers(capacity or config.max_iterations)
        t, tp = _d12(initial)
        cfg = config.cstruct()
        self._err(self.lib.kref_register_clouds(X.view(), Z.view(), tp, params.cstruct(), C.byref(cfg), C.byref(buf.struct)))
        return RegistrationResult.from_buffers(buf)

    def register_batch(self, Xs, Zs, initials, params, config, capacity=None):
        """OpenMP over pairs, one thread each (eval.cpp:323). Returns (results, statuses, seconds)."""
        n = len(Xs)
        xv = (_abi.kreg_cloud_view * n)(*[x.view() for x in Xs])
        zv = (_abi.kreg_cloud_view * n)(*[z.view() for z in Zs])
        inits = np.ascontiguousarray(np.stack([T.as12() if isinstance(T, Isometry) else np.asarray(T).reshape(12) for T in initials]))
        bufs = [_abi.TraceBuffers(capacity or config.max_iterations) for _ in range(n)]
        res = (_abi.kreg_registration_result * n)(*[b.struct for b in bufs])
        st = np.zeros(n, dtype=np.int32)
        secs = np.zeros(1)
        cfg = config.cstruct()
        self._err(self.lib.kref_register_batch(n, xv, zv, _abi.as_ptr(inits), params.cstruct(), C.byref(cfg), res,
                                               _abi.as_ptr(st, C.c_int32), _abi.as_ptr(secs)))
        out = []
        for k in range(n):
            bufs[k].struct = res[k]
            out.append(RegistrationResult.from_buffers(bufs[k]) if st[k] == 0 else None)
        return out, st, float(secs[0])

    def register_sequence(self, frames, params, config):
        n = len(frames)
        fv = (_abi.kreg_cloud_view * n)(*[f.view() for f in frames])
        sb = SequenceBuffers(n)
        cfg = config.cstruct()
        self._err(self.lib.kref_register_sequence(fv, n, params.cstruct(), C.byref(cfg), C.byref(sb.struct)))
        return sb.result()

    def anneal_step(self, l, history, config):
        h = np.ascontiguousarray(history, dtype=np.float64)
        out = np.zeros(1)
        self._err(self.lib.kref_anneal_step(l, _abi.as_ptr(h), len(h), C.byref(config.cstruct()), _abi.as_ptr(out)))
        return float(out[0])

    def line_search(self, X, Z, T, g, params, pairs, config):
        t, tp = _d12(T)
        gg = np.ascontiguousarray(g, dtype=np.float64)
        out = np.zeros(1)
        self._err(self.lib.kref_line_search(X.view(), Z.view(), tp, _abi.as_ptr(gg), params.cstruct(), pairs.h,
                                            C.byref(config.cstruct()), _abi.as_ptr(out)))
        return float(out[0])

    def check_config(self, config):
        self._err(self.lib.kref_check_config(C.byref(config.cstruct())))

    def exp(self, xi):
        xi = np.ascontiguousarray(xi, dtype=np.float64)
        out = np.zeros(12)
        self._err(self.lib.kref_se3_exp(_abi.as_ptr(xi), _abi.as_ptr(out)))
        return Isometry.from12(out)

    def compose(self, a, b):
        x, xp = _d12(a)
        y, yp = _d12(b)
        out = np.zeros(12)
        self.lib.kref_se3_compose(xp, yp, _abi.as_ptr(out))
        return Isometry.from12(out)

    def diameter(self, X):
        return self.lib.kref_diameter(X.view())

    def make_box_cloud(self, seed, n, with_color=False):
        from paper_2012_03683_b200.types import Channel, ChannelKind, FeatureSchema
        xyz = np.zeros((n, 3))
        feat = np.zeros((n, 3))
        self._err(self.lib.kref_make_box_cloud(seed, n, int(with_color), _abi.as_ptr(xyz), _abi.as_ptr(feat)))
        if with_color:
            return PointCloud(xyz, FeatureSchema([Channel("color", 3, ChannelKind.color)]), feat)
        return PointCloud(xyz)

    def make_ring_cloud(self, seed, sectors, per_sector, with_color=False):
        from paper_2012_03683_b200.types import Channel, ChannelKind, FeatureSchema
        n = sectors * per_sector
        xyz = np.zeros((n, 3))
        feat = np.zeros((n, 3))
        self._err(self.lib.kref_make_ring_cloud(seed, sectors, per_sector, int(with_color), _abi.as_ptr(xyz), _abi.as_ptr(feat)))
        if with_color:
            return PointCloud(xyz, FeatureSchema([Channel("color", 3, ChannelKind.color)]), feat)
        return PointCloud(xyz)


class _RefPairs:
    def __init__(self, owner, h, off, idx, cf):
        self.owner, self.h, self.offsets, self.x_index, self.coeff = owner, h, off, idx, cf

    def size(self):
        return len(self.x_index)

    def __del__(self):
        try:
            self.owner.lib.kref_pairs_destroy(self.h)
        except Exception:
            pass
