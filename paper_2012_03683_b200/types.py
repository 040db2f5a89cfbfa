"""Value types mirroring the reference's public C++ types.

Reference: /root/reference/proj/include/kreg/
  point_cloud.hpp:13-76  ChannelKind, Channel, FeatureSchema, PointCloud
  kernels.hpp:14-33      KernelForm, ChannelParams, KernelParams
  registration.hpp:13-100 RegistrationConfig, RegistrationResult, SequenceResult
  se3.hpp:11-34          Twist, Isometry
Validation and messages follow point_cloud.cpp:20-59.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from enum import IntEnum

import numpy as np

from . import _abi


class ChannelKind(IntEnum):
    color = 0
    intensity = 1
    semantic = 2
    custom = 3


class KernelForm(IntEnum):
    squared_exponential = 0
    linear = 1


@dataclasses.dataclass(frozen=True)
class Channel:
    name: str
    dim: int
    kind: ChannelKind = ChannelKind.custom


class FeatureSchema:
    """Ordered feature channels (point_cloud.hpp:27-46)."""

    def __init__(self, channels=()):
        self.channels = [c if isinstance(c, Channel) else Channel(*c) for c in channels]
        names = set()
        self.offsets = []
        total = 0
        for ch in self.channels:
            if ch.dim <= 0:
                raise ValueError(f"FeatureSchema: channel '{ch.name}' has non-positive dim")
            if ch.name in names:
                raise ValueError(f"FeatureSchema: duplicate channel name '{ch.name}'")
            names.add(ch.name)
            self.offsets.append(total)
            total += ch.dim
        self.total_dim = total

    def empty(self) -> bool:
        return not self.channels

    def __eq__(self, other) -> bool:
        return isinstance(other, FeatureSchema) and self.channels == other.channels

    def describe(self) -> str:
        if not self.channels:
            return "<geometric-only>"
        return ",".join(f"{c.name}({c.kind.name}:{c.dim})" for c in self.channels)


class PointCloud:
    """Immutable positions (n,3) FP64 + row-major features (n,D) FP64."""

    def __init__(self, positions, schema: FeatureSchema | None = None, features=None):
        self.positions = np.ascontiguousarray(np.asarray(positions, dtype=np.float64).reshape(-1, 3))
        self.schema = schema or FeatureSchema()
        n = self.positions.shape[0]
        d = self.schema.total_dim
        if features is None:
            features = np.zeros((n, d))
        self.features = np.ascontiguousarray(np.asarray(features, dtype=np.float64).reshape(n, d) if d else np.zeros((n, 0)))
        if self.features.size != n * d:
            raise ValueError(
                f"PointCloud: feature block has {self.features.size} values, schema "
                f"{self.schema.describe()} with {n} points requires {n * d}")
        self.positions.setflags(write=False)
        self.features.setflags(write=False)
        self._view = None

    def size(self) -> int:
        return self.positions.shape[0]

    def __len__(self) -> int:
        return self.size()

    def empty(self) -> bool:
        return self.size() == 0

    def view(self) -> _abi.kreg_cloud_view:
        """C descriptor (kreg_cloud_view); the cloud keeps the buffers alive."""
        if self._view is None:
            chans = (_abi.kreg_channel * max(1, len(self.schema.channels)))()
            self._names = [c.name.encode() for c in self.schema.channels]
            for k, c in enumerate(self.schema.channels):
                chans[k] = _abi.kreg_channel(self._names[k], c.dim, int(c.kind))
            self._chans = chans
            v = _abi.kreg_cloud_view()
            v.xyz = _abi.as_ptr(self.positions)
            v.n = self.size()
            v.features = _abi.as_ptr(self.features) if self.schema.total_dim else None
            v.dim = self.schema.total_dim
            v.channels = chans
            v.n_channels = len(self.schema.channels)
            self._view = v
        return self._view


@dataclasses.dataclass
class ChannelParams:
    sigma: float = 1.0
    lengthscale: float = 1.0
    form: KernelForm = KernelForm.squared_exponential


@dataclasses.dataclass
class KernelParams:
    sigma: float = 1.0
    lengthscale: float = 1.0
    per_channel: list = dataclasses.field(default_factory=list)

    def with_lengthscale(self, l: float) -> "KernelParams":
        return dataclasses.replace(self, lengthscale=l, per_channel=list(self.per_channel))

    def cstruct(self) -> _abi.kreg_kernel_params:
        arr = (_abi.kreg_channel_params * max(1, len(self.per_channel)))()
        for k, cp in enumerate(self.per_channel):
            arr[k] = _abi.kreg_channel_params(cp.sigma, cp.lengthscale, int(cp.form))
        s = _abi.kreg_kernel_params(self.sigma, self.lengthscale, arr, len(self.per_channel))
        s._keep = arr
        return s


@dataclasses.dataclass
class RegistrationConfig:
    """Defaults of registration.hpp:18-39."""
    init_lengthscale: float = 0.95
    subsequent_lengthscale: float = 0.1
    min_lengthscale: float = 0.0475
    decay_factor: float = 0.98
    stabilization_window: int = 5
    stabilization_rel_tol: float = 1e-5
    max_iterations: int = 2000
    step_init: float = 0.1
    step_shrink: float = 0.5
    step_grow: float = 1.2
    max_backtracks: int = 20
    convergence_twist_norm: float = 1e-5
    cutoff_multiplier: float = 3.0
    c_min: float = 1e-4

    def cstruct(self) -> _abi.kreg_registration_config:
        return _abi.kreg_registration_config(**dataclasses.asdict(self))


class Isometry:
    """Rotation (3,3) + translation (3,) (se3.hpp:27-34)."""

    def __init__(self, rotation=None, translation=None):
        self.rotation = np.eye(3) if rotation is None else np.array(rotation, dtype=np.float64).reshape(3, 3)
        self.translation = np.zeros(3) if translation is None else np.array(translation, dtype=np.float64).reshape(3)

    @staticmethod
    def identity() -> "Isometry":
        return Isometry()

    @staticmethod
    def from12(a) -> "Isometry":
        m = np.asarray(a, dtype=np.float64).reshape(3, 4)
        return Isometry(m[:, :3], m[:, 3])

    def as12(self) -> np.ndarray:
        return np.ascontiguousarray(np.hstack([self.rotation, self.translation[:, None]]).reshape(12))

    def matrix(self) -> np.ndarray:
        m = np.eye(4)
        m[:3, :3] = self.rotation
        m[:3, 3] = self.translation
        return m

    def apply(self, p):
        return np.asarray(p) @ self.rotation.T + self.translation

    def __repr__(self):
        return f"Isometry(R={self.rotation.tolist()}, t={self.translation.tolist()})"


def rotation_angle(T: Isometry) -> float:
    """se3.cpp:133-137."""
    c = 0.5 * (np.trace(T.rotation) - 1.0)
    return float(np.arccos(min(1.0, max(-1.0, c))))


def translation_norm(T: Isometry) -> float:
    return float(np.linalg.norm(T.translation))


def inverse(T: Isometry) -> Isometry:
    R = T.rotation.T
    return Isometry(R, -(R @ T.translation))


def compose(a: Isometry, b: Isometry) -> Isometry:
    return Isometry(a.rotation @ b.rotation, a.rotation @ b.translation + a.translation)


@dataclasses.dataclass
class RegistrationResult:
    transform: Isometry
    converged: bool
    iterations: int
    objective_trace: np.ndarray
    indicator_trace: np.ndarray
    lengthscale_trace: np.ndarray
    step_trace: np.ndarray
    twist_norm_trace: np.ndarray
    pair_count_trace: np.ndarray
    rebuild_trace: np.ndarray
    final_indicator: float
    sweeps: int = 0
    rebuilds: int = 0

    @staticmethod
    def from_buffers(buf: _abi.TraceBuffers) -> "RegistrationResult":
        s = buf.struct
        n = min(s.iterations, buf.capacity)
        return RegistrationResult(
            transform=Isometry.from12(list(s.transform)),
            converged=bool(s.converged),
            iterations=int(s.iterations),
            objective_trace=buf.objective[:n].copy(),
            indicator_trace=buf.indicator[:n].copy(),
            lengthscale_trace=buf.lengthscale[:n].copy(),
            step_trace=buf.step[:n].copy(),
            twist_norm_trace=buf.twist_norm[:n].copy(),
            pair_count_trace=buf.pair_count[:n].copy(),
            rebuild_trace=buf.rebuild[:n].copy(),
            final_indicator=float(s.final_indicator),
            sweeps=int(s.sweeps),
            rebuilds=int(s.rebuilds),
        )


@dataclasses.dataclass
class SequenceResult:
    relative: list
    trajectory: list
    fallback: np.ndarray
    converged: np.ndarray
    final_indicator: np.ndarray
    iterations: np.ndarray


class SequenceBuffers:
    def __init__(self, n_frames: int):
        m = max(n_frames - 1, 0)
        self.relative = np.zeros((max(m, 1), 12))
        self.trajectory = np.zeros((n_frames, 12))
        self.fallback = np.zeros(max(m, 1), dtype=np.uint8)
        self.converged = np.zeros(max(m, 1), dtype=np.uint8)
        self.final_indicator = np.zeros(max(m, 1))
        self.iterations = np.zeros(max(m, 1), dtype=np.int32)
        self.m = m
        self.struct = _abi.kreg_sequence_result(
            _abi.as_ptr(self.relative), _abi.as_ptr(self.trajectory),
            _abi.as_ptr(self.fallback, C.c_uint8), _abi.as_ptr(self.converged, C.c_uint8),
            _abi.as_ptr(self.final_indicator), _abi.as_ptr(self.iterations, C.c_int32))

    def result(self) -> SequenceResult:
        m = self.m
        return SequenceResult(
            relative=[Isometry.from12(r) for r in self.relative[:m]],
            trajectory=[Isometry.from12(r) for r in self.trajectory],
            fallback=self.fallback[:m].copy(), converged=self.converged[:m].copy(),
            final_indicator=self.final_indicator[:m].copy(), iterations=self.iterations[:m].copy())


class NoOverlapError(RuntimeError):
    """kreg::NoOverlapError (errors.hpp:25-36)."""

    def __init__(self, message: str, cutoff_radius: float | None = None):
        super().__init__(message)
        if cutoff_radius is None:
            import re
            m = re.search(r"radius ([0-9.eE+-]+)", message)
            cutoff_radius = float(m.group(1)) if m else float("nan")
        self.cutoff_radius = cutoff_radius


class ParseError(RuntimeError):
    """kreg::ParseError (errors.hpp:9-22): "path:line: message"."""

    @property
    def line(self) -> int:
        import re
        m = re.search(r":(\d+): ", str(self))
        return int(m.group(1)) if m else 0


class CudaError(RuntimeError):
    pass


def raise_for(code: int, message: str):
    if code == _abi.KREG_OK:
        return
    if code == _abi.KREG_INVALID_ARGUMENT:
        raise ValueError(message)
    if code == _abi.KREG_NO_OVERLAP:
        raise NoOverlapError(message)
    if code in (_abi.KREG_CUDA_ERROR, _abi.KREG_OUT_OF_MEMORY, _abi.KREG_NO_DEVICE):
        raise CudaError(message)
    if code == _abi.KREG_PARSE_ERROR:
        raise ParseError(message)
    raise RuntimeError(message)


@dataclasses.dataclass
class CameraIntrinsics:
    """kreg::CameraIntrinsics (projection.hpp:12-19)."""
    fx: float = 0.0
    fy: float = 0.0
    cx: float = 0.0
    cy: float = 0.0
    depth_scale: float = 1.0
    max_depth: float = 55.0
    skip_top_rows: int = 100

    def cstruct(self):
        return _abi.kreg_camera_intrinsics(self.fx, self.fy, self.cx, self.cy, self.depth_scale, self.max_depth,
                                           self.skip_top_rows)


@dataclasses.dataclass
class SelectorConfig:
    """kreg::SelectorConfig (selector.hpp:12-18)."""
    target_min: int = 3000
    target_max: int = 15000
    initial_threshold: float = 20.0
    adjust_factor: float = 1.5
    max_adjust_rounds: int = 20

    def cstruct(self):
        return _abi.kreg_selector_config(self.target_min, self.target_max, self.initial_threshold, self.adjust_factor,
                                         self.max_adjust_rounds)


@dataclasses.dataclass
class Selection:
    """kreg::Selection (selector.hpp:22-27): (u, v) pixels in raster order."""
    pixels: list
    threshold: float = 0.0
    in_band: bool = False
    note: str = ""
