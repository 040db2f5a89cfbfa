"""Synthetic inputs: the reference's seeded generators and the KITTI/TUM-shaped
scenes the benchmark configurations name.

* SplitMix64 (reference include/kreg/rng.hpp:11-46) — bit-exact.
* random_labeled_cloud / clustered_cloud / random_twist / params_for
  (reference tests/test_helpers.hpp:14-118) and make_box_cloud /
  make_ring_cloud (src/eval.cpp:248-300) — bit-exact replicas, so fixtures can
  be regenerated from seeds on a box without the reference tree.
* kitti_pair / tum_pair — ray-cast street / room scenes (numpy, seeded).
"""
from __future__ import annotations

import math

import numpy as np

from .types import (Channel, ChannelKind, ChannelParams, FeatureSchema, Isometry, KernelForm,
                    KernelParams, PointCloud, RegistrationConfig)

M64 = (1 << 64) - 1


class SplitMix64:
    def __init__(self, seed: int):
        self.state = seed & M64

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & M64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        return z ^ (z >> 31)

    def uniform(self, lo: float = None, hi: float = None) -> float:
        u = float(self.next() >> 11) * (2.0 ** -53)
        if lo is None:
            return u
        return lo + (hi - lo) * u

    def gaussian(self) -> float:
        u1 = self.uniform()
        while u1 <= 0.0:
            u1 = self.uniform()
        u2 = self.uniform()
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(6.283185307179586 * u2)

    @staticmethod
    def derive(seed: int, index: int) -> int:
        s = SplitMix64((seed ^ ((0x9E3779B97F4A7C15 * (index + 1)) & M64)) & M64)
        return s.next()


# ------------------------------------------------------------ SE(3) (numpy)
def skew(w):
    return np.array([[0.0, -w[2], w[1]], [w[2], 0.0, -w[0]], [-w[1], w[0], 0.0]])


def se3_exp(xi) -> Isometry:
    """Same formula as reference se3.cpp:48-76 (input generation only)."""
    xi = np.asarray(xi, dtype=np.float64)
    w, v = xi[:3], xi[3:]
    theta = math.sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2])
    W = skew(w)
    W2 = W @ W
    I = np.eye(3)
    if theta < 1e-8:
        R = I + W + 0.5 * W2
        V = I + 0.5 * W + W2 / 6.0
    else:
        t2 = theta * theta
        s = math.sin(theta)
        hs = math.sin(0.5 * theta)
        omc = 2.0 * hs * hs
        a, b, c = s / theta, omc / t2, (theta - s) / (t2 * theta)
        R = I + a * W + b * W2
        V = I + b * W + c * W2
    return Isometry(R, V @ v)


def _normalized(v):
    n = math.sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2])
    return np.array(v) / n if n > 0 else np.array(v, dtype=float)


def _vec3(draw):
    """Eigen::Vector3d(f(), f(), f()) as GCC evaluates it: arguments right to left."""
    c = draw()
    b = draw()
    a = draw()
    return [a, b, c]


def random_twist(rng: SplitMix64, max_angle: float, max_translation: float) -> np.ndarray:
    """test_helpers.hpp:14-22 (GCC right-to-left argument evaluation included)."""
    axis = _vec3(rng.gaussian)
    while math.sqrt(sum(a * a for a in axis)) < 1e-9:
        e2 = rng.gaussian()
        e1 = rng.gaussian()
        axis = [e1, e2, 1.0]
    omega = rng.uniform(0.0, max_angle) * _normalized(axis)
    u = rng.uniform(0.0, max_translation)  # operator*(vec, u): right operand first
    v = _normalized(_vec3(rng.gaussian)) * u
    return np.concatenate([omega, v])


def random_isometry(rng: SplitMix64, max_angle: float, max_translation: float) -> Isometry:
    return se3_exp(random_twist(rng, max_angle, max_translation))


def random_labeled_cloud(seed: int, n: int, scale: float, with_color: bool,
                         semantic_classes: int = 0) -> PointCloud:
    """test_helpers.hpp:30-59."""
    rng = SplitMix64(seed)
    pos = np.zeros((n, 3))
    for i in range(n):
        pos[i] = [scale * c for c in _vec3(rng.uniform)]
    chans = []
    if with_color:
        chans.append(Channel("color", 3, ChannelKind.color))
    if semantic_classes > 0:
        chans.append(Channel("semantic", semantic_classes, ChannelKind.semantic))
    if not chans:
        return PointCloud(pos)
    schema = FeatureSchema(chans)
    feat = []
    for i in range(n):
        if with_color:
            feat += [rng.uniform(), rng.uniform(), rng.uniform()]
        if semantic_classes > 0:
            cls = rng.next() % semantic_classes
            feat += [1.0 if c == cls else 0.0 for c in range(semantic_classes)]
    return PointCloud(pos, schema, np.array(feat).reshape(n, -1))


def clustered_cloud(seed: int, clusters: int, per_cluster: int, center_box: float,
                    cluster_radius: float, with_color: bool) -> PointCloud:
    """test_helpers.hpp:64-88."""
    rng = SplitMix64(seed)
    centers = [center_box * np.array(_vec3(rng.uniform)) for _ in range(clusters)]
    pos, cols = [], []
    for c in centers:
        for _ in range(per_cluster):
            g = np.array(_vec3(rng.gaussian))
            pos.append(c + cluster_radius * g)
            if with_color:
                cols += [rng.uniform(), rng.uniform(), rng.uniform()]
    pos = np.array(pos)
    if not with_color:
        return PointCloud(pos)
    return PointCloud(pos, FeatureSchema([Channel("color", 3, ChannelKind.color)]),
                      np.array(cols).reshape(-1, 3))


def params_for(cloud: PointCloud, lengthscale: float, channel_lengthscale: float = 0.3) -> KernelParams:
    """test_helpers.hpp:106-118."""
    p = KernelParams(lengthscale=lengthscale)
    for ch in cloud.schema.channels:
        if ch.kind == ChannelKind.semantic:
            p.per_channel.append(ChannelParams(1.0, 1.0, KernelForm.linear))
        else:
            p.per_channel.append(ChannelParams(1.0, channel_lengthscale, KernelForm.squared_exponential))
    return p


def make_box_cloud(seed: int, n: int, with_color: bool = False) -> PointCloud:
    """eval.cpp:248-266 (vectorised SplitMix64; bit-exact)."""
    u = np.ascontiguousarray(_splitmix_uniform_stream(seed, 3 * n).reshape(n, 3)[:, ::-1])  # GCC arg order
    if not with_color:
        return PointCloud(u)
    return PointCloud(u, FeatureSchema([Channel("color", 3, ChannelKind.color)]), u.copy())


def make_ring_cloud(seed: int, sectors: int, per_sector: int, with_color: bool) -> PointCloud:
    """eval.cpp:268-300."""
    rng = SplitMix64(seed)
    sector_angle = 2.0 * math.pi / sectors
    pattern = []
    for _ in range(per_sector):
        a = rng.uniform(0.0, sector_angle)
        r = rng.uniform(0.85, 1.15)
        z = rng.uniform(-0.15, 0.15)
        pattern.append((a, r, z))
    pos, feat = [], []
    for s in range(sectors):
        for (a, r, z) in pattern:
            phi = s * sector_angle + a
            pos.append([r * math.cos(phi), r * math.sin(phi), z])
            if with_color:
                feat += [0.5 + 0.5 * math.cos(phi), 0.5 + 0.5 * math.cos(phi - 2.0 * math.pi / 3.0),
                         0.5 + 0.5 * math.cos(phi + 2.0 * math.pi / 3.0)]
    pos = np.array(pos)
    if not with_color:
        return PointCloud(pos)
    return PointCloud(pos, FeatureSchema([Channel("color", 3, ChannelKind.color)]), np.array(feat).reshape(-1, 3))


def _splitmix_stream(seed: int, count: int) -> np.ndarray:
    """The first `count` outputs of SplitMix64(seed), vectorised (uint64 wraps)."""
    k = np.arange(1, count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & M64) + k * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def _splitmix_uniform_stream(seed: int, count: int) -> np.ndarray:
    return (_splitmix_stream(seed, count) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


# ---------------------------------------------------------------- scenes
# KITTI-shaped street: camera frame x right, y down, z fwd.
KITTI_INTRINSICS = dict(fx=718.856, fy=718.856, cx=607.1928, cy=185.2157, width=1241, height=376,
                        skip_top=100, min_depth=2.0, max_depth=55.0)
TUM_INTRINSICS = dict(fx=517.3, fy=516.5, cx=318.6, cy=255.3, width=640, height=480, skip_top=0,
                      min_depth=0.3, max_depth=5.0)

# 19 Cityscapes-style classes used by KITTI semantic CVO
CLS_ROAD, CLS_SIDEWALK, CLS_BUILDING, CLS_POLE, CLS_CAR, CLS_VEGETATION = 0, 1, 2, 5, 13, 8


class _Scene:
    """Axis-aligned boxes + infinite planes with per-primitive colour/class."""

    def __init__(self):
        self.boxes = []  # (lo[3], hi[3], base_rgb[3], cls, texture_freq)

    def add_box(self, lo, hi, rgb, cls, freq=1.0):
        self.boxes.append((np.asarray(lo, float), np.asarray(hi, float), np.asarray(rgb, float), cls, freq))

    def raycast(self, origin, dirs, forward=None, depth_range=(0.0, np.inf)):
        """Nearest hit along each ray (world frame). Returns t, primitive id.
        Boxes entirely outside depth_range along `forward` are culled."""
        n = dirs.shape[0]
        best_t = np.full(n, np.inf)
        best_id = np.full(n, -1, dtype=np.int64)
        inv = 1.0 / np.where(np.abs(dirs) < 1e-12, 1e-12, dirs)
        ix, iy, iz = (np.ascontiguousarray(inv[:, k]) for k in range(3))
        for b, (lo, hi, _, _, _) in enumerate(self.boxes):
            if forward is not None:
                corners = np.array([[x, y, z] for x in (lo[0], hi[0]) for y in (lo[1], hi[1]) for z in (lo[2], hi[2])])
                depth = (corners - origin) @ forward
                if depth.max() < depth_range[0] or depth.min() > depth_range[1]:
                    continue
            # slab test per axis on contiguous columns (same arithmetic as before)
            ax = (lo[0] - origin[0]) * ix, (hi[0] - origin[0]) * ix
            ay = (lo[1] - origin[1]) * iy, (hi[1] - origin[1]) * iy
            az = (lo[2] - origin[2]) * iz, (hi[2] - origin[2]) * iz
            tmin = np.maximum(np.maximum(np.minimum(*ax), np.minimum(*ay)), np.minimum(*az))
            tmax = np.minimum(np.minimum(np.maximum(*ax), np.maximum(*ay)), np.maximum(*az))
            t = np.where(tmin > 1e-6, tmin, tmax)  # camera inside the box → exit face
            hit = (tmax >= np.maximum(tmin, 1e-6)) & (t > 1e-6) & (t < best_t)
            best_t = np.where(hit, t, best_t)
            best_id = np.where(hit, b, best_id)
        return best_t, best_id

    def shade(self, pts, ids, rng, n_classes=19):
        """Colour (n,3) in [0,1] from a smooth world-space texture; class ids."""
        base = np.stack([self.boxes[i][2] for i in range(len(self.boxes))])[ids]
        freq = np.array([self.boxes[i][4] for i in range(len(self.boxes))])[ids]
        tex = (np.sin(freq * 2.1 * pts[:, 0] + 0.3) * np.sin(freq * 1.7 * pts[:, 1] + 1.1) *
               np.sin(freq * 1.3 * pts[:, 2] + 0.7))
        rgb = np.clip(base + 0.18 * tex[:, None] * np.array([1.0, 0.8, 0.6]), 0.0, 1.0)
        cls = np.array([self.boxes[i][3] for i in range(len(self.boxes))])[ids]
        return rgb, cls


def _street_scene(seed: int, length: float = 200.0) -> _Scene:
    rng = np.random.default_rng(seed)
    s = _Scene()
    # ground (road + sidewalks), y = +1.65 is the road surface (y down)
    s.add_box([-6.0, 1.65, -50.0], [6.0, 3.0, length], [0.35, 0.35, 0.37], CLS_ROAD, 3.0)
    s.add_box([-9.0, 1.50, -50.0], [-6.0, 3.0, length], [0.55, 0.52, 0.50], CLS_SIDEWALK, 4.0)
    s.add_box([6.0, 1.50, -50.0], [11.0, 3.0, length], [0.55, 0.52, 0.50], CLS_SIDEWALK, 4.0)
    # facades x = -9 / +11, broken into buildings of varying colour
    z = -50.0
    while z < length:
        w = rng.uniform(8.0, 20.0)
        h = rng.uniform(8.0, 20.0)
        s.add_box([-14.0, 1.5 - h, z], [-9.0, 1.6, z + w], rng.uniform(0.3, 0.8, 3), CLS_BUILDING, 1.5)
        z += w
    z = -50.0
    while z < length:
        w = rng.uniform(8.0, 20.0)
        h = rng.uniform(8.0, 20.0)
        s.add_box([11.0, 1.5 - h, z], [16.0, 1.6, z + w], rng.uniform(0.3, 0.8, 3), CLS_BUILDING, 1.5)
        z += w
    # parked cars (boxes on the road edges) and poles
    n_cars = int(25 * length / 60.0)
    for _ in range(n_cars):
        side = rng.choice([-1.0, 1.0])
        x0 = (-5.8 if side < 0 else 3.8) + rng.uniform(-0.2, 0.2)
        zc = rng.uniform(0.0, length)
        s.add_box([x0, 0.15, zc], [x0 + 1.8, 1.65, zc + rng.uniform(3.8, 4.8)], rng.uniform(0.05, 0.95, 3), CLS_CAR, 6.0)
    n_poles = int(30 * length / 60.0)
    for _ in range(n_poles):
        side = rng.choice([-1.0, 1.0])
        x0 = -7.5 if side < 0 else 8.5
        zc = rng.uniform(0.0, length)
        s.add_box([x0, -4.0, zc], [x0 + 0.2, 1.5, zc + 0.2], [0.5, 0.5, 0.5], CLS_POLE, 10.0)
    return s


def _room_scene(seed: int) -> _Scene:
    rng = np.random.default_rng(seed)
    s = _Scene()
    # room 5 x 4 x 3 m (x in [-2.5,2.5], y (down) in [-1.5,1.5], z in [-0.5,3.5])
    s.add_box([-2.6, 1.5, -0.6], [2.6, 1.7, 3.6], [0.6, 0.5, 0.4], 0, 4.0)    # floor
    s.add_box([-2.6, -1.7, -0.6], [2.6, -1.5, 3.6], [0.9, 0.9, 0.85], 0, 2.0)  # ceiling
    s.add_box([-2.7, -1.7, -0.6], [-2.5, 1.7, 3.6], [0.7, 0.6, 0.5], 0, 3.0)   # walls
    s.add_box([2.5, -1.7, -0.6], [2.7, 1.7, 3.6], [0.5, 0.6, 0.7], 0, 3.0)
    s.add_box([-2.6, -1.7, 3.5], [2.6, 1.7, 3.7], [0.6, 0.7, 0.5], 0, 3.0)
    for _ in range(6):
        c = np.array([rng.uniform(-2.0, 2.0), rng.uniform(0.5, 1.3), rng.uniform(0.8, 3.2)])
        e = rng.uniform(0.15, 0.45, 3)
        lo, hi = c - e, c + e
        hi[1] = 1.5
        s.add_box(lo, hi, rng.uniform(0.05, 0.95, 3), 0, 8.0)
    return s


def _render(scene: _Scene, pose: Isometry, intr: dict, n_points: int, depth_noise: float, rng):
    """Pixel-uniform ray-cast from a camera at `pose` (camera→world)."""
    fx, fy, cx, cy = intr["fx"], intr["fy"], intr["cx"], intr["cy"]
    pts_c, ids_all = [], []
    need = n_points
    while need > 0:
        m = int(need * 1.6) + 1024
        u = rng.uniform(0, intr["width"], m)
        v = rng.uniform(intr["skip_top"], intr["height"], m)
        d_cam = np.stack([(u - cx) / fx, (v - cy) / fy, np.ones(m)], axis=1)
        d_w = d_cam @ pose.rotation.T
        t, ids = scene.raycast(pose.translation, d_w, pose.rotation[:, 2], (0.0, intr["max_depth"]))
        z = t  # depth along the optical axis (d_cam.z = 1)
        ok = np.isfinite(t) & (z >= intr["min_depth"]) & (z <= intr["max_depth"])
        z = z[ok]
        z_noisy = z + depth_noise * z * z * rng.standard_normal(z.shape[0])
        p = d_cam[ok] * z_noisy[:, None]
        pts_c.append(p)
        ids_all.append(ids[ok])
        need -= p.shape[0]
    P = np.concatenate(pts_c)[:n_points]
    I = np.concatenate(ids_all)[:n_points]
    return P, I


def _semantic(cls: np.ndarray, rng, n_classes: int = 19) -> np.ndarray:
    logits = rng.standard_normal((cls.shape[0], n_classes))
    logits[np.arange(cls.shape[0]), cls] = 3.0 + 0.5 * rng.standard_normal(cls.shape[0])
    e = np.exp(logits - logits.max(axis=1, keepdims=True))
    return e / e.sum(axis=1, keepdims=True)


KITTI_SCHEMA = FeatureSchema([Channel("color", 3, ChannelKind.color), Channel("semantic", 19, ChannelKind.semantic)])


def kitti_params() -> KernelParams:
    """proj/profiles/kitti-stereo.json:2-7 via config_io.cpp:176-190."""
    return KernelParams(1.0, 0.1, [ChannelParams(1.0, 0.15, KernelForm.squared_exponential),
                                   ChannelParams(1.0, 0.6, KernelForm.linear)])


def kitti_subsequent_config() -> RegistrationConfig:
    """kitti-stereo.json:8-17 for a subsequent frame pair as register_sequence
    runs it (registration.cpp:200-203): init = subsequent = 0.1,
    min = 0.05 * 0.95 (config_io.cpp:126)."""
    return RegistrationConfig(init_lengthscale=0.1, subsequent_lengthscale=0.1, min_lengthscale=0.05 * 0.95,
                              decay_factor=0.98, stabilization_window=5, stabilization_rel_tol=1e-5,
                              max_iterations=2000, cutoff_multiplier=3.0, c_min=1e-4)


def kitti_first_config() -> RegistrationConfig:
    c = kitti_subsequent_config()
    c.init_lengthscale = 0.95
    return c


def _frame_cloud(scene, pose, intr, n_points, depth_noise, rng, schema_kind):
    P, ids = _render(scene, pose, intr, n_points, depth_noise, rng)
    world = pose.apply(P)
    rgb, cls = scene.shade(world, ids, rng)
    if schema_kind == "kitti":
        feat = np.concatenate([rgb, _semantic(cls, rng)], axis=1)
        return PointCloud(P, KITTI_SCHEMA, feat)
    # TUM: 5-dim colour channel (r, g, b, intensity, texture)
    inten = rgb.mean(axis=1, keepdims=True)
    tex = 0.5 + 0.5 * np.sin(3.0 * world[:, :1] + 2.0 * world[:, 1:2]) * np.cos(2.5 * world[:, 2:3])
    feat = np.concatenate([rgb, inten, tex], axis=1)
    return PointCloud(P, FeatureSchema([Channel("color", 5, ChannelKind.color)]), feat)


def camera_pose(z_forward: float, yaw_rad: float, x: float = 0.0) -> Isometry:
    c, s = math.cos(yaw_rad), math.sin(yaw_rad)
    R = np.array([[c, 0.0, s], [0.0, 1.0, 0.0], [-s, 0.0, c]])  # yaw about camera y (down)
    return Isometry(R, [x, 0.0, z_forward])


def kitti_pair(seed: int, n_points: int = 40000, forward: float = 1.0, yaw_deg: float = 0.5,
               start: float = 0.0):
    """Frame pair (X = frame k-1 = target, Z = frame k = source) with truth
    T* (maps Z onto X). Returns (X, Z, T_star)."""
    rng = np.random.default_rng(seed)
    scene = _street_scene(int(rng.integers(1 << 31)))
    p0 = camera_pose(start, 0.0)
    p1 = camera_pose(start + forward, math.radians(yaw_deg))
    X = _frame_cloud(scene, p0, KITTI_INTRINSICS, n_points, 2e-3, rng, "kitti")
    Z = _frame_cloud(scene, p1, KITTI_INTRINSICS, n_points, 2e-3, rng, "kitti")
    from .types import compose, inverse
    T_star = compose(inverse(p0), p1)
    return X, Z, T_star


def kitti_sequence(seed: int, n_frames: int, n_points: int = 40000, step: float = 1.0):
    """Frames along a smooth trajectory through one long street."""
    rng = np.random.default_rng(seed)
    length = n_frames * step + 120.0
    scene = _street_scene(int(rng.integers(1 << 31)), length=length)
    frames, poses = [], []
    for k in range(n_frames):
        yaw = math.radians(2.0) * math.sin(0.05 * k)
        x = 1.0 * math.sin(0.03 * k)
        pose = camera_pose(k * step, yaw, x)
        poses.append(pose)
        frames.append(_frame_cloud(scene, pose, KITTI_INTRINSICS, n_points, 2e-3, rng, "kitti"))
    return frames, poses


def tum_pair(seed: int, n_points: int = 20000, shift: float = 0.02, yaw_deg: float = 1.0):
    rng = np.random.default_rng(seed)
    scene = _room_scene(int(rng.integers(1 << 31)))
    p0 = camera_pose(-0.4, 0.0)
    p1 = camera_pose(-0.4 + shift, math.radians(yaw_deg))
    X = _frame_cloud(scene, p0, TUM_INTRINSICS, n_points, 1.5e-3, rng, "tum")
    Z = _frame_cloud(scene, p1, TUM_INTRINSICS, n_points, 1.5e-3, rng, "tum")
    from .types import compose, inverse
    return X, Z, compose(inverse(p0), p1)


def tum_params() -> KernelParams:
    """proj/profiles/tum-rgbd.json:2-6."""
    return KernelParams(1.0, 0.05, [ChannelParams(1.0, 0.15, KernelForm.squared_exponential)])


def tum_subsequent_config() -> RegistrationConfig:
    return RegistrationConfig(init_lengthscale=0.05, subsequent_lengthscale=0.05, min_lengthscale=0.025,
                              decay_factor=0.98, stabilization_window=5, stabilization_rel_tol=1e-5,
                              max_iterations=2000, cutoff_multiplier=3.0, c_min=1e-4)


def perturbed(T: Isometry, seed: int, angle: float = math.radians(0.5), trans: float = 0.05) -> Isometry:
    """Constant-velocity initial guess: truth composed with a small error."""
    rng = SplitMix64(seed)
    from .types import compose
    return compose(random_isometry(rng, angle, trans), T)


def kitti_frame(seed: int, width: int = 1241, height: int = 376, classes: int = 19, block: int = 4):
    """Synthetic KITTI-sized stereo frame for the ingest path (SURVEY §8f rank
    3): blocky random texture (FAST corners at block corners), a depth image in
    KITTI's 1/256 m units with holes and far pixels, and per-pixel class
    probabilities (normalised). Returns (depth u16 h x w, rgb u8 h x w x 3,
    semantics f32 h x w x classes, intrinsics)."""
    from .types import CameraIntrinsics
    rng = np.random.default_rng(seed)
    bh, bw = (height + block - 1) // block, (width + block - 1) // block
    tex = rng.integers(0, 256, size=(bh, bw, 3), dtype=np.uint8)
    rgb = np.repeat(np.repeat(tex, block, axis=0), block, axis=1)[:height, :width].copy()
    v = np.arange(height)[:, None].astype(np.float64)
    z = 4.0 + 60.0 * np.clip((height - v) / height, 0.02, 1.0) ** 2 + rng.normal(0.0, 0.05, size=(height, width))
    depth = np.clip(z * 256.0, 0, 65535).astype(np.uint16)
    depth[rng.random((height, width)) < 0.1] = 0  # holes
    sem = rng.random((height, width, classes)).astype(np.float32)
    sem /= sem.sum(axis=2, keepdims=True)
    intr = CameraIntrinsics(fx=718.856, fy=718.856, cx=607.1928, cy=185.2157, depth_scale=1.0 / 256.0,
                            max_depth=55.0, skip_top_rows=100)
    return depth, rgb, sem, intr
