"""Frame ingest on the B200: kreg_select_points /
kreg_depth_rgb_to_cloud against the compiled reference (selector.cpp:63-125,
projection.cpp:30-75) — identical pixel lists, thresholds, notes, and bitwise
identical positions and features."""
import numpy as np
import pytest

from _checkers import Reference, ref_available
from paper_2012_03683_b200 import api, synth
from paper_2012_03683_b200.types import CameraIntrinsics, Isometry, SelectorConfig

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not ref_available(), reason="compiled reference missing")]


def _cases():
    rng = np.random.default_rng(5)
    img = rng.integers(0, 256, (64, 64, 3), dtype=np.uint8)
    every3 = np.zeros((64, 64), np.uint8)
    every3.flat[::3] = 1
    yield "in_band", img, every3, SelectorConfig(target_min=50, target_max=200)
    yield "out_of_band", img, every3, SelectorConfig(target_min=150, target_max=151, max_adjust_rounds=3)
    yield "fallback", img, every3, SelectorConfig(target_min=5000, target_max=6000)
    yield "uniform", np.full((40, 40, 3), 100, np.uint8), np.ones((40, 40), np.uint8), SelectorConfig(10, 20)
    gray = rng.integers(0, 256, (48, 56), dtype=np.uint8)
    yield "one_channel", gray, np.ones((48, 56), np.uint8), SelectorConfig(target_min=100, target_max=400)
    yield "zero_rounds", img, every3, SelectorConfig(target_min=50, target_max=200, max_adjust_rounds=0)
    big = synth.kitti_frame(9)[1]
    yield "kitti_size", big, (rng.random(big.shape[:2]) < 0.7).astype(np.uint8), SelectorConfig()
    yield "tiny", img[:5, :6], np.ones((5, 6), np.uint8), SelectorConfig(target_min=1, target_max=2)


@pytest.mark.parametrize("name,img,valid,sel", list(_cases()), ids=[c[0] for c in _cases()])
def test_select_points_matches_reference(ctx, name, img, valid, sel):
    s = api.select_points(img, valid, sel)
    px, thr, band, note = Reference().select_points(img, valid, sel)
    assert s.pixels == px and s.threshold == thr and s.in_band == band
    assert s.note == note


@pytest.mark.parametrize("seed,classes", [(1, 19), (2, 0), (3, 5)])
def test_depth_rgb_to_cloud_bitwise_vs_reference(ctx, seed, classes):
    depth, rgb, sem, intr = synth.kitti_frame(seed, classes=max(classes, 1))
    sem = sem if classes else None
    warnings = []
    c = api.depth_rgb_to_cloud(depth, rgb, sem, intr, SelectorConfig(), warnings=warnings)
    xr, fr, note = Reference().depth_rgb_to_cloud(depth, rgb, sem, intr, SelectorConfig())
    assert c.size() == len(xr) > 3000
    assert np.array_equal(c.positions, xr) and np.array_equal(c.features, fr)
    assert (warnings[0] if warnings else "") == note
    assert c.schema.channels[0].name == "color" and (len(c.schema.channels) == 2) == bool(classes)


def test_known_answers_and_errors(ctx):
    intr = CameraIntrinsics(fx=500.0, fy=500.0, cx=4.0, cy=3.0, depth_scale=0.001, max_depth=10.0, skip_top_rows=0)
    depth = np.zeros((8, 10), np.uint16)
    depth[3, 4] = 2500
    rgb = np.full((8, 10, 3), 128, np.uint8)
    w = []
    c = api.depth_rgb_to_cloud(depth, rgb, None, intr, SelectorConfig(), warnings=w)
    assert c.size() == 1 and np.array_equal(c.positions[0], [0.0, 0.0, 2.5]) and w and "fallback" in w[0]
    assert api.depth_rgb_to_cloud(np.zeros((8, 10), np.uint16), rgb, None, intr).size() == 0
    with pytest.raises(ValueError, match="depth and rgb resolutions differ"):
        api.depth_rgb_to_cloud(depth, rgb[:7], None, intr)
    with pytest.raises(ValueError, match="fx and fy must be > 0"):
        api.depth_rgb_to_cloud(depth, rgb, None, CameraIntrinsics())
    with pytest.raises(ValueError, match="need 0 < target_min < target_max"):
        api.select_points(rgb, np.ones((8, 10)), SelectorConfig(target_min=5, target_max=5))
    with pytest.raises(ValueError, match="adjust_factor must be > 1"):
        api.select_points(rgb, np.ones((8, 10)), SelectorConfig(adjust_factor=1.0))


def test_ingested_frames_register(ctx):
    """Two ingested frames of one scene register through the engine (the
    ingest output is a regular cloud for register_clouds)."""
    depth, rgb, sem, intr = synth.kitti_frame(4)
    X = api.depth_rgb_to_cloud(depth, rgb, sem, intr)
    p = synth.kitti_params()
    res = api.register_clouds(X, X, Isometry(), p, synth.kitti_subsequent_config())
    assert res.iterations > 0
    assert np.linalg.norm(res.transform.as12()[[3, 7, 11]]) < 1e-3
