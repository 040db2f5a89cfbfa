"""Frame ingest — CPU: the C oracle (oracle/kreg_oracle.c)
against the compiled reference (selector.cpp / projection.cpp), including the
reference's own known answers (tests/test_ingest.cpp:304-492)."""
import numpy as np
import pytest

from _checkers import Oracle, Reference, ref_available
from paper_2012_03683_b200 import synth
from paper_2012_03683_b200.types import CameraIntrinsics, SelectorConfig

pytestmark = pytest.mark.skipif(not ref_available(), reason="compiled reference missing (make -C oracle ref)")


def _cases():
    rng = np.random.default_rng(5)
    img = rng.integers(0, 256, (64, 64, 3), dtype=np.uint8)
    every3 = np.zeros((64, 64), np.uint8)
    every3.flat[::3] = 1
    yield "in_band", img, every3, SelectorConfig(target_min=50, target_max=200)
    yield "out_of_band", img, every3, SelectorConfig(target_min=150, target_max=151, max_adjust_rounds=3)
    yield "fallback", img, every3, SelectorConfig(target_min=5000, target_max=6000)
    flat = np.full((40, 40, 3), 100, np.uint8)
    yield "uniform", flat, np.ones((40, 40), np.uint8), SelectorConfig(target_min=10, target_max=20)
    gray = rng.integers(0, 256, (48, 56), dtype=np.uint8)
    yield "one_channel", gray, np.ones((48, 56), np.uint8), SelectorConfig(target_min=100, target_max=400)
    yield "zero_rounds", img, every3, SelectorConfig(target_min=50, target_max=200, max_adjust_rounds=0)


@pytest.mark.parametrize("name,img,valid,sel", list(_cases()), ids=[c[0] for c in _cases()])
def test_oracle_selector_matches_reference(name, img, valid, sel):
    px_o, thr_o, band_o, fb_o = Oracle().select_points(img, valid, sel)
    px_r, thr_r, band_r, note_r = Reference().select_points(img, valid, sel)
    assert px_o == px_r and thr_o == thr_r and band_o == band_r
    assert fb_o == ("fallback" in note_r)


def test_oracle_cloud_matches_reference_kitti_frame():
    depth, rgb, sem, intr = synth.kitti_frame(3, 320, 180, classes=5)
    intr.skip_top_rows = 20
    sel = SelectorConfig(target_min=300, target_max=1500)
    xo, fo, fbo = Oracle().depth_rgb_to_cloud(depth, rgb, sem, intr, sel)
    xr, fr, note = Reference().depth_rgb_to_cloud(depth, rgb, sem, intr, sel)
    assert len(xo) == len(xr) > 0
    assert np.array_equal(xo, xr) and np.array_equal(fo, fr)


def test_reference_known_answers_principal_point_and_uniform():
    # test_ingest.cpp "principal point and exclusion rules": one valid pixel at
    # the principal point of a uniform image -> fallback keeps it at (0, 0, z)
    intr = CameraIntrinsics(fx=500.0, fy=500.0, cx=4.0, cy=3.0, depth_scale=0.001, max_depth=10.0, skip_top_rows=0)
    depth = np.zeros((8, 10), np.uint16)
    depth[3, 4] = 2500
    rgb = np.full((8, 10, 3), 128, np.uint8)
    for chk in (Oracle(), Reference()):
        out = chk.depth_rgb_to_cloud(depth, rgb, None, intr, SelectorConfig())
        assert len(out[0]) == 1 and np.array_equal(out[0][0], [0.0, 0.0, 2.5])
