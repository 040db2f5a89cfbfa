"""PLY ingest: kreg_cloud_read_ply against the
compiled reference read_ply (/root/reference/proj/src/cloud_io.cpp:141-297).

CPU tests pin the checker (reference write/read round trip, error texts);
the GPU tests compare the device reader with it: positions bit-exact,
features equal to the FP32 rounding of the reference's FP64 values, the same
schema, warnings and ParseError messages, and a registration on the device-read
clouds bitwise equal to one on host-uploaded reference clouds."""
import os
import struct

import numpy as np
import pytest

from _checkers import Reference, ref_available
from paper_2012_03683_b200 import synth
from paper_2012_03683_b200.types import ParseError, PointCloud

pytestmark = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")


def _ply(path, header_lines, body: bytes):
    with open(path, "wb") as f:
        f.write(("\n".join(header_lines) + "\n").encode())
        f.write(body)


def _typed_file(path):
    """uchar colour, ushort intensity, a skipped property, two semantic
    classes and a fixed-size element before the vertices (binary)."""
    rng = np.random.default_rng(5)
    n = 300
    xyz = rng.normal(size=(n, 3)) * 4.0
    rgb = rng.integers(0, 256, size=(n, 3))
    inten = rng.integers(0, 65536, size=n)
    sem = rng.random((n, 2)).astype(np.float32)
    hdr = ["ply", "format binary_little_endian 1.0", "comment typed", "element camera 2",
           "property float fx", "property int id", f"element vertex {n}", "property double x",
           "property float confidence", "property double y", "property double z", "property uchar red",
           "property uchar green", "property uchar blue", "property ushort intensity", "property float semantic_1",
           "property float semantic_0", "end_header"]
    body = b"".join(struct.pack("<fi", 1.5 * k, k) for k in range(2))
    for i in range(n):
        body += struct.pack("<dfddBBBHff", xyz[i, 0], 0.5, xyz[i, 1], xyz[i, 2], *rgb[i], inten[i], sem[i, 1], sem[i, 0])
    _ply(path, hdr, body)


BAD = {
    "magic": (["plx", "format ascii 1.0", "element vertex 0", "end_header"], b""),
    "format": (["ply", "format binary_big_endian 1.0", "element vertex 0", "end_header"], b""),
    "type": (["ply", "format ascii 1.0", "element vertex 1", "property float128 x", "end_header"], b""),
    "xyz": (["ply", "format ascii 1.0", "element vertex 1", "property float x", "property float y", "end_header"],
            b"1 2\n"),
    "rgb": (["ply", "format ascii 1.0", "element vertex 1", "property float x", "property float y",
             "property float z", "property uchar red", "end_header"], b"1 2 3 4\n"),
    "semantic": (["ply", "format ascii 1.0", "element vertex 1", "property float x", "property float y",
                  "property float z", "property float semantic_1", "end_header"], b"1 2 3 0.5\n"),
    "truncated": (["ply", "format binary_little_endian 1.0", "element vertex 4", "property double x",
                   "property double y", "property double z", "end_header"], b"\x00" * 40),
    "few_values": (["ply", "format ascii 1.0", "element vertex 2", "property float x", "property float y",
                    "property float z", "end_header"], b"1 2 3\n4 5\n"),
    "trailing": (["ply", "format ascii 1.0", "element vertex 1", "property float x", "property float y",
                  "property float z", "end_header"], b"1 2 3 4\n"),
    "keyword": (["ply", "format ascii 1.0", "element vertex 1", "bogus line", "end_header"], b""),
}


@pytest.fixture(scope="module")
def ref():
    return Reference()


def test_reference_binary_round_trip_is_bit_exact(ref, tmp_path):
    X, _, _ = synth.kitti_pair(11, 2000)
    p = str(tmp_path / "c.ply")
    ref.write_ply(X, p, binary=True)
    back, warns = ref.read_ply(p)
    assert warns == []
    assert np.array_equal(back.positions, X.positions)
    assert np.array_equal(back.features, X.features.astype(np.float32).astype(np.float64))


@pytest.mark.parametrize("case", sorted(BAD))
def test_reference_parse_errors(ref, tmp_path, case):
    p = str(tmp_path / f"{case}.ply")
    _ply(p, *BAD[case])
    with pytest.raises(ParseError):
        ref.read_ply(p)


@pytest.mark.gpu
@pytest.mark.parametrize("binary", [True, False])
def test_device_read_matches_reference(ref, ctx, tmp_path, binary):
    from paper_2012_03683_b200 import api
    X, _, _ = synth.kitti_pair(12, 5000)
    p = str(tmp_path / "k.ply")
    ref.write_ply(X, p, binary=binary)
    rc, rw = ref.read_ply(p)
    w = []
    dc = api.read_ply(p, ctx, warnings=w)
    assert w == rw
    assert dc.size() == rc.size()
    assert [(c.name, c.dim, int(c.kind)) for c in dc.cloud.schema.channels] == \
        [(c.name, c.dim, int(c.kind)) for c in rc.schema.channels]
    assert np.array_equal(dc.cloud.positions, rc.positions)
    assert np.array_equal(dc.cloud.features, rc.features.astype(np.float32).astype(np.float64))


@pytest.mark.gpu
def test_device_read_typed_properties(ref, ctx, tmp_path):
    from paper_2012_03683_b200 import api
    p = str(tmp_path / "typed.ply")
    _typed_file(p)
    rc, rw = ref.read_ply(p)
    w = []
    dc = api.read_ply(p, ctx, warnings=w)
    assert w == rw == ["property 'confidence' skipped"]
    assert np.array_equal(dc.cloud.positions, rc.positions)
    assert np.array_equal(dc.cloud.features, rc.features.astype(np.float32).astype(np.float64))


@pytest.mark.gpu
@pytest.mark.parametrize("case", sorted(BAD))
def test_device_parse_errors_match_reference(ref, ctx, tmp_path, case):
    from paper_2012_03683_b200 import api
    p = str(tmp_path / f"{case}.ply")
    _ply(p, *BAD[case])
    with pytest.raises(ParseError) as r_err:
        ref.read_ply(p)
    with pytest.raises(ParseError) as d_err:
        api.read_ply(p, ctx)
    assert str(d_err.value) == str(r_err.value)


@pytest.mark.gpu
def test_device_read_empty_and_geometric(ref, ctx, tmp_path):
    from paper_2012_03683_b200 import api
    p = str(tmp_path / "geo.ply")
    ref.write_ply(PointCloud(np.random.default_rng(1).normal(size=(1500, 3))), p, binary=True)
    dc = api.read_ply(p, ctx)
    rc, _ = ref.read_ply(p)
    assert dc.cloud.schema.channels == [] and np.array_equal(dc.cloud.positions, rc.positions)
    _ply(str(tmp_path / "empty.ply"), ["ply", "format ascii 1.0", "element vertex 0", "property float x",
                                        "property float y", "property float z", "end_header"], b"")
    assert api.read_ply(str(tmp_path / "empty.ply"), ctx).size() == 0


@pytest.mark.gpu
def test_registration_on_device_read_clouds_is_bitwise_the_host_upload(ref, ctx, tmp_path):
    """A cloud read by the device reader is the cloud kreg_cloud_create makes
    from read_ply's PointCloud: same order, same rows, same results."""
    from paper_2012_03683_b200 import api
    X, Z, T = synth.kitti_pair(13, 8000)
    px, pz = str(tmp_path / "x.ply"), str(tmp_path / "z.ply")
    ref.write_ply(X, px)
    ref.write_ply(Z, pz)
    rx, _ = ref.read_ply(px)
    rz, _ = ref.read_ply(pz)
    cfg = synth.kitti_subsequent_config()
    cfg.max_iterations = 60
    params = synth.kitti_params()
    init = synth.perturbed(T, 13)
    a = api.register_clouds(api.read_ply(px, ctx), api.read_ply(pz, ctx), init, params, cfg, ctx=ctx)
    b = api.register_clouds(rx, rz, init, params, cfg, ctx=ctx)
    assert np.array_equal(a.transform.as12(), b.transform.as12())
    assert np.array_equal(a.objective_trace, b.objective_trace)
