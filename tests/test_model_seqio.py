"""Host-side model preprocessing and sequence I/O against the reference
(fixtures from make_golden.py; live reference where built). CPU only.

  finalize / build_neighbors  skinmesh.cpp:13-58, 196-247
  subdivide                   skinmesh.cpp:490-511
  rigidify                    tracker.cpp:24-43
  .wts / depth_to_cloud       seqio.cpp:419-535, test_seqio.cpp:154-200
"""
import numpy as np
import pytest

from oracle import c_oracle
from paper_1711_07999_b200 import _lib as W
from paper_1711_07999_b200 import seqio
from paper_1711_07999_b200.model import build_neighbors, finalize, rigidify, subdivide
from paper_1711_07999_b200.tracker import Intrinsics

from .test_kats import kat_bundle

DERIVED = ["triangles", "vtri_offsets", "vtri_items", "nbr_offsets", "nbr_items"]


@pytest.mark.parametrize("rig", ["arm", "sphere", "sphere_sub1"])
def test_finalize_and_neighbors_match_reference(rig):
    b = kat_bundle(rig)
    tri, off, items = finalize(b.v0, b.polys)
    assert np.array_equal(tri, b.triangles)
    assert np.array_equal(off, b.vtri_offsets)
    assert np.array_equal(items, b.vtri_items)
    noff, nitems = build_neighbors(b.v0, 4)
    assert np.array_equal(noff, b.nbr_offsets)
    assert np.array_equal(nitems, b.nbr_items)


def test_subdivide_matches_reference():
    base, want = kat_bundle("sphere"), kat_bundle("sphere_sub1")
    got = subdivide(base, 1)
    assert got.vertex_count == want.vertex_count > 3 * base.vertex_count
    for k in ["v0", "phi", "weight_count", "weight_link", "weight"] + DERIVED:
        assert np.array_equal(getattr(got, k), getattr(want, k)), k
    assert got.polys == want.polys


def test_rigidify_matches_reference():
    got, want = rigidify(kat_bundle("arm")), kat_bundle("arm_rigid")
    for k in ["weight_count", "weight_link", "weight", "phi"]:
        assert np.array_equal(getattr(got, k), getattr(want, k)), k


def test_depth_to_cloud_principal_ray():
    """test_seqio.cpp:154-170, numpy tooling version and the C oracle."""
    intr = Intrinsics(10, 10, 4, 3, 8, 6)
    depth = np.zeros(48, np.float32)
    depth[3 * 8 + 4] = 2.0
    for pts, valid in (seqio.depth_to_cloud(intr, depth), c_oracle.depth_to_cloud(intr.c(), depth)):
        assert valid.sum() == 1
        assert np.abs(pts[3 * 8 + 4] - [0, 0, 2]).max() <= 1e-12
    assert seqio.depth_to_cloud(intr, np.zeros(48, np.float32))[1].sum() == 0


def test_depth_to_cloud_numpy_equals_oracle():
    z = np.load(__import__("tests.helpers", fromlist=["GOLDEN"]).GOLDEN / "biped_160x132.npz")
    fx, fy, cx, cy, w, h = z["intr"]
    intr = Intrinsics(fx, fy, cx, cy, int(w), int(h))
    d = z["depth1"].copy()
    d[0, :3] = [np.nan, np.inf, -1.0]
    a = seqio.depth_to_cloud(intr, d, 0.001)
    b = c_oracle.depth_to_cloud(intr.c(), d, 0.001)
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[0], b[0])


def test_sequence_round_trip_bitwise(tmp_path):
    """test_seqio.cpp:172-200."""
    rng = np.random.default_rng(3)
    frames = rng.uniform(0, 3, (5, 12, 16)).astype(np.float32)
    frames[frames < 0.5] = 0
    h = seqio.SequenceHeader(16, 12, 10.0, 11.0, 8.0, 6.0, 5, 0.001)
    w = seqio.SequenceWriter(tmp_path / "a.wts", h)
    for f in frames:
        w.write_depth(f)
    w.close()
    r = seqio.SequenceReader(tmp_path / "a.wts")
    assert r.header == h
    assert np.array_equal(r.frames(), frames)
    assert all(np.array_equal(r.read_depth(k), frames[k]) for k in range(5))
    with pytest.raises(W.ValidationError):
        r.read_depth(5)


def test_sequence_errors(tmp_path):
    (tmp_path / "bad.wts").write_bytes(b"NOTMAGIC" + bytes(56))
    with pytest.raises(W.ValidationError):
        seqio.SequenceReader(tmp_path / "bad.wts")
    h = seqio.SequenceHeader(4, 4, 1.0, 1.0, 2.0, 2.0, 2)
    w = seqio.SequenceWriter(tmp_path / "short.wts", h)
    w.write_depth(np.zeros(16, np.float32))
    with pytest.raises(W.ValidationError):
        w.close()
    with pytest.raises(W.ValidationError):
        seqio.SequenceReader(tmp_path / "short.wts")
    with pytest.raises(W.LengthMismatch):
        seqio.SequenceWriter(tmp_path / "x.wts", h).write_depth(np.zeros(15, np.float32))


@pytest.mark.ref
def test_sequence_format_identical_to_reference(tmp_path):
    from oracle import ref
    rng = np.random.default_rng(5)
    frames = rng.uniform(0, 3, (3, 10, 14)).astype(np.float32)
    intr = Intrinsics(9.0, 9.5, 7.0, 5.0, 14, 10)
    ref.write_sequence(tmp_path / "ref.wts", intr.c(), frames, 0.5)
    w = seqio.SequenceWriter(tmp_path / "ours.wts", seqio.SequenceHeader(14, 10, 9.0, 9.5, 7.0, 5.0, 3, 0.5))
    for f in frames:
        w.write_depth(f)
    w.close()
    assert (tmp_path / "ref.wts").read_bytes() == (tmp_path / "ours.wts").read_bytes()
    ri, scale, n, d = ref.read_depth(tmp_path / "ours.wts", 2)
    assert (ri.width, ri.height, scale, n) == (14, 10, 0.5, 3) and np.array_equal(d, frames[2])


def test_ground_truth_csv_round_trip(tmp_path):
    rng = np.random.default_rng(9)
    theta = rng.normal(size=(4, 3))
    joints = rng.normal(size=(4, 3, 3))
    vis = rng.integers(0, 2, (4, 3))
    seqio.save_ground_truth(tmp_path / "gt.csv", ["a", "b", "c"], theta, joints, vis)
    gt = seqio.load_ground_truth(tmp_path / "gt.csv")
    assert gt["joint_names"] == ["a", "b", "c"]
    assert np.array_equal(gt["theta"], theta) and np.array_equal(gt["joints"], joints)
    assert np.array_equal(gt["visible"], vis)
