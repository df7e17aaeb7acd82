"""Model preprocessing on the GPU (wt_gpu_mesh_subdivide / wt_gpu_build_neighbors,
csrc/wt_model.cu) against the reference:

  subdivide          skinmesh.cpp:249-511 (Catmull-Clark of positions, phi
                     and skin weights, truncate_weights)
  finalize           skinmesh.cpp:13-58   (shorter-diagonal split, CSR)
  build_neighbors    skinmesh.cpp:145-247 (exact k-NN, (d^2, index) order)

Every output is compared BITWISE: with the live reference (oracle/_ref) on its
own rigs, with the committed reference fixtures (tests/golden) and with the
host restatement (model.py, itself pinned to the reference) on the
400k-vertex C4 humanoid.
"""
import numpy as np
import pytest

from paper_1711_07999_b200 import _lib as W
from paper_1711_07999_b200.model import (_humanoid_at, build_neighbors, build_neighbors_on_device, subdivide,
                                         subdivide_on_device)

from .test_kats import kat_bundle

pytestmark = pytest.mark.gpu

MESH = ["v0", "phi", "weight_count", "weight_link", "weight", "triangles", "vtri_offsets", "vtri_items",
        "nbr_offsets", "nbr_items"]


def assert_same_mesh(got, want, tag):
    assert got.vertex_count == want.vertex_count, tag
    for k in MESH:
        a, b = getattr(got, k), getattr(want, k)
        assert a.shape == b.shape, (tag, k, a.shape, b.shape)
        assert np.array_equal(a, b), (tag, k)
    assert got.polys == [list(p) for p in want.polys], tag


def test_subdivide_sphere_matches_reference_fixture():
    base, want = kat_bundle("sphere"), kat_bundle("sphere_sub1")
    assert_same_mesh(subdivide_on_device(base, 1), want, "sphere sub1")


def test_finalize_and_neighbors_only_match_fixture():
    for rig in ("arm", "sphere", "sphere_sub1"):
        b = kat_bundle(rig)
        got = subdivide_on_device(b, 0, 4)
        for k in ("triangles", "vtri_offsets", "vtri_items", "nbr_offsets", "nbr_items"):
            assert np.array_equal(getattr(got, k), getattr(b, k)), (rig, k)


@pytest.mark.ref
@pytest.mark.parametrize("levels", [1, 2, 3])
def test_subdivide_biped_matches_live_reference(levels):
    """The reference's own biped rig (synth.cpp:496-569) subdivided 1-3 times
    by the reference (subdivide + build_neighbors, bindings.cpp:154-161) and on
    the GPU: identical to the last bit (3 levels: 165,912 vertices)."""
    from oracle import ref
    rm = ref.RefModel.rig("biped")
    base = rm.to_bundle()
    want = rm.subdivide(levels).to_bundle()
    got = subdivide_on_device(base, levels, 4)
    assert_same_mesh(got, want, f"biped sub{levels}")
    print(f"[preprocess] biped sub{levels}: {got.vertex_count} vertices bitwise the reference's")


def test_c4_humanoid_device_equals_host():
    """The 409k-vertex C4 model: three levels on the GPU vs the host
    restatement (model.subdivide, pinned to the reference by the tests above
    and test_model_seqio.py)."""
    import time
    b = _humanoid_at(0.0205, 1.6)  # ~6.2k base vertices: ~400k after three levels
    b.finalize()
    t0 = time.perf_counter()
    host = subdivide(b, 3, 4)
    t1 = time.perf_counter()
    dev = subdivide_on_device(b, 3, 4)
    t2 = time.perf_counter()
    assert dev.vertex_count > 300_000
    assert_same_mesh(dev, host, "humanoid sub3")
    print(f"[preprocess] humanoid sub3 ({dev.vertex_count} vertices): host {t1 - t0:.2f} s, device {t2 - t1:.2f} s")


@pytest.mark.ref
def test_build_neighbors_matches_live_reference():
    from oracle import ref
    rng = np.random.default_rng(7)
    # a noisy cloud with exact ties (duplicated points, a lattice) to exercise the index tie-break
    lattice = np.stack(np.meshgrid(np.arange(12), np.arange(12), np.arange(12)), -1).reshape(-1, 3) * 0.01
    v0 = np.concatenate([rng.normal(size=(20_000, 3)), lattice, lattice[:50]])
    for k in (1, 4, 8):
        items, counts = ref.build_neighbors(v0, k)
        off, got = build_neighbors_on_device(v0, k)
        assert np.array_equal(got.reshape(-1, k), items), k
        host_off, host = build_neighbors(v0, k)
        assert np.array_equal(host, got), k


def test_subdivide_rejects_non_manifold():
    b = kat_bundle("sphere")
    bad = b.copy()
    bad.polys = list(b.polys) + [list(b.polys[0])]  # a face repeated: its edges get a third face
    with pytest.raises(W.ValidationError, match="more than two"):
        subdivide_on_device(bad, 1)
