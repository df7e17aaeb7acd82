"""GPU path vs the reference CPU implementation (oracle/_ref) on identical
seeded inputs. Tolerances (fp32 storage / fp64 solves on the device):
  * skinned vertices: |v_gpu - v_ref| <= 1e-5 * max(1, |v_ref|)  (north_star 1e-5 rel)
  * normals: angle <= 1e-3 rad
  * winner (correspondence index) map: >= 99.9% agreement
  * rendered depth: >= 99.99% of pixels bit-identical
  * JtJ / Jtr for a fixed association: 1e-6 relative (Frobenius)
  * theta after N GN iterations: 1e-4 rad / m;  Phi: 2e-5 m
"""
import numpy as np
import pytest

from oracle import ref
from paper_1711_07999_b200 import _lib as W
from paper_1711_07999_b200.tracker import KinSolverConfig, ShapeSolverConfig, Tracker, solve_step, solve_vertices

from .helpers import cfg, humanoid, intr640, theta_at

pytestmark = [pytest.mark.gpu, pytest.mark.ref]


@pytest.fixture(scope="module")
def setup():
    b = humanoid(25000)
    intr = intr640()
    rm = ref.RefModel.from_bundle(b)
    trk = Tracker(b, intr)
    yield b, intr, rm, trk
    trk.close()


def test_skin_matches_reference(setup):
    b, intr, rm, trk = setup
    th = theta_at(b, 7)
    v, n, valid = trk.skin(th)
    rv, rn, rvalid = rm.skin(th)
    err = np.abs(v - rv).max(axis=1) / np.maximum(1.0, np.abs(rv).max(axis=1))
    assert err.max() <= 1e-5
    assert np.array_equal(valid, rvalid)
    cos = np.clip(np.sum(n * rn, axis=1), -1, 1)
    assert np.arccos(cos[valid.astype(bool)]).max() <= 1e-3


def test_render_matches_reference(setup):
    b, intr, rm, trk = setup
    th = theta_at(b, 3)
    d, vis = trk.render_depth(th)
    rd, rvis = rm.render_depth(th, intr.c())
    same = np.mean(d == rd)
    assert same >= 0.9999, f"identical pixels {same}"
    assert np.array_equal(vis, rvis)
    assert (rd > 0).sum() > 5000


def test_associate_matches_reference(setup):
    b, intr, rm, trk = setup
    th_true = theta_at(b, 5)
    depth, _ = rm.render_depth(th_true, intr.c())
    th = theta_at(b, 4)  # one frame behind, as in tracking
    trk.load_depth(depth)
    trk.skin(th)
    g = trk.associate(5, 0.10)
    rv, rn, rvalid = rm.skin(th)
    pts, pvalid = ref.depth_to_cloud(intr.c(), depth)
    r = ref.associate(intr.c(), rv, rn, rvalid, pts, pvalid, 5, 0.10)
    valid_px = pvalid.astype(bool)
    agree = np.mean(g["winners"][valid_px] == r["winners"][valid_px])
    assert agree >= 0.999, f"winner agreement {agree}"
    both = (g["count"] > 0) & (r["count"] > 0) & (g["count"] == r["count"])
    assert both.sum() > 0.99 * (r["count"] > 0).sum()
    assert np.abs(g["p_tilde"][both] - r["p_tilde"][both]).max() <= 1e-9
    assert np.abs(g["residual"][both] - r["residual"][both]).max() <= 2e-6


def test_normal_system_matches_reference(setup):
    b, intr, rm, trk = setup
    th = theta_at(b, 9)
    rng = np.random.default_rng(5)
    count = (rng.random(b.vertex_count) < 0.3).astype(np.int32)
    res = rng.uniform(-0.01, 0.01, b.vertex_count) * count
    kin = KinSolverConfig()
    jtj, jtr = trk.normal_system(th, kin, count, res)
    rjtj, rjtr = rm.normal_system(th, kin.c(), count, res)
    assert np.linalg.norm(jtj - rjtj) <= 1e-6 * np.linalg.norm(rjtj)
    assert np.linalg.norm(jtr - rjtr) <= 1e-6 * np.linalg.norm(rjtr)


def test_solve_step_kat():
    # kinopt test "solve_step basics" (test_kinopt.cpp:237-269)
    kin = KinSolverConfig(lambda_k=0.0, diag_floor=0.0)
    x = solve_step(np.eye(3), np.array([1.0, -2.0, 0.5]), kin)
    assert np.abs(x - [1, -2, 0.5]).max() <= 1e-14
    with pytest.raises(W.NotPositiveDefinite):
        solve_step(-np.eye(2), np.ones(2), kin)


def test_solve_vertex_kat():
    # rank-one system lands on the observed plane (test_shapeopt.cpp:62-78)
    cfg0 = ShapeSolverConfig(lambda_phi=0.0, lambda_nbr=0.0, lambda_w=0.0, diag_floor=1e-12)
    d, s = solve_vertices([[0, 0, -1]], [0.5], [[0, 0, 0]], [[0, 0, 0]], [4], cfg0)
    assert not s[0]
    assert np.allclose(-d[0], [0, 0, 0.5], atol=1e-6)


@pytest.mark.parametrize("mode", ["dynamic", "smooth-bind"])
def test_track_frames_match_reference(setup, mode):
    b, intr, rm, trk = setup
    c = cfg(mode)
    th0 = theta_at(b, 0)
    trk.set_state(theta=th0, phi=np.zeros((b.vertex_count, 3)), frame_index=0)
    rt = ref.RefTracker(rm, th0)
    for f in range(1, 4):
        depth, _ = rm.render_depth(theta_at(b, f), intr.c(), frame=f)
        st = trk.track_frame(c, depth=depth)
        rst = rt.track_frame_depth(intr.c(), depth, c.c())
        th, ph, _ = trk.get_state()
        rth, rph, _ = rt.get_state()
        assert np.abs(th - rth).max() <= 1e-4, (f, np.abs(th - rth).max())
        assert np.abs(ph - rph).max() <= 2e-5, (f, np.abs(ph - rph).max())
        assert st.kin[-1].associated == pytest.approx(rst.kin[rst.n_kin - 1].associated, rel=2e-3)


def test_associate_1080p_matches_reference():
    """The C4 frame size (1920x1080, a 2M-pixel bucket CSR, 32-column
    valid-pixel runs across 60 segments per row): the winner map and the
    per-vertex counts are the reference's, pixel for pixel."""
    from paper_1711_07999_b200.tracker import Intrinsics
    b = humanoid(7000)
    intr = Intrinsics.scaled(1920, 1080)
    rm = ref.RefModel.from_bundle(b)
    trk = Tracker(b, intr)
    try:
        depth, _ = rm.render_depth(theta_at(b, 5), intr.c())
        th = theta_at(b, 4)
        trk.load_depth(depth)
        trk.skin(th)
        g = trk.associate(5, 0.10)
        rv, rn, rvalid = rm.skin(th)
        pts, pvalid = ref.depth_to_cloud(intr.c(), depth)
        r = ref.associate(intr.c(), rv, rn, rvalid, pts, pvalid, 5, 0.10)
        valid_px = pvalid.astype(bool)
        assert valid_px.sum() > 50_000
        assert np.array_equal(g["winners"][valid_px], r["winners"][valid_px])
        assert np.array_equal(g["count"], r["count"])
    finally:
        trk.close()
