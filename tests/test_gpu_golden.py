"""GPU path vs the reference's stored answers (tests/golden, generated from
the unmodified reference by make_golden.py) and vs the C oracle -- no
oracle/_ref needed, so these run on any GPU box.

Tolerances:
  posed vertices        bitwise (fp64, no FMA contraction, reference operation order)
  normals               bitwise after rounding to the float32 the device stores
  winners / counts      exact (index work)
  p~                    1e-12 m (2^-44 m fixed-point accumulation)
  residual              1e-8 m (float32 normals: |p~ - v| <= cutoff times 2^-24)
  JtJ / Jtr             1e-8 relative (float32 normals in the row, 2^-40 fixed point)
  theta per frame       1e-6 (rad or m); Phi 1e-6 m
"""
import ctypes as C

import numpy as np
import pytest

from oracle import c_oracle
from paper_1711_07999_b200 import _lib as W
from paper_1711_07999_b200 import api, seqio
from paper_1711_07999_b200.model import rigidify
from paper_1711_07999_b200.tracker import (AssocConfig, Intrinsics, KinSolverConfig, ShapeSolverConfig,
                                           TrackConfig, Tracker, associate_posed)

from .helpers import GOLDEN, load_golden

pytestmark = pytest.mark.gpu

TH_TOL, PHI_TOL = 1e-6, 1e-6


def pyintr(ci: W.Intrinsics) -> Intrinsics:
    return Intrinsics(ci.fx, ci.fy, ci.cx, ci.cy, ci.width, ci.height)


def track_cfg(mode: str, kin: int, shape: int) -> TrackConfig:
    return TrackConfig(mode=mode, kin=KinSolverConfig(iterations=kin), shape=ShapeSolverConfig(iterations=shape),
                       assoc=AssocConfig())


@pytest.fixture(scope="module")
def biped():
    z, b, ci = load_golden("biped_160x132")
    trk = Tracker(b, pyintr(ci))
    yield z, b, pyintr(ci), trk
    trk.close()


def test_skin_bitwise(biped):
    """Skinning and normals run in a unit without FMA contraction: posed
    vertices are bitwise the reference's, normals are the reference's fp64
    normals rounded to the fp32 the device stores."""
    z, b, intr, trk = biped
    v, n, valid = trk.skin(z["theta1"])
    assert np.array_equal(v, z["skin_v"])
    assert np.array_equal(valid, z["skin_valid"])
    ok = valid.astype(bool)
    assert np.array_equal(n[ok].astype(np.float32), z["skin_n"][ok].astype(np.float32))


def test_associate_exact(biped):
    z, b, intr, trk = biped
    trk.load_depth(z["depth1"])
    trk.skin(z["theta0"])
    a = trk.associate(5, 0.10)
    assert np.array_equal(a["winners"], z["assoc_winners"])
    assert np.array_equal(a["count"], z["assoc_count"])
    m = z["assoc_count"] > 0
    assert np.abs(a["p_tilde"][m] - z["assoc_p_tilde"][m]).max() <= 1e-12
    assert np.abs(a["residual"][m] - z["assoc_residual"][m]).max() <= 1e-8


def test_normal_system(biped):
    z, b, intr, trk = biped
    jtj, jtr = trk.normal_system(z["theta0"], KinSolverConfig(), z["assoc_count"], z["assoc_residual"])
    assert np.abs(jtj - z["jtj"]).max() <= 1e-8 * np.abs(z["jtj"]).max()
    assert np.abs(jtr - z["jtr"]).max() <= 1e-8 * np.abs(z["jtr"]).max()


def test_track_two_frames(biped):
    z, b, intr, trk = biped
    trk.set_state(z["theta0"], np.zeros((b.vertex_count, 3)), 0)
    c = track_cfg("dynamic", 5, 2)
    st = trk.track_frame(c, depth=z["depth1"])
    th, ph, fi = trk.get_state()
    assert fi == 1
    assert np.abs(th - z["track_theta1"]).max() <= TH_TOL
    assert np.abs(ph - z["track_phi1"]).max() <= PHI_TOL
    assert [s.associated for s in st.kin] == z["kin1"][:, 0].astype(int).tolist()
    assert [s.singular for s in st.shape] == z["shape1"][:, 0].astype(int).tolist()
    trk.track_frame(c, depth=z["depth2"])
    th, ph, _ = trk.get_state()
    assert np.abs(th - z["track_theta2"]).max() <= TH_TOL
    assert np.abs(ph - z["track_phi2"]).max() <= PHI_TOL


def test_association_scenes_exact():
    z = dict(np.load(GOLDEN / "association_scenes.npz"))
    intr = Intrinsics(500.0, 500.0, 256.0, 212.0, 512, 424)
    P = intr.width * intr.height
    for s in range(int(z["n"])):
        v, n = z[f"s{s}_verts"], z[f"s{s}_normals"]
        pts = np.zeros((P, 3))
        pval = np.zeros(P, np.uint8)
        pts[z[f"s{s}_pix"]] = z[f"s{s}_pts"]
        pval[z[f"s{s}_pix"]] = 1
        a = associate_posed(intr, v, n, np.ones(len(v), np.uint8), pts, pval, 5, 0.10)
        assert np.array_equal(a["winners"][z[f"s{s}_pix"]], z[f"s{s}_winners"])
        assert np.array_equal(a["count"], z[f"s{s}_count"])
        m = z[f"s{s}_count"] > 0
        assert np.abs(a["p_tilde"][m] - z[f"s{s}_p_tilde"][m]).max() <= 1e-12
        assert np.abs(a["residual"][m] - z[f"s{s}_residual"][m]).max() <= 1e-8


@pytest.mark.parametrize("mode,key,kin,shape", [("smooth-bind", "smooth", 12, 0), ("dynamic", "dynamic", 5, 2)])
def test_humanoid_track_sequence(mode, key, kin, shape):
    """The sequence driver (wt_gpu_track_sequence: pinned double-buffered
    uploads overlapping the solves) against the reference's run."""
    z, b, ci = load_golden("humanoid7k_320x240")
    trk = Tracker(b, pyintr(ci), z["theta0"])
    th, joints = trk.track_sequence(z["depths"][1:4], track_cfg(mode, kin, shape))
    assert np.abs(th - z[f"{key}_theta"]).max() <= TH_TOL
    if key == "dynamic":
        assert np.abs(trk.get_state()[1] - z["dynamic_phi"][-1]).max() <= 1e-6
    assert trk.get_state()[2] == 3
    assert np.abs(joints[-1] - trk.joint_positions()).max() == 0.0
    trk.close()


def test_track_sequence_device_frames_and_determinism():
    import torch
    z, b, ci = load_golden("humanoid7k_320x240")
    intr = pyintr(ci)
    c = track_cfg("dynamic", 5, 2)
    a = Tracker(b, intr, z["theta0"])
    tha, ja = a.track_sequence(z["depths"][1:4], c)
    dev = torch.from_numpy(z["depths"][1:4].astype(np.float32)).cuda().contiguous()
    bt = Tracker(b, intr, z["theta0"])
    thb, jb = bt.track_sequence((dev.data_ptr(), 3), c)
    assert np.array_equal(tha, thb) and np.array_equal(ja, jb)
    assert np.array_equal(a.get_state()[1], bt.get_state()[1])  # run-to-run bitwise
    a.close()
    bt.close()


def test_api_track_sequence_file(tmp_path):
    """api.track_sequence on a .wts file, as bindings.cpp:241-303 returns it;
    joints = origins of FK(theta) recomputed by the C oracle."""
    z, b, ci = load_golden("humanoid7k_320x240")
    h = seqio.SequenceHeader(ci.width, ci.height, ci.fx, ci.fy, ci.cx, ci.cy, 3)
    w = seqio.SequenceWriter(tmp_path / "s.wts", h)
    for f in range(1, 4):
        w.write_depth(z["depths"][f])
    w.close()
    out = api.track_sequence(b, tmp_path / "s.wts", init_theta=z["theta0"], mode="dynamic", iterations=5,
                             shape_iterations=2)
    assert set(out) == {"theta", "joints", "final_phi"}
    assert np.abs(out["theta"] - z["dynamic_theta"]).max() <= TH_TOL
    assert np.abs(out["final_phi"] - z["dynamic_phi"][-1]).max() <= 1e-6
    ot = c_oracle.OracleTracker(b, ci)
    fk, _, _ = ot.pose_derivatives(out["theta"][-1])
    # origin of a unit DQ: 2 * dual * conj(real), vector part
    r, d = fk[:, :4], fk[:, 4:]
    w_, x, y, zz = r.T
    dw, dx, dy, dz = d.T
    org = 2 * np.stack([-dw * x + dx * w_ - dy * zz + dz * y,
                        -dw * y + dx * zz + dy * w_ - dz * x,
                        -dw * zz - dx * y + dy * x + dz * w_], 1)
    assert np.abs(out["joints"][-1] - org).max() <= 1e-12


def test_modes_against_oracle():
    """rigid (rigidify, tracker.cpp:24-43), shape-match (shape on frame 0
    only), smooth-bind -- GPU vs the C oracle over two frames."""
    z, b, ci = load_golden("humanoid7k_320x240")
    for mode in ("rigid", "shape-match", "smooth-bind"):
        bb = rigidify(b) if mode == "rigid" else b
        c = track_cfg(mode, 5, 2)
        g = Tracker(bb, pyintr(ci), z["theta0"])
        o = c_oracle.OracleTracker(bb, ci, z["theta0"])
        for f in (1, 2):
            g.track_frame(c, depth=z["depths"][f])
            o.load_depth(z["depths"][f])
            o.track_loaded(c.c())
            gt, gp, gf = g.get_state()
            ot, op, of = o.get_state()
            assert gf == of == f
            assert np.abs(gt - ot).max() <= TH_TOL, (mode, f)
            assert np.abs(gp - op).max() <= PHI_TOL, (mode, f)
        g.close()


def test_empty_frame_only_prior_acts():
    z, b, ci = load_golden("humanoid7k_320x240")
    c = track_cfg("dynamic", 3, 1)
    g = Tracker(b, pyintr(ci), z["theta0"])
    o = c_oracle.OracleTracker(b, ci, z["theta0"])
    empty = np.zeros((ci.height, ci.width), np.float32)
    st = g.track_frame(c, depth=empty)
    o.load_depth(empty)
    o.track_loaded(c.c())
    assert all(s.associated == 0 for s in st.kin)
    assert np.abs(g.get_state()[0] - o.get_state()[0]).max() <= 1e-12
    assert np.abs(g.get_state()[1] - o.get_state()[1]).max() <= 1e-12


def test_errors_surface():
    z, b, ci = load_golden("biped_160x132")
    t = Tracker(b, pyintr(ci))
    with pytest.raises(W.LengthMismatch):
        t.load_depth(np.zeros(10, np.float32))
    with pytest.raises(W.ValidationError):
        t.track_frame(TrackConfig(assoc=AssocConfig(window_radius=-1)), depth=z["depth1"])
    lib = W.lib()
    rc = lib.wt_gpu_track_loaded(t._ctx, None, None)
    assert rc == W.WT_EINVAL
    t.close()


@pytest.mark.parametrize("links", [6, 20, 21, 27, 28, 40, 48])
def test_long_chains_against_oracle(links):
    """Every JtJ accumulation layout (3x3 lane tiles up to 20 links, 4x4 up to
    27, lane-owned entries beyond; 128-thread pose CTAs for the 48-link chain,
    whose row tiles do not fit 8 warps' shared memory) and both solvers (one-warp LDL^T up to 32 links,
    block LDL^T beyond): normal system and two pose iterations on a cloud vs
    the C oracle."""
    from . import rigs
    rng = np.random.default_rng(links)
    b, pose = rigs.random_rig(rng, links, 400)
    intr = Intrinsics(40.0, 40.0, 80.0, 60.0, 160, 120)  # wide view: the rig spans x in [-2, 2]
    g = Tracker(b, intr, pose)
    o = c_oracle.OracleTracker(b, intr.c(), pose)
    V = b.vertex_count
    count = (rng.random(V) < 0.5).astype(np.int32)
    res = rng.uniform(-0.01, 0.01, V) * count
    jtj, jtr = g.normal_system(pose, KinSolverConfig(), count, res)
    ojtj, ojtr = o.normal_system(pose, KinSolverConfig().c(), count, res)
    # rows use the fp32-stored normals: 2^-24 relative per entry
    assert np.abs(jtj - ojtj).max() <= 1e-6 * np.abs(ojtj).max()
    assert np.abs(jtr - ojtr).max() <= 1e-6 * np.abs(ojtr).max()
    # a cloud of the posed vertices nudged along z, one point per pixel
    v, n, valid = g.skin(pose)
    pts, pv = rigs.frame_from_points(intr, v[valid.astype(bool)] + [0.0, 0.0, 0.004])
    g.load_cloud(pts, pv)
    o.load_cloud(pts, pv)
    kin = KinSolverConfig(iterations=2)
    sg = g.optimize_pose(kin)
    so = o.optimize_pose(kin.c(), AssocConfig().c())
    assert [s.associated for s in sg] == [s.associated for s in so]
    assert sg[0].associated > 20
    assert np.abs(g.get_state()[0] - o.get_state()[0]).max() <= 1e-6
    g.close()


def test_reconstruction_error_bitwise():
    """reconstruction_error_frame (metrics.cpp:110-142): same visible set and
    bitwise the same distances as the reference (exact brute-force NN)."""
    z, b, ci = load_golden("humanoid7k_320x240")
    trk = Tracker(b, pyintr(ci))
    trk.set_state(z["dynamic_theta"][2], np.asarray(z["dynamic_phi"][2], np.float64), 3)
    trk.load_depth(z["depths"][3])
    d = trk.reconstruction_error()
    assert d.shape == z["recon_frame3"].shape
    assert np.array_equal(d, z["recon_frame3"])
    per = trk.reconstruction_error(per_vertex=True)
    assert np.isnan(per).sum() == b.vertex_count - d.size
    trk.load_depth(np.zeros((ci.height, ci.width), np.float32))  # no observations: zeros
    assert np.all(trk.reconstruction_error() == 0.0)
    trk.close()


@pytest.mark.ref
def test_reconstruction_error_matches_live_reference():
    from oracle import ref
    from .helpers import humanoid, intr320, theta_at
    b = humanoid(7000)
    intr = intr320()
    rm = ref.RefModel.from_bundle(b)
    depth, _ = rm.render_depth(theta_at(b, 6), intr.c(), frame=6)
    th = theta_at(b, 5)
    trk = Tracker(b, intr, th)
    trk.load_depth(depth)
    pts, val = ref.depth_to_cloud(intr.c(), depth)
    want = ref.recon_error(rm, th, intr.c(), pts, val)
    assert np.array_equal(trk.reconstruction_error(), want)
    trk.close()


def test_set_state_invalidates_cached_fk():
    """The frame graph skips the leading FK while theta is unchanged since the
    last solve; set_state must force it again."""
    z, b, ci = load_golden("humanoid7k_320x240")
    c = track_cfg("dynamic", 5, 2)
    a = Tracker(b, pyintr(ci), z["theta0"])
    a.track_frame(c, depth=z["depths"][2])
    b2 = Tracker(b, pyintr(ci), z["theta0"])
    b2.track_frame(c, depth=z["depths"][1])  # FK now cached for another theta
    b2.set_state(z["theta0"], np.zeros((b.vertex_count, 3)), 0)
    b2.track_frame(c, depth=z["depths"][2])
    ta, pa, _ = a.get_state()
    tb, pb, _ = b2.get_state()
    assert np.array_equal(ta, tb) and np.array_equal(pa, pb)
    a.close()
    b2.close()
