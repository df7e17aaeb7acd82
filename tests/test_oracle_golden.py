"""The C restatement oracle (oracle/wt_oracle.c) against fixtures produced by
the unmodified reference (tests/golden/make_golden.py). CPU only."""
import numpy as np
import pytest

from oracle import c_oracle
from paper_1711_07999_b200 import _lib as W

from .helpers import load_golden, track_cfg_c


@pytest.fixture(scope="module")
def biped():
    return load_golden("biped_160x132")


def test_skin_bitwise(biped):
    z, b, intr = biped
    ot = c_oracle.OracleTracker(b, intr)
    v, n, valid = ot.skin(z["theta1"])
    assert np.array_equal(v, z["skin_v"])
    assert np.array_equal(valid, z["skin_valid"])
    assert np.abs(n - z["skin_n"]).max() <= 1e-15


def test_pose_derivatives(biped):
    z, b, intr = biped
    ot = c_oracle.OracleTracker(b, intr)
    _, _, dch = ot.pose_derivatives(z["theta0"])
    assert np.abs(dch - z["dchain"]).max() <= 1e-15


def test_association_bitwise(biped):
    z, b, intr = biped
    ot = c_oracle.OracleTracker(b, intr)
    v, n, valid = ot.skin(z["theta0"])
    pts, pval = c_oracle.depth_to_cloud(intr, z["depth1"])
    a = c_oracle.associate(intr, v, n, valid, pts, pval, 5, 0.10)
    assert pval.sum() > 2000
    assert np.array_equal(a["winners"], z["assoc_winners"])
    assert np.array_equal(a["count"], z["assoc_count"])
    assert np.array_equal(a["p_tilde"], z["assoc_p_tilde"])
    assert np.array_equal(a["residual"], z["assoc_residual"])


def test_normal_system_and_step(biped):
    z, b, intr = biped
    ot = c_oracle.OracleTracker(b, intr)
    kin = W.KinConfig(12, 1, 1e-2, 1e-4, 1e-9, 0, 0, 0.0)
    jtj, jtr = ot.normal_system(z["theta0"], kin, z["assoc_count"], z["assoc_residual"])
    assert np.abs(jtj - z["jtj"]).max() <= 1e-12 * np.abs(z["jtj"]).max()
    assert np.abs(jtr - z["jtr"]).max() <= 1e-12 * np.abs(z["jtr"]).max()
    x, rc = c_oracle.solve_step(z["jtj"], z["jtr"])
    assert rc == 0 and np.abs(x - z["step"]).max() <= 1e-12 * np.abs(z["step"]).max()


def test_track_frames(biped):
    z, b, intr = biped
    ot = c_oracle.OracleTracker(b, intr, z["theta0"])
    c = track_cfg_c(W.MODE_DYNAMIC, 5, 2)
    ot.load_depth(z["depth1"])
    st = ot.track_loaded(c)
    th, ph, fi = ot.get_state()
    assert fi == 1
    assert np.abs(th - z["track_theta1"]).max() <= 1e-12
    assert np.abs(ph - z["track_phi1"]).max() <= 1e-13
    kin = np.array([[s.associated, s.residual_sum, s.step_norm, s.solver_skipped] for s in st.kin[:st.n_kin]])
    assert np.array_equal(kin[:, 0], z["kin1"][:, 0])
    assert np.allclose(kin[:, 1:], z["kin1"][:, 1:], rtol=1e-10, atol=1e-15)
    shp = np.array([[s.singular, s.mean_phi, s.max_phi, s.mean_abs_r_before, s.mean_abs_r_after]
                    for s in st.shape[:st.n_shape]])
    assert np.allclose(shp, z["shape1"], rtol=1e-10, atol=1e-15)
    ot.load_depth(z["depth2"])
    ot.track_loaded(c)
    th, ph, _ = ot.get_state()
    assert np.abs(th - z["track_theta2"]).max() <= 1e-11
    assert np.abs(ph - z["track_phi2"]).max() <= 1e-12


@pytest.mark.parametrize("mode,key", [(W.MODE_SMOOTH_BIND, "smooth"), (W.MODE_DYNAMIC, "dynamic")])
def test_humanoid_sequence(mode, key):
    z, b, intr = load_golden("humanoid7k_320x240")
    c = track_cfg_c(mode, 12 if key == "smooth" else 5, 0 if key == "smooth" else 2)
    ot = c_oracle.OracleTracker(b, intr, z["theta0"])
    for f in range(1, 4):
        ot.load_depth(z["depths"][f])
        ot.track_loaded(c)
        th, ph, _ = ot.get_state()
        assert np.abs(th - z[f"{key}_theta"][f - 1]).max() <= 1e-10
        if key == "dynamic":
            assert np.abs(ph - z["dynamic_phi"][f - 1]).max() <= 1e-7  # stored as float32


def test_association_scenes():
    z = dict(np.load(__import__("tests.helpers", fromlist=["GOLDEN"]).GOLDEN / "association_scenes.npz"))
    intr = W.Intrinsics(500.0, 500.0, 256.0, 212.0, 512, 424)
    P = intr.width * intr.height
    for s in range(int(z["n"])):
        v, n = z[f"s{s}_verts"], z[f"s{s}_normals"]
        pts = np.zeros((P, 3))
        pval = np.zeros(P, np.uint8)
        pts[z[f"s{s}_pix"]] = z[f"s{s}_pts"]
        pval[z[f"s{s}_pix"]] = 1
        a = c_oracle.associate(intr, v, n, np.ones(len(v), np.uint8), pts, pval, 5, 0.10)
        assert np.array_equal(a["winners"][z[f"s{s}_pix"]], z[f"s{s}_winners"])
        assert np.array_equal(a["count"], z[f"s{s}_count"])
        assert np.abs(a["p_tilde"] - z[f"s{s}_p_tilde"]).max() <= 1e-15
        assert np.abs(a["residual"] - z[f"s{s}_residual"]).max() <= 1e-15
