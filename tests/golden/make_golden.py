"""Generates tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref,
built from /root/reference by oracle/ref/Makefile). Run in the build
container (the GPU box has no /root/reference):

    python tests/golden/make_golden.py

Each fixture holds the model arrays, the inputs and the reference outputs, so
tests can pin the oracle restatement and the GPU path without the reference.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import ref  # noqa: E402
from paper_1711_07999_b200 import _lib as W  # noqa: E402
from paper_1711_07999_b200.model import ModelBundle, humanoid_trajectory, make_humanoid  # noqa: E402
from tests import rigs  # noqa: E402

OUT = Path(__file__).resolve().parent
MODEL_KEYS = ["parent", "parent_offset", "joint_kind", "joint_axis", "theta_index", "v0", "phi", "weight_count",
              "weight_link", "weight", "triangles", "vtri_offsets", "vtri_items", "nbr_offsets", "nbr_items"]


def model_arrays(b: ModelBundle) -> dict:
    return {f"model_{k}": getattr(b, k) for k in MODEL_KEYS}


def intr_scaled(w, h):
    f = 365.456 * w / 512.0
    return W.Intrinsics(f, f, w / 2.0, h / 2.0, w, h)


def track_cfg(mode, kin, shape):
    return W.TrackConfigC(mode, 1, W.KinConfig(kin, 1, 1e-2, 1e-4, 1e-9, 0, 0, 0.0),
                          W.ShapeConfig(shape, 0, 0.05, 0.5, 1e-2, 1e-9), W.AssocConfig(5, 0, 0.10), 1, 0)


def biped_fixture() -> None:
    """The reference's own biped rig (make_biped_rig, synth.cpp:496-569): skin,
    association, normal system and two tracked frames at 160x132."""
    rm = ref.RefModel.rig("biped")
    b = rm.to_bundle()
    intr = intr_scaled(160, 132)
    rng = np.random.default_rng(11)
    L = b.link_count
    theta0 = rng.uniform(-0.2, 0.2, L)
    theta0[0] = -0.5  # prismatic root: toward the camera
    theta1 = theta0 + rng.uniform(-0.05, 0.05, L)
    theta2 = theta1 + rng.uniform(-0.05, 0.05, L)
    v, n, valid = rm.skin(theta1)
    depth1, vis1 = rm.render_depth(theta1, intr, frame=1)
    depth2, _ = rm.render_depth(theta2, intr, frame=2)
    pts, pvalid = ref.depth_to_cloud(intr, depth1)
    v0s, n0s, val0 = rm.skin(theta0)
    assoc = ref.associate(intr, v0s, n0s, val0, pts, pvalid, 5, 0.10)
    kin = W.KinConfig(12, 1, 1e-2, 1e-4, 1e-9, 0, 0, 0.0)
    jtj, jtr = rm.normal_system(theta0, kin, assoc["count"], assoc["residual"])
    x, rc = ref.solve_step(jtj, jtr)
    dchain = rm.pose_derivatives(theta0)
    S = rm.influence_counts()
    rt = ref.RefTracker(rm, theta0)
    c = track_cfg(W.MODE_DYNAMIC, 5, 2)
    st1 = rt.track_frame_depth(intr, depth1, c)
    th1, ph1, _ = rt.get_state()
    kin1 = np.array([[s.associated, s.residual_sum, s.step_norm, s.solver_skipped] for s in st1.kin[:st1.n_kin]])
    shp1 = np.array([[s.singular, s.mean_phi, s.max_phi, s.mean_abs_r_before, s.mean_abs_r_after]
                     for s in st1.shape[:st1.n_shape]])
    rt.track_frame_depth(intr, depth2, c)  # reuses the stats buffers
    th2, ph2, _ = rt.get_state()
    np.savez_compressed(OUT / "biped_160x132.npz", **model_arrays(b), intr=np.array([intr.fx, intr.fy, intr.cx, intr.cy,
                        intr.width, intr.height]), theta0=theta0, theta1=theta1, theta2=theta2,
                        skin_v=v, skin_n=n, skin_valid=valid, depth1=depth1, depth2=depth2, vis1=vis1,
                        assoc_winners=assoc["winners"], assoc_p_tilde=assoc["p_tilde"], assoc_count=assoc["count"],
                        assoc_residual=assoc["residual"], jtj=jtj, jtr=jtr, step=x, dchain=dchain, S=S,
                        track_theta1=th1, track_phi1=ph1, track_theta2=th2, track_phi2=ph2, kin1=kin1, shape1=shp1)


def humanoid_fixture() -> None:
    """The benchmark rig at C1 scale (~7k vertices, 320x240): three frames of
    smooth-bind (12 pose iterations) and of dynamic (5 + 2) tracking."""
    b = make_humanoid(7000)
    rm = ref.RefModel.from_bundle(b)
    intr = intr_scaled(320, 240)
    L = b.link_count
    depths = [rm.render_depth(humanoid_trajectory(L, f), intr, frame=f)[0] for f in range(4)]
    out = {}
    for tag, c in (("smooth", track_cfg(W.MODE_SMOOTH_BIND, 12, 0)), ("dynamic", track_cfg(W.MODE_DYNAMIC, 5, 2))):
        rt = ref.RefTracker(rm, humanoid_trajectory(L, 0))
        th, ph = [], []
        for f in range(1, 4):
            rt.track_frame_depth(intr, depths[f], c)
            t_, p_, _ = rt.get_state()
            th.append(t_)
            ph.append(p_.astype(np.float32) if tag == "dynamic" else np.zeros(1))
        out[f"{tag}_theta"] = np.array(th)
        if tag == "dynamic":
            out["dynamic_phi"] = np.array(ph)
    # reconstruction error of the frame-3 dynamic state against frame 3
    pts, val = ref.depth_to_cloud(intr, depths[3])
    out["recon_frame3"] = ref.recon_error(rm, out["dynamic_theta"][2], intr, pts, val,
                                          phi=np.asarray(out["dynamic_phi"][2], np.float64))
    np.savez_compressed(OUT / "humanoid7k_320x240.npz", **model_arrays(b),
                        intr=np.array([intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height]),
                        theta0=humanoid_trajectory(L, 0), depths=np.array(depths), **out)


def association_scenes() -> None:
    """Loose-vertex scenes in the style of test_association.cpp:124-180: random
    vertices with camera-facing normals and one point per pixel."""
    intr = W.Intrinsics(500.0, 500.0, 256.0, 212.0, 512, 424)
    rng = np.random.default_rng(17)
    rec = {}
    for s in range(6):
        nv = int(rng.integers(50, 500))
        verts = np.stack([rng.uniform(-0.35, 0.35, nv), rng.uniform(-0.35, 0.35, nv), rng.uniform(1.2, 2.2, nv)], 1)
        normals = np.tile([0.0, 0.0, -1.0], (nv, 1))
        if s % 2:  # random camera-facing normals exercise the dot products
            g = rng.normal(size=(nv, 3))
            g /= np.linalg.norm(g, axis=1, keepdims=True)
            g[g[:, 2] > 0] *= -1
            normals = g
        valid = np.ones(nv, np.uint8)
        P = intr.width * intr.height
        pts = np.zeros((P, 3))
        pval = np.zeros(P, np.uint8)
        for _ in range(int(rng.integers(200, 2000))):
            if rng.random() < 0.5:
                p = verts[rng.integers(nv)] + rng.uniform(-0.35, 0.35, 3) * 0.02
            else:
                p = np.array([rng.uniform(-0.35, 0.35), rng.uniform(-0.35, 0.35), rng.uniform(1.2, 2.2)])
            pc = ref.project(intr, p)
            if pc is None:
                continue
            i = pc[1] * intr.width + pc[0]
            if pval[i]:
                continue
            pts[i], pval[i] = p, 1
        a = ref.associate(intr, verts, normals, valid, pts, pval, 5, 0.10)
        idx = np.nonzero(pval)[0]
        rec[f"s{s}_verts"], rec[f"s{s}_normals"] = verts, normals
        rec[f"s{s}_pix"], rec[f"s{s}_pts"] = idx.astype(np.int32), pts[idx]
        rec[f"s{s}_winners"] = a["winners"][idx]
        rec[f"s{s}_count"], rec[f"s{s}_p_tilde"], rec[f"s{s}_residual"] = a["count"], a["p_tilde"], a["residual"]
    np.savez_compressed(OUT / "association_scenes.npz", n=6, **rec)


def bundle_arrays(prefix: str, b: ModelBundle) -> dict:
    out = {f"{prefix}_{k}": getattr(b, k) for k in MODEL_KEYS}
    out[f"{prefix}_poly_offsets"] = np.concatenate([[0], np.cumsum([len(p) for p in b.polys])]).astype(np.int32)
    out[f"{prefix}_poly_items"] = np.concatenate([np.asarray(p, np.int32) for p in b.polys]).astype(np.int32)
    return out


def kat_fixture() -> None:
    """The reference's own arm and sphere rigs (synth.cpp:425-494) with the
    frames its closed-loop unit tests render (test_kinopt.cpp:320-446,
    test_shapeopt.cpp:141-288), and the reference's answers on them."""
    intr = rigs.kinect()
    ic = intr.c()
    arm = ref.RefModel.rig("arm")
    sphere = ref.RefModel.rig("sphere")
    ab, sb = arm.to_bundle(), sphere.to_bundle()
    plate = rigs.camera_plate()
    rp = ref.RefModel.from_bundle(plate)
    out = {**bundle_arrays("arm", ab), **bundle_arrays("sphere", sb),
           **bundle_arrays("sphere_sub1", sphere.subdivide(1).to_bundle()),
           **bundle_arrays("arm_rigid", arm.rigidify().to_bundle())}
    truth = np.zeros(3)
    truth[1] = 0.1
    out["arm_hinge_depth"] = arm.render_depth(truth, ic)[0]
    out["plate_depth"] = rp.render_depth(np.zeros(1), ic)[0]
    out["arm_traj_depth"] = np.array([arm.render_depth(rigs.arm_curves(3, f), ic, frame=f)[0] for f in range(10)])
    bump = (sb.v0 - np.array([0.0, 0.0, 1.2]))
    bump = bump / np.linalg.norm(bump, axis=1, keepdims=True) * 0.01
    out["sphere_bump_phi"] = bump
    out["sphere_bump_depth"] = sphere.render_depth(np.zeros(1), ic, phi=bump)[0]
    out["sphere_depth"] = sphere.render_depth(np.zeros(1), ic)[0]
    dent = rigs.dent_phi(sb.v0)
    out["sphere_dent_phi"] = dent
    out["sphere_dent_depth"] = sphere.render_depth(np.zeros(1), ic, phi=dent)[0]
    # reference answers (threads = 1)
    kin = W.KinConfig(12, 1, 1e-2, 1e-4, 1e-9, 0, 0, 0.0)
    ac = W.AssocConfig(5, 0, 0.10)
    pts, val = ref.depth_to_cloud(ic, out["arm_hinge_depth"])
    for refresh in (1, 3):
        kin.assoc_refresh = refresh
        rt = ref.RefTracker(arm, np.zeros(3))
        st = rt.optimize_pose(ic, pts, val, kin, ac)
        out[f"arm_hinge_theta_r{refresh}"] = rt.get_state()[0]
        out[f"arm_hinge_stats_r{refresh}"] = np.array([[s.associated, s.residual_sum, s.step_norm,
                                                         s.solver_skipped] for s in st])
    rt = ref.RefTracker(sphere, np.zeros(1))
    pts, val = ref.depth_to_cloud(ic, out["sphere_dent_depth"])
    sc = W.ShapeConfig(2, 0, 0.05, 0.5, 1e-2, 1e-9)
    for f in range(3):
        rt.optimize_shape(ic, pts, val, sc, ac, stats=False)
    out["sphere_dent_phi3"] = rt.get_state()[1]
    np.savez_compressed(OUT / "kat_rigs.npz", **out)


if __name__ == "__main__":
    kat_fixture()
    biped_fixture()
    humanoid_fixture()
    association_scenes()
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size // 1024, "KiB")
