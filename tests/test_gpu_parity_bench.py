"""Parity at the configurations bench.py measures, against the unmodified
reference (oracle/_ref) on identical inputs.

  C3  640x480, 102k-vertex 20-link humanoid at 1.6 m (~40k valid pixels),
      dynamic 5 pose + 2 surface iterations + stats pass: 3 tracked frames.
  C4  1920x1080, 409k vertices: 1 tracked frame + the winner map.
  C5  batches of 16 and 64 C3 sequences (the narrow 3x3-core search from 8
      sequences, multi-vertex normals from 16 and skin from 32, the batch pose
      and shape grids): every sequence against the same sequence tracked
      alone, and sequence 0 against the reference.
  noise  sigma 5 mm, 5 % dropout, seed 404 (acceptance.cpp:445-449): the
      rendered frame and tracking on it.

Tolerances (asserted; the achieved maxima are printed, run with -s):
  winner map / per-vertex counts   identical (index work)
  theta per frame                  1e-6 rad / m   (north_star: "stated fp32 tolerance")
  Phi per frame                    1e-6 m
  per-iteration residual_sum       1e-6 relative; associated: identical
  batch vs lone sequence           1e-8 (theta, Phi): a 64-sequence batch regroups the
                                   fp64 row batches of the pose system
  rendered depth (noisy)           >= 99.99 % of pixels bit-identical
"""
import numpy as np
import pytest

from oracle import ref
from paper_1711_07999_b200 import _lib as W
from paper_1711_07999_b200.tracker import BatchTracker, Intrinsics, Tracker

from .helpers import bench_humanoid, cfg, theta_at

pytestmark = [pytest.mark.gpu, pytest.mark.ref]

TH_TOL, PHI_TOL, RES_REL = 1e-6, 1e-6, 1e-6


def report(name, **kv):
    print(f"[parity] {name}: " + ", ".join(f"{k}={v:.3g}" if isinstance(v, float) else f"{k}={v}"
                                          for k, v in kv.items()), flush=True)


def compare_stats(st, rst, tag):
    """GPU FrameStats vs the reference's FrameStatsC: associated identical,
    residual_sum / step_norm relative."""
    assert len(st.kin) == rst.n_kin, tag
    worst_r = worst_s = 0.0
    for k, g in enumerate(st.kin):
        r = rst.kin[k]
        assert g.associated == r.associated, (tag, k, g.associated, r.associated)
        assert g.solver_skipped == bool(r.solver_skipped), (tag, k)
        worst_r = max(worst_r, abs(g.residual_sum - r.residual_sum) / max(abs(r.residual_sum), 1e-300))
        worst_s = max(worst_s, abs(g.step_norm - r.step_norm) / max(abs(r.step_norm), 1e-12))
    assert worst_r <= RES_REL, (tag, worst_r)
    assert len(st.shape) == rst.n_shape, tag
    for k, g in enumerate(st.shape):
        r = rst.shape[k]
        assert g.singular == r.singular, (tag, k)
        assert abs(g.mean_abs_r_before - r.mean_abs_r_before) <= RES_REL * max(r.mean_abs_r_before, 1e-12)
        assert abs(g.mean_abs_r_after - r.mean_abs_r_after) <= RES_REL * max(r.mean_abs_r_after, 1e-12)
        assert abs(g.max_phi - r.max_phi) <= PHI_TOL
    return worst_r, worst_s


def track_against_reference(b, intr, frames, th0, c, tag):
    """Tracks `frames` on the GPU and in the reference from th0; asserts per
    frame and returns the worst theta / Phi deviation."""
    rm = ref.RefModel.from_bundle(b)
    trk = Tracker(b, intr, th0)
    rt = ref.RefTracker(rm, th0)
    worst_th = worst_ph = worst_r = worst_s = 0.0
    try:
        for f, depth in enumerate(frames):
            st = trk.track_frame(c, depth=depth)
            rst = rt.track_frame_depth(intr.c(), depth, c.c())
            th, ph, _ = trk.get_state()
            rth, rph, _ = rt.get_state()
            dth, dph = np.abs(th - rth).max(), np.abs(ph - rph).max()
            wr, ws = compare_stats(st, rst, (tag, f))
            worst_th, worst_ph = max(worst_th, dth), max(worst_ph, dph)
            worst_r, worst_s = max(worst_r, wr), max(worst_s, ws)
            assert dth <= TH_TOL, (tag, f, dth)
            assert dph <= PHI_TOL, (tag, f, dph)
            assert st.kin[0].associated > 1000
    finally:
        trk.close()
    report(tag, frames=len(frames), max_dtheta=worst_th, max_dphi=worst_ph, residual_sum_rel=worst_r,
           step_norm_rel=worst_s, associated="identical")
    return worst_th, worst_ph


def winner_map_against_reference(b, intr, depth, th, tag):
    """The correspondence index map of one association (posed at th, frame
    `depth`), GPU vs reference, pixel for pixel."""
    rm = ref.RefModel.from_bundle(b)
    trk = Tracker(b, intr)
    try:
        trk.load_depth(depth)
        trk.skin(th)
        g = trk.associate(5, 0.10)
    finally:
        trk.close()
    rv, rn, rvalid = rm.skin(th, threads=0)
    pts, pvalid = ref.depth_to_cloud(intr.c(), depth)
    r = ref.associate(intr.c(), rv, rn, rvalid, pts, pvalid, 5, 0.10, threads=0)
    valid_px = pvalid.astype(bool)
    same = float(np.mean(g["winners"][valid_px] == r["winners"][valid_px]))
    both = g["count"] > 0
    report(tag, valid_pixels=int(valid_px.sum()), winners_identical=same,
           associated=int((r["count"] > 0).sum()),
           p_tilde_max=float(np.abs(g["p_tilde"][both] - r["p_tilde"][both]).max()))
    assert np.array_equal(g["winners"][valid_px], r["winners"][valid_px])
    assert np.array_equal(g["count"], r["count"])
    assert np.abs(g["p_tilde"][both] - r["p_tilde"][both]).max() <= 1e-12


# ---- C3 ------------------------------------------------------------------------

@pytest.fixture(scope="module")
def c3():
    b = bench_humanoid(100_000)
    intr = Intrinsics.scaled(640, 480)
    rm = ref.RefModel.from_bundle(b)
    frames = [rm.render_depth(theta_at(b, f), intr.c(), frame=f)[0] for f in range(5)]
    return b, intr, frames


def test_c3_frame_has_survey_pixel_count(c3):
    b, intr, frames = c3
    n = [int((d > 0).sum()) for d in frames[1:]]
    report("c3 frames", vertices=b.vertex_count, valid_pixels=n)
    assert b.vertex_count > 95_000 and min(n) > 35_000


@pytest.mark.parametrize("mode", ["dynamic", "smooth-bind"])
def test_c3_tracking_matches_reference(c3, mode):
    b, intr, frames = c3
    track_against_reference(b, intr, frames[1:4], theta_at(b, 0), cfg(mode), f"c3 {mode} 5+2")


def test_c3_winner_map_bitwise(c3):
    b, intr, frames = c3
    winner_map_against_reference(b, intr, frames[4], theta_at(b, 3), "c3 winner map")


# ---- C4 ------------------------------------------------------------------------

def test_c4_tracking_and_winner_map_match_reference():
    b = bench_humanoid(400_000)
    intr = Intrinsics.scaled(1920, 1080)
    rm = ref.RefModel.from_bundle(b)
    frames = [rm.render_depth(theta_at(b, f), intr.c(), frame=f)[0] for f in range(3)]
    assert (frames[1] > 0).sum() > 300_000
    winner_map_against_reference(b, intr, frames[2], theta_at(b, 1), "c4 winner map")
    track_against_reference(b, intr, frames[1:3], theta_at(b, 0), cfg("dynamic"), "c4 dynamic 5+2")


# ---- C5 batches -------------------------------------------------------------------

@pytest.mark.parametrize("nseq", [16, 64])
def test_c5_batch_matches_lone_sequences_and_reference(c3, nseq):
    """Each sequence s of the batch follows its own trajectory phase (as in
    bench.py's C5): every one against a lone Tracker on the same frames, and
    sequence 0 against the reference."""
    b, intr, _ = c3
    c = cfg("dynamic")
    nframes = 2
    renderer = Tracker(b, intr)
    frames = np.zeros((nframes, nseq, intr.height, intr.width), np.float32)
    for f in range(nframes):
        for s in range(nseq):
            frames[f, s] = renderer.render_depth(theta_at(b, f + 1, 0.7 * s), frame=f + 1)[0]
    renderer.close()
    th0 = np.stack([theta_at(b, 0, 0.7 * s) for s in range(nseq)])
    bt = BatchTracker(b, intr, nseq, init_theta=th0)
    worst_th = worst_ph = 0.0
    per_seq = []
    assoc_same = True
    try:
        bstats = [bt.track_frame(c, depth=frames[f]) for f in range(nframes)]
        for s in range(nseq):
            solo = Tracker(b, intr, th0[s])
            try:
                for f in range(nframes):
                    st = solo.track_frame(c, depth=frames[f, s])
                    assoc_same &= [k.associated for k in st.kin] == [k.associated for k in bstats[f][s].kin]
                th_s, ph_s, _ = solo.get_state()
            finally:
                solo.close()
            th_b, ph_b = bt.get_state(s)
            per_seq.append(float(np.abs(th_b - th_s).max()))
            worst_th = max(worst_th, float(np.abs(th_b - th_s).max()))
            worst_ph = max(worst_ph, float(np.abs(ph_b - ph_s).max()))
        th_b0, ph_b0 = bt.get_state(0)
    finally:
        bt.close()
    report(f"c5 batch of {nseq} vs lone", max_dtheta=worst_th, max_dphi=worst_ph, associated_identical=assoc_same)
    rt = ref.RefTracker(ref.RefModel.from_bundle(b), th0[0])
    for f in range(nframes):
        rt.track_frame_depth(intr.c(), frames[f, 0], c.c())
    rth, rph, _ = rt.get_state()
    report(f"c5 batch of {nseq} seq 0 vs reference", max_dtheta=float(np.abs(th_b0 - rth).max()),
           max_dphi=float(np.abs(ph_b0 - rph).max()))
    if not assoc_same or worst_th > 1e-8:
        report(f"c5 batch of {nseq} per sequence", dtheta=str([f"{x:.2g}" for x in per_seq]))
    assert assoc_same
    assert worst_th <= 1e-8 and worst_ph <= 1e-8
    assert np.abs(th_b0 - rth).max() <= TH_TOL
    assert np.abs(ph_b0 - rph).max() <= PHI_TOL


# ---- noisy frames (acceptance.cpp:445-449) -------------------------------------------

NOISE = dict(sigma=0.005, dropout=0.05, quantization=0.0, seed=404)


def test_noisy_render_matches_reference(c3):
    b, intr, _ = c3
    rm = ref.RefModel.from_bundle(b)
    trk = Tracker(b, intr)
    try:
        worst = 1.0
        for f in (1, 2, 7):
            th = theta_at(b, f)
            d, vis = trk.render_depth(th, frame=f, **NOISE)
            rd, rvis = rm.render_depth(th, intr.c(), noise=W.Noise(**NOISE), frame=f)
            same = float(np.mean(d == rd))
            worst = min(worst, same)
            assert same >= 0.9999, (f, same)
            assert np.array_equal(vis, rvis)
            # dropout and noise really happened
            clean, _ = rm.render_depth(th, intr.c(), frame=f)
            dropped = float(np.mean(rd[clean > 0] == 0))
            assert 0.03 < dropped < 0.07, dropped
            assert np.abs(rd[(rd > 0) & (clean > 0)] - clean[(rd > 0) & (clean > 0)]).std() > 0.003
    finally:
        trk.close()
    report("noisy render", identical_pixels_min=worst)


def test_noisy_tracking_matches_reference(c3):
    b, intr, _ = c3
    rm = ref.RefModel.from_bundle(b)
    frames = [rm.render_depth(theta_at(b, f), intr.c(), noise=W.Noise(**NOISE), frame=f)[0] for f in range(1, 4)]
    track_against_reference(b, intr, frames, theta_at(b, 0), cfg("dynamic"), "c3 noisy dynamic 5+2")
