"""Batched sequences (wt_gpu_create_batch / BatchTracker): B independent
sequences tracked in lockstep, the sequence index in blockIdx.y.

Every kernel's result is independent of the grid it runs in (exact search,
integer fixed-point reductions, per-vertex solves), so each sequence of a
batch must be BITWISE the same as the sequence tracked alone -- theta, Phi
and the per-iteration stats -- and sequence 0 also matches the reference's
stored run (1e-6, as in test_gpu_golden).
"""
import numpy as np
import pytest

from paper_1711_07999_b200 import _lib as W
from paper_1711_07999_b200.tracker import (AssocConfig, BatchTracker, Intrinsics, KinSolverConfig,
                                           ShapeSolverConfig, TrackConfig, Tracker)

from .helpers import load_golden

pytestmark = pytest.mark.gpu


def pyintr(ci: W.Intrinsics) -> Intrinsics:
    return Intrinsics(ci.fx, ci.fy, ci.cx, ci.cy, ci.width, ci.height)


def cfg(mode="dynamic", kin=5, shape=2) -> TrackConfig:
    return TrackConfig(mode=mode, kin=KinSolverConfig(iterations=kin), shape=ShapeSolverConfig(iterations=shape),
                       assoc=AssocConfig())


def scenario():
    """Three different sequences over the humanoid fixture's frames."""
    z, b, ci = load_golden("humanoid7k_320x240")
    d = z["depths"][1:4].astype(np.float32)
    frames = np.stack([d, d[::-1].copy(), np.roll(d, 3, axis=2)], axis=1)  # [F, B, H, W]
    rng = np.random.default_rng(5)
    th0 = np.stack([z["theta0"], z["theta0"] + 0.02 * rng.standard_normal(b.link_count),
                    z["theta0"] - 0.01])
    return z, b, pyintr(ci), frames, th0


@pytest.mark.parametrize("mode,kin,shape", [("dynamic", 5, 2), ("shape-match", 4, 3), ("smooth-bind", 6, 0)])
def test_batch_equals_independent_sequences(mode, kin, shape):
    z, b, intr, frames, th0 = scenario()
    B = frames.shape[1]
    c = cfg(mode, kin, shape)
    bt = BatchTracker(b, intr, B, init_theta=th0)
    solo = [Tracker(b, intr, th0[s]) for s in range(B)]
    for f in range(frames.shape[0]):
        bst = bt.track_frame(c, depth=frames[f])
        for s in range(B):
            st = solo[s].track_frame(c, depth=frames[f, s])
            th_b, ph_b = bt.get_state(s)
            th_s, ph_s, fi = solo[s].get_state()
            assert np.array_equal(th_b, th_s), (f, s)
            assert np.array_equal(ph_b, ph_s), (f, s)
            assert bst[s].frame == st.frame == fi - 1
            assert [(k.associated, k.residual_sum, k.step_norm, k.solver_skipped) for k in bst[s].kin] == \
                   [(k.associated, k.residual_sum, k.step_norm, k.solver_skipped) for k in st.kin]
            assert [(k.singular, k.mean_phi, k.max_phi, k.mean_abs_r_after) for k in bst[s].shape] == \
                   [(k.singular, k.mean_phi, k.max_phi, k.mean_abs_r_after) for k in st.shape]
    if mode == "dynamic":
        # sequence 0 is the reference's stored run
        assert np.abs(bt.get_state(0)[0] - z["dynamic_theta"][-1]).max() <= 1e-6
        assert np.abs(bt.get_state(0)[1] - z["dynamic_phi"][-1]).max() <= 1e-6
    bt.close()
    for t in solo:
        t.close()


def test_batch_of_one_and_device_frames():
    import torch
    z, b, intr, frames, th0 = scenario()
    c = cfg()
    one = BatchTracker(b, intr, 1, init_theta=th0[:1])
    solo = Tracker(b, intr, th0[0])
    big = BatchTracker(b, intr, 3, init_theta=th0)
    for f in range(frames.shape[0]):
        one.track_frame(c, depth=frames[f, :1])
        solo.track_frame(c, depth=frames[f, 0])
        dev = torch.from_numpy(frames[f]).cuda().contiguous()
        big.load_depth((dev.data_ptr(),))
        torch.cuda.synchronize()
        big.track_async(c)
        big.sync()
    assert np.array_equal(one.get_state(0)[0], solo.get_state()[0])
    assert np.array_equal(one.get_state(0)[1], solo.get_state()[1])
    assert np.array_equal(big.get_state(0)[0], solo.get_state()[0])
    for t in (one, solo, big):
        t.close()


def test_batch_set_state_per_sequence():
    z, b, intr, frames, th0 = scenario()
    bt = BatchTracker(b, intr, 3)
    assert np.array_equal(bt.thetas(), np.zeros((3, b.link_count)))
    ph = np.full((b.vertex_count, 3), 1e-3)
    bt.set_state(1, theta=th0[1], phi=ph)
    th, p = bt.get_state(1)
    assert np.array_equal(th, th0[1]) and np.array_equal(p, ph)
    assert np.array_equal(bt.get_state(0)[1], np.zeros((b.vertex_count, 3)))
    bt.close()


def test_batch_rejects_per_frame_calls():
    z, b, intr, frames, th0 = scenario()
    bt = BatchTracker(b, intr, 2)
    with pytest.raises(W.ValidationError):
        bt.set_state(2, theta=th0[0])
    import ctypes as C
    lib = W.lib()
    d = np.ascontiguousarray(frames[0, 0])
    assert lib.wt_gpu_load_depth(bt._ctx, W.ptr(d), 1.0) == W.WT_EINVAL
    assert lib.wt_gpu_batch_size(bt._ctx) == 2
    with pytest.raises(W.LengthMismatch):
        bt.load_depth(frames[0, :1])
    with pytest.raises(W.ValidationError):
        bt.track_frame(cfg(kin=65), depth=frames[0, :2])  # > 64 recorded pose iterations
    bad = C.c_void_p()
    desc, keep = b.to_desc()
    assert lib.wt_gpu_create_batch(0, C.byref(desc), C.byref(intr.c()), 0, C.byref(bad)) == W.WT_EINVAL
    bt.close()


def test_batch_vga_equals_independent_sequences():
    """640x480 frames of the 25k-vertex humanoid, two sequences: the batched
    search's fp32 prefilter (k_search<true>, float4 bucket items) must pick
    exactly the exact search's winners -- theta, Phi and the statistics
    stay bitwise those of the lone sequences."""
    from .helpers import cfg as mkcfg, humanoid, intr640, theta_at
    b = humanoid(25000)
    intr = intr640()
    c = mkcfg("dynamic")
    th0 = np.stack([theta_at(b, 0), theta_at(b, 0, phase=0.7)])
    bt = BatchTracker(b, intr, 2, init_theta=th0)
    solo = [Tracker(b, intr, th0[s]) for s in range(2)]
    try:
        for f in range(1, 4):
            frames = np.stack([solo[s].render_depth(theta_at(b, f, phase=0.7 * s), frame=f)[0] for s in range(2)])
            bst = bt.track_frame(c, depth=frames)
            for s in range(2):
                st = solo[s].track_frame(c, depth=frames[s])
                th_b, ph_b = bt.get_state(s)
                th_s, ph_s, _ = solo[s].get_state()
                assert np.array_equal(th_b, th_s), (f, s)
                assert np.array_equal(ph_b, ph_s), (f, s)
                assert [k.associated for k in bst[s].kin] == [k.associated for k in st.kin]
    finally:
        bt.close()
        for t in solo:
            t.close()
