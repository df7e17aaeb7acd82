"""Robustness of the device path beyond the benchmark workload:

  * millimetre units: the reference sums in fp64 and tracks a model and depth
    given in millimetres exactly as in metres; the device's fixed-point sums
    pick their scales per frame / per call (wt_kernels.cuh, kObsExpBudget;
    wt_gpu.cu pose_scales) so nothing wraps -- checked against the reference
    on a millimetre-scaled copy of the same scene;
  * a stats buffer reallocation (an optimize_shape with more iterations than
    the stats buffer held) must invalidate EVERY cached frame graph, including
    the pinned-upload form of track_frame, or later frames report stale stats;
  * more than 64 iterations per call: the Python mirror sizes its stats arrays
    per call (the reference has no iteration cap).
"""
import ctypes as C

import numpy as np
import pytest

from oracle import ref
from paper_1711_07999_b200 import _lib as W
from paper_1711_07999_b200.tracker import Intrinsics, KinSolverConfig, ShapeSolverConfig, Tracker

from .helpers import cfg, humanoid, intr320, theta_at

pytestmark = pytest.mark.gpu


def scaled_bundle(b, k: float):
    """The same model with every length multiplied by k (template vertices,
    link offsets' translation parts, phi): a unit change, joint angles unchanged."""
    s = b.copy()
    s.v0 = b.v0 * k
    s.phi = None if b.phi is None else b.phi * k
    off = b.parent_offset.copy()
    off[:, 4:] *= k  # dual part = translation / 2 * real part: linear in the translation
    s.parent_offset = off
    return s


@pytest.mark.ref
def test_millimetre_scene_matches_reference():
    b = humanoid(7000)
    intr = intr320()
    mm = scaled_bundle(b, 1000.0)
    # prismatic root moves in metres in the base model: scale its trajectory too
    th = [theta_at(b, f) for f in range(4)]
    for t in th:
        t[0] *= 1000.0
    c = cfg("dynamic")
    c.assoc.cutoff = 100.0  # 0.10 m
    rm = ref.RefModel.from_bundle(mm)
    frames = [rm.render_depth(th[f], intr.c(), frame=f)[0] for f in range(1, 4)]
    assert frames[0].max() > 1000.0  # millimetre depth
    trk = Tracker(mm, intr, th[0])
    rt = ref.RefTracker(rm, th[0])
    try:
        worst = 0.0
        for d in frames:
            st = trk.track_frame(c, depth=d)
            rst = rt.track_frame_depth(intr.c(), d, c.c())
            assert [k.associated for k in st.kin] == [rst.kin[k].associated for k in range(rst.n_kin)]
            assert not any(k.solver_skipped for k in st.kin)
            gth, gph, _ = trk.get_state()
            rth, rph, _ = rt.get_state()
            dth = np.abs(gth[1:] - rth[1:]).max()  # hinge angles (rad)
            worst = max(worst, dth, np.abs(gth[0] - rth[0]) / 1000.0)
            assert dth <= 1e-6 and np.abs(gth[0] - rth[0]) <= 1e-3  # prismatic: mm
            assert np.abs(gph - rph).max() <= 1e-3                   # Phi: mm
        print(f"[robustness] millimetre scene: max dtheta {worst:.3g}")
    finally:
        trk.close()


def test_stats_reallocation_invalidates_pinned_graphs():
    import torch
    b = humanoid(7000)
    intr = intr320()
    c = cfg("dynamic")
    th0 = theta_at(b, 0)
    a, o = Tracker(b, intr, th0), Tracker(b, intr, th0)
    L = W.lib()
    try:
        frames = [a.render_depth(theta_at(b, f), frame=f)[0] for f in range(1, 4)]
        pinned = [torch.from_numpy(np.ascontiguousarray(d, dtype=np.float32)).pin_memory() for d in frames]

        def pinned_frame(f):
            sb = o._stats()
            W.check(L.wt_gpu_track_frame(o._ctx, pinned[f].data_ptr(), 1.0, C.byref(c.c()), C.byref(sb)), o._ctx)
            return [o._kin[k].residual_sum for k in range(sb.n_kin)], [o._shape[k].mean_phi for k in range(sb.n_shape)]

        for t in (a, o):
            t._ensure_stats(64, 64)
        sa = a.track_frame(c, depth=frames[0])
        ko, so = pinned_frame(0)  # captures the pinned-upload graph
        assert ko == [k.residual_sum for k in sa.kin]
        # grow the shape stats buffer (> 32 surface iterations) on both
        for t in (a, o):
            t.load_depth(frames[1])
            t.optimize_shape(ShapeSolverConfig(iterations=40))
        sa = a.track_frame(c, depth=frames[2])
        ko, so = pinned_frame(2)
        assert ko == [k.residual_sum for k in sa.kin]
        assert so == [s.mean_phi for s in sa.shape]
        assert np.array_equal(a.get_state()[0], o.get_state()[0])
    finally:
        a.close()
        o.close()


def test_more_than_64_iterations_per_call():
    b = humanoid(7000)
    intr = intr320()
    trk = Tracker(b, intr, theta_at(b, 0))
    try:
        d, _ = trk.render_depth(theta_at(b, 1), frame=1)
        c = cfg("dynamic", kin_its=70, shape_its=66)
        st = trk.track_frame(c, depth=d)
        assert len(st.kin) == 70 and len(st.shape) == 66
        assert [k.iteration for k in st.kin] == list(range(70))
        assert st.kin[-1].associated > 100
        ks = trk.optimize_pose(KinSolverConfig(iterations=80))
        assert len(ks) == 80
    finally:
        trk.close()
