"""wt_gpu_track_frame with a pinned host frame forks the upload and ingest
off inside the frame graph (wt_gpu.cu track_frame_overlapped) and joins them
before the first search. It must track exactly like load_depth +
track_loaded: theta, Phi and every per-iteration statistic bitwise, frame
after frame, with a different host buffer each frame (the graph's upload node
is re-pointed per launch)."""
import ctypes as C

import numpy as np
import pytest

from paper_1711_07999_b200 import _lib as W
from paper_1711_07999_b200.tracker import Tracker

from .helpers import cfg, humanoid, intr320, theta_at

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", ["dynamic", "smooth-bind"])
def test_pinned_track_frame_equals_loaded(mode):
    import torch
    b = humanoid(7000)
    intr = intr320()
    c = cfg(mode)
    th0 = theta_at(b, 0)
    a = Tracker(b, intr, th0)
    o = Tracker(b, intr, th0)
    L = W.lib()
    try:
        frames = [a.render_depth(theta_at(b, f), frame=f)[0] for f in range(1, 5)]
        pinned = [torch.from_numpy(np.ascontiguousarray(d, dtype=np.float32)).pin_memory() for d in frames]
        for f, d in enumerate(frames):
            st_a = a.track_frame(c, depth=d)
            sb = o._stats()
            W.check(L.wt_gpu_track_frame(o._ctx, pinned[f].data_ptr(), 1.0, C.byref(c.c()), C.byref(sb)), o._ctx)
            th_a, ph_a, fa = a.get_state()
            th_o = np.zeros(b.link_count)
            W.check(L.wt_gpu_get_state(o._ctx, th_o.ctypes.data, None, None), o._ctx)  # from the host mirror
            _, ph_o, fo = o.get_state()
            assert np.array_equal(th_a, th_o), f
            assert np.array_equal(ph_a, ph_o), f
            assert fa == fo == f + 1
            assert sb.n_kin == len(st_a.kin)
            for k in range(sb.n_kin):
                assert (o._kin[k].associated, o._kin[k].residual_sum, o._kin[k].step_norm) == \
                    (st_a.kin[k].associated, st_a.kin[k].residual_sum, st_a.kin[k].step_norm)
            for k in range(sb.n_shape):
                assert (o._shape[k].mean_phi, o._shape[k].max_phi) == (st_a.shape[k].mean_phi, st_a.shape[k].max_phi)
    finally:
        a.close()
        o.close()


def test_pinned_batch_track_equals_loaded():
    """wt_gpu_batch_track with pinned host frames (the [n][H][W] upload forked
    inside the batch frame graph, its 2D memcpy node re-pointed per call)
    tracks exactly like batch load_depth + track_async."""
    import torch
    from paper_1711_07999_b200.tracker import BatchTracker
    b = humanoid(7000)
    intr = intr320()
    c = cfg("dynamic")
    n = 3
    th0 = np.stack([theta_at(b, 0, phase=0.5 * s) for s in range(n)])
    ref_t = Tracker(b, intr, th0[0])
    a = BatchTracker(b, intr, n, init_theta=th0)
    o = BatchTracker(b, intr, n, init_theta=th0)
    L = W.lib()
    try:
        for f in range(1, 4):
            frames = np.stack([ref_t.render_depth(theta_at(b, f, phase=0.5 * s), frame=f)[0] for s in range(n)])
            pinned = torch.from_numpy(np.ascontiguousarray(frames, dtype=np.float32)).pin_memory()
            a.track_frame(c, depth=frames)
            stats = (W.FrameStatsC * n)(*[W.FrameStatsC(0, 0, 0, 64, 32, 0, o._kin[s], o._shape[s]) for s in range(n)])
            W.check(L.wt_gpu_batch_track(o._ctx, pinned.data_ptr(), 1.0, C.byref(c.c()), stats), o._ctx)
            for s in range(n):
                th_a, ph_a = a.get_state(s)
                th_o, ph_o = o.get_state(s)
                assert np.array_equal(th_a, th_o), (f, s)
                assert np.array_equal(ph_a, ph_o), (f, s)
                assert stats[s].n_kin == c.kin.iterations
    finally:
        ref_t.close()
        a.close()
        o.close()
