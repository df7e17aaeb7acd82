"""Experiment: per-kernel times of a C3 frame with the humanoid's vertices in
their subdivision order vs re-ordered along a Morton curve of the rest pose
(same mesh, same parity inputs; only the vertex numbering differs)."""
import ctypes as C
import sys

sys.path.insert(0, ".")
import numpy as np

from bench import make_workload, trajectory
from paper_1711_07999_b200 import _lib as W
from paper_1711_07999_b200.model import ModelBundle
from paper_1711_07999_b200.tracker import Tracker


def morton_order(v0):
    q = ((v0 - v0.min(0)) / (np.ptp(v0, 0).max() + 1e-12) * 1023).astype(np.uint64)

    def spread(x):
        x = (x | (x << 16)) & 0x030000FF
        x = (x | (x << 8)) & 0x0300F00F
        x = (x | (x << 4)) & 0x030C30C3
        x = (x | (x << 2)) & 0x09249249
        return x
    code = spread(q[:, 0]) | (spread(q[:, 1]) << 1) | (spread(q[:, 2]) << 2)
    return np.argsort(code, kind="stable")


def renumber(b: ModelBundle, order):
    inv = np.empty_like(order)
    inv[order] = np.arange(order.size)
    nb = b.copy()
    for k in ("v0", "phi", "weight_count", "weight_link", "weight"):
        setattr(nb, k, getattr(b, k)[order])
    nb.polys = [[int(inv[i]) for i in p] for p in b.polys]
    nb.finalize()
    nb.with_neighbors(4)
    return nb


def frame_times(bundle, intr, cfg):
    trk = Tracker(bundle, intr, trajectory(bundle, 0, 0))
    L = W.lib()
    ccfg = cfg.c()
    kinds, ms, n = (C.c_int32 * 512)(), (C.c_float * 512)(), C.c_int32()
    frames = [trk.render_depth(trajectory(bundle, f, 0), frame=f)[0] for f in range(6)]
    for f in range(1, 3):
        trk.track_frame(cfg, depth=frames[f])
    tot = {}
    for f in range(3, 6):
        trk.load_depth(frames[f])
        W.check(L.wt_gpu_profile_frame(trk._ctx, C.byref(ccfg), kinds, ms, 512, C.byref(n)), trk._ctx)
        for k in range(n.value):
            tot.setdefault(W.KERNEL_KINDS[kinds[k]], []).append(ms[k] * 1e3)
    return " ".join(f"{k}={np.mean(v):.1f}" for k, v in tot.items())


bundle, intr, cfg = make_workload("c3")
print("subdivision order:", frame_times(bundle, intr, cfg))
print("morton order:     ", frame_times(renumber(bundle, morton_order(bundle.v0)), intr, cfg))
