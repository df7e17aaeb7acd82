"""Per-kernel in-graph times (events between kernels) of a few C3 frames."""
import ctypes as C
import sys

sys.path.insert(0, ".")
import numpy as np

from bench import make_workload, trajectory
from paper_1711_07999_b200 import _lib as W
from paper_1711_07999_b200.tracker import Tracker

bundle, intr, cfg = make_workload("c3")
trk = Tracker(bundle, intr, trajectory(bundle, 0, 0))
L = W.lib()
ccfg = cfg.c()
kinds = (C.c_int32 * 512)()
ms = (C.c_float * 512)()
n = C.c_int32()
frames = [trk.render_depth(trajectory(bundle, f, 0), frame=f)[0] for f in range(6)]
for f in range(1, 3):
    trk.track_frame(cfg, depth=frames[f])
tot = {}
for f in range(3, 6):
    trk.load_depth(frames[f])
    W.check(L.wt_gpu_profile_frame(trk._ctx, C.byref(ccfg), kinds, ms, 512, C.byref(n)), trk._ctx)
    for k in range(n.value):
        nm = W.KERNEL_KINDS[kinds[k]]
        tot.setdefault(nm, []).append(ms[k] * 1e3)
print(" ".join(f"{k}={np.mean(v):.1f}" for k, v in tot.items()))
