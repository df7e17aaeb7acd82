"""Per-warp phase timing of k_search inside tracked C3 frames (WT_DEBUG_SEARCH)."""
import ctypes as C
import os
import sys

os.environ["WT_DEBUG_SEARCH"] = "1"
sys.path.insert(0, ".")
import numpy as np

from bench import make_workload, trajectory
from paper_1711_07999_b200 import _lib as W
from paper_1711_07999_b200.tracker import Tracker

bundle, intr, cfg = make_workload("c3")
trk = Tracker(bundle, intr, trajectory(bundle, 0, 0))
L = W.lib()
L.wt_gpu_debug_search.argtypes = [C.c_void_p, C.c_void_p]
buf = np.zeros(8 * 4096, np.int64)
for f in range(1, 4):
    d, _ = trk.render_depth(trajectory(bundle, f, 0), frame=f)
    trk.track_frame(cfg, depth=d)
L.wt_gpu_debug_search(trk._ctx, buf.ctypes.data)
r = buf.reshape(4096, 8)
r = r[r[:, 7] == 1]
print("warps with work", len(r), "pixels", r[:, 6].sum(), "open", r[:, 4].sum(), "overflow", (r[:, 5] < 0).sum())
for k, nm in enumerate(["stage", "core scan", "emit", "phase2"]):
    print(f"{nm:10s} cycles: median {np.median(r[:, k]):8.0f}  p90 {np.percentile(r[:, k], 90):8.0f}  max {r[:, k].max():8.0f}")
print("staged items median", np.median(r[r[:, 5] >= 0, 5]))
